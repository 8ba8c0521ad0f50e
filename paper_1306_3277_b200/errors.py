"""Exception classes with the reference's names and constructor contract
(errors.py:1-84 of the reference), raised by the host layer when the device
reports the corresponding condition."""


class SsmError(Exception):
    """Base class for all engine errors."""


class DistributionParameterError(SsmError):
    """Invalid distribution parameter at evaluation time (distributions.py:55-57)."""


class NonFiniteStateError(SsmError):
    """A state variable became NaN or infinite (simulate.py:158-162)."""

    def __init__(self, message, time=None):
        self.time = time
        super().__init__(message)


class DegenerateEnsembleError(SsmError):
    """All particle weights vanished at some time step (particle.py:128-131)."""

    def __init__(self, message, time=None):
        self.time = time
        super().__init__(message)


class UnsupportedModelError(SsmError):
    """The model has no hand-written sm_100a kernel (no CPU fallback exists)."""


class MissingInputError(SsmError):
    """A required input value is not available at the requested time."""


class DataFormatError(SsmError):
    """Malformed or schema-inconsistent data."""


class NonlinearModelError(SsmError):
    """The model is not linear-Gaussian, so the Kalman filter does not apply
    (lineargauss.py:1-12)."""


class CholeskyError(SsmError):
    """A covariance is not positive (semi-)definite (linalg.py:21-50)."""

    def __init__(self, message, index=None):
        self.index = index
        super().__init__(message)
