"""paper_1306_3277_b200: the B200-native (sm_100a) bootstrap particle filter
of LibBi (arXiv 1306.3277), behind the reference `ssmkit` API.

Host code is Python/PyTorch (device memory, streams); every per-particle
operation runs in the hand-written CUDA kernels of lib/libssm_b200.so,
bound through the C ABI declared in include/ssm_b200.h.
"""

from .models import LORENZ96, WINDKESSEL, ModelSpec, load_model, resolve_model
from .rng import RngStream

__version__ = "0.1.0"

__all__ = ["RngStream", "ModelSpec", "LORENZ96", "WINDKESSEL", "load_model", "resolve_model",
           "__version__"]
