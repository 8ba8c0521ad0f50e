"""Host side of the device Kalman filter: the linear-Gaussian
extraction against the reference's own extracted systems (tests/golden/kalman.npz,
made by make_golden.gen_kalman from lineargauss.extract_linear_gaussian)."""

import json
import os

import numpy as np
import pytest

from paper_1306_3277_b200 import LORENZ96, WINDKESSEL
from paper_1306_3277_b200.errors import CholeskyError, NonlinearModelError
from paper_1306_3277_b200.inference.kalman import psd_cholesky_upper
from paper_1306_3277_b200.lineargauss import extract_linear_gaussian
from tests.conftest import LocfInputs, load_golden

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIELDS = ("A", "b", "Q", "H", "c", "r_sd")


def _lowered(name):
    with open(os.path.join(ROOT, "tests", "golden", "gen_models.json")) as fh:
        d = dict(json.load(fh)["lowered"][name])
    d.pop("fingerprint", None)
    return d


def _flow(t, f_max=500.0, t_s=0.3, t_d=0.5):
    tp = np.mod(t, t_s + t_d)
    return np.where(tp < t_s, f_max * np.sin(np.pi * tp / t_s) ** 2, 0.0)


def _check(sys_, g, tag, n):
    for j in range(n):
        np.testing.assert_array_equal(sys_.mu0[j], g[f"{tag}/{j}/mu0"])
        np.testing.assert_allclose(sys_.P0[j], g[f"{tag}/{j}/P0"], rtol=1e-15, atol=1e-18)
        for f in FIELDS:
            np.testing.assert_allclose(getattr(sys_, f)[j], g[f"{tag}/{j}/{f}"], rtol=1e-14, atol=1e-18,
                                       err_msg=f"{tag} {j} {f}")


@pytest.mark.parametrize("src", ["builtin", "lowered"])
def test_windkessel_system_matches_reference(src):
    g = load_golden("kalman.npz")
    in_times = np.round(np.arange(0, 1.0001, 0.01), 10)
    model = WINDKESSEL if src == "builtin" else _lowered("Windkessel")
    sys_ = extract_linear_gaussian(model, g["wk/thetas"], g["wk/times"], LocfInputs(in_times, _flow(in_times)))
    _check(sys_, g, "wk", 2)


def test_linosc_system_matches_reference():
    g = load_golden("kalman.npz")
    d = json.loads(str(g["osc/desc"]))
    sys_ = extract_linear_gaussian(d, g["osc/thetas"], g["osc/times"],
                                   LocfInputs(g["osc/in_times"], g["osc/in_values"]))
    _check(sys_, g, "osc", 3)


def test_wide_system_matches_reference():
    g = load_golden("kalman.npz")
    gg = load_golden("generic.npz")
    sys_ = extract_linear_gaussian(_lowered("Wide"), g["wide/thetas"], np.linspace(0.0, 2.0, 21),
                                   LocfInputs(gg["Wide/in_times"], gg["Wide/in_values"]))
    _check(sys_, g, "wide", 2)


@pytest.mark.parametrize("name", ["Lorenz96", "StochVol", "PredatorPrey"])
def test_nonlinear_models_rejected(name):
    with pytest.raises(NonlinearModelError):
        extract_linear_gaussian(_lowered(name), np.array([[1.0, 0.1, 0.1]])[:, : len(_lowered(name)["parameter"])],
                                np.linspace(0, 1, 3))
    if name == "Lorenz96":
        with pytest.raises(NonlinearModelError):
            extract_linear_gaussian(LORENZ96, np.array([[10.0, 0.1]]), np.linspace(0, 1, 3))


def test_psd_cholesky():
    rs = np.random.default_rng(0)
    M = rs.normal(size=(5, 3))
    S = M @ M.T  # rank 3
    U = psd_cholesky_upper(S)
    np.testing.assert_allclose(U.T @ U, S, atol=1e-12)
    assert np.allclose(np.tril(U, -1), 0)
    np.testing.assert_array_equal(psd_cholesky_upper(np.zeros((3, 3))), np.zeros((3, 3)))
    with pytest.raises(CholeskyError):
        psd_cholesky_upper(np.diag([1.0, -1.0]))
