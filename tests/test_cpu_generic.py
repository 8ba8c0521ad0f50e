"""Generic-model path on the CPU: the lowering of the
reference IR is pinned against the reference's own expression sources
(tests/golden/gen_models.json, written by make_golden.py from the reference),
the generated CUDA compiles with NVRTC for sm_100a (no device needed), the
hand-written kernels are chosen exactly for the two reference models, and
the host-side initial draws equal the reference's."""

import json
import os

import numpy as np
import pytest

from tests.conftest import GOLDEN, load_golden
from paper_1306_3277_b200 import codegen, generic, models
from paper_1306_3277_b200.rng import RngStream

with open(os.path.join(GOLDEN, "gen_models.json")) as fh:
    FIX = json.load(fh)
NAMES = ["Lorenz96", "Windkessel", "StochVol", "PredatorPrey", "Wide"]


def _desc(name):
    d = dict(FIX["lowered"][name])
    d.pop("fingerprint", None)
    return d


def _exprs(desc):
    """Every lowered expression in the order make_golden.py lists the reference's."""
    out = []
    for bn in ("initial", "transition", "observation"):
        for op in desc[bn]:
            if op["op"] == "sample":
                out += [a for row in op["args"] for a in row]
            else:
                out += op["exprs"]
    return out


@pytest.mark.parametrize("name", NAMES)
def test_lowering_prints_the_reference_sources(name):
    got = [codegen.numpy_source(e) for e in _exprs(_desc(name))]
    assert got == FIX["reference_sources"][name]


@pytest.mark.parametrize("name", NAMES)
def test_generated_source_compiles_for_sm100a(name):
    m = generic.from_description(_desc(name))
    m.check_compiles()
    src = m.source
    assert "struct Model" in src and f"NX = {m.n_state}" in src
    assert m.digest == codegen.source_digest(codegen.cuda_source(_desc(name)))


def test_hand_written_fingerprints_pin_the_reference_models():
    assert models._FINGERPRINTS["lorenz96"] == FIX["lowered"]["Lorenz96"]["fingerprint"]
    assert models._FINGERPRINTS["windkessel"] == FIX["lowered"]["Windkessel"]["fingerprint"]


def test_resolve_model_generic_descriptions():
    m = models.resolve_model(_desc("StochVol"))
    assert isinstance(m, generic.GenericModel)
    assert models.resolve_model(_desc("StochVol")) is m  # one compile per model
    assert m.kernel == 2 and m.nx == 1 and m.theta_stride == 3
    assert m.draw_kinds == ["gaussian"]
    pp = models.resolve_model(_desc("PredatorPrey"))
    assert pp.draw_kinds == ["wiener", "wiener", "uniform"]
    np.testing.assert_array_equal(pp.derived([1.0, 2.0, 3.0]), [[1.0, 2.0, 3.0]])


@pytest.mark.parametrize("name", ["StochVol", "PredatorPrey"])
def test_host_initial_block_equals_reference_draws(name):
    g = load_golden("generic.npz")
    m = generic.from_description(_desc(name))
    x0 = m.host_initial(RngStream(5).child(0), 300, g[f"{name}/theta"])
    np.testing.assert_array_equal(x0, g[f"{name}/x0"])


def test_codegen_limits_and_unsupported_statements():
    d = _desc("StochVol")
    big = json.loads(json.dumps(d))
    big["transition"][0]["kind"] = "gamma"
    m = generic.GenericModel(big)
    with pytest.raises(models.UnsupportedModelError):
        m.check_host_noise()  # gamma transition noise: device draws only
    bad = json.loads(json.dumps(d))
    bad["observation"][0]["kind"] = "wiener"
    with pytest.raises(models.UnsupportedModelError):
        codegen.cuda_source(bad)


@pytest.mark.parametrize("name", ["StochVol", "PredatorPrey"])
def test_theta_level_blocks_equal_reference(name):
    """Prior draws / densities and the parameter proposal (with its fallback to
    the prior when the model has no proposal_parameter block) on the host,
    bitwise the reference's (simulate.py:96-108, 219-352)."""
    g = load_golden("generic.npz")
    m = generic.from_description(_desc(name))
    th = m.sample_parameter(RngStream(3), size=5)
    np.testing.assert_array_equal(th, g[f"{name}/prior_draws"])
    np.testing.assert_array_equal([m.parameter_logpdf(t) for t in th], g[f"{name}/prior_logpdf"])
    props = [m.propose_parameters(t, RngStream(4).child(k)) for k, t in enumerate(th)]
    np.testing.assert_array_equal([p[0] for p in props], g[f"{name}/prop"])
    np.testing.assert_array_equal([p[1] for p in props], g[f"{name}/prop_logq"])
    np.testing.assert_array_equal([m.proposal_parameter_logpdf(p[0], t) for p, t in zip(props, th)],
                                  g[f"{name}/prop_rev"])
    assert m.has_proposal_initial is False
    assert (m.block("proposal_parameter") is not None) == (name == "PredatorPrey")
