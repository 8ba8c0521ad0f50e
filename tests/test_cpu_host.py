"""CPU-only tests: the C-ABI library loads and exports every symbol the
header declares; host-side logic (theta-level blocks, grids, derived kernel
constants, schedules) matches the reference's golden vectors / the oracle."""

import os
import re

import numpy as np
import pytest

from oracle import ssm_oracle as O
from paper_1306_3277_b200 import LORENZ96, WINDKESSEL, RngStream, _lib, load_model, resolve_model
from paper_1306_3277_b200.errors import DataFormatError, UnsupportedModelError
from paper_1306_3277_b200.inference import build_filter_grid
from paper_1306_3277_b200.rng import device_key
from tests.conftest import ROOT, load_golden

HEADER = os.path.join(ROOT, "include", "ssm_b200.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int|size_t)\s+(ssm_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.load_library()
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.SIGNATURES, f"{n} has no ctypes signature"
    assert lib.ssm_version().decode().startswith("ssm_b200")


def test_library_is_sm100a():
    so = _lib.LIB_PATH
    out = os.popen(f"cuobjdump --list-elf {so} 2>&1").read()
    assert "sm_100a" in out


def test_struct_layouts_match_header(tmp_path):
    """ABI check: compile the header with gcc and compare sizeof/offsetof of
    every struct with the ctypes mirrors in _lib."""
    import ctypes as C
    import subprocess

    structs = {"ssm_pw_args": _lib.PwArgs, "ssm_substep": _lib.Substep, "ssm_step_desc": _lib.StepDesc,
               "ssm_advance_args": _lib.AdvanceArgs, "ssm_small_args": _lib.SmallArgs,
               "ssm_replay_args": _lib.ReplayArgs, "ssm_theta_args": _lib.ThetaArgs,
               "ssm_kalman_args": _lib.KalmanArgs}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "ssm_b200.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'  printf("{name} %zu\\n", sizeof({name}));')
        for fname, _ in cls._fields_:
            lines.append(f'  printf("{name}.{fname} %zu\\n", offsetof({name}, {fname}));')
    lines.append('  printf("ssm_filter_state %zu\\n", sizeof(ssm_filter_state));')
    lines.append('  printf("ssm_tile_rec %zu\\n", sizeof(ssm_tile_rec));')
    lines.append("  return 0; }")
    src = tmp_path / "abi.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "abi"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines())
    for name, cls in structs.items():
        assert int(got[name]) == C.sizeof(cls), name
        for fname, _ in cls._fields_:
            assert int(got[f"{name}.{fname}"]) == getattr(cls, fname).offset, (name, fname)
    assert int(got["ssm_filter_state"]) == _lib.FILTER_STATE_DTYPE.itemsize
    assert int(got["ssm_tile_rec"]) == 16
    assert int(got["ssm_step_desc"]) == _lib.STEP_DESC_DTYPE.itemsize


def test_status_strings_no_device_needed():
    lib = _lib.load_library()
    assert lib.ssm_status_string(0) == b"ok"
    assert lib.ssm_status_string(1) == b"invalid argument"
    assert lib.ssm_pw_workspace_bytes(2, 1024) > 0
    assert lib.ssm_scan_workspace_bytes(1, 1 << 20) > 0


def test_invalid_args_rejected_without_device():
    lib = _lib.load_library()
    assert lib.ssm_propagate_weight(None, None) == _lib.SSM_ERR_INVALID_ARG
    assert lib.ssm_gather(1, 0, 8, 16, None, None, None, None) == _lib.SSM_ERR_INVALID_ARG
    assert lib.ssm_resample_search(1, 4, 4, 9, 0, None, None, None, 0, None, None, None, None) == _lib.SSM_ERR_INVALID_ARG
    a = _lib.ThetaArgs()
    a.model, a.n_chains, a.n_param, a.nx = _lib.SSM_MODEL_WINDKESSEL, 4, 4, 1
    assert lib.ssm_theta_propose(a, None) == _lib.SSM_ERR_INVALID_ARG  # no keys, no injected draws
    a.model = _lib.SSM_MODEL_GENERIC
    assert lib.ssm_theta_propose(a, None) == _lib.SSM_ERR_UNSUPPORTED
    assert lib.ssm_theta_draws(_lib.SSM_MODEL_LORENZ96, 1) == 1 + 8 + 2 + 1
    assert lib.ssm_theta_draws(_lib.SSM_MODEL_GENERIC, 1) == -1
    assert lib.ssm_gen_theta_propose(None, a, None) == _lib.SSM_ERR_INVALID_ARG
    assert lib.ssm_gen_theta_draws(None, 0) == -1


def test_generic_theta_blocks_generated():
    """Generic models carry device theta-level blocks (codegen `struct Theta`):
    one draw per sampled slot of the proposal walk (or the prior when the
    proposal is absent); a statement the walk cannot sample gives stubs and
    DeviceThetaChains refuses the model before touching a device."""
    import copy
    import json

    from paper_1306_3277_b200 import codegen, generic
    from paper_1306_3277_b200.errors import UnsupportedModelError
    from paper_1306_3277_b200.inference.theta_mh import DeviceThetaChains

    with open(os.path.join(ROOT, "tests", "golden", "gen_models.json")) as fh:
        low = json.load(fh)["lowered"]
    want = {"Lorenz96": ((2, 8), ("proposal_parameter", "proposal_initial")),
            "PredatorPrey": ((3, 2), ("proposal_parameter", "initial")),
            "StochVol": ((3, 1), ("parameter", "initial"))}
    for name, (counts, blocks) in want.items():
        d = dict(low[name])
        d.pop("fingerprint", None)
        assert codegen.theta_draw_counts(d) == counts
        assert codegen.theta_walk_blocks(d) == blocks
        assert codegen.theta_supported(d)
        src = codegen.cuda_source(d)
        assert "struct Theta" in src and "th_sample_" in src
    d = copy.deepcopy(dict(low["StochVol"]))
    d.pop("fingerprint", None)
    d["parameter"][0]["kind"] = "wiener"
    assert not codegen.theta_supported(d)
    assert "perr = true; }" in codegen.cuda_source(d)
    with pytest.raises(UnsupportedModelError):
        DeviceThetaChains(generic.from_description(d), [])


def test_resolve_model():
    assert resolve_model("lorenz96") is LORENZ96
    assert load_model("/x/y/Windkessel.bi") is WINDKESSEL
    with pytest.raises(UnsupportedModelError):
        resolve_model("SIR")


@pytest.mark.parametrize("name,spec", [("lorenz96", LORENZ96), ("windkessel", WINDKESSEL)])
def test_theta_level_blocks_match_reference(name, spec):
    g = load_golden("theta.npz")
    th = spec.sample_parameter(RngStream(3), size=5)
    np.testing.assert_array_equal(th, g[f"{name}/prior_draws"])
    np.testing.assert_array_equal([spec.parameter_logpdf(t) for t in th], g[f"{name}/prior_logpdf"])
    for k, t in enumerate(th):
        tn, lq = spec.propose_parameters(t, RngStream(4, (k,)))
        np.testing.assert_array_equal(tn, g[f"{name}/proposals"][k])
        assert lq == g[f"{name}/logq_fwd"][k]
        assert spec.proposal_parameter_logpdf(tn, t) == g[f"{name}/logq_rev"][k]
    if spec.has_proposal_initial:
        x0 = spec.sample_initial(th, RngStream(5), size=5)
        np.testing.assert_array_equal(x0, g[f"{name}/init_draws"])
        for k in range(5):
            assert spec.initial_logpdf(th[k], x0[k]) == g[f"{name}/init_logpdf"][k]
            xp, lq = spec.propose_initial(th[k], x0[k], RngStream(6, (k,)))
            np.testing.assert_array_equal(xp, g[f"{name}/init_props"][k])
            assert lq == g[f"{name}/init_logq"][k]
            assert spec.proposal_initial_logpdf(th[k], xp, x0[k]) == g[f"{name}/init_logq_rev"][k]


def test_windkessel_derived_constants_bitwise():
    for theta in ([1.8, 3.0, 0.06, 25.0], [0.9, 1.5, 0.03, 10.0]):
        d = WINDKESSEL.derived(theta)[0]
        a, b = O.wk_coeffs(theta)
        assert d[0] == a and d[1] == b
        assert d[3] == 0.01 * np.sqrt(np.array([theta[3]]))[0]
    d = LORENZ96.derived([10.0, 0.1])[0]
    assert d[0] == 10.0 and d[1] == np.sqrt(0.1)


def test_filter_grid_matches_reference():
    g = load_golden("pf.npz")
    grid = build_filter_grid(0.0, 2.0, 20, g["l96/obs_t"], g["l96/obs_v"], g["l96/obs_m"], n_obs=8)
    np.testing.assert_array_equal(grid.times, g["l96/times"])
    assert grid.obs_steps == list(range(1, 21))


def test_device_key_is_seedsequence_hash():
    k1 = device_key(RngStream(7, (1,)))
    k2 = device_key(RngStream(7, (2,)))
    assert k1.dtype == np.uint32 and k1.shape == (2,)
    assert not np.array_equal(k1, k2)
    np.testing.assert_array_equal(k1, device_key(RngStream(7).child(1)))


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1306_3277_b200")
    pat = re.compile(r"^\s*(from|import)\s+\S*oracle", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                assert not pat.search(open(os.path.join(dirpath, f)).read()), f


def test_batched_streams_bit_exact_with_numpy():
    """rng.device_keys / first_uniforms / prime_streams restate numpy's
    SeedSequence + Philox4x64-10 vectorised; every draw must equal numpy's
    (including continuation draws of the same stream afterwards)."""
    from paper_1306_3277_b200.rng import RngStream, device_key, device_keys, first_uniforms, prime_streams

    def ref_gen(seed, key):
        return np.random.Generator(np.random.Philox(np.random.SeedSequence(entropy=seed, spawn_key=key)))

    r = np.random.default_rng(0)
    cases = []
    for i in range(120):
        seed = int(r.integers(0, 2**63)) if i % 4 == 0 else int(r.integers(0, 1000))
        key = tuple(int(x) for x in r.integers(0, 2**40 if i % 5 == 0 else 100, size=int(r.integers(0, 6))))
        cases.append((seed, key))
    streams = [RngStream(s, k) for s, k in cases]
    assert (device_keys(streams) == np.stack([device_key(x) for x in streams])).all()
    for n in (1, 4, 6):
        streams = [RngStream(s, k) for s, k in cases]
        got = first_uniforms(streams, n)
        gens = [ref_gen(s, k) for s, k in cases]
        assert (got == np.stack([g.uniform(size=n) for g in gens])).all()
        for st, g in list(zip(streams, gens))[:30]:
            assert st.gamma(2.0, 0.3, size=1).tolist() == g.gamma(2.0, 0.3, size=1).tolist()
            assert st.uniform(size=3).tolist() == g.uniform(size=3).tolist()
            assert st.normal(1.0, 2.0) == g.normal(1.0, 2.0)
    streams = [RngStream(s, k) for s, k in cases]
    prime_streams(streams)
    assert all(st._state is not None for st in streams)
    for st, (s, k) in zip(streams, cases):
        g = ref_gen(s, k)
        assert st.uniform() == g.uniform()
        assert st.generator.uniform(size=2).tolist() == g.uniform(size=2).tolist()


def test_batched_chain_log_priors_equal_per_chain():
    """SMC^2's batched prior evaluation (_chain_log_priors) gives bitwise the
    per-chain _chain_log_prior values (mcmc.py:118-132 / simulate.parameter_logpdf),
    including out-of-support parameters and initial states (-inf)."""
    from paper_1306_3277_b200 import LORENZ96, WINDKESSEL
    from paper_1306_3277_b200.inference.mcmc import _chain_log_prior, _chain_log_priors

    rs = np.random.default_rng(3)
    th = np.column_stack([rs.uniform(7.0, 13.0, 50), rs.uniform(-0.1, 1.0, 50)])
    x0 = rs.uniform(-1.5, 3.5, (50, 8))
    for init in (None, x0):
        got = _chain_log_priors(LORENZ96, list(th), None if init is None else list(init))
        want = [_chain_log_prior(LORENZ96, th[k], None if init is None else init[k]) for k in range(50)]
        assert [float(v).hex() for v in got] == [float(v).hex() for v in want]
    thw = np.abs(rs.normal(1.0, 1.0, (40, 4))) * np.array([1.0, 1.0, 0.03, 20.0])
    thw[3, 1] = -1.0
    xw = rs.normal(90.0, 20.0, (40, 1))
    for init in (None, xw):
        got = _chain_log_priors(WINDKESSEL, list(thw), None if init is None else list(init))
        want = [_chain_log_prior(WINDKESSEL, thw[k], None if init is None else init[k]) for k in range(40)]
        assert [float(v).hex() for v in got] == [float(v).hex() for v in want]


def _grid_by_event_loop(start, end, n_out, t_obs, n_obs_slots, mask):
    """Restatement of the reference's grid merge (inference/timegrid.py:53-97) as a
    plain event loop: outputs before observations at equal times, each event folded
    into the previous grid point when within the relative 1e-9 tolerance."""
    def close(a, b):
        return abs(a - b) <= 1e-9 * max(1.0, abs(a), abs(b))

    outs = np.linspace(start, end, n_out + 1)
    keep = [k for k, t in enumerate(t_obs) if t > start and not close(t, start) and (t < end or close(t, end))]
    t_obs, mask = [t_obs[k] for k in keep], mask[keep]
    ev = sorted([(t, 0, -1) for t in outs] + [(t, 1, r) for r, t in enumerate(t_obs)], key=lambda e: e[0])
    times, is_out, rows = [], [], []
    for t, kind, r in ev:
        if times and close(times[-1], t):
            is_out[-1] |= kind == 0
            rows[-1] = r if r >= 0 else rows[-1]
            continue
        times.append(t)
        is_out.append(kind == 0)
        rows.append(r)
    steps = [i for i in range(1, len(times)) if rows[i] >= 0 and mask[rows[i]].any()]
    return np.array(times), np.array(is_out), np.array(rows), steps


def test_filter_grid_merge_rules():
    """build_filter_grid against the event-loop restatement on random grids with
    observation times on, within 1e-12 / 3e-9 of, and outside the output times and
    the (start, end] boundaries, and rows with no present slot."""
    rs = np.random.default_rng(11)
    for trial in range(400):
        start = float(rs.choice([0.0, 1.5, -2.0]))
        end = start + float(rs.uniform(0.5, 10.0))
        n_out = int(rs.integers(1, 25))
        outs = np.linspace(start, end, n_out + 1)
        t = rs.uniform(start - 1.0, end + 1.0, int(rs.integers(0, 30)))
        if t.size:
            j = rs.integers(0, t.size, size=min(t.size, 6))
            t[j] = outs[rs.integers(0, n_out + 1, size=j.size)] * (1.0 + rs.choice([0.0, 1e-12, -1e-12, 3e-9], j.size))
        t = np.unique(t)
        nslot = int(rs.integers(1, 4))
        mask = rs.random((t.size, nslot)) < 0.5
        vals = rs.normal(size=(t.size, nslot))
        grid = build_filter_grid(start, end, n_out, t, vals, mask, n_obs=nslot)
        times, is_out, rows, steps = _grid_by_event_loop(start, end, n_out, list(t), nslot, mask)
        np.testing.assert_array_equal(grid.times, times)
        np.testing.assert_array_equal(grid.is_output, is_out)
        np.testing.assert_array_equal(grid.obs_row, rows)
        assert grid.obs_steps == steps
    with pytest.raises(DataFormatError):
        build_filter_grid(0.0, 1.0, 4, [0.5, 0.5], np.zeros((2, 1)), np.ones((2, 1), bool), n_obs=1)
    with pytest.raises(DataFormatError):
        build_filter_grid(1.0, 1.0, 4)
