"""Posterior runs of the device samplers written as samples files (SURVEY 8f
row 4, runner.py:84-146 + sampleio.py:39-68) against the files the
REFERENCE's own `sample` driver wrote for the same configuration
(tests/golden/io, make_io_golden.py), with the reference's draws (noise="host",
host theta-level draws): every line is byte-identical except the
log-likelihood column (and SMC^2's weights, exp of normalised log-likelihood
increments), which the device accumulates in a different (fixed-point tile)
order -- those agree to 1e-12 relative (-m gpu)."""

import os

import numpy as np
import pytest

from paper_1306_3277_b200 import LORENZ96, WINDKESSEL, RngStream
from paper_1306_3277_b200.inference import FilterRunner, build_filter_grid
from paper_1306_3277_b200.sampleio import posterior_output, read_run_output, write_run_output
from paper_1306_3277_b200.timeseries import InputProvider, read_timeseries, role_arrays
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu
IO = os.path.join(GOLDEN, "io")


def _compare(got_path, ref_path, float_cols):
    got = open(got_path).read().splitlines()
    ref = open(ref_path).read().splitlines()
    assert len(got) == len(ref)
    section = None
    for a, b in zip(got, ref):
        if a.startswith("["):
            section = a
        if a == b:
            continue
        assert section == "[parameters]", (a, b)
        fa, fb = a.split(","), b.split(",")
        for k, (x, y) in enumerate(zip(fa, fb)):
            if k in float_cols:
                assert abs(float(x) - float(y)) <= 1e-12 * max(abs(float(y)), 1e-300), (k, x, y)
            else:
                assert x == y, (k, a, b)


def _grid(model, obs_file, start, end, noutputs):
    t, v, m = role_arrays(read_timeseries(obs_file, model, roles=("obs",)), model, "obs")
    return build_filter_grid(start, end, noutputs, obs_times=t, obs_values=v, obs_mask=m, n_obs=model.n_obs)


def test_l96_pmmh_samples_file_matches_reference(tmp_path):
    ref_path = os.path.join(IO, "l96_mh_samples.txt")
    ref = read_run_output(ref_path)
    grid = _grid(LORENZ96, os.path.join(IO, "l96_obs.csv"), 0.0, 1.0, 10)
    runner = FilterRunner(LORENZ96, grid, n_particles=128, resampler="systematic", noise="host")
    out = posterior_output(LORENZ96, runner, "mh", 6, RngStream(31), metadata=ref.metadata)
    p = tmp_path / "samples.txt"
    write_run_output(p, out)
    _compare(p, ref_path, float_cols={2})  # loglik


def test_windkessel_smc2_samples_file_matches_reference(tmp_path):
    ref_path = os.path.join(IO, "wk_smc_samples.txt")
    ref = read_run_output(ref_path)
    inputs = InputProvider(WINDKESSEL, read_timeseries(os.path.join(IO, "wk_input.csv"), WINDKESSEL, ("input",)))
    grid = _grid(WINDKESSEL, os.path.join(IO, "wk_obs.csv"), 0.0, 0.4, 20)
    runner = FilterRunner(WINDKESSEL, grid, inputs=inputs, n_particles=256, resampler="systematic", noise="host")
    out = posterior_output(WINDKESSEL, runner, "smc2", 8, RngStream(32), metadata=ref.metadata)
    p = tmp_path / "samples.txt"
    write_run_output(p, out)
    _compare(p, ref_path, float_cols={1, 2})  # weight, loglik
    got = read_run_output(p)
    assert np.allclose([r.weight for r in got.records], [r.weight for r in ref.records], rtol=1e-10, atol=0)
