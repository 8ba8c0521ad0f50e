"""The benchmark inputs (bench.py / bench_outer.py) are simulated with this
package's own simulate API on the device; with the reference's draws they are
bitwise the data the reference's simulator makes (restated by the oracle)."""

import numpy as np
import pytest

import bench
import bench_outer as B
from oracle import ssm_oracle as O

pytestmark = pytest.mark.gpu


def test_l96_bench_data_bitwise_reference():
    _, ot, ov, om = bench.synthetic_data(40)
    _, ot2, ov2, om2 = bench._cpu_data(40)
    np.testing.assert_array_equal(ot, ot2)
    np.testing.assert_array_equal(ov, ov2)
    np.testing.assert_array_equal(om, om2)


def test_l96_sparse_data_bitwise_reference():
    th, times, ov, om = B.l96_sparse(40)
    obs = O.simulate_l96(th, times, O.Stream(1), obs_slots=range(4), obs_every=2)
    np.testing.assert_array_equal(ov, np.array([obs[k][0] for k in range(1, 41)]))
    np.testing.assert_array_equal(om, np.array([obs[k][1] for k in range(1, 41)]))


def test_windkessel_bench_data_bitwise_reference():
    theta, times, obs, inputs = B.wk_data()
    in_times = np.round(np.arange(0, 1 + 1e-9, 0.01), 10)
    np.testing.assert_array_equal(B.flow(in_times), O.windkessel_flow(in_times))
    rng = O.Stream(1)
    x = np.array([[rng.child(1).normal(90.0, 15.0)]])
    ref = []
    for k in range(1, 101):
        rk = rng.child(2, k)
        x, _ = O.wk_transition(theta, x, times[k - 1], times[k] - times[k - 1],
                               lambda kk, sd, rk=rk: rk.normal(0.0, np.array([sd]), size=1), inputs.at)
        ref.append([rng.child(3, k).normal(x[0, 0] + theta[2] * float(inputs.at(times[k])[0]), 2.0)])
    np.testing.assert_array_equal(obs, np.array(ref))
