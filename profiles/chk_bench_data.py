import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import bench, bench_outer as B
from oracle import ssm_oracle as O
T = 40
t, ot, ov, om = bench.synthetic_data(T)
ov2, om2 = bench._cpu_data(T)[2:]
print("bench data equal", np.array_equal(ov, ov2), np.array_equal(om, om2))
th, times, ov, om = B.l96_sparse(40)
obs = O.simulate_l96(th, times, O.Stream(1), obs_slots=range(4), obs_every=2)
print("sparse equal", np.array_equal(ov, np.array([obs[k][0] for k in range(1, 41)])), np.array_equal(om, np.array([obs[k][1] for k in range(1, 41)])))
theta, times, obs, inputs = B.wk_data()
rng = O.Stream(1)
x = np.array([[rng.child(1).normal(90.0, 15.0)]])
ref = []
for k in range(1, 101):
    rk = rng.child(2, k)
    x, _ = O.wk_transition(theta, x, times[k - 1], times[k] - times[k - 1],
                           lambda kk, sd, rk=rk: rk.normal(0.0, np.array([sd]), size=1), inputs.at)
    F = float(inputs.at(times[k])[0])
    ref.append([rng.child(3, k).normal(x[0, 0] + theta[2] * F, 2.0)])
print("wk equal", np.array_equal(obs, np.array(ref)), np.abs(obs - np.array(ref)).max())
print("flow equal", np.array_equal(B.flow(np.round(np.arange(0, 1 + 1e-9, 0.01), 10)), O.windkessel_flow(np.round(np.arange(0, 1 + 1e-9, 0.01), 10))))
