"""Generate the data-file fixtures (tests/golden/io/) by running the REFERENCE.

Run in this container only:  python tests/golden/make_io_golden.py

  wk_input.csv / wk_obs.csv   windkessel flow input and observations, written
                              by the reference's write_timeseries (one masked
                              observation cell);
  wk_input_at.npz             the reference InputProvider.at(t) on a time grid
                              (LOCF lookups at, between and before the rows);
  l96_obs.csv                 sparse L96 observations (masked cells);
  l96_mh_samples.txt          `sample --target posterior --sampler mh` on L96
                              (runner.run_sample: 6 samples, 128 particles,
                              systematic, 11 output times over 20 grid steps);
  wk_smc_samples.txt          the same with the SMC^2 sampler on the
                              windkessel (inf shim of SURVEY 8c applied).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as M  # noqa: E402  (imports the reference from /root/reference/pkg/src)
from ssmkit.config import RunConfig  # noqa: E402
from ssmkit.runner import run_sample  # noqa: E402
from ssmkit.timeseries import InputProvider, TimeSeries, read_timeseries, write_timeseries  # noqa: E402

OUT = os.path.join(HERE, "io")
MODELS = "/root/reference/pkg/models"


def main():
    os.makedirs(OUT, exist_ok=True)
    import ssmkit.core.ir as I

    I.compile_expr = lambda e, t, b: eval(
        f"lambda T, X, W, U: {I.expr_source(e, t, b)}", {"np": np, "inf": np.inf, "__builtins__": {}}
    )
    wk = M.load("windkessel")
    l96 = M.load("lorenz96")
    g = np.load(os.path.join(HERE, "pf.npz"))
    # windkessel input (flow every 0.01 s) and observations (Pa, one masked)
    ts = TimeSeries(times=g["wk/in_times"]).add("F", g["wk/in_values"])
    write_timeseries(os.path.join(OUT, "wk_input.csv"), ts, wk)
    obs = g["wk/obs_v"][:40, 0].copy()
    mask = np.ones(40, bool)
    mask[7] = False
    ots = TimeSeries(times=np.linspace(0, 0.4, 41)[1:]).add("Pa", obs, mask)
    write_timeseries(os.path.join(OUT, "wk_obs.csv"), ots, wk)
    prov = InputProvider(wk, read_timeseries(os.path.join(OUT, "wk_input.csv"), wk, roles=("input",)))
    tq = np.concatenate([np.linspace(0.0, 1.0, 301), g["wk/in_times"] - 1e-12, g["wk/in_times"] + 5e-10])
    tq = tq[(tq >= 0.0) & (tq <= 1.0)]
    np.savez_compressed(os.path.join(OUT, "wk_input_at.npz"), t=tq, v=np.array([prov.at(t) for t in tq]))
    # sparse L96 observations on the benchmark step (slots 0-3 every other step, 20 steps of 0.05)
    ir, theta, times, ot, ov, om = M.l96_data(obs_every=2, slots=range(4), T=40)
    keep = ot <= 1.0 + 1e-12
    lts = TimeSeries(times=ot[keep]).add("y", ov[keep], om[keep])
    write_timeseries(os.path.join(OUT, "l96_obs.csv"), lts, l96)
    # posterior runs through the reference's own driver (runner.run_sample)
    cfg = RunConfig(model_file=os.path.join(MODELS, "lorenz96/Lorenz96.bi"), target="posterior", sampler="mh",
                    nsamples=6, nparticles=128, noutputs=10, start_time=0.0, end_time=1.0,
                    obs_file=os.path.join(OUT, "l96_obs.csv"), output_file=os.path.join(OUT, "l96_mh_samples.txt"),
                    seed=31, resampler="systematic")
    run_sample(cfg)
    cfg = RunConfig(model_file=os.path.join(MODELS, "windkessel/Windkessel.bi"), target="posterior",
                    sampler="smc2", nsamples=8, nparticles=256, noutputs=20, start_time=0.0, end_time=0.4,
                    input_file=os.path.join(OUT, "wk_input.csv"), obs_file=os.path.join(OUT, "wk_obs.csv"),
                    output_file=os.path.join(OUT, "wk_smc_samples.txt"), seed=32, resampler="systematic")
    run_sample(cfg)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
