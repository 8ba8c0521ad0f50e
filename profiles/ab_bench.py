"""Interleaved A/B timing of bench.py configurations (run under gpurun).

usage: python profiles/ab_bench.py REPS NAME=ENV[,ENV...] ...   e.g.
       python profiles/ab_bench.py 3 lean= general=SSM_NO_LEAN=1
Each configuration runs REPS times, interleaved (A B A B ...), as a separate
bench.py process (no CPU legs); prints the median of ms/step and the per-phase
kernel times."""
import json
import os
import statistics
import subprocess
import sys

reps = int(sys.argv[1])
configs = []
for spec in sys.argv[2:]:
    name, _, envs = spec.partition("=")
    env = dict(os.environ)
    for kv in filter(None, envs.split(",")):
        k, _, v = kv.partition(":") if ":" in kv else kv.partition("=")
        env[k] = v
    configs.append((name, env))
extra = os.environ.get("BENCH_EXTRA", "").split()
res = {n: [] for n, _ in configs}
for r in range(reps):
    for name, env in configs:
        out = subprocess.run([sys.executable, "bench.py", "--steps", os.environ.get("STEPS", "10"), "--warmup", "3",
                              "--cpu-baseline", "0", "--e2e-steps", "0", "--variants", "0"] + extra,
                             env=env, capture_output=True, text=True)
        try:
            d = json.loads(out.stdout.strip().splitlines()[-1])
            k = d["kernels"]
            res[name].append((d["ms_per_step"], k["propagate_weight"]["avg_ms"], k.get("resample", {}).get("avg_ms", 0.0),
                              d["clocks"]["sm_mhz"]))
        except Exception as e:  # noqa: BLE001
            print(name, "FAILED", e, out.stderr[-800:], flush=True)
for name, rows in res.items():
    if rows:
        med = [statistics.median(c) for c in zip(*rows)]
        print(f"{name:16s} ms/step {med[0]:.3f}  pw {med[1]:.4f} ms  resample {med[2]:.4f} ms  sm {med[3]}  "
              f"(n={len(rows)}: pw {[round(r[1], 4) for r in rows]})", flush=True)
