#!/bin/bash
# Time each built variant with the bench (no CPU legs); one JSON line each.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for d in paper_1306_3277_b200/lib/variants/*/; do
  name=$(basename $d)
  SSM_LIB_PATH=$d/libssm_b200.so timeout 300 python bench.py --steps ${STEPS:-5} --warmup 3 --cpu-baseline 0 \
      --e2e-steps 0 --variants 0 ${BENCH_EXTRA} > gpurun_out/var_$name.json 2> gpurun_out/var_$name.err
  python - "$name" <<'PY'
import json, sys
name = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/var_{name}.json").read().strip().splitlines()[-1])
    k = d["kernels"]
    print(f"{name:28s} value {d['value']:.4g}  ms/step {d['ms_per_step']:.3f}  pw {k['propagate_weight']['avg_ms']:.4f} ms"
          f"  resample {k.get('resample', {}).get('avg_ms', 0):.4f} ms  clocks {d['clocks']['sm_mhz']}")
except Exception as e:
    print(name, "FAILED", e, open(f"gpurun_out/var_{name}.err").read()[-500:])
PY
done
