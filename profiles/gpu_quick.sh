#!/bin/bash
# One iteration of the build -> measure loop under gpurun: GPU tests, then the
# bench (f64 FMA headline + exact/f32/multinomial variants), no CPU baseline.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/q_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/q_pytest.log
tail -3 gpurun_out/q_pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 --cpu-baseline 0 ${BENCH_EXTRA} > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/q_bench.json").read().strip().splitlines()[-1])
print("value %.4g  pw %.4f ms  frac %.3f  resample %.4f ms" % (d["value"], d["kernels"]["propagate_weight"]["avg_ms"], d["roofline"]["frac"], d["kernels"]["resample"]["avg_ms"]))
for k, v in d.get("variants", {}).items(): print(k, "%.4g" % v["value"], v.get("pw_GB_s"))
print("clocks", d["clocks"])
PY
