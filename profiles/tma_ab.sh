# TMA-staged gather in the lagged headline kernel (SSM_PW_TMA=1) vs register prefetch: correctness then timing
SSM_PW_TMA=1 timeout 300 python -m pytest tests/test_gpu_parity_baseline.py -q -p no:cacheprovider -x -k "headline or config2" 2>&1 | tail -2
for r in 1 2 3; do
  for v in tma lag; do
    unset SSM_PW_TMA; [ $v = tma ] && export SSM_PW_TMA=1
    timeout 300 python bench.py --steps 10 --e2e-steps 0 --cpu-baseline 0 > gpurun_out/tma_$v.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/tma_$v.json').read().strip().splitlines()[-1]); k=d['kernels']; print('$v', round(d['ms_per_step'],3), d['value'], round(d['roofline']['frac'],4), {n: round(v['avg_ms'],4) for n, v in k.items() if n in ('propagate_weight','resample')}, d['clocks']['sm_mhz'])"
  done
done
unset SSM_PW_TMA
