# pw_body_lag (weighting one tile behind) vs pw_body for the headline step, interleaved
mkdir -p gpurun_out
for r in 1 2 3; do
  for v in lag nolag; do
    if [ $v = nolag ]; then export SSM_NO_PW_LAG=1; else unset SSM_NO_PW_LAG; fi
    python bench.py --steps 10 --e2e-steps 0 --cpu-baseline 0 > gpurun_out/lag_$v.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/lag_$v.json').read().strip().splitlines()[-1]); k=d['kernels']; print('$v', round(d['ms_per_step'],3), d['value'], round(d['roofline']['frac'],4), {n: round(v['avg_ms'],4) for n, v in k.items() if n in ('propagate_weight','resample')}, d['clocks']['sm_mhz'])"
  done
done
unset SSM_NO_PW_LAG
