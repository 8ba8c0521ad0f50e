# offspring_lean_kernel (default) vs the general offspring_tiles_kernel (SSM_NO_OFFSPRING_LEAN=1):
# bench.py headline resample phase, and the r microbench split (resample_from_logw + gather)
for r in 1 2; do
  for v in lean general; do
    if [ $v = general ]; then export SSM_NO_OFFSPRING_LEAN=1; else unset SSM_NO_OFFSPRING_LEAN; fi
    python bench.py --steps 10 --e2e-steps 0 --cpu-baseline 0 > gpurun_out/lean_$v.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/lean_$v.json').read().strip().splitlines()[-1]); k=d['kernels']; print('$v', round(d['value']/1e10,4), round(d['ms_per_step'],3), {n: round(v['avg_ms'],4) for n, v in k.items() if n in ('propagate_weight','resample')}, d['clocks']['sm_mhz'])"
  done
done
unset SSM_NO_OFFSPRING_LEAN
for v in lean general; do
  if [ $v = general ]; then export SSM_NO_OFFSPRING_LEAN=1; else unset SSM_NO_OFFSPRING_LEAN; fi
  echo "== gather_probe $v"; python profiles/gather_probe.py
done
unset SSM_NO_OFFSPRING_LEAN
