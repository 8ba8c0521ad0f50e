# offspring_tiles_kernel register cap: default (64 regs, 4 CTAs/SM) vs 5 / 6 CTAs/SM, bench.py resample phase
for r in 1 2; do
  for v in default off5 off6; do
    if [ $v = default ]; then unset SSM_LIB_PATH; else export SSM_LIB_PATH=paper_1306_3277_b200/lib/variants/$v/libssm_b200.so; fi
    python bench.py --steps 10 --e2e-steps 0 --cpu-baseline 0 > gpurun_out/off_$v.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/off_$v.json').read().strip().splitlines()[-1]); k=d['kernels']; print('$v', round(d['ms_per_step'],3), {n: round(v['avg_ms'],4) for n, v in k.items() if n in ('propagate_weight','resample')})"
  done
done
unset SSM_LIB_PATH
