# offspring_pipe_kernel (default) vs offspring_tiles_kernel (SSM_NO_OFFSPRING_PIPE=1): bench A/B, alternating
for r in 1 2 3; do
  for v in pipe tiles; do
    if [ $v = tiles ]; then export SSM_NO_OFFSPRING_PIPE=1; else unset SSM_NO_OFFSPRING_PIPE; fi
    python bench.py --steps 10 --e2e-steps 0 --cpu-baseline 0 --variants 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e10,4), {k:v['avg_ms'] for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
  done
done
unset SSM_NO_OFFSPRING_PIPE
