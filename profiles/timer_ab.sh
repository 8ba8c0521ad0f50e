# A/B: per-kernel event sampling inside bench.py's timed region (1 = every launch, 8 = default,
# 1000 = none of the grid steps), interleaved, 3 rounds
mkdir -p gpurun_out
for r in 1 2 3; do
  for e in 1 8 1000; do
    SSM_BENCH_TIMER_EVERY=$e python bench.py --steps 10 > gpurun_out/tab_$e.json 2>/dev/null
    python -c "import json,sys; d=json.loads(open('gpurun_out/tab_$e.json').read().strip().splitlines()[-1]); print('every=$e', round(d['ms_per_step'],3), d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
  done
done
