#!/bin/bash
# ncu --set full capture of the three per-step kernels at the bench size (run under gpurun).
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --cpu-baseline 0"
$CMD > gpurun_out/plain.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"pw_kernel|scan_kernel|merge_search_kernel" -s 120 -c 3 \
    -o gpurun_out/prof_r1 $CMD > gpurun_out/ncu_full.log 2>&1
