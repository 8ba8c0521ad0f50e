#!/bin/bash
# ncu --set full capture of the three per-step kernels at the bench size (run under gpurun).
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --cpu-baseline 0 ${EXTRA}"
$CMD > gpurun_out/plain.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"${KREGEX:-pw_kernel|offspring_kernel|expand_kernel|tile_sums}" -s ${KSKIP:-160} -c ${KCOUNT:-4} \
    -o gpurun_out/${KOUT:-prof} $CMD > gpurun_out/ncu_full.log 2>&1
