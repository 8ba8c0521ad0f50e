#!/bin/bash
# Per-launch device times (cold-cache, serialised) for one bench step, after 3 warm-up runs.
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --cpu-baseline 0 ${EXTRA}"
$CMD > gpurun_out/plain_launches.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s ${SKIP:-600} -c ${COUNT:-200} --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
