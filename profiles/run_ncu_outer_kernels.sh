#!/bin/bash
# ncu --set full capture of the theta-level MH and Kalman kernels (run under gpurun).
set -e
mkdir -p gpurun_out
python bench_outer.py --configs k,3d --quick > gpurun_out/outer_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"kalman_kernel|theta_propose|theta_accept" \
    -c 4 -o gpurun_out/r1_outer_kernels python bench_outer.py --configs k,3d --quick > gpurun_out/ncu_outer.log 2>&1
ncu -i gpurun_out/r1_outer_kernels.ncu-rep --page raw --csv > gpurun_out/r1_outer_raw.csv
python profiles/ncu_summary.py gpurun_out/r1_outer_raw.csv > gpurun_out/r1_ncu_outer_kernels_summary.txt
