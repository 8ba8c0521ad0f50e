#!/bin/bash
# Refresh the round's committed evidence: default bench line, ncu launch list
# and a --set full capture of the per-step kernels (run under gpurun).
mkdir -p gpurun_out
python bench.py > gpurun_out/r_bench_default.json 2> gpurun_out/r_bench_default.err
SKIP=483 COUNT=161 bash profiles/run_ncu_launches.sh
python profiles/launch_summary.py gpurun_out/launches.csv > gpurun_out/r_launch_summary.txt
export KREGEX="pw_kernel|offspring_tiles_kernel|tile_scale|blk_prefix" KSKIP=100 KCOUNT=4 KOUT=r_full
bash profiles/run_ncu_full.sh
ncu -i gpurun_out/r_full.ncu-rep --page raw --csv > gpurun_out/r_full_raw.csv
python profiles/ncu_summary.py gpurun_out/r_full_raw.csv > gpurun_out/r_full_summary.txt
ncu -i gpurun_out/r_full.ncu-rep --page source --print-source sass --csv --kernel-name regex:pw_kernel > gpurun_out/r_pw_sass.csv 2>&1
