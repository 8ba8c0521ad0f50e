#!/bin/bash
# Refresh round 2's committed evidence under gpurun: the default bench line and the
# reference arm, an ncu launch list of one bench step, one --set full capture of the
# per-step kernels at grid step ~30 of a filter run, and bench_outer's other configs.
mkdir -p gpurun_out
python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err
SKIP=483 COUNT=161 bash profiles/run_ncu_launches.sh
python profiles/launch_summary.py gpurun_out/launches.csv > gpurun_out/r2_launch_summary.txt
export KREGEX="pw_lag_kernel|offspring_tiles_kernel|tile_scale" KSKIP=125 KCOUNT=3 KOUT=r2_full
bash profiles/run_ncu_full.sh
ncu -i gpurun_out/r2_full.ncu-rep --page raw --csv > gpurun_out/r2_full_raw.csv
python profiles/ncu_summary.py gpurun_out/r2_full_raw.csv > gpurun_out/r2_full_summary.txt
ncu -i gpurun_out/r2_full.ncu-rep --page source --print-source sass --csv --kernel-name regex:pw_lag_kernel > gpurun_out/r2_pw_sass.csv 2>&1
python bench_outer.py --configs 1,3,3d,4,4d,5,g,k,r > gpurun_out/r2_bench_outer.jsonl 2> gpurun_out/r2_bench_outer.err
