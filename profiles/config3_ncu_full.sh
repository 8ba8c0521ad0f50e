# ncu --set full of config 3's per-step kernels (windkessel, 8 filters x 2^16) in one MH step
mkdir -p gpurun_out
python profiles/one_mh_step.py > gpurun_out/c3_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"pw_kernel|offspring_tiles|tile_scale|long_runs" \
    -s 800 -c 4 -o gpurun_out/c3_full python profiles/one_mh_step.py > gpurun_out/c3_ncu_full.log 2>&1
ncu -i gpurun_out/c3_full.ncu-rep --page raw --csv > gpurun_out/c3_full_raw.csv
python profiles/ncu_summary.py gpurun_out/c3_full_raw.csv
