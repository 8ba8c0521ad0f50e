# ncu --set full of the persistent small-P kernel in config 1 (windkessel, P=1024, T=100, one launch)
mkdir -p gpurun_out
python profiles/one_wk_filter.py > gpurun_out/small_plain.log 2>&1 || exit 1
cat gpurun_out/small_plain.log
ncu --set full --clock-control none --import-source on -k regex:small_filter -s 3 -c 1 -o gpurun_out/small_full \
    python profiles/one_wk_filter.py > gpurun_out/small_ncu.log 2>&1
ncu -i gpurun_out/small_full.ncu-rep --page raw --csv > gpurun_out/small_raw.csv
python profiles/ncu_summary.py gpurun_out/small_raw.csv
ncu -i gpurun_out/small_full.ncu-rep --page source --print-source sass --csv > gpurun_out/small_sass.csv 2>&1
