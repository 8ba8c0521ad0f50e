# ncu launch list of one config-3 MH step (8 windkessel filters x 2^16, T=100) after a warm-up
mkdir -p gpurun_out
W=$(python profiles/one_mh_step.py 2>/dev/null | grep "warm launches" | awk '{print $3}')
echo "warm launches $W"
ncu --metrics gpu__time_duration.sum --clock-control none -s $W -c 420 --csv --log-file gpurun_out/c3_launches.csv \
    python profiles/one_mh_step.py > gpurun_out/c3_ncu.log 2>&1
python profiles/launch_summary.py gpurun_out/c3_launches.csv
