# ssm_resample_from_logw: tile-record path (default) vs the previous log-weight scan paths
python profiles/gather_probe.py > gpurun_out/logw_tiles.txt 2>&1
SSM_LIB_PATH=paper_1306_3277_b200/lib/variants/logwscan/libssm_b200.so python profiles/gather_probe.py > gpurun_out/logw_scan.txt 2>&1
echo "== tiles"; cat gpurun_out/logw_tiles.txt; echo "== scan"; cat gpurun_out/logw_scan.txt
