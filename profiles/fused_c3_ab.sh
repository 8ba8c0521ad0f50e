# config 3 / L96 sweep points with the one-kernel nominal-total resample (SSM_RESAMPLE_FUSED) vs the default
for r in 1 2; do
  python bench_outer.py --configs 3d > gpurun_out/fab_def.jsonl 2>/dev/null
  SSM_LIB_PATH=paper_1306_3277_b200/lib/variants/fused/libssm_b200.so python bench_outer.py --configs 3d > gpurun_out/fab_fused.jsonl 2>/dev/null
  python -c "import json; a=json.loads(open('gpurun_out/fab_def.jsonl').read()); b=json.loads(open('gpurun_out/fab_fused.jsonl').read()); print('default', round(a['ms_per_mh_step'],3), 'fused', round(b['ms_per_mh_step'],3))"
done
