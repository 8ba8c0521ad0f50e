# tiles per pw block at moderate P (config 3: 8 windkessel filters x 2^16; L96 2^16 / 2^18 / 2^20 sweep points)
for r in 1 2; do
  for v in default tpb2 tpb1; do
    if [ $v = default ]; then unset SSM_LIB_PATH; else export SSM_LIB_PATH=paper_1306_3277_b200/lib/variants/$v/libssm_b200.so; fi
    python bench_outer.py --configs 3d 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v config3', round(d['ms_per_mh_step'],3))"
  done
done
unset SSM_LIB_PATH
