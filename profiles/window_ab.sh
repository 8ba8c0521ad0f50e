# offspring window 4096 (default) vs 8192 outputs per block (SSM_OFF_WINDOW; minBlocks 4 or 6): ncu per-launch + bench
for v in default w8k4 w8k6; do
  if [ $v = default ]; then unset SSM_LIB_PATH; else export SSM_LIB_PATH=paper_1306_3277_b200/lib/variants/$v/libssm_b200.so; fi
  bash profiles/ts_ncu.sh > /dev/null 2>&1
  python - $v <<'PY'
import csv, collections, sys
rows = [r for r in csv.reader(open("gpurun_out/ts_ncu.csv")) if len(r) > 10]
h = rows[0]; d = rows[1:]
iK, iV = h.index("Kernel Name"), h.index("Metric Value")
acc = collections.defaultdict(list)
for r in d:
    if "offspring" in r[iK]: acc["offspring"].append(float(r[iV].replace(",", "")))
print(sys.argv[1], {k: round(sum(t)/len(t)/1e3, 2) for k, t in acc.items()})
PY
done
for r in 1 2; do
  for v in default w8k4 w8k6; do
    if [ $v = default ]; then unset SSM_LIB_PATH; else export SSM_LIB_PATH=paper_1306_3277_b200/lib/variants/$v/libssm_b200.so; fi
    python bench.py --steps 10 --e2e-steps 0 --cpu-baseline 0 --variants 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e10,4), {k:v['avg_ms'] for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
  done
done
unset SSM_LIB_PATH
