# per-launch tile_scale / offspring times (ncu launch list, cold, serialised) of the current build
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"offspring|tile_scale|long_runs" -c 60 --csv \
  --log-file gpurun_out/ts_ncu.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --cpu-baseline 0 --variants 0 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/ts_ncu.csv")) if len(r) > 10]
h = rows[0]; d = rows[1:]
iK, iV = h.index("Kernel Name"), h.index("Metric Value")
acc = collections.defaultdict(list)
for r in d:
    acc[r[iK].split("(")[0][:40]].append(float(r[iV].replace(",", "")))
for k, t in acc.items():
    print(f"{k:40s} n={len(t):3d} avg={sum(t)/len(t)/1e3:7.2f} us")
PY
