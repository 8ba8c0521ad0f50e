# per-launch times of the sorted-multinomial resample kernels at the bench size (ncu launch list, cold, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"spacing|tile_scale" -c 60 --csv \
  --log-file gpurun_out/mn_ncu.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --cpu-baseline 0 --variants 0 --resampler multinomial > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/mn_ncu.csv")) if len(r) > 10]
h = rows[0]; d = rows[1:]
iK, iV = h.index("Kernel Name"), h.index("Metric Value")
acc = collections.defaultdict(list)
for r in d:
    acc[r[iK][:50]].append(float(r[iV].replace(",", "")))
for k, t in acc.items():
    print(f"{k:50s} n={len(t):3d} avg={sum(t)/len(t)/1e3:8.2f} us")
PY
