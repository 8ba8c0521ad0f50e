# per-launch times (ncu launch list, cold cache, serialised) of the offspring kernels: lean (minBlocks 4 / 3) vs general
run() {  # tag, env...
  local tag=$1; shift
  env "$@" ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"offspring|tile_scale" -c 60 --csv \
    --log-file gpurun_out/lean_ncu_$tag.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --cpu-baseline 0 > /dev/null 2>&1
  python - "$tag" <<'PY'
import csv, sys, collections
tag = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/lean_ncu_{tag}.csv")) if len(r) > 10]
h = rows[0]; d = rows[1:]
iK, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
acc = collections.defaultdict(lambda: collections.defaultdict(list))
for r in d:
    acc[r[iK].split("(")[0][:40]][r[iM]].append(float(r[iV].replace(",", "")))
for k, m in acc.items():
    t = m["gpu__time_duration.sum"]; rd = m["dram__bytes_read.sum"]; wr = m["dram__bytes_write.sum"]
    print(f"{tag:8s} {k:40s} n={len(t):3d} avg={sum(t)/len(t)/1e3:7.1f} us rd={sum(rd)/len(rd)/1e6:6.1f} MB wr={sum(wr)/len(wr)/1e6:6.1f} MB")
PY
}
run lean4
run lean3 SSM_LIB_PATH=paper_1306_3277_b200/lib/variants/lean3/libssm_b200.so
run general SSM_NO_OFFSPRING_LEAN=1
