"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,... --csv) per kernel."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        name = d["Kernel Name"].split("(")[0][:56]
        a = agg.setdefault(name, collections.defaultdict(list))
        a[d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
    total = sum(sum(a["gpu__time_duration.sum"]) for a in agg.values())
    print(f"{'kernel':56s} {'n':>4s} {'avg_us':>9s} {'share':>6s} {'rd_MB':>8s} {'wr_MB':>8s}")
    for k, a in agg.items():
        t = a["gpu__time_duration.sum"]
        n = len(t)
        rd = sum(a.get("dram__bytes_read.sum", [0])) / n / 1e6
        wr = sum(a.get("dram__bytes_write.sum", [0])) / n / 1e6
        print(f"{k:56s} {n:4d} {sum(t) / n / 1e3:9.1f} {sum(t) / total:6.1%} {rd:8.1f} {wr:8.1f}")
    print(f"total device time {total / 1e6:.3f} ms over {sum(len(a['gpu__time_duration.sum']) for a in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
