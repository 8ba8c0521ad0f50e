"""Summarise an ncu --set full report (raw page CSV) -> key metrics + top stalls per kernel.
usage: ncu -i X.ncu-rep --page raw --csv > raw.csv; python profiles/ncu_summary.py raw.csv"""
import csv
import sys

WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu%"),
    ("sm__inst_executed.avg.per_cycle_active", "ipc"),
    ("smsp__inst_executed.sum", "inst"),
    ("launch__grid_size", "grid"),
]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    for d in data:
        print("-----", d[hdr.index("Kernel Name")][:90])
        out = []
        for key, short in WANT:
            if key in hdr:
                i = hdr.index(key)
                out.append(f"{short}={d[i]}{units[i]}")
        print("  " + "  ".join(out))
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(d[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        print("  stalls: " + ", ".join(f"{n}={v:.2f}" for v, n in st[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
