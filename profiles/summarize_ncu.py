"""Summarise an ncu --set full report into the per-kernel numbers the
roofline needs (duration, DRAM bytes, DRAM/tensor/SM utilisation).

    python profiles/summarize_ncu.py gpurun_out/prof.ncu-rep > profiles/rNN_ncu_summary.md
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clk"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_%"),
]


def launch_shares(path):
    """Per-kernel totals and shares from a `--metrics gpu__time_duration.sum` launch list."""
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = {}
    for r in rows[1:]:
        n = r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").split("(")[0]
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(a[1] for a in agg.values())
    print(f"# launch list `{path}` (cold-cache, serialised: compare shares)\n")
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {n} | {c} | {t / 1e6:.3f} | {100 * t / tot:.1f}% |")


def main(path):
    if path.endswith(".csv"):
        return launch_shares(path)
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu summary of `{path}`\n")
    print("| kernel | " + " | ".join(k[1] for k in KEYS) + " |")
    print("|---|" + "---|" * len(KEYS))
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?").replace("(anonymous namespace)::", "").split("(")[0]
        cells = []
        for key, _ in KEYS:
            v = d.get(key, "")
            cells.append(f"{v} {u.get(key, '')}".strip())
        print(f"| {name} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
