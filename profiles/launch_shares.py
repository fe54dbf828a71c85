"""Per-kernel time shares from an `ncu --metrics gpu__time_duration.sum --csv`
launch list: python profiles/launch_shares.py LIST.csv [skip_launches]"""
import collections
import csv
import sys


def main(path, skip=0):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hd = rows[h]
    ki, vi, ui = hd.index("Kernel Name"), hd.index("Metric Value"), hd.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[h + 1 + skip:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        k = r[ki].split("(")[0].replace("(anonymous namespace)::", "").replace("occ::", "")
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k[:70]}` | {a[0]} | {a[1]:.1f} | {100 * a[1] / tot:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
