"""Print an `ncu --metrics ... --csv --log-file F` capture compactly:
one line per launch, `name metric=value ...`.  python profiles/ncu_brief.py F"""
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ii, ki, mi, vi = (h.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    cur, out = None, []
    for r in rows[1:]:
        if r[ii] != cur:
            cur = r[ii]
            out.append([r[ki].split("(")[0].replace("(anonymous namespace)::", "")[-48:], {}])
        out[-1][1][r[mi]] = r[vi]
    for name, m in out:
        print(name, " ".join(f"{k.split('.')[0].split('__')[-1]}={v}" for k, v in m.items()))


if __name__ == "__main__":
    main(sys.argv[1])
