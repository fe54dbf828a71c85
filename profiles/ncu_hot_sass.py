"""Top SASS instructions of one kernel in an ncu report by warp-stall samples,
with their dominant stall reasons.
python profiles/ncu_hot_sass.py REPORT KERNEL_REGEX [N] [LAUNCH_SKIP]"""
import csv
import io
import subprocess
import sys


def main(rep, kern, n=30, skip=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--launch-skip", str(skip), "--launch-count", "1", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = next(r for r in rows if r and r[0] == "Address")
    body = [r for r in rows[rows.index(h) + 1:] if len(r) == len(h) and r[0] != "Address"]
    si = h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_")]
    tot = sum(float(r[si] or 0) for r in body)
    print(f"{len(body)} SASS lines, {tot:.0f} samples")
    for idx, r in sorted(enumerate(body), key=lambda x: -float(x[1][si] or 0))[:n]:
        s = float(r[si] or 0)
        reasons = sorted(((float(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:3]
        rs = " ".join(f"{name}={v:.0f}" for v, name in reasons if v > 0)
        print(f"{idx:5d} {100 * s / tot:5.1f}%  {r[1].strip()[:60]:60s} {rs}")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], a[1], int(a[2]) if len(a) > 2 else 30, int(a[3]) if len(a) > 3 else 0)
