"""Top SASS instructions of an ncu report by warp-stall samples (with the
dominant stall reason), for reading a kernel's hot spots here without the GUI.

usage: python tools/ncu_hot.py <report.ncu-rep> [n]
"""
import csv
import io
import subprocess
import sys


def main(path, n=30):
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    h = rows[hi]
    si = h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    data = []
    for idx, r in enumerate(rows[hi + 1:]):
        if len(r) <= si or not r[si].strip().isdigit():
            continue
        s = int(r[si])
        top = max(stall_cols, key=lambda i: float(r[i] or 0))
        data.append((s, idx, r[1].strip()[:80], h[top][6:], r[h.index("Instructions Executed")]))
    tot = sum(d[0] for d in data) or 1
    print(f"total samples {tot}")
    for s, idx, src, why, ex in sorted(data, reverse=True)[:n]:
        print(f"{s:6d} {s / tot:6.3f}  #{idx:5d}  {why:14s} exec={ex:>8s}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
