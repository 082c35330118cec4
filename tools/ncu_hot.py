"""Hot spots of an ncu report by warp-stall samples, for reading a kernel
here without the GUI.

usage: python tools/ncu_hot.py <report.ncu-rep> [n]          top SASS instructions
       python tools/ncu_hot.py <report.ncu-rep> [n] --lines  top CUDA source lines
"""
import collections
import csv
import io
import subprocess
import sys


def _rows(path, view):
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", view],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(txt)))


def sass(path, n):
    rows = _rows(path, "sass")
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


def lines(path, n):
    rows = _rows(path, "cuda,sass")
    fname, h = "?", None
    agg = collections.defaultdict(lambda: [0, collections.Counter(), ""])
    for r in rows:
        if r[:1] == ["File Path"]:
            fname = r[1].split("/")[-1]
            continue
        if r[:2] == ["Line No", "Source"]:
            h = r
            si = h.index("Warp Stall Sampling (All Samples)")
            stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
            continue
        if h is None or len(r) <= si or not r[0].strip().isdigit():
            continue
        s = int(r[si]) if r[si].strip().isdigit() else 0
        key = (fname, int(r[0]))
        agg[key][0] += s
        agg[key][2] = r[1].strip()[:90]
        for i in stall_cols:
            try:
                agg[key][1][h[i][6:]] += float(r[i] or 0)
            except ValueError:
                pass
    tot = sum(v[0] for v in agg.values()) or 1
    print(f"total samples {tot}")
    for (f, ln), (s, why, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
        top = ",".join(f"{k}:{int(v)}" for k, v in why.most_common(2))
        print(f"{s:6d} {s / tot:6.3f}  {f}:{ln:<5d} [{top}]  {src}")


if __name__ == "__main__":
    n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 30
    (lines if "--lines" in sys.argv else sass)(sys.argv[1], n)
