"""Aggregate ncu warp-stall samples per CUDA source line (reads a .ncu-rep through the
ncu CLI's source page). Usage: python tools/ncu_lines.py REPORT [top] [line_lo line_hi]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
f = None
agg, tot, hdr = {}, 0, None
stall_cols = None
for r in rows:
    if len(r) >= 2 and r[0] in ("File Path", "File Name"):
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit() and r[2] == "-":
        s = int(r[4] or 0)
        k = (f, int(r[0]), r[1][:100])
        agg[k] = agg.get(k, 0) + s
        tot += s
print("total samples", tot)
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (None, None)
items = sorted(agg.items(), key=lambda x: -x[1])
if lo is not None:
    items = sorted([kv for kv in agg.items() if lo <= kv[0][1] <= hi], key=lambda x: x[0][1])
    print("range share", round(100 * sum(v for _, v in items) / tot, 1), "%")
for k, v in items[:top] if lo is None else items:
    print(f"{v * 100 / tot:5.1f}% {k[0]}:{k[1]} {k[2]}")
