"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, data = rows[0], rows[1:]
iN, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
iG = hdr.index("Grid Size")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(list)
for r in data:
    v = float(r[iV].replace(",", "")) * scale.get(r[iU], 1.0)
    agg[r[iN].split("(")[0].replace("void ", "")].append((v, r[iG]))
tot = sum(v for l in agg.values() for v, _ in l)
print(f"launches {len(data)}  total {tot:.1f} us")
for k, l in sorted(agg.items(), key=lambda kv: -sum(v for v, _ in kv[1])):
    vs = [v for v, _ in l]
    print(f"{k[:36]:36s} n={len(vs):4d} sum={sum(vs):9.1f}us ({100*sum(vs)/tot:4.1f}%) mean={sum(vs)/len(vs):7.2f} "
          f"min={min(vs):6.2f} max={max(vs):7.2f} grid={collections.Counter(g for _, g in l).most_common(1)[0][0]}")
