"""Summarise an ncu --csv launch list (gpu__time_duration.sum per kernel)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
seq = []
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0][:70]
    v = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)
    agg.setdefault(name, []).append(v)
    seq.append((name, v, d.get("Grid Size", "")))
tot = sum(v for _, v, _ in seq)
print(f"{'kernel':72s} {'n':>5s} {'mean_us':>9s} {'sum_us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:72s} {len(v):5d} {sum(v)/len(v):9.2f} {sum(v):10.1f} {sum(v)/tot:6.1%}")
if "--seq" in sys.argv:
    for n, v, g in seq:
        print(f"  {n[:50]:50s} {v:8.2f} {g}")
