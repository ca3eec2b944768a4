"""Attribute ncu stall samples of mbarrier wait loops to barrier offsets.

    python tools/ncu_waits.py sass.csv     (ncu --page source --csv --print-source sass)
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
S = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[ix[S]] or 0) for r in data)
addr = {r[ix["Address"]]: i for i, r in enumerate(data)}
agg = collections.Counter()


def wait_off(i):
    for j in range(i, max(-1, i - 6), -1):
        m = re.search(r"TRYWAIT P\d+, \[R\d+\+URZ\+(0x[0-9a-f]+)\]", data[j][ix["Source"]])
        if m:
            return m.group(1)
    return None


for i, r in enumerate(data):
    smp = float(r[ix[S]] or 0)
    if not smp:
        continue
    src = r[ix["Source"]]
    m = re.search(r"BRA (0x[0-9a-f]+)", src)
    off = None
    if m and m.group(1) in addr:               # branch into an out-of-line retry loop
        k = addr[m.group(1)]
        for j in range(k, min(k + 4, len(data))):
            mm = re.search(r"TRYWAIT P\d+, \[R\d+\+URZ\+(0x[0-9a-f]+)\]", data[j][ix["Source"]])
            if mm:
                off = mm.group(1)
                break
    if off is None and ("TRYWAIT" in src or "YIELD" in src or "BRA" in src):
        off = wait_off(i)
    if off:
        agg[off] += smp
for k, v in sorted(agg.items()):
    print(k, f"{100 * v / tot:.2f}%")
