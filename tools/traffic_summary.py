"""Per-dialogue-token DRAM traffic of the decode kernels from an ncu metric CSV
(--metrics dram__bytes_read.sum,dram__bytes_write.sum of one eager engine turn
with the question token + N decode tokens), vs the algorithmic KV bytes.

    python tools/traffic_summary.py launches.csv --batch 16 --token-steps 2 --out traffic.json
"""
import argparse
import collections
import csv
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--token-steps", type=int, default=2)
ap.add_argument("--out")
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
hdr = next(r for r in rows if r and r[0] == "ID")
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
agg = collections.defaultdict(float)
unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for d in data:
    kn = d["Kernel Name"]
    name = ("decode_mma" if "decode_mma" in kn else "decode_cluster" if "decode_cluster" in kn
            else "merge" if "merge" in kn else None)
    if name is None:
        continue
    v = float(d["Metric Value"].replace(",", "")) * unit.get(d["Metric Unit"], 1)
    agg[f"{name}_{'read' if 'read' in d['Metric Name'] else 'write'}_bytes"] += v
from bench import WORKLOADS  # noqa: E402
w = WORKLOADS["c2"]
row = w["hkv"] * w["head_dim"] * 2
K = 4
hist = w["rounds"] * w["round_tokens"]
alg = (w["watershed"] * hist + (w["num_layers"] - w["watershed"]) * K * w["round_tokens"]) * row * 2
tot = sum(agg.values())
out = dict(config=f"c2 shapes, one group of {a.batch} dialogues, {a.token_steps} token-steps (question token + "
                  f"{a.token_steps - 1} decode), eager, ncu cold-cache", **agg,
           per_dialogue_token_bytes=tot / a.batch / a.token_steps,
           algorithmic_per_dialogue_token_bytes=alg)
print(json.dumps(out, indent=1))
if a.out:
    Path(a.out).write_text(json.dumps(out, indent=1))
