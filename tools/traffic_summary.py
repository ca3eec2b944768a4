"""DRAM traffic of one dialogue group's token steps from an ncu metric CSV
(--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
of `tools/profile_engine.py --eager --turns 1`: one turn = the question token +
N decode tokens), per kernel family and per token step, against the algorithmic
bytes (KV of every visible key + the weights of every layer).

    python tools/traffic_summary.py launches.csv --batch 16 --decode-steps 4 --out traffic.json
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
ap.add_argument("--decode-steps", type=int, default=4)
ap.add_argument("--workload", default="c2")
ap.add_argument("--out")
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
hdr = next(r for r in rows if r and r[0] == "ID")
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3}
agg = collections.defaultdict(lambda: collections.defaultdict(float))
for d in data:
    kn = d["Kernel Name"]
    fam = ("proj_tc" if "proj_tc" in kn else "decode_cluster" if "decode_cluster" in kn
           else "decode_mma" if "decode_mma" in kn else "decode_merge" if "merge" in kn
           else "score_exact" if "exact" in kn else "argmax_embed" if "argmax" in kn else kn.split("(")[0][:40])
    v = float(d["Metric Value"].replace(",", "")) * unit.get(d["Metric Unit"], 1)
    key = "read" if "read" in d["Metric Name"] else "write" if "write" in d["Metric Name"] else "us"
    agg[fam][key] += v
    if key == "us":
        agg[fam]["launches"] += 1
from bench import WORKLOADS  # noqa: E402
from paper_2502_15294_b200.decode_model import ModelShape  # noqa: E402
w = WORKLOADS[a.workload]
row = w["hkv"] * w["head_dim"] * 2
K = 4 if a.workload == "c2" else 13
hist = w["rounds"] * w["round_tokens"]
kv = (w["watershed"] * hist + (w["num_layers"] - w["watershed"]) * K * w["round_tokens"]) * row * 2 * a.batch
sh = ModelShape(w["num_layers"], w["hq"], w["hkv"], w["head_dim"])
wb = 2 * (sh.num_layers * (sh.d_model * sh.qkv_width + sh.d_model * sh.d_model) + sh.vocab * sh.d_model)
steps = 1 + a.decode_steps                    # the 1-row question runs as one token step
tot = sum(f["read"] + f["write"] for f in agg.values())
out = {"config": f"{a.workload} shapes, one group of {a.batch} dialogues, one eager turn = question token + "
                 f"{a.decode_steps} decode tokens ({steps} token steps), ncu cold-cache, serialised",
       "batch_per_group": a.batch, "token_steps": steps,
       "per_family": {k: {kk: vv for kk, vv in v.items()} for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["us"])},
       "per_token_step_bytes_per_group": tot / steps,
       "algorithmic_per_token_step_bytes_per_group": kv + wb,
       "algorithmic_kv_bytes": kv, "algorithmic_weight_bytes": wb,
       "ratio_measured_to_algorithmic": tot / steps / (kv + wb)}
s = json.dumps(out, indent=1)
print(s)
if a.out:
    Path(a.out).write_text(s + "\n")
