"""Decode-step time vs batch (CUDA-graph replay of the decode loop only):
separates the per-layer fixed overhead from the bandwidth term.

    python tools/bench_layers.py --workload c2 --batches 1,4,16
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2502_15294_b200.decode_engine import EngineConfig, RoundDecodeEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--batches", default="1,4,16")
ap.add_argument("--decode-steps", type=int, default=32)
a = ap.parse_args()
peak = 6549.4
for B in [int(x) for x in a.batches.split(",")]:
    w = dict(WORKLOADS[a.workload])
    w.update(batch=B, decode_steps=a.decode_steps, host_unique=1)
    eng = RoundDecodeEngine(EngineConfig(**w))
    eng.prepare(e2e=False)
    for _ in range(2):
        eng.run_turn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        eng.run_turn()
        torch.cuda.synchronize()
        ts.append(eng.turn_breakdown_ms()["decode"])
    ms = sorted(ts)[len(ts) // 2] / a.decode_steps
    bt = eng.kv_bytes_per_token()
    print(json.dumps(dict(B=B, us_per_token_step=ms * 1000, GBps=bt / (ms / 1e3) / 1e9,
                          frac=bt / (ms / 1e3) / 1e9 / peak, bytes=bt, tok_s=B / (ms / 1e3))), flush=True)
    del eng
    torch.cuda.empty_cache()
