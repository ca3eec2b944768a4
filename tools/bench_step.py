"""Token-step time of the persistent whole-step kernel (rk_decode_step, one
launch per token) against the layered path (qkv_rope + decode attention +
out_proj per layer, then lm_head), both replayed from CUDA graphs and timed
with CUDA events.  One JSON line per batch: us per step and GB/s over the
algorithmic KV + weight bytes of the step.

    python tools/bench_step.py --workload c2 --batch 1 2 4 8 16 [--steps 32]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2502_15294_b200 import kernels  # noqa: E402
from paper_2502_15294_b200.decode_engine import EngineConfig, RoundDecodeEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--batch", type=int, nargs="+", default=[1, 2, 4, 8, 16])
ap.add_argument("--steps", type=int, default=32, help="token steps per graph replay")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()


def graph_time(fn, reset, reps, steps):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        reset()
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        best = None
        for _ in range(reps + 1):
            reset()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) * 1000.0 / steps
            best = t if best is None else min(best, t)
    return best


for B in a.batch:
    w = dict(WORKLOADS[a.workload])
    w.update(batch=B, decode_steps=a.steps, plant=0, host_unique=1, step_kernel="persistent")
    eng = RoundDecodeEngine(EngineConfig(**w))
    c, m = eng.cfg, eng.model

    def reset():
        eng.lower_len.copy_(eng.lower_len0)
        eng.upper_len.copy_(eng.upper_len0)
        eng.pos.copy_(eng.pos_dec0)

    def layered():
        for _ in range(a.steps):
            for l in range(c.num_layers):
                eng._layer(l, advance=(l == c.watershed - 1 or l == c.num_layers - 1))
            kernels.lm_head(eng.x, m.emb_packed, m.shape.vocab, m.emb, eng.x, eng.tokens, eng.pos, ws=eng.lm_ws)

    def persistent():
        for t in range(a.steps):
            kernels.decode_step(eng.step_args[t])

    nbytes = eng.kv_bytes_per_token() + eng.weight_bytes_per_token()
    res = {"workload": a.workload, "batch": B, "GB_per_step": round(nbytes / 1e9, 3)}
    for name, fn in (("layers", layered), ("persistent", persistent)):
        us = graph_time(fn, reset, a.reps, a.steps)
        res[name + "_us"] = round(us, 1)
        res[name + "_GBps"] = round(nbytes / (us * 1e-6) / 1e9, 1)
    res["speedup"] = round(res["layers_us"] / res["persistent_us"], 3)
    print(json.dumps(res), flush=True)
    del eng
    torch.cuda.empty_cache()
