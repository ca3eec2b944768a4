"""Time one decode token step of one dialogue group and its parts (CUDA graphs,
CUDA events): the whole step (per layer qkv_rope + decode attention + out_proj,
then lm_head), the projections alone, and the attention alone.  Prints one
JSON line per (batch) with us per step and GB/s against the algorithmic bytes.

    python tools/bench_token_step.py --workload c2 --batch 16 [--reps 20]
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
ap.add_argument("--batch", type=int, nargs="+", default=[16])
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()


def graph_time(fn, reps):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000.0 / reps


for B in a.batch:
    w = dict(WORKLOADS[a.workload])
    w.update(batch=B, decode_steps=2, plant=0, host_unique=1)
    eng = RoundDecodeEngine(EngineConfig(**w))
    c, m = eng.cfg, eng.model
    eng.lower_len.copy_(eng.lower_len0)
    eng.upper_len.copy_(eng.upper_len0)
    eng.pos.copy_(eng.pos_dec0)

    def step():
        for l in range(c.num_layers):
            eng._layer(l, advance=False)
        kernels.lm_head(eng.x, m.emb_packed, m.shape.vocab, m.emb, eng.x, eng.tokens, None, ws=eng.lm_ws)

    def proj():
        for l in range(c.num_layers):
            kernels.qkv_rope(eng.x, m.w_qkv_packed[l], c.hq, c.hkv, c.head_dim, eng.pos, m.freq, eng.q_buf,
                             eng.k_new, eng.v_new)
            kernels.out_proj(eng.attn, m.w_o_packed[l], eng.x)
        kernels.lm_head(eng.x, m.emb_packed, m.shape.vocab, m.emb, eng.x, eng.tokens, None, ws=eng.lm_ws)

    def qkv_only():
        for l in range(c.num_layers):
            kernels.qkv_rope(eng.x, m.w_qkv_packed[l], c.hq, c.hkv, c.head_dim, eng.pos, m.freq, eng.q_buf,
                             eng.k_new, eng.v_new)

    def oproj_only():
        for l in range(c.num_layers):
            kernels.out_proj(eng.attn, m.w_o_packed[l], eng.x)

    def attn():
        for l in range(c.num_layers):
            kc, vc, ln, cap = eng._caches(l)
            kernels.decode_attention(eng.q_buf, kc, vc, ln, cap, k_new=eng.k_new, v_new=eng.v_new,
                                     out=eng.attn.view(c.batch, c.hq, c.head_dim), ws=eng.ws)

    res = {"workload": a.workload, "batch": B}
    kv = eng.kv_bytes_per_token()
    wb = eng.weight_bytes_per_token()
    qkv_b = sum(x.numel() * 2 for x in m.w_qkv_packed)
    o_b = sum(x.numel() * 2 for x in m.w_o_packed)
    for name, fn, nbytes in (("step", step, kv + wb), ("proj", proj, wb), ("qkv", qkv_only, qkv_b),
                             ("oproj", oproj_only, o_b), ("attn", attn, kv)):
        us = graph_time(fn, a.reps)
        res[name + "_us"] = round(us, 1)
        res[name + "_GBps"] = round(nbytes / (us * 1e-6) / 1e9, 1)
    print(json.dumps(res), flush=True)
    del eng
    torch.cuda.empty_cache()
