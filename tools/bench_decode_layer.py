"""Per-call time of the decode attention (rk_decode_attention: cluster decode, or persistent split-K + merge with RK_DECODE_CLUSTER=0) on one layer
shape, replayed back to back from a CUDA graph (N dependent calls, as the
layers of one decode token): separates the fixed per-layer cost from the
bandwidth term at small batch.

    python tools/bench_decode_layer.py --batches 1,4,16 --keys 2177,16513
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2502_15294_b200 import kernels  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", default="1,2,4,8,16")
ap.add_argument("--keys", default="2177,16513")       # C2 upper (4 x 512 + turn) / lower (16 K + turn)
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--hkv", type=int, default=8)
ap.add_argument("--calls", type=int, default=64)
ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
a = ap.parse_args()
dt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
es = 2 if a.dtype == "bf16" else 4
peak = 6547.2
d = 128
for S in [int(x) for x in a.keys.split(",")]:
    for B in [int(x) for x in a.batches.split(",")]:
        kc = torch.randn(B, S + 1, a.hkv, d, device="cuda").to(dt)
        vc = torch.randn(B, S + 1, a.hkv, d, device="cuda").to(dt)
        q = torch.randn(B, a.hq, d, device="cuda")
        kn = torch.randn(B, a.hkv, d, device="cuda").to(dt)
        vn = torch.randn(B, a.hkv, d, device="cuda").to(dt)
        sl = torch.full((B,), S, dtype=torch.int32, device="cuda")
        out = torch.empty(B, a.hq, d, device="cuda")
        ws = kernels.decode_workspace(B, a.hq, a.hkv, d, 592, "cuda", tag=f"l{B}_{S}")
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())      # inputs were written on the default stream
        with torch.cuda.stream(st):
            for _ in range(3):
                kernels.decode_attention(q, kc, vc, sl, S + 1, k_new=kn, v_new=vn, out=out, ws=ws)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for _ in range(a.calls):
                    kernels.decode_attention(q, kc, vc, sl, S + 1, k_new=kn, v_new=vn, out=out, ws=ws)
            ts = []
            for _ in range(7):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                g.replay()
                e1.record(st)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / a.calls)
        ms = sorted(ts)[3]
        byts = B * (S + 1) * a.hkv * d * 2 * es
        plan = kernels.decode_plan(B, a.hq, a.hkv, d, dt, S + 1, kc.stride(0))
        print(json.dumps(dict(dtype=a.dtype, keys=S, B=B, plan=plan, us_per_call=round(ms * 1000, 2), GBps=round(byts / ms / 1e6),
                              frac=round(byts / ms / 1e6 / peak, 3), MB=round(byts / 1e6, 1))), flush=True)
        del kc, vc, g
        torch.cuda.empty_cache()
