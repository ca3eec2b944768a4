"""Same-box comparison point (library code, not on the product path): FlashInfer's
paged batch decode on the shapes of tools/bench_decode_layer.py (bf16 KV, NHD,
page 16), replayed from a CUDA graph of N back-to-back calls.

    python tools/bench_flashinfer_decode.py --batches 1,4,16 --keys 2177,16513
"""
import argparse
import json

import torch

import flashinfer

ap = argparse.ArgumentParser()
ap.add_argument("--batches", default="1,4,16")
ap.add_argument("--keys", default="2177,16513")
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--hkv", type=int, default=8)
ap.add_argument("--calls", type=int, default=64)
a = ap.parse_args()
peak, d, page = 6547.2, 128, 16
for S in [int(x) for x in a.keys.split(",")]:
    for B in [int(x) for x in a.batches.split(",")]:
        L = S + 1
        npg = (L + page - 1) // page
        kv = torch.randn(B * npg, 2, page, a.hkv, d, device="cuda").bfloat16()
        indptr = torch.arange(0, (B + 1) * npg, npg, dtype=torch.int32, device="cuda")
        indices = torch.arange(B * npg, dtype=torch.int32, device="cuda")
        last = torch.full((B,), L - (npg - 1) * page, dtype=torch.int32, device="cuda")
        q = torch.randn(B, a.hq, d, device="cuda").bfloat16()
        wsb = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        w = flashinfer.CUDAGraphBatchDecodeWithPagedKVCacheWrapper(wsb, indptr, indices, last, kv_layout="NHD")
        w.plan(indptr, indices, last, a.hq, a.hkv, d, page, q_data_type=torch.bfloat16,
               kv_data_type=torch.bfloat16)
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())      # inputs were written on the default stream
        with torch.cuda.stream(st):
            for _ in range(3):
                o = w.run(q, kv)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for _ in range(a.calls):
                    o = w.run(q, kv)
            ts = []
            for _ in range(7):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                g.replay()
                e1.record(st)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / a.calls)
        ms = sorted(ts)[3]
        byts = B * L * a.hkv * d * 2 * 2
        print(json.dumps(dict(impl="flashinfer", keys=S, B=B, us_per_call=round(ms * 1000, 2),
                              GBps=round(byts / ms / 1e6), frac=round(byts / ms / 1e6 / peak, 3))), flush=True)
        del kv, g, w
        torch.cuda.empty_cache()
