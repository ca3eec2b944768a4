"""Same-box comparison point (library code, not on the product path): FlashInfer
single_prefill_with_kv_cache at the C3 prefill shape (bf16 q / K / V, causal
aligned to the end of the history; bf16 softmax P), vs tools/bench_prefill.py.

    python tools/bench_flashinfer_prefill.py --nq 128,512,1024
"""
import argparse
import json

import torch

import flashinfer

ap = argparse.ArgumentParser()
ap.add_argument("--nq", default="128,512,1024")
ap.add_argument("--hq", type=int, default=28)
ap.add_argument("--hkv", type=int, default=4)
a = ap.parse_args()
d, hist = 128, 64 * 1024
for nq in [int(x) for x in a.nq.split(",")]:
    s = hist + nq
    q = torch.randn(nq, a.hq, d, device="cuda").bfloat16()
    k = torch.randn(s, a.hkv, d, device="cuda").bfloat16()
    v = torch.randn(s, a.hkv, d, device="cuda").bfloat16()
    f = lambda: flashinfer.single_prefill_with_kv_cache(q, k, v, causal=True)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[5]
    flop = 4.0 * a.hq * d * (nq * hist + nq * (nq + 1) / 2)
    print(json.dumps(dict(impl="flashinfer", n_q=nq, ms=round(ms, 4), algo_tflops=round(flop / ms / 1e9))), flush=True)

# FlashInfer's Blackwell backends through the ragged batch-prefill wrapper (one request)
for backend in ("cutlass", "trtllm-gen", "fa2"):
    for nq in [int(x) for x in a.nq.split(",")]:
        s = hist + nq
        try:
            q = torch.randn(nq, a.hq, d, device="cuda").bfloat16()
            k = torch.randn(s, a.hkv, d, device="cuda").bfloat16()
            v = torch.randn(s, a.hkv, d, device="cuda").bfloat16()
            wsb = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
            w = flashinfer.BatchPrefillWithRaggedKVCacheWrapper(wsb, "NHD", backend=backend)
            qo = torch.tensor([0, nq], dtype=torch.int32, device="cuda")
            kvi = torch.tensor([0, s], dtype=torch.int32, device="cuda")
            w.plan(qo, kvi, a.hq, a.hkv, d, causal=True, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
            f = lambda: w.run(q, k, v)  # noqa: E731
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            ts = []
            for _ in range(10):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                f()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = sorted(ts)[5]
            flop = 4.0 * a.hq * d * (nq * hist + nq * (nq + 1) / 2)
            print(json.dumps(dict(impl=f"flashinfer-{backend}", n_q=nq, ms=round(ms, 4),
                                  algo_tflops=round(flop / ms / 1e9))), flush=True)
        except Exception as exc:  # backend unavailable on this build
            print(json.dumps(dict(impl=f"flashinfer-{backend}", n_q=nq, error=repr(exc)[:160])), flush=True)
            break
