"""Kernel microbenchmarks (device-resident inputs, CUDA events, L2 flushed
between launches by using KV far larger than L2 or an explicit flush).

    python tools/bench_kernels.py [--json out.json]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2502_15294_b200 import kernels  # noqa: E402

PEAK = 6549.4


def flush(buf):
    buf.zero_()


def time_decode(B, S, hkv, G, d, dtype=torch.bfloat16, iters=20, append=True, items=None):
    dev = "cuda"
    kc = torch.randn(B, S + 1, hkv, d, device=dev).to(dtype)
    vc = torch.randn(B, S + 1, hkv, d, device=dev).to(dtype)
    q = torch.randn(B, hkv * G, d, device=dev)
    kn = torch.randn(B, hkv, d, device=dev).to(dtype) if append else None
    vn = torch.randn(B, hkv, d, device=dev).to(dtype) if append else None
    sl = torch.full((B,), S, dtype=torch.int32, device=dev)
    out = torch.empty(B, hkv * G, d, device=dev)
    l2 = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        kernels.decode_attention(q, kc, vc, sl, S + 1, k_new=kn, v_new=vn, out=out)
    torch.cuda.synchronize()
    times = []
    for _ in range(iters):
        flush(l2)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        kernels.decode_attention(q, kc, vc, sl, S + 1, k_new=kn, v_new=vn, out=out)
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) * 1e-3)
    times.sort()
    t = times[len(times) // 2]
    elem = 2 if dtype == torch.bfloat16 else 4
    nbytes = B * (S + 1) * hkv * d * elem * 2
    return dict(B=B, S=S, hkv=hkv, G=G, d=d, us=t * 1e6, GBps=nbytes / t / 1e9, frac=nbytes / t / 1e9 / PEAK)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json")
    args = ap.parse_args()
    rows = []
    for cfg in [(1, 16384, 8, 4, 128), (1, 2048, 8, 4, 128), (1, 65536, 4, 7, 128), (1, 7168, 4, 7, 128),
                (16, 131072, 8, 4, 128), (16, 13312, 8, 4, 128), (8, 16384, 8, 4, 128), (64, 16384, 8, 4, 128)]:
        r = time_decode(*cfg)
        rows.append(r)
        print(json.dumps(r), flush=True)
    if args.json:
        Path(args.json).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
