"""Multi-row watershed scoring at the C3 shape (Qwen2-7B-shaped layer Lw-1:
Hq=28, Hkv=4, d=128, 64 rounds x 1024 history keys, n_q question rows).

    python tools/bench_scoring.py [--nq 128,512,1024] [--json out.json]
Run with RK_SCORE_TC=0 to time the CUDA-core split kernel instead.
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_15294_b200 import stats  # noqa: E402

PEAK_TF = 1633.6          # MEASURED_PEAKS bf16 burst
ap = argparse.ArgumentParser()
ap.add_argument("--nq", default="128,512,1024")
ap.add_argument("--rounds", type=int, default=64)
ap.add_argument("--T", type=int, default=1024)
ap.add_argument("--json")
ap.add_argument("--exact", action="store_true", help="time rk_round_scores_exact (fp64) instead of the tcgen05 scorer")
a = ap.parse_args()
hq, hkv, d = 28, 4, 128
rows = []
for nq in [int(x) for x in a.nq.split(",")]:
    hist = a.rounds * a.T
    s = hist + nq
    k = torch.randn(s, hkv, d, device="cuda").bfloat16()
    q = torch.randn(nq, hq, d, device="cuda")
    qp = torch.arange(hist, s, device="cuda")
    kp = torch.arange(s, device="cuda")
    bounds = [(r * a.T, (r + 1) * a.T, r) for r in range(a.rounds)] + [(hist, s, a.rounds)]
    for _ in range(2):
        stats.round_scores(q, k, qp, kp, bounds, a.rounds, chunk=1024, exact=a.exact)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        stats.round_scores(q, k, qp, kp, bounds, a.rounds, chunk=1024, exact=a.exact)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    ms_dev = None
    if not a.exact and os.environ.get("RK_SCORE_TC", "1") != "0":
        # the same scoring through the C ABI with the item table already on the device: the
        # kernels alone (prep, scores-only pass, score_rows, score_sum_rows), no host work inside
        from paper_2502_15294_b200 import _lib
        from paper_2502_15294_b200.workspace import scratch
        items = torch.from_numpy(stats.build_round_items(bounds, 1024)).to("cuda")
        raw = torch.zeros(a.rounds, dtype=torch.float64, device="cuda")
        wsb = _lib.lib.rk_round_scores_workspace_bytes(nq, hq, hkv, items.shape[0], d, a.rounds)
        ws = scratch(wsb, torch.device("cuda"), "bench_scores")

        def direct():
            _lib.call("rk_round_scores", _lib.ptr(q), nq, hq, d, _lib.ptr(k), _lib.RK_BF16, s, hkv, _lib.ptr(qp),
                      _lib.ptr(kp), _lib.ptr(items), items.shape[0], a.rounds, None, _lib.ptr(raw), _lib.ptr(ws),
                      ws.numel(), _lib.stream_ptr())
        direct()
        torch.cuda.synchronize()
        td = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            direct()
            e1.record()
            torch.cuda.synchronize()
            td.append(e0.elapsed_time(e1))
        ms_dev = sorted(td)[len(td) // 2]
        ref = stats.round_scores(q, k, qp, kp, bounds, a.rounds, chunk=1024, exact=False)
        assert torch.equal(raw, ref), "direct ABI call differs from stats.round_scores"
    visible = nq * hist + nq * (nq + 1) / 2            # causal keys per head
    flop = 2.0 * hq * d * nq * s                        # algorithmic QK^T (all tiles)
    exps = hq * visible
    r = dict(n_q=nq, keys=s, ms=ms, ms_device=ms_dev, algo_tflops=flop / ms / 1e9, frac_bf16_peak=flop / ms / 1e9 / PEAK_TF,
             tensor_tflops_issued=2 * flop / ms / 1e9, gexp_s=exps / ms / 1e6,
             path="exact fp64" if a.exact else "tcgen05" if os.environ.get("RK_SCORE_TC", "1") != "0" else "cuda-core")
    rows.append(r)
    print(json.dumps(r), flush=True)
if a.json:
    Path(a.json).write_text(json.dumps(rows, indent=1))
