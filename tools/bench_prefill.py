"""Question prefill attention at the C3 shape (Qwen2-7B-shaped: Hq=28, Hkv=4,
d=128, 64 rounds x 1024 history keys + an n_q-row question, causal), on the
tcgen05 kernel (rk_prefill_attention), plain and with the fused round scoring
of layer Lw-1; the separate scorer (rk_round_scores) is timed beside it.

    python tools/bench_prefill.py [--nq 128,512,1024] [--json out.json]
Algorithmic FLOPs = 4 * Hq * d * (visible (row, key) pairs): QK^T + PV once,
causal pairs only; the q and P splits double the issued tensor work.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2502_15294_b200 import kernels, stats  # noqa: E402
from paper_2502_15294_b200.stats import build_round_items  # noqa: E402

REPO = Path(__file__).resolve().parents[1]
peaks = json.loads((REPO / "MEASURED_PEAKS.json").read_text()) if (REPO / "MEASURED_PEAKS.json").exists() else {}
PEAK_TF = float(peaks.get("bf16_tflops", 1590.0))
ap = argparse.ArgumentParser()
ap.add_argument("--nq", default="128,512,1024")
ap.add_argument("--rounds", type=int, default=64)
ap.add_argument("--T", type=int, default=1024)
ap.add_argument("--hq", type=int, default=28)
ap.add_argument("--hkv", type=int, default=4)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--json")
a = ap.parse_args()
hq, hkv, d = a.hq, a.hkv, 128


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


rows = []
for nq in [int(x) for x in a.nq.split(",")]:
    hist = a.rounds * a.T
    s = hist + nq
    k = torch.randn(s, hkv, d, device="cuda").bfloat16()
    v = torch.randn(s, hkv, d, device="cuda").bfloat16()
    q = torch.randn(nq, hq, d, device="cuda")
    qp = torch.arange(hist, s, device="cuda")
    kp = torch.arange(s, device="cuda")
    bounds = [(r * a.T, (r + 1) * a.T, r) for r in range(a.rounds)] + [(hist, s, a.rounds)]
    items = torch.from_numpy(build_round_items(bounds, 1024)).cuda()
    out = torch.empty(nq, hq, d, device="cuda")
    visible = nq * hist + nq * (nq + 1) / 2
    flop = 4.0 * hq * d * visible
    ms_plain = timed(lambda: kernels.prefill_attention(q, k, v, qp, kp, out=out), a.reps)
    ms_fused = timed(lambda: kernels.prefill_attention(q, k, v, qp, kp, items=items, n_bins=a.rounds, out=out),
                     a.reps)
    ms_score = timed(lambda: stats.round_scores(q, k, qp, kp, bounds, a.rounds, chunk=1024, exact=False), a.reps)
    ms_single = timed(lambda: kernels.prefill_attention(q, k, v, qp, kp, out=out, single_pass=True), a.reps)
    r = dict(n_q=nq, keys=s, hq=hq, hkv=hkv, ms_prefill=ms_plain, ms_prefill_fused_scoring=ms_fused,
             ms_separate_scorer=ms_score, ms_single_pass_bf16=ms_single,
             algo_tflops_single_pass=flop / ms_single / 1e9, algo_tflops=flop / ms_plain / 1e9,
             frac_bf16_peak=flop / ms_plain / 1e9 / PEAK_TF, issued_tflops=2 * flop / ms_plain / 1e9,
             fused_scoring_overhead=ms_fused / ms_plain - 1.0, peak_tflops=PEAK_TF)
    rows.append(r)
    print(json.dumps(r), flush=True)
if a.json:
    Path(a.json).write_text(json.dumps(rows, indent=1))
