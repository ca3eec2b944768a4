"""ORACLE (test infrastructure only): the reference's CPU path, timed on the
host cores, for bench.py's `cpu_baseline` and `--impl reference` legs.

Composition of one decode token of one dialogue, exactly as BASELINE.md §3
prescribes for the GQA configs (the reference has no GQA and a full pipeline
at 16K-128K tokens is infeasible on the CPU):
  * Lw   x attention_forward over the full history (+ the new token),
  * L-Lw x attention_forward over the kept rounds (+ the new token),
  * one capture call at layer Lw-1 + aggregate_round_attention + normalize +
    select (stats.py:59-115, selection.py:87-97),
  * np.copyto of the kept rounds' upper blocks (the CPU "transfer"),
with K/V expanded to Hq heads (repeat_kv) because the kernel is MHA only, and
KV in float32 — the reference's storage precision (_attn_np.py:26-28): it
reads 2x the bytes of the GPU's bf16 KV.

`kind="reference"` runs the reference package itself — its public
`backend.attention_forward` (the compiled `_attn_ext` kernel), `stats` and
`selection` — staged from /root/reference into oracle/_ref by
`make -C oracle ref`; this process never imports the product package.
`kind="port"` runs oracle/attn_ref.c (the kernel's plain-C restatement) with
the oracle's restated Eq. 1 / selection.

Dialogues are independent, so the host cores run one dialogue per process
(SURVEY.md §8d).  Every worker generates its inputs first, then all workers
meet at a barrier and time only the decode tokens: tokens/s = all tokens /
(last worker's end - first worker's start), data generation excluded.
"""

from __future__ import annotations

import math
import multiprocessing as mp
import os
import time

import numpy as np

_BARRIER = None


def _init(barrier):
    global _BARRIER
    _BARRIER = barrier


def _api(kind):
    """(attention_forward, aggregate, normalize, select, policy, Round) of the arm."""
    if kind == "reference":
        from . import refkernel
        rk = refkernel.load_package()
        import roundkv.backend as be
        import roundkv.conversation as conv
        import roundkv.selection as sel
        import roundkv.stats as st
        assert be.BACKEND_NAME == "ext" and rk.BACKEND_NAME == "ext"
        return (be.attention_forward, st.aggregate_round_attention, st.normalize, sel.select,
                sel.SelectionPolicy("top_percent", fraction=0.10), conv.Round)
    from . import cref
    from . import rounds as orr
    return (lambda *a, **kw: cref.attention_forward(*a, **kw, threads=1), orr.aggregate_round_attention,
            orr.normalize, orr.select, orr.SelectionPolicy("top_percent", fraction=0.10), orr.Round)


def _worker(args):
    """One dialogue: generate inputs, wait for every worker, time `tokens`
    decode tokens.  Returns (t_start, t_end, tokens)."""
    (kind, L, lw, hq, hkv, d, rounds, T, K, seed, tokens) = args
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    attn, aggregate, normalize, select, policy, Round = _api(kind)
    rng = np.random.default_rng(seed)
    G = hq // hkv
    S = rounds * T + 1
    kv = rng.standard_normal((S, hkv, d), dtype=np.float32)
    kve = np.repeat(kv, G, axis=1)                       # repeat_kv expansion (MHA kernel)
    q = rng.standard_normal((1, hq, d), dtype=np.float32)
    upper_blocks = [rng.standard_normal((L - lw, 2, T, hkv * d), dtype=np.float32) for _ in range(K)]
    work = np.empty((L - lw, 2, K * T, hkv * d), np.float32)
    rnds = [Round(m, (m * T, m * T + 1), (m * T + 1, (m + 1) * T)) for m in range(rounds)]
    rnds.append(Round(rounds, (S - 1, S), (S, S)))
    pos_lo = np.arange(S)
    up = work[0].reshape(2, K * T, hkv, d)
    ku = np.repeat(np.concatenate([up[0], kv[:1]]), G, axis=1)
    vu = np.repeat(np.concatenate([up[1], kv[:1]]), G, axis=1)
    pos_up = np.arange(K * T + 1)
    if _BARRIER is not None:
        _BARRIER.wait()
    t0 = time.perf_counter()
    for _ in range(tokens):
        # scoring at layer Lw-1 (capture) + Eq. 1 + normalize + select
        _, cap = attn(q, kve, kve, np.array([S - 1]), pos_lo, capture=True)
        raw = aggregate(cap, rnds, "question", rounds, row_offset=S - 1)
        select(normalize(raw), policy)
        for i in range(K):                               # the CPU "transfer" of kept upper blocks
            np.copyto(work[:, :, i * T:(i + 1) * T], upper_blocks[i])
        for _ in range(lw - 1):                          # the other lower layers over the full history
            attn(q, kve, kve, np.array([S - 1]), pos_lo)
        for _ in range(L - lw):                          # upper layers over the kept rounds + the new token
            attn(q, ku, vu, np.array([K * T]), pos_up)
    return t0, time.perf_counter(), tokens


def kept_count(rounds: int, fraction: float = 0.10, min_rounds: int = 1) -> int:
    """K of select_top_percent (selection.py:23,93), stated without importing any package."""
    return min(rounds, max(min_rounds, math.ceil(fraction * rounds - 1e-9)))


def decode_tokens_per_s(kind: str, *, L, lw, hq, hkv, d, rounds, T, K, processes=None, tokens_per_proc=1,
                        seed=0):
    """Reference CPU decode throughput on the host: `processes` dialogues in
    parallel (default: all cores), `tokens_per_proc` timed tokens each."""
    procs = processes or os.cpu_count() or 1
    args = [(kind, L, lw, hq, hkv, d, rounds, T, K, seed + i, tokens_per_proc) for i in range(procs)]
    ctx = mp.get_context("fork")
    barrier = ctx.Barrier(procs)
    t_wall = time.perf_counter()
    with ctx.Pool(procs, initializer=_init, initargs=(barrier,)) as pool:
        per = pool.map(_worker, args, chunksize=1)
    wall = time.perf_counter() - t_wall
    start = min(p[0] for p in per)
    end = max(p[1] for p in per)
    tokens = sum(p[2] for p in per)
    out = dict(tokens_per_s=tokens / (end - start), timed_s=end - start, wall_s=wall, cores=procs, tokens=tokens,
               mean_token_s=float(np.mean([(p[1] - p[0]) / p[2] for p in per])), kind=kind)
    if kind == "reference":
        from . import refkernel
        out["kernel"] = refkernel.kernel_identity()
    return out
