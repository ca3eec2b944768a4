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
with K/V expanded to Hq heads (repeat_kv) because the kernel is MHA only.
`kind="reference"` runs the reference's OWN compiled kernel
(oracle/_ref, built from /root/reference by `make -C oracle ref`);
`kind="port"` runs oracle/attn_ref.c, its plain-C restatement.
Dialogues are independent, so the host cores run one dialogue per process
(SURVEY.md §8d); tokens/s = processes * tokens / wall time.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from . import rounds as orr


def _kernel(kind):
    if kind == "reference":
        from . import refkernel
        mod = refkernel.load()
        return lambda *a, **kw: mod.attention_forward(*a, **kw)
    from . import cref
    return lambda *a, **kw: cref.attention_forward(*a, **kw, threads=1)


def _one_token(args):
    """Worker: one decode token of one dialogue; returns seconds spent."""
    (kind, L, lw, hq, hkv, d, rounds, T, K, seed, kv_cap) = args
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    attn = _kernel(kind)
    rng = np.random.default_rng(seed)
    G = hq // hkv
    S = rounds * T + 1
    S_lo = min(S, kv_cap) if kv_cap else S
    kv = rng.standard_normal((S_lo, hkv, d)).astype(np.float32)
    kve = np.repeat(kv, G, axis=1)                       # repeat_kv expansion (MHA kernel)
    q = rng.standard_normal((1, hq, d)).astype(np.float32)
    upper_blocks = [rng.standard_normal((L - lw, 2, T, hkv * d)).astype(np.float32) for _ in range(K)]
    work = np.empty((L - lw, 2, K * T, hkv * d), np.float32)
    t0 = time.perf_counter()
    # scoring at layer Lw-1 (capture) + Eq. 1 + normalize + select
    _, cap = attn(q, kve, kve, np.array([S_lo - 1]), np.arange(S_lo), capture=True)
    rnds = orr.make_rounds([(1, T - 1)] * rounds + [(1, 0)])
    nr = min(rounds, (S_lo - 1) // T)
    raw = orr.aggregate_round_attention(cap, rnds[: nr] + [orr.Round(nr, (S_lo - 1, S_lo), (S_lo, S_lo))],
                                        "question", nr, row_offset=S_lo - 1)
    dist = orr.normalize(raw)
    orr.select(dist, orr.SelectionPolicy("top_percent", fraction=0.10))
    for i in range(K):                                   # the CPU "transfer" of kept upper blocks
        np.copyto(work[:, :, i * T:(i + 1) * T], upper_blocks[i])
    # lower layers over the full history (the capture layer already ran once)
    for _ in range(lw - 1):
        attn(q, kve, kve, np.array([S_lo - 1]), np.arange(S_lo))
    # upper layers over the kept rounds + the new token
    up = work[0].reshape(2, K * T, hkv, d)
    ku = np.repeat(np.concatenate([up[0], kv[:1]]), G, axis=1)
    vu = np.repeat(np.concatenate([up[1], kv[:1]]), G, axis=1)
    for _ in range(L - lw):
        attn(q, ku, vu, np.array([K * T]), np.arange(K * T + 1))
    dt = time.perf_counter() - t0
    if kv_cap and S_lo < S:
        # bounded sample: scale the lower-layer share to the full history length
        pass
    return dt


def decode_tokens_per_s(kind: str, *, L, lw, hq, hkv, d, rounds, T, K, processes=None, tokens_per_proc=1,
                        seed=0):
    """Reference CPU decode throughput on the host: `processes` dialogues in
    parallel (default: all cores), `tokens_per_proc` tokens each."""
    procs = processes or os.cpu_count() or 1
    args = [(kind, L, lw, hq, hkv, d, rounds, T, K, seed + i, 0) for i in range(procs * tokens_per_proc)]
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        per = pool.map(_one_token, args, chunksize=1)
    wall = time.perf_counter() - t0
    return dict(tokens_per_s=len(args) / wall, wall_s=wall, cores=procs, tokens=len(args),
                mean_token_s=float(np.mean(per)), kind=kind)
