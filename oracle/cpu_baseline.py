"""ORACLE (test infrastructure only): the reference's CPU path, timed on the
host cores, for bench.py's `cpu_baseline` and `--impl reference` legs.

Composition of one decode token of one dialogue, as BASELINE.md §3 prescribes
for the GQA configs (the reference has no GQA and a full pipeline at 16K-128K
tokens is infeasible on the CPU), with the model's layer body of
forward_range (engine.py:244-267) around every attention call:
  * per layer: q, k = RoPE(x W_q), RoPE(x W_k), v = x W_v (float32 BLAS; the
    reference's own Model._rope for kind="reference"), attention, x += out W_o;
    after the last layer the tied logits x E^T and the first argmax
    (engine.py:270-271, pipeline.py:308); the float32 weights are allocated
    once in the parent and shared read-only by the forked workers,
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
_WEIGHTS: dict = {}


def _weights(L, hq, hkv, d, vocab=258):
    """float32 weights of the config's shape (values irrelevant to timing),
    created once per process tree before the workers fork."""
    key = (L, hq, hkv, d)
    if key not in _WEIGHTS:
        D = hq * d
        w = 1.0 / math.sqrt(D)
        _WEIGHTS.clear()
        _WEIGHTS[key] = dict(
            wq=np.full((L, D, hq * d), w, np.float32), wk=np.full((L, D, hkv * d), w, np.float32),
            wv=np.full((L, D, hkv * d), w, np.float32), wo=np.full((L, hq * d, D), w / 8, np.float32),
            emb=np.full((vocab, D), 0.01, np.float32))
    return _WEIGHTS[key]


def _init(barrier):
    global _BARRIER
    _BARRIER = barrier


def _rope_fn(kind, d):
    """RoPE of (rows, heads, d) at absolute positions: the reference's own
    Model._rope for kind="reference" (engine.py:175-185), else its restatement."""
    freq = 10000.0 ** (-np.arange(d // 2, dtype=np.float64) * 2.0 / d)      # engine.py:162-164
    if kind == "reference":
        import roundkv.engine as eng

        class _Self:
            _rope_freq = freq
        return lambda x, pos: eng.Model._rope(_Self, x, pos)

    def rope(x, pos):
        ang = pos[:, None].astype(np.float64) * freq[None, :]
        c, s_ = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
        x64 = x.astype(np.float64)
        out = np.empty_like(x64)
        out[..., 0::2] = x64[..., 0::2] * c - x64[..., 1::2] * s_
        out[..., 1::2] = x64[..., 0::2] * s_ + x64[..., 1::2] * c
        return out.astype(np.float32)
    return rope


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
    (kind, L, lw, hq, hkv, d, rounds, T, K, seed, tokens, model) = args
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    attn, aggregate, normalize, select, policy, Round = _api(kind)
    W = _WEIGHTS.get((L, hq, hkv, d)) if model else None
    rope = _rope_fn(kind, d)
    rng = np.random.default_rng(seed)
    G = hq // hkv
    S = rounds * T + 1
    kv = rng.standard_normal((S, hkv, d), dtype=np.float32)
    kve = np.repeat(kv, G, axis=1)                       # repeat_kv expansion (MHA kernel)
    q = rng.standard_normal((1, hq, d), dtype=np.float32)
    x = rng.standard_normal((1, hq * d), dtype=np.float32)
    upper_blocks = [rng.standard_normal((L - lw, 2, T, hkv * d), dtype=np.float32) for _ in range(K)]
    work = np.empty((L - lw, 2, K * T, hkv * d), np.float32)
    rnds = [Round(m, (m * T, m * T + 1), (m * T + 1, (m + 1) * T)) for m in range(rounds)]
    rnds.append(Round(rounds, (S - 1, S), (S, S)))
    pos_lo = np.arange(S)
    pos_q = np.array([S - 1])
    up = work[0].reshape(2, K * T, hkv, d)
    ku = np.repeat(np.concatenate([up[0], kv[:1]]), G, axis=1)
    vu = np.repeat(np.concatenate([up[1], kv[:1]]), G, axis=1)
    pos_up = np.arange(K * T + 1)

    def body(l, att_k, att_v, qpos, kpos, capture=False):
        """forward_range's layer body (engine.py:244-267) around the attention call."""
        nonlocal x
        qq = q
        if W is not None:
            qq = rope((x @ W["wq"][l]).reshape(1, hq, d), pos_q)
            rope((x @ W["wk"][l]).reshape(1, hkv, d), pos_q)      # the new key (appended in the reference)
            x @ W["wv"][l]
        out, cap = attn(qq, att_k, att_v, qpos, kpos, capture=capture)
        if W is not None:
            x = x + out.reshape(1, -1) @ W["wo"][l]
        return cap

    if _BARRIER is not None:
        _BARRIER.wait()
    t0 = time.perf_counter()
    for _ in range(tokens):
        for l in range(lw - 1):                          # the lower layers over the full history
            body(l, kve, kve, pos_q, pos_lo)
        # layer Lw-1 with the capture (scoring) + Eq. 1 + normalize + select
        cap = body(lw - 1, kve, kve, pos_q, pos_lo, capture=True)
        raw = aggregate(cap, rnds, "question", rounds, row_offset=S - 1)
        select(normalize(raw), policy)
        for i in range(K):                               # the CPU "transfer" of kept upper blocks
            np.copyto(work[:, :, i * T:(i + 1) * T], upper_blocks[i])
        for l in range(lw, L):                           # upper layers over the kept rounds + the new token
            body(l, ku, vu, np.array([K * T]), pos_up)
        if W is not None:
            int(np.argmax(x @ W["emb"].T))               # tied logits + first argmax
    return t0, time.perf_counter(), tokens


def kept_count(rounds: int, fraction: float = 0.10, min_rounds: int = 1) -> int:
    """K of select_top_percent (selection.py:23,93), stated without importing any package."""
    return min(rounds, max(min_rounds, math.ceil(fraction * rounds - 1e-9)))


def decode_tokens_per_s(kind: str, *, L, lw, hq, hkv, d, rounds, T, K, processes=None, tokens_per_proc=1,
                        seed=0, model=True):
    """Reference CPU decode throughput on the host: `processes` dialogues in
    parallel (default: all cores), `tokens_per_proc` timed tokens each; with
    `model` every layer also runs its projections (float32 BLAS, weights
    shared by the forked workers)."""
    procs = processes or os.cpu_count() or 1
    if model:
        _weights(L, hq, hkv, d)
    args = [(kind, L, lw, hq, hkv, d, rounds, T, K, seed + i, tokens_per_proc, model) for i in range(procs)]
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
