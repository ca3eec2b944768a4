"""ORACLE (test infrastructure only): one serving turn of the batched engine
(paper_2502_15294_b200/decode_engine.py) restated on the CPU in NumPy float64,
for the engine's GQA-shaped version of the reference model.

Follows the reference step by step:
  * forward_range per layer, engine.py:244-267: q, k = RoPE(x W_q), RoPE(x W_k)
    (interleaved pairs, float64 trig, fp32 result, engine.py:175-185); v = x W_v;
    append; attention over the layer's cache (_attn_ext.pyx:41-80: fp64
    logits / softmax / weighted sum); x += out W_o — with GQA (query head h
    reads kv-head h // (Hq / Hkv), HF repeat_kv) and the cached K/V rounded to
    bf16 as the engine stores them;
  * the capture at layer L_w-1 + Eq. 1 + normalize + select (pipeline.py:225-251,
    stats.py:59-115, selection.py:87-97);
  * upper layers over the kept rounds' blocks + the turn's rows (splice ==
    mask, engine.py:94-112);
  * the greedy decode (pipeline.py:298-313): SEP, then first-max argmax of the
    tied logits (engine.py:270-271) for a fixed number of forwards.
Weights are the engine's bf16 weights (DecodeModel.host_weights()).
"""

from __future__ import annotations

import numpy as np

from . import rounds as orr
from .attention import capture_pre, round_to_bf16

SEP_TOKEN = 256


def rope(x, positions, freq):
    """(rows, heads, d) rotated by absolute position (engine.py:175-185)."""
    ang = np.asarray(positions, dtype=np.float64)[:, None] * freq[None, :]
    cos, sin = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    x64 = x.astype(np.float64)
    ev, od = x64[..., 0::2], x64[..., 1::2]
    out = np.empty_like(x64)
    out[..., 0::2] = ev * cos - od * sin
    out[..., 1::2] = ev * sin + od * cos
    return out.astype(np.float32)


def attend(q, K, V, capture=False):
    """One query row per head over all cached keys (decode: every key visible):
    q (Hq, d), K/V (S, Hkv, d) -> out (Hq*d,) fp32 and the head-summed,
    row-normalised capture (S,) when asked (_attn_ext.pyx:41-80,113-114)."""
    hq, d = q.shape
    G = hq // K.shape[1]
    Ke = np.repeat(K.astype(np.float64), G, axis=1)
    Ve = np.repeat(V.astype(np.float64), G, axis=1)
    s = np.einsum("hd,shd->hs", q.astype(np.float64), Ke) * (1.0 / np.sqrt(float(d)))
    s -= s.max(axis=1, keepdims=True)
    w = np.exp(s)
    p = w / w.sum(axis=1, keepdims=True)
    out = np.einsum("hs,shd->hd", p, Ve).astype(np.float32).reshape(-1)
    cap = None
    if capture:
        cap = p.sum(axis=0)
        cap = cap / cap.sum()
    return out, cap


class TurnOracle:
    """State of one dialogue for one turn: lower caches (history), the kept
    rounds' upper blocks are given after selection."""

    def __init__(self, weights, hq, hkv, d, freq, kv_bf16=True):
        self.w = weights
        self.hq, self.hkv, self.d = hq, hkv, d
        self.freq = freq
        self.L = len(weights["wq"])
        self.kv_round = round_to_bf16 if kv_bf16 else (lambda a: np.asarray(a, dtype=np.float32))

    def layer(self, l, x, pos, K, V, capture=False):
        """x (D,) fp32; K/V caches (S, Hkv, d) of layer l BEFORE the append.
        Returns (x', K', V', capture-or-None, q)."""
        w = self.w
        x64 = x.astype(np.float64)
        q = (x64 @ w["wq"][l]).astype(np.float32).reshape(1, self.hq, self.d)
        k = (x64 @ w["wk"][l]).astype(np.float32).reshape(1, self.hkv, self.d)
        v = (x64 @ w["wv"][l]).astype(np.float32).reshape(1, self.hkv, self.d)
        q = rope(q, [pos], self.freq)[0]
        k = self.kv_round(rope(k, [pos], self.freq))      # the cache's dtype (bf16 or the reference's fp32)
        v = self.kv_round(v)
        K = np.concatenate([K, k])
        V = np.concatenate([V, v])
        out, cap = attend(q, K, V, capture)
        x = (x64 + out.astype(np.float64) @ w["wo"][l]).astype(np.float32)
        return x, K, V, cap, q

    def logits(self, x):
        return x.astype(np.float64) @ self.w["emb"].astype(np.float64).T


def run_turn(oracle: TurnOracle, lower_k, lower_v, upper_blocks_fn, question_token, hist, round_tokens, n_rounds,
             lw, policy, decode_steps, capture_mode="post", active=None):
    """One turn of one dialogue.  lower_k/v: [lw] arrays (hist, Hkv, d);
    upper_blocks_fn(kept) -> [L-lw] pairs (K, V) of the kept rounds' keys in
    the engine's slot order.  capture_mode "pre": the head-summed-logit capture
    (engine.py:187-200); active: the candidate rounds (the drop policy's
    active_rounds, pipeline.py:238-245; None = every round).
    Returns dict(kept, raw, masses, answer, x)."""
    L = oracle.L
    T = round_tokens
    x = oracle.w["emb"][question_token].astype(np.float32)
    pos = hist
    lk = [k.copy() for k in lower_k]
    lv = [v.copy() for v in lower_v]
    cap = None
    for l in range(lw):
        x, lk[l], lv[l], c, q = oracle.layer(l, x, pos, lk[l], lv[l], capture=(l == lw - 1))
        if c is not None:
            cap = c
            if capture_mode == "pre":
                cap = capture_pre(q[None], lk[l], [pos], np.arange(lk[l].shape[0]))[0]
    act = list(range(n_rounds)) if active is None else list(active)
    raw = np.array([cap[r * T:(r + 1) * T].sum() for r in act])
    dist = orr.normalize(raw, round_indices=act)
    kept = orr.select(dist, policy)
    uk, uv = [], []
    blocks = upper_blocks_fn(kept)
    for u, l in enumerate(range(lw, L)):
        K, V = blocks[u]
        x, K, V, _, _ = oracle.layer(l, x, pos, K, V)
        uk.append(K)
        uv.append(V)
    answer = [SEP_TOKEN]
    x = oracle.w["emb"][SEP_TOKEN].astype(np.float32)
    pos = hist + 1
    gaps = []
    for t in range(decode_steps):
        for l in range(L):
            if l < lw:
                x, lk[l], lv[l], _, _ = oracle.layer(l, x, pos, lk[l], lv[l])
            else:
                u = l - lw
                x, uk[u], uv[u], _, _ = oracle.layer(l, x, pos, uk[u], uv[u])
        z = oracle.logits(x)
        top = np.sort(z)[::-1]
        gaps.append(float(top[0] - top[1]))
        nxt = int(np.argmax(z))
        answer.append(nxt)
        x = oracle.w["emb"][nxt].astype(np.float32)
        pos += 1
    return dict(kept=kept, raw=raw, masses=np.asarray(dist.masses), answer=answer, x=x, logit_gaps=gaps)
