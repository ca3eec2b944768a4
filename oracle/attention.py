"""ORACLE (test infrastructure only): the reference attention kernel contract.

Restates `pkg/src/roundkv/_attn_np.py:19-92` and the compiled twin
`pkg/src/roundkv/_attn_ext.pyx:20-116`:

* inputs coerced to C-contiguous float32 / int64 / bool (`_attn_np.py:26-47`);
* visibility `k_pos[j] <= q_pos[i]` and `allowed[j]` (`_attn_ext.pyx:43-48`);
* float64 logits `q.k / sqrt(d)`, max-subtracted exp, float64 weighted sum of
  values (`_attn_ext.pyx:51-80`), float32 output;
* capture: per-head probabilities summed over heads, then every row divided by
  its own sum (`_attn_ext.pyx:75-76,113-114`);
* a row with no visible key raises InvariantError (`_attn_ext.pyx:49-50,110`).

The reference is MHA only (`_attn_np.py:33-36`).  `attention_forward_gqa`
extends it with the HF `repeat_kv` convention (query head h reads key head
h // (Hq/Hkv)) by expanding K/V and calling the MHA restatement, which is the
parity convention fixed in SURVEY.md §7 hard part 7.
"""

from __future__ import annotations

import numpy as np

from paper_2502_15294_b200.errors import DomainError, InvariantError


def check_inputs(q, k, v, q_pos, k_pos, allowed, *, gqa=False):
    """Shape/dtype normalisation of `_attn_np.check_attention_inputs` (:19-47)."""
    q = np.ascontiguousarray(q, dtype=np.float32)
    k = np.ascontiguousarray(k, dtype=np.float32)
    v = np.ascontiguousarray(v, dtype=np.float32)
    if q.ndim != 3 or k.ndim != 3 or v.ndim != 3:
        raise DomainError("q, k, v must be (rows, heads, head_dim) arrays")
    if k.shape != v.shape:
        raise DomainError(f"key/value shape mismatch: {k.shape} vs {v.shape}")
    if gqa:
        ok = q.shape[2] == k.shape[2] and k.shape[1] > 0 and q.shape[1] % k.shape[1] == 0
    else:
        ok = q.shape[1:] == k.shape[1:]
    if not ok:
        raise DomainError(f"query heads {q.shape[1:]} do not match key heads {k.shape[1:]}")
    if q.shape[2] == 0:
        raise DomainError("head_dim must be positive")
    q_pos = np.ascontiguousarray(q_pos, dtype=np.int64)
    k_pos = np.ascontiguousarray(k_pos, dtype=np.int64)
    if q_pos.shape != (q.shape[0],) or k_pos.shape != (k.shape[0],):
        raise DomainError("position arrays must match q/k row counts")
    if allowed is not None:
        allowed = np.ascontiguousarray(allowed, dtype=bool)
        if allowed.shape != (k.shape[0],):
            raise DomainError("allowed mask must have one entry per key row")
    return q, k, v, q_pos, k_pos, allowed


def attention_forward(q, k, v, q_pos, k_pos, allowed=None, capture=False):
    """fp64 restatement of the reference kernel contract (MHA)."""
    q, k, v, q_pos, k_pos, allowed = check_inputs(q, k, v, q_pos, k_pos, allowed)
    return _forward(q, k, v, q_pos, k_pos, allowed, capture)


def attention_forward_gqa(q, k, v, q_pos, k_pos, allowed=None, capture=False):
    """GQA by expansion: repeat each key/value head Hq/Hkv times (repeat_kv)."""
    q, k, v, q_pos, k_pos, allowed = check_inputs(q, k, v, q_pos, k_pos, allowed, gqa=True)
    group = q.shape[1] // k.shape[1]
    if group > 1:
        k = np.repeat(k, group, axis=1)
        v = np.repeat(v, group, axis=1)
    return _forward(q, k, v, q_pos, k_pos, allowed, capture)


def _forward(q, k, v, q_pos, k_pos, allowed, capture):
    n, heads, d = q.shape
    s = k.shape[0]
    out = np.zeros((n, heads * d), dtype=np.float32)
    if n == 0:
        return out, (np.zeros((0, s)) if capture else None)
    vis = k_pos[None, :] <= q_pos[:, None]
    if allowed is not None:
        vis &= allowed[None, :]
    has_key = vis.any(axis=1)
    if not has_key.all():
        raise InvariantError(f"query row {int(np.argmin(has_key))} has no visible key")
    scale = 1.0 / np.sqrt(float(d))
    cap = np.zeros((n, s), dtype=np.float64) if capture else None
    q64 = q.astype(np.float64)
    k64 = k.astype(np.float64)
    v64 = v.astype(np.float64)
    for h in range(heads):
        logits = (q64[:, h, :] @ k64[:, h, :].T) * scale        # (n, s)
        logits = np.where(vis, logits, -np.inf)
        logits -= logits.max(axis=1, keepdims=True)
        w = np.exp(logits)
        w /= w.sum(axis=1, keepdims=True)
        out[:, h * d:(h + 1) * d] = (w @ v64[:, h, :]).astype(np.float32)
        if capture:
            cap += w
    if capture:
        cap /= cap.sum(axis=1, keepdims=True)
    return out, cap


def capture_pre(q, k, q_pos, k_pos, allowed=None):
    """engine.py:187-200 (Model._capture_pre, capture_mode="pre"): one softmax per
    query row over the head-summed fp64 logits sum_h q_h . k_h / (H sqrt(d)),
    masked keys excluded.  q (n, Hq, d); k (s, Hkv, d) with GQA heads expanded
    as repeat_kv (Hkv = Hq for the reference's MHA model).  Returns (n, s)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    hq, hkv, d = q.shape[1], k.shape[1], q.shape[2]
    k = np.repeat(k, hq // hkv, axis=1)
    logits = np.einsum("nhd,shd->ns", q, k) / (hq * np.sqrt(d))
    vis = np.asarray(k_pos)[None, :] <= np.asarray(q_pos)[:, None]
    if allowed is not None:
        vis = vis & np.asarray(allowed, dtype=bool)[None, :]
    logits = np.where(vis, logits, -np.inf)
    logits -= logits.max(axis=1, keepdims=True)
    w = np.exp(logits)
    return w / w.sum(axis=1, keepdims=True)


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """float32 values rounded to the nearest bf16 (round-to-nearest-even),
    returned as float32 — the identical inputs fed to both sides for bf16 parity."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    bits = x.view(np.uint32).astype(np.uint64)
    lsb = (bits >> 16) & 1
    rounded = ((bits + 0x7FFF + lsb) >> 16) << 16
    return rounded.astype(np.uint32).view(np.float32).reshape(x.shape)
