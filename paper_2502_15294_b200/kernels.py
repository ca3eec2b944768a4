"""Thin torch-facing wrappers over the librk decode / scoring entry points.

These take and return torch CUDA tensors (no host copies) and are what the
pipeline and the batched decode engine call on the hot path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .workspace import scratch


def kv_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.RK_BF16
    if t.dtype == torch.float32:
        return _lib.RK_F32
    raise TypeError(f"KV dtype {t.dtype} unsupported (float32, bfloat16)")


def decode_workspace(batch: int, hq: int, hkv: int, d: int, splits: int, device, tag: str = "decode"):
    nbytes = _lib.lib.rk_decode_workspace_bytes(batch, hq, hkv, d, max(1, splits))
    return scratch(nbytes, device, tag)


def decode_attention(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor, seq_len: torch.Tensor,
                     max_seq_len: int, *, k_new=None, v_new=None, items=None, n_items=None,
                     out: torch.Tensor | None = None, ws: torch.Tensor | None = None,
                     advance: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Batched single-token attention over contiguous per-dialogue caches.

    q (B, Hq, d) f32; k_cache/v_cache (B, S_cap, Hkv, d) or (S_cap, Hkv, d) for
    B == 1; seq_len (B,) int32 device = cached keys per dialogue; k_new/v_new
    (B, Hkv, d) appended at seq_len[b] and attended (seq_len not advanced).
    items (B, n_items_max, 3) int32 device enables the fused round scoring.
    """
    B, hq, d = q.shape
    if k_cache.dim() == 3:
        stride = 0
        hkv = k_cache.shape[1]
    else:
        stride = k_cache.stride(0)
        hkv = k_cache.shape[2]
    if out is None:
        out = torch.empty((B, hq, d), dtype=torch.float32, device=q.device)
    items_stride = 0 if items is None else items.shape[1]
    if ws is None:
        splits = items_stride if items is not None else 148
        ws = decode_workspace(B, hq, hkv, d, splits, q.device)
    _lib.call("rk_decode_attention", _lib.ptr(q), B, hq, d, _lib.ptr(k_cache), _lib.ptr(v_cache),
              kv_code(k_cache), hkv, stride, _lib.ptr(seq_len), int(max_seq_len), _lib.ptr(k_new),
              _lib.ptr(v_new), _lib.ptr(items), _lib.ptr(n_items), items_stride, _lib.ptr(out),
              _lib.ptr(advance), _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream))
    return out


def decode_attention_rows(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor, seq_len: torch.Tensor,
                          max_seq_len: int, row_active: torch.Tensor, *, k_new=None, v_new=None,
                          out: torch.Tensor | None = None, advance: torch.Tensor | None = None,
                          stream=None) -> torch.Tensor:
    """rk_decode_attention_rows: decode_attention over the rows with
    row_active[b] != 0 (int32 device); the other rows are not touched."""
    B, hq, d = q.shape
    stride, hkv = k_cache.stride(0), k_cache.shape[2]
    if out is None:
        out = torch.empty((B, hq, d), dtype=torch.float32, device=q.device)
    if row_active.dtype != torch.int32 or row_active.numel() != B:
        raise ValueError("row_active must be (B,) int32")
    _lib.call("rk_decode_attention_rows", _lib.ptr(q), B, hq, d, _lib.ptr(k_cache), _lib.ptr(v_cache),
              kv_code(k_cache), hkv, stride, _lib.ptr(seq_len), int(max_seq_len), _lib.ptr(k_new), _lib.ptr(v_new),
              _lib.ptr(row_active), _lib.ptr(out), _lib.ptr(advance), _lib.stream_ptr(stream))
    return out


def decode_plan(batch: int, hq: int, hkv: int, d: int, kv_dtype: torch.dtype, max_seq_len: int,
                cache_stride: int = 0, has_items: bool = False) -> int:
    """rk_decode_plan: C > 0 = cluster decode with C CTAs per (dialogue, kv-head),
    0 = persistent split-K + merge, -1 = generic split kernel."""
    code = _lib.RK_BF16 if kv_dtype == torch.bfloat16 else _lib.RK_F32
    return int(_lib.lib.rk_decode_plan(batch, hq, hkv, d, code, int(max_seq_len), int(cache_stride),
                                         int(has_items)))


def decode_scores_finalize(batch: int, hq: int, hkv: int, d: int, items: torch.Tensor, n_items: torch.Tensor,
                           n_bins: int, ws: torch.Tensor, active=None, raw: torch.Tensor | None = None,
                           kv_dtype: torch.dtype = torch.bfloat16, stream=None) -> torch.Tensor:
    """Per-dialogue raw round masses (B, n_bins) from the statistics a
    decode_attention(items=...) call left in `ws` (same kv dtype / shape)."""
    if raw is None:
        raw = torch.empty((batch, n_bins), dtype=torch.float64, device=items.device)
    code = _lib.RK_BF16 if kv_dtype == torch.bfloat16 else _lib.RK_F32
    _lib.call("rk_round_scores_finalize", batch, hq, hkv, d, code, items.shape[1], _lib.ptr(items),
              _lib.ptr(n_items), n_bins, _lib.ptr(active), _lib.ptr(raw), _lib.ptr(ws), _lib.stream_ptr(stream))
    return raw


def select_batch(raw: torch.Tensor, kind: str, *, v=0.1, k_top=0, kappa=1.0, normalize=True, stream=None):
    """rk_select_batch over rows of a (B, n) float64 device tensor.  Returns
    device (masses (B, n), kept (B, n) int32, meta (B, 3) int32 = n_kept,
    degenerate, status)."""
    raw = raw.contiguous()         # select_kernel offsets raw, masses and kept by the same ld
    B, n = raw.shape
    masses = torch.empty((B, n), dtype=torch.float64, device=raw.device)
    kept = torch.zeros((B, n), dtype=torch.int32, device=raw.device)
    meta = torch.zeros((3, B), dtype=torch.int32, device=raw.device)
    _lib.call("rk_select_batch", _lib.ptr(raw), n, n, B, 1 if normalize else 0, _lib.SEL_KINDS[kind],
              float(v), int(k_top), float(kappa), _lib.ptr(masses), _lib.ptr(kept), _lib.ptr(meta[0]),
              _lib.ptr(meta[1]), _lib.ptr(meta[2]), _lib.stream_ptr(stream))
    return masses, kept, meta


def select_batch_active(raw: torch.Tensor, policy, *, active: torch.Tensor | None = None, k_top: int = 0,
                        out=None, stream=None):
    """rk_select_batch_active: selection over each dialogue's active rounds (the
    drop policy's candidate set) for a SelectionPolicy-like `policy` (kind, v,
    fraction, kappa, min_rounds).  raw (B, n) float64 device, one mass per round;
    active (B, n) uint8 device or None.  Returns device (masses (B, n), kept
    ROUND IDS (B, n) int32, meta (3, B) int32 = n_kept, degenerate, status,
    margin (B,) float64); `out` = a previous return value to reuse."""
    raw = raw.contiguous()
    B, n = raw.shape
    if out is None:
        out = (torch.empty((B, n), dtype=torch.float64, device=raw.device),
               torch.zeros((B, n), dtype=torch.int32, device=raw.device),
               torch.zeros((3, B), dtype=torch.int32, device=raw.device),
               torch.zeros(B, dtype=torch.float64, device=raw.device))
    masses, kept, meta, margin = out
    if active is not None and (active.dtype != torch.uint8 or tuple(active.shape) != (B, n)
                               or not active.is_contiguous()):
        raise ValueError("active must be a contiguous (B, n) uint8 tensor")
    _lib.call("rk_select_batch_active", _lib.ptr(raw), n, n, B, _lib.ptr(active), 1, _lib.SEL_KINDS[policy.kind],
              float(policy.v), int(k_top), float(policy.fraction), int(policy.min_rounds), float(policy.kappa),
              _lib.ptr(masses), _lib.ptr(kept), _lib.ptr(meta[0]), _lib.ptr(meta[1]), _lib.ptr(meta[2]),
              _lib.ptr(margin), _lib.stream_ptr(stream))
    return out


def selection_margin(masses: torch.Tensor, kind: str, *, v=0.1, k_top=0, kappa=1.0, out=None, stream=None):
    """rk_selection_margin over rows of a (B, n) float64 device tensor of masses:
    the relative distance of the deciding masses from the decision threshold
    (top_percent: (m_(K) - m_(K+1)) / m_(K)).  Returns (B,) float64 device."""
    masses = masses.contiguous()
    B, n = masses.shape
    if out is None:
        out = torch.empty(B, dtype=torch.float64, device=masses.device)
    _lib.call("rk_selection_margin", _lib.ptr(masses), n, n, B, _lib.SEL_KINDS[kind], float(v), int(k_top),
              float(kappa), _lib.ptr(out), _lib.stream_ptr(stream))
    return out


def round_scores_exact(q: torch.Tensor, k_cache: torch.Tensor, q_pos: torch.Tensor, items: torch.Tensor,
                       n_bins: int, *, seq_len: torch.Tensor | None = None, n_items: torch.Tensor | None = None,
                       k_pos: torch.Tensor | None = None, active: torch.Tensor | None = None,
                       raw: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None,
                       capture_mode: str = "post") -> torch.Tensor:
    """Exact (fp64) Eq. 1 masses for B dialogues (rk_round_scores_exact; with
    capture_mode="pre" rk_round_scores_exact_pre, engine.py:187-200).

    q (B, n_q, Hq, d) f32; k_cache (B, S_cap, Hkv, d) with any batch stride
    (layer Lw-1 keys); q_pos (n_q,) int64 device; items (B, n_items_max, 3)
    int32 round-aligned (bin n_bins = the question) + n_items (B,) int32;
    seq_len (B,) int32 = visible keys per dialogue (None: S_cap); k_pos (S,)
    int64 or None (key j at position j).  Returns raw (B, n_active) float64."""
    B, n_q, hq, d = q.shape
    hkv = k_cache.shape[2]
    stride = k_cache.stride(0)
    n_out = n_bins if active is None else int(active.sum().item())
    if raw is None:
        raw = torch.empty((B, max(1, n_out)), dtype=torch.float64, device=q.device)
    if ws is None:
        nbytes = _lib.lib.rk_round_scores_exact_workspace_bytes(B, n_q, hq, items.shape[1], n_bins)
        ws = scratch(nbytes, q.device, "scores_exact")
    if capture_mode not in ("post", "pre"):
        raise ValueError(f"capture_mode {capture_mode!r}")
    entry = "rk_round_scores_exact" if capture_mode == "post" else "rk_round_scores_exact_pre"
    _lib.call(entry, _lib.ptr(q), B, n_q, hq, d, _lib.ptr(k_cache), kv_code(k_cache), hkv, stride,
              _lib.ptr(seq_len), k_cache.shape[1], _lib.ptr(q_pos), _lib.ptr(k_pos), _lib.ptr(items), items.shape[1],
              _lib.ptr(n_items), n_bins, _lib.ptr(active), max(1, n_out), _lib.ptr(raw), _lib.ptr(ws), ws.numel(),
              _lib.stream_ptr(stream))
    return raw


def advance_lengths(seq_len: torch.Tensor, delta: int = 1, stream=None) -> None:
    _lib.call("rk_advance_lengths", _lib.ptr(seq_len), seq_len.numel(), int(delta), _lib.stream_ptr(stream))


def select_device(raw: torch.Tensor, kind: str, *, v=0.1, k_top=0, kappa=1.0, normalize=True, stream=None):
    """rk_select on a device float64 vector; returns device (masses, ints) where
    ints = [kept positions (n) | n_kept | degenerate | status]."""
    n = raw.numel()
    masses = torch.empty(n, dtype=torch.float64, device=raw.device)
    ints = torch.zeros(n + 3, dtype=torch.int32, device=raw.device)
    base = ints.data_ptr()
    _lib.call("rk_select", _lib.ptr(raw), n, 1 if normalize else 0, _lib.SEL_KINDS[kind], float(v), int(k_top),
              float(kappa), _lib.ptr(masses), base, base + 4 * n, base + 4 * (n + 1), base + 4 * (n + 2),
              _lib.stream_ptr(stream))
    return masses, ints


def items_tensor(per_dialogue_bounds, chunk: int, device) -> tuple[torch.Tensor, torch.Tensor]:
    """Pack per-dialogue round-aligned items into (B, max_items, 3) + counts."""
    from .stats import build_round_items
    packs = [build_round_items(b, chunk) for b in per_dialogue_bounds]
    width = max(1, max(len(p) for p in packs))
    arr = np.zeros((len(packs), width, 3), dtype=np.int32)
    for i, p in enumerate(packs):
        arr[i, : len(p)] = p
    counts = np.array([len(p) for p in packs], dtype=np.int32)
    return torch.from_numpy(arr).to(device), torch.from_numpy(counts).to(device)


def prefill_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, q_pos: torch.Tensor, k_pos: torch.Tensor,
                      *, allowed: torch.Tensor | None = None, items: torch.Tensor | None = None, n_bins: int = 0,
                      active: torch.Tensor | None = None, out: torch.Tensor | None = None,
                      raw: torch.Tensor | None = None, bad_row: torch.Tensor | None = None,
                      single_pass: bool = False, stream=None):
    """Question-prefill attention on the tensor cores (rk_prefill_attention).

    q (n_q, Hq, 128) f32; k/v (S, Hkv, 128) bf16; q_pos (n_q,) / k_pos (S,)
    int64 device; allowed (S,) uint8 or None.  single_pass: the bf16 path (q and
    P rounded to bf16, one MMA pass each; ~1e-2 relative).  With `items` ((n_items, 3)
    int32 round-aligned (lo, hi, bin)) and n_bins > 0 the Eq. 1 masses of the
    active bins come back in `raw` (float64) from the same pass.  Returns
    (out (n_q, Hq, 128) f32, raw or None, bad_row (1,) int32 device).
    """
    n_q, hq, d = q.shape
    s, hkv = k.shape[0], k.shape[1]
    dev = q.device
    if out is None:
        out = torch.empty((n_q, hq, d), dtype=torch.float32, device=dev)
    n_items = 0 if items is None else items.shape[0]
    if n_bins > 0 and raw is None:
        n_out = n_bins if active is None else int(active.sum().item())
        raw = torch.zeros(max(1, n_out), dtype=torch.float64, device=dev)
    if bad_row is None:
        bad_row = torch.empty(1, dtype=torch.int32, device=dev)
    nbytes = _lib.lib.rk_prefill_workspace_bytes(n_q, hq, hkv, s, d, n_items, n_bins if raw is not None else 0)
    ws = scratch(nbytes, dev, "prefill")
    _lib.call("rk_prefill_attention", _lib.ptr(q), n_q, hq, d, _lib.ptr(k), _lib.ptr(v), kv_code(k), s, hkv,
              _lib.ptr(q_pos), _lib.ptr(k_pos), _lib.ptr(allowed), _lib.ptr(items), n_items,
              n_bins if raw is not None else 0, _lib.ptr(active), _lib.ptr(out), _lib.ptr(raw), _lib.ptr(bad_row),
              _lib.ptr(ws), ws.numel(), _lib.RK_PREFILL_SINGLE_PASS if single_pass else 0, _lib.stream_ptr(stream))
    return out, raw, bad_row


# ---------------------------------------------------------------- layer body (proj.cu)
def pack_weight(w: torch.Tensor, stream=None) -> torch.Tensor:
    """(k, n) weight of x @ W (fp32 or bf16, device) -> W^T [n_pad][k] bf16
    (n padded to 128 with zero rows), the K-major tcgen05 A operand."""
    k, n = w.shape
    w = w.contiguous()
    out = torch.empty(_lib.lib.rk_packed_weight_bytes(k, n) // 2, dtype=torch.bfloat16, device=w.device)
    _lib.call("rk_pack_weight", _lib.ptr(w), kv_code(w), k, n, _lib.ptr(out), _lib.stream_ptr(stream))
    return out


def proj_workspace(m: int, k: int, n: int, device) -> torch.Tensor:
    """A zeroed split-K workspace for one stream's projections of m rows
    (k inputs, n outputs); the kernels leave it zeroed."""
    return torch.zeros(max(256, int(_lib.lib.rk_proj_workspace_bytes(m, k, n))), dtype=torch.uint8, device=device)


def _proj_ws(ws, m, k, n, device, tag):
    need = _lib.lib.rk_proj_workspace_bytes(m, k, n)
    if ws is None or ws.numel() < need:
        ws = scratch(need, device, tag)
    return ws


def qkv_rope(x: torch.Tensor, w_qkv_packed: torch.Tensor, hq: int, hkv: int, d: int, pos: torch.Tensor,
             freq: torch.Tensor, q_out: torch.Tensor, k_out: torch.Tensor, v_out: torch.Tensor,
             kv_row_stride: int | None = None, ws: torch.Tensor | None = None, stream=None) -> None:
    """q, k, v = RoPE(x W_q), RoPE(x W_k), x W_v for m rows of x (m, d_model) f32;
    k / v rows in k_out's dtype (bf16 or fp32 caches)."""
    m, dm = x.shape
    if k_out.dtype != v_out.dtype:
        raise ValueError("k_out and v_out must share a dtype")
    ws = _proj_ws(ws, m, dm, (hq + 2 * hkv) * d, x.device, "proj")
    _lib.call("rk_qkv_rope_kv", _lib.ptr(x), m, dm, _lib.ptr(w_qkv_packed), hq, hkv, d, _lib.ptr(pos),
              _lib.ptr(freq), _lib.ptr(q_out), _lib.ptr(k_out), _lib.ptr(v_out), kv_code(k_out),
              int(hkv * d if kv_row_stride is None else kv_row_stride), _lib.ptr(ws), ws.numel(),
              _lib.stream_ptr(stream))


def out_proj(a: torch.Tensor, w_o_packed: torch.Tensor, resid: torch.Tensor, ws: torch.Tensor | None = None,
             stream=None, row_active: torch.Tensor | None = None) -> None:
    """resid (m, d_model) += a (m, k) W_o (only the rows with row_active != 0 when given)."""
    m, k = a.shape
    ws = _proj_ws(ws, m, k, resid.shape[1], a.device, "proj")
    _lib.call("rk_out_proj_rows", _lib.ptr(a), m, k, _lib.ptr(w_o_packed), resid.shape[1], _lib.ptr(resid),
              _lib.ptr(row_active), _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream))


def lm_head(x: torch.Tensor, emb_packed: torch.Tensor, vocab: int, emb: torch.Tensor, x_next: torch.Tensor,
            tokens: torch.Tensor | None, pos: torch.Tensor | None, tokens_log: torch.Tensor | None = None,
            log_stride: int = 0, ws: torch.Tensor | None = None, stream=None,
            row_active: torch.Tensor | None = None, log_pos_base: int = -1) -> None:
    """tokens = first argmax of x E^T; x_next = E[tokens]; pos += 1 (when given);
    rows with row_active == 0 (when given) are left unchanged."""
    m, dm = x.shape
    need = _lib.lib.rk_lm_head_workspace_bytes(m, vocab, dm)
    if ws is None or ws.numel() < need:
        ws = scratch(need, x.device, "lm_head")
    _lib.call("rk_lm_head_rows", _lib.ptr(x), m, dm, _lib.ptr(emb_packed), vocab, _lib.ptr(emb), _lib.ptr(x_next),
              _lib.ptr(tokens), _lib.ptr(pos), _lib.ptr(tokens_log), int(log_stride), _lib.ptr(row_active),
              int(log_pos_base), _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream))


def small_qkv_rope(x: torch.Tensor, w_q: torch.Tensor, w_k: torch.Tensor, w_v: torch.Tensor, heads: int,
                   positions: torch.Tensor, freq: torch.Tensor, stream=None):
    """The drop-in model's q, k = RoPE(x W_q), RoPE(x W_k); v = x W_v (float32,
    rk_small_qkv_rope): returns q (n, heads, d_k), k (n, d_model), v (n, d_model)."""
    x = x.contiguous()
    n, dm = x.shape
    q = torch.empty((n, dm), dtype=torch.float32, device=x.device)
    k = torch.empty_like(q)
    v = torch.empty_like(q)
    pos = positions.to(torch.int64).contiguous()
    _lib.call("rk_small_qkv_rope", _lib.ptr(x), n, dm, _lib.ptr(w_q), _lib.ptr(w_k), _lib.ptr(w_v), heads,
              _lib.ptr(pos), _lib.ptr(freq), _lib.ptr(q), _lib.ptr(k), _lib.ptr(v), _lib.stream_ptr(stream))
    return q.view(n, heads, dm // heads), k, v


def small_out_proj(a: torch.Tensor, w_o: torch.Tensor, x: torch.Tensor, stream=None) -> torch.Tensor:
    """x + a W_o (float32, rk_small_out_proj), a new tensor."""
    a, x = a.contiguous(), x.contiguous()
    out = torch.empty_like(x)
    _lib.call("rk_small_out_proj", _lib.ptr(a), a.shape[0], a.shape[1], _lib.ptr(w_o), _lib.ptr(x), _lib.ptr(out),
              _lib.stream_ptr(stream))
    return out


def small_logits(x: torch.Tensor, emb: torch.Tensor, want_logits: bool = True, stream=None):
    """(logits = x E^T or None, first-max argmax per row) (float32, rk_small_logits)."""
    x = x.contiguous()
    n, dm = x.shape
    logits = torch.empty((n, emb.shape[0]), dtype=torch.float32, device=x.device) if want_logits else None
    am = torch.empty(n, dtype=torch.int32, device=x.device)
    _lib.call("rk_small_logits", _lib.ptr(x), n, dm, _lib.ptr(emb), emb.shape[0], _lib.ptr(logits), _lib.ptr(am),
              _lib.stream_ptr(stream))
    return logits, am


def capture_pre(q: torch.Tensor, k: torch.Tensor, q_pos: torch.Tensor, k_pos: torch.Tensor,
                allowed: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """capture_mode="pre" score matrix (rk_capture_pre): q (n, H, d_k), k (s, H*d_k)
    float32 -> (n, s) float64 softmax of the head-summed logits / (H sqrt(d_k))."""
    q = q.contiguous().to(torch.float32)
    n, heads, dk = q.shape
    k = k.contiguous().to(torch.float32)
    s = k.shape[0]
    out = torch.empty((n, s), dtype=torch.float64, device=q.device)
    qp = q_pos.to(device=q.device, dtype=torch.int64).contiguous()
    kp = k_pos.to(device=q.device, dtype=torch.int64).contiguous()
    al = None if allowed is None else allowed.to(device=q.device, dtype=torch.uint8).contiguous()
    _lib.call("rk_capture_pre", _lib.ptr(q), n, heads, dk, _lib.ptr(k), s, _lib.ptr(qp), _lib.ptr(kp), _lib.ptr(al),
              _lib.ptr(out), _lib.stream_ptr(stream))
    return out


def decode_step_supported(batch: int, hq: int, hkv: int, head_dim: int, kv_dtype=torch.bfloat16) -> bool:
    """Whether rk_decode_step (the persistent whole-step kernel) covers this shape."""
    code = {torch.bfloat16: _lib.RK_BF16, torch.float32: _lib.RK_F32}.get(kv_dtype, -1)
    return bool(_lib.lib.rk_decode_step_supported(batch, hq, hkv, head_dim, code))


def decode_step_workspace(batch: int, num_layers: int, hq: int, hkv: int, head_dim: int, vocab: int,
                          device) -> torch.Tensor:
    """The zeroed workspace rk_decode_step reuses across launches (monotonic counters)."""
    need = _lib.lib.rk_decode_step_workspace_bytes(batch, num_layers, hq, hkv, head_dim, vocab)
    return torch.zeros(max(256, int(need)), dtype=torch.uint8, device=device)


def decode_step_args(x, lower, upper, lower_len, upper_len, pos, freq, w_qkv_table, w_o_table, emb_packed, emb,
                     hq: int, hkv: int, watershed: int, ws, tokens=None, tokens_log=None, log_stride: int = 0,
                     vocab: int | None = None):
    """rk_decode_step_args for one token step over all layers (see the header):
    lower (B, Lw, 2, S_lo, hkv, d), upper (B, L - Lw, 2, S_up, hkv, d) bf16;
    w_*_table: int64 device tensors of the layers' packed-weight addresses."""
    B, d = x.shape[0], lower.shape[-1]
    a = _lib.DecodeStepArgs()
    a.batch, a.num_layers, a.watershed = B, int(w_qkv_table.numel()), int(watershed)
    a.hq, a.hkv, a.head_dim, a.vocab = hq, hkv, d, int(emb.shape[0] if vocab is None else vocab)
    a.x = _lib.ptr(x)
    a.lower, a.lower_seq = _lib.ptr(lower), int(lower.shape[3])
    a.upper, a.upper_seq = _lib.ptr(upper), int(upper.shape[3])
    a.lower_len, a.upper_len, a.pos, a.rope_freq = (_lib.ptr(lower_len), _lib.ptr(upper_len), _lib.ptr(pos),
                                                     _lib.ptr(freq))
    a.w_qkv, a.w_o = _lib.ptr(w_qkv_table), _lib.ptr(w_o_table)
    a.emb_packed, a.emb = _lib.ptr(emb_packed), _lib.ptr(emb)
    a.tokens, a.tokens_log, a.log_stride = _lib.ptr(tokens), _lib.ptr(tokens_log), int(log_stride)
    a.workspace, a.workspace_bytes = _lib.ptr(ws), ws.numel()
    return a


def decode_step(args, stream=None) -> None:
    """One persistent launch of the whole decode token step (rk_decode_step)."""
    import ctypes
    _lib.call("rk_decode_step", ctypes.addressof(args), _lib.stream_ptr(stream))


def embed(tokens: torch.Tensor, emb: torch.Tensor, x: torch.Tensor, stream=None) -> None:
    """x (m, d_model) f32 = emb[tokens] (bf16 table)."""
    _lib.call("rk_embed", _lib.ptr(tokens), tokens.numel(), _lib.ptr(emb), emb.shape[1], _lib.ptr(x),
              _lib.stream_ptr(stream))


def rope_rows(qkv: torch.Tensor, hq: int, hkv: int, d: int, pos: torch.Tensor, freq: torch.Tensor,
              q_out: torch.Tensor, k_out: torch.Tensor, v_out: torch.Tensor, kv_row_stride: int,
              rows_per_group: int, kv_group_stride: int, stream=None) -> None:
    """RoPE + bf16 cache append of m projected rows (qkv (m, (hq+2hkv)d) f32)."""
    _lib.call("rk_rope_rows", _lib.ptr(qkv), qkv.shape[0], hq, hkv, d, _lib.ptr(pos), _lib.ptr(freq),
              _lib.ptr(q_out), _lib.ptr(k_out), _lib.ptr(v_out), int(kv_row_stride), int(rows_per_group),
              int(kv_group_stride), _lib.stream_ptr(stream))
