"""Attention kernel backend — the reference's plug-in point, CUDA only.

Mirrors `pkg/src/roundkv/backend.py:21-47`: exports `BACKEND_NAME`,
`attention_forward` and `available_backends()`.  There is exactly one backend
("cuda", librk.so on sm_100a); `ROUNDKV_BACKEND` may be `cuda` or `auto`, and
asking for the reference's CPU backends (`ext`, `numpy`) raises ImportError,
the same way the reference rejects an unknown name (backend.py:40-44).

`attention_forward(q, k, v, q_pos, k_pos, allowed=None, capture=False)` keeps
the reference contract (_attn_np.py:50-92 / _attn_ext.pyx:84-116):
  * NumPy inputs are validated and coerced like check_attention_inputs
    (_attn_np.py:19-47) and NumPy results come back: out (n, H*d) float32,
    scores (n, S) float64 row-normalised or None;
  * torch CUDA tensors stay on the device (fp32 or bf16 K/V) and torch tensors
    come back — the zero-copy path used by the pipeline;
  * shape errors raise DomainError, a query row with no visible key raises
    InvariantError("query row i has no visible key").
`attention_forward_gqa` additionally accepts Hq = G * Hkv (HF repeat_kv).
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib
from .errors import DomainError, InvariantError
from .workspace import scratch

BACKEND_NAME = "cuda"

_requested = os.environ.get("ROUNDKV_BACKEND", "auto").lower()
if _requested not in ("auto", "cuda"):
    raise ImportError(
        f"ROUNDKV_BACKEND={_requested!r}: this package only has the CUDA backend (use cuda or auto)")


def available_backends() -> dict:
    """Name -> kernel module (backend.py:21-28)."""
    import sys
    return {BACKEND_NAME: sys.modules[__name__]}


def _is_torch(x) -> bool:
    try:
        import torch
        return isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


def _check_numpy(q, k, v, q_pos, k_pos, allowed, gqa):
    """check_attention_inputs (_attn_np.py:19-47) on host arrays."""
    q = np.ascontiguousarray(q, dtype=np.float32)
    k = np.ascontiguousarray(k, dtype=np.float32)
    v = np.ascontiguousarray(v, dtype=np.float32)
    _check_shapes(q.shape, k.shape, v.shape, q.ndim, k.ndim, v.ndim, gqa)
    q_pos = np.ascontiguousarray(q_pos, dtype=np.int64)
    k_pos = np.ascontiguousarray(k_pos, dtype=np.int64)
    if q_pos.shape != (q.shape[0],) or k_pos.shape != (k.shape[0],):
        raise DomainError("position arrays must match q/k row counts")
    if allowed is not None:
        allowed = np.ascontiguousarray(allowed, dtype=bool)
        if allowed.shape != (k.shape[0],):
            raise DomainError("allowed mask must have one entry per key row")
    return q, k, v, q_pos, k_pos, allowed


def _check_shapes(qs, ks, vs, qn, kn, vn, gqa):
    if qn != 3 or kn != 3 or vn != 3:
        raise DomainError("q, k, v must be (rows, heads, head_dim) arrays")
    if tuple(ks) != tuple(vs):
        raise DomainError(f"key/value shape mismatch: {tuple(ks)} vs {tuple(vs)}")
    if gqa:
        ok = qs[2] == ks[2] and ks[1] > 0 and qs[1] % ks[1] == 0
    else:
        ok = tuple(qs[1:]) == tuple(ks[1:])
    if not ok:
        raise DomainError(f"query heads {tuple(qs[1:])} do not match key heads {tuple(ks[1:])}")
    if qs[2] == 0:
        raise DomainError("head_dim must be positive")


def _run(q, k, v, q_pos, k_pos, allowed, capture):
    """Device call on torch tensors (q f32; k/v f32 or bf16), returns torch."""
    torch = _lib.require_cuda()
    n, hq, d = q.shape
    s, hkv = k.shape[0], k.shape[1]
    dev = q.device
    out = torch.empty((n, hq * d), dtype=torch.float32, device=dev)
    scores = torch.empty((n, s), dtype=torch.float64, device=dev) if capture else None
    if n == 0:
        return out, (torch.zeros((0, s), dtype=torch.float64, device=dev) if capture else None)
    kv_dtype = _lib.RK_BF16 if k.dtype == torch.bfloat16 else _lib.RK_F32
    q = q.contiguous().to(torch.float32)
    k = k.contiguous()
    v = v.contiguous().to(k.dtype)
    q_pos = q_pos.to(device=dev, dtype=torch.int64).contiguous()
    k_pos = k_pos.to(device=dev, dtype=torch.int64).contiguous()
    allowed_u8 = None if allowed is None else allowed.to(device=dev, dtype=torch.uint8).contiguous()
    bad = torch.empty(1, dtype=torch.int32, device=dev)
    ws_bytes = _lib.lib.rk_attention_workspace_bytes(n, hq, hkv, s, d)
    ws = scratch(ws_bytes, dev, "attention")
    _lib.call("rk_attention_forward", _lib.ptr(q), n, hq, d, _lib.ptr(k), _lib.ptr(v), kv_dtype, s, hkv,
              _lib.ptr(q_pos), _lib.ptr(k_pos), _lib.ptr(allowed_u8), _lib.ptr(out), _lib.ptr(scores),
              _lib.ptr(bad), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    bad_row = int(bad.item())
    if bad_row != 2**31 - 1:
        raise InvariantError(f"query row {bad_row} has no visible key")
    return out, scores


def _forward(q, k, v, q_pos, k_pos, allowed, capture, gqa):
    if _is_torch(q):
        torch = _lib.require_cuda()
        _check_shapes(tuple(q.shape), tuple(k.shape), tuple(v.shape), q.dim(), k.dim(), v.dim(), gqa)
        q_pos = torch.as_tensor(q_pos)
        k_pos = torch.as_tensor(k_pos)
        if tuple(q_pos.shape) != (q.shape[0],) or tuple(k_pos.shape) != (k.shape[0],):
            raise DomainError("position arrays must match q/k row counts")
        if allowed is not None:
            allowed = torch.as_tensor(allowed)
            if tuple(allowed.shape) != (k.shape[0],):
                raise DomainError("allowed mask must have one entry per key row")
        return _run(q, k, v, q_pos, k_pos, allowed, capture)
    torch = _lib.require_cuda()
    q, k, v, q_pos, k_pos, allowed = _check_numpy(q, k, v, q_pos, k_pos, allowed, gqa)
    n, hq, d = q.shape
    if n == 0:
        out = np.zeros((0, hq * d), dtype=np.float32)
        return out, (np.zeros((0, k.shape[0])) if capture else None)
    dev = torch.device("cuda", torch.cuda.current_device())
    t = lambda a: torch.from_numpy(a).to(dev, non_blocking=False)  # noqa: E731
    out, scores = _run(t(q), t(k), t(v), t(q_pos), t(k_pos),
                       None if allowed is None else t(allowed.view(np.uint8)), capture)
    return out.cpu().numpy(), (scores.cpu().numpy() if capture else None)


def attention_forward(q, k, v, q_pos, k_pos, allowed=None, capture=False):
    """Causal multi-head attention over cached keys/values (MHA contract)."""
    return _forward(q, k, v, q_pos, k_pos, allowed, capture, gqa=False)


def attention_forward_gqa(q, k, v, q_pos, k_pos, allowed=None, capture=False):
    """Same contract with Hq = G * Hkv query heads (query head h -> kv head h // G)."""
    return _forward(q, k, v, q_pos, k_pos, allowed, capture, gqa=True)
