"""ORACLE (test infrastructure only): ctypes binding of oracle/attn_ref.c,
the threaded plain-C restatement of the reference kernel (_attn_ext.pyx:20-116),
used as the CPU-baseline port."""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

from paper_2502_15294_b200.errors import InvariantError

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libattnref.so"


def build():
    subprocess.run(["make", "-C", str(HERE), "_build/libattnref.so"], check=True, capture_output=True)


def _lib():
    if not LIB.exists():
        build()
    lib = C.CDLL(str(LIB))
    lib.attn_ref_forward.restype = C.c_int
    lib.attn_ref_forward.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                     C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
    return lib


_LIB = None


def attention_forward(q, k, v, q_pos, k_pos, allowed=None, capture=False, threads=1):
    """Same contract as the reference kernel; K/V may have fewer heads (GQA)."""
    global _LIB
    if _LIB is None:
        _LIB = _lib()
    q = np.ascontiguousarray(q, np.float32)
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    q_pos = np.ascontiguousarray(q_pos, np.int64)
    k_pos = np.ascontiguousarray(k_pos, np.int64)
    n, hq, d = q.shape
    s, hkv = k.shape[0], k.shape[1]
    out = np.zeros((n, hq * d), np.float32)
    cap = np.zeros((n, s), np.float64) if capture else None
    if n == 0:
        return out, cap
    al = None if allowed is None else np.ascontiguousarray(allowed, np.uint8)
    p = lambda a: None if a is None else a.ctypes.data  # noqa: E731
    bad = _LIB.attn_ref_forward(p(q), n, hq, d, p(k), p(v), s, hkv, p(q_pos), p(k_pos), p(al), p(out), p(cap),
                                int(threads))
    if bad >= 0:
        raise InvariantError(f"query row {bad} has no visible key")
    return out, cap


def round_masses(q, k, q_pos, k_pos, spans, n_bins, threads=None):
    """Eq. 1 raw masses per bin from q (n, Hq, d) and K (S, Hkv, d) with the
    reference kernel's capture arithmetic (attn_ref.c:attn_ref_round_masses);
    spans = [(key_lo, key_hi, bin)], bins >= n_bins ignored."""
    import os
    global _LIB
    if _LIB is None:
        _LIB = _lib()
    fn = _LIB.attn_ref_round_masses
    fn.restype = None
    fn.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                   C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int]
    q = np.ascontiguousarray(q, np.float32)
    k = np.ascontiguousarray(k, np.float32)
    q_pos = np.ascontiguousarray(q_pos, np.int64)
    k_pos = np.ascontiguousarray(k_pos, np.int64)
    sp = np.ascontiguousarray(np.asarray(spans, dtype=np.int32).reshape(-1, 3))
    n, hq, d = q.shape
    s, hkv = k.shape[0], k.shape[1]
    raw = np.zeros(n_bins, np.float64)
    fn(q.ctypes.data, n, hq, d, k.ctypes.data, s, hkv, q_pos.ctypes.data, k_pos.ctypes.data, sp.ctypes.data,
       len(sp), n_bins, raw.ctypes.data, int(threads or os.cpu_count() or 1))
    return raw
