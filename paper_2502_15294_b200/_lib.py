"""ctypes binding of librk.so (include/roundkv_b200.h).

The library is the product: there is no CPU fallback.  Importing this module
on a machine without the built library raises ImportError, and every entry
point raises the reference's exception classes for non-zero statuses.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import DeviceError, from_status

LIB_PATH = Path(os.environ.get("ROUNDKV_B200_LIB", Path(__file__).resolve().parent / "librk.so"))

if not LIB_PATH.exists():
    raise ImportError(
        f"librk.so not found at {LIB_PATH}; build it with `python -m paper_2502_15294_b200.build` "
        "(the round-attention path has no CPU fallback)")

lib = C.CDLL(str(LIB_PATH))

_p = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_sz = C.c_size_t
_d = C.c_double

_SIGS = {
    "rk_abi_version": (_i, []),
    "rk_last_error": (C.c_char_p, []),
    "rk_attention_workspace_bytes": (_sz, [_i, _i, _i, _i, _i]),
    "rk_attention_forward": (_i, [_p, _i, _i, _i, _p, _p, _i, _i, _i, _p, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "rk_decode_workspace_bytes": (_sz, [_i, _i, _i, _i, _i]),
    "rk_decode_attention": (_i, [_p, _i, _i, _i, _p, _p, _i, _i, _i64, _p, _i, _p, _p, _p, _p, _i, _p, _p, _p, _sz, _p]),
    "rk_advance_lengths": (_i, [_p, _i, _i, _p]),
    "rk_decode_attention_rows": (_i, [_p, _i, _i, _i, _p, _p, _i, _i, _i64, _p, _i, _p, _p, _p, _p, _p, _p]),
    "rk_out_proj_rows": (_i, [_p, _i, _i, _p, _i, _p, _p, _p, _sz, _p]),
    "rk_lm_head_rows": (_i, [_p, _i, _i, _p, _i, _p, _p, _p, _p, _p, _i, _p, _i, _p, _sz, _p]),
    "rk_decode_plan": (_i, [_i, _i, _i, _i, _i, _i, _i64, _i]),
    "rk_round_scores_workspace_bytes": (_sz, [_i, _i, _i, _i, _i, _i]),
    "rk_round_scores": (_i, [_p, _i, _i, _i, _p, _i, _i, _i, _p, _p, _p, _i, _i, _p, _p, _p, _sz, _p]),
    "rk_round_scores_finalize": (_i, [_i, _i, _i, _i, _i, _i, _p, _p, _i, _p, _p, _p, _p]),
    "rk_aggregate_rounds": (_i, [_p, _i64, _i, _i, _p, _i, _p, _p]),
    "rk_select": (_i, [_p, _i, _i, _i, _d, _i, _d, _p, _p, _p, _p, _p, _p]),
    "rk_select_batch": (_i, [_p, _i, _i, _i, _i, _i, _d, _i, _d, _p, _p, _p, _p, _p, _p]),
    "rk_select_batch_active": (_i, [_p, _i, _i, _i, _p, _i, _i, _d, _i, _d, _i, _d, _p, _p, _p, _p, _p, _p, _p]),
    "rk_selection_margin": (_i, [_p, _i, _i, _i, _i, _d, _i, _d, _p, _p]),
    "rk_round_scores_exact_workspace_bytes": (_sz, [_i, _i, _i, _i, _i]),
    "rk_round_scores_exact": (_i, [_p, _i, _i, _i, _i, _p, _i, _i, _i64, _p, _i, _p, _p, _p, _i, _p, _i, _p, _i,
                                   _p, _p, _sz, _p]),
    "rk_round_scores_exact_pre": (_i, [_p, _i, _i, _i, _i, _p, _i, _i, _i64, _p, _i, _p, _p, _p, _i, _p, _i, _p, _i,
                                       _p, _p, _sz, _p]),
    "rk_h2d_gather": (_i, [_i, _p, _p, _p, _p, _p, _p, _p, _p]),
    "rk_peer_gather": (_i, [_i, _p, _p, _p, _p, _p, _p, _p, _p]),
    "rk_enable_peer_access": (_i, [_i]),
    "rk_d2h_scatter": (_i, [_i, _p, _p, _p, _p, _p, _p, _p, _p]),
    "rk_prefill_workspace_bytes": (_sz, [_i, _i, _i, _i, _i, _i, _i]),
    "rk_prefill_attention": (_i, [_p, _i, _i, _i, _p, _p, _i, _i, _i, _p, _p, _p, _p, _i, _i, _p, _p, _p, _p, _p,
                                  _sz, _i, _p]),
    "rk_packed_weight_bytes": (_sz, [_i, _i]),
    "rk_pack_weight": (_i, [_p, _i, _i, _i, _p, _p]),
    "rk_proj_workspace_bytes": (_sz, [_i, _i, _i]),
    "rk_qkv_rope": (_i, [_p, _i, _i, _p, _i, _i, _i, _p, _p, _p, _p, _p, _i64, _p, _sz, _p]),
    "rk_qkv_rope_kv": (_i, [_p, _i, _i, _p, _i, _i, _i, _p, _p, _p, _p, _p, _i, _i64, _p, _sz, _p]),
    "rk_out_proj": (_i, [_p, _i, _i, _p, _i, _p, _p, _sz, _p]),
    "rk_lm_head_workspace_bytes": (_sz, [_i, _i, _i]),
    "rk_lm_head": (_i, [_p, _i, _i, _p, _i, _p, _p, _p, _p, _p, _i, _p, _sz, _p]),
    "rk_embed": (_i, [_p, _i, _p, _i, _p, _p]),
    "rk_rope_rows": (_i, [_p, _i, _i, _i, _i, _p, _p, _p, _p, _p, _i64, _i, _i64, _p]),
    "rk_small_qkv_rope": (_i, [_p, _i, _i, _p, _p, _p, _i, _p, _p, _p, _p, _p, _p]),
    "rk_small_out_proj": (_i, [_p, _i, _i, _p, _p, _p, _p]),
    "rk_small_logits": (_i, [_p, _i, _i, _p, _i, _p, _p, _p]),
    "rk_capture_pre": (_i, [_p, _i, _i, _i, _p, _i, _p, _p, _p, _p, _p]),
    "rk_decode_step_workspace_bytes": (_sz, [_i, _i, _i, _i, _i, _i]),
    "rk_decode_step_supported": (_i, [_i, _i, _i, _i, _i]),
    "rk_decode_step": (_i, [_p, _p]),
    "rk_decode_step_watchdog": (_i, [_p, _p, _p]),
}


class DecodeStepArgs(C.Structure):
    """rk_decode_step_args (include/roundkv_b200.h)."""
    _fields_ = [(n, _i) for n in ("batch", "num_layers", "watershed", "hq", "hkv", "head_dim", "vocab")] + [
        ("x", _p), ("lower", _p), ("lower_seq", _i64), ("upper", _p), ("upper_seq", _i64),
        ("lower_len", _p), ("upper_len", _p), ("pos", _p), ("rope_freq", _p), ("w_qkv", _p), ("w_o", _p),
        ("emb_packed", _p), ("emb", _p), ("tokens", _p), ("tokens_log", _p), ("log_stride", _i),
        ("workspace", _p), ("workspace_bytes", _sz)]

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

ABI_VERSION = lib.rk_abi_version()

RK_F32, RK_BF16 = 0, 1
RK_PREFILL_SINGLE_PASS = 1
SEL_KINDS = {"fixed": 0, "top_percent": 1, "adaptive": 2, "all": 3}


def last_error() -> str:
    msg = lib.rk_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str) -> None:
    """Raise the reference exception class mapped from a negative status."""
    if status != 0:
        raise from_status(status, f"{what}: {last_error()}")


def call(name: str, *args) -> None:
    check(getattr(lib, name)(*args), name)


def ptr(t) -> int | None:
    """Device/host address of a torch tensor (None passes NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the round-attention path runs only on the GPU (sm_100a)")
    return torch


def symbols() -> list[str]:
    return sorted(_SIGS)
