"""Round-level attention statistics on the device (Eq. 1 + normalisation).

Mirrors the hot-path half of `pkg/src/roundkv/stats.py`:
  * `RoundDistribution`            stats.py:28-40
  * `aggregate_round_attention`    stats.py:59-94  (same validation; the sum
    runs in rk_aggregate_rounds on the GPU)
  * `normalize`                    stats.py:97-115 (rk_select with kind=all:
    NumPy-order pairwise sum, so masses are bit-identical to the reference)
plus the fused path the pipeline uses:
  * `round_scores`  — the Eq. 1 masses straight from Q and K of layer Lw-1
    (rk_round_scores) without materialising the capture matrix; equals
    aggregate_round_attention(attention_forward(..., capture=True)[1], ...).
The calibration half of the reference module (KL curves, watershed detection,
Spearman, CSV) is offline analysis and out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DomainError
from .workspace import scratch

SEGMENT_QUESTION = "question"
SEGMENT_ANSWER = "answer"


@dataclass(frozen=True)
class Round:
    """One question/answer pair; half-open token spans (conversation.py:38-68)."""

    index: int
    q_span: tuple
    a_span: tuple

    @property
    def completed(self) -> bool:
        return self.a_span[1] > self.a_span[0]

    @property
    def start(self) -> int:
        return self.q_span[0]

    @property
    def end(self) -> int:
        return self.a_span[1] if self.completed else self.q_span[1]


@dataclass
class RoundDistribution:
    """Normalised attention mass over prior rounds at one layer (stats.py:28-40)."""

    layer: int
    segment: str
    round_indices: list
    raw: np.ndarray
    masses: np.ndarray
    degenerate: bool = False

    def __len__(self) -> int:
        return len(self.round_indices)


def _device():
    torch = _lib.require_cuda()
    return torch, torch.device("cuda", torch.cuda.current_device())


def aggregate_round_attention(scores, rounds, segment, current_round, *, active_rounds=None,
                              row_offset: int = 0):
    """Sum the current segment's capture rows over each prior round's columns."""
    if segment not in (SEGMENT_QUESTION, SEGMENT_ANSWER):
        raise DomainError(f"unknown segment {segment!r}")
    if not 0 <= current_round < len(rounds):
        raise DomainError(f"current_round {current_round} out of range")
    rnd = rounds[current_round]
    span = rnd.q_span if segment == SEGMENT_QUESTION else rnd.a_span
    if span[1] <= span[0]:
        raise DomainError(f"round {current_round} has an empty {segment} span")
    row_lo, row_hi = span[0] - row_offset, span[1] - row_offset
    n_rows = scores.shape[0]
    if row_lo < 0 or row_hi > n_rows:
        raise DomainError(f"{segment} rows [{span[0]}, {span[1]}) absent from scores")
    active = list(active_rounds) if active_rounds is not None else list(range(current_round))
    spans = np.zeros((len(active), 4), dtype=np.int64)
    cols = scores.shape[1]
    for i, k in enumerate(active):
        if not 0 <= k < current_round:
            raise DomainError(f"round {k} is not prior to round {current_round}")
        pr = rounds[k]
        q0, q1 = min(pr.q_span[0], cols), min(pr.q_span[1], cols)
        a0, a1 = min(pr.a_span[0], cols), min(pr.a_span[1], cols)
        spans[i] = (q0, max(q0, q1), a0, max(a0, a1))
    torch, dev = _device()
    on_device = isinstance(scores, torch.Tensor)
    s = scores if on_device else torch.from_numpy(np.ascontiguousarray(scores, dtype=np.float64))
    s = s.to(device=dev, dtype=torch.float64).contiguous()
    raw = torch.zeros(len(active), dtype=torch.float64, device=dev)
    if len(active):
        sp = torch.from_numpy(spans).to(dev)
        _lib.call("rk_aggregate_rounds", _lib.ptr(s), s.shape[1], row_lo, row_hi, _lib.ptr(sp), len(active),
                  _lib.ptr(raw), _lib.stream_ptr())
    return raw if on_device else raw.cpu().numpy()


def _select_device(values: np.ndarray, normalize: int, kind: str, v=0.1, k_top=0, kappa=1.0):
    """One rk_select launch; returns (masses, kept_positions, degenerate)."""
    torch, dev = _device()
    n = len(values)
    x = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float64)).to(dev)
    masses = torch.empty(n, dtype=torch.float64, device=dev)
    ints = torch.zeros(n + 3, dtype=torch.int32, device=dev)   # kept[n] | n_kept | degenerate | status
    _lib.call("rk_select", _lib.ptr(x), n, normalize, _lib.SEL_KINDS[kind], float(v), int(k_top),
              float(kappa), _lib.ptr(masses), _lib.ptr(ints), ints.data_ptr() + 4 * n,
              ints.data_ptr() + 4 * (n + 1), ints.data_ptr() + 4 * (n + 2), _lib.stream_ptr())
    host = ints.cpu().numpy()
    if host[n + 2] != 0:
        raise DomainError("raw attention masses must be non-negative")
    kept = [int(i) for i in host[: host[n]]]
    return masses.cpu().numpy(), kept, bool(host[n + 1])


def normalize(raw, *, layer: int = 0, segment: str = SEGMENT_QUESTION,
              round_indices=None) -> RoundDistribution:
    """raw / raw.sum(); uniform with degenerate=True when the sum is 0."""
    raw = np.asarray(raw.cpu().numpy() if hasattr(raw, "cpu") else raw, dtype=np.float64)
    if np.any(raw < 0):
        raise DomainError("raw attention masses must be non-negative")
    if round_indices is None:
        round_indices = list(range(len(raw)))
    if len(raw) == 0:
        return RoundDistribution(layer, segment, list(round_indices), raw, raw.copy(), True)
    masses, _, degenerate = _select_device(raw, 1, "all")
    return RoundDistribution(layer=layer, segment=segment, round_indices=list(round_indices),
                             raw=raw, masses=masses, degenerate=degenerate)


def build_round_items(bounds, chunk: int = 256):
    """Round-aligned work items (key_lo, key_hi, bin) for rk_round_scores.

    `bounds` = [(key_lo, key_hi, bin), ...] in ascending key order; every
    range is cut into pieces of at most `chunk` keys (items stay sorted by bin).
    """
    items = []
    for lo, hi, b in bounds:
        for s in range(lo, hi, chunk):
            items.append((s, min(hi, s + chunk), b))
    return np.asarray(items, dtype=np.int32).reshape(-1, 3)


_ITEMS_CACHE: dict = {}          # (bounds, chunk, device, stream) -> device item table (read-only to the kernels)


def _device_items(torch, dev, key_bounds, chunk: int):
    """The round items on the device, uploaded once per distinct (bounds, chunk):
    the calibration pass scores every layer of a conversation with one table, and
    a pipeline's turns repeat it until a round is added.  Keyed by the current
    stream too, so a table is only read on the stream it was allocated on and an
    evicted one is reused by the caching allocator in stream order."""
    key = (tuple((int(lo), int(hi), int(b)) for lo, hi, b in key_bounds), int(chunk), str(dev),
           torch.cuda.current_stream(dev).cuda_stream)
    t = _ITEMS_CACHE.get(key)
    if t is None:
        if len(_ITEMS_CACHE) >= 64:
            _ITEMS_CACHE.pop(next(iter(_ITEMS_CACHE)))
        t = _ITEMS_CACHE[key] = torch.from_numpy(build_round_items(key_bounds, chunk)).to(dev)
    return t


def round_scores(q, k, q_pos, k_pos, key_bounds, n_bins, active=None, *, chunk: int = 256, exact: bool = True,
                 capture_mode: str = "post"):
    """Fused capture + Eq. 1: raw mass per ACTIVE prior round (float64, device).

    q: (n_q, Hq, d) float32 cuda; k: (S, Hkv, d) fp32/bf16 cuda (layer Lw-1
    keys, ascending positions); key_bounds: [(lo, hi, bin)] covering [0, S)
    with bin == n_bins for the current round's keys (denominator only).
    exact=True (default): rk_round_scores_exact, the reference kernel's fp64
    arithmetic (kept sets bit-exact by construction); exact=False: the
    fp32-class rk_round_scores (tcgen05 scores-only pass for large bf16
    questions).  capture_mode="pre" (engine.py:187-200): one softmax per row
    over the head-summed logits / (Hq sqrt(d)) (rk_round_scores_exact_pre;
    exact scoring only).
    """
    torch, dev = _device()
    n_q, hq, d = q.shape
    s, hkv = k.shape[0], k.shape[1]
    items = _device_items(torch, dev, key_bounds, chunk)
    n_items = items.shape[0]
    act = None
    n_out = n_bins
    if active is not None:
        a = np.asarray(active, dtype=np.uint8)
        n_out = int(a.sum())
        act = torch.from_numpy(a).to(dev)
    raw = torch.zeros(max(n_out, 1), dtype=torch.float64, device=dev)
    kv_dtype = _lib.RK_BF16 if k.dtype == torch.bfloat16 else _lib.RK_F32
    if capture_mode not in ("post", "pre"):
        raise DomainError(f"capture_mode must be 'post' or 'pre', got {capture_mode!r}")
    if capture_mode == "pre" and not exact:
        raise DomainError("capture_mode='pre' is scored by the exact (fp64) scorer only")
    if exact:
        q_pos = torch.as_tensor(q_pos, dtype=torch.int64, device=dev)
        k_pos = torch.as_tensor(k_pos, dtype=torch.int64, device=dev)
        qc = q.contiguous().float()
        kc = k.contiguous()
        ws_bytes = _lib.lib.rk_round_scores_exact_workspace_bytes(1, n_q, hq, n_items, n_bins)
        ws = scratch(ws_bytes, dev, "scores_exact")
        entry = "rk_round_scores_exact" if capture_mode == "post" else "rk_round_scores_exact_pre"
        _lib.call(entry, _lib.ptr(qc), 1, n_q, hq, d, _lib.ptr(kc), kv_dtype, hkv, 0, None, s,
                  _lib.ptr(q_pos), _lib.ptr(k_pos), _lib.ptr(items), n_items, None, n_bins, _lib.ptr(act),
                  max(n_out, 1), _lib.ptr(raw), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
        return raw[:n_out]
    ws_bytes = _lib.lib.rk_round_scores_workspace_bytes(n_q, hq, hkv, n_items, d, n_bins)
    ws = scratch(ws_bytes, dev, "scores")
    q_pos = torch.as_tensor(q_pos, dtype=torch.int64, device=dev)
    k_pos = torch.as_tensor(k_pos, dtype=torch.int64, device=dev)
    qc = q.contiguous()            # bound to a name: alive until the call is enqueued
    _lib.call("rk_round_scores", _lib.ptr(qc), n_q, hq, d, _lib.ptr(k), kv_dtype, s, hkv,
              _lib.ptr(q_pos), _lib.ptr(k_pos), _lib.ptr(items), n_items, n_bins, _lib.ptr(act),
              _lib.ptr(raw), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    return raw[:n_out]


# The reference's stats module also carries the KL / watershed helpers
# (stats.py:118-181); they live in calibration.py (which imports this module),
# re-exported here lazily.
_CALIBRATION_NAMES = ("KL_EPSILON", "KLCurve", "WatershedResult", "kl_divergence", "kl_curve", "mean_curve",
                      "detect_watershed")


def __getattr__(name):
    if name in _CALIBRATION_NAMES:
        from . import calibration
        return getattr(calibration, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
