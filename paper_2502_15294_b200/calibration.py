"""Watershed calibration on the GPU.

Restates the reference's calibration path (`pkg/src/roundkv/pipeline.py:439-494`,
`pkg/src/roundkv/stats.py:118-181`):

  capture_all_layers    teacher-forced full prefill capturing every layer
  layer_distributions   Eq. 1 round masses of the analysis round's question
  kl_curve              D(l) = mean KL from layer l to every later layer
  detect_watershed      max_drop / threshold criterion over the corpus mean

The O(L * S^2) part — every layer's capture matrix — never exists here: the
prefill runs on the device (`engine.Model.forward_range`) and at every layer a
hook hands the analysis round's question rows to the fused scorer
(`stats.round_scores` -> `rk_round_scores`: softmax statistics per round item,
no capture matrix), so each layer yields its n-round distribution directly.
The KL curve and the watershed choice are L x n host arithmetic, restated
from the reference with the same NumPy expressions.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import DomainError
from .stats import SEGMENT_QUESTION, Round, aggregate_round_attention, normalize, round_scores

KL_EPSILON = 1e-10          # stats.py:22 smoothing
SEP_TOKEN = 256             # conversation.py:24


@dataclass
class Conversation:
    """The slice of the reference's Conversation (conversation.py:71-100) the
    calibration reads: the token stream and its rounds."""

    rounds: list = field(default_factory=list)
    token_ids: list = field(default_factory=list)

    @property
    def T(self) -> int:
        return sum(1 for r in self.rounds if r.completed)

    @property
    def num_tokens(self) -> int:
        return len(self.token_ids)

    @property
    def has_inflight(self) -> bool:
        return bool(self.rounds) and not self.rounds[-1].completed


@dataclass(frozen=True)
class KLCurve:
    values: np.ndarray
    num_layers: int


@dataclass(frozen=True)
class WatershedResult:
    layer: int
    curve: KLCurve
    criterion: str
    corpus_size: int


def kl_divergence(p, q, epsilon: float = KL_EPSILON) -> float:
    """Smoothed forward KL in nats; exactly 0 for identical inputs (stats.py:118-128)."""
    p = np.asarray(p, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    if p.shape != q.shape:
        raise DomainError(f"length mismatch: {p.shape} vs {q.shape}")
    if np.array_equal(p, q):
        return 0.0
    ps = (p + epsilon) / (p + epsilon).sum()
    qs = (q + epsilon) / (q + epsilon).sum()
    return float(np.sum(ps * np.log(ps / qs)))


def kl_curve(per_layer_masses) -> KLCurve:
    """stats.py:131-144."""
    dists = [np.asarray(d, dtype=np.float64) for d in per_layer_masses]
    L = len(dists)
    if L < 2:
        raise DomainError("cross-layer curve needs at least 2 layers")
    if len({d.shape for d in dists}) != 1:
        raise DomainError("per-layer distributions must share one length")
    values = np.empty(L - 1, dtype=np.float64)
    for l in range(L - 1):
        values[l] = float(np.mean([kl_divergence(dists[l], dists[lp]) for lp in range(l + 1, L)]))
    return KLCurve(values=values, num_layers=L)


def mean_curve(curves) -> KLCurve:
    """stats.py:147-154."""
    if not curves:
        raise DomainError("empty calibration corpus")
    if len({c.num_layers for c in curves}) != 1:
        raise DomainError("curves disagree on layer count")
    return KLCurve(values=np.stack([c.values for c in curves]).mean(axis=0), num_layers=curves[0].num_layers)


def detect_watershed(curves, criterion: str = "max_drop", tau: float = 0.1) -> WatershedResult:
    """stats.py:157-181: max_drop = the l in [1, L-1) maximising D(l-1) - D(l)
    (smallest on ties); threshold = the smallest l with D(l) <= tau, else argmin."""
    avg = mean_curve(curves)
    d, L = avg.values, avg.num_layers
    if L < 3:
        raise DomainError("watershed detection needs at least 3 layers")
    cand = np.arange(1, L - 1)
    if criterion == "max_drop":
        layer = int(cand[np.argmax(d[cand - 1] - d[cand])])
    elif criterion == "threshold":
        below = cand[d[cand] <= tau]
        layer = int(below[0]) if below.size else int(cand[np.argmin(d[cand])])
    else:
        raise DomainError(f"unknown watershed criterion {criterion!r}")
    return WatershedResult(layer=layer, curve=avg, criterion=criterion, corpus_size=len(curves))


def analysis_round_index(conv) -> int | None:
    """pipeline.py:439-449."""
    if conv.has_inflight and conv.T >= 1:
        return len(conv.rounds) - 1
    if conv.T >= 2:
        return conv.T - 1
    return None


def layer_round_masses(model, conv, n: int, *, chunk: int = 256) -> np.ndarray:
    """(L, n) normalised question-segment round distributions of round n at
    every layer (pipeline.py:452-471), from one device prefill with fused
    scoring — the capture matrices of capture_all_layers are never formed."""
    import torch

    c = model.config
    L, H, dk = c.num_layers, c.num_heads, c.d_k
    r_n = conv.rounds[n]
    q0, q1 = r_n.q_span
    if q1 <= q0:
        raise DomainError(f"round {n} has an empty question segment")
    # every prior round receives a bin; keys from round n onwards are the
    # denominator-only bin (causal visibility keeps later keys out)
    bounds = [(conv.rounds[m].start, conv.rounds[m].end, m) for m in range(n)]
    bounds.append((conv.rounds[n].start, conv.num_tokens, n))
    q_pos = np.arange(q0, q1, dtype=np.int64)
    raws = [None] * L

    def hook(l, q, kv):
        keys = kv.keys.view(-1, H, dk)
        raws[l] = round_scores(q[q0:q1].contiguous(), keys, q_pos, kv.positions, bounds, n, chunk=chunk,
                               capture_mode=c.capture_mode)

    cache = model.new_cache()
    model.forward_range(cache, 0, L, tokens=conv.token_ids, positions=np.arange(conv.num_tokens),
                        layer_hook=hook)
    torch.cuda.synchronize()
    return np.stack([normalize(r.cpu().numpy(), layer=l).masses for l, r in enumerate(raws)])


def capture_all_layers(model, conv) -> dict:
    """pipeline.py:452-460: teacher-forced full prefill capturing every layer's
    (tokens, tokens) score matrix on the device — the reference's materialised
    route (and the one capture_mode="pre" needs); layer_round_masses computes the
    same distributions without the matrices."""
    L = model.config.num_layers
    positions = np.arange(conv.num_tokens, dtype=np.int64)
    _, captures = model.forward_range(model.new_cache(), 0, L, tokens=conv.token_ids, positions=positions,
                                      capture_layers=range(L))
    return captures


def layer_distributions(matrices, rounds, current_round: int, segment: str = SEGMENT_QUESTION) -> list:
    """pipeline.py:463-471: per-layer normalised round distributions from full
    score matrices (rk_aggregate_rounds + the device normalisation)."""
    return [normalize(aggregate_round_attention(m, rounds, segment, current_round), layer=l, segment=segment)
            for l, m in enumerate(matrices)]


def conversation_kl_curve(model, conv) -> KLCurve:
    """pipeline.py:474-481."""
    n = analysis_round_index(conv)
    if n is None:
        raise DomainError("conversation has no prior completed round to analyze")
    return kl_curve(layer_round_masses(model, conv, n))


def calibrate_watershed(model, conversations, *, criterion: str = "max_drop", tau: float = 0.1) -> WatershedResult:
    """pipeline.py:484-494: detect the watershed layer over a corpus."""
    curves = [conversation_kl_curve(model, conv) for conv in conversations if analysis_round_index(conv) is not None]
    if not curves:
        raise DomainError("calibration corpus has no multi-round conversation")
    return detect_watershed(curves, criterion=criterion, tau=tau)


def make_conversation(q_lens, a_lens, rng) -> Conversation:
    """Synthetic token stream with the reference's round layout
    (conversation.py:164-186: SEP before every later question and every answer);
    a_len 0 makes the last round the in-flight question."""
    ids, rounds = [], []
    for m, (ql, al) in enumerate(zip(q_lens, a_lens)):
        qs = len(ids)
        if m > 0:
            ids.append(SEP_TOKEN)
        ids.extend(int(x) for x in rng.integers(0, 256, size=ql))
        qe = len(ids)
        ae = qe
        if al > 0:
            ids.append(SEP_TOKEN)
            ids.extend(int(x) for x in rng.integers(0, 256, size=al))
            ae = len(ids)
        rounds.append(Round(m, (qs, qe), (qe, ae)))
    return Conversation(rounds=rounds, token_ids=ids)
