"""ORACLE (test infrastructure only): round statistics, selection, store ledger,
memory model — restated from the reference.

* `aggregate_round_attention` / `normalize` — `pkg/src/roundkv/stats.py:59-115`
* selection strategies — `pkg/src/roundkv/selection.py:20-126`
* `TieredStore` + `TransferLedger` — `pkg/src/roundkv/store.py:52-302`
* Eq. 2 memory model — `pkg/src/roundkv/store.py:308-357`
* `np_pairwise_sum` — NumPy's float64 `add.reduce` order for a contiguous 1-D
  array (8-way unrolled blocks of <=128, recursive halving at multiples of 8).
  The reference's selection thresholds depend on `masses = raw / raw.sum()`,
  `masses.mean()` and `masses.std()` (`stats.py:100-101`, `selection.py:104`);
  the device selector reproduces this order so kept sets are bit-exact.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from paper_2502_15294_b200.errors import (
    CapacityError,
    ConsistencyError,
    DomainError,
)

SEP_TOKEN = 256      # conversation.py:24
EOT_TOKEN = 257      # conversation.py:25
VOCAB_SIZE = 258     # conversation.py:26


@dataclass(frozen=True)
class Round:
    """Half-open token spans of one question/answer pair (conversation.py:38-68)."""

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


def make_rounds(lengths):
    """Rounds tiled from (q_len, a_len) pairs (tests/conftest.py:64-73)."""
    rounds, pos = [], 0
    for m, (ql, al) in enumerate(lengths):
        rounds.append(Round(m, (pos, pos + ql), (pos + ql, pos + ql + al)))
        pos += ql + al
    return rounds


# --------------------------------------------------------------------------
# numpy-exact reductions
# --------------------------------------------------------------------------

def np_pairwise_sum(values) -> float:
    """float64 sum in NumPy's pairwise order (see module docstring)."""
    a = [float(x) for x in values]

    def rec(lo, n):
        if n < 8:
            r = 0.0
            for i in range(lo, lo + n):
                r += a[i]
            return r
        if n <= 128:
            r = a[lo:lo + 8]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] += a[lo + i + j]
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res += a[lo + i]
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return rec(lo, n2) + rec(lo + n2, n - n2)

    return rec(0, len(a))


def np_mean_std(masses):
    """`masses.mean()` and population `masses.std()` with NumPy's operation order
    (_methods._mean / _var: pairwise sum, true divide, squared deviations)."""
    n = len(masses)
    mean = np_pairwise_sum(masses) / n
    dev = [(float(m) - mean) * (float(m) - mean) for m in masses]
    var = np_pairwise_sum(dev) / n
    return mean, math.sqrt(var)


# --------------------------------------------------------------------------
# Eq. 1 aggregation and normalisation (stats.py)
# --------------------------------------------------------------------------

@dataclass
class RoundDistribution:
    """stats.py:28-40"""

    layer: int
    segment: str
    round_indices: list
    raw: np.ndarray
    masses: np.ndarray
    degenerate: bool = False

    def __len__(self):
        return len(self.round_indices)


def aggregate_round_attention(scores, rounds, segment, current_round, *,
                              active_rounds=None, row_offset=0):
    """stats.py:59-94: per prior round, the capture mass of the current
    round's segment rows falling on that round's question+answer columns."""
    if segment not in ("question", "answer"):
        raise DomainError(f"unknown segment {segment!r}")
    if not 0 <= current_round < len(rounds):
        raise DomainError(f"current_round {current_round} out of range")
    cur = rounds[current_round]
    lo, hi = cur.q_span if segment == "question" else cur.a_span
    if hi <= lo:
        raise DomainError(f"round {current_round} has an empty {segment} span")
    r0, r1 = lo - row_offset, hi - row_offset
    scores = np.asarray(scores, dtype=np.float64)
    if r0 < 0 or r1 > scores.shape[0]:
        raise DomainError(f"{segment} rows [{lo}, {hi}) absent from scores")
    rows = scores[r0:r1]
    active = list(range(current_round)) if active_rounds is None else list(active_rounds)
    raw = np.empty(len(active), dtype=np.float64)
    for i, k in enumerate(active):
        if not 0 <= k < current_round:
            raise DomainError(f"round {k} is not prior to round {current_round}")
        pr = rounds[k]
        raw[i] = rows[:, pr.q_span[0]:pr.q_span[1]].sum() + rows[:, pr.a_span[0]:pr.a_span[1]].sum()
    return raw


def normalize(raw, *, layer=0, segment="question", round_indices=None):
    """stats.py:97-115: raw / sum, uniform + degenerate flag when the sum is 0."""
    raw = np.asarray(raw, dtype=np.float64)
    if np.any(raw < 0):
        raise DomainError("raw attention masses must be non-negative")
    if round_indices is None:
        round_indices = list(range(len(raw)))
    total = np_pairwise_sum(raw)
    if total > 0:
        masses, degenerate = raw / total, False
    else:
        masses = np.full(len(raw), 1.0 / len(raw)) if len(raw) else raw.copy()
        degenerate = True
    return RoundDistribution(layer, segment, list(round_indices), raw, masses, degenerate)


# --------------------------------------------------------------------------
# selection (selection.py)
# --------------------------------------------------------------------------

POLICY_KINDS = ("fixed", "top_percent", "adaptive", "all", "token_baseline")
CEIL_SLACK = 1e-9  # selection.py:23


@dataclass(frozen=True)
class SelectionPolicy:
    """selection.py:26-42"""

    kind: str = "top_percent"
    v: float = 0.1
    fraction: float = 0.10
    kappa: float = 1.0
    min_rounds: int = 1

    def __post_init__(self):
        if self.kind not in POLICY_KINDS:
            raise DomainError(f"policy kind must be one of {POLICY_KINDS}")
        if not 0.0 < self.v < 1.0:
            raise DomainError("fixed threshold v must lie in (0, 1)")
        if not 0.0 < self.fraction <= 1.0:
            raise DomainError("fraction must lie in (0, 1]")
        if self.min_rounds < 1:
            raise DomainError("min_rounds must be >= 1")


def top_k_count(n, fraction, min_rounds):
    """selection.py:93-94"""
    return min(n, max(min_rounds, math.ceil(fraction * n - CEIL_SLACK)))


def select_positions(masses, policy: SelectionPolicy):
    """Kept positions (indices into `masses`), ascending — selection.py:63-126."""
    m = [float(x) for x in masses]
    n = len(m)
    if n == 0:
        return []
    if policy.kind == "all":
        return list(range(n))
    if policy.kind == "top_percent":
        k = top_k_count(n, policy.fraction, policy.min_rounds)
        # stable descending sort: ties resolve to the smaller index (:95-96)
        order = sorted(range(n), key=lambda i: (-m[i], i))
        return sorted(order[:k])
    if policy.kind == "fixed":
        kept = [i for i in range(n) if m[i] > policy.v]
    elif policy.kind == "adaptive":
        mean, std = np_mean_std(m)
        cut = mean + policy.kappa * std
        kept = [i for i in range(n) if m[i] > cut]
    else:
        raise DomainError(f"policy {policy.kind!r} is not a round-selection strategy")
    if not kept:                       # _argmax_fallback :71-73 (first max)
        kept = [max(range(n), key=lambda i: (m[i], -i))]
    return kept


def select(dist: RoundDistribution, policy: SelectionPolicy):
    """Kept round ids, ascending (selection.py:117-126 with _result :63-68)."""
    pos = select_positions(dist.masses, policy)
    return tuple(sorted(dist.round_indices[i] for i in pos))


# --------------------------------------------------------------------------
# tiered store ledger (store.py)
# --------------------------------------------------------------------------

MODELED_ELEM_BYTES = 2
MIB = 1 << 20
DEFAULT_DEVICE_CAPACITY = 64 * MIB


def block_nbytes(tokens, hidden, layers):
    """store.py:34-36"""
    return 2 * MODELED_ELEM_BYTES * tokens * hidden * layers


class ActivityLedger:
    """selection.py:168-204: last-active turn per round and the inactivity drop rule."""

    def __init__(self, window=math.inf, protect_recent=2):
        self.window = window
        self.protect_recent = protect_recent
        self.last_active = {}
        self.dropped = set()

    def register_round(self, round_index, turn):
        self.last_active.setdefault(round_index, turn)

    def active_rounds(self, upto):
        return [m for m in range(upto) if m not in self.dropped]

    def update_and_drop(self, kept, current_turn, total_rounds):
        kept = set(kept)
        for m in kept:
            self.last_active[m] = current_turn
        if math.isinf(self.window):
            return []
        drops = []
        for m in range(total_rounds):
            if m in self.dropped or m in kept:
                continue
            if m >= total_rounds - self.protect_recent:
                continue
            if current_turn - self.last_active.get(m, current_turn) >= self.window:
                drops.append(m)
        self.dropped.update(drops)
        return drops


@dataclass
class TurnRecord:
    turn: int
    h2d_events: int = 0
    h2d_bytes: int = 0
    d2h_events: int = 0
    d2h_bytes: int = 0
    device_used_bytes: int = 0


@dataclass
class Ledger:
    """store.py:62-107"""

    h2d_events: int = 0
    h2d_bytes: int = 0
    d2h_events: int = 0
    d2h_bytes: int = 0
    per_turn: list = field(default_factory=list)

    def begin_turn(self, turn):
        self.per_turn.append(TurnRecord(turn))

    def _cur(self):
        if not self.per_turn:
            self.begin_turn(0)
        return self.per_turn[-1]

    def h2d(self, nbytes):
        self.h2d_events += 1
        self.h2d_bytes += nbytes
        r = self._cur()
        r.h2d_events += 1
        r.h2d_bytes += nbytes

    def d2h(self, nbytes):
        self.d2h_events += 1
        self.d2h_bytes += nbytes
        r = self._cur()
        r.d2h_events += 1
        r.d2h_bytes += nbytes

    def note(self, used):
        r = self._cur()
        r.device_used_bytes = max(r.device_used_bytes, used)

    def rows(self):
        return [dict(turn=r.turn, h2d_events=r.h2d_events, h2d_bytes=r.h2d_bytes,
                     d2h_events=r.d2h_events, d2h_bytes=r.d2h_bytes,
                     device_used_bytes=r.device_used_bytes) for r in self.per_turn]


class StoreModel:
    """Tier/ledger state machine of TieredStore (store.py:110-302), payload-free."""

    def __init__(self, num_layers, watershed, d_model, *,
                 device_capacity=DEFAULT_DEVICE_CAPACITY, evict_lower_on_pressure=False):
        if not 0 < watershed < num_layers:
            raise DomainError(f"watershed must satisfy 0 < L_w < L, got {watershed} of {num_layers}")
        self.L, self.lw, self.d = num_layers, watershed, d_model
        self.cap = device_capacity
        self.evict = evict_lower_on_pressure
        self.tier = {}     # (round, half) -> tier
        self.size = {}
        self.used = 0
        self.ledger = Ledger()

    def _get(self, m, half):
        if (m, half) not in self.tier:
            raise ConsistencyError(f"round {m} has no {half} block")
        return (m, half)

    def _room(self, incoming):
        if self.used + incoming <= self.cap:
            return
        if self.evict:
            spilled = 0
            for key in sorted((k for k, t in self.tier.items() if k[1] == "lower" and t == "device"),
                              key=lambda k: k[0]):
                if self.used + incoming <= self.cap:
                    break
                self.tier[key] = "host"
                self.used -= self.size[key]
                spilled += self.size[key]
            if spilled:
                self.ledger.d2h(spilled)
            if self.used + incoming <= self.cap:
                return
        raise CapacityError(f"device tier needs {incoming} bytes, {self.cap - self.used} available")

    def _to_device(self, keys):
        pending = [k for k in keys if self.tier[k] == "host"]
        if not pending:
            return
        total = sum(self.size[k] for k in pending)
        self._room(total)
        for k in pending:
            self.tier[k] = "device"
        self.used += total
        self.ledger.h2d(total)
        self.ledger.note(self.used)

    def begin_turn(self, turn):
        self.ledger.begin_turn(turn)

    def put_round(self, m, tokens, *, upper_on_device=False):
        if (m, "lower") in self.tier:
            raise ConsistencyError(f"round {m} already stored")
        lo_b = block_nbytes(tokens, self.d, self.lw)
        up_b = block_nbytes(tokens, self.d, self.L - self.lw)
        # store.py:432-445 — blocks are registered only after both room checks;
        # a CapacityError on the upper half leaves the lower bytes counted
        self._room(lo_b)
        self.used += lo_b
        if upper_on_device:
            self._room(up_b)
            self.used += up_b
            up_tier = "device"
        else:
            up_tier = "host"
            self.ledger.d2h(up_b)
        self.tier[(m, "lower")] = "device"
        self.size[(m, "lower")] = lo_b
        self.tier[(m, "upper")] = up_tier
        self.size[(m, "upper")] = up_b
        self.ledger.note(self.used)

    def fetch_lower_all(self, upto):
        self._to_device([self._get(m, "lower") for m in range(upto)])

    def fetch_upper(self, selected):
        keys = []
        for m in selected:
            k = self._get(m, "upper")
            if self.tier[k] == "dropped":
                raise ConsistencyError(f"round {m} upper block was dropped")
            keys.append(k)
        self._to_device(keys)

    def writeback_upper(self, rounds):
        moving = [self._get(m, "upper") for m in rounds]
        moving = [k for k in moving if self.tier[k] == "device"]
        if not moving:
            return
        for k in moving:
            self.tier[k] = "host"
            self.used -= self.size[k]
        self.ledger.d2h(sum(self.size[k] for k in moving))

    def drop_upper(self, m):
        k = self._get(m, "upper")
        if self.tier[k] == "device":
            self.used -= self.size[k]
        self.tier[k] = "dropped"

    def end_session(self):
        moving = [k for k, t in self.tier.items() if t == "device"]
        if not moving:
            return
        for k in moving:
            self.tier[k] = "host"
            self.used -= self.size[k]
        self.ledger.d2h(sum(self.size[k] for k in moving))


# --------------------------------------------------------------------------
# Eq. 2 memory model (store.py:308-357)
# --------------------------------------------------------------------------

def memory_ratio(num_layers, watershed, kept_rounds, total_rounds):
    if not 0 < watershed < num_layers:
        raise DomainError("watershed must satisfy 0 < L_w < L")
    if total_rounds < 1:
        raise DomainError("total rounds must be >= 1")
    if not 0 <= kept_rounds <= total_rounds:
        raise DomainError("kept rounds must satisfy 0 <= K <= T")
    f = watershed / num_layers
    return f + (kept_rounds / total_rounds) * (1.0 - f)


def save_percent(num_layers, watershed):
    if not 0 < watershed < num_layers:
        raise DomainError("watershed must satisfy 0 < L_w < L")
    return (200 * (num_layers - watershed) + num_layers) // (2 * num_layers)


def footprint_report(batch, seq_len, hidden, num_layers, watershed, kept_rounds, total_rounds):
    for name, value in (("batch", batch), ("seq_len", seq_len), ("hidden", hidden)):
        if value < 1:
            raise DomainError(f"{name} must be >= 1")
    ratio = memory_ratio(num_layers, watershed, kept_rounds, total_rounds)
    m_orig = 4.0 * batch * seq_len * hidden * num_layers
    m_round = (4.0 * batch * seq_len * hidden * watershed
               + 4.0 * batch * (kept_rounds / total_rounds) * seq_len * hidden * (num_layers - watershed))
    return {"m_orig_bytes": m_orig, "m_round_bytes": m_round, "ratio": m_round / m_orig,
            "closed_form_ratio": ratio, "save_percent_at_k0": save_percent(num_layers, watershed)}


# ---------------------------------------------------------------- calibration
# stats.py:118-181 (KL curve, watershed detection) and the conversation token
# layout of conversation.py:164-186 — restated for the calibration fixtures.

KL_EPSILON = 1e-10          # stats.py:22


def make_conversation_layout(q_lens, a_lens, rng):
    """Token ids and (q_span, a_span) per round: SEP (256) before every later
    question and before every answer (conversation.py:164-186); a_len 0 = the
    in-flight question."""
    ids, spans = [], []
    for m, (ql, al) in enumerate(zip(q_lens, a_lens)):
        qs = len(ids)
        if m > 0:
            ids.append(256)
        ids.extend(int(x) for x in rng.integers(0, 256, size=ql))
        qe = len(ids)
        ae = qe
        if al > 0:
            ids.append(256)
            ids.extend(int(x) for x in rng.integers(0, 256, size=al))
            ae = len(ids)
        spans.append(((qs, qe), (qe, ae)))
    return ids, spans


def kl_divergence(p, q, epsilon=KL_EPSILON):
    """stats.py:118-128."""
    p = np.asarray(p, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    if np.array_equal(p, q):
        return 0.0
    ps = (p + epsilon) / (p + epsilon).sum()
    qs = (q + epsilon) / (q + epsilon).sum()
    return float(np.sum(ps * np.log(ps / qs)))


def kl_curve(per_layer_masses):
    """stats.py:131-144: D(l) = mean KL from layer l to every later layer."""
    d = [np.asarray(x, dtype=np.float64) for x in per_layer_masses]
    L = len(d)
    return np.array([np.mean([kl_divergence(d[l], d[lp]) for lp in range(l + 1, L)]) for l in range(L - 1)])


def detect_watershed(curves, criterion="max_drop", tau=0.1):
    """stats.py:157-181 over the corpus mean curve (stats.py:147-154)."""
    d = np.stack(curves).mean(axis=0)
    L = d.shape[0] + 1
    cand = np.arange(1, L - 1)
    if criterion == "max_drop":
        return int(cand[np.argmax(d[cand - 1] - d[cand])])
    below = cand[d[cand] <= tau]
    return int(below[0]) if below.size else int(cand[np.argmin(d[cand])])
