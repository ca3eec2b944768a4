"""Per-turn Round-Attention serving pipeline on the GPU (drop-in for
`pkg/src/roundkv/pipeline.py:114-433`, modes "round" and "baseline").

`RoundPipeline.run_turn(question, max_decode_steps)` follows Algorithm 1 of
the reference step by step (pipeline.py:192-394):
  1. lower blocks for all prior rounds (device tier, no transfer in steady state);
  2. lower-layer prefill of the question (SEP + tokens) with the Eq. 1 round
     masses at layer Lw-1 computed by the fused librk scorer (`round_scores`:
     softmax statistics per round, no capture matrix) over the same keys the
     reference's capture sees (every prior round incl. dropped ones + the causal
     question prefix); with capture_mode="pre" the head-summed-logit capture is
     materialised and aggregated instead (engine.py:187-200); `normalize` +
     `select` on the device (bit-exact);
  3. ONE batched H2D of the kept rounds' upper blocks (TieredStore.fetch_upper,
     rk_h2d_gather);
  4. upper-layer prefill over kept rounds + the question;
  5. greedy decode (argmax, first maximum) until EOT=257 or max_decode_steps;
  6. put_round(upper_on_device=True) + one batched writeback of kept + [n].
`attend_mode = "mask"` (pipeline.py:150, 271-280) assembles every upper block
and restricts visibility with `restricted_attention_mask` instead of splicing.
The token-granularity comparator and the simulated cost model are out of scope;
`TurnMetrics` keeps the transfer / selection fields of the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .engine import KVCache, Model
from .errors import DomainError
from .selection import ActivityLedger, SelectionPolicy, SelectionResult, select
from .stats import SEGMENT_QUESTION, Round, RoundDistribution, aggregate_round_attention, normalize, round_scores
from .store import TieredStore
# the reference module's calibration entry points (pipeline.py:439-494) live in calibration.py
from .calibration import (analysis_round_index, calibrate_watershed, capture_all_layers,  # noqa: F401
                          conversation_kl_curve, layer_distributions)

SEP_TOKEN = 256
EOT_TOKEN = 257
MODES = ("round", "baseline")


def tokenize(text: str) -> list:
    """One token id per UTF-8 byte (conversation.py:113-115)."""
    return list(text.encode("utf-8"))


def restricted_attention_mask(kept, rounds, current_start, key_positions, upper: bool):
    """Full causal below the watershed, kept rounds + current round above (pipeline.py:55-67)."""
    if not upper:
        return None
    kp = torch.as_tensor(key_positions)
    allowed = kp >= current_start
    for m in kept:
        r = rounds[m]
        allowed |= (kp >= r.start) & (kp < r.end)
    return allowed


@dataclass
class TurnMetrics:
    round_index: int
    mode: str
    policy: str
    append_rows: int
    decode_steps: int
    kept: tuple
    K: int
    selection_invocations: int
    upper_h2d_events: int
    upper_h2d_bytes: int
    lower_h2d_events: int
    lower_h2d_bytes: int
    d2h_events: int
    d2h_bytes: int
    device_used_peak: int
    hist_tokens: int
    hist_tokens_attended: int
    # the reference's simulated cost fields (costs.py, out of scope: real timings come from CUDA
    # events in bench.py); kept so TurnMetrics has the reference's field names and order
    total_cost_us: float | None = None
    curves: object = None
    shape: object = None
    distribution: RoundDistribution | None = None
    token_stats: object = None
    dropped_rounds: tuple = ()


@dataclass
class TurnResult:
    answer_ids: list
    metrics: TurnMetrics


class RoundPipeline:
    """Owns one conversation's serving state; strictly sequential per turn."""

    def __init__(self, model: Model, watershed: int, *, policy: SelectionPolicy | None = None,
                 mode: str = "round", store: TieredStore | None = None, cost_model=None,
                 drop_window: float = float("inf"), drop_protect: int = 2, conversation_id: str = "conv0"):
        if mode not in MODES:
            raise DomainError(f"mode must be one of {MODES}")
        L = model.config.num_layers
        if not 0 < watershed < L:
            raise DomainError(f"watershed must satisfy 0 < L_w < L, got {watershed} of {L}")
        if mode == "round" and policy is None:
            raise DomainError("round mode needs a selection policy")
        self.model = model
        self.watershed = watershed
        self.policy = policy
        self.mode = mode
        self.cost_model = cost_model          # accepted like the reference (cli.py:212-222); not simulated here
        self.store = store or TieredStore(L, watershed, model.config.d_model, conversation_id=conversation_id,
                                          device=model.device)
        self.activity = ActivityLedger(window=drop_window if mode == "round" else float("inf"),
                                       protect_recent=drop_protect)
        self.rounds: list = []
        self.token_ids: list = []
        self.attend_mode = "splice"

    @classmethod
    def baseline(cls, model: Model, watershed: int, **kwargs) -> "RoundPipeline":
        return cls(model, watershed, mode="baseline", **kwargs)

    # -- cache assembly (pipeline.py:158-180) -----------------------------------
    def _assemble(self, cache: KVCache, layer_lo: int, layer_hi: int, blocks) -> int:
        total = 0
        for block in blocks:
            payload = block.payload.to(self.model.device, non_blocking=True)
            pos = block.positions.to(self.model.device)
            for off, l in enumerate(range(layer_lo, layer_hi)):
                cache.layer(l).append(payload[off, 0], payload[off, 1], pos)
            total += block.tokens
        return total

    @staticmethod
    def _extract_new_rows(cache: KVCache, layer_lo: int, layer_hi: int, start_len: int):
        return torch.stack([torch.stack([cache.layer(l).keys[start_len:], cache.layer(l).values[start_len:]])
                            for l in range(layer_lo, layer_hi)])

    def _score(self, captures_q, working, q_start, n, rounds_now, active):
        """Fused Eq. 1 at layer Lw-1: raw mass per active prior round."""
        lw = self.watershed
        c = self.model.config
        kv = working.layer(lw - 1)
        q, q_pos = captures_q
        bounds = []
        for m in range(n):                                  # every prior round holds keys (dropped too)
            r = rounds_now[m]
            bounds.append((r.start, r.end, m))
        bounds.append((q_start, len(kv), n))
        # capture_mode="pre" (engine.py:187-200): the head-summed-logit softmax,
        # scored by rk_round_scores_exact_pre without a capture matrix
        active_mask = [m in set(active) for m in range(n)]
        raw = round_scores(q, kv.keys.view(-1, c.num_heads, c.d_k), q_pos, kv.positions, bounds, n,
                           active=active_mask, capture_mode=c.capture_mode)
        return raw.cpu().numpy()

    def run_turn(self, question, max_decode_steps: int = 16) -> TurnResult:
        if max_decode_steps <= 0:
            raise DomainError("max_decode_steps must be positive")
        model, c = self.model, self.model.config
        L, lw = c.num_layers, self.watershed
        n = len(self.rounds)
        self.store.begin_turn(n)
        ledger = self.store.ledger

        q_body = tokenize(question) if isinstance(question, str) else list(question)
        q_ids = ([SEP_TOKEN] if n > 0 else []) + q_body
        if not q_ids:
            raise DomainError("question must contain at least one token")
        q_start = len(self.token_ids)
        q_positions = np.arange(q_start, q_start + len(q_ids), dtype=np.int64)
        current = Round(n, (q_start, q_start + len(q_ids)), (q_start + len(q_ids), q_start + len(q_ids)))
        rounds_now = self.rounds + [current]

        # step 1: lower blocks on device
        h2d0 = (ledger.h2d_events, ledger.h2d_bytes)
        lower_blocks = self.store.fetch_lower_all(n)
        lower_h2d = (ledger.h2d_events - h2d0[0], ledger.h2d_bytes - h2d0[1])
        working = model.new_cache()
        hist_tokens = self._assemble(working, 0, lw, lower_blocks)

        # step 2: lower-layer prefill; keep the question's rotated queries at Lw-1 for scoring
        if lw > 1:
            hidden, _ = model.forward_range(working, 0, lw - 1, tokens=q_ids, positions=q_positions)
            hidden, q_lw1 = self._forward_capture_q(working, lw - 1, None, hidden, q_positions)
        else:
            hidden, q_lw1 = self._forward_capture_q(working, 0, q_ids, None, q_positions)

        selection_invocations = 0
        distribution = None
        kept: tuple = ()
        active = self.activity.active_rounds(n)
        if n > 0:
            if self.mode == "round":
                raw = self._score((q_lw1, q_positions), working, q_start, n, rounds_now, active)
                distribution = normalize(raw, layer=lw - 1, round_indices=active)
                selection = select(distribution, self.policy)
                selection_invocations = 1
                kept = selection.kept
            else:
                kept = tuple(range(n))

        # step 3: upper blocks for the kept rounds, one batched fetch
        h2d0 = (ledger.h2d_events, ledger.h2d_bytes)
        if self.mode == "round":
            upper_blocks = self.store.fetch_upper(kept)
        else:
            upper_blocks = [self.store.get_block(m, "upper") for m in range(n)]
        upper_h2d = (ledger.h2d_events - h2d0[0], ledger.h2d_bytes - h2d0[1])

        allowed_fn = None
        if self.mode == "round" and self.attend_mode == "mask":
            upper_blocks = [self.store.get_block(m, "upper") for m in range(n)]
            mask_kept = kept

            def allowed_fn(layer, key_positions, _kept=mask_kept):
                return restricted_attention_mask(_kept, rounds_now, q_start, key_positions, upper=layer >= lw)

        upper_assembled = self._assemble(working, lw, L, upper_blocks)

        # step 4: upper-layer prefill
        hidden, _ = model.forward_range(working, lw, L, hidden=hidden, positions=q_positions, allowed_fn=allowed_fn)

        # step 5: greedy decode
        answer_ids = []
        cur, pos = SEP_TOKEN, q_start + len(q_ids)
        generated = 0
        while True:
            answer_ids.append(cur)
            hid, _ = model.forward_range(working, 0, L, tokens=[cur], positions=[pos], allowed_fn=allowed_fn)
            nxt = model.greedy(hid) if hasattr(model, "greedy") else int(torch.argmax(model.logits(hid)[0]))
            if nxt == EOT_TOKEN or generated >= max_decode_steps:
                break
            cur, pos, generated = nxt, pos + 1, generated + 1

        # turn end: store the new round, one batched writeback
        new_count = len(q_ids) + len(answer_ids)
        new_positions = np.arange(q_start, q_start + new_count, dtype=np.int64)
        lower_payload = self._extract_new_rows(working, 0, lw, hist_tokens)
        upper_payload = self._extract_new_rows(working, lw, L, upper_assembled)
        d2h0 = (ledger.d2h_events, ledger.d2h_bytes)
        self.store.put_round(n, lower_payload, upper_payload, new_positions, upper_on_device=True)
        if self.mode == "round":
            self.store.writeback_upper(list(kept) + [n])
        d2h = (ledger.d2h_events - d2h0[0], ledger.d2h_bytes - d2h0[1])

        self.rounds.append(Round(n, (q_start, q_start + len(q_ids)), (q_start + len(q_ids), q_start + new_count)))
        self.token_ids.extend(q_ids + answer_ids)
        self.activity.register_round(n, n)
        dropped = []
        if self.mode == "round":
            dropped = self.activity.update_and_drop(kept, n, len(self.rounds))
            for m in dropped:
                self.store.drop_upper(m)

        kept_tokens = hist_tokens if self.mode == "baseline" else sum(
            self.rounds[m].end - self.rounds[m].start for m in kept)
        peak = ledger.per_turn[-1].device_used_bytes if ledger.per_turn else 0
        metrics = TurnMetrics(
            round_index=n, mode=self.mode, policy=self.policy.kind if self.policy else self.mode,
            append_rows=len(q_ids), decode_steps=len(answer_ids), kept=kept,
            K=len(kept), selection_invocations=selection_invocations,
            upper_h2d_events=upper_h2d[0], upper_h2d_bytes=upper_h2d[1],
            lower_h2d_events=lower_h2d[0], lower_h2d_bytes=lower_h2d[1],
            d2h_events=d2h[0], d2h_bytes=d2h[1], device_used_peak=peak, hist_tokens=hist_tokens,
            hist_tokens_attended=lw * hist_tokens + (L - lw) * kept_tokens,
            distribution=distribution, dropped_rounds=tuple(dropped))
        return TurnResult(answer_ids=answer_ids, metrics=metrics)

    def _forward_capture_q(self, working, l, tokens, hidden, positions):
        """Layer l (= Lw-1) of the question prefill, returning the hidden state
        after the layer and the layer's rotated queries (the scorer's input)."""
        model = self.model
        if tokens is not None:
            x = model.embed_tokens(tokens)
        else:
            x = hidden
        seen = {}
        out, _ = model.forward_range(working, l, l + 1, hidden=x, positions=positions,
                                     layer_hook=lambda _l, q, _kv: seen.setdefault("q", q))
        return out, seen["q"]

    def run_conversation(self, questions, max_decode_steps: int = 16) -> list:
        return [self.run_turn(q, max_decode_steps) for q in questions]

    def end_session(self) -> None:
        self.store.end_session()
