"""ORACLE (test infrastructure only): the reference's toy model and per-turn
round pipeline, restated on the CPU in float32/float64 NumPy.

* model init / RoPE / forward — `pkg/src/roundkv/engine.py:27-287`
  (seeded `default_rng`, draw order embedding then per layer q,k,v,o
  :152-161; interleaved-pair RoPE with float64 trig :175-185; attention +
  residual only, tied logits :270-271)
* `run_turn` round/baseline modes — `pkg/src/roundkv/pipeline.py:192-394`
  (steps 1-5 + writeback; cost simulation omitted: out of scope)

Used to pin the C1 whole-turn parity of the GPU pipeline (kept rounds, answer
ids, ledger) together with golden vectors from the real reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2502_15294_b200.errors import DomainError

from .attention import attention_forward
from .rounds import (
    EOT_TOKEN,
    SEP_TOKEN,
    VOCAB_SIZE,
    Round,
    SelectionPolicy,
    StoreModel,
    aggregate_round_attention,
    normalize,
    select,
)


@dataclass(frozen=True)
class ModelConfig:
    """engine.py:27-55 (capture_mode "post" only: the pipeline default)."""

    num_layers: int = 4
    num_heads: int = 4
    d_model: int = 32
    vocab_size: int = VOCAB_SIZE
    rng_seed: int = 42
    rope_theta: float = 10000.0

    @property
    def d_k(self):
        return self.d_model // self.num_heads


class Model:
    """engine.py:146-287"""

    def __init__(self, c: ModelConfig):
        self.config = c
        rng = np.random.default_rng(c.rng_seed)
        scale = c.d_model ** -0.5
        self.embedding = rng.standard_normal((c.vocab_size, c.d_model)).astype(np.float32)
        out_scale = scale / np.sqrt(2.0 * c.num_layers)
        self.w_q, self.w_k, self.w_v, self.w_o = [], [], [], []
        for _ in range(c.num_layers):
            self.w_q.append((rng.standard_normal((c.d_model, c.d_model)) * scale).astype(np.float32))
            self.w_k.append((rng.standard_normal((c.d_model, c.d_model)) * scale).astype(np.float32))
            self.w_v.append((rng.standard_normal((c.d_model, c.d_model)) * scale).astype(np.float32))
            self.w_o.append((rng.standard_normal((c.d_model, c.d_model)) * out_scale).astype(np.float32))
        half = c.d_k // 2
        self.rope_freq = c.rope_theta ** (-np.arange(half, dtype=np.float64) * 2.0 / c.d_k)

    def rope(self, x, positions):
        """(rows, heads, d_k) rotated by absolute position, engine.py:175-185."""
        ang = positions[:, None].astype(np.float64) * self.rope_freq[None, :]
        cos, sin = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
        x64 = x.astype(np.float64)
        ev, od = x64[..., 0::2], x64[..., 1::2]
        out = np.empty_like(x64)
        out[..., 0::2] = ev * cos - od * sin
        out[..., 1::2] = ev * sin + od * cos
        return out.astype(np.float32)

    def forward_range(self, cache, lo, hi, x, positions, capture_layer=None, allowed_fn=None):
        """engine.py:202-268; `cache[l]` = dict(keys, values, positions)."""
        c = self.config
        h, dk = c.num_heads, c.d_k
        n = x.shape[0]
        cap = None
        for l in range(lo, hi):
            q = self.rope((x @ self.w_q[l]).reshape(n, h, dk), positions)
            k = self.rope((x @ self.w_k[l]).reshape(n, h, dk), positions)
            v = (x @ self.w_v[l]).reshape(n, h, dk)
            kv = cache[l]
            kv["keys"] = np.concatenate([kv["keys"], k.reshape(n, -1)])
            kv["values"] = np.concatenate([kv["values"], v.reshape(n, -1)])
            kv["positions"] = np.concatenate([kv["positions"], positions])
            allowed = allowed_fn(l, kv["positions"]) if allowed_fn else None
            out, scores = attention_forward(
                q, kv["keys"].reshape(-1, h, dk), kv["values"].reshape(-1, h, dk),
                positions, kv["positions"], allowed=allowed, capture=(l == capture_layer))
            if l == capture_layer:
                cap = scores
            x = x + out @ self.w_o[l]
        return x, cap

    def new_cache(self):
        d = self.config.d_model
        return [dict(keys=np.zeros((0, d), np.float32), values=np.zeros((0, d), np.float32),
                     positions=np.zeros(0, np.int64)) for _ in range(self.config.num_layers)]


class Pipeline:
    """pipeline.py:114-433, modes "round" and "baseline", splice attend mode."""

    def __init__(self, model: Model, watershed: int, policy: SelectionPolicy | None = None,
                 mode: str = "round"):
        L = model.config.num_layers
        if not 0 < watershed < L:
            raise DomainError("watershed must satisfy 0 < L_w < L")
        self.model, self.lw, self.policy, self.mode = model, watershed, policy, mode
        self.store = StoreModel(L, watershed, model.config.d_model)
        self.rounds: list[Round] = []
        self.token_ids: list[int] = []
        self.payload = {}            # round -> (lower (lw,2,T,D), upper (L-lw,2,T,D), positions)

    def run_turn(self, question_ids, max_decode_steps=16):
        m, c = self.model, self.model.config
        L, lw = c.num_layers, self.lw
        n = len(self.rounds)
        self.store.begin_turn(n)
        q_ids = ([SEP_TOKEN] if n > 0 else []) + list(question_ids)
        q_start = len(self.token_ids)
        q_pos = np.arange(q_start, q_start + len(q_ids), dtype=np.int64)
        rounds_now = self.rounds + [Round(n, (q_start, q_start + len(q_ids)),
                                          (q_start + len(q_ids), q_start + len(q_ids)))]
        self.store.fetch_lower_all(n)                                   # :218
        work = m.new_cache()
        hist = self._assemble(work, 0, lw, range(n), lower=True)        # :222-223
        x, cap = m.forward_range(work, 0, lw, m.embedding[np.asarray(q_ids)], q_pos,
                                 capture_layer=(lw - 1) if n > 0 else None)
        kept, raw, masses = (), None, None
        if n > 0:
            if self.mode == "round":
                raw = aggregate_round_attention(cap, rounds_now, "question", n, row_offset=q_start)
                dist = normalize(raw, layer=lw - 1)
                masses = dist.masses
                kept = select(dist, self.policy)
            else:
                kept = tuple(range(n))
        if self.mode == "round":
            self.store.fetch_upper(kept)                                # :264
        up = self._assemble(work, lw, L, kept, lower=False)             # :290
        x, _ = m.forward_range(work, lw, L, x, q_pos)                   # :293-296
        answer, cur, pos, gen = [], SEP_TOKEN, q_start + len(q_ids), 0
        while True:                                                     # :302-313
            answer.append(cur)
            hid, _ = m.forward_range(work, 0, L, m.embedding[[cur]], np.array([pos], np.int64))
            nxt = int(np.argmax(hid @ m.embedding.T))
            if nxt == EOT_TOKEN or gen >= max_decode_steps:
                break
            cur, pos, gen = nxt, pos + 1, gen + 1
        cnt = len(q_ids) + len(answer)
        lower = np.stack([np.stack([work[l]["keys"][hist:], work[l]["values"][hist:]]) for l in range(lw)])
        upper = np.stack([np.stack([work[l]["keys"][up:], work[l]["values"][up:]]) for l in range(lw, L)])
        self.payload[n] = (lower, upper, np.arange(q_start, q_start + cnt, dtype=np.int64))
        self.store.put_round(n, cnt, upper_on_device=True)              # :321-323
        if self.mode == "round":
            self.store.writeback_upper(list(kept) + [n])                # :324-325
        self.rounds.append(Round(n, (q_start, q_start + len(q_ids)), (q_start + len(q_ids), q_start + cnt)))
        self.token_ids.extend(q_ids + answer)
        return dict(answer_ids=answer, kept=tuple(kept), raw=raw, masses=masses)

    def _assemble(self, work, lo, hi, rounds, lower):
        total = 0
        for r in rounds:
            lo_p, up_p, pos = self.payload[r]
            p = lo_p if lower else up_p
            for off, l in enumerate(range(lo, hi)):
                work[l]["keys"] = np.concatenate([work[l]["keys"], p[off, 0]])
                work[l]["values"] = np.concatenate([work[l]["values"], p[off, 1]])
                work[l]["positions"] = np.concatenate([work[l]["positions"], pos])
            total += len(pos)
        return total
