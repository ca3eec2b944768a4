"""Batched round-sparse serving engine: one GPU, B independent dialogues.

The B200 restatement of `RoundPipeline.run_turn` (pipeline.py:192-394) for the
BASELINE configurations, with the reference's model (engine.py:146-287:
attention + residual, RoPE, tied logits; here GQA-shaped with bf16 weights,
decode_model.py) running on the GPU for every token:

  1. lower layers [0, Lw) hold every round's KV in HBM
     (`lower`  [B][Lw][K|V][S_lo][Hkv][d]);
     upper layers [Lw, L) of every round live in pinned host memory, one
     contiguous block per round ([L-Lw][K|V][T][Hkv][d], store.py:225-242);
  2. the question runs the lower layers (fused QKV projection + RoPE + KV
     append, decode attention, output projection + residual per layer); at
     layer Lw-1 the exact fp64 scorer (rk_round_scores_exact) gives the Eq. 1
     masses (pipeline.py:225-245), no capture matrix;
  3. rk_select_batch picks the kept rounds bit-exactly (selection.py:87-97),
     and the K ids come back to the host (the API returns a host tuple);
  4. rk_h2d_gather copies the kept rounds' upper KV into the per-dialogue
     working cache (`upper` [B][L-Lw][K|V][S_up][Hkv][d]) on a copy stream, one
     event per upper layer, so upper layer l starts as soon as its rows land
     (store.fetch_upper :254-263 + _assemble :158-169);
  5. the question's upper layers, then the greedy decode (pipeline.py:298-313):
     SEP, then argmax tokens, every token through all L layers and the tied
     logits, replayed from a CUDA graph;
  6. the new round's upper rows are written back to pinned host memory
     (writeback_upper :265-278).

A multi-row question (n_q > 1) takes the tensor-core prefill
(rk_prefill_attention) with the Lw-1 scoring fused, its projections as library
GEMMs (bf16 hi + lo halves of the activations, fp32 output), and an fp64
re-score when the fused scoring's K-boundary margin is small.

Each dialogue's synthetic history (lower KV, host blocks, questions, planted
relevance) is seeded by its GLOBAL dialogue id, so a dialogue gets the same
data and the same kept rounds whichever rank or group serves it.  The decode
runs a fixed number of answer tokens per turn (EOT does not stop a dialogue:
the work per turn is fixed).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, kernels
from .decode_model import SEP_TOKEN, DecodeModel, ModelShape
from .selection import SelectionPolicy, top_k_count
from .stats import build_round_items


@dataclass
class EngineConfig:
    num_layers: int = 32
    watershed: int = 5            # L_w: layers [0, L_w) stay in HBM; scoring at L_w - 1
    hq: int = 32
    hkv: int = 8
    head_dim: int = 128
    rounds: int = 32              # prior rounds in the history
    round_tokens: int = 512       # tokens per prior round
    batch: int = 1                # dialogues on this GPU
    decode_steps: int = 128       # answer tokens per turn (SEP + generated), each through all L layers
    policy: SelectionPolicy = field(default_factory=lambda: SelectionPolicy("top_percent", fraction=0.10))
    host_unique: int = 0          # distinct host round sets (0 = one per dialogue); >0 aliases
    item_chunk: int = 1024        # keys per scoring work item (round-aligned)
    plant: int = 2                # rounds per dialogue with planted relevance at L_w-1 (0 = none)
    plant_beta: float = 0.25
    question_rows: int = 1        # n_q: 1 = single-token question (decode path); > 1 = tensor-core prefill
    round_cache: bool = True      # keep rounds kept again in their working-cache slots (no re-fetch)
    question_variants: int = 4    # distinct questions cycled over turns
    refine_margin: float = 1e-5   # multi-row questions: re-score in fp64 the dialogues whose K-boundary gap
                                  # of the fp32-class fused scoring is below this (measured fused error vs the
                                  # exact masses <= 3e-8 relative on C3, profiles/r02_bench_c3.json;
                                  # 1-row questions always score in fp64)
    model_seed: int = 42
    capture_mode: str = "post"    # "pre": head-summed-logit softmax scoring (engine.py:187-200)
    max_kept: int = 0             # working-cache capacity in rounds (0: top_percent -> its K, else every round)
    drop_window: float = math.inf  # inactivity drop policy (selection.py:168-204); inf = off
    drop_protect: int = 2         # newest rounds never dropped
    kv_dtype: str = "bf16"        # KV caches and host blocks: "bf16" or "f32" (the reference's float32 KV)
    upper_tier: str = "host"      # where the rounds' deep-layer blocks live: "host" (pinned host memory) or
                                  # "hbm" (a GPU's HBM: the peer-HBM tier)
    tier_device: int = -1         # the GPU holding an "hbm" tier (-1: this engine's GPU; another GPU = peer over NVLink)
    step_kernel: str = "layers"   # answer loop: "persistent" = one rk_decode_step launch per token (whole step,
                                  # every layer, one CTA per SM); "layers" = qkv / attention / out kernels per
                                  # layer; "auto" = persistent when supported (batch <= 16, bf16 KV, d = 128)
                                  # and the engine has the GPU to itself (one group)

    @property
    def group(self) -> int:
        return self.hq // self.hkv

    @property
    def shape(self) -> ModelShape:
        return ModelShape(self.num_layers, self.hq, self.hkv, self.head_dim)


def _ptr_array(values) -> np.ndarray:
    return np.asarray(values, dtype=np.uint64)


def _dialogue_gen(device, gid: int, salt: int) -> torch.Generator:
    return torch.Generator(device=device).manual_seed(1_000_003 * (gid + 1) + salt)


class RoundDecodeEngine:
    @staticmethod
    def shapes(c: EngineConfig) -> dict:
        """Round slots K of the working cache and the per-dialogue cache capacities
        (keys) of the lower (s_lo) and upper (s_up) tiers for a config."""
        R, T = c.rounds, c.round_tokens
        k_policy = top_k_count(R, c.policy.fraction, c.policy.min_rounds) if c.policy.kind == "top_percent" else R
        K = min(R, c.max_kept) if c.max_kept > 0 else k_policy
        turn_rows = max(1, c.question_rows) + c.decode_steps
        return dict(K=K, s_lo=R * T + turn_rows, s_up=K * T + turn_rows)

    def __init__(self, cfg: EngineConfig, device: str = "cuda", model: DecodeModel | None = None,
                 dialogues=None, seed: int | None = None, shared: dict | None = None,
                 head_shard: tuple[int, int] = (0, 1), all_reduce=None):
        """shared (cohort serving, cohort.py): views of a larger batch's caches and
        length arrays ('lower', 'upper', 'lower_len', 'upper_len') this engine's
        dialogues live in, so one decode loop can serve several engines' rows.

        head_shard = (rank, world): KV-head sharding of every dialogue over `world`
        ranks (the option for fewer dialogues than GPUs): this engine
        holds kv-heads [rank hkv/world, (rank+1) hkv/world) of every layer (caches,
        host rounds, projections' columns, W_o's rows) and exchanges two things
        through `all_reduce(tensor)` (in-place sum over the ranks, e.g.
        torch.distributed.all_reduce): each layer's output-projection partial
        (B x d_model f32) and, before selection, the per-round fp64 masses of its
        heads — so every rank keeps the same rounds and the same residual stream."""
        self.cfg = c = cfg
        self.dev = torch.device(device)
        self.shard_rank, self.shard_world = head_shard
        if self.shard_world > 1:
            if all_reduce is None:
                raise ValueError("head sharding needs an all_reduce")
            if c.hkv % self.shard_world:
                raise ValueError(f"{c.hkv} kv-heads do not split over {self.shard_world} ranks")
            if c.question_rows > 1 or c.capture_mode != "post" or shared is not None:
                raise ValueError("head sharding serves 1-row questions, capture_mode='post', no cohorts")
            if c.step_kernel == "persistent":
                raise ValueError("head sharding runs the layered answer loop")
        self.all_reduce = all_reduce
        self.hq_l, self.hkv_l = c.hq // self.shard_world, c.hkv // self.shard_world
        self.h0 = self.shard_rank * self.hkv_l              # first kv-head of this shard
        if c.policy.kind not in ("top_percent", "fixed", "adaptive", "all"):
            raise ValueError(f"policy {c.policy.kind!r} is not a round-selection strategy")
        if c.capture_mode not in ("post", "pre"):
            raise ValueError(f"capture_mode must be 'post' or 'pre', got {c.capture_mode!r}")
        if c.kv_dtype not in ("bf16", "f32"):
            raise ValueError(f"kv_dtype must be 'bf16' or 'f32', got {c.kv_dtype!r}")
        if c.step_kernel not in ("auto", "persistent", "layers"):
            raise ValueError(f"step_kernel must be 'auto', 'persistent' or 'layers', got {c.step_kernel!r}")
        self.dtype = torch.bfloat16 if c.kv_dtype == "bf16" else torch.float32
        self.es = 2 if c.kv_dtype == "bf16" else 4           # bytes per KV element
        if c.kv_dtype == "f32" and c.question_rows > 1:
            raise ValueError("multi-row questions (tcgen05 prefill) need bf16 KV")
        L, lw, B, T, R = c.num_layers, c.watershed, c.batch, c.round_tokens, c.rounds
        if dialogues is None:
            base = 0 if seed is None else int(seed)
            dialogues = list(range(base, base + B))
        self.dialogues = [int(x) for x in dialogues]
        if len(self.dialogues) != B:
            raise ValueError(f"{len(self.dialogues)} dialogue ids for batch {B}")
        self.model = model if model is not None else DecodeModel(c.shape, self.dev, seed=c.model_seed,
                                                                 prefill_gemm=c.question_rows > 1,
                                                                 shard=head_shard)
        if self.model.shape != c.shape:
            raise ValueError("model shape does not match the engine config")
        if getattr(self.model, "shard", (0, 1)) != tuple(head_shard):
            raise ValueError(f"model shard {self.model.shard} != engine head_shard {head_shard}")
        self.L_up = L - lw
        # K = the working cache's round slots.  top_percent keeps the same number of
        # rounds every turn (uniform K); fixed / adaptive thresholds and the drop
        # policy's shrinking candidate set keep a data-dependent count per dialogue
        # (<= K), and the upper caches / writeback follow each dialogue's count.
        k_policy = top_k_count(R, c.policy.fraction, c.policy.min_rounds) if c.policy.kind == "top_percent" else R
        self.K = min(R, c.max_kept) if c.max_kept > 0 else k_policy
        if c.policy.kind in ("top_percent", "all") and self.K < k_policy:
            raise ValueError(f"max_kept {c.max_kept} below the {c.policy.kind} kept count {k_policy}")
        self.uniform_k = c.policy.kind in ("top_percent", "all") and math.isinf(c.drop_window)
        if not self.uniform_k and c.question_rows > 1:
            raise ValueError("multi-row questions need a uniform kept count (top_percent / all, no drop policy)")
        from .selection import ActivityLedger
        self.activity = [ActivityLedger(window=c.drop_window, protect_recent=c.drop_protect) for _ in range(B)]
        for led in self.activity:
            for r in range(R):
                led.register_round(r, r)          # round r completed at turn r (pipeline.py:333)
        self.dropped = [[] for _ in range(B)]
        self.n_kept = [self.K] * B                # kept rounds per dialogue, last turn
        self.hist = R * T
        self.nq = nq = max(1, c.question_rows)
        # rows appended to the caches per turn; tokens the decode metric counts
        # (a 1-row question runs through the decode path and counts as one)
        self.turn_rows = nq + c.decode_steps
        self.turn_tokens = 1 + c.decode_steps if nq == 1 else c.decode_steps
        self.s_lo = self.hist + self.turn_rows
        self.s_up = self.K * T + self.turn_rows
        hq_l, hkv_l = self.hq_l, self.hkv_l
        hs = slice(self.h0, self.h0 + hkv_l)                  # this shard's kv-heads of a full-width draw
        self.row = hkv_l * c.head_dim                         # elements per key (this shard's heads)
        D = c.hq * c.head_dim                                 # d_model

        # ---- HBM tiers (per-dialogue synthetic history, seeded by the global dialogue id)
        if shared is not None:
            self.lower, self.upper = shared["lower"], shared["upper"]
            if (tuple(self.lower.shape) != (B, lw, 2, self.s_lo, hkv_l, c.head_dim)
                    or tuple(self.upper.shape) != (B, self.L_up, 2, self.s_up, hkv_l, c.head_dim)):
                raise ValueError("shared caches do not match the engine shape")
        else:
            self.lower = torch.empty((B, lw, 2, self.s_lo, hkv_l, c.head_dim), dtype=self.dtype, device=self.dev)
            self.upper = torch.zeros((B, self.L_up, 2, self.s_up, hkv_l, c.head_dim), dtype=self.dtype,
                                     device=self.dev)
        for b, gid in enumerate(self.dialogues):
            g = _dialogue_gen(self.dev, gid, 1)
            self.lower[b, :, :, : self.hist] = torch.randn((lw, 2, self.hist, c.hkv, c.head_dim), generator=g,
                                                           device=self.dev)[..., hs, :].to(self.dtype)
        # ---- upper tier: one contiguous upper block per (dialogue set, round), in pinned host
        # memory (the reference's host tier) or in a GPU's HBM (the peer-HBM tier)
        if c.upper_tier not in ("host", "hbm"):
            raise ValueError(f"upper_tier must be 'host' or 'hbm', got {c.upper_tier!r}")
        tier_dev = None
        if c.upper_tier == "hbm":
            tier_dev = torch.device("cuda", self.dev.index if c.tier_device < 0 else c.tier_device)
            if tier_dev != self.dev:
                with torch.cuda.device(self.dev):
                    _lib.call("rk_enable_peer_access", tier_dev.index)
        self.tier_dev = tier_dev
        n_sets = B if c.host_unique <= 0 else min(B, c.host_unique)
        self.host_sets = n_sets
        self.host_blocks = []
        pool = torch.randn(1 << 24, generator=torch.Generator().manual_seed(7)).to(self.dtype)   # 16 M noise values
        for u in range(n_sets):
            gid = self.dialogues[u]
            offs = np.random.default_rng(gid + 17).integers(0, 1 << 23, size=R)
            blocks = []
            for r in range(R):
                full = torch.empty((self.L_up, 2, T, c.hkv, c.head_dim), dtype=self.dtype,
                                   pin_memory=self.shard_world == 1)
                flat = full.view(-1)
                o = int(offs[r])
                for s0 in range(0, flat.numel(), 1 << 23):       # distinct window of the pool per block
                    n = min(1 << 23, flat.numel() - s0)
                    flat[s0:s0 + n].copy_(pool[o:o + n])
                blk = full if self.shard_world == 1 else full[..., hs, :].contiguous().pin_memory()
                if tier_dev is not None:
                    blk = blk.to(tier_dev)
                blocks.append(blk)
            self.host_blocks.append(blocks)
        wb_shape = (B, self.L_up, 2, self.turn_rows, hkv_l, c.head_dim)
        self.writeback = (torch.empty(wb_shape, dtype=self.dtype, pin_memory=True) if tier_dev is None
                          else torch.empty(wb_shape, dtype=self.dtype, device=tier_dev))    # the new round's tier

        # ---- lengths and positions (device) and their per-turn reset values
        if shared is not None:
            self.lower_len, self.upper_len = shared["lower_len"], shared["upper_len"]
        else:
            self.lower_len = torch.zeros(B, dtype=torch.int32, device=self.dev)
            self.upper_len = torch.zeros(B, dtype=torch.int32, device=self.dev)
        self.lower_len0 = torch.full((B,), self.hist, dtype=torch.int32, device=self.dev)
        self.upper_len0 = torch.full((B,), self.K * T, dtype=torch.int32, device=self.dev)
        self.pos = torch.zeros(B, dtype=torch.int32, device=self.dev)
        self.pos_q0 = torch.full((B,), self.hist, dtype=torch.int32, device=self.dev)        # 1-row question
        self.pos_dec0 = torch.full((B,), self.hist + nq, dtype=torch.int32, device=self.dev)  # SEP of the answer

        # ---- round-aligned scoring items at layer L_w-1 (prior rounds + the question)
        bounds = [[(r * T, (r + 1) * T, r) for r in range(R)] + [(self.hist, self.hist + nq, R)] for _ in range(B)]
        self.items, self.n_items = kernels.items_tensor(bounds, c.item_chunk, self.dev)
        self.n_items_host = [len(build_round_items(b_, c.item_chunk)) for b_ in bounds]

        # ---- activations (one decode row per dialogue)
        self.x = torch.zeros((B, D), dtype=torch.float32, device=self.dev)          # residual stream
        self.q_buf = torch.zeros((B, hq_l, c.head_dim), dtype=torch.float32, device=self.dev)
        self.k_new = torch.zeros((B, hkv_l, c.head_dim), dtype=self.dtype, device=self.dev)
        self.v_new = torch.zeros((B, hkv_l, c.head_dim), dtype=self.dtype, device=self.dev)
        self.attn = torch.zeros((B, hq_l * c.head_dim), dtype=torch.float32, device=self.dev)   # attention output
        # head sharding: this shard's output-projection partial, summed over the ranks
        self.delta = torch.zeros((B, D), dtype=torch.float32, device=self.dev) if self.shard_world > 1 else None
        self.tokens = torch.zeros(B, dtype=torch.int32, device=self.dev)
        self.sep = torch.full((B,), SEP_TOKEN, dtype=torch.int32, device=self.dev)
        # answer ids of the turn: [SEP, generated...] (the last entry is the argmax after the final forward)
        self.answer = torch.full((B, c.decode_steps + 1), SEP_TOKEN, dtype=torch.int32, device=self.dev)
        self.answer_host = torch.zeros((B, c.decode_steps + 1), dtype=torch.int32, pin_memory=True)
        # this engine's own split-K workspaces (groups run concurrently on their own streams)
        self.lm_ws = torch.zeros(max(256, _lib.lib.rk_lm_head_workspace_bytes(B, self.model.shape.vocab, D)),
                                 dtype=torch.uint8, device=self.dev)
        self.proj_ws = kernels.proj_workspace(B, D, max(self.model.shape.qkv_width, D), self.dev)
        if nq > 1:
            self.xq = torch.zeros((B * nq, D), dtype=torch.float32, device=self.dev)
            self.qq = torch.zeros((B * nq, hq_l, c.head_dim), dtype=torch.float32, device=self.dev)
            self.qout = torch.zeros((B, nq, hq_l, c.head_dim), dtype=torch.float32, device=self.dev)
            self.q_pos = torch.arange(self.hist, self.hist + nq, dtype=torch.int64, device=self.dev)
            self.pos_rows = torch.arange(self.hist, self.hist + nq, dtype=torch.int32,
                                         device=self.dev).repeat(B).contiguous()
            self.k_pos_lo = torch.arange(self.hist + nq, dtype=torch.int64, device=self.dev)
            self.k_pos_up = torch.zeros((B, self.K * T + nq), dtype=torch.int64, device=self.dev)
            self.k_pos_up_host = torch.zeros((B, self.K * T + nq), dtype=torch.int64, pin_memory=True)
            self.bad_row = torch.zeros(1, dtype=torch.int32, device=self.dev)
            self.lower_len_q = torch.full((B,), self.hist + nq, dtype=torch.int32, device=self.dev)
            self.upper_len_q = torch.full((B,), self.K * T + nq, dtype=torch.int32, device=self.dev)

        # ---- questions: `question_variants` token sequences per dialogue, cycled over turns
        V = max(1, c.question_variants)
        qt = np.stack([np.stack([np.random.default_rng([gid, v, 99]).integers(0, 256, size=nq)
                                 for gid in self.dialogues]) for v in range(V)]).astype(np.int32)   # (V, B, nq)
        self.q_tok_all = torch.from_numpy(qt).to(self.dev)
        self.q_tok_host = torch.from_numpy(qt).pin_memory()
        self.q_tok = torch.zeros((B, nq), dtype=torch.int32, device=self.dev)      # this turn's question (graph input)
        self.turn = 0
        if c.plant:
            self._plant()
        # working-cache slot -> round id per dialogue (-1 = empty); see assign_slots
        self.slot_round = np.full((B, self.K), -1, dtype=np.int64)
        self.last_copied_rounds = 0

        # ---- scratch (this engine's own: groups run concurrently on their own streams)
        self.raw = torch.empty((B, R), dtype=torch.float64, device=self.dev)
        self.active_host = torch.ones((B, R), dtype=torch.uint8, pin_memory=True)
        self.active_dev = torch.ones((B, R), dtype=torch.uint8, device=self.dev)
        self.sel_out = None
        ws_bytes = _lib.lib.rk_decode_workspace_bytes(B, hq_l, hkv_l, c.head_dim, max(592, self.items.shape[1] * 8))
        self.ws = torch.zeros(max(256, int(ws_bytes)), dtype=torch.uint8, device=self.dev)
        ex_bytes = _lib.lib.rk_round_scores_exact_workspace_bytes(B, nq, hq_l, self.items.shape[1], R)
        self.ws_exact = torch.zeros(max(256, int(ex_bytes)), dtype=torch.uint8, device=self.dev)
        self.q_pos_1 = torch.full((1,), self.hist, dtype=torch.int64, device=self.dev)
        self.margin = torch.zeros(B, dtype=torch.float64, device=self.dev)
        self.margin_host = torch.zeros(B, dtype=torch.float64, pin_memory=True)
        self.min_margin = math.inf            # smallest K-boundary margin seen (fp64 masses)
        self.refined_turns = 0                # multi-row turns re-scored in fp64
        self.refined_dialogues = 0            # dialogue-turns re-scored
        self.max_fused_rel_err = 0.0          # largest |fused - exact| / exact mass seen when re-scoring
        self.copy_stream = torch.cuda.Stream(self.dev)
        self.compute_stream = torch.cuda.Stream(self.dev)
        # torch creates CUDA events lazily: record once so the handles exist
        # before librk records them on the copy stream (rk_h2d_gather)
        self.layer_events = [torch.cuda.Event() for _ in range(self.L_up)]
        for ev in self.layer_events:
            ev.record(self.copy_stream)
        self.decode_done = torch.cuda.Event()
        self.decode_done.record(self.compute_stream)
        torch.cuda.synchronize()
        assert all(ev.cuda_event for ev in self.layer_events)
        self.kept_host = torch.empty((B, R), dtype=torch.int32, pin_memory=True)
        self.meta_host = torch.empty((3, B), dtype=torch.int32, pin_memory=True)
        self.graph_a = None
        self.graph_b = None
        self.graphs_b1 = None      # multi-row questions: one graph per upper layer (replayed between gather waits)
        # ---- the persistent whole-step kernel (rk_decode_step) for the answer loop
        supported = self.shard_world == 1 and kernels.decode_step_supported(B, c.hq, c.hkv, c.head_dim, self.dtype)
        if c.step_kernel == "persistent" and not supported:
            raise ValueError("step_kernel='persistent' needs batch <= 16, group <= 8, head_dim 128 and bf16 KV")
        self.persistent = supported and c.step_kernel in ("auto", "persistent")
        if self.persistent:
            m = self.model
            self.w_qkv_table = torch.tensor([w.data_ptr() for w in m.w_qkv_packed], dtype=torch.int64, device=self.dev)
            self.w_o_table = torch.tensor([w.data_ptr() for w in m.w_o_packed], dtype=torch.int64, device=self.dev)
            self.step_ws = kernels.decode_step_workspace(B, L, c.hq, c.hkv, c.head_dim, m.shape.vocab, self.dev)
            self.step_args = [kernels.decode_step_args(
                self.x, self.lower, self.upper, self.lower_len, self.upper_len, self.pos, m.freq, self.w_qkv_table,
                self.w_o_table, m.emb_packed, m.emb, c.hq, c.hkv, lw, self.step_ws, tokens=self.tokens,
                tokens_log=self.answer[:, t + 1:], log_stride=self.answer.shape[1], vocab=m.shape.vocab)
                for t in range(c.decode_steps)]
        self.last_kept = None
        self.marks = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        self.window_log = None        # list of (start, end) decode-loop events per turn when enabled
        self.copy_marks = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    # ------------------------------------------------------------------ data
    def _plant(self):
        """Raise the question's attention on `plant` rounds per dialogue at
        layer L_w-1 (SURVEY.md §8d planted relevance): add beta * sqrt(d) * u
        to those rounds' keys, u the unit query direction of the question's
        first variant at that layer, approximated by its last token's embedding
        projected and rotated (x W_q, RoPE at that token's position)."""
        c = self.cfg
        lw1 = c.watershed - 1
        m = self.model
        tok = self.q_tok_all[0, :, -1].long()                            # (B,) last question token
        x = m.emb[tok].float().contiguous()
        q = torch.zeros((c.batch, self.hq_l, c.head_dim), dtype=torch.float32, device=self.dev)
        kd = torch.zeros((c.batch, self.hkv_l, c.head_dim), dtype=self.dtype, device=self.dev)
        vd = torch.zeros_like(kd)
        pos = torch.full((c.batch,), self.hist + self.nq - 1, dtype=torch.int32, device=self.dev)
        kernels.qkv_rope(x, m.w_qkv_packed[lw1], self.hq_l, self.hkv_l, c.head_dim, pos, m.freq, q, kd, vd)
        qm = q.view(c.batch, self.hkv_l, c.group, c.head_dim).mean(dim=2)
        u = qm / qm.norm(dim=-1, keepdim=True)
        self.planted = []
        for b, gid in enumerate(self.dialogues):
            rng = np.random.default_rng(gid + 1234)
            rs = sorted(rng.choice(c.rounds, size=min(c.plant, c.rounds), replace=False).tolist())
            self.planted.append(rs)
            for r in rs:
                sl = self.lower[b, lw1, 0, r * c.round_tokens:(r + 1) * c.round_tokens].float()
                sl += c.plant_beta * math.sqrt(c.head_dim) * u[b][None]
                self.lower[b, lw1, 0, r * c.round_tokens:(r + 1) * c.round_tokens] = sl.to(self.dtype)

    # ------------------------------------------------------------------ kernels
    def _caches(self, l: int):
        c = self.cfg
        if l < c.watershed:
            return self.lower[:, l, 0], self.lower[:, l, 1], self.lower_len, self.s_lo
        u = l - c.watershed
        return self.upper[:, u, 0], self.upper[:, u, 1], self.upper_len, self.s_up

    def _layer(self, l: int, advance: bool):
        """One decode row per dialogue through layer l: fused QKV projection +
        RoPE (rk_qkv_rope), decode attention with the KV append
        (rk_decode_attention), output projection + residual (rk_out_proj)."""
        c, m = self.cfg, self.model
        kc, vc, ln, cap = self._caches(l)
        kernels.qkv_rope(self.x, m.w_qkv_packed[l], self.hq_l, self.hkv_l, c.head_dim, self.pos, m.freq, self.q_buf,
                         self.k_new, self.v_new, ws=self.proj_ws)
        kernels.decode_attention(self.q_buf, kc, vc, ln, cap, k_new=self.k_new, v_new=self.v_new,
                                 out=self.attn.view(c.batch, self.hq_l, c.head_dim), ws=self.ws,
                                 advance=ln if advance else None)
        if self.shard_world > 1:
            # row-parallel W_o: this shard's heads' contribution, summed over the ranks
            self.delta.zero_()
            kernels.out_proj(self.attn, m.w_o_packed[l], self.delta, ws=self.proj_ws)
            self.all_reduce(self.delta)
            self.x += self.delta
        else:
            kernels.out_proj(self.attn, m.w_o_packed[l], self.x, ws=self.proj_ws)

    def _attn_launches(self, l: int, advance: bool = False) -> int:
        c = self.cfg
        kc, _, _, cap = self._caches(l)
        plan = kernels.decode_plan(c.batch, self.hq_l, self.hkv_l, c.head_dim, kc.dtype, cap, kc.stride(0), False)
        return (1 + int(advance)) if plan > 0 else 2

    def decode_kernel_desc(self) -> str:
        """The decode attention kernels the answer tokens run (lower / upper layers)."""
        c = self.cfg
        if self.persistent:
            return "step_kernel (one persistent launch per token: every layer's projections, attention, merge)"
        out = []
        for name, kc, cap in (("lower", self.lower[:, 0, 0], self.s_lo), ("upper", self.upper[:, 0, 0], self.s_up)):
            plan = kernels.decode_plan(c.batch, self.hq_l, self.hkv_l, c.head_dim, kc.dtype, cap, kc.stride(0))
            out.append(f"{name}: " + (f"decode_cluster_kernel, {plan} CTA(s) per (dialogue, kv-head)" if plan > 0
                                      else "decode_mma_kernel + decode_merge_kernel"))
        return "; ".join(out)

    def launches_per_token(self) -> int:
        """Kernels of one answer token: per layer qkv_rope + attention (+ length
        advance) + out_proj; then the logits GEMV + argmax/embed."""
        c = self.cfg
        if self.persistent:
            return 1
        return sum(2 + self._attn_launches(l, advance=(l == c.watershed - 1 or l == c.num_layers - 1))
                   for l in range(c.num_layers)) + 2

    def _set_turn_lengths(self):
        self.lower_len.copy_(self.lower_len0)
        self.upper_len.copy_(self.upper_len0)

    def _phase_a(self):
        """Question through the lower layers, watershed scoring, selection.

        A 1-row question is scored exactly: after layer Lw-1 appended the
        question's key, rk_round_scores_exact recomputes the layer's logits with
        the reference kernel's fp64 arithmetic (one extra read of that layer's
        keys, ~5 us per dialogue), so the kept rounds are the reference's by
        construction, not within a tolerance."""
        if self.nq > 1:
            return self._phase_a_prefill()
        c = self.cfg
        self._set_turn_lengths()
        self.pos.copy_(self.pos_q0)
        kernels.embed(self.q_tok.view(-1), self.model.emb, self.x)
        for l in range(c.watershed):
            self._layer(l, advance=(l == c.watershed - 1))
        lw1 = c.watershed - 1
        kernels.round_scores_exact(self.q_buf.unsqueeze(1), self.lower[:, lw1, 0], self.q_pos_1, self.items,
                                   c.rounds, seq_len=self.lower_len, n_items=self.n_items, raw=self.raw,
                                   ws=self.ws_exact, capture_mode=c.capture_mode)
        if self.shard_world > 1:
            self.all_reduce(self.raw)      # Eq. 1 sums over heads: every rank selects from the same masses
        self._select()

    def _select(self):
        """Device selection over every dialogue's active rounds (bit-exact,
        selection.py:63-126): kept round ids, counts and the K-boundary margin.
        With a per-dialogue kept count the upper caches' lengths follow it."""
        pol = self.cfg.policy
        if self.uniform_k and pol.kind == "top_percent":
            self.masses, self.kept_pos, self.sel_meta = kernels.select_batch(self.raw, "top_percent", k_top=self.K)
            kernels.selection_margin(self.masses, "top_percent", k_top=self.K, out=self.margin)
            return
        self.sel_out = kernels.select_batch_active(self.raw, pol, active=self.active_dev, out=self.sel_out)
        self.masses, self.kept_pos, self.sel_meta, margin = self.sel_out
        self.margin.copy_(margin)
        if not self.uniform_k:
            torch.mul(self.sel_meta[0], self.cfg.round_tokens, out=self.upper_len)

    def _refine_exact(self, dialogues):
        """Multi-row question whose fused fp32-class scoring left a K-boundary
        gap below cfg.refine_margin: re-score those dialogues with
        rk_round_scores_exact (fp64, the reference's arithmetic) and select
        again (eager, on the current stream).  Records the largest relative
        difference between the fused and the exact masses (the fused scorer's
        measured error, which the margin must exceed)."""
        c = self.cfg
        lw1 = c.watershed - 1
        qq = self.qq.view(c.batch, self.nq, c.hq, c.head_dim)
        fused = self.raw.clone()
        for b in dialogues:
            kernels.round_scores_exact(qq[b:b + 1], self.lower[b:b + 1, lw1, 0], self.q_pos, self.items[b:b + 1],
                                       c.rounds, seq_len=self.lower_len[b:b + 1], n_items=self.n_items[b:b + 1],
                                       raw=self.raw[b:b + 1], ws=self.ws_exact, capture_mode=c.capture_mode)
        if c.capture_mode == "post":
            rows = torch.as_tensor(list(dialogues), device=self.dev)
            ex, fu = self.raw[rows], fused[rows]
            err = ((fu - ex).abs() / ex.abs().clamp_min(1e-300)).max()
            self.max_fused_rel_err = max(self.max_fused_rel_err, float(err))
        self._select()
        self.refined_turns += 1
        self.refined_dialogues += len(dialogues)

    # ---- multi-row question: projections as library GEMMs, tensor-core prefill attention
    @staticmethod
    def _proj_rows(x: torch.Tensor, w_kn: torch.Tensor) -> torch.Tensor:
        """x (m, k) f32 @ w (k, n) bf16 with fp32 output, x split into bf16
        hi + lo halves (~16 mantissa bits, as the decode projections)."""
        hi = x.to(torch.bfloat16)
        lo = (x - hi.float()).to(torch.bfloat16)
        return torch.mm(hi, w_kn, out_dtype=torch.float32) + torch.mm(lo, w_kn, out_dtype=torch.float32)

    def _prefill_layer(self, l: int, items: bool):
        c, m = self.cfg, self.model
        nq, hist, KT = self.nq, self.hist, self.K * c.round_tokens
        lower = l < c.watershed
        qkv = self._proj_rows(self.xq, m.w_qkv_kn[l])
        if lower:
            kb, vb = self.lower[0, l, 0, hist], self.lower[0, l, 1, hist]
            gstride = self.lower.stride(0)
        else:
            u = l - c.watershed
            kb, vb = self.upper[0, u, 0, KT], self.upper[0, u, 1, KT]
            gstride = self.upper.stride(0)
        kernels.rope_rows(qkv, c.hq, c.hkv, c.head_dim, self.pos_rows, m.freq, self.qq, kb, vb, self.row, nq,
                          gstride)
        qq = self.qq.view(c.batch, nq, c.hq, c.head_dim)
        for b in range(c.batch):
            if lower:
                kernels.prefill_attention(
                    qq[b], self.lower[b, l, 0, :hist + nq], self.lower[b, l, 1, :hist + nq], self.q_pos,
                    self.k_pos_lo, out=self.qout[b], bad_row=self.bad_row,
                    items=self.items[b, :self.n_items_host[b]] if items else None,
                    n_bins=c.rounds if items else 0, raw=self.raw[b] if items else None)
            else:
                u = l - c.watershed
                kernels.prefill_attention(
                    qq[b], self.upper[b, u, 0, :KT + nq], self.upper[b, u, 1, :KT + nq], self.q_pos,
                    self.k_pos_up[b], out=self.qout[b], bad_row=self.bad_row)
        self.xq += self._proj_rows(self.qout.view(c.batch * nq, -1), m.w_o_kn[l])

    def _phase_a_prefill(self):
        """n_q question rows through the lower layers (causal over the full
        history + the question, pipeline.py:225-230); at layer L_w-1 the same
        pass leaves the Eq. 1 round masses (fused scoring), then selection."""
        c = self.cfg
        self._set_turn_lengths()
        kernels.embed(self.q_tok.view(-1), self.model.emb, self.xq)
        for l in range(c.watershed):
            self._prefill_layer(l, items=(l == c.watershed - 1))
        self.lower_len.copy_(self.lower_len_q)
        self._select()

    def _phase_b1_prefill(self, layer_wait: bool):
        """n_q question rows through the upper layers over the kept rounds +
        the question (pipeline.py:292-296); positions keep their original
        values, so the splice equals the masked attention (engine.py:94-112)."""
        c = self.cfg
        nq, T, KT = self.nq, c.round_tokens, self.K * c.round_tokens
        for b in range(c.batch):       # key positions of the working cache: its round slots, then the question
            pos = self.k_pos_up_host[b]
            for i, r in enumerate(self.slot_round[b]):
                pos[i * T:(i + 1) * T] = torch.arange(int(r) * T, (int(r) + 1) * T)
            pos[KT:KT + nq] = torch.arange(self.hist, self.hist + nq)
        self.k_pos_up.copy_(self.k_pos_up_host, non_blocking=True)
        for l in range(c.watershed, c.num_layers):
            if layer_wait:
                torch.cuda.current_stream().wait_event(self.layer_events[l - c.watershed])
            if self.graphs_b1 is not None:
                self.graphs_b1[l - c.watershed].replay()
            else:
                self._prefill_layer(l, items=False)
        self.upper_len.copy_(self.upper_len_q)

    def _phase_b1(self, layer_wait: bool):
        """The question through the upper layers (each waits for its rows)."""
        if self.nq > 1:
            return self._phase_b1_prefill(layer_wait)
        c = self.cfg
        for l in range(c.watershed, c.num_layers):
            if layer_wait:
                torch.cuda.current_stream().wait_event(self.layer_events[l - c.watershed])
            self._layer(l, advance=(l == c.num_layers - 1))

    def prefill_flops_per_turn(self) -> float:
        """Algorithmic attention FLOPs of the question prefill (QK^T + PV once,
        causal visible pairs only): 4 * Hq * d per visible (row, key) pair."""
        if self.nq == 1:
            return 0.0
        c = self.cfg
        nq = self.nq
        causal = nq * (nq + 1) / 2
        pairs = c.watershed * (nq * self.hist + causal) + self.L_up * (nq * self.K * c.round_tokens + causal)
        return 4.0 * c.hq * c.head_dim * pairs * c.batch

    def _phase_b2(self):
        """The answer (pipeline.py:298-313): SEP at the position after the
        question, then `decode_steps` forwards through all L layers, each
        followed by the tied logits + first-max argmax (rk_lm_head), which also
        embeds the next token and advances the position."""
        c, m = self.cfg, self.model
        self.pos.copy_(self.pos_dec0)
        kernels.embed(self.sep, m.emb, self.x)
        if self.persistent:
            for t in range(c.decode_steps):
                kernels.decode_step(self.step_args[t])
            return
        for t in range(c.decode_steps):
            for l in range(c.num_layers):
                self._layer(l, advance=(l == c.watershed - 1 or l == c.num_layers - 1))
            kernels.lm_head(self.x, m.emb_packed, m.shape.vocab, m.emb, self.x, self.tokens, self.pos,
                            tokens_log=self.answer[:, t + 1:], log_stride=self.answer.shape[1], ws=self.lm_ws)

    def _phase_wb(self):
        """Writeback of the new round's upper rows to pinned host memory
        (store.writeback_upper, pipeline.py:324-325): one strided D2H."""
        T = self.cfg.round_tokens
        if self.uniform_k:
            self.writeback.copy_(self.upper[:, :, :, self.K * T:], non_blocking=True)
            return
        for b, n in enumerate(self.n_kept):      # the turn's rows follow each dialogue's kept rounds
            self.writeback[b].copy_(self.upper[b, :, :, n * T:n * T + self.turn_rows], non_blocking=True)

    # ------------------------------------------------------------------ gather
    def assign_slots(self, kept):
        """Cross-turn round cache: the working cache's K
        round slots keep the rounds that stay kept; only newly kept rounds are
        fetched, into the slots of the rounds that left.  Decode attention is
        invariant to the order of the cached keys (every cached key is visible
        to a decode token), so the splice need not be ascending; the question
        prefill reads the slots' original positions (k_pos_up).  Without the
        cache every kept round is fetched, ascending (pipeline._assemble).
        Returns [(dialogue, slot, round)] copies."""
        copies = []
        for b in range(self.cfg.batch):
            new = [int(r) for r in kept[b]]
            nb = len(new)
            if nb > self.K:
                raise RuntimeError(f"dialogue {self.dialogues[b]} keeps {nb} rounds > working-cache capacity "
                                   f"{self.K} (raise EngineConfig.max_kept)")
            cur = self.slot_round[b]
            if not self.cfg.round_cache:
                cur[:] = -1
            # the kept rounds occupy slots [0, nb) (the cache rows stay contiguous)
            stay = set(new) & set(int(cur[i]) for i in range(nb) if cur[i] >= 0)
            for i in range(self.K):
                if i >= nb or cur[i] not in stay:
                    cur[i] = -1
            free = [i for i in range(nb) if cur[i] < 0]
            for i, r in zip(free, [r for r in new if r not in stay]):
                cur[i] = r
                copies.append((b, i, r))
        self.last_copied_rounds = len(copies)
        return copies

    def gather_plan(self, kept: list):
        """Per upper layer: (src, spitch, dst, dpitch, width, height) arrays, one
        2-row (K, V) strided copy per (dialogue, newly kept round)."""
        c = self.cfg
        es = self.es
        T = c.round_tokens
        width = T * self.row * es
        spitch = width
        dpitch = self.s_up * self.row * es
        copies = self.assign_slots(kept)
        plans = []
        for u in range(self.L_up):
            srcs, dsts = [], []
            for b, i, r in copies:
                blk = self.host_blocks[b % self.host_sets][r]
                srcs.append(blk.data_ptr() + u * 2 * T * self.row * es)
                dsts.append(self.upper[b, u, 0, i * T].data_ptr())
            n = len(srcs)
            plans.append(dict(n=n, src=_ptr_array(srcs), dst=_ptr_array(dsts),
                              spitch=np.full(n, spitch, np.uint64), dpitch=np.full(n, dpitch, np.uint64),
                              width=np.full(n, width, np.uint64), height=np.full(n, 2, np.uint64)))
        return plans

    def issue_gather(self, plans):
        """rk_h2d_gather (host tier) or rk_peer_gather (HBM tier) per upper layer
        on the copy stream, one event per layer."""
        vp = C.c_void_p
        s = self.copy_stream
        total = 0
        for u, pl in enumerate(plans):
            ev = self.layer_events[u]
            assert ev.cuda_event, "gather event not created"
            _lib.call("rk_h2d_gather" if self.tier_dev is None else "rk_peer_gather", pl["n"], pl["src"].ctypes.data_as(vp), pl["spitch"].ctypes.data_as(vp),
                      pl["dst"].ctypes.data_as(vp), pl["dpitch"].ctypes.data_as(vp), pl["width"].ctypes.data_as(vp),
                      pl["height"].ctypes.data_as(vp), s.cuda_stream, ev.cuda_event)
            total += int((pl["width"] * pl["height"]).sum())
        return total

    # ------------------------------------------------------------------ turn
    def prepare(self, e2e: bool = False, decode_graph: bool = True):
        """Warm up (module attributes, workspace) and capture the CUDA graphs
        (decode_graph=False: the answer loop runs elsewhere, cohort.py)."""
        with torch.cuda.stream(self.compute_stream):
            self.run_turn_eager()                     # warm-up, sets kernel attributes
            if self.nq > 1:                           # load the fp64 re-score kernels now, not in a timed turn
                c = self.cfg
                kernels.round_scores_exact(self.qq.view(c.batch, self.nq, c.hq, c.head_dim)[:1],
                                           self.lower[:1, c.watershed - 1, 0], self.q_pos, self.items[:1],
                                           c.rounds, seq_len=self.lower_len[:1], n_items=self.n_items[:1],
                                           raw=torch.empty_like(self.raw[:1]), ws=self.ws_exact,
                                           capture_mode=c.capture_mode)
                r0 = self.raw[torch.as_tensor([0], device=self.dev)]            # the error check's torch ops
                float(((r0 - r0).abs() / r0.abs().clamp_min(1e-300)).max())
            torch.cuda.synchronize()
            if self.graph_a is None:
                self.graph_a = torch.cuda.CUDAGraph()
                with torch.cuda.graph(self.graph_a, stream=self.compute_stream):
                    self._phase_a()
                if decode_graph:
                    self.graph_b = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(self.graph_b, stream=self.compute_stream):
                        self._phase_b2()
                if self.nq > 1 and self.uniform_k:
                    # the question's upper layers: ~40 launches per layer (projections, RoPE, one
                    # prefill per dialogue) whose host launch cost exceeded their GPU time at C3;
                    # one graph per layer keeps the per-layer wait on its gathered rows between
                    # replays.  Replayed in capture order on one stream, so they share one pool
                    pool = torch.cuda.graph_pool_handle()
                    graphs = []
                    for l in range(self.cfg.watershed, self.cfg.num_layers):
                        g = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(g, stream=self.compute_stream, pool=pool):
                            self._prefill_layer(l, items=False)
                        graphs.append(g)
                    self.graphs_b1 = graphs
        torch.cuda.synchronize()

    def _select_to_host(self, refine: bool = True):
        self.kept_host.copy_(self.kept_pos, non_blocking=True)
        self.meta_host.copy_(self.sel_meta, non_blocking=True)
        self.margin_host.copy_(self.margin, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        if int(self.meta_host[2].abs().sum()) != 0:
            raise RuntimeError("selection reported a negative raw mass")
        if refine and self.nq > 1:
            # the fused prefill scoring is the "post" statistic: "pre" questions are always
            # scored exactly; otherwise only the dialogues whose K-boundary gap is small
            if self.cfg.capture_mode == "pre":
                low = list(range(self.cfg.batch))
            else:
                low = [b for b in range(self.cfg.batch) if float(self.margin_host[b]) < self.cfg.refine_margin]
            if low:
                self._refine_exact(low)
                return self._select_to_host(refine=False)
        self.min_margin = min(self.min_margin, float(self.margin_host.min()))
        kept = []
        for b in range(self.cfg.batch):
            n = int(self.meta_host[0, b])
            kept.append(self.kept_host[b, :n].numpy().copy())
        self.n_kept = [len(k) for k in kept]
        self._update_activity(kept)
        return kept

    def _update_activity(self, kept):
        """The inactivity drop policy (pipeline.py:333-338, selection.py:183-204):
        record the turn's kept rounds, drop the rounds idle for drop_window turns
        (their upper blocks leave the host tier, store.drop_upper) and take them
        out of the next turn's candidate set (the active mask the selector reads)."""
        if math.isinf(self.cfg.drop_window):
            return
        R = self.cfg.rounds
        now = R + self.turn - 1                    # the turn being served (rounds 0..R-1 came before it)
        for b, k in enumerate(kept):
            drops = self.activity[b].update_and_drop([int(x) for x in k], now, R)
            self.dropped[b] = drops
            for r in drops:
                self.active_host[b, r] = 0
                if self.host_sets == self.cfg.batch:
                    self.host_blocks[b][r] = None   # store.drop_upper: the payload is gone
        self.active_dev.copy_(self.active_host, non_blocking=True)

    def _set_question(self, e2e: bool = False):
        """This turn's question (variant turn % V) into the question input: from
        pinned host memory through the public API (e2e), else device-resident."""
        v = self.turn % self.q_tok_all.shape[0]
        self.q_tok.copy_(self.q_tok_host[v] if e2e else self.q_tok_all[v], non_blocking=True)
        self.turn += 1

    def run_turn_eager(self):
        """Whole turn without graphs (first call / debugging)."""
        self._set_question()
        self._phase_a()
        kept = self._select_to_host()
        self.copy_stream.wait_stream(torch.cuda.current_stream())
        self.issue_gather(self.gather_plan(kept))
        self._phase_b1(layer_wait=True)
        self._phase_b2()
        self.decode_done.record()
        self.copy_stream.wait_event(self.decode_done)
        with torch.cuda.stream(self.copy_stream):
            self._phase_wb()
        torch.cuda.current_stream().wait_stream(self.copy_stream)
        self.last_kept = kept
        return kept

    def run_turn(self, e2e: bool = False, on_gather=None):
        """One turn on the compute stream with the captured graphs.  Returns the
        kept rounds per dialogue (host) and the H2D bytes moved.  With e2e the
        question tokens come from pinned host memory and the answer ids go back
        to it (the public API's input and output).  Timing marks (compute
        stream): 0 start, 1 after scoring+select, 2 after the question's upper
        layers, 3 after the decode tokens, 4 after writeback; copy_marks bracket
        the H2D gather on the copy stream."""
        m = self.marks
        with torch.cuda.stream(self.compute_stream):
            m[0].record()
            self._set_question(e2e)
            self.graph_a.replay()
            m[1].record()
            kept = self._select_to_host()
            self.copy_stream.wait_stream(self.compute_stream)
            plans = self.gather_plan(kept)
            self.copy_marks[0].record(self.copy_stream)
            nbytes = self.issue_gather(plans)
            self.copy_marks[1].record(self.copy_stream)
            if on_gather is not None:
                on_gather()
            self.last_h2d_bytes = nbytes
            self._phase_b1(layer_wait=True)
            m[2].record()
            if self.window_log is not None:          # per-turn decode window (bench roofline)
                a = torch.cuda.Event(enable_timing=True)
                a.record(self.compute_stream)
            self.graph_b.replay()
            m[3].record()
            if self.window_log is not None:
                b = torch.cuda.Event(enable_timing=True)
                b.record(self.compute_stream)
                self.window_log.append((a, b))
            if e2e:
                self.answer_host.copy_(self.answer, non_blocking=True)
            # writeback of the new round's upper rows on the copy stream: it
            # overlaps the next turn's scoring; the next gather queues behind it
            self.decode_done.record(self.compute_stream)
        self.copy_stream.wait_event(self.decode_done)
        with torch.cuda.stream(self.copy_stream):
            self._phase_wb()
            m[4].record(self.copy_stream)
        self.last_kept = kept
        return kept, nbytes

    def answers(self) -> np.ndarray:
        """(B, decode_steps) answer ids of the last turn (SEP first), as the reference's answer_ids."""
        torch.cuda.synchronize()
        return self.answer[:, : self.cfg.decode_steps].cpu().numpy()

    def turn_breakdown_ms(self) -> dict:
        """Elapsed times of the last turn (call after synchronising)."""
        m = self.marks
        return dict(score_select=m[0].elapsed_time(m[1]), gather_upper_prefill=m[1].elapsed_time(m[2]),
                    decode=m[2].elapsed_time(m[3]), writeback_copy_stream=m[3].elapsed_time(m[4]),
                    turn=m[0].elapsed_time(m[3]), h2d=self.copy_marks[0].elapsed_time(self.copy_marks[1]))

    def kernel_launches_per_turn(self) -> int:
        c = self.cfg
        answer = 1 + self.launches_per_token() * c.decode_steps            # SEP embed + tokens
        if self.nq > 1:   # embed; per layer rope_rows + per dialogue (bad-row fill, q prep, tcgen05 pass, merge)
            return 1 + c.num_layers * (1 + c.batch * 4) + 2 * c.batch + 2 + answer    # (+2 scoring) + select + margin
        upper_q = sum(2 + self._attn_launches(l, advance=(l == c.num_layers - 1))
                      for l in range(c.watershed, c.num_layers))
        lower_q = sum(2 + self._attn_launches(l, advance=(l == c.watershed - 1)) for l in range(c.watershed))
        return 1 + lower_q + 3 + 2 + upper_q + answer       # embed, lower layers, exact scorer, select + margin

    # ------------------------------------------------------------------ accounting
    def kv_bytes_per_token(self) -> int:
        """Algorithmic attention bytes of one decode token (all dialogues, all
        layers): K and V of every visible key, SURVEY.md §8d."""
        c = self.cfg
        es = self.es
        mid = self.nq + c.decode_steps // 2           # mean rows of the turn visible to a decode token
        lower = c.watershed * (self.hist + mid) * self.row * 2 * es
        upper = self.L_up * (self.K * c.round_tokens + mid) * self.row * 2 * es
        return c.batch * (lower + upper)

    def weight_bytes_per_token(self) -> int:
        """Weight bytes one token step of this group reads (projections of all
        layers + the tied logits), SURVEY.md §8d end-to-end roofline row."""
        return self.model.weight_bytes_per_token()

    def gpu_kv_bytes(self) -> tuple[int, int]:
        """(resident KV bytes of the round engine, full-cache bytes) at turn end."""
        c = self.cfg
        es = self.es
        full = c.batch * c.num_layers * 2 * (self.hist + self.turn_rows) * self.row * es
        resident = c.batch * 2 * self.row * es * (c.watershed * (self.hist + self.turn_rows)
                                                   + self.L_up * (self.K * c.round_tokens + self.turn_rows))
        return resident, full


class GroupedDecoder:
    """B dialogues served as G independent groups, each a RoundDecodeEngine on
    its own compute + copy streams, driven by one host thread per group, all
    sharing one model (weights are read-only).

    A group's turn has one host round trip (the kept ids) and an H2D gather
    that the decode cannot start without; with two or more groups in flight the
    gather and selection of one group overlap the decode kernels of the others,
    and the groups' programmatic-launch chains fill each other's per-layer
    latency gaps.  Dialogues stay independent: no data crosses groups.
    """

    def __init__(self, cfg: EngineConfig, groups: int = 2, device: str = "cuda", dialogues=None, seed: int = 0):
        import dataclasses
        import os
        if cfg.batch % groups:
            raise ValueError(f"batch {cfg.batch} not divisible by groups {groups}")
        per = cfg.batch // groups
        sub = dataclasses.replace(cfg, batch=per,
                                  host_unique=max(1, cfg.host_unique // groups) if cfg.host_unique else 0)
        if groups > 1 and cfg.step_kernel == "persistent":
            raise ValueError("step_kernel='persistent' needs the GPU to itself (one CTA on every SM): use groups=1")
        if groups > 1 and cfg.step_kernel == "auto":
            # concurrent groups share the SMs: the persistent step needs one CTA on every SM
            sub = dataclasses.replace(sub, step_kernel="layers")
        if dialogues is None:
            dialogues = list(range(seed, seed + cfg.batch))
        self.cfg = cfg
        self.dialogues = list(dialogues)
        self.model = DecodeModel(cfg.shape, device, seed=cfg.model_seed, prefill_gemm=cfg.question_rows > 1)
        self.groups = [RoundDecodeEngine(sub, device=device, model=self.model,
                                         dialogues=self.dialogues[g * per:(g + 1) * per]) for g in range(groups)]
        self.stagger = os.environ.get("RK_STAGGER", "1") != "0"

    def prepare(self, e2e: bool = False):
        for eng in self.groups:
            eng.prepare(e2e=e2e)

    def run_turns(self, turns: int, e2e: bool = False):
        """`turns` turns of every group, groups concurrent.  Returns (device ms
        from the first start to the last end, h2d bytes per turn (all groups),
        group-0 breakdown, kept of group 0's last turn)."""
        import threading
        starts = [torch.cuda.Event(enable_timing=True) for _ in self.groups]
        ends = [torch.cuda.Event(enable_timing=True) for _ in self.groups]
        h2d = [0] * len(self.groups)
        errors = []

        gathered = [threading.Event() for _ in self.groups]

        def work(g):
            eng = self.groups[g]
            try:
                if self.stagger and g > 0:
                    # start after the previous group's first KV gather has landed, so
                    # the groups' gathers alternate on the PCIe link instead of
                    # splitting it (each group's gather then overlaps the others' decode)
                    gathered[g - 1].wait(timeout=600)
                    if errors:           # the previous group failed before its gather: fail fast
                        return
                    eng.compute_stream.wait_event(self.groups[g - 1].copy_marks[1])
                starts[g].record(eng.compute_stream)
                for i in range(turns):
                    _, nb = eng.run_turn(e2e=e2e, on_gather=gathered[g].set if i == 0 else None)
                    h2d[g] += nb
                eng.compute_stream.wait_stream(eng.copy_stream)
                ends[g].record(eng.compute_stream)
            except Exception as exc:  # surfaced in the caller
                errors.append(exc)
                gathered[g].set()        # release a group waiting on this one's first gather

        for eng in self.groups:
            eng.window_log = []
        torch.cuda.synchronize()
        threads = [threading.Thread(target=work, args=(g,)) for g in range(len(self.groups))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        torch.cuda.synchronize()
        ref = starts[0]                                    # events are comparable across streams
        ms = max(ref.elapsed_time(e) for e in ends) - min(ref.elapsed_time(s) for s in starts)
        # decode-busy time: the union on the device timeline of every group's
        # decode-loop intervals over the timed turns (groups drift against each
        # other, so intervals are merged on the timeline, not per turn index)
        iv = sorted((ref.elapsed_time(a), ref.elapsed_time(b)) for e in self.groups for (a, b) in e.window_log)
        busy, cur0, cur1 = 0.0, None, None
        for a, b in iv:
            if cur1 is None or a > cur1:
                if cur1 is not None:
                    busy += cur1 - cur0
                cur0, cur1 = a, b
            else:
                cur1 = max(cur1, b)
        if cur1 is not None:
            busy += cur1 - cur0
        self.last_decode_busy_ms = busy
        self.last_decode_bytes = turns * sum(e.cfg.decode_steps * (e.kv_bytes_per_token() + e.weight_bytes_per_token())
                                             for e in self.groups)
        self.last_decode_kv_bytes = turns * sum(e.cfg.decode_steps * e.kv_bytes_per_token() for e in self.groups)
        self.last_decode_launches = turns * sum(e.launches_per_token() * e.cfg.decode_steps for e in self.groups)
        for eng in self.groups:
            eng.window_log = None
        return ms, sum(h2d) // max(turns, 1), self.groups[0].turn_breakdown_ms(), self.groups[0].last_kept

    # aggregate accounting over groups
    @property
    def turn_tokens(self):
        return self.groups[0].turn_tokens

    @property
    def min_margin(self):
        return min(e.min_margin for e in self.groups)

    @property
    def refined_turns(self):
        return sum(e.refined_turns for e in self.groups)

    @property
    def refined_dialogues(self):
        return sum(e.refined_dialogues for e in self.groups)

    @property
    def max_fused_rel_err(self):
        return max(e.max_fused_rel_err for e in self.groups)

    def kv_bytes_per_token(self):
        return sum(e.kv_bytes_per_token() for e in self.groups)

    def weight_bytes_per_token(self):
        return sum(e.weight_bytes_per_token() for e in self.groups)

    def gpu_kv_bytes(self):
        r = [e.gpu_kv_bytes() for e in self.groups]
        return sum(x[0] for x in r), sum(x[1] for x in r)

    def kernel_launches_per_turn(self):
        return sum(e.kernel_launches_per_turn() for e in self.groups)

    def decode_kernel_desc(self):
        return self.groups[0].decode_kernel_desc()
