"""Cohort serving: B dialogues in two phase-offset cohorts that share ONE decode loop.

The grouped decoder (decode_engine.GroupedDecoder) hides one group's per-turn
work — the question through the layers, the watershed scoring and selection,
the host->HBM gather of the kept rounds (pipeline.py:225-296) — under the other
group's answer decode, but each group reads every layer's weights once per
token step (2 x 2.69 GB per token step at C2 shapes).  Here the answer decode
(pipeline.py:298-313) of all B dialogues is one loop of token steps over all B
rows, each step reading the weights once for every dialogue in it:

  * each cohort (B/2 dialogues) is a RoundDecodeEngine over views of the shared
    caches and length arrays; its turn prologue (question, scoring, selection,
    gather, the question's upper layers) runs on its own streams, eagerly or
    from its captured graph, while the other cohort decodes;
  * the decode loop replays ONE captured token step over all B rows with a row
    mask (rk_decode_attention_rows, rk_out_proj_rows, rk_lm_head_rows): rows of
    a cohort outside the loop append nothing, advance nothing and keep their
    residual row, so the cohort's prologue may write its own caches and
    lengths concurrently;
  * a cohort joins the loop (SEP embedded, positions reset) once its prologue's
    event has completed on the device, decodes `decode_steps` tokens and
    leaves; the host keeps at most two token steps in flight so joins happen
    within ~two steps of readiness.

Every row's arithmetic is independent of the other rows (the projections
reduce over k per row, attention is per (dialogue, kv-head)), so a dialogue's
answer is the same whichever cohorts share its steps.
"""

from __future__ import annotations

import dataclasses
import threading

import numpy as np
import torch

from . import kernels
from .decode_engine import EngineConfig, RoundDecodeEngine
from .decode_model import SEP_TOKEN, DecodeModel


class CohortDecoder:
    def __init__(self, cfg: EngineConfig, cohorts: int = 2, device: str = "cuda", dialogues=None, seed: int = 0):
        if cfg.batch % cohorts:
            raise ValueError(f"batch {cfg.batch} not divisible by cohorts {cohorts}")
        self.cfg = c = cfg
        self.dev = torch.device(device)
        self.n_c = cohorts
        per = c.batch // cohorts
        self.per = per
        if dialogues is None:
            dialogues = list(range(seed, seed + c.batch))
        self.dialogues = list(dialogues)
        self.model = DecodeModel(c.shape, self.dev, seed=c.model_seed, prefill_gemm=c.question_rows > 1)
        m = self.model
        B, L, lw = c.batch, c.num_layers, c.watershed
        sub = dataclasses.replace(c, batch=per, host_unique=max(1, c.host_unique // cohorts) if c.host_unique else 0,
                                  step_kernel="layers")    # the masked answer loop is this class's own
        # the shared HBM tiers and length arrays, sized as one engine's
        probe = RoundDecodeEngine.shapes(sub)
        dt = torch.bfloat16 if c.kv_dtype == "bf16" else torch.float32
        self.lower = torch.empty((B, lw, 2, probe["s_lo"], c.hkv, c.head_dim), dtype=dt, device=self.dev)
        self.upper = torch.zeros((B, L - lw, 2, probe["s_up"], c.hkv, c.head_dim), dtype=dt, device=self.dev)
        self.lower_len = torch.zeros(B, dtype=torch.int32, device=self.dev)
        self.upper_len = torch.zeros(B, dtype=torch.int32, device=self.dev)
        self.engines = []
        for k in range(cohorts):
            rows = slice(k * per, (k + 1) * per)
            shared = dict(lower=self.lower[rows], upper=self.upper[rows], lower_len=self.lower_len[rows],
                          upper_len=self.upper_len[rows])
            self.engines.append(RoundDecodeEngine(sub, device=device, model=m, dialogues=self.dialogues[rows],
                                                  shared=shared))
        e0 = self.engines[0]
        self.s_lo, self.s_up = e0.s_lo, e0.s_up
        D = c.hq * c.head_dim
        # ---- the shared decode loop's own buffers (all B rows)
        self.x = torch.zeros((B, D), dtype=torch.float32, device=self.dev)
        self.q = torch.zeros((B, c.hq, c.head_dim), dtype=torch.float32, device=self.dev)
        self.k_new = torch.zeros((B, c.hkv, c.head_dim), dtype=dt, device=self.dev)
        self.v_new = torch.zeros((B, c.hkv, c.head_dim), dtype=dt, device=self.dev)
        self.attn = torch.zeros((B, D), dtype=torch.float32, device=self.dev)
        self.tokens = torch.zeros(B, dtype=torch.int32, device=self.dev)
        self.pos = torch.zeros(B, dtype=torch.int32, device=self.dev)
        self.pos_dec0 = int(e0.pos_dec0[0])
        self.answer = torch.full((B, c.decode_steps + 1), SEP_TOKEN, dtype=torch.int32, device=self.dev)
        self.answer_host = torch.zeros((B, c.decode_steps + 1), dtype=torch.int32, pin_memory=True)
        self.sep = torch.full((per,), SEP_TOKEN, dtype=torch.int32, device=self.dev)
        self.active = torch.zeros(B, dtype=torch.int32, device=self.dev)
        self.active_host = [torch.zeros(B, dtype=torch.int32, pin_memory=True) for _ in range(4)]
        self.proj_ws = kernels.proj_workspace(B, D, max(m.shape.qkv_width, D), self.dev)
        from . import _lib
        self.lm_ws = torch.zeros(max(256, _lib.lib.rk_lm_head_workspace_bytes(B, m.shape.vocab, D)),
                                 dtype=torch.uint8, device=self.dev)
        self.stream = torch.cuda.Stream(self.dev)
        self.graph = None
        self.dec_marks = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(cohorts)]

    # ------------------------------------------------------------------ the shared token step
    def _caches(self, l: int):
        c = self.cfg
        if l < c.watershed:
            return self.lower[:, l, 0], self.lower[:, l, 1], self.lower_len, self.s_lo
        u = l - c.watershed
        return self.upper[:, u, 0], self.upper[:, u, 1], self.upper_len, self.s_up

    def _step(self):
        """One answer token of every active row through all L layers and the
        tied logits (pipeline.py:298-313; engine.py:244-271)."""
        c, m = self.cfg, self.model
        for l in range(c.num_layers):
            kc, vc, ln, cap = self._caches(l)
            kernels.qkv_rope(self.x, m.w_qkv_packed[l], c.hq, c.hkv, c.head_dim, self.pos, m.freq, self.q,
                             self.k_new, self.v_new, ws=self.proj_ws)
            adv = l == c.watershed - 1 or l == c.num_layers - 1
            kernels.decode_attention_rows(self.q, kc, vc, ln, cap, self.active, k_new=self.k_new, v_new=self.v_new,
                                          out=self.attn.view(c.batch, c.hq, c.head_dim), advance=ln if adv else None)
            kernels.out_proj(self.attn, m.w_o_packed[l], self.x, ws=self.proj_ws, row_active=self.active)
        kernels.lm_head(self.x, m.emb_packed, m.shape.vocab, m.emb, self.x, self.tokens, self.pos,
                        tokens_log=self.answer, log_stride=self.answer.shape[1], ws=self.lm_ws,
                        row_active=self.active, log_pos_base=self.pos_dec0)

    def _join(self, k: int):
        """Cohort k enters the loop: SEP embedded, positions at the answer's start."""
        rows = slice(k * self.per, (k + 1) * self.per)
        kernels.embed(self.sep, self.model.emb, self.x[rows])
        self.pos[rows].fill_(self.pos_dec0)
        self.answer[rows].fill_(SEP_TOKEN)

    def prepare(self, e2e: bool = False):
        for eng in self.engines:
            eng.prepare(e2e=e2e, decode_graph=False)
        with torch.cuda.stream(self.stream):
            self.active.fill_(0)
            self._step()                          # warm-up (every row inactive: touches nothing)
            torch.cuda.synchronize()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=self.stream):
                self._step()
        torch.cuda.synchronize()

    # ------------------------------------------------------------------ serving
    def run_turns(self, turns: int, e2e: bool = False, timeout: float = 600.0):
        """`turns` turns of every dialogue.  Returns (device ms from the first
        cohort's start to the last token, H2D bytes per turn (all cohorts), the
        kept rounds of every dialogue's last turn by global id).  Sets
        last_decode_bytes / last_decode_busy_ms (KV of the rows in each step +
        the weights once per step, over the loop's device interval)."""
        c, per, n_c = self.cfg, self.per, self.n_c
        self.last_turns = turns
        first_ready = [threading.Event() for _ in range(n_c)]   # first prologue enqueued (never cleared)
        ready = [threading.Event() for _ in range(n_c)]         # a prologue is enqueued (host)
        done = [threading.Event() for _ in range(n_c)]          # the cohort left the loop (host)
        ev_ready = [torch.cuda.Event() for _ in range(n_c)]
        ev_done = [torch.cuda.Event() for _ in range(n_c)]
        start = torch.cuda.Event(enable_timing=True)
        loop0 = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        errors, h2d = [], [0] * n_c
        kept_last = [None] * n_c
        stop = threading.Event()

        def wait_flag(flag):
            while not flag.wait(0.05):
                if stop.is_set():
                    return False
            return True

        def cohort(k):
            eng = self.engines[k]
            try:
                with torch.cuda.stream(eng.compute_stream):
                    if k > 0:     # offset the cohorts: the previous cohort's first prologue goes first
                        if not wait_flag(first_ready[k - 1]):
                            return
                        eng.compute_stream.wait_event(ev_ready[k - 1])
                    else:
                        start.record(eng.compute_stream)
                    for i in range(turns):
                        if i > 0:
                            if not wait_flag(done[k]):
                                return
                            done[k].clear()
                            eng.compute_stream.wait_event(ev_done[k])
                            eng.copy_stream.wait_event(ev_done[k])
                            with torch.cuda.stream(eng.copy_stream):
                                eng._phase_wb()
                        mk = eng.marks
                        mk[0].record(eng.compute_stream)
                        eng._set_question(e2e)
                        eng.graph_a.replay()
                        mk[1].record(eng.compute_stream)
                        kept = eng._select_to_host()
                        eng.copy_stream.wait_stream(eng.compute_stream)
                        plans = eng.gather_plan(kept)
                        eng.copy_marks[0].record(eng.copy_stream)
                        nb = eng.issue_gather(plans)
                        eng.copy_marks[1].record(eng.copy_stream)
                        h2d[k] += nb
                        eng.last_h2d_bytes = nb
                        eng._phase_b1(layer_wait=True)
                        mk[2].record(eng.compute_stream)
                        ev_ready[k].record(eng.compute_stream)
                        eng.last_kept = kept
                        kept_last[k] = kept
                        ready[k].set()
                        first_ready[k].set()
                    if not wait_flag(done[k]):                # the last turn's decode
                        return
                    eng.copy_stream.wait_event(ev_done[k])
                    with torch.cuda.stream(eng.copy_stream):
                        eng._phase_wb()
            except Exception as exc:  # surfaced in the caller
                errors.append(exc)
                stop.set()

        copied = [None] * len(self.active_host)    # event of the last copy out of each pinned mask buffer

        def set_mask(mask, nbuf):
            i = nbuf % len(self.active_host)
            if copied[i] is not None:
                copied[i].synchronize()             # never rewrite a buffer a pending copy still reads
            hb = self.active_host[i]
            hb.copy_(torch.from_numpy(mask))
            self.active.copy_(hb, non_blocking=True)
            copied[i] = torch.cuda.Event()
            copied[i].record(self.stream)

        threads = [threading.Thread(target=cohort, args=(k,)) for k in range(n_c)]
        torch.cuda.synchronize()
        for t in threads:
            t.start()
        w_bytes = self.weight_bytes_per_token()
        kv_bytes = [e.kv_bytes_per_token() for e in self.engines]
        dec_bytes = 0
        try:
            left = [0] * n_c                       # tokens left in the loop per cohort
            served = [0] * n_c                     # turns decoded per cohort
            inflight = []                          # events of the last token steps (host throttle)
            nbuf = 0
            mask = np.zeros(c.batch, dtype=np.int32)
            looping = False
            steps = 0
            while not errors:
                if min(served) >= turns and not any(left):
                    break
                joined = False
                for k in range(n_c):
                    if left[k] or served[k] >= turns or not ready[k].is_set():
                        continue
                    if any(left) and not ev_ready[k].query():
                        continue                   # join only once its prologue is done on the device
                    ready[k].clear()
                    with torch.cuda.stream(self.stream):
                        self.stream.wait_event(ev_ready[k])
                        self._join(k)
                        self.dec_marks[k][0].record(self.stream)
                    mask[k * per:(k + 1) * per] = 1
                    left[k] = c.decode_steps
                    joined = True
                if not any(left):
                    if not any(t.is_alive() for t in threads) and not any(r.is_set() for r in ready):
                        raise RuntimeError("cohort threads ended before serving every turn")
                    for k in range(n_c):
                        ready[k].wait(0.01)
                    continue
                with torch.cuda.stream(self.stream):
                    if joined:
                        set_mask(mask, nbuf)
                        nbuf += 1
                    if not looping:
                        loop0.record(self.stream)
                        looping = True
                    self.graph.replay()
                    ev = torch.cuda.Event()
                    ev.record(self.stream)
                    steps += 1
                inflight.append(ev)
                if len(inflight) > 2:
                    inflight.pop(0).synchronize()
                dec_bytes += w_bytes + sum(kv_bytes[k] for k in range(n_c) if left[k])
                for k in range(n_c):
                    if left[k] == 0:
                        continue
                    left[k] -= 1
                    if left[k] == 0:                   # cohort k leaves the loop
                        mask[k * per:(k + 1) * per] = 0
                        with torch.cuda.stream(self.stream):
                            if e2e:
                                rows = slice(k * per, (k + 1) * per)
                                self.answer_host[rows].copy_(self.answer[rows], non_blocking=True)
                            set_mask(mask, nbuf)
                            nbuf += 1
                            ev_done[k].record(self.stream)
                            self.dec_marks[k][1].record(self.stream)
                        served[k] += 1
                        done[k].set()
            with torch.cuda.stream(self.stream):
                end.record(self.stream)
        except Exception as exc:
            errors.append(exc)
            stop.set()
        for t in threads:
            t.join(timeout)
        if errors:
            raise errors[0]
        torch.cuda.synchronize()
        self.last_decode_bytes = dec_bytes
        self.last_decode_kv_bytes = dec_bytes - steps * w_bytes
        self.last_decode_busy_ms = loop0.elapsed_time(end)
        self.last_steps = steps
        self.last_decode_launches = steps * self.engines[0].launches_per_token()
        kept = {}
        for k in range(n_c):
            for gid, kk in zip(self.engines[k].dialogues, kept_last[k]):
                kept[int(gid)] = [int(x) for x in kk]
        self.last_kept_by_dialogue = kept
        return start.elapsed_time(end), sum(h2d) // max(turns, 1), self.turn_breakdown_ms(), kept_last[0]

    def turn_breakdown_ms(self) -> dict:
        """Cohort 0's last turn: prologue parts on its stream, its decode window on the loop's."""
        e, m = self.engines[0], self.engines[0].marks
        return dict(score_select=m[0].elapsed_time(m[1]), gather_upper_prefill=m[1].elapsed_time(m[2]),
                    decode=self.dec_marks[0][0].elapsed_time(self.dec_marks[0][1]), writeback_copy_stream=0.0,
                    turn=m[0].elapsed_time(self.dec_marks[0][1]),
                    h2d=e.copy_marks[0].elapsed_time(e.copy_marks[1]))

    def answers(self) -> np.ndarray:
        torch.cuda.synchronize()
        return self.answer[:, : self.cfg.decode_steps].cpu().numpy()

    # ------------------------------------------------------------------ accounting (GroupedDecoder's interface)
    @property
    def groups(self):
        return self.engines

    @property
    def turn_tokens(self):
        return self.engines[0].turn_tokens

    @property
    def min_margin(self):
        return min(e.min_margin for e in self.engines)

    @property
    def refined_turns(self):
        return sum(e.refined_turns for e in self.engines)

    @property
    def refined_dialogues(self):
        return sum(e.refined_dialogues for e in self.engines)

    @property
    def max_fused_rel_err(self):
        return max(e.max_fused_rel_err for e in self.engines)

    def gpu_kv_bytes(self):
        r = [e.gpu_kv_bytes() for e in self.engines]
        return sum(x[0] for x in r), sum(x[1] for x in r)

    def decode_kernel_desc(self) -> str:
        return (f"decode_cluster_kernel over all {self.cfg.batch} rows with a row mask (rk_decode_attention_rows), "
                f"{self.n_c} cohorts")

    def kernel_launches_per_turn(self) -> int:
        """Per turn: every cohort's prologue (question layers, scoring, selection) and the
        shared loop's token steps of the last run, per turn."""
        e = self.engines[0]
        prologue = e.kernel_launches_per_turn() - 1 - e.launches_per_token() * self.cfg.decode_steps
        steps = getattr(self, "last_steps", self.cfg.decode_steps) / max(1, getattr(self, "last_turns", 1))
        return int(self.n_c * prologue + steps * e.launches_per_token())

    def kv_bytes_per_token(self):
        return sum(e.kv_bytes_per_token() for e in self.engines)

    def weight_bytes_per_token(self):
        return self.model.weight_bytes_per_token()
