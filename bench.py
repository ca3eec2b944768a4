"""Round-Attention serving benchmark (B200, sm_100a).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c4]
                    [--batch B] [--decode-steps T] [--impl ours|reference]

A "step" is one serving TURN for every dialogue on the GPU, with the model
(the reference's attention + residual transformer, engine.py:146-287, at the
Llama-3-8B / Qwen2-7B shapes with bf16 weights) running every token on the GPU:
the question through the lower layers (fused QKV projection + RoPE + KV append,
decode attention, output projection per layer), exact fp64 watershed scoring at
layer Lw-1, device round selection, the kept rounds' deep-layer KV gathered
from pinned host memory, the question's upper layers, then T greedy answer
tokens (SEP + argmax of the tied logits) through all L layers (BASELINE.json
north star).  `value` = decode tokens/s of the whole job
(B * (T + 1) tokens per turn per GPU, summed over GPUs) with the questions
already in HBM; `e2e` = the same through the public turn API: every turn's
question ids come from pinned host memory and its answer ids (plus the kept
ids and the new round's KV writeback) go back to it.  Dialogues are
independent: each rank runs its own batch (weak scaling, no collective on the
data path).

Under torchrun (N > 1) every rank runs its own engine; rank 0 prints ONE JSON
line with the max-over-ranks device time.  RK_SHARE_GPU=1 maps every rank to
GPU local_rank % device_count (the multi-rank path on a one-GPU box; the
barrier then runs on gloo).  `--impl reference` times the reference package's
own CPU path (oracle/_ref) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

WORKLOADS = {
    # Llama-3-8B-shaped GQA, 32 rounds x 512 tokens, single-token decode (BASELINE configs[1]);
    # 32 independent dialogues per GPU served as 2 groups of 16 (8 GPUs x 32 = the 256-dialogue end of
    # the configs[4] batch sweep); --batch 1 --groups 1 for a single dialogue
    # every dialogue has its own pinned host rounds (32 x 32 x 54 MiB = 55 GiB of the box's 196 GB)
    "c2": dict(num_layers=32, watershed=5, hq=32, hkv=8, head_dim=128, rounds=32, round_tokens=512, batch=32,
               decode_steps=128, host_unique=0),
    # Qwen2-7B-shaped, 64 rounds x 1K tokens, 512-row question: tcgen05 prefill of the lower layers with the
    # round scoring fused at layer Lw-1, then the upper layers over the kept rounds, then 128 answer tokens
    "c3": dict(num_layers=28, watershed=10, hq=28, hkv=4, head_dim=128, rounds=64, round_tokens=1024, batch=8,
               decode_steps=128, host_unique=0, question_rows=512),
    # Llama-3-8B-shaped 128K context, 16 dialogues, deep layers in pinned host memory; unique host rounds
    # would need 16 x 128 x 108 MiB = 216 GiB > the box's 196 GB, so 2 host round sets are shared (aliased)
    "c4": dict(num_layers=32, watershed=5, hq=32, hkv=8, head_dim=128, rounds=128, round_tokens=1024, batch=16,
               decode_steps=64, host_unique=2),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--decode-steps", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--host-unique", type=int, default=None,
                    help="distinct pinned host round sets (0 = one per dialogue)")
    ap.add_argument("--no-fetch-all", action="store_true",
                    help="skip the reference transfer pattern pass (every kept round fetched every turn)")
    ap.add_argument("--no-round-cache", action="store_true",
                    help="fetch every kept round every turn (the reference's transfer pattern)")
    ap.add_argument("--kv-dtype", default="bf16", choices=["bf16", "f32"],
                    help="KV caches / host blocks: bf16 (BASELINE configs[1]) or f32 (the reference's precision)")
    ap.add_argument("--upper-tier", default="host", choices=["host", "hbm"],
                    help="deep-layer round blocks in pinned host memory (default) or in HBM (peer-HBM tier)")
    ap.add_argument("--serving", default="groups", choices=["groups", "cohorts"],
                    help="groups: independent dialogue groups, each with its own decode loop; cohorts: two "
                         "phase-offset cohorts sharing one row-masked decode loop (weights read once per step)")
    ap.add_argument("--cohorts", type=int, default=2, help="cohorts sharing the decode loop (--serving cohorts)")
    ap.add_argument("--step-kernel", default="layers", choices=["layers", "persistent"],
                    help="answer loop: per-layer kernels, or one persistent rk_decode_step launch per token "
                         "(batch <= 16 per group, one group; DESIGN 3.2: measured slower)")
    ap.add_argument("--groups", type=int, default=None,
                    help="dialogue groups in flight per GPU (default: 2 when batch >= 2)")
    return ap.parse_args()


def measured_peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md recipe)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and "Active" in r[3 + i]
                          and "Not" not in r[3 + i]})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


def pcie_h2d_peak(torch, dev_index: int) -> float:
    """Practical H2D peak of this GPU's link: a 256 MiB pinned copy."""
    n = 256 << 20
    src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(n, dtype=torch.uint8, device=f"cuda:{dev_index}")
    best = 0.0
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        b.synchronize()
        best = max(best, n / (a.elapsed_time(b) / 1000.0) / 1e9)
    del src, dst
    return best


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def reference_arm(args, world, rank):
    """--impl reference: the reference package itself (its public
    backend.attention_forward on the compiled `_attn_ext` kernel, stats,
    selection; staged into oracle/_ref by `make -C oracle ref`) composing the
    workload's decode tokens on the host cores (rank 0).  This process never
    imports the product package, so librk.so is never mapped here."""
    if rank != 0:
        return 0
    from oracle import cpu_baseline, refkernel
    w = dict(WORKLOADS[args.workload])
    if args.batch:
        w["batch"] = args.batch
    kind = "reference" if refkernel.available() else "port"
    k = cpu_baseline.kept_count(w["rounds"])
    cores = os.cpu_count() or 1
    samples = []
    for i in range(args.warmup + args.steps):
        r = cpu_baseline.decode_tokens_per_s(kind, L=w["num_layers"], lw=w["watershed"], hq=w["hq"],
                                             hkv=w["hkv"], d=w["head_dim"], rounds=w["rounds"],
                                             T=w["round_tokens"], K=k, processes=cores, seed=100 * i)
        if i >= args.warmup:
            samples.append(r)
    tps = sum(s["tokens_per_s"] for s in samples) / len(samples)
    sample = (f"{cores} dialogues x 1 decode token per step ({args.workload} shapes: every layer's projections "
              f"(float32 BLAS) + RoPE + attention (GQA expanded to MHA, fp32 KV = 2x the GPU arm's bf16 bytes) + "
              f"residual, Lw-1 scoring + selection, tied logits + argmax), one process per core, inputs generated "
              f"before the timed region; {args.steps} steps")
    line = {
        "metric": "decode tokens/s", "value": tps, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * samples[-1]["timed_s"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64 accumulate (fp32 KV)", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"{args.workload}: reference CPU decode path", "parallelism": f"{cores} processes"},
        "cpu_baseline": {"value": tps, "unit": "tokens/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": tps, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if kind == "reference":
        line["reference_kernel"] = samples[-1]["kernel"]
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        return reference_arm(args, world, rank)

    import torch
    import torch.distributed as dist

    from paper_2502_15294_b200.decode_engine import EngineConfig, GroupedDecoder
    from paper_2502_15294_b200.sharding import (bind_numa_local, dialogues_for_rank, gpu_for_rank,
                                                host_available_bytes, host_sets_that_fit, max_over_ranks)

    dev_index, shared = gpu_for_rank(local)
    torch.cuda.set_device(dev_index)
    numa = bind_numa_local(dev_index)            # pinned host pools are allocated NUMA-local to the GPU
    if world > 1:
        if shared:       # several ranks on one GPU (a one-GPU box): NCCL refuses duplicate devices
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
    w = dict(WORKLOADS[args.workload])
    if args.batch:
        w["batch"] = args.batch
    if args.decode_steps:
        w["decode_steps"] = args.decode_steps
    if args.no_round_cache:
        w["round_cache"] = False
    if args.host_unique is not None:
        w["host_unique"] = args.host_unique
    w["kv_dtype"] = args.kv_dtype
    w["upper_tier"] = args.upper_tier
    w["step_kernel"] = args.step_kernel
    cfg = EngineConfig(**w)
    # pinned host rounds: one set per dialogue unless the node's ranks together would not fit in host
    # memory (an 8-GPU node pins 8 x the one-GPU footprint); then sets are aliased and config says so
    host_cap = None
    if cfg.host_unique <= 0 and cfg.upper_tier == "host":
        es = 2 if cfg.kv_dtype == "bf16" else 4
        set_bytes = ((cfg.num_layers - cfg.watershed) * 2 * cfg.rounds * cfg.round_tokens * cfg.hkv
                     * cfg.head_dim * es)
        ranks_on_node = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        avail = host_available_bytes()
        fit = host_sets_that_fit(cfg.batch, set_bytes, ranks_on_node, avail)
        if fit < cfg.batch:
            cfg.host_unique = fit
            host_cap = (f"{fit} host round sets per rank ({ranks_on_node} ranks x {cfg.batch} dialogues x "
                        f"{set_bytes / 2**30:.2f} GiB would exceed 0.6 x {avail / 2**30:.0f} GiB available)")
    # this rank's dialogues (b mod world == rank): its own HBM tiers, pinned host blocks, copy streams
    shard = dialogues_for_rank(cfg.batch * world, world, rank)
    # dialogue groups in flight: two groups hide one group's per-turn KV gather under the other's decode,
    # but each group reads the weights once per token step.  Measured (C2 shapes): one group is faster up
    # to 16 dialogues (B=2 1.82 K vs 1.32 K tok/s, B=8 4.40 K vs 3.89 K), two from 32 (7.64 K vs 6.85 K);
    # C3 (gathers mostly served by the round cache): one group 2.35 K vs 2.17 K; C4 (1.4 GB gathered per
    # dialogue-turn): two groups 1.30 K vs 0.98 K
    default_groups = {"c2": 2 if cfg.batch >= 32 else 1, "c3": 1, "c4": 2}[args.workload]
    groups = args.groups if args.groups else default_groups
    if cfg.batch % groups or args.step_kernel == "persistent":
        groups = 1                  # the persistent step holds one CTA on every SM
    if args.serving == "cohorts":
        from paper_2502_15294_b200.cohort import CohortDecoder
        groups = args.cohorts
        eng = CohortDecoder(cfg, cohorts=groups, dialogues=shard)
    else:
        eng = GroupedDecoder(cfg, groups=groups, dialogues=shard)
    eng.prepare(e2e=not args.no_e2e)
    link_peak = pcie_h2d_peak(torch, dev_index)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(e2e: bool, k: int):
        eng.run_turns(args.warmup, e2e=e2e)
        barrier()
        with ClockSampler(dev_index) as clk:
            ms, h2d, brk, kept = eng.run_turns(k, e2e=e2e)
        barrier()
        ms = max_over_ranks(ms)                  # the job ends with its slowest rank
        return ms, clk.summary(), brk, h2d, kept

    ms, clocks, brk, h2d_bytes, kept0 = timed(False, args.steps)
    # kept rounds of the last timed turn of every dialogue, keyed by its global id (gathered on rank 0):
    # a dialogue's data and questions are seeded by its global id, so this is independent of the sharding
    kept_by_dialogue = {int(gid): [int(x) for x in k] for e in eng.groups for gid, k in zip(e.dialogues, e.last_kept)}
    if world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, kept_by_dialogue)
        kept_by_dialogue = {k: v for part in parts for k, v in part.items()}
    # decode-loop statistics of THIS (device-resident) timed run, before the next runs overwrite them
    dec_busy_ms, dec_bytes, dec_kv_bytes = eng.last_decode_busy_ms, eng.last_decode_bytes, eng.last_decode_kv_bytes
    dec_launches = eng.last_decode_launches
    tokens_per_turn = cfg.batch * eng.turn_tokens
    value = world * tokens_per_turn * args.steps / (ms / 1000.0)
    g0 = eng.groups[0]

    e2e = None
    if not args.no_e2e:
        ms_e, _, brk_e, h2d_e, _ = timed(True, args.steps)
        # the public turn API's own transfers: question ids in; answer ids, kept ids + selection
        # metadata and the new round's upper KV (writeback) out; plus the kept rounds' KV gathers
        step_in = sum(e.q_tok.numel() * 4 for e in eng.groups)
        step_out = sum(e.answer_host.numel() * 4 + e.writeback.numel() * e.es + e.kept_host.numel() * 4
                       + e.meta_host.numel() * 4 + e.margin_host.numel() * 8 for e in eng.groups)
        e2e = {"value": world * tokens_per_turn * args.steps / (ms_e / 1000.0), "unit": "tokens/s",
               "h2d_bytes_per_step": int(h2d_e + step_in), "d2h_bytes_per_step": int(step_out),
               "ms_per_step": ms_e / args.steps, "breakdown_ms_group0": brk_e}

    fetch_all = None
    if cfg.round_cache and not args.no_fetch_all:
        # the reference's transfer pattern (store.fetch_upper of every kept round, every turn)
        for e in eng.groups:
            e.cfg.round_cache = False
        ms_f, _, _, h2d_f, _ = timed(False, args.steps)
        for e in eng.groups:
            e.cfg.round_cache = True
        fetch_all = {"value": world * tokens_per_turn * args.steps / (ms_f / 1000.0), "unit": "tokens/s",
                     "h2d_bytes_per_turn_all_groups": h2d_f,
                     "note": "round cache off: every kept round's deep-layer KV crosses PCIe every turn"}

    # roofline: the decode loop streams the KV of every visible key AND every layer's weights per token step
    # (SURVEY §8d end-to-end row); achieved = algorithmic bytes of every timed decode token / the union of
    # the groups' decode-loop intervals on the device timeline (CUDA events on each group's compute stream)
    peak, peak_kind = measured_peaks()
    bytes_tok = eng.kv_bytes_per_token() + eng.weight_bytes_per_token()
    achieved = dec_bytes / (dec_busy_ms / 1000.0) / 1e9
    step_bw = bytes_tok * eng.turn_tokens * args.steps / (ms / 1000.0) / 1e9
    resident, full = eng.gpu_kv_bytes()
    traffic = None      # DRAM bytes per token-step from the committed ncu capture (same shapes)
    tp = REPO / "profiles" / f"r02_traffic_{args.workload}_tokenstep.json"      # c2, c4: one group's token steps
    if (tp.exists() and args.kv_dtype == "bf16" and args.step_kernel == "layers" and args.serving == "groups"
            and args.upper_tier == "host"):
        t = json.loads(tp.read_text())
        if t.get("batch_per_group") == g0.cfg.batch:
            traffic = t["per_token_step_bytes_per_group"] * len(eng.groups)

    prefill = None
    if g0.nq > 1:
        # question prefill (tcgen05): lower layers incl. fused scoring = marks 0 -> 1 of group 0 (its own
        # stream; the other group's decode runs beside it), algorithmic FLOPs of those layers
        lw, nq = cfg.watershed, g0.nq
        lower_flops = 4.0 * cfg.hq * cfg.head_dim * lw * (nq * g0.hist + nq * (nq + 1) / 2) * g0.cfg.batch
        prefill = {"question_rows": nq, "flops_per_turn_all_layers": sum(e.prefill_flops_per_turn() for e in eng.groups),
                   "lower_layers_ms_group0": brk["score_select"],
                   "lower_layers_attention_tflops_group0": lower_flops / (brk["score_select"] / 1000.0) / 1e12,
                   "note": "lower-layer prefill (projections + attention + fused Lw-1 scoring) + select, timed on "
                           "group 0's stream while the other group decodes; attention FLOPs only; kernel-alone "
                           "figures: profiles/r01_prefill_c3.json"}
    line = {
        "metric": "decode tokens/s", "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None,
        "dtype": f"bf16 weights, {args.kv_dtype} KV, fp32 activations / accumulate",
        "data": "synthetic (random-init weights of the config's shape, random KV history, random question ids)",
        "config": {"workload": f"{args.workload}: L={cfg.num_layers} Lw={cfg.watershed} Hq={cfg.hq} "
                               f"Hkv={cfg.hkv} d={cfg.head_dim} rounds={cfg.rounds}x{cfg.round_tokens} "
                               f"K={g0.K} batch/GPU={cfg.batch} in {groups} {'cohorts sharing one decode loop' if args.serving == 'cohorts' else 'groups'} question_rows={g0.nq} "
                               f"decode tokens/turn={eng.turn_tokens} (fixed; EOT ignored) "
                               f"host_round_sets/group={g0.host_sets} (unique per dialogue: "
                               f"{g0.host_sets == g0.cfg.batch}) round_cache={cfg.round_cache} "
                               f"question_variants={cfg.question_variants} kv_dtype={args.kv_dtype} "
                               f"upper_tier={args.upper_tier}",
                   "model": "reference toy transformer (attention + residual, RoPE, tied logits) at "
                            f"{'Llama-3-8B' if cfg.hq == 32 else 'Qwen2-7B'} shapes, GQA, bf16 weights",
                   "global_batch": cfg.batch * world, "parallelism": f"dialogues x{world} (no collective)",
                   "l2": "inputs larger than L2 (KV + weights read per token step >> 126 MB)",
                   **({"host_memory_cap": host_cap} if host_cap else {})},
        "gpu_launches": eng.kernel_launches_per_turn() * args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "kernel": (f"decode step (per layer: rk_qkv_rope + rk decode attention [{eng.decode_kernel_desc()}]"
                                " + rk_out_proj; rk_lm_head)" if args.step_kernel == "layers" else
                                f"decode step ({eng.decode_kernel_desc()})")
                               + ": KV + weight bytes of every timed decode token / union "
                               "of the groups' decode-loop intervals (CUDA events)",
                     "decode_busy_ms": dec_busy_ms, "launches": dec_launches,
                     "kv_GBps": dec_kv_bytes / (dec_busy_ms / 1000.0) / 1e9,
                     "whole_step_GBps": step_bw, "whole_step_frac": step_bw / peak,
                     "bytes_per_token_step": bytes_tok, "kv_bytes_per_token_step": eng.kv_bytes_per_token(),
                     "weight_bytes_per_token_step": eng.weight_bytes_per_token(), "peak_source": peak_kind},
        "h2d": {"bytes_per_turn_all_groups": h2d_bytes, "group0_bytes": g0.last_h2d_bytes, "group0_ms": brk["h2d"],
                "round_cache": {"enabled": cfg.round_cache, "question_variants": cfg.question_variants,
                                "rounds_fetched_group0_last_turn": g0.last_copied_rounds,
                                "rounds_kept_group0": g0.cfg.batch * g0.K},
                "GBps": g0.last_h2d_bytes / (brk["h2d"] / 1000.0) / 1e9 if brk["h2d"] > 0 else None,
                "link": ("PCIe Gen5 x16 (~63 GB/s/dir theoretical)" if args.upper_tier == "host"
                 else "HBM tier on this GPU (a peer GPU's HBM over NVLink on a multi-GPU box)"),
                "link_peak_GBps": link_peak,
                "link_peak_how": "one 256 MiB pinned-host -> HBM copy, best of 5, CUDA events, before the timed region"},
        "k_boundary": {"min_rel_gap": eng.min_margin, "scorer": "fp64 exact (rk_round_scores_exact)" if g0.nq == 1
                       else "tcgen05 fused fp32-class, fp64 re-score below the margin",
                       "refine_margin": cfg.refine_margin, "refined_turns": eng.refined_turns,
                       "refined_dialogue_turns": eng.refined_dialogues,
                       "max_fused_rel_err": eng.max_fused_rel_err,
                       "note": "relative gap between the K-th and (K+1)-th largest masses, minimum over every "
                               "dialogue and turn of the run"},
        "gpu_kv_saved": {"resident_bytes": resident, "full_cache_bytes": full, "saved_frac": 1 - resident / full},
        "breakdown_ms_group0": brk,
        "clocks": clocks,
        "kept_dialogue0": [int(x) for x in kept0[0]],
        "kept_by_dialogue": ({str(k): kept_by_dialogue[k] for k in sorted(kept_by_dialogue)}
                             if len(kept_by_dialogue) <= 64 else None),
        "host": {"numa_node": numa, "pinned_round_bytes": sum(e.host_sets * e.cfg.rounds for e in eng.groups)
                 * g0.host_blocks[0][0].numel() * g0.es},
    }
    if fetch_all:
        line["fetch_all"] = fetch_all
    if prefill:
        line["prefill"] = prefill
    if e2e:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            from oracle import cpu_baseline, refkernel
            kind = "reference" if refkernel.available() else "port"
            cores = os.cpu_count() or 1
            r = cpu_baseline.decode_tokens_per_s(kind, L=cfg.num_layers, lw=cfg.watershed, hq=cfg.hq,
                                                 hkv=cfg.hkv, d=cfg.head_dim, rounds=cfg.rounds,
                                                 T=cfg.round_tokens, K=g0.K, processes=cores)
            line["cpu_baseline"] = {"value": r["tokens_per_s"], "unit": "tokens/s", "cores": cores, "kind": kind,
                                    "sample": f"{cores} dialogues x 1 decode token ({args.workload} shapes: projections "
                                              f"(float32 BLAS) + RoPE + attention (fp32 KV) + residual per layer, "
                                              f"scoring + selection, tied logits), one process per core, timed "
                                              f"{r['timed_s']:.1f}s after input generation"}
        except Exception as exc:  # the GPU number stands on its own
            line["cpu_baseline"] = {"value": None, "error": repr(exc)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
