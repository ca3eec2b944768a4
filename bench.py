"""Round-Attention decode benchmark (B200, sm_100a).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c4]
                    [--batch B] [--decode-steps T] [--impl ours|reference]

A "step" is one serving TURN for every dialogue on the GPU: the question token
through the lower layers with fused watershed scoring (layer Lw-1), device
round selection, the kept rounds' deep-layer KV gathered from pinned host
memory, the question's upper layers, then T answer tokens through all L
layers (BASELINE.json north star).  `value` = decode tokens/s
of the whole job (B * (T + 1) tokens per turn per GPU, summed over GPUs) with
per-token activations already in HBM; `e2e` = the same with every token's
q/k/v read from pinned host memory and every layer's attention output written
back to host inside the timed region.  Dialogues are independent: each rank
runs its own batch (weak scaling, no collective on the data path).

Under torchrun (N > 1) every rank runs its own engine; rank 0 prints ONE JSON
line with the max-over-ranks device time.  `--impl reference` times the
reference's own CPU kernel (oracle/_ref, else the C port) on the host cores.
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
    "c2": dict(num_layers=32, watershed=5, hq=32, hkv=8, head_dim=128, rounds=32, round_tokens=512, batch=32,
               decode_steps=128, host_unique=4),
    # Qwen2-7B-shaped, 64 rounds x 1K tokens, 512-row question: tcgen05 prefill of the lower layers with the
    # round scoring fused at layer Lw-1, then the upper layers over the kept rounds, then 128 answer tokens
    "c3": dict(num_layers=28, watershed=10, hq=28, hkv=4, head_dim=128, rounds=64, round_tokens=1024, batch=8,
               decode_steps=128, host_unique=2, question_rows=512),
    # Llama-3-8B-shaped 128K context, 16 dialogues, deep layers in pinned host memory
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
    ap.add_argument("--question-noise", type=float, default=None,
                    help="per-turn question variation (EngineConfig.question_noise)")
    ap.add_argument("--input-period", type=int, default=None,
                    help="per-token input slots (EngineConfig.input_period; e2e loads run P-2 tokens ahead)")
    ap.add_argument("--no-round-cache", action="store_true",
                    help="fetch every kept round every turn (the reference's transfer pattern)")
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
    sample = (f"{cores} dialogues x 1 decode token per step ({args.workload} shapes, GQA expanded to MHA, "
              f"fp32 KV = 2x the GPU arm's bf16 bytes), one process per core, inputs generated before the "
              f"timed region; {args.steps} steps")
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
    from paper_2502_15294_b200.sharding import dialogues_for_rank, max_over_ranks

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = dict(WORKLOADS[args.workload])
    if args.batch:
        w["batch"] = args.batch
    if args.decode_steps:
        w["decode_steps"] = args.decode_steps
    if args.no_round_cache:
        w["round_cache"] = False
    if args.question_noise is not None:
        w["question_noise"] = args.question_noise
    if args.input_period:
        w["input_period"] = args.input_period
    cfg = EngineConfig(**w)
    # this rank's dialogues (b mod world == rank): its own HBM tiers, pinned host blocks, copy streams
    shard = dialogues_for_rank(cfg.batch * world, world, rank)
    groups = args.groups if args.groups else (2 if cfg.batch >= 2 and cfg.batch % 2 == 0 else 1)
    eng = GroupedDecoder(cfg, groups=groups, seed=1000 * shard[0])
    eng.prepare(e2e=not args.no_e2e)
    link_peak = pcie_h2d_peak(torch, local)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(e2e: bool, k: int):
        eng.run_turns(args.warmup, e2e=e2e)
        barrier()
        with ClockSampler(local) as clk:
            ms, h2d, brk, kept = eng.run_turns(k, e2e=e2e)
        barrier()
        ms = max_over_ranks(ms)                  # the job ends with its slowest rank
        return ms, clk.summary(), brk, h2d, kept

    ms, clocks, brk, h2d_bytes, kept0 = timed(False, args.steps)
    # decode-kernel statistics of THIS (device-resident) timed run, before the e2e run overwrites them
    dec_busy_ms, dec_bytes, dec_launches = eng.last_decode_busy_ms, eng.last_decode_bytes, eng.last_decode_launches
    tokens_per_turn = cfg.batch * eng.turn_tokens
    value = world * tokens_per_turn * args.steps / (ms / 1000.0)
    g0 = eng.groups[0]

    e2e = None
    if not args.no_e2e:
        ms_e, _, brk_e, h2d_e, _ = timed(True, args.steps)
        step_in = sum(e.turn_tokens * (e.q_in[0].numel() * 4 + e.kv_in[0].numel() * 2)
                      + (e.qq_in.numel() * 4 + e.qkv_in.numel() * 2 + e.q_var[0].numel() * 4 if e.nq > 1 else 0)
                      for e in eng.groups)
        step_out = sum(e.cfg.decode_steps * e.out.numel() * 4 + e.writeback.numel() * 2 + e.kept_host.numel() * 4
                       for e in eng.groups)
        e2e = {"value": world * tokens_per_turn * args.steps / (ms_e / 1000.0), "unit": "tokens/s",
               "h2d_bytes_per_step": int(h2d_e + step_in), "d2h_bytes_per_step": int(step_out),
               "ms_per_step": ms_e / args.steps, "breakdown_ms_group0": brk_e}

    # roofline of the dominant kernel (the decode attention) from the timed turns:
    # decode-loop time per token vs algorithmic KV bytes per token
    peak, peak_kind = measured_peaks()
    # decode kernels of all groups: algorithmic KV bytes of
    # every timed decode token / the union of the decode-loop intervals on the
    # device timeline (CUDA events on each group's compute stream)
    bytes_tok = eng.kv_bytes_per_token()
    achieved = dec_bytes / (dec_busy_ms / 1000.0) / 1e9
    step_bw = bytes_tok * eng.turn_tokens * args.steps / (ms / 1000.0) / 1e9
    resident, full = eng.gpu_kv_bytes()
    traffic = None      # DRAM bytes per token-step from the committed ncu capture of this kernel (same shapes)
    tp = REPO / "profiles" / "r01_traffic_c2_tokenstep.json"
    if tp.exists() and args.workload == "c2":
        t = json.loads(tp.read_text())
        traffic = t["per_dialogue_token_bytes"] * cfg.batch

    prefill = None
    if g0.nq > 1:
        # question prefill (tcgen05): lower layers incl. fused scoring = marks 0 -> 1 of group 0 (its own
        # stream; the other group's decode runs beside it), algorithmic FLOPs of those layers
        lw, nq = cfg.watershed, g0.nq
        lower_flops = 4.0 * cfg.hq * cfg.head_dim * lw * (nq * g0.hist + nq * (nq + 1) / 2) * g0.cfg.batch
        prefill = {"question_rows": nq, "flops_per_turn_all_layers": sum(e.prefill_flops_per_turn() for e in eng.groups),
                   "lower_layers_ms_group0": brk["score_select"],
                   "lower_layers_tflops_group0": lower_flops / (brk["score_select"] / 1000.0) / 1e12,
                   "note": "lower-layer prefill + fused Lw-1 scoring + select, timed on group 0's stream while "
                           "the other group decodes; kernel-alone figures: profiles/r01_prefill_c3.json"}
        pk = json.loads((REPO / "MEASURED_PEAKS.json").read_text()) if (REPO / "MEASURED_PEAKS.json").exists() else {}
        tpk = float(pk.get("bf16_tflops", 2250.0))
        achieved_tf = prefill["lower_layers_tflops_group0"]
        prefill["roofline"] = {"bound": "tensor", "achieved": achieved_tf, "peak": tpk, "unit": "TFLOP/s",
                               "frac": achieved_tf / tpk,
                               "peak_source": "measured" if pk else "nominal dense bf16",
                               "note": "algorithmic FLOPs (QK^T + PV once over causal-visible pairs); the kernel "
                                       "issues 2x (q and P hi/lo bf16 splits for fp32-class accuracy)"}
    line = {
        "metric": "decode tokens/s", "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16 KV, fp32 accumulate", "data": "synthetic (random KV + activations)",
        "config": {"workload": f"{args.workload}: L={cfg.num_layers} Lw={cfg.watershed} Hq={cfg.hq} "
                               f"Hkv={cfg.hkv} d={cfg.head_dim} rounds={cfg.rounds}x{cfg.round_tokens} "
                               f"K={g0.K} batch/GPU={cfg.batch} in {groups} groups question_rows={g0.nq} "
                               f"decode tokens/turn={eng.turn_tokens}",
                   "global_batch": cfg.batch * world, "parallelism": f"dialogues x{world} (no collective)",
                   "l2": "inputs larger than L2 (KV read per token >> 126 MB)"},
        "gpu_launches": eng.kernel_launches_per_turn() * args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": f"rk decode attention ({eng.decode_kernel_desc()}): KV bytes of every timed decode "
                                                "token / union of the groups' decode-loop intervals (CUDA events)",
                     "decode_busy_ms": dec_busy_ms, "launches": dec_launches,
                     "whole_step_GBps": step_bw, "whole_step_frac": step_bw / peak,
                     "bytes_per_token": bytes_tok, "peak_source": peak_kind},
        "h2d": {"bytes_per_turn_all_groups": h2d_bytes, "group0_bytes": g0.last_h2d_bytes, "group0_ms": brk["h2d"],
                "round_cache": {"enabled": cfg.round_cache, "question_variants": cfg.question_variants,
                                "rounds_fetched_group0_last_turn": g0.last_copied_rounds,
                                "rounds_kept_group0": g0.cfg.batch * g0.K},
                "GBps": g0.last_h2d_bytes / (brk["h2d"] / 1000.0) / 1e9 if brk["h2d"] > 0 else None,
                "link": "PCIe Gen5 x16 (~63 GB/s/dir theoretical)",
                "link_peak_GBps": link_peak,
                "link_peak_how": "one 256 MiB pinned-host -> HBM copy, best of 5, CUDA events, before the timed region"},
        "gpu_kv_saved": {"resident_bytes": resident, "full_cache_bytes": full, "saved_frac": 1 - resident / full},
        "breakdown_ms_group0": brk,
        "clocks": clocks,
        "kept_dialogue0": [int(x) for x in kept0[0]],
    }
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
                                    "sample": f"{cores} dialogues x 1 decode token ({args.workload} shapes, fp32 KV), "
                                              f"one process per core, timed {r['timed_s']:.1f}s after input "
                                              f"generation"}
        except Exception as exc:  # the GPU number stands on its own
            line["cpu_baseline"] = {"value": None, "error": repr(exc)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
