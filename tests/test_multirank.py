"""N>1 path on the CPU with the gloo backend (world size 2): dialogue sharding
is disjoint and complete, each rank's round selection for its dialogues equals
a single-process run (no data crosses ranks), and the timing reduction takes
the max over ranks."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import attention as oatt
from oracle import rounds as orr
from paper_2502_15294_b200.sharding import dialogues_for_rank, max_over_ranks, per_rank_batch

N_DIALOGUES, R, T, HKV, G, D = 6, 8, 16, 2, 2, 16


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dialogue_selection(b):
    """Oracle watershed scoring + top-k for synthetic dialogue b (deterministic per b)."""
    rng = np.random.default_rng(100 + b)
    hist = R * T
    k = rng.standard_normal((hist + 1, HKV, D)).astype(np.float32)
    q = rng.standard_normal((1, HKV * G, D)).astype(np.float32)
    _, cap = oatt.attention_forward_gqa(q, k, k, [hist], np.arange(hist + 1), capture=True)
    raw = np.array([cap[0, r * T:(r + 1) * T].sum() for r in range(R)])
    return orr.select(orr.normalize(raw), orr.SelectionPolicy("top_percent", fraction=0.25))


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = dialogues_for_rank(N_DIALOGUES, world, rank)
    kept = {b: _dialogue_selection(b) for b in mine}
    gathered = [None] * world
    dist.all_gather_object(gathered, kept)
    ms = max_over_ranks(10.0 + rank, device="cpu")
    if rank == 0:
        out.put((gathered, ms))
    dist.barrier()
    dist.destroy_process_group()


def test_sharding_plan():
    assert dialogues_for_rank(5, 2, 0) == [0, 2, 4]
    assert dialogues_for_rank(5, 2, 1) == [1, 3]
    assert per_rank_batch(256, 8) == 32
    with pytest.raises(ValueError):
        per_rank_batch(10, 4)
    with pytest.raises(ValueError):
        dialogues_for_rank(4, 2, 2)


def test_two_ranks_gloo_independent_dialogues():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, ms = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    merged = {}
    for part in gathered:
        assert not set(part) & set(merged)          # disjoint shards
        merged.update(part)
    assert sorted(merged) == list(range(N_DIALOGUES))   # complete coverage
    for b in range(N_DIALOGUES):                     # identical to a single-process run
        assert merged[b] == _dialogue_selection(b)
    assert ms == 11.0                                # max over ranks


def test_gpu_for_rank_sharing(monkeypatch):
    """RK_SHARE_GPU=1 maps ranks onto the visible GPUs round-robin (the
    multi-rank bench on a one-GPU box); without it a rank needs its own GPU."""
    from paper_2502_15294_b200 import sharding
    monkeypatch.setattr(torch.cuda, "device_count", lambda: 1)
    monkeypatch.setenv("RK_SHARE_GPU", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")
    assert sharding.gpu_for_rank(0) == (0, True)
    assert sharding.gpu_for_rank(1) == (0, True)
    monkeypatch.setenv("RK_SHARE_GPU", "0")
    assert sharding.gpu_for_rank(0) == (0, False)
    with pytest.raises(RuntimeError):
        sharding.gpu_for_rank(1)
    # NUMA binding degrades to a no-op when the topology is not exposed
    node = sharding.bind_numa_local(0)
    assert node is None or node >= 0


def test_bench_reference_arm_under_torchrun():
    """The driver's N=2 launch of the reference arm: torchrun with two ranks,
    rank 0 prints exactly one JSON line, rank 1 exits 0 without work."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    repo = Path(__file__).resolve().parents[1]
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), str(repo / "bench.py"), "--impl", "reference", "--gpus", "2",
           "--steps", "1", "--warmup", "0"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=repo)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0


def test_host_sets_that_fit():
    """Pinned host round sets per rank: unique per dialogue when the node's ranks fit, aliased down otherwise."""
    from paper_2502_15294_b200.sharding import host_available_bytes, host_sets_that_fit
    gib = 1 << 30
    assert host_sets_that_fit(32, 2 * gib, 1, 196 * gib) == 32            # one GPU: 64 GiB of 196
    assert host_sets_that_fit(32, 2 * gib, 8, 196 * gib) == 7             # 8 ranks: floor(0.6*196/16)
    assert host_sets_that_fit(32, 2 * gib, 8, 2048 * gib) == 32           # a 2 TiB node keeps them unique
    assert host_sets_that_fit(32, 200 * gib, 8, 196 * gib) == 1           # never below one set
    assert host_sets_that_fit(32, 2 * gib, 8, 0) == 32                    # unknown host size: unchanged
    assert host_available_bytes() >= 0
