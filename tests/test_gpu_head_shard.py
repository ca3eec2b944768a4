"""KV-head sharding of every dialogue (SURVEY §8e's option for fewer dialogues
than GPUs): `world` engines each hold kv-heads [rank hkv/world, ...) of every
layer — caches, host rounds, the projections' columns and W_o's rows — and
exchange only (a) each layer's output-projection partial and (b) the per-round
fp64 masses before selection, through an all-reduce.  Here the ranks run as
threads on one GPU with an in-process all-reduce (summing in rank order, like a
ring), and must keep the same rounds, answers and residual stream as the
unsharded engine over several turns (gathers, writebacks and the round cache
included)."""

from __future__ import annotations

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2502_15294_b200.decode_engine import RoundDecodeEngine  # noqa: E402
from paper_2502_15294_b200.decode_model import DecodeModel  # noqa: E402

from test_gpu_engine import _small_cfg  # noqa: E402


class ThreadAllReduce:
    """In-place sum over `world` threads' device tensors (rank order)."""

    def __init__(self, world: int):
        self.world = world
        self.bar = threading.Barrier(world, timeout=120)
        self.slots = [None] * world
        self.calls = 0

    def fn(self, rank: int):
        def all_reduce(t):
            torch.cuda.current_stream().synchronize()
            self.slots[rank] = t
            self.bar.wait()
            total = self.slots[0].clone()
            for r in range(1, self.world):
                total += self.slots[r]
            torch.cuda.current_stream().synchronize()
            self.bar.wait()                       # every rank has read every slot
            t.copy_(total)
            torch.cuda.current_stream().synchronize()
            if rank == 0:
                self.calls += 1
        return all_reduce


def _run_threads(engines, turns):
    out = [[] for _ in engines]
    errors = []

    def work(i):
        try:
            eng = engines[i]
            with torch.cuda.stream(eng.compute_stream):
                for _ in range(turns):
                    kept = eng.run_turn_eager()
                    torch.cuda.current_stream().synchronize()
                    out[i].append(([tuple(int(r) for r in k) for k in kept], eng.answers().copy(),
                                   eng.x.cpu().numpy().copy()))
        except Exception as e:      # pragma: no cover - surfaced below
            errors.append(e)
    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(engines))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return out


@pytest.mark.parametrize("world,hkv,G,batch", [(2, 2, 4, 2), (2, 4, 7, 1), (4, 4, 4, 3)])
def test_head_sharded_turns_match_unsharded(world, hkv, G, batch):
    cfg = _small_cfg(hq=hkv * G, hkv=hkv, batch=batch, decode_steps=5, question_variants=2)
    dialogues = [3 + 5 * b for b in range(batch)]
    turns = 3
    full = RoundDecodeEngine(cfg, model=DecodeModel(cfg.shape, "cuda", seed=3), dialogues=dialogues)
    ref = _run_threads([full], turns)[0]
    ar = ThreadAllReduce(world)
    shards = [RoundDecodeEngine(cfg, model=DecodeModel(cfg.shape, "cuda", seed=3, shard=(r, world)),
                                dialogues=dialogues, head_shard=(r, world), all_reduce=ar.fn(r))
              for r in range(world)]
    assert shards[0].lower.shape[4] == hkv // world
    got = _run_threads(shards, turns)
    # per layer of every token one exchange, plus the masses once per turn
    steps = cfg.decode_steps + 1
    assert ar.calls == turns * (1 + cfg.num_layers * steps)
    for t in range(turns):
        k_ref, a_ref, x_ref = ref[t]
        for r in range(world):
            k, a, x = got[r][t]
            assert k == k_ref, (t, r)                               # every rank keeps the reference's rounds
            np.testing.assert_array_equal(a, a_ref)                 # greedy answers
            np.testing.assert_array_equal(x, got[0][t][2])          # ranks agree bit for bit
            np.testing.assert_array_equal(x, x_ref)                 # embedding of the same final token


def test_head_shard_validation():
    cfg = _small_cfg(batch=1)
    with pytest.raises(ValueError):
        RoundDecodeEngine(cfg, head_shard=(0, 2))                   # no all_reduce
    with pytest.raises(ValueError):
        DecodeModel(cfg.shape, "cuda", seed=1, shard=(0, 3))       # 2 kv-heads over 3 ranks
    m = DecodeModel(cfg.shape, "cuda", seed=1, shard=(1, 2))
    with pytest.raises(ValueError):
        RoundDecodeEngine(cfg, model=m)                             # model / engine shard mismatch


def _dist_rank(rank, world, port, out_dir):
    import os

    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = _small_cfg(batch=2, decode_steps=4)
        eng = RoundDecodeEngine(cfg, model=DecodeModel(cfg.shape, "cuda", seed=3, shard=(rank, world)),
                                dialogues=[3, 8], head_shard=(rank, world), all_reduce=dist.all_reduce)
        res = _run_threads([eng], 2)[0]
        np.savez(f"{out_dir}/rank{rank}.npz", **{f"kept{t}": np.array(k) for t, (k, _, _) in enumerate(res)},
                 **{f"ans{t}": a for t, (_, a, _) in enumerate(res)}, **{f"x{t}": x for t, (_, _, x) in enumerate(res)})
    finally:
        dist.destroy_process_group()


def test_head_shard_over_torch_distributed(tmp_path):
    """The same exchange through torch.distributed.all_reduce (two processes on
    this GPU, gloo on CUDA tensors; NCCL between GPUs): both ranks reproduce the
    unsharded turns."""
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mp.start_processes(_dist_rank, args=(2, port, str(tmp_path)), nprocs=2, start_method="spawn")
    cfg = _small_cfg(batch=2, decode_steps=4)
    full = RoundDecodeEngine(cfg, model=DecodeModel(cfg.shape, "cuda", seed=3), dialogues=[3, 8])
    ref = _run_threads([full], 2)[0]
    for r in range(2):
        z = np.load(tmp_path / f"rank{r}.npz")
        for t, (k, a, x) in enumerate(ref):
            np.testing.assert_array_equal(z[f"kept{t}"], np.array(k))
            np.testing.assert_array_equal(z[f"ans{t}"], a)
            np.testing.assert_array_equal(z[f"x{t}"], x)
