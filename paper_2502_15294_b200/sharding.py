"""Multi-GPU layout of the round-attention path: independent dialogues.

Dialogues share nothing (pipeline.py:115 "one pipeline per conversation",
SPEC.md:518), so N GPUs serve N disjoint dialogue shards with no collective on
the data path: dialogue b belongs to rank b mod N, every rank
owns its HBM tiers, pinned host blocks and copy stream.  torch.distributed is
used only for the launch barrier and the max-over-ranks timing.
"""

from __future__ import annotations


def dialogues_for_rank(total: int, world: int, rank: int) -> list:
    """Round-robin shard: dialogue b -> rank b % world."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return list(range(rank, total, world))


def per_rank_batch(total: int, world: int) -> int:
    """Dialogues per rank for weak scaling (equal shards)."""
    if total % world:
        raise ValueError(f"{total} dialogues do not split evenly over {world} ranks")
    return total // world


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank timing (the job finishes with its slowest rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], device=device or ("cuda" if dist.get_backend() == "nccl" else "cpu"))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gpu_for_rank(local_rank: int) -> tuple[int, bool]:
    """(device index, shared) for this rank: one GPU per rank (local_rank);
    RK_SHARE_GPU=1 maps ranks onto the visible GPUs round-robin
    (local_rank % device_count) so the multi-rank path runs on a one-GPU box."""
    import os

    import torch
    n = torch.cuda.device_count()
    if os.environ.get("RK_SHARE_GPU", "0") == "1":
        return local_rank % max(1, n), int(os.environ.get("WORLD_SIZE", "1")) > n
    if local_rank >= n:
        raise RuntimeError(f"local rank {local_rank} but only {n} visible GPUs (set RK_SHARE_GPU=1 to share)")
    return local_rank, False


def _cpulist(text: str) -> set:
    cpus = set()
    for part in text.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        else:
            cpus.add(int(part))
    return cpus


def bind_numa_local(device_index: int):
    """Pin this process to the CPUs of its GPU's NUMA node, so the pinned host
    pools it allocates next (the deep-layer round blocks, first touched by this
    process) are NUMA-local to the GPU's PCIe root.  Returns the
    node, or None when the topology is not exposed (no binding)."""
    import os
    from pathlib import Path

    import torch
    try:
        props = torch.cuda.get_device_properties(device_index)
        bus = f"{props.pci_domain_id:04x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
        node = int(Path(f"/sys/bus/pci/devices/{bus}/numa_node").read_text())
        if node < 0:
            return None
        cpus = _cpulist(Path(f"/sys/devices/system/node/node{node}/cpulist").read_text())
        if cpus:
            os.sched_setaffinity(0, cpus)
        return node
    except Exception:
        return None


def host_available_bytes() -> int:
    """MemAvailable of this host (bytes), 0 when /proc/meminfo is not readable."""
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def host_sets_that_fit(wanted: int, set_bytes: int, ranks_on_node: int, available: int,
                       frac: float = 0.6) -> int:
    """Distinct pinned host round sets per rank that fit this node.

    Every rank on the node pins `wanted` sets of `set_bytes` (one per dialogue,
    the reference's one store per conversation, store.py:110-129); when all of
    them would exceed `frac` of the host's available memory the sets are aliased
    (the engine's host_unique) down to what fits, at least one.  Returns `wanted`
    when it fits or the host size is unknown (available == 0)."""
    if wanted < 1 or set_bytes <= 0 or available <= 0:
        return wanted
    fit = int(frac * available) // (set_bytes * max(1, ranks_on_node))
    return max(1, min(wanted, fit))
