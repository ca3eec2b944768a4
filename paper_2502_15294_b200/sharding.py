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
