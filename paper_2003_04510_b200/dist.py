"""Multi-GPU batching of independent HE Muls.

One process per GPU; a batch of B ciphertext pairs is split into contiguous
blocks, one per rank, with the evaluation key replicated (each rank builds
its own level tables and evk forms). There is no collective on the compute
path: ranks only agree on the slowest rank's time (max all-reduce) and send
their outputs / digests to rank 0 after the timed region. The reference has
no multi-process path at all (thread_pool.hpp:17-98 is its only
parallelism), so this module adds the one thing a batch needs.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Any, Callable


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    start: int  # first pair of this rank
    count: int  # pairs on this rank


def shard(total: int, rank: int, world: int) -> Shard:
    """Contiguous, balanced split of `total` pairs: the first total % world
    ranks get one extra pair."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError("bad shard request")
    base, extra = divmod(total, world)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return Shard(rank, world, start, count)


def max_over_ranks(value: float, device: Any = None) -> float:
    """The slowest rank's time (all-reduce MAX); identity without a process
    group."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    if dist.get_backend() != "nccl":  # gloo reduces host tensors
        device = None
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_to_rank0(obj: Any) -> list[Any] | None:
    """Every rank's `obj` on rank 0 (None elsewhere); [obj] without a group."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [obj]
    world = dist.get_world_size()
    out = [None] * world if dist.get_rank() == 0 else None
    dist.gather_object(obj, out, dst=0)
    return out


def run_sharded(total: int, rank: int, world: int,
                compute: Callable[[int, int], list[Any]]) -> list[Any] | None:
    """compute(start, count) -> per-pair results for this rank's block;
    returns all results in pair order on rank 0 (None on other ranks)."""
    s = shard(total, rank, world)
    local = compute(s.start, s.count) if s.count else []
    parts = gather_to_rank0(local)
    if parts is None:
        return None
    return [r for part in parts for r in part]
