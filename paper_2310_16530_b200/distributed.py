"""Data-parallel sharding of independent encrypted inferences across GPUs.

The path partitions naturally: every encrypted image is an
independent ``graph.execute`` with read-only keys and masks, so N GPUs run N
shards with no collective on the data path.  One process per GPU
(torchrun); each rank owns a contiguous block of the batch, keys are
replicated (generated from the same seed on every rank, bit-identical), and
the only communication is control-plane: a barrier around timed regions,
a MAX reduction of the per-rank device time, and an optional gather of the
decrypted results to rank 0.  Works over NCCL (GPU) and gloo (CPU tests).
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Any, Callable, Sequence


@dataclass(frozen=True)
class ShardPlan:
    """Contiguous block partition of `total` items over `world` ranks
    (the first total % world ranks get one extra item)."""

    total: int
    world: int

    def bounds(self, rank: int) -> tuple[int, int]:
        base, extra = divmod(self.total, self.world)
        lo = rank * base + min(rank, extra)
        return lo, lo + base + (1 if rank < extra else 0)

    def indices(self, rank: int) -> range:
        lo, hi = self.bounds(rank)
        return range(lo, hi)


def env_rank() -> tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def max_over_ranks(value: float, device=None) -> float:
    """MAX-reduce a scalar over the default process group (identity when
    torch.distributed is not initialised)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_sharded(items: Sequence[Any], fn: Callable[[Any], Any], gather: bool = True) -> list[Any] | None:
    """Apply `fn` to this rank's shard of `items`; with `gather`, rank 0
    receives the full, ordered result list (other ranks get None)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return [fn(x) for x in items]
    rank, world = dist.get_rank(), dist.get_world_size()
    plan = ShardPlan(len(items), world)
    mine = [(i, fn(items[i])) for i in plan.indices(rank)]
    if not gather:
        return None
    parts: list[Any] = [None] * world
    dist.all_gather_object(parts, mine)
    if rank != 0:
        return None
    out: list[Any] = [None] * len(items)
    for part in parts:
        for i, v in part:
            out[i] = v
    return out
