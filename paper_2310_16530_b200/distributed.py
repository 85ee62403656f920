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
import socket
import subprocess
import sys
import time
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


class Cluster:
    """One process per GPU (torchrun environment): device binding, process
    group (NCCL on GPUs, gloo on CPU), barrier, MAX over ranks, ordered
    gather to rank 0 and the timed region every multi-rank number goes
    through.  world_size 1 needs no process group and is the identity."""

    def __init__(self, backend: str | None = None):
        import torch
        self.torch = torch
        self.rank, self.local, self.world = env_rank()
        self.cuda = torch.cuda.is_available() and backend != "gloo"
        if self.cuda:
            torch.cuda.set_device(self.local)
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            be = backend or ("nccl" if self.cuda else "gloo")
            if not dist.is_initialized():
                kw = {"device_id": torch.device(f"cuda:{self.local}")} if be == "nccl" else {}
                dist.init_process_group(be, rank=self.rank, world_size=self.world, **kw)
            self.dist = dist

    def sync(self):
        if self.cuda:
            self.torch.cuda.synchronize()

    def barrier(self):
        self.sync()
        if self.dist is not None:
            self.dist.barrier()
        self.sync()

    def max(self, v: float) -> float:
        if self.dist is None:
            return float(v)
        dev = "cuda" if self.cuda else "cpu"
        t = self.torch.tensor([float(v)], device=dev, dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def gather(self, obj: Any) -> list[Any] | None:
        """Rank 0 gets [obj of rank 0, obj of rank 1, ...]; others None."""
        if self.dist is None:
            return [obj]
        parts: list[Any] = [None] * self.world
        self.dist.all_gather_object(parts, obj)
        return parts if self.rank == 0 else None

    def shard(self, total: int) -> range:
        return ShardPlan(total, self.world).indices(self.rank)

    def timed(self, fn: Callable[[], Any], steps: int, nvtx: str | None = None) -> float:
        """ms over `steps` calls of fn between two barriers (+ device syncs),
        CUDA events on the current stream (wall clock on CPU); MAX over ranks."""
        torch = self.torch
        self.barrier()
        if self.cuda:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if nvtx:
                torch.cuda.nvtx.range_push(nvtx)
            e0.record()
            for _ in range(steps):
                fn()
            e1.record()
            if nvtx:
                torch.cuda.nvtx.range_pop()
            self.barrier()
            ms = e0.elapsed_time(e1)
        else:
            t0 = time.perf_counter()
            for _ in range(steps):
                fn()
            self.barrier()
            ms = (time.perf_counter() - t0) * 1e3
        return self.max(ms)

    def close(self):
        if self.dist is not None and self.dist.is_initialized():
            self.dist.destroy_process_group()


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(nproc: int, script: str, argv: Sequence[str]) -> int:
    """Re-run `script argv` as `nproc` ranks under torch.distributed.run on
    this node (one process per GPU, rendezvous on 127.0.0.1); returns the
    launcher's exit code.  Used when a multi-GPU run is started without
    torchrun (bench.py --gpus N)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", script, *argv]
    return subprocess.call(cmd)
