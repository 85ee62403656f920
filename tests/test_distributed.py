"""Multi-rank host logic over gloo (world_size 2, CPU): shard partition,
ordered gather to rank 0, MAX-over-ranks timing -- the same code bench.py
and multi-GPU inference use over NCCL."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def test_shard_plan_covers_exactly_once():
    from paper_2310_16530_b200.distributed import ShardPlan
    for total in range(0, 23):
        for world in (1, 2, 3, 4, 8):
            p = ShardPlan(total, world)
            seen = [i for r in range(world) for i in p.indices(r)]
            assert seen == list(range(total))
            sizes = [len(p.indices(r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2310_16530_b200 import distributed as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        items = list(range(7))
        out = D.run_sharded(items, lambda x: (x * x, rank))
        t = D.max_over_ranks(10.0 + rank)
        if rank == 0:
            q.put((out, t))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [v for v, _ in out] == [x * x for x in range(7)]
    # first 4 items on rank 0, last 3 on rank 1
    assert [r for _, r in out] == [0, 0, 0, 0, 1, 1, 1]
    assert t == 11.0


def test_bench_multi_rank_path_gloo():
    """bench.py --gpus 2 without torchrun re-launches itself as 2 ranks under
    torch.distributed.run (127.0.0.1 rendezvous) and runs the same
    Cluster -> shard -> timed -> gather skeleton the GPU workloads use
    (here over gloo with a CPU stub step): one JSON line from rank 0 with
    every image owned by exactly one rank."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--workload", "selftest",
                        "--images-per-gpu", "3", "--steps", "2", "--warmup", "1"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["backend"] == "gloo" and line["warmup"] == 3
    owned = sorted(i for p in line["per_rank"] for i in p["images"])
    assert owned == list(range(6))
    assert [p["images"] for p in sorted(line["per_rank"], key=lambda p: p["rank"])] == [[0, 1, 2], [3, 4, 5]]
    assert line["ms_per_step"] > 0 and line["value"] > 0
