"""Benchmark workload builders (BASELINE.json configs), shared by bench.py
and tools/.  All data is synthetic and seeded; weights are random-init of
the named architecture (no checkpoints exist offline)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import bootstrap as bt
from . import ckks, graph, packing


@dataclass
class ResNet20Setup:
    params: ckks.CkksParams
    cfg: bt.BootConfig
    boot: bt.Bootstrapper
    fixture: dict
    graph: graph.HcnnGraph
    plan: graph.LevelPlan
    ks: ckks.KeySet


def resnet20_setup(app_levels: int = 14, seed: int = 3, key_seed: int = 20) -> ResNet20Setup:
    """BASELINE config 4: AESPA-ResNet20 (CIFAR-10 shape 3x32x32), HyPHEN
    packing with multiplex 4 at N=2^16 (r >= m for FormatB, packing.py:489),
    bootstrappable chain with `app_levels` computation levels, real CKKS
    bootstrapping at the snapshot-aware planner's refresh points."""
    packing.set_mask_mode("compact")
    cfg = bt.BootConfig()
    params = bt.boot_params("resnet20-16", 1 << 16, app_levels, cfg)
    boot = bt.Bootstrapper(params, cfg)
    fx = graph.gen_fixture("resnet20", seed, params, golden_count=1)
    g = graph.build_graph("resnet20", fx, multiplex=4)
    plan = graph.plan_levels(g, boot.output_level, refresh_target=boot.output_level, count_snapshots=True)
    steps = graph.required_rotation_steps(g, params.slots) | graph.refresh_rotation_steps(g, plan, params.slots)
    ks = boot.keygen(np.random.default_rng(key_seed), rotations=sorted(steps))
    # keys used only at application levels keep their low-level rows (HBM for resident masks)
    ks.truncate_rotations(sorted(set(steps) - boot.rotation_steps()), boot.output_level)
    return ResNet20Setup(params, cfg, boot, fx, g, plan, ks)


def encrypt_image(s: ResNet20Setup, x: np.ndarray, rng: np.random.Generator) -> packing.PackedTensor:
    return packing.encrypt_tensor(x, s.graph.input_format, s.ks, rng, s.plan.entry_levels[0])


CFG2 = dict(n=1 << 16, log_q0=59, log_qi=40, levels=24, log_p=59, n_special=4)


def cfg2_params() -> ckks.CkksParams:
    """BASELINE config 2: CkksParams.build("bench16", 1<<16, 59, 40, 24, 59, 4)."""
    return ckks.CkksParams.build("bench16", CFG2["n"], CFG2["log_q0"], CFG2["log_qi"], CFG2["levels"],
                                 CFG2["log_p"], CFG2["n_special"])


# per-image op tally of resnet20_setup()'s encrypted inference
# (graph.CostReport.totals(); profiles/r01_resnet20_graph.json) -- lets the
# host-only reference arm extrapolate without running the GPU executor
RESNET20_TALLY = {"rotations": 1964, "hmults": 172, "pmults": 44464, "hadds": 44856, "rescales": 793,
                  "refreshes": 32}


def resnet20_plan_only(app_levels: int = 14, seed: int = 3):
    """Host-only part of resnet20_setup (params, graph, plan; no keys/GPU)."""
    cfg = bt.BootConfig()
    params = bt.boot_params("resnet20-16", 1 << 16, app_levels, cfg)
    fx = graph.gen_fixture("resnet20", seed, params, golden_count=1)
    g = graph.build_graph("resnet20", fx, multiplex=4)
    out_level = params.max_level - cfg.depth()
    plan = graph.plan_levels(g, out_level, refresh_target=out_level, count_snapshots=True)
    return params, g, plan
