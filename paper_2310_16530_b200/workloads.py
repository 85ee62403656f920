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


# the ResNet20 chain: q0 + application levels + bootstrapping depth = 30 q-limbs
# (+ RESNET20_N_SPECIAL specials: logQP 1759 <= 1772, the 128-bit bound at N=2^16).
# 30 keeps the 6-bootstrap refresh plan of 31 (refresh points 7/17/27/37) with
# every op one limb narrower (29 re-plans to 7 bootstraps: 601 ms/image)
RESNET20_Q_LIMBS = 30
# EvalMod's Chebyshev degree before the 3 double angles.  The bootstrap
# multiplies the sin approximation error by ~sqrt(N) q0 / (2 pi Delta_1) =
# 2^8 * 2^12 / 2 pi ~ 2^17.3 (every slot sums N coefficients), so 59 (2^-43)
# keeps bootstraps at the noise floor (19.6 bits, boot16) while 31 (2^-25.5,
# one level less) measured 8 bits (tools/boot_precision.py) -- rejected
RESNET20_EVALMOD_DEGREE = 59


def resnet20_boot_config(stc_stages=None, degree=None) -> bt.BootConfig:
    """Bootstrapping configuration of the ResNet20 workload (HCNN_STC env:
    e.g. "8,7"; HCNN_EVALMOD_DEGREE: the Chebyshev degree before the double
    angles)."""
    import os
    env = os.environ.get("HCNN_STC")
    if stc_stages is None and env:
        stc_stages = tuple(int(v) for v in env.split(","))
    if degree is None:
        degree = int(os.environ.get("HCNN_EVALMOD_DEGREE", RESNET20_EVALMOD_DEGREE))
    kw = {}
    if stc_stages is not None:
        kw["stc_stages"] = tuple(stc_stages)
    if degree is not None:
        kw["degree"] = int(degree)
    if os.environ.get("HCNN_BSGS_BABY"):
        kw["bsgs_baby"] = int(os.environ["HCNN_BSGS_BABY"])
    if os.environ.get("HCNN_DOUBLE_ANGLE"):
        kw["double_angle"] = int(os.environ["HCNN_DOUBLE_ANGLE"])
    return bt.BootConfig(**kw)


# special primes K (= alpha, the key-switch digit size): 5 x 61 bits spends
# the slack of the 30-limb chain under logQP 1772 on fewer digits --
# ceil(n_q/5) instead of ceil(n_q/4): fewer ModUp NTTs, 23 % smaller keys
# (360.3 -> 354.5 ms/image on the same chain)
RESNET20_N_SPECIAL = 5


def resnet20_n_special() -> int:
    """Special primes of the ResNet20 chain (HCNN_N_SPECIAL overrides)."""
    import os
    return int(os.environ.get("HCNN_N_SPECIAL", RESNET20_N_SPECIAL))


# bits of the CtS / EvalMod primes at the top of the chain (HCNN_BIG_BITS overrides)
RESNET20_BIG_BITS = 58


def resnet20_big_bits() -> int:
    import os
    return int(os.environ.get("HCNN_BIG_BITS", RESNET20_BIG_BITS))


def resnet20_special_bits():
    """Bits of each special prime (HCNN_SPECIAL_BITS, e.g. "61,40,40,40,40";
    default: RESNET20_N_SPECIAL primes of 61 bits)."""
    import os
    env = os.environ.get("HCNN_SPECIAL_BITS")
    if env:
        return tuple(int(v) for v in env.split(","))
    return (61,) * resnet20_n_special()


def resnet20_params(name: str, app_levels: int, cfg: bt.BootConfig) -> ckks.CkksParams:
    sb = resnet20_special_bits()
    return bt.boot_params(name, 1 << 16, app_levels, cfg, n_special=len(sb), special_bits=sb,
                          big_bits=resnet20_big_bits())


def resnet20_app_levels(cfg: bt.BootConfig) -> int:
    """Application levels of a fixed-length chain: what the bootstrap does not
    use (HCNN_Q_LIMBS overrides the chain length)."""
    import os
    return int(os.environ.get("HCNN_Q_LIMBS", RESNET20_Q_LIMBS)) - 1 - cfg.depth()


def resnet20_setup(app_levels: int | None = None, seed: int = 3, key_seed: int = 20) -> ResNet20Setup:
    """BASELINE config 4: AESPA-ResNet20 (CIFAR-10 shape 3x32x32), HyPHEN
    packing with multiplex 4 at N=2^16 (r >= m for FormatB, packing.py:489),
    bootstrappable chain with `app_levels` computation levels, real CKKS
    bootstrapping at the snapshot-aware planner's refresh points."""
    packing.set_mask_mode("compact")
    cfg = resnet20_boot_config()
    if app_levels is None:  # keep the chain length (logQP) fixed: bootstrap levels trade for application levels
        app_levels = resnet20_app_levels(cfg)
    params = resnet20_params("resnet20-16", app_levels, cfg)
    boot = bt.Bootstrapper(params, cfg)
    fx = graph.gen_fixture("resnet20", seed, params, golden_count=1)
    g = graph.build_graph("resnet20", fx, multiplex=4)
    plan = graph.plan_levels(g, boot.output_level, refresh_target=boot.output_level,
                             refresh_cost=graph.refresh_bootstraps(g, params.slots))
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


def resnet20_plan_only(app_levels: int | None = None, seed: int = 3):
    """Host-only part of resnet20_setup (params, graph, plan; no keys/GPU)."""
    cfg = resnet20_boot_config()
    if app_levels is None:
        app_levels = resnet20_app_levels(cfg)
    params = resnet20_params("resnet20-16", app_levels, cfg)
    fx = graph.gen_fixture("resnet20", seed, params, golden_count=1)
    g = graph.build_graph("resnet20", fx, multiplex=4)
    out_level = params.max_level - cfg.depth()
    plan = graph.plan_levels(g, out_level, refresh_target=out_level, refresh_cost=graph.refresh_bootstraps(g, params.slots))
    return params, g, plan


def warm_up(s: ResNet20Setup, ct, cache: dict) -> dict:
    """First two eager inferences of a workload, sizing mask residency from
    measurement instead of a guess: run 1 builds every mask (compact, none
    resident) and measures the largest transient working set of any layer
    W (peak minus the layer's starting footprint); run 2 keeps masks
    resident while 1.5 W + 3 GiB stays free -- room for the CUDA-graph
    capture (graph.CapturedInference) and the live activations.  `ct` may
    be a list of images: both runs then go through graph.execute_many, so
    W includes the batched bootstraps of all of them."""
    cts = list(ct) if isinstance(ct, (list, tuple)) else [ct]
    import os
    import time
    import torch
    packing.set_residency(False)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    marks: dict = {}
    work = [0]

    def hook(i, phase):
        torch.cuda.synchronize()
        if phase == "start":
            marks["start"] = torch.cuda.memory_allocated()
            torch.cuda.reset_peak_memory_stats()
        else:  # transient only: compact masks created by the layer persist and are not working set
            end = torch.cuda.memory_allocated()
            work[0] = max(work[0], torch.cuda.max_memory_allocated() - max(marks["start"], end))

    t0 = time.time()
    graph.execute_many(s.graph, s.plan, cts, s.ks, cache=cache, layer_hook=hook)
    torch.cuda.synchronize()
    t_build = time.time() - t0
    after = torch.cuda.memory_allocated()
    # headroom for the graph pool and live activations: HCNN_RESERVE_MULT x the
    # largest transient layer working set + 3 GiB (1.5 measured safe)
    reserve = int(float(os.environ.get("HCNN_RESERVE_MULT", "1.5")) * work[0]) + (3 << 30)
    torch.cuda.empty_cache()
    packing.set_residency(True, reserve)
    t0 = time.time()
    graph.execute_many(s.graph, s.plan, cts, s.ks, cache=cache)
    torch.cuda.synchronize()
    return {"first_image_s": round(t_build, 2), "residency_fill_s": round(time.time() - t0, 2),
            "layer_working_set_gb": round(work[0] / 2 ** 30, 2),
            "persistent_growth_gb": round((after - base) / 2 ** 30, 2),
            "reserve_gb": round(reserve / 2 ** 30, 2), "resident_mask_gb": round(packing.resident_bytes() / 2 ** 30, 1)}
