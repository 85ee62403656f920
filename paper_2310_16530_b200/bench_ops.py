"""`bench-ops` on the GPU (the reference's
cli.py:259-310 `_bench_closures` / `_cmd_bench_ops`).

    python -m paper_2310_16530_b200.bench_ops [--params desk-A] [--reps 25] [--seed 0] [--batch 1] [--out FILE]

Same report schema as the reference (version, command, params, reps,
ops{name: median_ms, iqr_ms}, hmult_gt_hadd, note, insecure), timed the same
way (3 warm-up calls, then per-call wall clock around a synchronised call),
plus the GPU fields SURVEY §8f asks for: per-op device time from CUDA
events, algorithmic bytes and the HBM roofline fraction, GPU
name/count.  --batch B times every op on B ciphertexts at once (the batched
engine entry points) and reports per-ciphertext numbers.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import time

import numpy as np
import torch

from . import ckks, graph
from .ring import to_mont_rows

BENCH_OPS = ("encode", "hadd", "pmult", "hmult", "rescale", "rotate")


def _peak_gbs() -> float:
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(here, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f).get("hbm_gbs", 6450.0))
    except OSError:
        return 6450.0


def algorithmic_bytes(op: str, params: ckks.CkksParams, level: int) -> float:
    """Minimal one-pass traffic per op, bytes."""
    lb = params.n * 8
    nq = level + 1
    K = len(params.p_mods)
    d = -(-nq // K) if K else 0
    return lb * {
        "encode": nq,                                   # write the residues
        "hadd": 6 * nq,
        "pmult": 5 * nq,
        "hmult": 4 * nq + 2 * d * (nq + K) + 2 * nq,
        "rescale": 2 * nq + 2 * (nq - 1),
        "rotate": 2 * nq + 2 * d * (nq + K) + 2 * nq,
    }[op]


def bench_closures(params: ckks.CkksParams, ks: ckks.KeySet, rng: np.random.Generator, batch: int = 1):
    """The reference's closures (cli.py:259-276); batch > 1 stacks ciphertexts."""
    vals = rng.uniform(-1, 1, params.slots)
    level = params.max_level
    pt = ckks.encode(vals, params, level)
    enc = lambda: ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, level), ks, rng)
    if batch > 1:
        a = ckks.stack([enc() for _ in range(batch)])
        b = ckks.stack([enc() for _ in range(batch)])
    else:
        a, b = ckks.encrypt(pt, ks, rng), enc()
    rows = to_mont_rows(pt.poly)
    product = ckks.hmult(a, b, ks)
    return {
        "encode": lambda: ckks.encode(vals, params, level),
        "hadd": lambda: ckks.hadd(a, b),
        "pmult": lambda: ckks.pmult_mont(a, rows, pt.scale),
        "hmult": lambda: ckks.hmult(a, b, ks),
        "rescale": lambda: ckks.rescale(product, params),
        "rotate": lambda: ckks.rotate(a, 1, ks),
    }


def run(params_name: str = "desk-A", reps: int = 25, seed: int = 0, batch: int = 1) -> dict:
    params = ckks.params_by_name(params_name)
    rng = np.random.default_rng(seed)
    ks = ckks.keygen(params, rng, rotations=[1])
    closures = bench_closures(params, ks, rng, batch)
    peak = _peak_gbs()
    results = {}
    for name in BENCH_OPS:
        fn = closures[name]
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            times.append((time.perf_counter() - t0) * 1e3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        dev_ms = e0.elapsed_time(e1) / reps
        q1, med, q3 = statistics.quantiles(times, n=4) if reps >= 2 else (times[0],) * 3
        nb = 1 if name == "encode" else batch
        by = algorithmic_bytes(name, params, params.max_level) * nb
        gbs = by / (dev_ms / 1e3) / 1e9
        results[name] = {
            "median_ms": round(med / nb, 4),
            "iqr_ms": round((q3 - q1) / nb, 4),
            "device_ms": round(dev_ms / nb, 5),
            "algorithmic_bytes": int(by / nb),
            "GBps": round(gbs, 1),
            "roofline_frac": round(gbs / peak, 4),
        }
    return {
        "version": graph.REPORT_VERSION,
        "command": "bench-ops",
        "params": params.name,
        "reps": reps,
        "batch": batch,
        "ops": results,
        "hmult_gt_hadd": results["hmult"]["median_ms"] > results["hadd"]["median_ms"],
        "note": "B200 engine: median_ms = wall clock per synchronised call (per ciphertext for --batch); "
                "device_ms from CUDA events; encode runs its FFT on the host",
        "insecure": params.toy,
        "gpu": torch.cuda.get_device_name(0),
        "gpu_count": 1,
        "hbm_peak_gbs": peak,
    }


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="bench-ops")
    ap.add_argument("--params", default="desk-A", help="parameter preset (desk-A, desk-B, unit, bench16)")
    ap.add_argument("--reps", type=int, default=25)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--out", default=None)
    args = ap.parse_args(argv)
    rep = run(args.params, args.reps, args.seed, args.batch)
    txt = json.dumps(rep, indent=1)
    if args.out:
        with open(args.out, "w") as f:
            f.write(txt + "\n")
    print(txt)
    return 0


if __name__ == "__main__":
    sys.exit(main())
