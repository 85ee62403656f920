"""BASELINE config 3: full-slot CKKS bootstrapping at N=2^16 (32768 slots).

Prints one JSON line: latency (CUDA events, warm), precision (max abs error
and bits vs the encrypted values), level budget, and the per-kernel device
time breakdown of one bootstrap."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HCNN_TEST_MODE", "1")
import numpy as np
import torch

from paper_2310_16530_b200 import _native, bootstrap as bt, ckks


def main(reps: int = 3, app_levels: int = 8):
    cfg = bt.BootConfig()
    params = bt.boot_params("boot16", 1 << 16, app_levels, cfg)
    b = bt.Bootstrapper(params, cfg)
    t0 = time.time()
    ks = b.keygen(np.random.default_rng(16), rotations=[1])
    torch.cuda.synchronize()
    t_key = time.time() - t0
    rng = np.random.default_rng(3)
    vals = rng.uniform(-1, 1, params.slots)
    ct = ckks.encrypt(ckks.encode(vals, params, 0), ks, rng)
    t0 = time.time()
    out = b.bootstrap(ct, ks)  # first run: builds masks (host encode) and tables
    torch.cuda.synchronize()
    t_first = time.time() - t0
    got = ckks.decode(ckks.decrypt(out, ks), params, imag_tol=None)
    err = float(np.max(np.abs(got - vals)))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    k0 = _native.kernel_launches()
    ev0.record()
    for _ in range(reps):
        out = b.bootstrap(ct, ks)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / reps
    launches = (_native.kernel_launches() - k0) // reps
    _native.profile_read(reset=True)
    _native.profile_enable(True)
    b.bootstrap(ct, ks)
    torch.cuda.synchronize()
    _native.profile_enable(False)
    prof = _native.profile_read(reset=True)
    tot = sum(v["ms"] for v in prof.values())
    kern = {k: {"ms": round(v["ms"], 3), "share": round(v["ms"] / tot, 3), "launches": v["launches"]}
            for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}
    print(json.dumps({
        "config": "boot16", "n": params.n, "slots": params.slots, "q_limbs": len(params.q_mods),
        "special_limbs": len(params.p_mods), "depth": cfg.depth(), "output_level": b.output_level,
        "rotation_keys": len(ks.gks), "keygen_s": round(t_key, 2), "first_bootstrap_s": round(t_first, 2),
        "bootstrap_ms": round(ms, 3), "kernel_launches": launches, "max_abs_err": err,
        "precision_bits": round(-np.log2(err), 2), "kernels": kern}))


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
