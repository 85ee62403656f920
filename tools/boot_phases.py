"""Per-phase device time of a batched bootstrap on the ResNet20 chain
(N=2^16, 31 q-limbs): CoeffToSlot, conjugate/split, EvalMod (both halves of
every entry in one pass), SlotToCoeff; plus the per-kernel split.

    python tools/boot_phases.py [nb] [reps]"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HCNN_TEST_MODE", "1")
import numpy as np
import torch

from paper_2310_16530_b200 import _native, bootstrap as bt, ckks


def main(nb: int = 8, reps: int = 3):
    cfg = bt.BootConfig()
    params = bt.boot_params("resnet20-16", 1 << 16, 14, cfg)
    b = bt.Bootstrapper(params, cfg)
    ks = b.keygen(np.random.default_rng(16), rotations=[1])
    rng = np.random.default_rng(3)
    vals = [rng.uniform(-1, 1, params.slots) for _ in range(nb)]
    cts = [ckks.encrypt(ckks.encode(v, params, 3), ks, rng) for v in vals]
    X = ckks.stack(cts) if nb > 1 else cts[0]
    out = b.bootstrap(X, ks)  # warm: masks, tables
    got = [ckks.decode(ckks.decrypt(o, ks), params, imag_tol=None) for o in ckks.unstack(out)]
    err = max(float(np.max(np.abs(g - v))) for g, v in zip(got, vals))
    phases: dict = {}
    for _ in range(reps):
        marks = []
        b.phase_hook = lambda name: marks.append((name, torch.cuda.Event(enable_timing=True)))
        torch.cuda.synchronize()
        orig = b.phase_hook

        def hook(name, marks=marks):
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append((name, e))
        b.phase_hook = hook
        b.bootstrap(X, ks)
        torch.cuda.synchronize()
        for (n0, e0), (n1, e1) in zip(marks, marks[1:]):
            phases[n1] = phases.get(n1, 0.0) + e0.elapsed_time(e1) / reps
    b.phase_hook = None
    _native.profile_read(reset=True)
    _native.profile_enable(True)
    b.bootstrap(X, ks)
    torch.cuda.synchronize()
    _native.profile_enable(False)
    prof = _native.profile_read(reset=True)
    print(json.dumps({"nb": nb, "q_limbs": len(params.q_mods), "ms_total": round(sum(phases.values()), 3),
                      "ms_per_ct": round(sum(phases.values()) / nb, 3),
                      "phases_ms": {k: round(v, 3) for k, v in phases.items()}, "max_abs_err": err,
                      "kernels_ms": {k: round(v["ms"], 3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}}),
          flush=True)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
