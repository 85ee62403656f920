"""Batched vs per-ciphertext key switching on the ResNet20 bootstrapping
chain (N=2^16, 31 q-limbs, 4 special): hmult and one rotation of nb
ciphertexts, at a high and a low level.  Prints one JSON line per case with
per-kernel device time."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HCNN_TEST_MODE", "1")
import numpy as np
import torch

from paper_2310_16530_b200 import _native, bootstrap as bt, ckks


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def profile(fn):
    _native.profile_read(reset=True)
    _native.profile_enable(True)
    fn()
    torch.cuda.synchronize()
    _native.profile_enable(False)
    p = _native.profile_read(reset=True)
    return {k: round(v["ms"], 3) for k, v in sorted(p.items(), key=lambda kv: -kv[1]["ms"])}


def main(nb: int = 8, ks_batch: int = 4):
    _native.set_option("ks_batch", ks_batch)
    cfg = bt.BootConfig()
    params = bt.boot_params("resnet20-16", 1 << 16, 14, cfg)
    ks = ckks.keygen(params, np.random.default_rng(1), rotations=[1])
    rng = np.random.default_rng(2)
    for level in (params.max_level, 10):
        cts = [ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, level), ks, rng) for _ in range(nb)]
        B = ckks.stack(cts)
        cases = {
            "hmult_single": lambda: [ckks.hmult(c, c, ks) for c in cts],
            "hmult_batch": lambda: ckks.hmult(B, B, ks),
            "rot_single": lambda: [ckks.rotate(c, 1, ks) for c in cts],
            "rot_batch": lambda: ckks.rotate(B, 1, ks),
            "rescale_single": lambda: [ckks.rescale(c, params) for c in cts],
            "rescale_batch": lambda: ckks.rescale(B, params),
        }
        for name, fn in cases.items():
            ms = timed(fn)
            print(json.dumps({"case": name, "level": level, "nb": nb, "ks_batch": ks_batch, "ms_total": round(ms, 3),
                              "ms_per_ct": round(ms / nb, 4), "kernels": profile(fn)}), flush=True)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
