"""NTT / key-switch microbenchmark over the engine's tuning knobs (N=2^16,
BASELINE config 2 chain).  Prints one JSON line per setting."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HCNN_TEST_MODE", "1")
import numpy as np
import torch

from paper_2310_16530_b200 import _native, ckks


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    params = ckks.bench16()
    ctx = params.ctx
    ks = ckks.keygen(params, np.random.default_rng(1), rotations=[1])
    rng = np.random.default_rng(5)
    L = params.max_level
    a = ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, L), ks, rng)
    b = ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, L), ks, rng)
    big = ctx.zeros(7, 29, params.n)
    small = ctx.zeros(2, 29, params.n)
    settings = [(0, 1, 0), (0, 1, 1), (0, 0, 1)]
    if len(sys.argv) > 1:
        settings = [tuple(int(v) for v in s.split(",")) for s in sys.argv[1:]]
    for group, hints, occ, split in [tuple(s) + (0,) * (4 - len(s)) for s in settings]:
        _native.set_option("ntt_group_limbs", group)
        _native.set_option("ntt_hints", hints)
        _native.set_option("ntt_occupancy", occ)
        _native.set_option("ntt_split", split)
        res = {"group_limbs": group, "hints": hints, "occupancy": occ, "split": split}
        for name, t, nq, np_ in (("203limbs", big, 25, 4), ("58limbs", small, 25, 4)):
            f = timed(lambda: ctx.ntt(t, nq, np_))
            i = timed(lambda: ctx.ntt(t, nq, np_, inverse=True))
            limbs = t.numel() // params.n
            res[name] = {"fwd_us_per_limb": round(f * 1e3 / limbs, 3), "inv_us_per_limb": round(i * 1e3 / limbs, 3)}
        res["hmult_ms"] = round(timed(lambda: ckks.hmult(a, b, ks)), 4)
        res["rotate_ms"] = round(timed(lambda: ckks.rotate(a, 1, ks)), 4)
        res["rescale_ms"] = round(timed(lambda: ckks.rescale(a, params)), 4)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
