"""A/B of NTT launch options at N=2^16 on the BASELINE cfg 2 chain: each
argument is "opt=v,opt=v"; prints device ms per forward / inverse NTT of a
[7][29] batch (the ModUp shape, 25 q + 4 special limbs) and asserts every
setting returns the residues of the first."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HCNN_TEST_MODE", "1")
import numpy as np
import torch

from paper_2310_16530_b200 import _native, ckks


def timed(fn, reps=30):
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
    rng = np.random.default_rng(0)
    mods = [m.q for m in params.q_mods] + [m.q for m in params.p_mods]
    host = np.stack([np.stack([rng.integers(0, q, params.n, dtype=np.uint64) for q in mods]) for _ in range(7)])
    src = torch.from_numpy(host.view(np.int64)).to(ctx.torch_device)
    settings = sys.argv[1:] or ["ntt_f64_minb=1"]
    ref = None
    for s in settings:
        for item in s.split(","):
            k, _, v = item.partition("=")
            _native.set_option(k, int(v))
        t = src.clone()
        ctx.ntt(t, 25, 4)
        f = t.clone()
        ctx.ntt(t, 25, 4, inverse=True)
        if ref is None:
            ref = f
        ok = torch.equal(f, ref) and torch.equal(t, src)
        w = src.clone()
        tf = timed(lambda: ctx.ntt(w, 25, 4))
        ti = timed(lambda: ctx.ntt(w, 25, 4, inverse=True))
        print(json.dumps({"setting": s, "fwd_ms": round(tf, 4), "inv_ms": round(ti, 4),
                          "fwd_us_per_limb": round(tf * 1e3 / 203, 3), "inv_us_per_limb": round(ti * 1e3 / 203, 3),
                          "bit_identical": ok}), flush=True)
        assert ok


if __name__ == "__main__":
    main()
