"""Key-switch inner-product variants on the ResNet20 bootstrapping chain
(N=2^16, 31 q-limbs + 4 special): hoisted rotation batches (conv tap
pattern), a batched hmult and a high-level rotation batch (bootstrapping),
for each `ks_pipe` setting.  Prints per-kernel device time and the
ks_inner algorithmic GB/s; asserts every setting is bit-identical with
ks_pipe=0 (the reference-order kernel)."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HCNN_TEST_MODE", "1")
import numpy as np
import torch

from paper_2310_16530_b200 import _native, bootstrap as bt, ckks


def profile(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    _native.profile_read(reset=True)
    _native.profile_enable(True)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    _native.profile_enable(False)
    return {k: {"ms": v["ms"] / reps, "GBps": v["bytes"] / (v["ms"] / 1e3) / 1e9}
            for k, v in _native.profile_read(reset=True).items()}


def main():
    # each argument: comma-separated engine options, e.g. "ks_tma=0,ks_pipe=0"
    settings = sys.argv[1:] or ["ks_tma=0,ks_pipe=0", "ks_tma=0,ks_pipe=2", "ks_tma=1"]
    cfg = bt.BootConfig()
    params = bt.boot_params("resnet20-16", 1 << 16, 14, cfg)
    steps = [1, 2, 3, 4, 5, 6, 7, 8]
    ks = ckks.keygen(params, np.random.default_rng(1), rotations=steps)
    rng = np.random.default_rng(2)
    ctx = params.ctx
    keys = [(ks.gks[k].rows_b, ks.gks[k].rows_a) for k in steps]
    gal = [ckks.galois_element(k, params.n) for k in steps]
    cases = {}
    for level, nb in ((14, 4), (14, 1), (params.max_level, 8)):
        cts = [ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, level), ks, rng) for _ in range(nb)]
        B = ckks.stack(cts) if nb > 1 else cts[0]
        cases[f"rot8_l{level}_nb{nb}"] = (lambda B=B, level=level: ctx.rotate_hoisted(B.data, level, gal, keys))
        cases[f"hmult_l{level}_nb{nb}"] = (lambda B=B: [ckks.hmult(B, B, ks).data])
    ref = {}
    for pipe in settings:
        for item in pipe.split(","):
            key, _, val = item.partition("=")
            _native.set_option(key, int(val))
        for name, fn in cases.items():
            outs = fn()
            torch.cuda.synchronize()
            if pipe == settings[0]:
                ref[name] = [o.clone() for o in outs]
            same = all(torch.equal(a, b) for a, b in zip(ref[name], outs))
            p = profile(fn)
            ki = p.get("ks_inner", {"ms": 0, "GBps": 0})
            print(json.dumps({"options": pipe, "case": name, "bit_identical": same,
                              "total_ms": round(sum(v["ms"] for v in p.values()), 3),
                              "ks_inner_ms": round(ki["ms"], 3), "ks_inner_GBps": round(ki["GBps"], 1)}), flush=True)
            assert same, f"{pipe} changed {name}"


if __name__ == "__main__":
    main()
