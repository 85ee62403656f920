"""Steady-state key-switch traffic probe for ncu (--cache-control none):
BASELINE cfg 2 chain (N=2^16, 25 q-limbs, K=4), a batch of 4 ciphertexts at
the top level: hmult + rescale + a hoisted rotation group of 4 steps per
iteration, 8 iterations (the first 2 warm the tables).  Run plain first;
ncu then reads per-launch DRAM bytes of every kernel of iterations 3..8."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HCNN_TEST_MODE", "1")
import numpy as np
import torch

from paper_2310_16530_b200 import _native, ckks, workloads


def main(iters: int = 8, nb: int = 4):
    params = workloads.cfg2_params()
    steps = [1, 2, 3, 4]
    ks = ckks.keygen(params, np.random.default_rng(1), rotations=steps)
    rng = np.random.default_rng(2)
    L = params.max_level
    B = ckks.stack([ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, L), ks, rng)
                    for _ in range(nb)])
    torch.cuda.synchronize()
    k0 = _native.kernel_launches()
    for it in range(iters):
        if it == 2:
            torch.cuda.synchronize()
            torch.cuda.nvtx.range_push("probe")
        ckks.rescale(ckks.hmult(B, B, ks), params)
        ckks.rotate_many(B, steps, ks)
        if it == 0:
            torch.cuda.synchronize()
            print("launches per iteration", _native.kernel_launches() - k0, flush=True)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print("ok", flush=True)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
