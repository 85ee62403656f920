"""Short N=2^16 workload for ncu captures: keygen, then R rounds of
hmult+rescale and rotate(1) on one ciphertext pair (bench.py's step shape)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HCNN_TEST_MODE", "1")
import numpy as np
import torch

from paper_2310_16530_b200 import ckks

R = int(sys.argv[1]) if len(sys.argv) > 1 else 3
params = ckks.bench16()
ks = ckks.keygen(params, np.random.default_rng(1), rotations=[1])
rng = np.random.default_rng(5)
L = params.max_level
a = ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, L), ks, rng)
b = ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, L), ks, rng)
for _ in range(R):
    ckks.rescale(ckks.hmult(a, b, ks), params)
    ckks.rotate(a, 1, ks)
torch.cuda.synchronize()
print("prof_step done")
