"""Large-batch NTT launches for ncu (203 limbs fwd + inv at N=2^16)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2310_16530_b200 import ckks
params = ckks.bench16()
ctx = params.ctx
t = ctx.zeros(7, 29, params.n)
for _ in range(3):
    ctx.ntt(t, 25, 4)
    ctx.ntt(t, 25, 4, inverse=True)
torch.cuda.synchronize()
print("ok")
