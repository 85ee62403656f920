"""Launch the NTT butterfly probes once each (ncu target: k_bfly_peak*)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2310_16530_b200 import _native
torch.zeros(1).cuda()
for f in (4, 2, 0):
    print(f, _native.ntt_butterfly_peak(f) / 1e9)
