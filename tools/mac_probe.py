"""Plane-MAC probe for ncu: k_mac_multi_tma2 at a ResNet20 conv shape
(N=2^16, ResNet20 chain, level 10, 36 terms = 9 taps x 4 input
ciphertexts, 4 outputs per launch, packed resident masks), 6 launches in
an NVTX range "probe" after 2 warm-up launches."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HCNN_TEST_MODE", "1")
import numpy as np
import torch

from paper_2310_16530_b200 import bootstrap as bt


def main(level: int = 10, T: int = 36, G: int = 4, settings=("mac_tma=3",)):
    from paper_2310_16530_b200 import _native
    cfg = bt.BootConfig()
    params = bt.boot_params("resnet20-16", 1 << 16, 14, cfg)
    ctx = params.ctx
    rng = np.random.default_rng(0)
    qs = [m.q for m in params.q_mods[: level + 1]]

    def rows(k):
        return torch.from_numpy(np.stack([np.stack([rng.integers(0, q, params.n, dtype=np.uint64) for q in qs])
                                          for _ in range(k)]).view(np.int64)).to(ctx.torch_device)

    images = int(os.environ.get("MAC_PROBE_IMAGES", "1"))
    cts = [rows(2) for _ in range(T)] if images == 1 else \
        [torch.stack([rows(2) for _ in range(images)]).contiguous() for _ in range(T)]
    packed = os.environ.get("MAC_PROBE_UNPACKED") is None
    masks = [[ctx.pack_masks(rows(1), level)[0] if packed else rows(1)[0] for _ in range(T)] for _ in range(G)]
    ref = None
    for st in settings:
        for item in st.split(","):
            k, _, v = item.partition("=")
            _native.set_option(k, int(v))
        for _ in range(2):
            outs = ctx.mac_terms_multi(cts, masks, level)
        torch.cuda.synchronize()
        same = True
        if ref is None:
            ref = [o.clone() for o in outs]
        else:
            same = all(torch.equal(a, b) for a, b in zip(ref, outs))
        torch.cuda.nvtx.range_push("probe")
        runs = []
        for rep in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10 if rep else 2):
                ctx.mac_terms_multi(cts, masks, level)
            e1.record()
            torch.cuda.synchronize()
            if rep:
                runs.append(e0.elapsed_time(e1) / 10)
        torch.cuda.nvtx.range_pop()
        ms = sorted(runs)[len(runs) // 2]
        lb = params.n * 8
        mb = ctx.packed_mask_bytes(level) if packed else (level + 1) * lb
        alg = (2 * T * images * (level + 1) * lb + G * T * mb + 2 * G * images * (level + 1) * lb)
        print(f"{st} images={images} mac_multi T={T} G={G} level={level}: {ms:.4f} ms, {alg / ms / 1e6:.1f} GB/s algorithmic (median of {len(runs)}, "
              f"min {min(runs):.4f}), bit_identical={same}", flush=True)
        assert same


if __name__ == "__main__":
    nums = [int(a) for a in sys.argv[1:] if "=" not in a]
    sets = [a for a in sys.argv[1:] if "=" in a] or ["mac_tma=3"]
    main(*nums, settings=sets)
