"""Where one eager ResNet20 image spends its device time: bootstrapping
(Bootstrapper.bootstrap calls, bracketed by CUDA events) vs the rest."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HCNN_TEST_MODE", "1")
import numpy as np
import torch

from paper_2310_16530_b200 import bootstrap as bt, graph, workloads


def main():
    s = workloads.resnet20_setup()
    rng = np.random.default_rng(1)
    ct = workloads.encrypt_image(s, rng.uniform(-1, 1, (3, 32, 32)), rng)
    cache: dict = {}
    graph.execute(s.graph, s.plan, ct, s.ks, "encrypted", cache=cache)  # warm (masks, tables)
    torch.cuda.synchronize()
    marks = []
    orig = bt.Bootstrapper.bootstrap

    def timed(self, x, ks, out_scale=None):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = orig(self, x, ks, out_scale)
        e1.record()
        marks.append((x.batch or 1, x.level, e0, e1))
        return out

    bt.Bootstrapper.bootstrap = timed
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    graph.execute(s.graph, s.plan, ct, s.ks, "encrypted", cache=cache)
    b.record()
    torch.cuda.synchronize()
    total = a.elapsed_time(b)
    boot = sum(e0.elapsed_time(e1) for _, _, e0, e1 in marks)
    print(f"image {total:.1f} ms (eager), bootstrapping {boot:.1f} ms in {len(marks)} calls:",
          [(nb, lvl, round(e0.elapsed_time(e1), 1)) for nb, lvl, e0, e1 in marks])


if __name__ == "__main__":
    main()
