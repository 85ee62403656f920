"""One eager encrypted ResNet20 image (workloads.resnet20_setup) -- a
target for ncu kernel captures (-k regex:<kernel> -s <skip> -c <count>)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HCNN_TEST_MODE", "1")
import numpy as np
import torch

from paper_2310_16530_b200 import graph, workloads


def main():
    s = workloads.resnet20_setup()
    rng = np.random.default_rng(1)
    ct = workloads.encrypt_image(s, rng.uniform(-1, 1, (3, 32, 32)), rng)
    graph.execute(s.graph, s.plan, ct, s.ks, "encrypted", cache={})
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
