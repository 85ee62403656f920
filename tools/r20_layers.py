"""Per-layer device time of one ResNet20 image (eager, masks resident,
sync_timing: the device is synchronised around every layer and refresh)."""
import json
import os
import sys
from collections import defaultdict
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
    cache: dict = {}
    workloads.warm_up(s, ct, cache)
    graph.execute(s.graph, s.plan, ct, s.ks, "encrypted", cache=cache)
    torch.cuda.synchronize()
    _, rep = graph.execute(s.graph, s.plan, ct, s.ks, "encrypted", cache=cache, sync_timing=True)
    by = defaultdict(float)
    for r in rep.per_layer:
        by[r["kind"]] += r["ms"]
    tot = sum(by.values())
    print(json.dumps({"total_ms": round(tot, 1), "by_kind_ms": {k: round(v, 1) for k, v in by.items()},
                      "layers": [(r["name"], r["kind"], r["entry_level"], r["ms"]) for r in rep.per_layer]}))


if __name__ == "__main__":
    main()
