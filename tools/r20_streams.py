"""Throughput of K ResNet20 inferences replayed concurrently (K captured
CUDA graphs on K streams) vs one at a time.

    python tools/r20_streams.py [K] [reps]"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HCNN_TEST_MODE", "1")
import numpy as np
import torch

from paper_2310_16530_b200 import graph, packing, workloads


def main(K: int = 2, reps: int = 4):
    s = workloads.resnet20_setup()
    rng = np.random.default_rng(1)
    raw = [rng.uniform(-1, 1, (3, 32, 32)) for _ in range(K)]
    cts = [workloads.encrypt_image(s, x, rng) for x in raw]
    cache: dict = {}
    graph.execute(s.graph, s.plan, cts[0], s.ks, "encrypted", cache=cache)
    torch.cuda.synchronize()
    runners = [graph.CapturedInference(s.graph, s.plan, s.ks, cts[0], cache, warmup=False) for _ in range(K)]
    streams = [torch.cuda.Stream() for _ in range(K)]
    for r, c in zip(runners, cts):
        r.run(c)
    torch.cuda.synchronize()

    def timed(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    seq = timed(lambda: [r.cuda_graph.replay() for r in runners])
    cur = torch.cuda.current_stream()

    def conc():
        for r, st in zip(runners, streams):
            st.wait_stream(cur)
            with torch.cuda.stream(st):
                r.cuda_graph.replay()
        for st in streams:
            cur.wait_stream(st)

    par = timed(conc)
    errs = []
    for r, c, x in zip(runners, cts, raw):
        lg = packing.read_logits(r.out, s.graph.n_classes, s.graph.formats[-1], s.ks)
        ref, _ = graph.execute(s.graph, s.plan, x, mode="plaintext-ref")
        errs.append(float(np.max(np.abs(lg - ref))))
    print(json.dumps({"K": K, "sequential_ms_per_image": round(seq / K, 2), "concurrent_ms_per_image": round(par / K, 2),
                      "speedup": round(seq / par, 3), "max_logit_err": max(errs),
                      "resident_mask_gb": round(packing.resident_bytes() / 2 ** 30, 1),
                      "gpu_mem_gb": round(torch.cuda.max_memory_allocated() / 2 ** 30, 1)}), flush=True)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
