"""BASELINE config 4 breakdown: encrypted AESPA-ResNet20 (workloads.resnet20_setup).

    python tools/resnet20.py [images] [use_graph]

Prints one JSON line: s/image (captured replay), logits error vs the
plaintext mirror, a device-synchronised per-layer-kind breakdown (refresh =
bootstrapping rows) and per-kernel device time of one eager image."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HCNN_TEST_MODE", "1")
import numpy as np
import torch

from paper_2310_16530_b200 import _native, graph, packing, workloads


def main(images: int = 2, use_graph: int = 1):
    t0 = time.time()
    s = workloads.resnet20_setup()
    torch.cuda.synchronize()
    t_setup = time.time() - t0
    rng = np.random.default_rng(0xC1FA)
    xs = [rng.uniform(-1.0, 1.0, (3, 32, 32)) for _ in range(images)]
    cts = [workloads.encrypt_image(s, x, rng) for x in xs]
    cache: dict = {}
    warm = workloads.warm_up(s, cts[0], cache)
    t_first = warm["first_image_s"]
    # device-synchronised layer breakdown (eager)
    _, rep = graph.execute(s.graph, s.plan, cts[0], s.ks, "encrypted", cache=cache, sync_timing=True)
    kinds: dict = {}
    for row in rep.per_layer:
        kinds[row["kind"]] = kinds.get(row["kind"], 0.0) + row["ms"]
    per_refresh = [r["ms"] / max(1, r["tally"]["refreshes"]) for r in rep.per_layer if r["kind"] == "refresh"]
    # per-kernel device time of one eager image
    _native.profile_read(reset=True)
    _native.profile_enable(True)
    graph.execute(s.graph, s.plan, cts[0], s.ks, "encrypted", cache=cache)
    torch.cuda.synchronize()
    _native.profile_enable(False)
    prof = _native.profile_read(reset=True)
    dev_ms = sum(v["ms"] for v in prof.values())
    kern = {k: {"ms": round(v["ms"], 1), "share": round(v["ms"] / dev_ms, 3), "launches": v["launches"]}
            for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}
    runner = graph.CapturedInference(s.graph, s.plan, s.ks, cts[0], cache, warmup=False) if use_graph else None
    errs, agree, times = [], 0, []
    for x, ct in zip(xs, cts):
        torch.cuda.synchronize()
        t0 = time.time()
        o = runner.run(ct) if runner else graph.execute(s.graph, s.plan, ct, s.ks, "encrypted", cache=cache)[0]
        logits = packing.read_logits(o, s.graph.n_classes, s.graph.formats[-1], s.ks)
        torch.cuda.synchronize()
        times.append(time.time() - t0)
        ref, _ = graph.execute(s.graph, s.plan, x, mode="plaintext-ref")
        errs.append(float(np.max(np.abs(logits - ref))))
        agree += int(np.argmax(logits) == np.argmax(ref))
    print(json.dumps({
        "config": "resnet20-cifar10 AESPA+HyPHEN, N=2^16, multiplex 4, bootstrapping",
        "q_limbs": len(s.params.q_mods), "special_limbs": len(s.params.p_mods),
        "refresh_points": list(s.plan.refresh_points), "rotation_keys": len(s.ks.gks),
        "setup_s": round(t_setup, 1), "first_image_s": round(t_first, 2), "cuda_graph": bool(use_graph),
        "s_per_image": round(float(np.median(times)), 3), "images": images,
        "max_logit_err_vs_plain": max(errs), "argmax_agree": f"{agree}/{images}",
        "tally": rep.totals().as_dict(), "layer_ms_by_kind_synced": {k: round(v, 1) for k, v in kinds.items()},
        "ms_per_bootstrap_by_point": [round(v, 2) for v in per_refresh],
        "layer_rows": [(r["name"], r["ms"]) for r in rep.per_layer],
        "mask_cache_entries": len(cache), "device_ms_profiled_image": round(dev_ms, 1), "kernels": kern,
        "resident_mask_gb": round(packing.resident_bytes() / 2 ** 30, 1), "warm_up": warm,
        "gpu_mem_gb": round(torch.cuda.max_memory_allocated() / 2 ** 30, 1)}), flush=True)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
