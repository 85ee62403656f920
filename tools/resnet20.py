"""BASELINE config 4: encrypted AESPA-ResNet20 on a CIFAR-10-shaped input,
HyPHEN packing (multiplex 4, N=2^16, 32768 slots) with real CKKS
bootstrapping at the refresh points.  Synthetic seeded weights
(graph.gen_fixture("resnet20", ...)) and a U(-1,1) 3x32x32 input.

Prints one JSON line: s/image (warm: masks and keys resident, the first
image builds the mask set), logits error vs the plaintext mirror, argmax,
bootstrap count, per-kind layer time."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HCNN_TEST_MODE", "1")
import numpy as np
import torch

from paper_2310_16530_b200 import _native, bootstrap as bt, graph, packing


def build(app_levels: int = 14, seed: int = 3, key_seed: int = 20):
    cfg = bt.BootConfig()
    params = bt.boot_params("resnet20-16", 1 << 16, app_levels, cfg)
    b = bt.Bootstrapper(params, cfg)
    fx = graph.gen_fixture("resnet20", seed, params, golden_count=2)
    g = graph.build_graph("resnet20", fx, multiplex=4)
    plan = graph.plan_levels(g, b.output_level, refresh_target=b.output_level, count_snapshots=True)
    steps = sorted(graph.required_rotation_steps(g, params.slots))
    ks = b.keygen(np.random.default_rng(key_seed), rotations=steps)
    return params, cfg, b, fx, g, plan, ks


def infer(g, plan, ks, x, cache, rng):
    packed = packing.encrypt_tensor(x, g.input_format, ks, rng, plan.entry_levels[0])
    out, rep = graph.execute(g, plan, packed, ks, "encrypted", cache=cache)
    logits = packing.read_logits(out, g.n_classes, g.formats[-1], ks)
    return logits, rep


def main(images: int = 2, app_levels: int = 14, use_graph: int = 1):
    packing.set_mask_mode("compact")
    t0 = time.time()
    params, cfg, b, fx, g, plan, ks = build(app_levels)
    torch.cuda.synchronize()
    t_setup = time.time() - t0
    cache: dict = {}
    rng = np.random.default_rng(0xC1FA)
    x0 = np.asarray(fx["golden"][0]["input"])
    t0 = time.time()
    logits0, rep0 = infer(g, plan, ks, x0, cache, rng)
    torch.cuda.synchronize()
    t_first = time.time() - t0
    runner = None
    t_capture = None
    if use_graph:
        t0 = time.time()
        example = packing.encrypt_tensor(x0, g.input_format, ks, rng, plan.entry_levels[0])
        runner = graph.CapturedInference(g, plan, ks, example, cache)
        t_capture = time.time() - t0
        eager_out, _ = graph.execute(g, plan, example, ks, "encrypted", cache=cache)
        replay_out = runner.run(example)
        assert torch.equal(eager_out.data, replay_out.data), "graph replay differs from eager execution"
    errs, agree, times = [], 0, []
    kinds: dict = {}
    refreshes = 0
    for k in range(images):
        x = rng.uniform(-1.0, 1.0, (3, 32, 32))
        torch.cuda.synchronize()
        t0 = time.time()
        if runner is not None:
            packed = packing.encrypt_tensor(x, g.input_format, ks, rng, plan.entry_levels[0])
            out = runner.run(packed)
            logits = packing.read_logits(out, g.n_classes, g.formats[-1], ks)
            rep = runner.report
        else:
            logits, rep = infer(g, plan, ks, x, cache, rng)
        torch.cuda.synchronize()
        times.append(time.time() - t0)
        ref, _ = graph.execute(g, plan, x, mode="plaintext-ref")
        errs.append(float(np.max(np.abs(logits - ref))))
        agree += int(np.argmax(logits) == np.argmax(ref))
        refreshes = rep.totals().refreshes
        for row in rep.per_layer:
            kinds[row["kind"]] = kinds.get(row["kind"], 0.0) + row["ms"] / images
    tot = rep.totals().as_dict()
    # per-kernel device time of one more warm image
    _native.profile_read(reset=True)
    _native.profile_enable(True)
    infer(g, plan, ks, x0, cache, rng)
    torch.cuda.synchronize()
    _native.profile_enable(False)
    prof = _native.profile_read(reset=True)
    dev_ms = sum(v["ms"] for v in prof.values())
    kern = {k: {"ms": round(v["ms"], 1), "share": round(v["ms"] / dev_ms, 3), "launches": v["launches"]}
            for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}
    print(json.dumps({
        "config": "resnet20-cifar10 AESPA+HyPHEN, N=2^16, multiplex 4, bootstrapping",
        "q_limbs": len(params.q_mods), "special_limbs": len(params.p_mods), "app_levels": app_levels,
        "refresh_points": list(plan.refresh_points), "bootstraps_per_image": refreshes,
        "rotation_keys": len(ks.gks), "setup_s": round(t_setup, 1), "first_image_s": round(t_first, 2),
        "cuda_graph": bool(use_graph), "capture_s": None if t_capture is None else round(t_capture, 1),
        "s_per_image": round(float(np.median(times)), 3), "images": images,
        "max_logit_err_vs_plain": max(errs), "argmax_agree": f"{agree}/{images}",
        "tally": tot, "layer_ms_by_kind": {k: round(v, 1) for k, v in kinds.items()},
        "mask_cache_entries": len(cache), "device_ms_profiled_image": round(dev_ms, 1), "kernels": kern,
        "gpu_mem_gb": round(torch.cuda.max_memory_allocated() / 2 ** 30, 1)}), flush=True)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
