"""Benchmark driver (graft contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload resnet20|cfg2] [--impl ours|reference]

Default workload = the BASELINE.json metric: encrypted AESPA-ResNet20 on a
CIFAR-10-shaped (3x32x32) synthetic input, HyPHEN packing (multiplex 4,
N=2^16), real CKKS bootstrapping at the planner's refresh points
(workloads.resnet20_setup).  One step = one encrypted image through the
captured inference (graph.CapturedInference: the whole executor, ~10^5
kernels with 32 bootstraps, replayed as one CUDA graph).  Random-init
weights of the architecture (seeded), synthetic images.  Encrypted
inputs/keys/masks exceed the 126 MB L2 by orders of magnitude (no flush).

`value` = whole-job images/s with encrypted inputs resident in HBM;
`ms_per_step` = s/image x 1e3.  `e2e` = the same through the public API with
the encrypted input copied from pinned host memory and the encrypted logits
copied back each step.  `roofline` = the kernel with the largest device-time
share in an event-profiled eager run of one image.  `cpu_baseline` = the
C/numpy oracle (tests' checker; the Python reference cannot travel to the
GPU box) timed per primitive on the host cores and extrapolated over this
image's op tally (bootstraps excluded: the reference has none).

`--workload cfg2` runs BASELINE config 2 instead: HMult+relin, rescale and
HRot(1) on batches of ciphertext pairs at N=2^16, L=24.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("HCNN_TEST_MODE", "1")
# before any CUDA allocation (see paper_2310_16530_b200/__init__.py)
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

PAPER_A100_MS = 1402.0  # ResNet20 AESPA+HyPHEN on A100


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout: float = 5.0) -> None:
        """block until nvidia-smi has produced a sample (its start-up takes
        longer than a short timed region)"""
        t0 = time.time()
        while self.proc is not None and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.05)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


class Dist:
    """torchrun plumbing: barrier and MAX over ranks (identity on 1 GPU)."""

    def __init__(self):
        import torch
        self.torch = torch
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local)
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{self.local}"))
            self.dist = dist

    def barrier(self):
        self.torch.cuda.synchronize()
        if self.dist is not None:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def max(self, v: float) -> float:
        if self.dist is None:
            return v
        t = self.torch.tensor([v], device="cuda", dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.dist is not None:
            self.dist.destroy_process_group()


def timed_steps(d: Dist, fn, steps: int, nvtx: str | None = None) -> float:
    """device ms over `steps` calls of fn, CUDA events on the current stream,
    MAX over ranks.  nvtx: name of an NVTX range around the timed region (ncu
    --nvtx --nvtx-include "<name>/" captures exactly these launches)."""
    torch = d.torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d.barrier()
    if nvtx:
        torch.cuda.nvtx.range_push(nvtx)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    if nvtx:
        torch.cuda.nvtx.range_pop()
    d.barrier()
    return d.max(e0.elapsed_time(e1))


def _kernel_family(label: str) -> str:
    """profile labels carry the call site (ntt_fwd_modup, ntt_fwd_rescale ...);
    the roofline is per kernel, so sites of one kernel are merged"""
    for fam in ("ntt_fwd", "ntt_inv"):
        if label.startswith(fam):
            return fam
    return label


def roofline_from_profile(prof: dict) -> tuple[dict, dict]:
    peak, kind = _peaks()
    total = sum(v["ms"] for v in prof.values()) or 1.0
    fam: dict = {}
    for k, v in prof.items():
        f = fam.setdefault(_kernel_family(k), {"ms": 0.0, "bytes": 0.0, "launches": 0})
        f["ms"] += v["ms"]
        f["bytes"] += v["bytes"]
        f["launches"] += v["launches"]
    kernels = {}
    for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
        gbs = v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] > 0 else 0.0
        kernels[k] = {"share": round(v["ms"] / total, 4), "ms_per_launch": round(v["ms"] / v["launches"], 5),
                      "GBps": round(gbs, 1), "launches": v["launches"]}
    name, tv = max(fam.items(), key=lambda kv: kv[1]["ms"])
    achieved = tv["bytes"] / (tv["ms"] / 1e3) / 1e9
    roof = {"kernel": name, "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_kind_note(kind),
            "algorithmic_bytes_per_launch": tv["bytes"] / tv["launches"], "share_of_device_time": round(tv["ms"] / total, 4),
            "note": "the 64-bit NTT is integer-pipe bound (SURVEY 8d); HBM fraction reported per contract, "
                    "ncu issue/pipe utilisation in profiles/"}
    return roof, kernels


def int_roofline(roof: dict, prof: dict, limbs: dict, n: int) -> dict:
    """The NTT family is integer-pipe bound: its roofline is the
    butterfly rate of the same radix-16 register network with no memory
    traffic (hcnn_ntt_butterfly_peak, measured here on this GPU, per modulus
    class).  ideal = sum over limbs of N/2 log2 N / peak(class); frac =
    ideal / measured device time of the family.  The HBM view is kept under
    "hbm"."""
    from paper_2310_16530_b200 import _native
    fam = roof["kernel"]
    if fam not in ("ntt_fwd", "ntt_inv"):
        return roof
    d = "fwd" if fam == "ntt_fwd" else "inv"
    fast, full = limbs[f"{d}_fast"], limbs[f"{d}_full"]
    ms = sum(v["ms"] for k, v in prof.items() if _kernel_family(k) == fam)
    if fast + full == 0 or ms <= 0:
        return roof
    # fast limbs (q < 2^44 here) run the FP64-quotient network: its probe is their ceiling
    pf, ps = _native.ntt_butterfly_peak(2), _native.ntt_butterfly_peak(0)
    per_limb = n // 2 * (n.bit_length() - 1)
    ideal_s = per_limb * (fast / pf + full / ps)
    bfly = per_limb * (fast + full)
    achieved = bfly / (ms / 1e3)
    peak = bfly / ideal_s
    hbm = {k: roof[k] for k in ("achieved", "peak", "unit", "frac", "peak_source", "algorithmic_bytes_per_launch")}
    # DRAM traffic per launch from the committed ncu --set full capture, scaled per limb
    traffic = roof.get("traffic")
    tf = ROOT / "profiles" / "r01_ncu_ntt_traffic.json"
    if traffic is None and fam == "ntt_fwd" and tf.exists():
        per_limb = json.loads(tf.read_text())["dram_bytes_per_limb"]
        launches = sum(v["launches"] for k, v in prof.items() if _kernel_family(k) == fam)
        traffic = round(per_limb * (fast + full) / max(launches, 1))
        hbm["traffic_source"] = ("profiles/r01_ncu_ntt_traffic.json (ncu, cold L2) x mean limbs per launch "
                                 "(one launch = the cols + chunks pass pair)")
    out = {"kernel": fam, "bound": "int", "achieved": round(achieved / 1e9, 2), "peak": round(peak / 1e9, 2),
           "unit": "Gbutterfly/s", "frac": round(ideal_s / (ms / 1e3), 4), "traffic": traffic,
           "peak_source": (f"measured on this GPU: radix-16 register network without memory traffic "
                           f"(hcnn_ntt_butterfly_peak) {pf/1e9:.1f} Gbfly/s for the FP64-quotient network of "
                           f"q<2^44 limbs, {ps/1e9:.1f} for full-width limbs, weighted by this image's {fast} + {full} limbs"),
           "limbs": {"fast": fast, "full": full}, "share_of_device_time": roof["share_of_device_time"],
           "hbm": hbm}
    return out


def peak_kind_note(kind: str) -> str:
    return f"{kind} (MEASURED_PEAKS.json hbm_gbs)" if kind == "measured" else "fallback 6650 GB/s"


# ---------------------------------------------------------------------------
# CPU oracle (test infrastructure): per-primitive timings, extrapolated
# ---------------------------------------------------------------------------

class OracleSampler:
    """Per-primitive host timings of the C/numpy oracle at one level (keys
    generated once; every sample re-times the five primitives)."""

    def __init__(self, qs, ps, n, level, delta):
        from oracle import ckks_oracle as O
        self.O, self.level = O, level
        self.P = O.OParams(n, list(qs), list(ps), float(delta))
        self.K = O.keygen(self.P, np.random.default_rng(1), rotations=[1])
        rng = np.random.default_rng(5)
        a, sc = O.encode(rng.uniform(-1, 1, self.P.slots), self.P, level)
        b, _ = O.encode(rng.uniform(-1, 1, self.P.slots), self.P, level)
        self.ca, self.cb = O.encrypt(a, sc, self.K, rng)[0], O.encrypt(b, sc, self.K, rng)[0]
        self.mask = a
        self.cores = int(O.lib().o_num_threads())

    def sample(self) -> dict:
        O, ca, cb, mods = self.O, self.ca, self.cb, self.P.qs[: self.level + 1]
        ops = {
            "rotate": lambda: O.rotate(ca, 1, self.K),
            "hmult": lambda: O.hmult(ca, cb, self.K),
            "rescale": lambda: O.rescale(ca, self.P),
            "pmult": lambda: O.pmult(ca, self.mask, mods),
            "hadd": lambda: np.stack([O.add(ca[0], cb[0], mods), O.add(ca[1], cb[1], mods)]),
        }
        out = {}
        for name, fn in ops.items():
            t0 = time.perf_counter()
            fn()
            out[name] = time.perf_counter() - t0
        return out


def extrapolate(op_s: dict, tally: dict) -> float:
    return (tally["rotations"] * op_s["rotate"] + tally["hmults"] * op_s["hmult"]
            + tally["rescales"] * op_s["rescale"] + tally["pmults"] * op_s["pmult"]
            + tally["hadds"] * op_s["hadd"])


def resnet_cpu_baseline(sampler: OracleSampler, tally: dict, samples: int = 1) -> dict:
    runs = [sampler.sample() for _ in range(samples)]
    op_s = {k: statistics.median(r[k] for r in runs) for k in runs[0]}
    s_img = extrapolate(op_s, tally)
    return {"value": 1.0 / s_img, "unit": "images/s", "cores": sampler.cores, "kind": "port",
            "sample": f"extrapolated: C/numpy oracle primitive times at level {sampler.level} "
                      f"(rotate {op_s['rotate']:.3f}s, hmult {op_s['hmult']:.3f}s, rescale {op_s['rescale']:.3f}s, "
                      f"pmult {op_s['pmult']*1e3:.1f}ms, hadd {op_s['hadd']*1e3:.1f}ms; median of {samples}) "
                      f"x the image's op tally {tally}; bootstraps excluded (the reference has none)",
            "s_per_image_extrapolated": s_img}


def _oracle_for(params, level):
    return OracleSampler([m.q for m in params.q_mods], [m.q for m in params.p_mods], params.n, level,
                         params.delta)


# ---------------------------------------------------------------------------
# ResNet20 (default)
# ---------------------------------------------------------------------------

def _median_conv_level_of(g, plan) -> int:
    lv = sorted(plan.entry_levels[i] for i, l in enumerate(g.layers) if l.kind == "conv")
    return int(lv[len(lv) // 2])


def _median_conv_level(s) -> int:
    return _median_conv_level_of(s.graph, s.plan)


def run_resnet20(args, d: Dist):
    import torch
    from paper_2310_16530_b200 import _native, graph, packing, workloads

    s = workloads.resnet20_setup()
    rng = np.random.default_rng(100 + d.rank)
    raw = [rng.uniform(-1.0, 1.0, (3, 32, 32)) for _ in range(3)]
    imgs = [workloads.encrypt_image(s, x, rng) for x in raw]
    cache: dict = {}
    # eager runs first (mask build, measured residency fill, lazy tables;
    # then one event-profiled image for the kernel table / roofline / launch
    # count), then capture -- so the capture pool reuses the eager memory
    warm = workloads.warm_up(s, imgs[0], cache)
    k0 = _native.kernel_launches()
    _native.profile_read(reset=True)
    _native.ntt_limb_counts(reset=True)
    _native.profile_enable(True)
    graph.execute(s.graph, s.plan, imgs[1], s.ks, "encrypted", cache=cache)
    torch.cuda.synchronize()
    _native.profile_enable(False)
    prof = _native.profile_read(reset=True)
    limbs = _native.ntt_limb_counts(reset=True)
    launches = _native.kernel_launches() - k0
    roofline, kernels = roofline_from_profile(prof)
    roofline = int_roofline(roofline, prof, limbs, s.params.n)
    runner = graph.CapturedInference(s.graph, s.plan, s.ks, imgs[0], cache, warmup=False)
    tally = runner.report.totals().as_dict()

    def step(i=[0]):
        runner.run(imgs[i[0] % len(imgs)])
        i[0] += 1

    for _ in range(args.warmup):
        step()
    sampler = ClockSampler(d.local)
    sampler.start()
    sampler.wait_first()
    ms = timed_steps(d, step, args.steps, nvtx="timed")
    clocks = sampler.stop()
    ms_img = ms / args.steps
    value = d.world / (ms_img / 1e3)

    # e2e: encrypted input from pinned host memory, encrypted logits back
    host_in = [[ct.data.to("cpu").pin_memory() for ct in im.cts] for im in imgs]
    out_ct = runner.out
    host_out = torch.empty(out_ct.data.shape, dtype=torch.int64).pin_memory()
    h2d = sum(t.numel() * 8 for t in host_in[0])

    def e2e_step(i=[0]):
        src = host_in[i[0] % len(host_in)]
        for dst, h in zip(runner.inp.cts, src):
            dst.data.copy_(h, non_blocking=True)
        runner.cuda_graph.replay()
        host_out.copy_(out_ct.data, non_blocking=True)
        i[0] += 1

    for _ in range(2):
        e2e_step()
    ms_e2e = timed_steps(d, e2e_step, args.steps)
    e2e = {"value": d.world / (ms_e2e / args.steps / 1e3), "unit": "images/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": host_out.numel() * 8}

    # correctness of the measured path: decrypt the replayed logits
    logits = packing.read_logits(runner.run(imgs[0]), s.graph.n_classes, s.graph.formats[-1], s.ks)
    plain, _ = graph.execute(s.graph, s.plan, raw[0], mode="plaintext-ref")

    cpu = None
    if d.rank == 0 and d.world == 1 and not args.no_cpu_baseline:
        try:
            cpu = resnet_cpu_baseline(_oracle_for(s.params, _median_conv_level(s)), tally)
        except Exception as e:  # the checker must not take the bench down
            cpu = {"value": None, "unit": "images/s", "cores": None, "kind": "port", "sample": f"failed: {e}"}

    if d.rank == 0:
        line = {
            "metric": "ResNet20 CIFAR-10 encrypted inference images/s (s/image = ms_per_step/1e3)",
            "value": value, "unit": "images/s", "n_gpus": d.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_img, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": round(PAPER_A100_MS / ms_img, 4), "dtype": "u64", "data": "synthetic",
            "config": {"workload": "resnet20-cifar10-aespa-hyphen-bootstrap", "model": "AESPA-ResNet20 (random init)",
                       "input": "3x32x32 U(-1,1), encrypted", "ring_n": s.params.n, "slots": s.params.slots,
                       "multiplex": 4, "q_limbs": len(s.params.q_mods), "special_limbs": len(s.params.p_mods),
                       "app_levels": s.boot.output_level, "bootstrap_depth": s.cfg.depth(),
                       "refresh_points": list(s.plan.refresh_points), "refreshed_ciphertexts_per_image": tally["refreshes"],
                       "bootstraps_per_image": sum(graph.refresh_bootstraps(s.graph, s.params.slots)[i]
                                                   for i in s.plan.refresh_points),
                       "images_per_step_per_gpu": 1, "parallelism": f"dp{d.world} (independent images per GPU)",
                       "cuda_graph": True,
                       "resident_mask_gb": round(packing.resident_bytes() / 2 ** 30, 1),
                       "l2": "working set >> L2 (rotation keys ~15 GB, masks > 100 GB); no flush"},
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks, "gpu_launches": launches,
            "tally_per_image": tally, "kernels": kernels,
            "logits_check": {"max_abs_err_vs_plaintext": float(np.max(np.abs(logits - plain))),
                             "argmax_agree": bool(np.argmax(logits) == np.argmax(plain))},
            "setup": warm,
            "vs_baseline_note": "paper A100 1402 ms / our ms_per_step (PAPER.md:189)",
        }
        print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# config 2 primitive set
# ---------------------------------------------------------------------------

def run_cfg2(args, d: Dist):
    import torch
    from paper_2310_16530_b200 import _native, ckks, workloads

    params = workloads.cfg2_params()
    ks = ckks.keygen(params, np.random.default_rng(1), rotations=[1])
    rng = np.random.default_rng(5 + d.rank)
    L, B = params.max_level, args.batch
    pairs = [(ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, L), ks, rng),
              ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, L), ks, rng)) for _ in range(B)]

    def step():
        for a, b in pairs:
            ckks.rescale(ckks.hmult(a, b, ks), params)
            ckks.rotate(a, 1, ks)

    for _ in range(args.warmup):
        step()
    sampler = ClockSampler(d.local)
    sampler.start()
    sampler.wait_first()
    k0 = _native.kernel_launches()
    ms = timed_steps(d, step, args.steps)
    launches = _native.kernel_launches() - k0
    clocks = sampler.stop()
    value = d.world * B * args.steps / (ms / 1e3)
    _native.profile_read(reset=True)
    _native.ntt_limb_counts(reset=True)
    _native.profile_enable(True)
    step()
    torch.cuda.synchronize()
    _native.profile_enable(False)
    prof = _native.profile_read(reset=True)
    roofline, kernels = roofline_from_profile(prof)
    roofline = int_roofline(roofline, prof, _native.ntt_limb_counts(reset=True), params.n)
    if d.rank == 0:
        print(json.dumps({
            "metric": "HMult+relin+rescale+HRot primitive sets/s at N=2^16, L=24, K=4, dnum=7 (BASELINE cfg 2)",
            "value": value, "unit": "sets/s", "n_gpus": d.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u64", "data": "synthetic",
            "config": {"workload": "ckks-bench16-hmult-rescale-hrot", "batch_per_step": B, "ring_n": params.n,
                       "q_limbs": L + 1, "special_limbs": 4, "dnum": params.dnum, "level": L},
            "roofline": roofline, "clocks": clocks, "gpu_launches": launches, "kernels": kernels}), flush=True)


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle (the reference's path restated; the Python
# reference cannot travel to the GPU box)
# ---------------------------------------------------------------------------

def run_reference(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from paper_2310_16530_b200 import workloads
    params, g, plan = workloads.resnet20_plan_only()
    level = _median_conv_level_of(g, plan)
    tally = dict(workloads.RESNET20_TALLY)
    t0 = time.perf_counter()
    sampler = _oracle_for(params, level)
    t_keys = time.perf_counter() - t0
    for _ in range(args.warmup):
        sampler.sample()
    runs, walls = [], []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        runs.append(sampler.sample())
        walls.append(time.perf_counter() - t0)
    op_s = {k: statistics.median(r[k] for r in runs) for k in runs[0]}
    s_img = extrapolate(op_s, tally)
    value = 1.0 / s_img
    sample = (f"C/numpy oracle (restatement of the reference path) per-primitive times at level {level}, "
              f"median of {args.steps} (rotate {op_s['rotate']:.3f}s, hmult {op_s['hmult']:.3f}s, "
              f"rescale {op_s['rescale']:.3f}s, pmult {op_s['pmult']*1e3:.1f}ms, hadd {op_s['hadd']*1e3:.1f}ms) "
              f"x the GPU arm's per-image op tally {tally}; bootstraps excluded (the reference has none)")
    line = {
        "impl": "reference", "metric": "ResNet20 CIFAR-10 encrypted inference images/s (s/image = ms_per_step/1e3)",
        "value": value, "unit": "images/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": s_img * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": "resnet20-cifar10-aespa-hyphen-bootstrap", "ring_n": params.n,
                   "q_limbs": len(params.q_mods), "special_limbs": len(params.p_mods), "level_sampled": level,
                   "keygen_s": round(t_keys, 1), "sample_wall_s": round(statistics.mean(walls), 2)},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": sampler.cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--workload", default="resnet20", choices=["resnet20", "cfg2"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)  # K timed samples after W warm-up samples (~1.2 s each on 8 host threads)
        return
    d = Dist()
    try:
        if args.workload == "resnet20":
            run_resnet20(args, d)
        else:
            run_cfg2(args, d)
    finally:
        d.close()


if __name__ == "__main__":
    main()
