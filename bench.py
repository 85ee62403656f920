"""Benchmark driver (graft contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--images-per-gpu B]
                    [--workload resnet20|cfg2|boot16] [--impl ours|reference]

Default workload = the BASELINE.json metric: encrypted AESPA-ResNet20 on a
CIFAR-10-shaped (3x32x32) synthetic input, HyPHEN packing (multiplex 4,
N=2^16), real CKKS bootstrapping at the planner's refresh points
(workloads.resnet20_setup).  One step = B encrypted images per GPU, each
through the captured inference (graph.CapturedInference: the whole
executor, ~10^4 kernels with 6 bootstraps, replayed as one CUDA graph).
Random-init weights of the architecture (seeded), synthetic images.
Encrypted inputs/keys/masks exceed the 126 MB L2 by orders of magnitude
(no flush).

Multi-GPU: images are independent, so N ranks (one process per
GPU; started by torchrun, or by this script re-launching itself under
torch.distributed.run when --gpus N > 1 is given without it) each own a
block of the N*B images of a step (distributed.ShardPlan), with keys and
masks replicated; the only communication is the barrier + MAX of device
time around the timed region and the gather of the per-image logits checks.

`value` = whole-job images/s with encrypted inputs resident in HBM;
`ms_per_step` = device ms per step (MAX over ranks).  `e2e` = the same
through the public API with each encrypted input copied from pinned host
memory and the encrypted logits copied back every step.  `roofline` = the
kernel family with the largest device-time share in an event-profiled
eager run of one image; `keyswitch` = the whole key switch (ModUp + inner
product + ModDown) against max(HBM, integer) ideal time.  `cpu_baseline` =
the C/numpy oracle (tests' checker; the Python reference cannot travel to
the GPU box) on the host cores: per-primitive samples at three levels,
extrapolated over this image's per-layer op tally (bootstraps excluded:
the reference has none) -- latency on one pinned core, throughput with
one pinned process per core.

`--workload cfg2` runs BASELINE config 2 (HMult+relin, rescale and HRot(1)
on batches of ciphertext pairs at N=2^16, L=24); `--workload boot16`
config 3 (full-slot bootstrapping at N=2^16: ms per bootstrap, precision).
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


def timed_steps(cl, fn, steps: int, nvtx: str | None = None) -> float:
    """device ms over `steps` calls of fn, CUDA events on the current stream,
    barrier + synchronize on both sides, MAX over ranks (Cluster.timed).
    nvtx: name of an NVTX range around the timed region (ncu --nvtx
    --nvtx-include "<name>/" captures exactly these launches)."""
    return cl.timed(fn, steps, nvtx=nvtx)


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
    # class-2 limbs (q < 2^41: the 40-bit primes) run the pure FP64 network:
    # its register-only probe is their ceiling; full-width limbs the integer one
    pf, ps = _native.ntt_butterfly_peak(4), _native.ntt_butterfly_peak(0)
    per_limb = n // 2 * (n.bit_length() - 1)
    ideal_s = per_limb * (fast / pf + full / ps)
    bfly = per_limb * (fast + full)
    achieved = bfly / (ms / 1e3)
    peak = bfly / ideal_s
    hbm = {k: roof[k] for k in ("achieved", "peak", "unit", "frac", "peak_source", "algorithmic_bytes_per_launch")}
    # DRAM traffic per launch from the committed ncu --set full capture, scaled per limb
    traffic = roof.get("traffic")
    tf = ROOT / "profiles" / "r02_ncu_ntt_traffic.json"
    if traffic is None and tf.exists():
        cls = json.loads(tf.read_text())["per_class"]
        launches = sum(v["launches"] for k, v in prof.items() if _kernel_family(k) == fam)
        traffic = round((cls[f"{d}_f64"]["dram_bytes_per_limb"] * fast + cls[f"{d}_int"]["dram_bytes_per_limb"] * full)
                        / max(launches, 1))
        hbm["traffic_source"] = ("profiles/r02_ncu_ntt_traffic.json (ncu --cache-control none, steady state, "
                                 "per-class DRAM bytes per limb) x this run's limbs per launch "
                                 "(one launch = the cols + chunks pass pair)")
    out = {"kernel": fam, "bound": "int", "achieved": round(achieved / 1e9, 2), "peak": round(peak / 1e9, 2),
           "unit": "Gbutterfly/s", "frac": round(ideal_s / (ms / 1e3), 4), "traffic": traffic,
           "peak_source": (f"measured on this GPU: the kernels' radix-16 register networks without memory traffic "
                           f"(hcnn_ntt_butterfly_peak) {pf/1e9:.1f} Gbfly/s for the FP64 network of the "
                           f"q<2^41 limbs, {ps/1e9:.1f} for the integer network of full-width limbs, weighted by "
                           f"this run's {fast} + {full} limbs"),
           "limbs": {"fast": fast, "full": full}, "share_of_device_time": roof["share_of_device_time"],
           "hbm": hbm}
    return out


def peak_kind_note(kind: str) -> str:
    return f"{kind} (MEASURED_PEAKS.json hbm_gbs)" if kind == "measured" else "fallback 6650 GB/s"




# ---------------------------------------------------------------------------
# whole key switch (ModUp + inner product + ModDown) against max(HBM, int)
# ---------------------------------------------------------------------------

KS_LABELS = ("ntt_inv_modup", "modup", "ntt_fwd_modup", "ks_inner", "ntt_inv_moddown", "moddown_fbc",
             "ntt_fwd_moddown", "moddown_combine", "add_pmul")


def keyswitch_roofline(prof: dict, ksc: dict, n: int) -> dict | None:
    """SURVEY 8d's key-switch unit: minimal HBM bytes (the digits read once,
    the switch keys, the outputs -- hcnn_ks_counters) and the limb-NTTs the
    hybrid key switch cannot avoid (ModUp iNTT + digit NTTs, ModDown iNTT of
    the specials + NTT of the lift); ideal = max(bytes / HBM peak,
    butterflies / butterfly peak), frac = ideal / measured device time of
    every kernel of the chain.  The butterfly peak is the faster (FP64)
    network's for every limb, so the integer bound is not flattered."""
    from paper_2310_16530_b200 import _native
    ms = sum(prof[k]["ms"] for k in KS_LABELS if k in prof)
    if ms <= 0 or not ksc.get("keyswitches"):
        return None
    total = sum(v["ms"] for v in prof.values()) or 1.0
    peak_gbs, kind = _peaks()
    per_limb = n // 2 * (n.bit_length() - 1)
    limbs = ksc["fwd_limbs"] + ksc["inv_limbs"]
    bfly = per_limb * limbs
    pf = _native.ntt_butterfly_peak(4)  # the FP64 network: the faster ceiling of the two
    t = ms / 1e3
    t_hbm = ksc["min_bytes"] / (peak_gbs * 1e9)
    t_int = bfly / pf
    ideal = max(t_hbm, t_int)
    return {"kernel": "keyswitch (ModUp + inner product + ModDown chain)", "bound": "int" if t_int >= t_hbm else "hbm",
            "frac": round(ideal / t, 4), "ms": round(ms, 3), "keyswitches": ksc["keyswitches"],
            "us_per_keyswitch": round(ms * 1e3 / ksc["keyswitches"], 2),
            "share_of_device_time": round(ms / total, 4),
            "hbm": {"achieved": round(ksc["min_bytes"] / t / 1e9, 1), "peak": peak_gbs, "unit": "GB/s",
                    "frac": round(t_hbm / t, 4), "min_bytes": ksc["min_bytes"]},
            "int": {"achieved": round(bfly / t / 1e9, 1), "peak": round(pf / 1e9, 1), "unit": "Gbutterfly/s",
                    "frac": round(t_int / t, 4), "limb_ntts": limbs,
                    "peak_source": "hcnn_ntt_butterfly_peak(4): the FP64 radix-16 network, register-only, measured here"}}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle on the host cores
# ---------------------------------------------------------------------------

def _layer_rows(per_layer: list[dict]) -> list[dict]:
    return [{"name": r["name"], "kind": r["kind"], "tally": r["tally"], "entry_level": r["entry_level"]}
            for r in per_layer]


def cpu_baseline(params, per_layer: list[dict], reps: int = 1, throughput: bool = True) -> dict:
    """Latency: one process pinned to one core (OMP_NUM_THREADS=1); the
    throughput run: one such process per available core, all at once,
    images/s = sum of their rates.  Each process samples the five
    primitives at three levels (min / median / max conv entry level) and
    extrapolates over the per-layer tally (oracle/cpu_bench.py)."""
    from oracle import cpu_bench
    lv = sorted({r["entry_level"] for r in per_layer if r["kind"] == "conv"})
    levels = sorted({lv[0], lv[len(lv) // 2], lv[-1]})
    spec = {"n": params.n, "qs": [m.q for m in params.q_mods], "ps": [m.q for m in params.p_mods],
            "delta": float(params.delta), "levels": levels, "reps": reps}
    cores = sorted(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    lat = cpu_bench.launch(spec, cores[:1])[0]
    t_lat = time.perf_counter() - t0
    lat_x = cpu_bench.extrapolate(lat["levels"], per_layer)
    out = {"latency_s_per_image": lat_x["s_per_image"], "latency_by_op_s": lat_x["by_op_s"],
           "latency_samples": lat["levels"], "latency_wall_s": round(t_lat, 1), "cpu_model": cpu_bench.host_cpu_model(),
           "levels_sampled": levels}
    if throughput:
        t0 = time.perf_counter()
        runs = cpu_bench.launch(spec, cores)
        out["throughput_wall_s"] = round(time.perf_counter() - t0, 1)
        rates = [1.0 / cpu_bench.extrapolate(r["levels"], per_layer)["s_per_image"] for r in runs]
        out["throughput_images_per_s"] = sum(rates)
        out["processes"] = len(runs)
    return out


def cpu_baseline_line(cb: dict, what: str) -> dict:
    thr = "throughput_images_per_s" in cb
    return {"value": cb["throughput_images_per_s"] if thr else 1.0 / cb["latency_s_per_image"], "unit": "images/s",
            "cores": cb.get("processes", 1), "kind": "port",
            "sample": (f"extrapolated: the C/numpy oracle (restatement of the reference path, single-threaded) "
                       f"times rotate/hmult/rescale/pmult/hadd once per level at levels {cb['levels_sampled']} "
                       f"(sub-chain keys per level), interpolated linearly in the level and multiplied by {what}; "
                       + (f"{cb['processes']} processes, one pinned per core, all at once (throughput); " if thr else "")
                       + f"latency on one pinned core {cb['latency_s_per_image']:.0f} s/image; bootstraps "
                       f"excluded (the reference has none); host {cb['cpu_model']}"),
            "latency_s_per_image": round(cb["latency_s_per_image"], 1), "latency_by_op_s": cb["latency_by_op_s"],
            "latency_samples": cb["latency_samples"],
            "wall_s": {"latency": cb["latency_wall_s"], "throughput": cb.get("throughput_wall_s")}}


# ---------------------------------------------------------------------------
# ResNet20 (default)
# ---------------------------------------------------------------------------

TALLY_FILE = ROOT / "paper_2310_16530_b200" / "data" / "resnet20_tally.json"


def resnet20_config(s_or_params, g, plan, boot_depth: int, out_level: int, world: int, B: int) -> dict:
    from paper_2310_16530_b200 import graph
    params = s_or_params
    return {"workload": "resnet20-cifar10-aespa-hyphen-bootstrap", "model": "AESPA-ResNet20 (random init)",
            "input": "3x32x32 U(-1,1), encrypted", "ring_n": params.n, "slots": params.slots, "multiplex": 4,
            "q_limbs": len(params.q_mods), "special_limbs": len(params.p_mods), "app_levels": out_level,
            "bootstrap_depth": boot_depth, "refresh_points": list(plan.refresh_points),
            "bootstraps_per_image": sum(graph.refresh_bootstraps(g, params.slots)[i] for i in plan.refresh_points),
            "images_per_step_per_gpu": B, "global_batch": B * world,
            "parallelism": f"dp{world} (independent images per GPU, keys and masks replicated)",
            "l2": "working set >> L2 (rotation keys ~15 GB, masks > 100 GB); no flush"}


def _image(i: int) -> np.ndarray:
    return np.random.default_rng(1000 + i).uniform(-1.0, 1.0, (3, 32, 32))


def run_resnet20(args, cl):
    import torch
    from paper_2310_16530_b200 import _native, ckks, graph, packing, workloads

    B = args.images_per_gpu
    s = workloads.resnet20_setup()
    mine = list(cl.shard(B * cl.world))  # this rank's global image indices
    raw = [_image(i) for i in mine]
    imgs = [workloads.encrypt_image(s, x, np.random.default_rng(2000 + i)) for i, x in zip(mine, raw)]
    cache: dict = {}
    # eager runs first (mask build, measured residency fill, lazy tables;
    # then one event-profiled image for the kernel table / roofline / launch
    # count), then capture -- so the capture pool reuses the eager memory
    # --batch-mode stack (default): the B images of a step are stacked into
    # [B, 2, l+1, N] ciphertexts and the executor runs ONCE for all of them
    # (graph.stack_images: every kernel covers the B images, bootstraps
    # included; each image's residues equal its single-image run);
    # lockstep: graph.execute_many (per-image layers, shared bootstraps)
    stacked = B > 1 and args.batch_mode == "stack"
    units = [graph.stack_images(imgs)] if stacked else imgs
    warm = workloads.warm_up(s, units, cache)
    k0 = _native.kernel_launches()
    _native.profile_read(reset=True)
    _native.ntt_limb_counts(reset=True)
    _native.ks_counters(reset=True)
    _native.profile_enable(True)
    graph.execute_many(s.graph, s.plan, units, s.ks, cache=cache)
    torch.cuda.synchronize()
    _native.profile_enable(False)
    prof = _native.profile_read(reset=True)
    limbs = _native.ntt_limb_counts(reset=True)
    ksc = _native.ks_counters(reset=True)
    launches = _native.kernel_launches() - k0
    roofline, kernels = roofline_from_profile(prof)
    roofline = int_roofline(roofline, prof, limbs, s.params.n)
    ks_roof = keyswitch_roofline(prof, ksc, s.params.n)
    # all B images of a step in one captured graph
    runner = graph.CapturedInference(s.graph, s.plan, s.ks, units[0], cache, warmup=False, images=len(units))
    per_layer = _layer_rows(runner.report.per_layer)
    tally = runner.report.totals().as_dict()

    def step():
        runner.run_many(units)

    for _ in range(args.warmup):
        step()
    sampler = ClockSampler(cl.local)
    sampler.start()
    sampler.wait_first()
    ms = timed_steps(cl, step, args.steps, nvtx="timed")
    clocks = sampler.stop()
    ms_step = ms / args.steps
    value = B * cl.world / (ms_step / 1e3)

    # e2e: every step's encrypted inputs from pinned host memory, encrypted logits back
    host_in = [[ct.data.to("cpu").pin_memory() for ct in im.cts] for im in units]
    host_out = [torch.empty(o.data.shape, dtype=torch.int64).pin_memory() for o in runner.outs]
    h2d = sum(t.numel() * 8 for src in host_in for t in src)

    def e2e_step():
        for src, inp in zip(host_in, runner.inps):
            for dst, h in zip(inp.cts, src):
                dst.data.copy_(h, non_blocking=True)
        runner.cuda_graph.replay()
        for o, hout in zip(runner.outs, host_out):
            hout.copy_(o.data, non_blocking=True)

    for _ in range(2):
        e2e_step()
    ms_e2e = timed_steps(cl, e2e_step, args.steps)
    torch.cuda.synchronize()
    e2e = {"value": B * cl.world / (ms_e2e / args.steps / 1e3), "unit": "images/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": sum(h.numel() * 8 for h in host_out)}
    out_ct = runner.out
    # one host logits tensor per image (the last e2e step's copies)
    per_image_out = [h[b] for h in host_out for b in range(h.shape[0])] if stacked else host_out

    # correctness of the measured path: decrypt each of this rank's replayed
    # logits against the float mirror
    checks = []
    for i, x, hout in zip(mine, raw, per_image_out):
        ct = ckks.Ciphertext(hout.to(s.params.ctx.torch_device), out_ct.scale, out_ct.n, s.params)
        lg = packing.read_logits(ct, s.graph.n_classes, s.graph.formats[-1], s.ks)
        pl, _ = graph.execute(s.graph, s.plan, x, mode="plaintext-ref")
        checks.append({"image": i, "max_abs_err": float(np.max(np.abs(lg - pl))),
                       "rel_err": float(np.max(np.abs(lg - pl)) / np.max(np.abs(pl))),
                       "argmax_agree": bool(np.argmax(lg) == np.argmax(pl))})
    all_checks = cl.gather({"rank": cl.rank, "checks": checks, "ms": ms, "value_rank": B / (ms_step / 1e3)})

    cpu = None
    if cl.rank == 0 and cl.world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_line(cpu_baseline(s.params, per_layer), "this image's per-layer op tally "
                                    "(graph.CostReport of the captured inference)")
        except Exception as e:  # the checker must not take the bench down
            cpu = {"value": None, "unit": "images/s", "cores": None, "kind": "port", "sample": f"failed: {e}"}

    if cl.rank == 0:
        flat = [c for part in all_checks for c in part["checks"]]
        line = {
            "metric": "ResNet20 CIFAR-10 encrypted inference images/s (s/image = ms_per_step/images_per_step_per_gpu/1e3)",
            "value": value, "unit": "images/s", "n_gpus": cl.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "s_per_image_per_gpu": ms_step / B / 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": round(PAPER_A100_MS / (ms_step / B), 4), "dtype": "u64",
            "data": "synthetic",
            "config": resnet20_config(s.params, s.graph, s.plan, s.cfg.depth(), s.boot.output_level, cl.world, B),
            "e2e": e2e, "roofline": roofline, "keyswitch": ks_roof, "cpu_baseline": cpu, "clocks": clocks,
            "gpu_launches": launches, "gpu_launches_per_image": launches / B, "cuda_graph": True,
            "resident_mask_gb": round(packing.resident_bytes() / 2 ** 30, 1),
            "tally_per_image": tally, "kernels": kernels,
            "per_rank": [{"rank": p["rank"], "ms": round(p["ms"], 3), "images_per_s": round(p["value_rank"], 4)}
                         for p in all_checks],
            "logits_check": {"images": len(flat), "max_rel_err_vs_plaintext": max(c["rel_err"] for c in flat),
                             "max_abs_err_vs_plaintext": max(c["max_abs_err"] for c in flat),
                             "argmax_agree": all(c["argmax_agree"] for c in flat)},
            "setup": warm, "batch_mode": (args.batch_mode if B > 1 else None),
            "vs_baseline_note": "paper A100 1402 ms / our s per image (PAPER.md:189)",
        }
        print(json.dumps(line), flush=True)
        if args.tally_out:
            Path(args.tally_out).write_text(json.dumps({"per_layer": per_layer, "totals": tally}, indent=1) + "\n")


# ---------------------------------------------------------------------------
# config 2 primitive set
# ---------------------------------------------------------------------------

def run_cfg2(args, cl):
    import torch
    from paper_2310_16530_b200 import _native, ckks, workloads

    params = workloads.cfg2_params()
    ks = ckks.keygen(params, np.random.default_rng(1), rotations=[1])
    rng = np.random.default_rng(5 + cl.rank)
    L, B = params.max_level, args.batch
    pairs = [(ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, L), ks, rng),
              ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, L), ks, rng)) for _ in range(B)]

    # batched (default): the B pairs stacked once into [B, 2, L+1, N] ciphertexts,
    # one hmult / rescale / rotate call each over the whole batch
    # (hcnn_hmult_batch, hcnn_rotate_hoisted_batch: keys read once per batch);
    # sequential: the reference's one-ciphertext-per-call loop, timed alongside
    sa, sb = ckks.stack([a for a, _ in pairs]), ckks.stack([b for _, b in pairs])

    def seq_step():
        for a, b in pairs:
            ckks.rescale(ckks.hmult(a, b, ks), params)
            ckks.rotate(a, 1, ks)

    def batch_step():
        ckks.rescale(ckks.hmult(sa, sb, ks), params)
        ckks.rotate(sa, 1, ks)

    step = seq_step if args.batch_mode == "lockstep" or B == 1 else batch_step
    for _ in range(args.warmup):
        seq_step()
        batch_step()
    sampler = ClockSampler(cl.local)
    sampler.start()
    sampler.wait_first()
    k0 = _native.kernel_launches()
    ms = timed_steps(cl, step, args.steps)
    launches = _native.kernel_launches() - k0
    seq_ms = timed_steps(cl, seq_step, args.steps)
    clocks = sampler.stop()
    value = cl.world * B * args.steps / (ms / 1e3)
    _native.profile_read(reset=True)
    _native.ntt_limb_counts(reset=True)
    _native.ks_counters(reset=True)
    _native.profile_enable(True)
    step()
    torch.cuda.synchronize()
    _native.profile_enable(False)
    prof = _native.profile_read(reset=True)
    ksc = _native.ks_counters(reset=True)
    roofline, kernels = roofline_from_profile(prof)
    roofline = int_roofline(roofline, prof, _native.ntt_limb_counts(reset=True), params.n)
    ks_roof = keyswitch_roofline(prof, ksc, params.n)
    if cl.rank == 0:
        print(json.dumps({
            "metric": "HMult+relin+rescale+HRot primitive sets/s at N=2^16, L=24, K=4, dnum=7 (BASELINE cfg 2)",
            "value": value, "unit": "sets/s", "n_gpus": cl.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u64", "data": "synthetic",
            "config": {"workload": "ckks-bench16-hmult-rescale-hrot", "batch_per_step": B, "ring_n": params.n,
                       "q_limbs": L + 1, "special_limbs": 4, "dnum": params.dnum, "level": L,
                       "calls": "sequential" if step is seq_step else "batched"},
            "sequential": {"ms_per_step": seq_ms / args.steps, "value": cl.world * B * args.steps / (seq_ms / 1e3),
                           "note": "one hmult / rescale / rotate call per ciphertext (the reference's loop)"},
            "roofline": roofline, "keyswitch": ks_roof, "clocks": clocks, "gpu_launches": launches // args.steps,
            "kernels": kernels}), flush=True)


# ---------------------------------------------------------------------------
# config 3: full-slot bootstrapping at N=2^16
# ---------------------------------------------------------------------------

def run_boot16(args, cl):
    """BASELINE cfg 3: one step = bootstrapping `--batch` level-0
    ciphertexts of U(-1,1) slot values (one batched bootstrap); precision =
    -log2 of the max abs slot error after decrypt-and-decode (parity
    unpinned: the reference has no bootstrapping)."""
    import torch
    from paper_2310_16530_b200 import _native, bootstrap as bt, ckks

    cfg = bt.BootConfig()
    params = bt.boot_params("boot16", 1 << 16, 8, cfg)
    boot = bt.Bootstrapper(params, cfg)
    t0 = time.time()
    ks = boot.keygen(np.random.default_rng(16), rotations=[1])
    t_key = time.time() - t0
    rng = np.random.default_rng(3 + cl.rank)
    nb = max(1, args.boot_batch)
    vals = [rng.uniform(-1, 1, params.slots) for _ in range(nb)]
    cts = [ckks.encrypt(ckks.encode(v, params, 0), ks, rng) for v in vals]

    x = ckks.stack(cts) if nb > 1 else cts[0]

    def eager():
        return boot.bootstrap(x, ks)

    t0 = time.time()
    eager()  # first run: bootstrapping masks (host encode), conversion tables
    torch.cuda.synchronize()
    t_first = time.time() - t0
    eager()
    # the whole batched bootstrap replayed as one CUDA graph (as inside the
    # captured ResNet20 inference): host dispatch off the timed path
    k0 = _native.kernel_launches()
    _native.profile_read(reset=True)
    _native.ntt_limb_counts(reset=True)
    _native.ks_counters(reset=True)
    _native.profile_enable(True)
    eager()
    torch.cuda.synchronize()
    _native.profile_enable(False)
    launches = _native.kernel_launches() - k0
    prof = _native.profile_read(reset=True)
    ksc = _native.ks_counters(reset=True)
    limbs = _native.ntt_limb_counts(reset=True)
    torch.cuda.synchronize()
    cg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(cg):
        out_c = eager()
    torch.cuda.synchronize()
    cg.replay()
    torch.cuda.synchronize()
    outs = ckks.unstack(out_c) if nb > 1 else [out_c]
    errs = [float(np.max(np.abs(ckks.decode(ckks.decrypt(o, ks), params, imag_tol=None) - v)))
            for o, v in zip(outs, vals)]
    step = cg.replay
    for _ in range(args.warmup):
        step()
    sampler = ClockSampler(cl.local)
    sampler.start()
    sampler.wait_first()
    ms = timed_steps(cl, step, args.steps)
    clocks = sampler.stop()
    roofline, kernels = roofline_from_profile(prof)
    roofline = int_roofline(roofline, prof, limbs, params.n)
    ks_roof = keyswitch_roofline(prof, ksc, params.n)
    ms_step = ms / args.steps
    if cl.rank == 0:
        err = max(errs)
        print(json.dumps({
            "metric": "full-slot CKKS bootstrapping at N=2^16 (BASELINE cfg 3): bootstraps/s",
            "value": cl.world * nb / (ms_step / 1e3), "unit": "bootstraps/s", "n_gpus": cl.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "ms_per_bootstrap": ms_step / nb,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": "ckks-boot16-full-slot", "ring_n": params.n, "slots": params.slots,
                       "q_limbs": len(params.q_mods), "special_limbs": len(params.p_mods), "depth": cfg.depth(),
                       "output_level": boot.output_level, "ciphertexts_per_step": nb,
                       "secret_hamming_weight": cfg.secret_weight, "rotation_keys": len(ks.gks),
                       "cuda_graph": True},
            "precision": {"max_abs_err": err, "bits": round(-float(np.log2(err)), 2),
                          "check": "decrypt-and-decode vs the encrypted U(-1,1) values (parity unpinned: the "
                                   "reference has no bootstrapping, ckks.py:667-690)"},
            "keygen_s": round(t_key, 2), "first_step_s": round(t_first, 2),
            "roofline": roofline, "keyswitch": ks_roof, "clocks": clocks, "gpu_launches": launches,
            "kernels": kernels, "cpu_baseline": None,
            "cpu_baseline_note": "n/a: the reference has no bootstrapping (BASELINE.md section 4)"}), flush=True)


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle (the reference's path restated; the Python
# reference cannot travel to the GPU box)
# ---------------------------------------------------------------------------

def run_reference(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from paper_2310_16530_b200 import workloads
    params, g, plan = workloads.resnet20_plan_only()
    depth = workloads.resnet20_boot_config().depth()
    out_level = params.max_level - depth
    saved = json.loads(TALLY_FILE.read_text())
    per_layer = saved["per_layer"]
    reps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    cb = cpu_baseline(params, per_layer, reps=reps)
    wall = time.perf_counter() - t0
    value = cb["throughput_images_per_s"]
    B = args.images_per_gpu
    cfg = resnet20_config(params, g, plan, depth, out_level, args.gpus, B)
    line = {
        "impl": "reference",
        "metric": "ResNet20 CIFAR-10 encrypted inference images/s (s/image = ms_per_step/images_per_step_per_gpu/1e3)",
        "value": value, "unit": "images/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": B * 1e3 / value, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic", "config": cfg,
        "cpu_baseline": cpu_baseline_line(cb, f"the GPU arm's per-layer op tally ({TALLY_FILE.name}, checked "
                                              f"against the executor by tests/test_gpu_resnet20.py)")
        | {"reps_per_primitive": reps},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": round(wall, 1),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# selftest: the multi-rank skeleton (relaunch -> Cluster -> shard -> timed
# -> gather -> one line) with a CPU stub step, run over gloo by the CPU tests
# ---------------------------------------------------------------------------

def run_selftest(args, cl):
    B = args.images_per_gpu
    mine = list(cl.shard(B * cl.world))
    work = [np.random.default_rng(1000 + i).uniform(-1, 1, 256) for i in mine]
    acc = [0.0]

    def step():
        for w in work:
            acc[0] += float(np.sum(w * w))

    for _ in range(args.warmup):
        step()
    ms = timed_steps(cl, step, args.steps)
    parts = cl.gather({"rank": cl.rank, "images": mine, "ms": ms})
    if cl.rank == 0:
        print(json.dumps({"metric": "selftest items/s", "value": B * cl.world / (ms / args.steps / 1e3),
                          "unit": "items/s", "n_gpus": cl.world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": ms / args.steps, "backend": "gloo" if not cl.cuda else "nccl",
                          "per_rank": parts}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=8, help="cfg2: ciphertext pairs per step")
    ap.add_argument("--boot-batch", type=int, default=1, help="boot16: ciphertexts bootstrapped per step")
    ap.add_argument("--images-per-gpu", type=int, default=1, help="resnet20: images per GPU per step")
    ap.add_argument("--batch-mode", default="stack", choices=["stack", "lockstep"],
                    help="resnet20, B > 1: stacked image batches (one executor pass) or execute_many; "
                         "cfg2: stack = one batched call per op, lockstep = one call per ciphertext")
    ap.add_argument("--workload", default="resnet20", choices=["resnet20", "cfg2", "boot16", "selftest"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tally-out", default=None, help="resnet20: write the per-layer op tally here")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)  # host cores only; rank 0 prints, other ranks exit 0
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        from paper_2310_16530_b200.distributed import relaunch
        sys.exit(relaunch(args.gpus, str(Path(__file__).resolve()), sys.argv[1:]))
    from paper_2310_16530_b200.distributed import Cluster
    cl = Cluster(backend="gloo" if args.workload == "selftest" else None)
    try:
        {"resnet20": run_resnet20, "cfg2": run_cfg2, "boot16": run_boot16,
         "selftest": run_selftest}[args.workload](args, cl)
    finally:
        cl.close()


if __name__ == "__main__":
    main()
