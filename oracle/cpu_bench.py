"""TEST INFRASTRUCTURE -- the CPU baseline sampler.  Never imported by the
product; run only by bench.py's cpu_baseline leg and its --impl reference
arm, always as a child process so the OpenMP thread
count and the core pinning are fixed before the C kernels load:

    taskset -c 0 env OMP_NUM_THREADS=1 python -m oracle.cpu_bench SPEC.json   (latency)
    P such processes, process i pinned to core i                          (throughput)

For each sampled level l it builds the oracle over the sub-chain
q_0..q_l || P (the reference's key switch at level l touches exactly
ceil((l+1)/alpha) digits over those moduli, ckks.py:548-602, so the work
is the full chain's at level l), generates a relinearisation key and one
rotation key, encrypts two ciphertexts at level l and times one call of
each primitive on the reference's path: rotate (ckks.py:620-657), hmult
(ckks.py:605-617), rescale (ckks.py:506-528), pmult (ckks.py:482-503),
hadd (ckks.py:457-466).  Prints {"levels": {l: {op: seconds}}, ...} as JSON.

extrapolate() turns those samples into seconds per image: every executed
layer's op tally (graph.CostReport rows of the GPU executor: count per op
and entry level) times the primitive time at that level, interpolated
linearly in the level between samples.  Bootstraps are excluded -- the
reference has none (its refresh slot is an insecure decrypt/re-encrypt,
ckks.py:667-690)."""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

OPS = ("rotate", "hmult", "rescale", "pmult", "hadd")


def sample_level(n: int, qs: list[int], ps: list[int], delta: float, level: int, seed: int = 1,
                 reps: int = 1) -> dict:
    from . import ckks_oracle as O
    P = O.OParams(n, list(qs[: level + 1]), list(ps), float(delta))
    rng = np.random.default_rng(seed)
    t0 = time.perf_counter()
    K = O.keygen(P, rng, rotations=[1])
    t_key = time.perf_counter() - t0
    a, sc = O.encode(rng.uniform(-1, 1, P.slots), P, level)
    b, _ = O.encode(rng.uniform(-1, 1, P.slots), P, level)
    ca, cb = O.encrypt(a, sc, K, rng)[0], O.encrypt(b, sc, K, rng)[0]
    mods = P.qs[: level + 1]
    ops = {
        "rotate": lambda: O.rotate(ca, 1, K),
        "hmult": lambda: O.hmult(ca, cb, K),
        "rescale": lambda: O.rescale(ca, P),
        "pmult": lambda: O.pmult(ca, a, mods),
        "hadd": lambda: np.stack([O.add(ca[0], cb[0], mods), O.add(ca[1], cb[1], mods)]),
    }
    out = {}
    for name, fn in ops.items():
        ts = []
        for _ in range(max(1, reps)):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        out[name] = float(np.median(ts))
    out["keygen_s"] = t_key
    return out


def run(spec: dict) -> dict:
    from . import ckks_oracle as O
    t0 = time.perf_counter()
    levels = {}
    for lv in spec["levels"]:
        levels[str(lv)] = sample_level(spec["n"], spec["qs"], spec["ps"], spec["delta"], int(lv),
                                       reps=int(spec.get("reps", 1)))
    return {"levels": levels, "threads": int(O.lib().o_num_threads()), "wall_s": time.perf_counter() - t0,
            "pid": os.getpid()}


def _at(samples: dict, op: str, level: int) -> float:
    pts = sorted((int(k), v[op]) for k, v in samples.items())
    if level <= pts[0][0]:
        lo = pts[0]
        hi = pts[1] if len(pts) > 1 else pts[0]
    elif level >= pts[-1][0]:
        lo, hi = (pts[-2] if len(pts) > 1 else pts[-1]), pts[-1]
    else:
        k = max(i for i, (l, _) in enumerate(pts) if l <= level)
        lo, hi = pts[k], pts[k + 1]
    if hi[0] == lo[0]:
        return lo[1]
    # linear in the level (clamped at zero when extrapolating below the lowest sample)
    return max(lo[1] + (hi[1] - lo[1]) * (level - lo[0]) / (hi[0] - lo[0]), 0.0)


def extrapolate(samples: dict, per_layer: list[dict]) -> dict:
    """Seconds per image: sum over executed layers of count(op) x t_op(level)."""
    total = 0.0
    by_op = {op: 0.0 for op in OPS}
    for row in per_layer:
        lv = row["entry_level"]
        t = row["tally"]
        for op, key in (("rotate", "rotations"), ("hmult", "hmults"), ("rescale", "rescales"),
                        ("pmult", "pmults"), ("hadd", "hadds")):
            c = t.get(key, 0)
            if c:
                s = c * _at(samples, op, lv)
                by_op[op] += s
                total += s
    return {"s_per_image": total, "by_op_s": {k: round(v, 3) for k, v in by_op.items()}}


def launch(spec: dict, cores: list[int]) -> list[dict]:
    """Run the sampler as one single-threaded process pinned to each listed
    core, all at once; returns their outputs (a one-element list is the
    latency run).  Called by bench.py only."""
    import subprocess
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        json.dump(spec, f)
        path = f.name
    env = dict(os.environ, OMP_NUM_THREADS="1", PYTHONPATH=root + os.pathsep + os.environ.get("PYTHONPATH", ""))
    procs = []
    for c in cores:
        procs.append(subprocess.Popen([sys.executable, "-m", "oracle.cpu_bench", path], cwd=root, env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True,
                                      preexec_fn=(lambda c=c: os.sched_setaffinity(0, {c}))))
    outs = []
    for pr in procs:
        o, e = pr.communicate()
        if pr.returncode != 0:
            raise RuntimeError(f"oracle sampler failed: {e[-500:]}")
        outs.append(json.loads(o.strip().splitlines()[-1]))
    os.unlink(path)
    return outs


def host_cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


if __name__ == "__main__":
    spec = json.loads(open(sys.argv[1]).read())
    print(json.dumps(run(spec)), flush=True)
