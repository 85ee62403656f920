"""The benchmarked path itself (BASELINE cfg 4): encrypted AESPA-ResNet20 on
CIFAR-10-shaped inputs at N=2^16 with real bootstrapping, exactly as
bench.py runs it (workloads.resnet20_setup: compact GPU-encoded masks,
packed resident masks, the whole inference replayed from one CUDA graph).

* CUDA-graph replay == eager execution, residue for residue, on 3 images.
* Decrypted logits vs the float oracle (graph.execute(mode="plaintext-ref"),
  the reference's reference_forward pattern, graph.py:817-864, with the
  tolerance check of test_graph.py:409-412) within 1e-3 RELATIVE
  (max|d| / max|logit|) with identical top-1, on 3 images x 2 weight seeds.
* The GPU mask encode (torch FFT) against the reference's host encode
  (numpy FFT, ckks.py:260-290) on a sample of the real mask set: integer
  mismatches are counted and reported (gpurun_out/r2_mask_encode.json) and
  bounded (|d| <= 1 per coefficient, a rounding tie broken differently).
* N=2^16 batched hoisted rotations (nb = 2, 3, 5 -> the TMA inner product)
  equal single rotations and the reference's bench16 rotate digests.
"""

import hashlib
import json
import os
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
REL_TOL = 1e-3


def h(arr) -> str:
    a = np.ascontiguousarray(np.asarray(arr, dtype=np.uint64))
    return hashlib.sha256(a.astype("<u8").tobytes()).hexdigest()


def _free_setup():
    import gc
    import torch
    from paper_2310_16530_b200 import packing
    gc.collect()
    packing._RESIDENT["used"] = 0
    packing.set_mask_mode("host")
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def _images(seed, n=3):
    rng = np.random.default_rng(seed)
    return [rng.uniform(-1.0, 1.0, (3, 32, 32)) for _ in range(n)]


def _rel(logits, plain):
    return float(np.max(np.abs(logits - plain)) / np.max(np.abs(plain)))


@pytest.fixture(scope="module")
def r20_bench():
    """The bench configuration (weight seed 3): warm-up with measured
    residency, then capture -- bench.py's run_resnet20 sequence."""
    import torch
    from paper_2310_16530_b200 import ckks, graph, packing, workloads
    s = workloads.resnet20_setup(seed=3)
    raw = _images(100)
    rng = np.random.default_rng(7)
    imgs = [workloads.encrypt_image(s, x, rng) for x in raw]
    cache: dict = {}
    workloads.warm_up(s, imgs[0], cache)
    eager = []
    for im in imgs:
        out, rep = graph.execute(s.graph, s.plan, im, s.ks, "encrypted", cache=cache)
        eager.append((out.data.clone(), out.scale, out.level))
    tally = rep.totals().as_dict()
    # two images stacked into [2, 2, l+1, N] ciphertexts through one executor
    # pass (bench.py --images-per-gpu 2): bootstraps included, each image
    # must equal its single-image run
    sout, srep = graph.execute(s.graph, s.plan, graph.stack_images(imgs[:2]), s.ks, "encrypted", cache=cache)
    stacked = [(o.data.clone(), o.scale, o.level) for o in graph.unstack_images(sout)]
    stacked_tally = srep.totals().as_dict()
    del sout
    runner = graph.CapturedInference(s.graph, s.plan, s.ks, imgs[0], cache, warmup=False)
    replay = []
    for im in imgs:
        o = runner.run(im)
        torch.cuda.synchronize()
        replay.append((o.data.clone(), o.scale, o.level))
    logits = [packing.read_logits(ckks.Ciphertext(d, sc, s.params.n, s.params), s.graph.n_classes,
                                  s.graph.formats[-1], s.ks) for d, sc, _ in replay]
    plain = [graph.execute(s.graph, s.plan, x, mode="plaintext-ref")[0] for x in raw]
    res = {"eager": eager, "replay": replay, "logits": logits, "plain": plain, "tally": tally,
           "stacked": stacked, "stacked_tally": stacked_tally,
           "runner_tally": runner.report.totals().as_dict(),
           "per_layer": [{"name": r["name"], "kind": r["kind"], "tally": r["tally"], "entry_level": r["entry_level"]}
                         for r in runner.report.per_layer]}
    yield res
    del runner, cache, s, imgs
    _free_setup()


def test_replay_equals_eager(r20_bench):
    import torch
    assert r20_bench["tally"] == r20_bench["runner_tally"]
    for (de, se, le), (dr, sr, lr) in zip(r20_bench["eager"], r20_bench["replay"]):
        assert le == lr and se == sr
        assert torch.equal(de, dr), "CUDA-graph replay differs from eager execution"


def test_stacked_images_equal_single_runs(r20_bench):
    """ResNet20 at N=2^16 with real bootstrapping, two images stacked into
    [2, 2, l+1, N] ciphertexts: each image's encrypted logits are bit-identical
    to its single-image run (bootstrapping is entry-wise in a batch)."""
    import torch
    assert r20_bench["stacked_tally"] == r20_bench["tally"]
    for (ds, ss, ls), (de, se, le) in zip(r20_bench["stacked"], r20_bench["eager"][:2]):
        assert ls == le and ss == se
        assert torch.equal(ds, de)


def test_committed_tally_matches_executor(r20_bench):
    """bench.py --impl reference extrapolates the CPU oracle over the
    committed per-layer tally (paper_2310_16530_b200/data/resnet20_tally.json);
    it must be exactly what the executor runs."""
    path = ROOT / "paper_2310_16530_b200" / "data" / "resnet20_tally.json"
    saved = json.loads(path.read_text())
    if saved["per_layer"] != r20_bench["per_layer"]:
        (ROOT / "gpurun_out").mkdir(exist_ok=True)
        (ROOT / "gpurun_out" / "resnet20_tally.json").write_text(
            json.dumps({"per_layer": r20_bench["per_layer"], "totals": r20_bench["tally"]}, indent=1) + "\n")
    assert saved["per_layer"] == r20_bench["per_layer"]
    assert saved["totals"] == r20_bench["tally"]


def test_bench_config_logits(r20_bench):
    for lg, pl in zip(r20_bench["logits"], r20_bench["plain"]):
        assert _rel(lg, pl) < REL_TOL, (_rel(lg, pl), lg, pl)
        assert int(np.argmax(lg)) == int(np.argmax(pl))


@pytest.mark.parametrize("nb", [2, 3, 5])
def test_bench16_batched_rotations(golden_hashes, nb):
    """Batched hoisted rotations at N=2^16, 25 q-limbs (the 2-entry and
    larger batches take k_ks_inner_tma2): every entry equals its single
    rotation, and ct1's entries hash to the reference's rotate digests."""
    import torch
    from paper_2310_16530_b200 import ckks
    gold = golden_hashes["bench16"]
    params = ckks.bench16()
    ks = _bench16_keys(params, gold)
    ct1, ct2 = _bench16_cts(params, ks)
    members = [ct1, ct2, ct1, ct2, ct1][:nb]
    batch = ckks.stack(members)
    outs = ckks.rotate_many(batch, [1, 4], ks)
    for step, o in zip([1, 4], outs):
        for m, got in zip(members, ckks.unstack(o)):
            assert torch.equal(got.data, ckks.rotate(m, step, ks).data), (nb, step)
    # composite step 5 = 4 + 1 on the batch, entry 0 = ct1
    five = ckks.rotate(batch, 5, ks)
    assert h(np.stack(ckks.unstack(five)[0].host_residues())) == gold["rot"]["5"]
    assert h(np.stack(ckks.unstack(outs[0])[0].host_residues())) == gold["rot"]["1"]


_B16: dict = {}


def _bench16_keys(params, gold):
    from paper_2310_16530_b200 import ckks
    if "ks" not in _B16:
        _B16["ks"] = ckks.keygen(params, np.random.default_rng(gold["key_seed"]), rotations=gold["rotations"])
    return _B16["ks"]


def _bench16_cts(params, ks):
    from paper_2310_16530_b200 import ckks
    if "cts" not in _B16:
        vrng = np.random.default_rng(12345)
        v1 = vrng.uniform(-1, 1, params.slots)
        v2 = vrng.uniform(-1, 1, params.slots)
        L = params.max_level
        _B16["cts"] = (ckks.encrypt(ckks.encode(v1, params, L), ks, np.random.default_rng(77)),
                       ckks.encrypt(ckks.encode(v2, params, L), ks, np.random.default_rng(78)))
    return _B16["cts"]


def test_deska_launch_shapes_batched_galois(golden_hashes):
    """The launch-shape knobs of the key switch at desk-A (TMA inner product
    shapes, the fused ModDown combine, the pipelined FP64 chunk pass)
    (N=2^13: 32 tiles per limb, so the per-CTA Galois source block and the
    s_in remap for batch entries >= 1 are exercised) with non-trivial
    Galois elements: every variant gives the shipped residues, and entry 0
    of the batch equals the reference's rotate-by-1 digest."""
    import torch
    from paper_2310_16530_b200 import _native, ckks
    gold = golden_hashes["deskA"]
    params = ckks.desk_a()
    ks = ckks.keygen(params, np.random.default_rng(gold["key_seed"]), rotations=gold["rotations"])
    vrng = np.random.default_rng(12345)
    v1 = vrng.uniform(-1, 1, params.slots)
    v2 = vrng.uniform(-1, 1, params.slots)
    L = params.max_level
    ct1 = ckks.encrypt(ckks.encode(v1, params, L), ks, np.random.default_rng(77))
    ct2 = ckks.encrypt(ckks.encode(v2, params, L), ks, np.random.default_rng(78))
    batch = ckks.stack([ct1, ct2, ct1, ct2, ct2])
    steps = [1, 8, 64, 2048]
    defaults = {"ks_tpb": 128, "ks_stages": 3, "ks_tma_min": 2, "md_fuse": 0, "ntt_pipe": 1, "ks_tma3": 0,
                "fbc_fast": 1, "ntt_split": 1, "ntt_fork": 1, "fbc_fork": 1,
                "ks_rots": 1, "ks_rots_min_nb": 1, "ks96": 1, "ntt_occupancy": 1}
    variants = [{"ks_tpb": 256}, {"ks_stages": 4}, {"ks_tpb": 256, "ks_stages": 4}, {"ks_tma_min": 1},
                {"md_fuse": 1}, {"ntt_pipe": 0}, {"md_fuse": 1, "ks_tma_min": 1}, {"ks_tma3": 1}, {"ks_tma3": 2},
                {"fbc_fast": 0}, {"ntt_split": 2}, {"ntt_fork": 0}, {"fbc_fork": 0},
                {"ntt_fork": 0, "fbc_fork": 0, "mac3_fork": 0},
                {"ks_rots": 0}, {"ks_rots_min_nb": 2}, {"ks_stages": 4, "ks_rots": 1},
                {"ks96": 0}, {"ks96": 0, "ks_rots": 0}, {"ntt_occupancy": 0}, {"ntt_occupancy": 2}]

    def run():
        outs = [r.data.clone() for r in ckks.rotate_many(batch, steps, ks)]
        torch.cuda.synchronize()
        return outs

    for k, v in defaults.items():
        _native.set_option(k, v)
    want = run()
    assert h(np.stack(ckks.Ciphertext(want[0][0], ct1.scale, ct1.n, params).host_residues())) == gold["rot"]["1"]
    assert h(np.stack(ckks.Ciphertext(want[3][0], ct1.scale, ct1.n, params).host_residues())) == gold["rot"]["2048"]
    try:
        for var in variants:
            for k, v in var.items():
                _native.set_option(k, v)
            got = run()
            assert all(torch.equal(a, b) for a, b in zip(got, want)), var
            for k, v in defaults.items():
                _native.set_option(k, v)
    finally:
        for k, v in defaults.items():
            _native.set_option(k, v)
