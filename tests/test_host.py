"""CPU-only tests: the C ABI boundary (load, exported symbols, error
mapping), parameter construction, and every host-side computation whose
floats feed encoded masks (AESPA folds, fixtures, layouts, planner,
rotation-step enumeration), against goldens frozen from the reference."""

import hashlib
import itertools
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def hf(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.float64)).astype("<f8").tobytes()).hexdigest()


# ---------------------------------------------------------------------------
# boundary
# ---------------------------------------------------------------------------

def test_abi_library_exports_every_header_symbol():
    from paper_2310_16530_b200 import _native
    lib = _native.load()  # loads without a GPU (cudart is static)
    header = (ROOT / "include" / "hcnn_b200.h").read_text()
    declared = set(re.findall(r"\b(hcnn_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    assert declared == set(_native.SIGNATURES), declared ^ set(_native.SIGNATURES)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.hcnn_abi_version() == 1


def test_abi_status_codes_map_to_reference_exceptions():
    import ctypes
    from paper_2310_16530_b200 import _native
    from paper_2310_16530_b200.errors import ParameterError, LevelError, HcnnError
    lib = _native.load()
    h = ctypes.c_void_p()
    q = _native.u64_array([17])
    rc = lib.hcnn_ctx_create(ctypes.byref(h), 0, 3, q, 1, None, 0)  # N=3: rejected before any CUDA call
    assert rc == 1
    with pytest.raises(ParameterError):
        _native.check(rc)
    with pytest.raises(LevelError):
        _native.check(4)
    assert issubclass(_native.NativeError if hasattr(_native, "NativeError") else HcnnError, HcnnError)


def test_no_cuda_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2310_16530_b200 import ckks
    from paper_2310_16530_b200.errors import NativeError
    params = ckks.CkksParams.build("t", 256, 50, 40, 2, 50, 2)
    with pytest.raises(NativeError):
        params.ctx


# ---------------------------------------------------------------------------
# parameters
# ---------------------------------------------------------------------------

def test_presets_match_reference_chains(golden_hashes):
    from paper_2310_16530_b200 import ckks
    a = ckks.desk_a()
    g = golden_hashes["deskA"]["params"]
    assert [m.q for m in a.q_mods] == g["q"] and [m.q for m in a.p_mods] == g["p"]
    b = ckks.bench16()
    g = golden_hashes["bench16"]["params"]
    assert [m.q for m in b.q_mods] == g["q"] and [m.q for m in b.p_mods] == g["p"]
    assert a.dnum == 6 and ckks.desk_b().dnum == 5 and b.dnum == 7
    assert a.alpha == 2 and a.max_level == 10 and a.slots == 4096


def test_prime_search_properties():
    from paper_2310_16530_b200.ring import find_ntt_primes, is_prime
    n = 1 << 13
    qs = find_ntt_primes(n, 40, 4, alternate=True)
    assert [q > 1 << 40 for q in qs] == [False, True, False, True]
    for q in qs:
        assert q % (2 * n) == 1 and is_prime(q)
    first = find_ntt_primes(64, 30, 2)
    assert not set(first) & set(find_ntt_primes(64, 30, 2, avoid=first))
    assert [p for p in range(2, 200) if is_prime(p)] == [p for p in range(2, 200)
                                                        if all(p % d for d in range(2, p))]


def test_params_validation():
    from paper_2310_16530_b200 import ckks
    from paper_2310_16530_b200.errors import ParameterError
    good = ckks.desk_a()
    with pytest.raises(ParameterError):
        ckks.CkksParams("bad", 12, good.q_mods, good.p_mods, 2.0 ** 40)
    with pytest.raises(ParameterError):
        ckks.CkksParams("bad", good.n, good.q_mods, good.q_mods[:1], 2.0 ** 40)
    with pytest.raises(ParameterError):
        ckks.params_by_name("desk-Z")


def test_galois_and_rotation_plan():
    from paper_2310_16530_b200 import ckks
    from paper_2310_16530_b200.errors import KeyError_
    assert ckks.galois_element(1, 16) == 5 and ckks.galois_element(8, 16) == 1
    assert ckks.rotation_plan(7, (1, 2, 4), 512) == [4, 2, 1]
    assert ckks.rotation_plan(0, (1, 2, 4), 512) == []
    with pytest.raises(KeyError_):
        ckks.rotation_plan(9, (2, 4), 512)


def test_encode_coefficients_known_answer():
    from paper_2310_16530_b200 import ckks
    p = ckks.desk_a()
    ints = ckks.encode_coeffs(np.ones(p.slots), p, 0, p.delta)
    assert abs(int(ints[0]) - 2 ** 40) <= 1 and int(np.max(np.abs(ints[1:]))) <= 1


# ---------------------------------------------------------------------------
# AESPA, fixtures, folds, plans, layouts (golden_hashes["host"])
# ---------------------------------------------------------------------------

def test_hermite_coefficients(golden_hashes):
    from paper_2310_16530_b200 import aespa
    g = golden_hashes["host"]
    assert list(aespa.hermite_coeffs(2).f_hat) == g["hermite2"]
    assert list(aespa.hermite_coeffs(4).f_hat) == g["hermite4"]
    f = aespa.hermite_coeffs(4).f_hat
    assert abs(f[0] - 0.3989422804014327) < 1e-15 and abs(f[1] - 0.5) < 1e-12
    assert abs(f[2] - 0.2820947917738781) < 1e-15 and abs(f[3]) < 1e-12


def test_fold_matches_expansion():
    from paper_2310_16530_b200 import aespa
    basis = aespa.hermite_coeffs(2)
    rng = np.random.default_rng(0xACC3)
    for _ in range(50):
        ch = aespa.AespaChannelParams(float(rng.uniform(0.5, 1.5)), float(rng.uniform(-1, 1)),
                                      tuple(rng.uniform(-0.5, 0.5, 3)), tuple(rng.uniform(0.5, 2.0, 3)), 1e-5)
        qa = aespa.fold_quadratic(ch, basis)
        x = rng.uniform(-6, 6, 256)
        assert np.max(np.abs(qa(x) - aespa.aespa_eval_plain(x, ch, basis))) < 1e-9


@pytest.mark.parametrize("key", ["tiny-cnn|42|desk-B", "basic-block-stack(1)|21|desk-A",
                                 "basic-block-stack(2)|7|desk-A"])
def test_fixture_fold_plan_steps(golden_hashes, key):
    from paper_2310_16530_b200 import ckks, graph
    g = golden_hashes["host"]["fixtures"][key]
    topo, seed, pname = key.split("|")
    params = ckks.params_by_name(pname)
    fx = graph.gen_fixture(topo, int(seed), params, golden_count=2)
    assert graph.weights_digest(fx) == g["digest"]
    assert fx["golden"] == g["golden"]
    gr = graph.build_graph(topo, fx, multiplex=8)
    assert graph.plan_levels(gr, params.max_level).as_dict() == g["plan"]
    assert graph.plan_levels(gr, 7, 5).as_dict() == g["plan_t5"]
    assert sorted(graph.required_rotation_steps(gr, params.slots)) == g["steps"]
    assert sorted(graph.required_rotation_steps(gr, params.slots, include_fixed=True)) == g["steps_fixed"]
    for L, row in zip(gr.layers, g["layers"]):
        assert L.kind == row["kind"] and L.fold_forward == row["fold_forward"]
        if L.kind == "conv":
            assert hf(L.spec.effective_weights()) == row["eff_w"]
            assert (None if L.spec.bias_map is None else hf(L.spec.bias_map)) == row["bias_map"]
            assert L.spec.low_scale_out == row["low_scale_out"]
        if L.kind == "act":
            assert [[q.a, q.b, q.c] for q in L.quads] == row["quads"]
    x = np.asarray(fx["golden"][0]["input"])
    out, _ = graph.execute(gr, graph.plan_levels(gr, params.max_level), x, mode="plaintext-ref")
    assert hf(out) == g["plain_out"]


def test_layouts(golden_hashes):
    from paper_2310_16530_b200 import packing
    for key, g in golden_hashes["host"]["layouts"].items():
        parts = key.split("|")
        fa = (parts[0], int(parts[1]), int(parts[2]), int(parts[3]))
        shape = tuple(int(v) for v in parts[4:7])
        slots = int(parts[7])
        fmt = packing.PackingFormat(*fa)
        t = np.asarray(g["input"])
        vecs = packing.pack(t, fmt, slots)
        assert [hf(v) for v in vecs] == g["pack"]
        lay = packing.Layout(fmt, packing.TensorShape(*shape), slots)
        assert [hf(lay.occupancy(i)) for i in range(lay.n_cts)] == g["occ"]
        assert np.array_equal(packing.unpack(vecs, fmt, packing.TensorShape(*shape), slots), t)
        assert sorted(packing.pool_fc_rotation_steps(packing.TensorShape(*shape), fmt, slots, shape[0], 3)) \
            == g["pool_fc_steps"]


def test_format_b_stagger_table():
    """FormatB m=4, span 4, 4x2x2 (the reference's frozen slot table,
    tests/data/format_b_m4_slots.txt): channel c lives at block c of replica
    0 and at block (c-1) mod 4 of replica 1."""
    from paper_2310_16530_b200 import packing
    fmt = packing.PackingFormat("B", 4, 1, 4)
    t = np.arange(16, dtype=float).reshape(4, 2, 2) + 1
    vec = packing.pack(t, fmt, 32)[0]
    for c in range(4):
        for y in range(2):
            for x in range(2):
                v = t[c, y, x]
                assert vec[c * 4 + y * 2 + x] == v
                assert vec[16 + ((c - 1) % 4) * 4 + y * 2 + x] == v


@pytest.mark.parametrize("variant,m,span,shape,slots", [
    ("B", 4, 1024, (16, 32, 32), 32768), ("A", 4, 1024, (16, 32, 32), 32768), ("B", 4, 1024, (64, 8, 8), 32768),
    ("B", 2, 16, (4, 4, 4), 64), ("A", 4, 16, (4, 4, 4), 64), ("B", 4, 16, (4, 4, 4), 64)])
def test_slot_period_is_a_true_period(variant, m, span, shape, slots):
    """packing.slot_period: every packed vector (and every mask built from
    the layout) repeats with the reported period -- the premise of pairing
    two ciphertexts per bootstrap."""
    from paper_2310_16530_b200 import packing
    fmt = packing.PackingFormat(variant, m, 1, span)
    per = packing.slot_period(fmt, packing.TensorShape(*shape), slots)
    t = np.random.default_rng(0).standard_normal(shape)
    lay = packing.Layout(fmt, packing.TensorShape(*shape), slots)
    for v in packing.pack(t, fmt, slots) + [lay.channel_values(0, np.arange(shape[0]) + 1.0)]:
        assert np.array_equal(v, np.roll(v, per))
    if per < slots:
        assert slots % per == 0
    if variant == "B" and slots // (m * span) >= 2 * m:
        assert per * 2 <= slots


def _exhaustive_refreshes(costs, max_level, target):
    n = len(costs)
    entry0 = min(max_level, sum(costs))
    for r in range(n + 1):
        for pts in itertools.combinations(range(n), r):
            lvl = entry0
            ok = True
            for i in range(n):
                if i in pts:
                    lvl = target
                if lvl < costs[i]:
                    ok = False
                    break
                lvl -= costs[i]
            if ok:
                return r
    raise AssertionError


def test_planner_optimal_vs_exhaustive():
    """Acceptance gate 6 (test_acceptance.py:384-408) on 120 random chains."""
    from paper_2310_16530_b200 import graph, packing
    rng = np.random.default_rng(0xACC6)
    fmt = packing.PackingFormat("A", 4, 1, 64)
    shape = packing.TensorShape(1, 8, 8)
    kinds = {0: "avgpool", 1: "act", 2: "conv"}
    for _ in range(120):
        n = int(rng.integers(1, 13))
        ml = int(rng.integers(4, 9))
        costs = [int(c) for c in rng.choice((0, 1, 2), size=n, p=(0.2, 0.3, 0.5))]
        g = graph.HcnnGraph("synthetic", [graph.Layer(kind=kinds[c], name=f"l{i}") for i, c in enumerate(costs)],
                            shape, fmt, 4, True, (shape,) * n, (fmt,) * n, (1,) * n)
        plan = graph.plan_levels(g, ml)
        assert len(plan.refresh_points) == _exhaustive_refreshes(costs, ml, ml - 1)
        assert plan == graph.plan_levels(g, ml)


def test_conv_rotation_step_counts():
    """Closed-form tap / landing step sets (test_packing.py:292-306)."""
    from paper_2310_16530_b200 import packing
    A = packing.PackingFormat("A", 4, 1, 16)
    B = packing.PackingFormat("B", 4, 1, 16)
    shape = packing.TensorShape(4, 4, 4)
    w = np.ones((4, 4, 3, 3))
    ab = packing.conv_rotation_steps(packing.ConvLayerSpec(w, 1, A, B), shape, 256)
    assert len(ab) == 8 + 3
    ba = packing.conv_rotation_steps(packing.ConvLayerSpec(w, 1, B, A), shape, 256)
    assert len(ba) == 8 + 2
    fixed = packing.conv_rotation_steps(packing.ConvLayerSpec(w, 1, A, A), shape, 256, fixed=True)
    assert len(fixed) == 9 * 4 - 1


_SHIM_SCRIPT = r"""
import os, sys, traceback
import numpy as np
sys.path.insert(0, sys.argv[1])
from hcnn import ckks as rc, packing as rp, graph as rg        # the unmodified reference
from paper_2310_16530_b200 import ckks as gc, ring as gr, refshim
from paper_2310_16530_b200.errors import NativeError
orig_hmult, orig_ct = rc.hmult, rp.Ciphertext
refshim.enable(rc, rp, rg)
assert rc.hmult is gc.hmult and rc.rotate is gc.rotate and rc.encode is gc.encode
assert rp.Ciphertext is gc.Ciphertext and rg.Ciphertext is gc.Ciphertext
assert rp.to_mont_rows is gr.to_mont_rows and rp._zero_ct is refshim._zero_ct
params = rc.CkksParams.build("shim", 256, 50, 40, 4, 50, 2)
assert type(params) is gc.CkksParams
class KS:                                  # only .params is read before the first device call
    pass
ks = KS(); ks.params = params
fmt = rp.PackingFormat("A", 4, 1, 4)
try:
    rp.encrypt_tensor(np.zeros((4, 2, 2)), fmt, ks, np.random.default_rng(0), 2)
    raise SystemExit("expected NativeError: no CUDA device")
except NativeError:
    frames = [f.filename for f in traceback.extract_tb(sys.exc_info()[2])]
    assert any(f.endswith("hcnn/packing.py") for f in frames), frames          # the reference's layer code ...
    assert any("paper_2310_16530_b200" in f for f in frames), frames           # ... called into the engine
refshim.disable()
assert rc.hmult is orig_hmult and rp.Ciphertext is orig_ct
print("shim ok")
"""


def test_reference_side_shim_routes_reference_layers_into_the_engine(tmp_path):
    """refshim.enable patches the reference's hcnn.ckks / packing / graph
    (including the name-bound hooks), so the reference's own
    packing code calls this engine -- here, without a GPU, its loud
    NativeError proves the routing.  Runs only where /root/reference exists
    (the build container); the GPU box has no reference to patch."""
    import os
    import subprocess
    import sys
    src = Path("/root/reference/pkg/src")
    if not (src / "hcnn" / "packing.py").exists():
        pytest.skip("reference package not present")
    import torch
    if torch.cuda.is_available():
        pytest.skip("routing check relies on the no-device NativeError")
    env = dict(os.environ, NUMBA_CACHE_DIR=str(tmp_path / "numba"), HCNN_TEST_MODE="1",
               PYTHONPATH=str(ROOT) + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-c", _SHIM_SCRIPT, str(src)], cwd=tmp_path, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "shim ok" in r.stdout


def test_stack_views_and_image_batches():
    """ckks.stack / unstack and graph.stack_images / unstack_images are pure
    tensor bookkeeping (host-checkable): consecutive slices of one buffer
    stack without a copy (the conv planes' MAC buffer, packing._mac_multi),
    other members are copied; under ckks.image_batched(B) members are
    [B, 2, l+1, N] image batches that stack along the image axis and unstack
    into B-image chunks; stack_images / unstack_images round-trip."""
    import torch
    from paper_2310_16530_b200 import ckks, graph, packing
    buf = torch.arange(3 * 2 * 4 * 8, dtype=torch.int64).reshape(3, 2, 4, 8)
    cts = [ckks.Ciphertext(buf[i], 2.0, 8, None) for i in range(3)]
    s = ckks.stack(cts)
    assert s.batch == 3 and s.data.data_ptr() == buf.data_ptr()        # a view, no copy
    apart = [ckks.Ciphertext(buf[i].clone(), 2.0, 8, None) for i in (2, 0)]
    s2 = ckks.stack(apart)
    assert s2.data.data_ptr() != buf.data_ptr() and torch.equal(s2.data[0], buf[2])
    assert [torch.equal(u.data, buf[i]) for i, u in enumerate(ckks.unstack(s))] == [True] * 3
    with pytest.raises(Exception):
        ckks.stack([cts[0], ckks.Ciphertext(buf[1], 3.0, 8, None)])   # scales differ
    with ckks.image_batched(2):
        x = [ckks.Ciphertext(torch.full((2, 2, 4, 8), i, dtype=torch.int64), 2.0, 8, None) for i in range(3)]
        st = ckks.stack(x)
        assert st.data.shape == (6, 2, 4, 8)
        un = ckks.unstack(st)
        assert [u.data.shape for u in un] == [(2, 2, 4, 8)] * 3 and int(un[2].data[1, 1, 3, 7]) == 2
    imgs = [packing.PackedTensor(cts=[ckks.Ciphertext(torch.full((2, 4, 8), 10 * b + i, dtype=torch.int64),
                                                      2.0, 8, None) for i in range(2)], fmt="F", shape=(1, 2, 2))
            for b in range(3)]
    both = graph.stack_images(imgs)
    assert [c.data.shape for c in both.cts] == [(3, 2, 4, 8)] * 2
    back = graph.unstack_images(both)
    assert all(torch.equal(back[b].cts[i].data, imgs[b].cts[i].data) for b in range(3) for i in range(2))
