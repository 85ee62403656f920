"""Layer-function parity on the reference's packing-unit setup
(test_packing.py:74-119: pack-unit N=512, L=7, K=2): every HyPHEN layer
function the ResNet20 path executes -- stride-2 conv in both directions,
convs at the doubled gap, downsample on both formats, the fixed-layout
baseline conv, the AESPA activation, pooling and the dense head -- and the
graph-level cost_report_compare reproduce the reference's residues bit for
bit, with identical op tallies and decrypted values (digests frozen by
tests/golden/make_golden.py gen_packing from the unmodified reference)."""

import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def h(arr) -> str:
    a = np.ascontiguousarray(np.asarray(arr, dtype=np.uint64))
    return hashlib.sha256(a.astype("<u8").tobytes()).hexdigest()


def _cts(x):
    return h(np.stack([np.stack(c.host_residues()) for c in x.cts]))


@pytest.fixture(scope="module")
def gold(golden_hashes):
    return golden_hashes["packing"]


@pytest.fixture(scope="module")
def setup(gold):
    from paper_2310_16530_b200 import ckks
    from paper_2310_16530_b200 import packing as P
    params = ckks.CkksParams.build("pack-unit", 512, 50, 40, 7, 50, 2)
    assert [m.q for m in params.q_mods] == gold["params"]["q"]
    A, B = P.FORMAT_A, P.FORMAT_B
    f = {"m4A": P.PackingFormat(A, 4, 1, 16), "m4B": P.PackingFormat(B, 4, 1, 16),
         "m2A": P.PackingFormat(A, 2, 1, 16), "m2B": P.PackingFormat(B, 2, 1, 16),
         "m2A2": P.PackingFormat(A, 2, 2, 16), "m2B2": P.PackingFormat(B, 2, 2, 16)}
    w4, w2 = np.ones((4, 4, 3, 3)), np.ones((2, 2, 3, 3))
    sh4, sh2 = P.TensorShape(4, 4, 4), P.TensorShape(2, 4, 4)
    layers = [
        (P.ConvLayerSpec(w4, 1, f["m4A"], f["m4B"]), sh4, False),
        (P.ConvLayerSpec(w4, 1, f["m4A"], f["m4A"]), sh4, True),
        (P.ConvLayerSpec(w2, 2, f["m2A"], f["m2B2"]), sh2, False),
        (P.ConvLayerSpec(w2, 2, f["m2B"], f["m2A2"]), sh2, False),
        (P.ConvLayerSpec(w2, 1, f["m2B2"], f["m2A2"]), P.TensorShape(2, 2, 2), False),
        (P.ConvLayerSpec(w2, 1, f["m2A2"], f["m2B2"]), P.TensorShape(2, 2, 2), False),
    ]
    steps = set()
    for layer, shape, fixed in layers:
        steps |= P.conv_rotation_steps(layer, shape, params.slots, fixed=fixed)
    steps |= P.pool_fc_rotation_steps(sh4, f["m4A"], params.slots, 4, 3)
    steps |= P.pool_fc_rotation_steps(sh4, f["m4B"], params.slots, 4, 3)
    assert sorted(steps) == gold["steps"]
    ks = ckks.keygen(params, np.random.default_rng(gold["key_seed"]), rotations=sorted(steps))
    return params, ks, f


def _check(gold, name, x_in, y, tally=None, ks=None):
    from paper_2310_16530_b200 import packing as P
    g = gold[name]
    assert _cts(x_in) == g["input"], f"{name}: input"
    if hasattr(y, "cts"):
        assert [y.fmt.variant, y.fmt.multiplex, y.fmt.gap, y.fmt.span] == g["fmt"]
        assert [y.shape.c, y.shape.h, y.shape.w] == g["shape"]
        assert _cts(y) == g["output"], f"{name}: output residues differ from the reference"
        assert [float(v) for v in P.decrypt_tensor(y, ks).ravel()] == g["dec"]
    else:
        assert h(np.stack(y.host_residues())) == g["output"], f"{name}: output residues differ"
    assert y.level == g["level"] and y.scale == g["scale"]
    if tally is not None:
        assert tally.as_dict() == g["tally"], f"{name}: op tally"


@pytest.mark.parametrize("name,seed,fin,fout", [("stride2_a2b", 11, "m2A", "m2B2"),
                                                ("stride2_b2a", 13, "m2B", "m2A2")])
def test_stride2_conv(gold, setup, name, seed, fin, fout):
    from paper_2310_16530_b200 import packing as P
    params, ks, f = setup
    rng = np.random.default_rng(seed)
    t = rng.standard_normal((2, 4, 4))
    w = rng.standard_normal((2, 2, 3, 3)) * 0.4
    b = rng.standard_normal(2) * 0.2
    x = P.encrypt_tensor(t, f[fin], ks, rng, params.max_level)
    tally = P.OpTally()
    y = P.conv2d(x, P.ConvLayerSpec(w, 2, f[fin], f[fout], bias=b), ks, tally)
    _check(gold, name, x, y, tally, ks)


def test_conv_at_doubled_gap(gold, setup):
    from paper_2310_16530_b200 import packing as P
    params, ks, f = setup
    rng = np.random.default_rng(12)
    t = rng.standard_normal((2, 4, 4))
    w = rng.standard_normal((2, 2, 3, 3)) * 0.4
    x = P.encrypt_tensor(t, f["m2A"], ks, rng, params.max_level)
    mid = P.conv2d(x, P.ConvLayerSpec(w, 2, f["m2A"], f["m2B2"]), ks)
    tally = P.OpTally()
    out = P.conv2d(mid, P.ConvLayerSpec(w, 1, f["m2B2"], f["m2A2"]), ks, tally)
    _check(gold, "gap2_b2a", mid, out, tally, ks)
    tally = P.OpTally()
    out2 = P.conv2d(out, P.ConvLayerSpec(w, 1, f["m2A2"], f["m2B2"]), ks, tally)
    _check(gold, "gap2_a2b", out, out2, tally, ks)


def test_fixed_baseline(gold, setup):
    from paper_2310_16530_b200 import packing as P
    params, ks, f = setup
    rng = np.random.default_rng(21)
    t = rng.standard_normal((4, 4, 4))
    w = rng.standard_normal((4, 4, 3, 3)) * 0.4
    b = rng.standard_normal(4) * 0.2
    xa = P.encrypt_tensor(t, f["m4A"], ks, rng, params.max_level)
    t_alt, t_fix = P.OpTally(), P.OpTally()
    y_alt = P.conv2d(xa, P.ConvLayerSpec(w, 1, f["m4A"], f["m4B"], bias=b), ks, t_alt)
    y_fix = P.conv2d_fixed_baseline(xa, P.ConvLayerSpec(w, 1, f["m4A"], f["m4A"], bias=b), ks, t_fix)
    _check(gold, "alt_a2b", xa, y_alt, t_alt, ks)
    _check(gold, "fixed", xa, y_fix, t_fix, ks)
    rng = np.random.default_rng(22)
    t = rng.standard_normal((4, 4, 4))
    w = rng.standard_normal((4, 4, 3, 3)) * 0.4
    x = P.encrypt_tensor(t, f["m4A"], ks, rng, 4)
    tally = P.OpTally()
    y = P.conv2d_fixed_baseline(x, P.ConvLayerSpec(w, 1, f["m4A"], f["m4A"]), ks, tally)
    _check(gold, "fixed_l4", x, y, tally, ks)


def test_activation(gold, setup):
    from paper_2310_16530_b200 import packing as P
    from paper_2310_16530_b200.aespa import AespaChannelParams, fold_channels, hermite_coeffs
    params, ks, f = setup
    rng = np.random.default_rng(31)
    t = rng.standard_normal((4, 4, 4))
    chans = [AespaChannelParams(gamma=0.8 + 0.1 * i, beta=0.05 * i, mu=(0.1, -0.05, 0.02),
                                sigma2=(1.1, 0.9, 1.3)) for i in range(4)]
    quads = fold_channels(chans, hermite_coeffs(2))
    x = P.encrypt_tensor(t, f["m4B"], ks, rng, 4)
    tally = P.OpTally()
    y = P.he_activation(x, quads, ks, tally)
    _check(gold, "act", x, y, tally, ks)


@pytest.mark.parametrize("name,seed,fmt", [("down_a", 32, "m2A"), ("down_b", 36, "m2B")])
def test_downsample(gold, setup, name, seed, fmt):
    from paper_2310_16530_b200 import packing as P
    params, ks, f = setup
    rng = np.random.default_rng(seed)
    t = rng.standard_normal((2, 4, 4))
    x = P.encrypt_tensor(t, f[fmt], ks, rng, 4)
    tally = P.OpTally()
    y = P.downsample(x, ks, tally)
    _check(gold, name, x, y, tally, ks)
    assert np.abs(P.decrypt_tensor(y, ks) - t[:, ::2, ::2]).max() < 1e-5


@pytest.mark.parametrize("variant", ["A", "B"])
def test_pool_and_fc(gold, setup, variant):
    from paper_2310_16530_b200 import packing as P
    params, ks, f = setup
    rng = np.random.default_rng(34)
    t = rng.standard_normal((4, 4, 4))
    wfc = rng.standard_normal((3, 4)) * 0.5
    bfc = rng.standard_normal(3) * 0.2
    fmt = P.PackingFormat(variant, 4, 1, 16)
    x = P.encrypt_tensor(t, fmt, ks, rng, 4)
    tally = P.OpTally()
    pooled = P.avgpool_global(x, ks, tally)
    _check(gold, f"pool_{variant}", x, pooled, tally, ks)
    tally = P.OpTally()
    out = P.fully_connected(pooled, wfc, bfc, ks, tally)
    _check(gold, f"fc_{variant}", pooled, out, tally, ks)
    assert [float(v) for v in P.read_logits(out, 3, fmt, ks)] == gold[f"fc_{variant}"]["logits"]


def test_cost_report_compare(gold):
    """graph.py:637-682 on the reference's own graph-unit fixture
    (test_graph.py:86-117, 504-508): rotation counts per conv for both
    layouts, and the decrypted difference between the two encrypted paths
    (a float of two bit-exact decodes, so compared exactly)."""
    from paper_2310_16530_b200 import ckks, graph
    g0 = gold["compare"]
    gp = ckks.CkksParams.build("graph-unit", 2048, 50, 40, 11, 50, 2)
    fx = graph.gen_fixture("tiny-cnn", 7, gp, golden_count=2)
    g = graph.build_graph("tiny-cnn", fx, multiplex=4)
    steps = sorted(graph.required_rotation_steps(g, gp.slots, include_fixed=True))
    assert steps == g0["steps"]
    gks = ckks.keygen(gp, np.random.default_rng(g0["key_seed"]), rotations=steps)
    plan = graph.plan_levels(g, gp.max_level)
    x = np.array(fx["golden"][0]["input"])
    rep = graph.cost_report_compare(g, plan, x, gks, np.random.default_rng(9))
    assert rep == g0["report"]
