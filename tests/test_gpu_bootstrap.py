"""Homomorphic bootstrapping on the B200 (BASELINE config 3).
No reference exists (parity unpinned): checked by decrypt-and-compare
against the input slot values, stage by stage."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def boot12():
    from paper_2310_16530_b200 import bootstrap as bt, ckks
    cfg = bt.BootConfig(cts_stages=(4, 4, 3), stc_stages=(3, 4, 4))
    params = bt.boot_params("boot12", 1 << 12, 4, cfg)
    b = bt.Bootstrapper(params, cfg)
    ks = b.keygen(np.random.default_rng(7), rotations=[1])
    return params, cfg, b, ks


def test_mod_raise_and_cts(boot12):
    """After ModRaise + CoeffToSlot the slots hold (t_lo + i t_hi)/(2 q0 B)
    with t = m + q0*I, I small integers."""
    from paper_2310_16530_b200 import bootstrap as bt, ckks
    params, cfg, b, ks = boot12
    rng = np.random.default_rng(1)
    vals = rng.uniform(-1, 1, params.slots)
    ct = ckks.encrypt(ckks.encode(vals, params, 0), ks, rng)
    u, delta1 = b.coeff_to_slot(ct, ks)
    assert u.level == params.max_level - len(cfg.cts_stages)
    got = ckks.decode(ckks.decrypt(u, ks), params, imag_tol=None)  # real parts only
    # plaintext expectation from the coefficient vector of m' (scaled-up message)
    t = ckks.encode_coeffs(vals, params, 0, delta1).astype(float)
    n = params.slots
    br = bt.bit_reverse_perm(n)
    frac = (t[:n] / b.q0)[br]
    # real part of slot = (t_lo + q0 I)/(2 q0 B): the fractional offset must match mod 1/(2B)
    r = got * 2 * b.B
    assert np.max(np.abs((r - frac) - np.round(r - frac))) < 1e-6
    assert np.max(np.abs(np.round(r - frac))) <= cfg.k_bound


def test_bootstrap_round_trip(boot12):
    from paper_2310_16530_b200 import ckks
    params, cfg, b, ks = boot12
    rng = np.random.default_rng(2)
    vals = rng.uniform(-1, 1, params.slots)
    ct = ckks.encrypt(ckks.encode(vals, params, 2), ks, rng)
    out = b.bootstrap(ct, ks)
    assert out.level == b.output_level == params.max_level - cfg.depth()
    assert abs(out.scale - ct.scale) < 1e-6 * ct.scale
    got = ckks.decode(ckks.decrypt(out, ks), params, imag_tol=None)
    err = float(np.max(np.abs(got - vals)))
    print("bootstrap max abs error", err)
    assert err < 1e-3
    # the refreshed ciphertext keeps computing: square it
    sq = ckks.rescale(ckks.hmult(out, out, ks), params)
    got2 = ckks.decode(ckks.decrypt(sq, ks), params, imag_tol=None)
    assert np.max(np.abs(got2 - vals * vals)) < 2e-3


def test_double_hoisted_matches_single_hoisted():
    """The double-hoisted linear transforms (Q||P babies and accumulator, one
    ModDown per giant) decrypt to the single-hoisted result."""
    from paper_2310_16530_b200 import bootstrap as bt, ckks
    outs = []
    for dh in (False, True):
        rng = np.random.default_rng(5)  # same keys, same ciphertext for both
        cfg = bt.BootConfig(cts_stages=(4, 4, 3), stc_stages=(3, 4, 4), double_hoist=dh)
        params = bt.boot_params("boot12", 1 << 12, 4, cfg)
        b = bt.Bootstrapper(params, cfg)
        ks = b.keygen(np.random.default_rng(7), rotations=[1])
        vals = np.random.default_rng(9).uniform(-1, 1, params.slots)
        ct = ckks.encrypt(ckks.encode(vals, params, 2), ks, rng)
        u, _ = b.coeff_to_slot(ct, ks)
        outs.append(ckks.decode(ckks.decrypt(u, ks), params, imag_tol=None))
        got = ckks.decode(ckks.decrypt(b.bootstrap(ct, ks), ks), params, imag_tol=None)
        assert np.max(np.abs(got - vals)) < 1e-3
    assert np.max(np.abs(outs[0] - outs[1])) < 1e-6


def test_bootstrap_many_matches_single(boot12):
    """The batched bootstrap (one pass over all members) is entry-wise
    bit-identical to bootstrapping each ciphertext alone."""
    import torch
    from paper_2310_16530_b200 import ckks
    params, cfg, b, ks = boot12
    rng = np.random.default_rng(3)
    cts = [ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, 1), ks, rng) for _ in range(3)]
    many = b.bootstrap_many(cts, ks)
    for ct, m in zip(cts, many):
        one = b.bootstrap(ct, ks)
        assert m.level == one.level and m.scale == one.scale
        assert torch.equal(m.data, one.data)


def test_bootstrap_pairs_round_trip(boot12):
    """Two half-periodic messages (even polynomials) share one bootstrap and
    come back separated, each within the single-bootstrap precision."""
    from paper_2310_16530_b200 import ckks
    params, cfg, b, ks = boot12
    rng = np.random.default_rng(4)
    h = params.slots // 2
    vals = [np.tile(rng.uniform(-1, 1, h), 2) for _ in range(4)]
    cts = [ckks.encrypt(ckks.encode(v, params, 1), ks, rng) for v in vals]
    outs = b.bootstrap_pairs([(cts[0], cts[1]), (cts[2], cts[3])], ks)
    got = [o for pair in outs for o in pair]
    for v, ct, o in zip(vals, cts, got):
        assert o.level == b.output_level and abs(o.scale - ct.scale) < 1e-9 * ct.scale
        err = float(np.max(np.abs(ckks.decode(ckks.decrypt(o, ks), params, imag_tol=None) - v)))
        assert err < 1e-3, err


def test_packed_refresh_of_sparse_layout(boot12):
    """Refresh of a gap-2 FormatB tensor: 2 ciphertexts interleaved into one
    (graph.refresh_shifts), paired, bootstrapped, moved back -- every
    occupied slot of every replica comes back within bootstrap precision."""
    from paper_2310_16530_b200 import bootstrap as bt, ckks, graph, packing
    params, cfg, b, ks0 = boot12
    fmt = packing.PackingFormat("B", 2, 2, 256)
    shape = packing.TensorShape(8, 8, 8)
    shifts = graph.refresh_shifts(fmt, shape, params.slots)
    assert shifts == [0, 1, 16, 17]
    ks = b.keygen(np.random.default_rng(7), rotations=sorted({s for s in shifts if s} | {-s % params.slots for s in shifts}))
    rng = np.random.default_rng(8)
    x = rng.uniform(-1, 1, (8, 8, 8))
    pt = packing.encrypt_tensor(x, fmt, ks, rng, 2)
    assert len(pt.cts) == 4
    tally = packing.OpTally()
    out = graph._refresh_tensors([pt], ks, b.output_level, tally, cache={})[0]
    assert tally.refreshes == 4
    lay = packing.Layout(fmt, shape, params.slots)
    want = packing.pack(x, fmt, params.slots)
    for j, ct in enumerate(out.cts):
        assert ct.level == b.output_level and abs(ct.scale - pt.cts[j].scale) < 1e-9 * ct.scale
        got = ckks.decode(ckks.decrypt(ct, ks), params, imag_tol=None)
        occ = lay.occupancy(j) > 0
        assert np.max(np.abs(got[occ] - want[j][occ])) < 2e-3


def test_graph_refresh_slot_bootstraps():
    """Two stacked basic blocks need a refresh between them (6 levels each):
    the executor's refresh slot bootstraps (no decryption), and the result
    matches the plaintext mirror."""
    from paper_2310_16530_b200 import bootstrap as bt, graph, packing
    cfg = bt.BootConfig(cts_stages=(4, 4, 4), stc_stages=(4, 4, 4))
    params = bt.boot_params("boot13", 1 << 13, 6, cfg)
    b = bt.Bootstrapper(params, cfg)
    fx = graph.gen_fixture("basic-block-stack(2)", 5, params)
    g = graph.build_graph("basic-block-stack(2)", fx, multiplex=8)
    plan = graph.plan_levels(g, b.output_level, refresh_target=b.output_level)
    assert plan.refresh_points
    ks = b.keygen(np.random.default_rng(9), rotations=sorted(graph.required_rotation_steps(g, params.slots)))
    x = np.asarray(fx["golden"][0]["input"])
    packed = packing.encrypt_tensor(x, g.input_format, ks, np.random.default_rng(4), plan.entry_levels[0])
    out, rep = graph.execute(g, plan, packed, ks, "encrypted")
    assert rep.totals().refreshes > 0
    dec = packing.decrypt_tensor(out, ks)
    ref, _ = graph.execute(g, plan, x, mode="plaintext-ref")
    err = float(np.max(np.abs(dec - ref)))
    print("stack(2) with bootstrapping: max abs err", err)
    assert err < 1e-3


def test_fused_moddown_rescale(boot12):
    """hcnn_moddown_rescale_batch divides a Q||P ciphertext by P q_l in one
    base conversion: on the lifted P*ct it decrypts to rescale(ct) up to the
    rounding, for a single ciphertext and a batch."""
    from paper_2310_16530_b200 import ckks
    from paper_2310_16530_b200.ckks import Ciphertext
    params, cfg, b, ks = boot12
    rng = np.random.default_rng(21)
    lvl = params.max_level - 1
    cts = [ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, lvl), ks, rng) for _ in range(3)]
    for ct in (cts[0], ckks.stack(cts)):
        want = ckks.rescale(ct, params)
        got = Ciphertext(params.ctx.moddown_rescale(b._lift_ext(ct), lvl), want.scale, ct.n, params)
        assert got.level == want.level
        for g, w in zip(ckks.unstack(got), ckks.unstack(want)):
            dg = ckks.decode(ckks.decrypt(g, ks), params, imag_tol=None)
            dw = ckks.decode(ckks.decrypt(w, ks), params, imag_tol=None)
            assert np.max(np.abs(dg - dw)) < 1e-7


def test_fused_hmult_rescale(boot12):
    """hcnn_hmult_rescale_batch == rescale(hmult(a, b)) up to one rounding
    (decrypt-and-compare, single ciphertext and batch)."""
    from paper_2310_16530_b200 import ckks
    from paper_2310_16530_b200.ckks import Ciphertext
    params, cfg, b, ks = boot12
    rng = np.random.default_rng(22)
    lvl = params.max_level
    # EvalMod multiplies at scale ~ q_l, so the product keeps scale ~ q_l after the
    # rescale; at Delta = 2^40 it would land at 2^22 and the two paths' (different)
    # rounding points alone differ by ~1e-4 in the slots
    sc = float(params.q_mods[lvl].q)
    xs = [ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, lvl, sc), ks, rng) for _ in range(3)]
    ys = [ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, lvl, sc), ks, rng) for _ in range(3)]
    for x, y in ((xs[0], ys[0]), (ckks.stack(xs), ckks.stack(ys))):
        want = ckks.rescale(ckks.hmult(x, y, ks), params)
        got = Ciphertext(params.ctx.hmult_rescale(x.data, y.data, lvl, ks.rlk.rows_b, ks.rlk.rows_a), want.scale,
                         x.n, params)
        for g, w in zip(ckks.unstack(got), ckks.unstack(want)):
            dg = ckks.decode(ckks.decrypt(g, ks), params, imag_tol=None)
            dw = ckks.decode(ckks.decrypt(w, ks), params, imag_tol=None)
            assert np.max(np.abs(dg - dw)) < 1e-6


def test_boot16_full_slot_precision():
    """BASELINE cfg 3 at full size: N=2^16, 32768 slots, the bench's
    boot16 chain.  A single bootstrap and a 2-entry batched bootstrap
    (entry-wise identical to it) keep >= 19 bits of precision, and the
    CUDA-graph replay bench.py times gives the eager residues."""
    import torch
    from paper_2310_16530_b200 import bootstrap as bt, ckks
    cfg = bt.BootConfig()
    params = bt.boot_params("boot16", 1 << 16, 8, cfg)
    b = bt.Bootstrapper(params, cfg)
    ks = b.keygen(np.random.default_rng(16), rotations=[1])
    rng = np.random.default_rng(3)
    vals = [rng.uniform(-1, 1, params.slots) for _ in range(2)]
    cts = [ckks.encrypt(ckks.encode(v, params, 0), ks, rng) for v in vals]
    single = b.bootstrap(cts[0], ks)
    assert single.level == b.output_level
    err = float(np.max(np.abs(ckks.decode(ckks.decrypt(single, ks), params, imag_tol=None) - vals[0])))
    print("boot16 bits", -np.log2(err))
    assert -np.log2(err) >= 19.0
    x = ckks.stack(cts)
    batch = ckks.unstack(b.bootstrap(x, ks))
    assert torch.equal(batch[0].data, single.data)
    err1 = float(np.max(np.abs(ckks.decode(ckks.decrypt(batch[1], ks), params, imag_tol=None) - vals[1])))
    assert -np.log2(err1) >= 19.0
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = b.bootstrap(x, ks)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(ckks.unstack(out)[0].data, single.data)
    assert torch.equal(ckks.unstack(out)[1].data, batch[1].data)


def test_resnet20_chain_bootstrap_precision():
    """The ResNet20 workload's own chain (workloads.resnet20_params: 30
    q-limbs, 5 specials, EvalMod degree RESNET20_EVALMOD_DEGREE) bootstraps
    full-slot U(-1,1) inputs to >= 19 bits -- the precision the bench's
    inference runs at (degree 31 measured 8 bits: tools/boot_precision.py)."""
    from paper_2310_16530_b200 import bootstrap as bt, ckks, workloads
    cfg = workloads.resnet20_boot_config()
    params = workloads.resnet20_params("resnet20-16", workloads.resnet20_app_levels(cfg), cfg)
    assert params.max_level + 1 == workloads.RESNET20_Q_LIMBS and len(params.p_mods) == workloads.RESNET20_N_SPECIAL
    b = bt.Bootstrapper(params, cfg)
    ks = b.keygen(np.random.default_rng(20), rotations=[])
    rng = np.random.default_rng(5)
    v = rng.uniform(-1, 1, params.slots)
    out = b.bootstrap(ckks.encrypt(ckks.encode(v, params, 0), ks, rng), ks)
    assert out.level == b.output_level
    err = float(np.max(np.abs(ckks.decode(ckks.decrypt(out, ks), params, imag_tol=None) - v)))
    print("resnet20-chain bootstrap bits", -np.log2(err))
    assert -np.log2(err) >= 19.0
