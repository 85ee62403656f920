"""Bit-exact parity of the CUDA engine against full residue arrays frozen
from the unmodified reference at a 256-ring (tests/golden/make_golden.py,
gen_small).  Every integer output must match with np.array_equal."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def small(golden_small):
    from paper_2310_16530_b200 import ckks
    params = ckks.CkksParams.build("unit-small", 256, 50, 40, 4, 50, 2)
    assert [m.q for m in params.q_mods] == golden_small["q"].tolist()
    assert [m.q for m in params.p_mods] == golden_small["p"].tolist()
    ks = ckks.keygen(params, np.random.default_rng(3), rotations=[1, 2, 4])
    return params, ks


def _ct(ct):
    c0, c1 = ct.host_residues()
    return np.stack([c0, c1])


def test_psi_matches_reference(small, golden_small):
    params, _ = small
    ctx = params.ctx
    got = [ctx.psi(i) for i in range(ctx.Lq + ctx.K)]
    assert got == golden_small["psi"].tolist()


def test_ntt_forward_inverse(small, golden_small):
    from paper_2310_16530_b200 import ring
    params, _ = small
    ext = params.q_mods + params.p_mods
    p = ring.RnsPoly(ext, golden_small["ntt_in"].copy(), ring.Domain.COEFF, params.ctx)
    f = ring.ntt_forward(p)
    assert np.array_equal(f.coeffs, golden_small["ntt_out"])
    back = ring.ntt_inverse(f)
    assert np.array_equal(back.coeffs, golden_small["ntt_in"])


def test_base_convert(small, golden_small):
    from paper_2310_16530_b200 import ring
    params, _ = small
    src = params.q_mods[:3]
    dst = params.p_mods + params.q_mods[3:4]
    p = ring.RnsPoly(src, golden_small["ntt_in"][:3].copy(), ring.Domain.COEFF, params.ctx)
    assert np.array_equal(ring.base_convert(p, dst).coeffs, golden_small["bc_out"])


def test_automorphism_coeff(small, golden_small):
    from paper_2310_16530_b200 import ckks, ring
    params, _ = small
    ext = params.q_mods + params.p_mods
    p = ring.RnsPoly(ext, golden_small["ntt_in"].copy(), ring.Domain.COEFF, params.ctx)
    assert np.array_equal(ring.automorphism(p, 5).coeffs, golden_small["auto5"])
    g = ckks.galois_element(3, params.n)
    assert np.array_equal(ring.automorphism(p, g).coeffs, golden_small["auto_g"])


def test_automorphism_eval_is_permutation(small, golden_small):
    from paper_2310_16530_b200 import ckks, ring
    params, _ = small
    ext = params.q_mods + params.p_mods
    p = ring.RnsPoly(ext, golden_small["ntt_in"].copy(), ring.Domain.COEFF, params.ctx)
    for g in (5, ckks.galois_element(3, params.n), 2 * params.n - 1):
        lhs = ring.ntt_forward(ring.automorphism(p, g))
        rhs = ring.automorphism_eval(ring.ntt_forward(p), g)
        assert np.array_equal(lhs.coeffs, rhs.coeffs)


def test_keygen_bit_exact(small, golden_small):
    from paper_2310_16530_b200.engine import to_host_u64
    _, ks = small
    assert np.array_equal(ks.sk.coeffs, golden_small["sk"])
    assert np.array_equal(ks.pk[0].coeffs, golden_small["pk_b"])
    assert np.array_equal(ks.pk[1].coeffs, golden_small["pk_a"])
    assert np.array_equal(to_host_u64(ks.rlk.rows_b), golden_small["rlk_b"])
    assert np.array_equal(to_host_u64(ks.rlk.rows_a), golden_small["rlk_a"])
    for s in (1, 2, 4):
        assert np.array_equal(to_host_u64(ks.gks[s].rows_b), golden_small[f"gk{s}_b"])
        assert np.array_equal(to_host_u64(ks.gks[s].rows_a), golden_small[f"gk{s}_a"])


@pytest.fixture(scope="module")
def cts(small, golden_small):
    from paper_2310_16530_b200 import ckks
    params, ks = small
    L = params.max_level
    pt1 = ckks.encode(golden_small["v1"], params, L)
    ct1 = ckks.encrypt(pt1, ks, np.random.default_rng(77))
    ct2 = ckks.encrypt(ckks.encode(golden_small["v2"], params, L), ks, np.random.default_rng(78))
    return pt1, ct1, ct2


def test_encode_encrypt(cts, golden_small):
    pt1, ct1, ct2 = cts
    assert np.array_equal(pt1.poly.coeffs, golden_small["pt1"])
    assert np.array_equal(_ct(ct1), golden_small["ct1"])
    assert np.array_equal(_ct(ct2), golden_small["ct2"])


def test_hmult_rescale(small, cts, golden_small):
    from paper_2310_16530_b200 import ckks
    params, ks = small
    _, ct1, ct2 = cts
    hm = ckks.hmult(ct1, ct2, ks)
    assert np.array_equal(_ct(hm), golden_small["hmult"])
    rs = ckks.rescale(hm, params)
    assert np.array_equal(_ct(rs), golden_small["rescale"])
    dec = ckks.decode(ckks.decrypt(rs, ks), params)
    np.testing.assert_array_equal(dec, golden_small["dec_hmult"])


@pytest.mark.parametrize("k", [1, 3, -1, 4])
def test_rotate(small, cts, golden_small, k):
    from paper_2310_16530_b200 import ckks
    _, ks = small
    _, ct1, _ = cts
    assert np.array_equal(_ct(ckks.rotate(ct1, k, ks)), golden_small[f"rot{k}"])


def test_rotate_many_hoisted(small, cts, golden_small):
    from paper_2310_16530_b200 import ckks
    _, ks = small
    _, ct1, _ = cts
    outs = ckks.rotate_many(ct1, [1, 4, 3], ks)
    assert np.array_equal(_ct(outs[0]), golden_small["rot1"])
    assert np.array_equal(_ct(outs[1]), golden_small["rot4"])
    assert np.array_equal(_ct(outs[2]), golden_small["rot3"])


def test_elementwise(small, cts, golden_small):
    from paper_2310_16530_b200 import ckks
    _, ks = small
    pt1, ct1, ct2 = cts
    assert np.array_equal(_ct(ckks.pmult(ct1, pt1)), golden_small["pmult"])
    assert np.array_equal(_ct(ckks.hadd(ct1, ct2)), golden_small["hadd"])
    assert np.array_equal(_ct(ckks.padd(ct1, pt1)), golden_small["padd"])


def test_scalar_mac_exact(small, cts):
    """sum_t k_t * src_t per limb (prefix read of a longer source), checked
    with Python integers; > 16 terms exercises the batched launches."""
    params, _ = small
    _, ct1, ct2 = cts
    ctx = params.ctx
    lvl = ct1.level - 1
    srcs = [ct1.data, ct2.data] * 9
    rng = np.random.default_rng(9)
    consts = [[int(v) for v in rng.integers(-(1 << 62), 1 << 62, size=lvl + 1)] for _ in srcs]
    out = ctx.scalar_mac(srcs, consts, lvl).cpu().numpy().astype(object)
    hs = [s.cpu().numpy().astype(object) for s in srcs]
    for r in range(lvl + 1):
        q = params.q_mods[r].q
        want = sum(h[:, r, :] * (c[r] % q) for h, c in zip(hs, consts)) % q
        assert np.array_equal(out[:, r, :], want)
    acc = ctx.scalar_mac(srcs[:1], consts[:1], lvl, out=ctx.scalar_mac(srcs[1:2], consts[1:2], lvl),
                         accumulate=True).cpu().numpy().astype(object)
    q0 = params.q_mods[0].q
    assert np.array_equal(acc[:, 0, :], (hs[0][:, 0, :] * (consts[0][0] % q0) + hs[1][:, 0, :] * (consts[1][0] % q0)) % q0)


def test_batched_ops_match_single(small, cts):
    """hmult / hoisted rotations / shared-mask MAC over a batch of
    ciphertexts equal the single-ciphertext results entry by entry."""
    import torch
    from paper_2310_16530_b200 import ckks
    params, ks = small
    _, ct1, ct2 = cts
    rng = np.random.default_rng(11)
    more = [ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, ct1.level), ks, rng)
            for _ in range(4)]
    A = ckks.stack([ct1, ct2] + more[:3])           # 5 entries: exercises the 4-wide kernels' tail
    B = ckks.stack([ct2, ct1] + more[1:])
    hm = ckks.unstack(ckks.hmult(A, B, ks))
    for a, b, h in zip(ckks.unstack(A), ckks.unstack(B), hm):
        assert torch.equal(h.data, ckks.hmult(a, b, ks).data)
    rots = ckks.rotate_many(A, [1, 2, 4], ks)
    for k, r in zip([1, 2, 4], rots):
        for a, got in zip(ckks.unstack(A), ckks.unstack(r)):
            assert torch.equal(got.data, ckks.rotate(a, k, ks).data)
    ctx = params.ctx
    masks = [ctx.unop("to_mont", ckks.encode(rng.uniform(-1, 1, params.slots), params, ct1.level).data,
                      ct1.level + 1) for _ in range(3)]
    outb = ctx.mac_terms([A.data, B.data, A.data], masks, ct1.level)
    for i, (a, b) in enumerate(zip(ckks.unstack(A), ckks.unstack(B))):
        assert torch.equal(outb[i], ctx.mac_terms([a.data, b.data, a.data], masks, ct1.level))
    # a ciphertext-batch rescale is the per-entry rescale
    rs = ckks.unstack(ckks.rescale(A, params))
    for a, r in zip(ckks.unstack(A), rs):
        assert torch.equal(r.data, ckks.rescale(a, params).data)


def test_mac_terms_multi_matches_per_output(small, cts):
    """Multi-output MAC over a shared term list (null = absent term) equals
    one mac_terms per output on its present terms."""
    import torch
    from paper_2310_16530_b200 import ckks
    params, ks = small
    _, ct1, ct2 = cts
    ctx = params.ctx
    rng = np.random.default_rng(12)
    lvl = ct1.level
    srcs = [ct1.data, ct2.data] + [ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, lvl), ks,
                                                 rng).data for _ in range(3)]
    mk = lambda: ctx.unop("to_mont", ckks.encode(rng.uniform(-1, 1, params.slots), params, lvl).data, lvl + 1)
    for G in (1, 2, 3, 4, 6, 9):
        masks = [[mk() if (g + t) % 3 else None for t in range(len(srcs))] for g in range(G)]
        got = ctx.mac_terms_multi(srcs, masks, lvl)
        # the same with every other mask in the 48-bit packed resident layout
        assert ctx.masks_packable(lvl)
        mixed = [[(ctx.pack_masks(m, lvl)[0] if (m is not None and (g + t) % 2) else m) for t, m in enumerate(row)]
                 for g, row in enumerate(masks)]
        got_p = ctx.mac_terms_multi(srcs, mixed, lvl)
        for g in range(G):
            terms = [(s, m) for s, m in zip(srcs, masks[g]) if m is not None]
            want = ctx.mac_terms([s for s, _ in terms], [m for _, m in terms], lvl)
            assert torch.equal(got[g], want)
            assert torch.equal(got_p[g], want)
    m = mk()
    assert torch.equal(ctx.unpack_mask(ctx.pack_masks(m, lvl)[0], lvl), m)


def test_truncated_rotation_keys(small, cts):
    """Rotation keys cut down to the rows levels <= 2 read give identical
    rotations there and refuse higher levels (KeyError_)."""
    import torch
    from paper_2310_16530_b200 import ckks
    from paper_2310_16530_b200.errors import KeyError_
    params, ks = small
    _, ct1, _ = cts
    kt = ckks.keygen(params, np.random.default_rng(3), rotations=[1, 2, 4])
    freed = kt.truncate_rotations([1, 4], 2)
    assert freed > 0 and kt.gks[2].rows_b.shape == ks.gks[2].rows_b.shape
    low = ckks.mod_drop(ct1, 2)
    for k in (1, 3, 4):
        assert torch.equal(ckks.rotate(low, k, kt).data, ckks.rotate(low, k, ks).data)
    many = ckks.rotate_many(ckks.stack([low, low]), [1, 4], kt)
    assert torch.equal(ckks.unstack(many[1])[1].data, ckks.rotate(low, 4, ks).data)
    with pytest.raises(KeyError_):
        ckks.rotate(ct1, 1, kt)


def test_lazy_mac_worst_case_residues(small):
    """Lazy 128-bit MACs fold the high word every 8 products and the plane MAC
    chunks its term list by 48: with every residue at q-1 (the largest
    products) and 53 terms (folds at 8, 16, ..., a 48 + 5 chunk split, mixed
    packed / unpacked masks) the outputs still equal sum (q-1)^2 R^-1 mod q."""
    import torch
    params, ks = small
    ctx = params.ctx
    lvl = params.max_level
    qs = [m.q for m in params.q_mods[: lvl + 1]]
    n = params.n
    full = torch.tensor([[q - 1] * n for q in qs], dtype=torch.int64, device=ctx.torch_device)
    ct = torch.stack([full, full]).contiguous()
    T = 53
    cts = [ct] * T
    masks = [[full.clone() for _ in range(T)], [full.clone() for _ in range(T)]]
    masks[1] = [ctx.pack_masks(m, lvl)[0] if t % 2 else m for t, m in enumerate(masks[1])]
    got = ctx.mac_terms_multi(cts, masks, lvl)
    got_terms = ctx.mac_terms(cts, masks[0], lvl)
    for i, q in enumerate(qs):
        r_inv = pow(1 << 64, -1, q)
        want = T * (q - 1) * (q - 1) * r_inv % q
        for out in (got[0], got[1], got_terms):
            row = out[:, i].cpu().numpy().view(np.uint64)
            assert (row == np.uint64(want)).all(), (i, q)


# launch-shape knobs of the TMA-staged plane MAC and key-switch inner product
# (threads per CTA, ring depth, register cap) and the values the engine ships with
_KNOB_DEFAULTS = {"mac_tma": 3, "mac3_stages": 4, "mac3_tpb": 128, "mac3_fork": 1, "mac_tpb": 128, "tma_stages": 3,
                  "mac_minb": 1,
                  "ks_tpb": 128, "ks_stages": 3, "ks_tma_min": 2, "ks_tma3": 0, "ks3_stages": 3, "md_fuse": 0,
                  "ntt_pipe": 1, "fbc_fast": 1, "ntt_fork": 1, "fbc_fork": 1,
                  "ks_rots": 1, "ks_rots_min_nb": 1, "ks96": 1}
_KNOB_VARIANTS = [
    {"mac_tma": 1},
    {"ntt_fork": 0},
    {"fbc_fork": 0},
    {"ks_rots": 0},
    {"ks_rots_min_nb": 2},
    {"ks96": 0},
    {"mac3_fork": 0},
    {"md_fuse": 1},
    {"ntt_pipe": 0},
    {"fbc_fast": 0},
    {"mac3_stages": 2},
    {"mac3_stages": 3},
    {"mac3_stages": 6},
    {"mac3_tpb": 256},
    {"mac3_tpb": 256, "mac3_stages": 4},
    {"mac_tma": 1, "mac_tpb": 256, "tma_stages": 4, "ks_tpb": 256},
    {"mac_tma": 1, "mac_tpb": 256, "tma_stages": 6, "ks_tpb": 256},
    {"mac_tma": 1, "mac_tpb": 256, "tma_stages": 4, "mac_minb": 4},
    {"mac_tma": 1, "mac_tpb": 128, "tma_stages": 4},
    {"mac_tma": 1, "mac_tpb": 128, "tma_stages": 3, "mac_minb": 5},
    {"mac_tma": 1, "mac_tpb": 128, "tma_stages": 2},
    {"ks_tpb": 128, "ks_stages": 4},
    {"ks_tma3": 1},
    {"ks_tma3": 1, "ks3_stages": 2},
    {"ks_tma3": 1, "ks3_stages": 4},
]


def test_launch_shape_variants_bit_identical(small, cts):
    """Every launch shape of k_mac_multi_tma(2/3) / k_ks_inner_tma(2) gives the
    residues of the shipped shape: plane MACs over mixed packed / unpacked /
    absent masks, and batched (>= 2 entries: TMA path) hoisted rotations."""
    import torch
    from paper_2310_16530_b200 import _native, ckks
    params, ks = small
    _, ct1, ct2 = cts
    ctx = params.ctx
    rng = np.random.default_rng(21)
    lvl = ct1.level
    srcs = [ct1.data, ct2.data] + [ckks.encrypt(ckks.encode(rng.uniform(-1, 1, params.slots), params, lvl), ks,
                                                 rng).data for _ in range(11)]
    mk = lambda: ctx.unop("to_mont", ckks.encode(rng.uniform(-1, 1, params.slots), params, lvl).data, lvl + 1)
    masks = [[mk() if (g + t) % 3 else None for t in range(len(srcs))] for g in range(4)]
    masks = [[(ctx.pack_masks(m, lvl)[0] if (m is not None and (g + t) % 2) else m) for t, m in enumerate(row)]
             for g, row in enumerate(masks)]
    batch = ckks.stack([ct1, ct2, ct1, ct2, ct1])

    def run():
        outs = [o.clone() for o in ctx.mac_terms_multi(srcs, masks, lvl)]
        outs += [r.data.clone() for r in ckks.rotate_many(batch, [1, 2, 4], ks)]
        torch.cuda.synchronize()
        return outs

    for k, v in _KNOB_DEFAULTS.items():
        _native.set_option(k, v)
    want = run()
    try:
        for var in _KNOB_VARIANTS:
            for k, v in var.items():
                _native.set_option(k, v)
            got = run()
            assert all(torch.equal(a, b) for a, b in zip(got, want)), var
            for k, v in _KNOB_DEFAULTS.items():
                _native.set_option(k, v)
    finally:
        for k, v in _KNOB_DEFAULTS.items():
            _native.set_option(k, v)
