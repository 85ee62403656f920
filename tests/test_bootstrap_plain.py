"""Plaintext simulation of every bootstrapping stage (CPU).  Bootstrapping
has no reference implementation (parity unpinned); these checks pin the
linear algebra and the EvalMod polynomial before any homomorphic run."""

import math

import numpy as np
import pytest

from paper_2310_16530_b200 import bootstrap as bt


@pytest.mark.parametrize("n_ring", [16, 32, 256])
def test_special_fft_factorises_embedding(n_ring):
    n = n_ring // 2
    u0 = bt.embedding_matrix(n_ring)
    prod = np.eye(n, dtype=complex)
    for s in range(1, n.bit_length()):
        prod = bt.special_fft_stage(n, 1 << s).toarray() @ prod
    br = bt.bit_reverse_perm(n)
    perm = np.zeros((n, n))
    perm[np.arange(n), br] = 1
    assert np.allclose(prod @ perm, u0)


def test_embedding_matches_reference_encoding():
    """slot j = m(zeta^(5^j)): decode of the engine's encode is U0 applied to
    (t_lo + i t_hi)/scale (ckks.py:241-308 conventions)."""
    from paper_2310_16530_b200 import ckks
    params = ckks.CkksParams.build("t", 64, 50, 40, 2, 50, 2)
    rng = np.random.default_rng(0)
    vals = rng.uniform(-1, 1, params.slots)
    t = ckks.encode_coeffs(vals, params, 0, 2.0 ** 30).astype(float)
    n = params.slots
    u = (t[:n] + 1j * t[n:]) / 2.0 ** 30
    assert np.max(np.abs(bt.embedding_matrix(params.n) @ u - vals)) < 1e-6


@pytest.mark.parametrize("n_ring,stages", [(64, (2, 3)), (256, (3, 2, 2)), (1 << 12, (4, 4, 3))])
def test_cts_stc_round_trip_and_cts_output(n_ring, stages):
    n = n_ring // 2
    rng = np.random.default_rng(1)
    t = rng.normal(size=2 * n)
    coeffs = t[:n] + 1j * t[n:]
    w = bt.embedding_matrix(n_ring) @ coeffs
    cts = [bt.diag_plan(m) for m in bt.cts_groups(n, stages, 0.5)]
    stc = [bt.diag_plan(m) for m in bt.stc_groups(n, stages[::-1], 2.0 / n)]
    u = bt.apply_plain(cts, w)
    br = bt.bit_reverse_perm(n)
    assert np.allclose(u, 0.5 * n * coeffs[br])
    assert np.allclose(bt.apply_plain(stc, u), w)
    # unit-magnitude diagonal entries (precision of the plaintext products)
    for plans, c0 in ((cts, 0.5), (stc, 2.0 / n)):
        for i, p in enumerate(plans):
            mags = np.concatenate([np.abs(pre) for terms in p.giants.values() for _, pre in terms])
            nz = mags[mags > 1e-12]
            assert np.allclose(nz, c0 if i == 0 else 1.0)
    # BSGS uses few rotations per level
    for p in cts:
        assert len(p.babies) + len(p.giants) <= 2 * (1 << max(stages)) + 2


def test_evalmod_polynomial_accuracy():
    cfg = bt.BootConfig()
    rng = np.random.default_rng(2)
    I = rng.integers(-cfg.k_bound + 1, cfg.k_bound, size=4000)
    eps = rng.uniform(-2.0 ** -10, 2.0 ** -10, size=4000)
    x = I + eps
    got = bt.evalmod_plain(cfg, x / (cfg.k_bound + 1))
    assert np.max(np.abs(got - np.sin(2 * np.pi * x))) < 1e-9
    # sin(2 pi eps)/(2 pi) ~ eps to the cubic term
    assert np.max(np.abs(got / (2 * np.pi) - eps)) < 1e-7


def test_depth_budget_and_chain():
    cfg = bt.BootConfig()
    assert cfg.depth() == 3 + (math.ceil(math.log2(cfg.degree)) + 1) + cfg.double_angle + 3
    p = bt.boot_params("b", 1 << 12, 4, bt.BootConfig(cts_stages=(4, 4, 3), stc_stages=(3, 4, 4)))
    assert p.max_level == 4 + 3 + cfg.evalmod_depth() + 3
    assert all(m.q.bit_length() <= 61 for m in p.q_mods + p.p_mods)


def _levels(tree, baby, top_level):
    """level simulation of eval_chebyshev: T_i at top - ceil(log2 i)"""
    lv = {i: top_level - math.ceil(math.log2(i)) if i > 1 else top_level for i in bt.bsgs_powers(tree, baby)}

    def top(t):
        if isinstance(t, np.ndarray):
            return min((lv[i] for i in range(1, len(t))), default=top_level) - 1
        m, q, r = t
        return min(lv[m] - 1, top(q) - 1, top(r))
    return top(tree)


def _products(tree):
    if isinstance(tree, np.ndarray):
        return 0
    return 1 + _products(tree[1]) + _products(tree[2])


@pytest.mark.parametrize("baby", [4, 8])
def test_bsgs_chebyshev_matches_direct_evaluation(baby):
    cfg = bt.BootConfig()
    c = bt.evalmod_coeffs(cfg)
    tree = bt.bsgs_split(c, baby)
    y = np.linspace(-1, 1, 2001)
    assert np.max(np.abs(bt.bsgs_eval_plain(tree, y) - np.polynomial.chebyshev.chebval(y, c))) < 1e-12
    # depth within the evalmod budget, far fewer ciphertext products than degree
    assert 40 - _levels(tree, baby, 40) <= math.ceil(math.log2(cfg.degree)) + 1
    powers = bt.bsgs_powers(tree, baby)
    assert len(powers) + _products(tree) <= 2 * int(math.sqrt(cfg.degree)) + 10


def test_cheb_divide_identity():
    rng = np.random.default_rng(4)
    for d, m in [(7, 4), (15, 8), (59, 32), (33, 32)]:
        c = rng.standard_normal(d + 1)
        q, r = bt.cheb_divide(c, m)
        y = np.linspace(-1, 1, 101)
        tm = np.polynomial.chebyshev.chebval(y, np.eye(m + 1)[m])
        ch = np.polynomial.chebyshev.chebval
        assert np.allclose(ch(y, r) + tm * ch(y, q), ch(y, c), atol=1e-12)


@pytest.mark.parametrize("n1", [4, 16, 32])
def test_diag_plan_any_baby_count(n1):
    """BSGS plans with a forced baby count apply the same matrix."""
    n = 256
    rng = np.random.default_rng(n1)
    v = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    for m in bt.cts_groups(n, (4, 4), 1.0):
        p = bt.diag_plan(m, n1)
        assert p.n1 == n1
        assert np.allclose(bt.apply_plain([p], v), m @ v)


def _evalmod_error(cfg):
    B = cfg.k_bound + 1
    I = np.arange(-cfg.k_bound + 1, cfg.k_bound)
    eps = np.linspace(-2 ** -10, 2 ** -10, 201)
    y = ((I[:, None] + eps[None, :]) / B).ravel()
    return np.max(np.abs(bt.evalmod_plain(cfg, y) - np.sin(2 * np.pi * B * y)))


def test_resnet20_evalmod_degree_is_precise_enough():
    """The ResNet20 workload's EvalMod (workloads.RESNET20_EVALMOD_DEGREE
    before 3 double angles) must approximate sin(2 pi x) near the integers
    (x = I + eps, |I| < k_bound, |eps| <= 2^-10) so well that the bootstrap's
    ~2^17.3 amplification (sqrt(N) coefficients per slot x q0 / (2 pi
    Delta_1), message ratio 2^12, N = 2^16) keeps slots within 2^-19:
    degree 59 does (2^-43); degree 31, one level shallower, does not (2^-25.5
    -> the 8-bit bootstraps tools/boot_precision.py measured)."""
    from paper_2310_16530_b200 import workloads
    cfg = workloads.resnet20_boot_config()
    assert cfg.degree == workloads.RESNET20_EVALMOD_DEGREE == 59
    amp = 2 ** 8 * 2 ** cfg.message_ratio_bits / (2 * np.pi)
    assert _evalmod_error(cfg) * amp < 2 ** -19
    shallow = bt.BootConfig(degree=31)
    assert shallow.evalmod_depth() == cfg.evalmod_depth() - 1
    assert _evalmod_error(shallow) * amp > 2 ** -10
