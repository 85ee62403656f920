"""NTT / iNTT parity over every ring size the engine dispatches (single-pass
smem kernels for small N, radix-16 register passes for 2^12..2^16) against
the C oracle (restated reference kernels.py:232-281), plus acceptance gate 1
(test_acceptance.py:128-156): transform products equal schoolbook negacyclic
products, run through the GPU."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _mods(n, bits=(59, 40, 45)):
    from paper_2310_16530_b200.ring import find_ntt_primes
    out = []
    for b in bits:
        out += find_ntt_primes(n, b, 1, avoid=out)
    return out


@pytest.mark.parametrize("logn", list(range(2, 17)))
def test_ntt_matches_oracle(logn):
    from oracle import ckks_oracle as O
    from paper_2310_16530_b200.engine import context_for, to_device_u64, to_host_u64
    n = 1 << logn
    qs = _mods(n)
    rng = np.random.default_rng(logn)
    rows = np.stack([rng.integers(0, q, size=(3, n), dtype=np.uint64) for q in qs], axis=1)  # [3 polys, 3 limbs, n]
    ctx = context_for(n, qs)
    d = to_device_u64(rows)
    ctx.ntt(d, len(qs))
    got = to_host_u64(d)
    for z in range(3):
        assert np.array_equal(got[z], O.ntt(rows[z], qs)), f"poly {z}"
    ctx.ntt(d, len(qs), inverse=True)
    assert np.array_equal(to_host_u64(d), rows)


@pytest.mark.parametrize("logn", [12, 13, 14, 16])
def test_ntt_ext_basis_and_skip(logn):
    """Ext-basis NTT (q prefix + specials) equals per-limb oracle transforms."""
    from oracle import ckks_oracle as O
    from paper_2310_16530_b200.engine import context_for, to_device_u64, to_host_u64
    n = 1 << logn
    qs = _mods(n, (59, 40, 41, 42))
    ps = _mods(n, (58, 57))
    ps = [p for p in ps if p not in qs]
    ctx = context_for(n, qs, ps)
    rng = np.random.default_rng(7)
    basis = qs[:2] + ps
    rows = np.stack([rng.integers(0, q, size=n, dtype=np.uint64) for q in basis])
    d = to_device_u64(rows)
    ctx.ntt(d, 2, len(ps))
    assert np.array_equal(to_host_u64(d), O.ntt(rows, basis))


def _schoolbook(a, b, q):
    n = len(a)
    out = [0] * n
    for i, ai in enumerate(a):
        for j, bj in enumerate(b):
            k = i + j
            if k < n:
                out[k] = (out[k] + ai * bj) % q
            else:
                out[k - n] = (out[k - n] - ai * bj) % q
    return out


@pytest.mark.parametrize("n", [4, 8, 16, 32])
def test_gate1_schoolbook(n):
    from paper_2310_16530_b200 import ring
    from paper_2310_16530_b200.ring import Modulus, find_ntt_primes
    qs = find_ntt_primes(n, 59, 1) + find_ntt_primes(n, 45, 1)
    mods = tuple(Modulus.make(q) for q in qs)
    rng = np.random.default_rng(0xACC1)
    for _ in range(50):
        a = rng.integers(-(1 << 61), 1 << 61, size=n).tolist()
        b = rng.integers(-(1 << 61), 1 << 61, size=n).tolist()
        pa = ring.from_int_coeffs(a, mods, n)
        pb = ring.from_int_coeffs(b, mods, n)
        got = ring.ntt_inverse(ring.poly_mul_pointwise(ring.ntt_forward(pa), ring.ntt_forward(pb))).coeffs
        for li, m in enumerate(mods):
            want = _schoolbook([v % m.q for v in a], [v % m.q for v in b], m.q)
            assert got[li].tolist() == want


@pytest.mark.parametrize("logn", [8, 12, 16])
@pytest.mark.parametrize("mont", [False, True])
def test_ntt_from_signed_fused(logn, mont):
    """The fused signed-load forward NTT equals from_signed (+ Montgomery
    lift) followed by the forward NTT, bit for bit, and the oracle."""
    import torch
    from oracle import ckks_oracle as O
    from paper_2310_16530_b200.engine import context_for, to_host_u64
    n = 1 << logn
    qs = _mods(n)
    ctx = context_for(n, qs)
    rng = np.random.default_rng(logn + 3)
    rows = rng.integers(-(1 << 62), 1 << 62, size=(5, n), dtype=np.int64)
    rows[0, :4] = [-(1 << 63), (1 << 63) - 1, 0, -1]
    dev = torch.from_numpy(rows).cuda()
    fused = ctx.ntt_from_signed(dev, len(qs), mont=mont)
    ref = ctx.from_signed(dev, len(qs), mont=mont)
    ctx.ntt(ref, len(qs))
    assert torch.equal(fused, ref)
    if not mont:
        want = np.stack([O.ntt(np.stack([(rows[p].astype(object) % q).astype(np.uint64) for q in qs]), qs)
                         for p in range(5)])
        assert np.array_equal(to_host_u64(fused), want)


def test_roofline_instrumentation():
    """bench.py's integer roofline: the butterfly-rate probes run and order
    as measured (pure FP64 network > FP64 quotient > integer fast > full
    width), and the limb counters classify one forward + one inverse
    transform by modulus width."""
    from paper_2310_16530_b200 import _native
    from paper_2310_16530_b200.engine import context_for, to_device_u64
    f64, fp, fast, full = (_native.ntt_butterfly_peak(k) for k in (4, 2, 1, 0))
    assert f64 > 0 and fp > 0 and fast > 0 and full > 0
    assert f64 > fp  # the network the class-2 (q < 2^41) limbs now run
    assert fast > full  # the unreduced network issues fewer instructions
    n = 1 << 16
    qs = _mods(n)  # 59-bit (full), 40-bit (FP64 class), 45-bit (integer fast class)
    ctx = context_for(n, qs)
    d = to_device_u64(np.zeros((2, len(qs), n), dtype=np.uint64))
    _native.ntt_limb_counts(reset=True)
    ctx.ntt(d, len(qs))
    ctx.ntt(d, len(qs), inverse=True)
    c = _native.ntt_limb_counts(reset=True)
    assert c == {"fwd_fast": 4, "fwd_full": 2, "inv_fast": 4, "inv_full": 2}
