"""TEST INFRASTRUCTURE -- the CPU oracle.  Never imported by the product.

A compact numpy + C restatement of the reference's RNS-CKKS path
(/root/reference/pkg/src/hcnn/ring.py and ckks.py), used (a) by the test
suite to recompute residues the CUDA engine must match bit for bit on
seeded inputs, and (b) as bench.py's CPU-baseline / ``--impl reference``
arm.  The per-row modular kernels are the C restatement in ref_kernels.c
(OpenMP over rows); everything here is host numpy.

Pinned against the reference by tests/test_oracle.py: every function here
reproduces tests/golden/golden_small.npz (full arrays frozen from the
reference) and the sha256 digests of tests/golden/golden_hashes.json.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_lib = None


def lib():
    global _lib
    if _lib is None:
        from . import build as _b
        path = _b.build()
        L = ctypes.CDLL(str(path))
        P = ctypes.c_void_p
        S = ctypes.c_size_t
        U = ctypes.c_uint64
        L.o_ntt_rows.argtypes = [P, S, S, P, P, P]
        L.o_intt_rows.argtypes = [P, S, S, P, P, P, P]
        L.o_mulmod_rows.argtypes = [P, P, P, S, S, ctypes.c_int, P, P]
        L.o_muladd_rows.argtypes = [P, P, P, S, S, P, P]
        L.o_fbc_rows.argtypes = [P, P, S, S, S, P, P, P, P, P]
        L.o_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _u(vals) -> np.ndarray:
    return np.ascontiguousarray(np.asarray([int(v) for v in vals], dtype=np.uint64))


# ---------------------------------------------------------------------------
# moduli, primes, twiddles (ring.py:32-197)
# ---------------------------------------------------------------------------

def ninv_of(q: int) -> int:
    return (-pow(q, -1, 1 << 64)) % (1 << 64)


def mont(a: int, q: int) -> int:
    return (a << 64) % q


def _probable_prime(n: int) -> bool:
    if n < 2:
        return False
    small = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41)
    for p in small:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while not d & 1:
        d >>= 1
        s += 1
    for a in small:
        x = pow(a, d, n)
        if x == 1 or x == n - 1:
            continue
        for _ in range(s - 1):
            x = pow(x, 2, n)
            if x == n - 1:
                break
        else:
            return False
    return True


def ntt_primes(n: int, bits: int, count: int, avoid=(), alternate=False) -> list[int]:
    """ring.py:84-126 walk: first candidate below is anchor-2N, above anchor+2*2N."""
    step = 2 * n
    anchor = (1 << bits) - (((1 << bits) - 1) % step)
    used = set(avoid)
    down, up = anchor, anchor + step
    res = []
    for i in range(count):
        if alternate and i % 2:
            up += step
            while up in used or not _probable_prime(up):
                up += step
            pick = up
        else:
            down -= step
            while down in used or not _probable_prime(down):
                down -= step
            pick = down
        used.add(pick)
        res.append(pick)
    return res


_tw_cache: dict = {}


def twiddles(q: int, n: int):
    """(forward_mont, inverse_mont, n_inv_mont, psi) per ring.py:160-197."""
    key = (q, n)
    if key in _tw_cache:
        return _tw_cache[key]
    psi = next(p for p in (pow(r, (q - 1) // (2 * n), q) for r in range(2, 1000))
               if p != 1 and pow(p, n, q) == q - 1)
    bits = n.bit_length() - 1
    brv = np.array([int(format(j, f"0{bits}b")[::-1], 2) if bits else 0 for j in range(n)])
    pw_f = [1] * n
    pw_i = [1] * n
    pinv = pow(psi, -1, q)
    for j in range(1, n):
        pw_f[j] = pw_f[j - 1] * psi % q
        pw_i[j] = pw_i[j - 1] * pinv % q
    fwd = _u([mont(pw_f[b], q) for b in brv])
    inv = _u([mont(pw_i[b], q) for b in brv])
    out = (fwd, inv, mont(pow(n, -1, q), q), psi)
    _tw_cache[key] = out
    return out


@dataclass
class OParams:
    n: int
    qs: list[int]
    ps: list[int]
    delta: float

    @classmethod
    def build(cls, n, log_q0, log_qi, levels, log_p, n_special):
        q0 = ntt_primes(n, log_q0, 1)
        qi = ntt_primes(n, log_qi, levels, avoid=q0, alternate=True)
        ps = ntt_primes(n, log_p, n_special, avoid=q0 + qi)
        return cls(n, q0 + qi, ps, float(2 ** log_qi))

    @property
    def slots(self):
        return self.n // 2

    @property
    def L(self):
        return len(self.qs) - 1

    @property
    def alpha(self):
        return len(self.ps)

    @property
    def dnum(self):
        return -(-len(self.qs) // self.alpha)

    @property
    def ext(self):
        return self.qs + self.ps


# ---------------------------------------------------------------------------
# row arithmetic (ring.py:264-336 over lists of moduli)
# ---------------------------------------------------------------------------

def _consts(mods):
    return _u(mods), _u([ninv_of(q) for q in mods])


def ntt(rows: np.ndarray, mods) -> np.ndarray:
    out = np.ascontiguousarray(rows, dtype=np.uint64).copy()
    n = out.shape[1]
    w = np.ascontiguousarray(np.stack([twiddles(q, n)[0] for q in mods]))
    qs, ni = _consts(mods)
    lib().o_ntt_rows(_p(out), out.shape[0], n, _p(w), _p(qs), _p(ni))
    return out


def intt(rows: np.ndarray, mods) -> np.ndarray:
    out = np.ascontiguousarray(rows, dtype=np.uint64).copy()
    n = out.shape[1]
    w = np.ascontiguousarray(np.stack([twiddles(q, n)[1] for q in mods]))
    nim = _u([twiddles(q, n)[2] for q in mods])
    qs, ni = _consts(mods)
    lib().o_intt_rows(_p(out), out.shape[0], n, _p(w), _p(qs), _p(ni), _p(nim))
    return out


def mul_mont(a: np.ndarray, b_mont: np.ndarray, mods) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b_mont, dtype=np.uint64)
    out = np.empty_like(a)
    qs, ni = _consts(mods)
    lib().o_mulmod_rows(_p(out), _p(a), _p(b), a.shape[0], a.shape[1], 0, _p(qs), _p(ni))
    return out


def to_mont(a: np.ndarray, mods) -> np.ndarray:
    r2 = np.ascontiguousarray(np.stack([np.full(a.shape[1], (1 << 128) % q, dtype=np.uint64) for q in mods]))
    return mul_mont(a, r2, mods)


def mul(a, b, mods):
    """poly_mul_pointwise ring.py:287-296 (two REDCs)."""
    return mul_mont(a, to_mont(b, mods), mods)


def add(a, b, mods):
    q = _u(mods)[:, None]
    t = a + b
    return np.where(t >= q, t - q, t)


def sub(a, b, mods):
    q = _u(mods)[:, None]
    return np.where(a >= b, a - b, a + (q - b))


def scalar_mul(a, consts, mods):
    """_scalar_mul_rows ckks.py:350-356"""
    c = np.ascontiguousarray(np.stack([np.full(a.shape[1], mont(int(k) % q, q), dtype=np.uint64)
                                       for k, q in zip(consts, mods)]))
    return mul_mont(a, c, mods)


def base_convert(x: np.ndarray, src, dst) -> np.ndarray:
    """_conv_table + base_convert ring.py:343-398"""
    n = x.shape[1]
    big = 1
    for q in src:
        big *= q
    punc = [big // q for q in src]
    inv_p = np.ascontiguousarray(np.stack([np.full(n, mont(pow(pu % q, -1, q), q), dtype=np.uint64)
                                           for pu, q in zip(punc, src)]))
    ys = mul_mont(x, inv_p, src)
    tmat = _u([mont(pu % t, t) for t in dst for pu in punc])
    out = np.zeros((len(dst), n), dtype=np.uint64)
    sq = _u(src)
    halves = _u([q // 2 for q in src])
    dq, dn = _consts(dst)
    lib().o_fbc_rows(_p(out), _p(np.ascontiguousarray(ys)), len(src), len(dst), n, _p(sq), _p(halves),
                     _p(tmat), _p(dq), _p(dn))
    return out


def automorphism(rows: np.ndarray, g: int, mods) -> np.ndarray:
    """ring.py:405-439 coefficient-domain X -> X^g"""
    n = rows.shape[1]
    j = (np.arange(n) * g) % (2 * n)
    flip = j >= n
    dst = np.where(flip, j - n, j)
    q = _u(mods)[:, None]
    vals = np.where(flip[None, :], np.where(rows == 0, rows, q - rows), rows)
    out = np.empty_like(rows)
    out[:, dst] = vals
    return out


# ---------------------------------------------------------------------------
# sampling (ring.py:446-468, identical draw order)
# ---------------------------------------------------------------------------

def small_rows(small: np.ndarray, mods) -> np.ndarray:
    return np.stack([np.where(small >= 0, small, small + q).astype(np.uint64) for q in mods])


def sample(mods, n, kind, rng, sigma=3.2):
    if kind == "uniform":
        return np.stack([rng.integers(0, q, size=n, dtype=np.uint64) for q in mods])
    if kind == "ternary":
        s = rng.integers(-1, 2, size=n, dtype=np.int64)
    else:
        s = np.rint(rng.normal(0.0, sigma, size=n)).astype(np.int64)
    return small_rows(s, mods)


# ---------------------------------------------------------------------------
# CKKS (ckks.py:241-657)
# ---------------------------------------------------------------------------

def _slot_positions(n):
    pos = np.array([(pow(5, j, 2 * n) - 1) // 2 for j in range(n // 2)], dtype=np.int64)
    return pos, np.exp(1j * np.pi * np.arange(n) / n)


def encode(values, P: OParams, level, scale=None):
    scale = P.delta if scale is None else float(scale)
    n = P.n
    vals = np.zeros(P.slots, dtype=np.complex128)
    v = np.asarray(values, dtype=np.complex128)
    vals[: v.shape[0]] = v
    pos, twist = _slot_positions(n)
    spec = np.zeros(n, dtype=np.complex128)
    spec[pos] = vals
    spec[n - 1 - pos] = np.conj(vals)
    ints = np.rint(np.real(np.fft.fft(spec) / n * np.conj(twist)) * scale).astype(np.int64)
    mods = P.qs[: level + 1]
    rows = np.stack([(ints % np.int64(q)).astype(np.uint64) for q in mods])
    return ntt(rows, mods), scale


def crt_center(rows, mods, bound_bits=None):
    use = len(mods)
    if bound_bits is not None:
        acc = 0
        for i, q in enumerate(mods):
            acc += q.bit_length() - 1
            if acc > bound_bits + 2:
                use = i + 1
                break
    big = 1
    for q in mods[:use]:
        big *= q
    tot = np.zeros(rows.shape[1], dtype=object)
    for i, q in enumerate(mods[:use]):
        pu = big // q
        tot = tot + rows[i].astype(object) * (pu * pow(pu % q, -1, q))
    tot = tot % big
    return np.where(tot > big // 2, tot - big, tot)


def decode(poly_eval, scale, P: OParams):
    mods = P.qs[: poly_eval.shape[0]]
    ints = crt_center(intt(poly_eval, mods), mods, int(np.log2(max(scale, 2.0))) + 34)
    c = np.array([float(v) for v in ints])
    pos, twist = _slot_positions(P.n)
    return np.real((np.fft.ifft(c * twist) * P.n)[pos] / scale)


@dataclass
class OKeys:
    P: OParams
    s_coeff: np.ndarray
    sk: np.ndarray
    pk_b: np.ndarray
    pk_a: np.ndarray
    rlk: tuple
    gks: dict = field(default_factory=dict)


def galois(step, n):
    return pow(5, step % (n // 2), 2 * n)


def _switch_key(P: OParams, s_ext, payload, rng):
    """_make_switch_key ckks.py:359-394"""
    ext = P.ext
    n = P.n
    pint = 1
    for q in P.ps:
        pint *= q
    qfull = 1
    for q in P.qs:
        qfull *= q
    bs, as_ = [], []
    for j in range(P.dnum):
        dp = 1
        for q in P.qs[j * P.alpha:(j + 1) * P.alpha]:
            dp *= q
        qh = qfull // dp
        lam = qh * pow(qh % dp, -1, dp)
        a = ntt(sample(ext, n, "uniform", rng), ext)
        e = ntt(sample(ext, n, "gaussian", rng), ext)
        b = add(sub(e, mul(a, s_ext, ext), ext), scalar_mul(payload, [(pint * lam) % q for q in ext], ext), ext)
        bs.append(to_mont(b, ext))
        as_.append(to_mont(a, ext))
    return np.stack(bs), np.stack(as_)


def keygen(P: OParams, rng, rotations=()):
    """ckks.py:397-424"""
    ext = P.ext
    s_c = sample(ext, P.n, "ternary", rng)
    sk = ntt(s_c, ext)
    nq = len(P.qs)
    a = ntt(sample(P.qs, P.n, "uniform", rng), P.qs)
    e = ntt(sample(P.qs, P.n, "gaussian", rng), P.qs)
    pk_b = sub(e, mul(a, sk[:nq], P.qs), P.qs)
    rlk = _switch_key(P, sk, mul(sk, sk, ext), rng)
    K = OKeys(P, s_c, sk, pk_b, a, rlk)
    for st in rotations:
        st %= P.slots
        if st == 0 or st in K.gks:
            continue
        s_rot = ntt(automorphism(s_c, galois(st, P.n), ext), ext)
        K.gks[st] = _switch_key(P, sk, s_rot, rng)
    return K


def encrypt(pt, scale, K: OKeys, rng):
    P = K.P
    mods = P.qs[: pt.shape[0]]
    nq = len(mods)
    v = ntt(sample(mods, P.n, "ternary", rng), mods)
    e0 = ntt(sample(mods, P.n, "gaussian", rng), mods)
    e1 = ntt(sample(mods, P.n, "gaussian", rng), mods)
    c0 = add(add(mul(v, K.pk_b[:nq], mods), e0, mods), pt, mods)
    c1 = add(mul(v, K.pk_a[:nq], mods), e1, mods)
    return np.stack([c0, c1]), scale


def decrypt(ct, K: OKeys):
    mods = K.P.qs[: ct.shape[1]]
    return add(ct[0], mul(ct[1], K.sk[: len(mods)], mods), mods)


def keyswitch(d_coeff, key, P: OParams):
    """_keyswitch_coeff ckks.py:548-602"""
    nq = d_coeff.shape[0]
    ext = P.qs[:nq] + P.ps
    n_ext = len(ext)
    n = P.n
    kb, ka = key
    sel = list(range(nq)) + list(range(len(P.qs), len(P.qs) + len(P.ps)))
    acc0 = np.zeros((n_ext, n), dtype=np.uint64)
    acc1 = np.zeros((n_ext, n), dtype=np.uint64)
    for j in range(-(-nq // P.alpha)):
        lo, hi = j * P.alpha, min(j * P.alpha + P.alpha, nq)
        others = [r for r in range(n_ext) if not lo <= r < hi]
        raised = np.empty((n_ext, n), dtype=np.uint64)
        raised[lo:hi] = d_coeff[lo:hi]
        raised[others] = base_convert(d_coeff[lo:hi], P.qs[lo:hi], [ext[r] for r in others])
        raised = ntt(raised, ext)
        acc0 = add(acc0, mul_mont(raised, kb[j][sel], ext), ext)
        acc1 = add(acc1, mul_mont(raised, ka[j][sel], ext), ext)
    pint = 1
    for q in P.ps:
        pint *= q
    qm = P.qs[:nq]
    out = []
    for acc in (acc0, acc1):
        lift = ntt(base_convert(intt(acc[nq:], P.ps), P.ps, qm), qm)
        out.append(scalar_mul(sub(acc[:nq], lift, qm), [pow(pint % q, -1, q) for q in qm], qm))
    return out


def hmult(a, b, K: OKeys):
    """ckks.py:605-613"""
    P = K.P
    mods = P.qs[: a.shape[1]]
    d0 = mul(a[0], b[0], mods)
    d1 = add(mul(a[0], b[1], mods), mul(a[1], b[0], mods), mods)
    d2 = mul(a[1], b[1], mods)
    k0, k1 = keyswitch(intt(d2, mods), K.rlk, P)
    return np.stack([add(d0, k0, mods), add(d1, k1, mods)])


def rescale(ct, P: OParams):
    """ckks.py:506-528"""
    l = ct.shape[1] - 1
    qt = P.qs[l]
    rem = P.qs[:l]
    out = []
    for poly in ct:
        top = intt(poly[l:l + 1], [qt])[0]
        big = top > np.uint64(qt // 2)
        lift = np.stack([np.where(big, (top % np.uint64(q) + np.uint64(q - qt % q)) % np.uint64(q),
                                  top % np.uint64(q)) for q in rem])
        diff = sub(poly[:l], ntt(lift, rem), rem)
        out.append(scalar_mul(diff, [pow(qt, -1, q) for q in rem], rem))
    return np.stack(out)


def rotation_plan(step, available, slots):
    step %= slots
    if step == 0:
        return []
    if step in available:
        return [step]
    plan, rem = [], step
    for s in sorted(available, reverse=True):
        while rem >= s:
            plan.append(s)
            rem -= s
    if rem:
        raise KeyError(step)
    return plan


def rotate(ct, k, K: OKeys):
    """rotate / _apply_step ckks.py:620-657"""
    P = K.P
    mods = P.qs[: ct.shape[1]]
    for st in rotation_plan(k, tuple(K.gks), P.slots):
        g = galois(st, P.n)
        c0 = ntt(automorphism(intt(ct[0], mods), g, mods), mods)
        a = automorphism(intt(ct[1], mods), g, mods)
        k0, k1 = keyswitch(a, K.gks[st], P)
        ct = np.stack([add(c0, k0, mods), k1])
    return ct


def pmult(ct, pt, mods):
    return np.stack([mul(ct[0], pt, mods), mul(ct[1], pt, mods)])
