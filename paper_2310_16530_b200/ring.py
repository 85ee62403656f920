"""RNS polynomials resident in HBM (drop-in for hcnn.ring).

Same public names and semantics as /root/reference/pkg/src/hcnn/ring.py, but
an ``RnsPoly`` holds its residue matrix as a CUDA tensor (uint64 bit
patterns in an int64 tensor of shape [nlimbs, N], limb-major like the
reference's ``coeffs``) and every arithmetic function runs a CUDA kernel
through the C ABI.  ``.coeffs`` materialises a host uint64 copy on demand.

Host-only pieces that fix the parameters and therefore must match the
reference exactly -- the NTT-prime search (ring.py:84-126), the Montgomery
constants (ring.py:32-72) and the seeded samplers (ring.py:446-468) -- are
restated here on the host; twiddle tables are derived from the same psi
rule inside the engine (include/hcnn_b200.h, hcnn_ctx_create).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Iterable, Sequence

import numpy as np
import torch

from .engine import DeviceContext, context_for, to_device_u64, to_host_u64
from .errors import BasisError, DomainError, ParameterError

_MASK64 = (1 << 64) - 1


class Domain(Enum):
    COEFF = "coeff"
    EVAL = "eval"


@dataclass(frozen=True)
class Modulus:
    """NTT prime < 2^62 with reduction constants (ring.py:32-72)."""

    q: int
    ninv: int
    r2: int
    barrett_mu: int

    @classmethod
    def make(cls, q: int) -> "Modulus":
        if not (2 < q < (1 << 62)):
            raise ParameterError(f"modulus {q} outside (2, 2^62)")
        return cls(q=q, ninv=(-pow(q, -1, 1 << 64)) & _MASK64, r2=(1 << 128) % q,
                   barrett_mu=(1 << 128) // q)

    def mul(self, a: int, b: int) -> int:
        assert 0 <= a < self.q and 0 <= b < self.q
        t = a * b
        r = t - ((t * self.barrett_mu) >> 128) * self.q
        return r - self.q if r >= self.q else r

    def to_mont(self, a: int) -> int:
        return (a << 64) % self.q

    def pow(self, a: int, e: int) -> int:
        return pow(a, e, self.q)

    def inv(self, a: int) -> int:
        return pow(a, -1, self.q)


def mod_mul(a: int, b: int, mod: Modulus) -> int:
    return mod.mul(a, b)


# ---------------------------------------------------------------------------
# primes
# ---------------------------------------------------------------------------

_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin; exact for n < 3.3e24 (all moduli here)."""
    if n < 2:
        return False
    for p in _MR_BASES:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in _MR_BASES:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def find_ntt_primes(n: int, bits: int, count: int, avoid: Iterable[int] = (),
                    alternate: bool = False) -> list[int]:
    """Primes = 1 mod 2N near 2^bits, the same sequence as ring.py:84-126:
    walk down (and, with ``alternate``, up on odd picks) from the largest
    candidate <= 2^bits in steps of 2N."""
    step = 2 * n
    base = 1 << bits
    anchor = base - ((base - 1) % step)
    taken = set(avoid)
    lo, hi = anchor, anchor + step
    out: list[int] = []
    for i in range(count):
        if alternate and i % 2 == 1:
            while True:
                hi += step
                if hi.bit_length() > bits + 1:
                    raise ParameterError(f"ran out of {bits}-bit primes above 2^{bits}")
                if hi not in taken and is_prime(hi):
                    p = hi
                    break
        else:
            while True:
                lo -= step
                if lo.bit_length() < bits - 1:
                    raise ParameterError(f"ran out of {bits}-bit primes below 2^{bits}")
                if lo not in taken and is_prime(lo):
                    p = lo
                    break
        taken.add(p)
        out.append(p)
    return out


def _bit_reverse(x: int, bits: int) -> int:
    return int(format(x, f"0{bits}b")[::-1], 2) if bits else 0


# ---------------------------------------------------------------------------
# RnsPoly on the device
# ---------------------------------------------------------------------------

def _basis_in(ctx: DeviceContext, mods: tuple[Modulus, ...]) -> tuple[int, int] | None:
    qs = [m.q for m in mods]
    nq = 0
    while nq < len(qs) and nq < ctx.Lq and qs[nq] == ctx.q_list[nq]:
        nq += 1
    rest = qs[nq:]
    if len(rest) > ctx.K or tuple(rest) != ctx.p_list[: len(rest)]:
        return None
    return nq, len(rest)


class RnsPoly:
    """Residue matrix [len(mods), N] on the device plus the domain flag.

    Treated as immutable like the reference's (ring.py:204-239); every
    operation writes a fresh tensor.
    """

    __slots__ = ("mods", "data", "domain", "ctx", "nq", "np")

    def __init__(self, mods, data, domain: Domain, ctx: DeviceContext | None = None,
                 basis: tuple[int, int] | None = None):
        mods = tuple(mods)
        if len(mods) == 0:
            raise BasisError("empty basis")
        if isinstance(data, np.ndarray):
            if data.dtype != np.uint64:
                raise ParameterError("residues must be uint64")
            if data.ndim != 2 or data.shape[0] != len(mods):
                raise BasisError("residue matrix shape disagrees with basis")
            n = data.shape[1]
            if ctx is None:
                ctx = context_for(n, [m.q for m in mods])
            data = to_device_u64(data, ctx.device)
        else:
            if data.dim() != 2 or data.shape[0] != len(mods):
                raise BasisError("residue matrix shape disagrees with basis")
            if ctx is None:
                ctx = context_for(data.shape[1], [m.q for m in mods])
        if basis is None:
            basis = _basis_in(ctx, mods)
            if basis is None:
                raise BasisError("modulus list is not a basis of the device context")
        self.mods = mods
        self.data = data
        self.domain = domain
        self.ctx = ctx
        self.nq, self.np = basis

    @property
    def n(self) -> int:
        return self.data.shape[1]

    @property
    def nlimbs(self) -> int:
        return len(self.mods)

    @property
    def coeffs(self) -> np.ndarray:
        """Host uint64 copy of the residues (synchronises)."""
        return to_host_u64(self.data)

    def qs(self) -> tuple[int, ...]:
        return tuple(m.q for m in self.mods)

    def copy(self) -> "RnsPoly":
        return RnsPoly(self.mods, self.data.clone(), self.domain, self.ctx, (self.nq, self.np))

    def limbs(self, idx: slice) -> "RnsPoly":
        mods = self.mods[idx]
        data = self.data[idx].clone()
        return RnsPoly(mods, data, self.domain, self.ctx if _basis_in(self.ctx, mods) else None)

    def _new(self, data: torch.Tensor, domain: Domain | None = None) -> "RnsPoly":
        return RnsPoly(self.mods, data, self.domain if domain is None else domain, self.ctx,
                       (self.nq, self.np))


def zero_poly(mods: Sequence[Modulus], n: int, domain: Domain = Domain.COEFF,
              ctx: DeviceContext | None = None) -> RnsPoly:
    mods = tuple(mods)
    ctx = ctx or context_for(n, [m.q for m in mods])
    return RnsPoly(mods, ctx.zeros(len(mods), n), domain, ctx)


def from_int_coeffs(values: Sequence[int], mods: Sequence[Modulus], n: int,
                    ctx: DeviceContext | None = None) -> RnsPoly:
    if len(values) > n:
        raise ParameterError("too many coefficients")
    vals = list(values) + [0] * (n - len(values))
    rows = np.array([[v % m.q for v in vals] for m in mods], dtype=np.uint64)
    return RnsPoly(tuple(mods), rows, Domain.COEFF, ctx)


def _check_same(a: RnsPoly, b: RnsPoly):
    if a.qs() != b.qs():
        raise BasisError("operand bases differ")
    if a.domain != b.domain:
        raise DomainError("operand domains differ")


def _same_ctx(a: RnsPoly, b: RnsPoly) -> torch.Tensor:
    if b.ctx is a.ctx:
        return b.data
    return b.data  # same modulus list -> identical residue semantics


def poly_add(a: RnsPoly, b: RnsPoly) -> RnsPoly:
    _check_same(a, b)
    return a._new(a.ctx.binop("add", a.data, _same_ctx(a, b), a.nq, a.np))


def poly_sub(a: RnsPoly, b: RnsPoly) -> RnsPoly:
    _check_same(a, b)
    return a._new(a.ctx.binop("sub", a.data, _same_ctx(a, b), a.nq, a.np))


def poly_neg(a: RnsPoly) -> RnsPoly:
    return a._new(a.ctx.unop("neg", a.data, a.nq, a.np))


def poly_mul_pointwise(a: RnsPoly, b: RnsPoly) -> RnsPoly:
    """Hadamard product in the evaluation domain (ring.py:287-296)."""
    _check_same(a, b)
    if a.domain is not Domain.EVAL:
        raise DomainError("pointwise product requires Evaluation domain")
    return a._new(a.ctx.binop("mul", a.data, _same_ctx(a, b), a.nq, a.np))


def to_mont_rows(p: RnsPoly) -> torch.Tensor:
    """Residues lifted to Montgomery form (device tensor, ring.py:299-304)."""
    return p.ctx.unop("to_mont", p.data, p.nq, p.np)


def poly_mul_mont_rows(a: RnsPoly, rows_mont) -> RnsPoly:
    if a.domain is not Domain.EVAL:
        raise DomainError("pointwise product requires Evaluation domain")
    rows = rows_mont if isinstance(rows_mont, torch.Tensor) else to_device_u64(rows_mont, a.ctx.device)
    return a._new(a.ctx.binop("mul_mont", a.data, rows[: a.nlimbs].contiguous(), a.nq, a.np))


def ntt_forward(p: RnsPoly) -> RnsPoly:
    if p.domain is not Domain.COEFF:
        raise DomainError("ntt_forward expects Coefficient domain")
    out = p.data.clone()
    p.ctx.ntt(out, p.nq, p.np, inverse=False)
    return p._new(out, Domain.EVAL)


def ntt_inverse(p: RnsPoly) -> RnsPoly:
    if p.domain is not Domain.EVAL:
        raise DomainError("ntt_inverse expects Evaluation domain")
    out = p.data.clone()
    p.ctx.ntt(out, p.nq, p.np, inverse=True)
    return p._new(out, Domain.COEFF)


def _mod_indices(ctx: DeviceContext, qs: Sequence[int]) -> list[int] | None:
    allm = list(ctx.q_list) + list(ctx.p_list)
    try:
        return [allm.index(q) for q in qs]
    except ValueError:
        return None


def base_convert(p: RnsPoly, new_mods: Sequence[Modulus]) -> RnsPoly:
    """Centred fast base conversion (ring.py:378-398), bit-exact."""
    if p.domain is not Domain.COEFF:
        raise DomainError("base_convert expects Coefficient domain")
    dst = tuple(new_mods)
    if len(dst) == 0:
        raise BasisError("empty target basis")
    ctx = p.ctx
    si = _mod_indices(ctx, p.qs())
    di = _mod_indices(ctx, [m.q for m in dst])
    data = p.data
    if si is None or di is None:
        union = list(dict.fromkeys(list(p.qs()) + [m.q for m in dst]))
        ctx = context_for(p.n, union)
        si = [union.index(q) for q in p.qs()]
        di = [union.index(m.q) for m in dst]
    out = ctx.base_convert(data, si, di)[0]
    return RnsPoly(dst, out, Domain.COEFF, ctx if _basis_in(ctx, dst) else None)


def automorphism(p: RnsPoly, g: int) -> RnsPoly:
    """X -> X^g in the coefficient domain (ring.py:427-439)."""
    if p.domain is not Domain.COEFF:
        raise DomainError("automorphism expects Coefficient domain")
    if g % 2 == 0:
        raise ParameterError("automorphism exponent must be odd")
    return p._new(p.ctx.automorphism(p.data, g % (2 * p.n), p.nq, p.np, eval_domain=False))


def automorphism_eval(p: RnsPoly, g: int) -> RnsPoly:
    """The same automorphism applied to an evaluation-domain poly: a pure
    index permutation of the bit-reversed NTT output."""
    if p.domain is not Domain.EVAL:
        raise DomainError("automorphism_eval expects Evaluation domain")
    if g % 2 == 0:
        raise ParameterError("automorphism exponent must be odd")
    return p._new(p.ctx.automorphism(p.data, g % (2 * p.n), p.nq, p.np, eval_domain=True))


# ---------------------------------------------------------------------------
# seeded sampling: host RNG (identical draw order to ring.py:446-468), device
# replication
# ---------------------------------------------------------------------------

def sample_small(n: int, dist: str, rng: np.random.Generator, sigma: float = 3.2) -> np.ndarray:
    if dist == "ternary":
        return rng.integers(-1, 2, size=n, dtype=np.int64)
    if dist == "gaussian":
        return np.rint(rng.normal(0.0, sigma, size=n)).astype(np.int64)
    raise ParameterError(f"unknown distribution {dist!r}")


def sample_uniform_rows(mods: Sequence[Modulus], n: int, rng: np.random.Generator) -> np.ndarray:
    out = np.empty((len(mods), n), dtype=np.uint64)
    for i, m in enumerate(mods):
        out[i] = rng.integers(0, m.q, size=n, dtype=np.uint64)
    return out


def sample_poly(mods: Sequence[Modulus], n: int, dist: str, rng: np.random.Generator,
                sigma: float = 3.2, ctx: DeviceContext | None = None) -> RnsPoly:
    mods = tuple(mods)
    if dist == "uniform":
        return RnsPoly(mods, sample_uniform_rows(mods, n, rng), Domain.COEFF, ctx)
    small = sample_small(n, dist, rng, sigma)
    ctx = ctx or context_for(n, [m.q for m in mods])
    basis = _basis_in(ctx, mods)
    if basis is None:
        raise BasisError("modulus list is not a basis of the device context")
    rows = torch.from_numpy(small).to(ctx.torch_device)
    data = ctx.from_signed(rows, basis[0], basis[1])[0]
    return RnsPoly(mods, data, Domain.COEFF, ctx, basis)


# ---------------------------------------------------------------------------
# CRT reconstruction (host; decode / test support, ring.py:475-519)
# ---------------------------------------------------------------------------

def crt_consts(mods: Sequence[Modulus]) -> tuple[int, list[int]]:
    big_q = 1
    for m in mods:
        big_q *= m.q
    consts = []
    for m in mods:
        punc = big_q // m.q
        consts.append(punc * pow(punc % m.q, -1, m.q))
    return big_q, consts


def crt_rows(rows: np.ndarray, mods: Sequence[Modulus], bound_bits: int | None = None) -> np.ndarray:
    """Centred integers (numpy object array) from host residue rows, using the
    limb prefix rule of ring.py:489-497."""
    use = len(mods)
    if bound_bits is not None:
        acc = 0
        for i, m in enumerate(mods):
            acc += m.q.bit_length() - 1
            if acc > bound_bits + 2:
                use = i + 1
                break
    mods = tuple(mods)[:use]
    big_q, consts = crt_consts(mods)
    total = np.zeros(rows.shape[1], dtype=object)
    for i in range(use):
        total = total + rows[i].astype(object) * consts[i]
    total = total % big_q
    half = big_q // 2
    return np.where(total > half, total - big_q, total)


def to_int_coeffs(p: RnsPoly, bound_bits: int | None = None) -> list[int]:
    if p.domain is not Domain.COEFF:
        raise DomainError("reconstruction expects Coefficient domain")
    return [int(v) for v in crt_rows(p.coeffs, p.mods, bound_bits)]
