"""Full-slot CKKS bootstrapping (BASELINE config 3).

The reference has no bootstrapping -- its refresh slot is the insecure
``debug_refresh`` (ckks.py:667-690, graph.py:493-497) -- so this module has
no oracle: **parity unpinned**.  It is validated by decrypt-and-compare
(tests/test_gpu_bootstrap.py) and by plaintext simulation of every linear
stage (tests/test_bootstrap_plain.py).

Pipeline, all on the engine's primitives:

1. ``mod_drop`` to level 0, exact integer scale-up so the message sits
   ``message_ratio_bits`` below q0, ``mod_raise`` to the top of the chain:
   the ciphertext now decrypts to t = m + q0*I, |I| < k_bound (sparse
   ternary secret of weight h).
2. CoeffToSlot: the inverse special FFT (HEAAN's decomposition of the
   canonical embedding, slots left in bit-reversed order) as
   ``len(cts_stages)`` level-collapsed sparse matrices; each is applied as a
   baby-step/giant-step diagonal product -- baby rotations hoisted on one
   ModUp (``rotate_many``), each giant group one fused MAC kernel
   (``mac_terms``), one rescale per level.  The constant Delta/(2 q0 B) is
   folded into the first matrix, so the slots hold (t_lo + i t_hi)/(2 q0 B).
3. Conjugation splits real and imaginary parts: y_lo = u + conj(u),
   y_hi = -X^(N/2) (u - conj(u)) -- slot values t/(q0 B) in [-1, 1].
4. EvalMod on each: Chebyshev interpolant of cos(2pi(B y - 1/4)/2^r),
   then r double-angle steps give sin(2pi x) ~ 2pi m/q0.  The evaluator
   keeps every addition between equal scales exactly (constants are folded
   in as integers at compensating scales), since a relative scale error
   would multiply the large q0*I part.
5. v = v_lo + X^(N/2) v_hi, then SlotToCoeff (the forward special FFT with
   q0/(2 pi Delta) folded in) returns the message at ``output_level`` with
   the input's scale.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import torch
from numpy.polynomial import chebyshev as npcheb

from . import ckks
from .ckks import Ciphertext, CkksParams, KeySet
from .errors import KeyError_, LevelError, ParameterError


def boot_params(name: str, n: int, app_levels: int, cfg: "BootConfig | None" = None, q0_bits: int = 60,
                app_bits: int = 40, big_bits: int = 58, n_special: int = 4,
                special_bits: "int | tuple[int, ...]" = 61) -> CkksParams:
    """A bootstrappable chain: q0, `app_levels` + StC levels of app_bits,
    then EvalMod + CtS levels of big_bits (top of the chain), Delta = 2^app_bits.
    Large top primes keep the CtS/EvalMod plaintext products precise.
    `special_bits` may list one size per special prime (n_special is then
    its length): P must exceed the largest key-switch digit product, so one
    wide special next to narrow ones covers a digit holding q0."""
    from .ring import Modulus, find_ntt_primes
    cfg = cfg or BootConfig()
    n_small = app_levels + len(cfg.stc_stages)
    n_big = cfg.evalmod_depth() + len(cfg.cts_stages)
    q0 = find_ntt_primes(n, q0_bits, 1)
    small = find_ntt_primes(n, app_bits, n_small, avoid=q0, alternate=True)
    big = find_ntt_primes(n, big_bits, n_big, avoid=q0 + small, alternate=True)
    sizes = [special_bits] * n_special if isinstance(special_bits, int) else list(special_bits)
    ps: list[int] = []
    for b in sorted(set(sizes), key=sizes.index):
        ps += find_ntt_primes(n, b, sizes.count(b), avoid=q0 + small + big + ps, alternate=b <= 41)
    return CkksParams(name=name, n=n, q_mods=tuple(Modulus.make(q) for q in q0 + small + big),
                      p_mods=tuple(Modulus.make(p) for p in ps), delta=float(2 ** app_bits))


@dataclass(frozen=True)
class BootConfig:
    cts_stages: tuple[int, ...] = (5, 5, 5)   # FFT stages merged per level, application order
    stc_stages: tuple[int, ...] = (5, 5, 5)
    k_bound: int = 16                         # |I| < k_bound after ModRaise
    double_angle: int = 3
    degree: int = 59                          # Chebyshev degree before the double angles
    message_ratio_bits: int = 12              # q0 / scaled-up Delta ~ 2^bits
    secret_weight: int = 64
    # baby steps per BSGS level matrix (None: ~sqrt of the diagonal span).
    # Double hoisting makes babies cheap (no ModDown each) and giants dear
    # (a ModUp each), so more babies / fewer giants wins.
    bsgs_baby: int | None = 16
    double_hoist: bool = True
    # linear-transform levels end with one base conversion dividing by P q_l
    # (ModDown + rescale fused, hcnn_moddown_rescale_batch)
    fused_moddown_rescale: bool = True

    def evalmod_depth(self) -> int:
        return max(1, math.ceil(math.log2(self.degree))) + 1 + self.double_angle

    def depth(self) -> int:
        return len(self.cts_stages) + self.evalmod_depth() + len(self.stc_stages)


# ---------------------------------------------------------------------------
# special FFT factorisation (host, exact float64 matrices)
# ---------------------------------------------------------------------------

def special_fft_stage(n: int, length: int, inverse: bool = False) -> sp.csr_matrix:
    """Butterfly stage of the size-n special FFT: within blocks of `length`,
    (a, a + length/2) -> (x_a + w_j x_b, x_a - w_j x_b), w_j = exp(pi i
    (5^j mod 4 length) / (2 length)).  The product F_n ... F_2 composed with
    the bit reversal is U0[j, k] = zeta^(5^j k), zeta = exp(i pi / N): the
    slot map of the reference's encoding (ckks.py:241-308)."""
    h = length // 2
    j = np.arange(h)
    w = np.exp(1j * np.pi * (np.array([pow(5, int(t), 4 * length) for t in j]) / (2.0 * length)))
    starts = np.arange(0, n, length)
    a = (starts[:, None] + j[None, :]).ravel()
    b = a + h
    ww = np.tile(w, len(starts))
    if not inverse:
        rows = np.concatenate([a, a, b, b])
        cols = np.concatenate([a, b, a, b])
        vals = np.concatenate([np.ones_like(ww), ww, np.ones_like(ww), -ww])
    else:
        rows = np.concatenate([a, a, b, b])
        cols = np.concatenate([a, b, a, b])
        vals = np.concatenate([0.5 * np.ones_like(ww), 0.5 * np.ones_like(ww), 0.5 / ww, -0.5 / ww])
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n), dtype=np.complex128)


def bit_reverse_perm(n: int) -> np.ndarray:
    bits = n.bit_length() - 1
    return np.array([int(format(i, f"0{bits}b")[::-1], 2) if bits else 0 for i in range(n)])


def embedding_matrix(n_ring: int) -> np.ndarray:
    """U0[j, k] = zeta^(5^j k) (dense; tests only)."""
    n = n_ring // 2
    e = np.array([pow(5, j, 2 * n_ring) for j in range(n)])
    return np.exp(1j * np.pi * np.outer(e, np.arange(n)) / n_ring)


def stc_groups(n: int, stages: tuple[int, ...], const: complex) -> list[sp.csr_matrix]:
    """SlotToCoeff = const * F_n ... F_2 (slots in bit-reversed order),
    grouped into level matrices in application order."""
    lens = [1 << s for s in range(1, n.bit_length())]
    if sum(stages) != len(lens):
        raise ParameterError(f"stc stages {stages} must sum to log2(slots)={len(lens)}")
    groups, pos = [], 0
    for g, cnt in enumerate(stages):
        m = sp.identity(n, dtype=np.complex128, format="csr")
        for length in lens[pos:pos + cnt]:
            m = special_fft_stage(n, length) @ m
        if g == 0:
            m = m * const
        groups.append(m.tocsr())
        pos += cnt
    return groups


def cts_groups(n: int, stages: tuple[int, ...], const: complex) -> list[sp.csr_matrix]:
    """CoeffToSlot = const * (2F_2)^-1... : the inverse of StC's product with
    every stage scaled by 2 (unit-magnitude entries), i.e. n * BR * U0^-1."""
    lens = [1 << s for s in range(1, n.bit_length())][::-1]
    if sum(stages) != len(lens):
        raise ParameterError(f"cts stages {stages} must sum to log2(slots)={len(lens)}")
    groups, pos = [], 0
    for g, cnt in enumerate(stages):
        m = sp.identity(n, dtype=np.complex128, format="csr")
        for length in lens[pos:pos + cnt]:
            m = (2.0 * special_fft_stage(n, length, inverse=True)) @ m
        if g == 0:
            m = m * const
        groups.append(m.tocsr())
        pos += cnt
    return groups


@dataclass
class DiagPlan:
    """Baby-step / giant-step schedule of one level matrix:
    M v = sum_g rot_{g n1 s}( sum_b P_{g,b} (.) rot_{b s}(v) )."""

    n: int
    stride: int
    n1: int
    babies: list[int]                          # rotation amounts b*s
    giants: dict[int, list[tuple[int, np.ndarray]]]  # giant amount -> [(baby amount, pre-rotated diag)]


def diag_plan(m: sp.csr_matrix, n1: int | None = None) -> DiagPlan:
    n = m.shape[0]
    coo = m.tocoo()
    keep = np.abs(coo.data) > 1e-300
    rows, cols, vals = coo.row[keep], coo.col[keep], coo.data[keep]
    d = (cols - rows) % n
    diags: dict[int, np.ndarray] = {}
    for off in np.unique(d):
        sel = d == off
        v = np.zeros(n, dtype=np.complex128)
        v[rows[sel]] = vals[sel]
        diags[int(off)] = v
    signed = {off: (off if off <= n // 2 else off - n) for off in diags}
    nz = [abs(k) for k in signed.values() if k]
    stride = int(np.gcd.reduce(nz)) if nz else 1
    ks = {off: k // stride for off, k in signed.items()}
    span = max(ks.values()) - min(ks.values()) + 1
    if n1 is None:
        n1 = 1 << max(0, math.ceil(math.log2(math.sqrt(span))))
    giants: dict[int, list] = {}
    babies: set[int] = set()
    for off, k in ks.items():
        b = k % n1
        g = (k - b) // n1
        gamt = (g * n1 * stride) % n
        pre = np.roll(diags[off], g * n1 * stride)
        giants.setdefault(gamt, []).append(((b * stride) % n, pre))
        babies.add((b * stride) % n)
    return DiagPlan(n, stride, n1, sorted(babies), giants)


def plan_rotations(plans: list[DiagPlan]) -> set[int]:
    steps = set()
    for p in plans:
        steps |= {b for b in p.babies if b}
        steps |= {g for g in p.giants if g}
    return steps


def apply_plain(plans: list[DiagPlan], v: np.ndarray) -> np.ndarray:
    """Host simulation of the homomorphic BSGS application (tests)."""
    for p in plans:
        out = np.zeros_like(v)
        for gamt, terms in p.giants.items():
            inner = np.zeros_like(v)
            for bamt, pre in terms:
                inner = inner + pre * np.roll(v, -bamt)
            out = out + np.roll(inner, -gamt)
        v = out
    return v


def evalmod_coeffs(cfg: BootConfig) -> np.ndarray:
    """Chebyshev coefficients (on y in [-1,1]) of cos(2 pi (B y - 1/4) / 2^r)."""
    B = cfg.k_bound + 1
    r = cfg.double_angle
    f = lambda y: np.cos(2 * np.pi * (B * y - 0.25) / (1 << r))
    return npcheb.chebinterpolate(f, cfg.degree)


def evalmod_plain(cfg: BootConfig, y: np.ndarray) -> np.ndarray:
    c = npcheb.chebval(y, evalmod_coeffs(cfg))
    for _ in range(cfg.double_angle):
        c = 2 * c * c - 1
    return c


# ---------------------------------------------------------------------------
# exact-scale homomorphic evaluator
# ---------------------------------------------------------------------------

class _Exact:
    """hmult / constants with scales tracked so that additions always meet
    equal scales (to float precision)."""

    def __init__(self, params: CkksParams, ks: KeySet, fused: bool = False):
        self.params, self.ks = params, ks
        self.ctx = params.ctx
        self.fused = fused  # products through hcnn_hmult_rescale_batch (one ModDown for relin + rescale)

    def drop(self, a: Ciphertext, level: int) -> Ciphertext:
        return a if a.level == level else ckks.mod_drop(a, level)

    def mul(self, a: Ciphertext, b: Ciphertext) -> Ciphertext:
        lvl = min(a.level, b.level)
        if lvl < 1:
            raise LevelError("bootstrap evaluator ran out of levels")
        a, b = self.drop(a, lvl), self.drop(b, lvl)
        if self.fused:
            out = self.ctx.hmult_rescale(a.data, b.data, lvl, self.ks.rlk.rows_b, self.ks.rlk.rows_a)
            return Ciphertext(out, a.scale * b.scale / self.params.q_mods[lvl].q, a.n, a.params)
        return ckks.rescale(ckks.hmult(a, b, self.ks), self.params)

    def double(self, a: Ciphertext) -> Ciphertext:
        return Ciphertext(self.ctx.binop("add", a.data, a.data, a.level + 1), a.scale, a.n, a.params)

    def add(self, a: Ciphertext, b: Ciphertext, sub: bool = False) -> Ciphertext:
        lvl = min(a.level, b.level)
        a, b = self.drop(a, lvl), self.drop(b, lvl)
        if abs(a.scale - b.scale) > 1e-9 * a.scale:
            raise ParameterError(f"exact evaluator: scales {a.scale} vs {b.scale}")
        out = self.ctx.binop("sub" if sub else "add", a.data, b.data, lvl + 1)
        return Ciphertext(out, a.scale, a.n, a.params)

    def _int_consts(self, k: int, level: int) -> list[int]:
        return [k % m.q for m in self.params.mods_at(level)]

    def add_const(self, a: Ciphertext, c: float, inplace: bool = False) -> Ciphertext:
        """a + c exactly at a's scale (every c0 of a batch)."""
        out = a.data if inplace else a.data.clone()
        self.ctx.scalar_mac([], [], a.level, out=out, accumulate=True, c0_add=int(round(c * a.scale)))
        return Ciphertext(out, a.scale, a.n, a.params)

    def mul_const(self, a: Ciphertext, c: float, target_scale: float) -> Ciphertext:
        """a * c, rescaled, landing exactly on target_scale (one level)."""
        if a.level < 1:
            raise LevelError("bootstrap evaluator ran out of levels")
        q = self.params.q_mods[a.level].q
        s_c = target_scale * q / a.scale
        k = int(round(c * s_c))
        out = self.ctx.scalar_mul(a.data, self._int_consts(k, a.level), a.level + 1)
        return ckks.rescale(Ciphertext(out, a.scale * s_c, a.n, a.params), self.params)


    def cheb_product(self, a: Ciphertext, b: Ciphertext, t1: Ciphertext | None) -> Ciphertext:
        """T_{i+j} = 2 T_i T_j - T_{|i-j|} with |i-j| in {0, 1}: the doubling
        and the T_1 (or constant) correction are folded into one scalar-MAC
        before the single rescale."""
        lvl = min(a.level, b.level)
        if lvl < 1:
            raise LevelError("bootstrap evaluator ran out of levels")
        p = ckks.hmult(self.drop(a, lvl), self.drop(b, lvl), self.ks)
        two = [2] * (lvl + 1)
        if t1 is None:  # 2 T_a^2 - 1: the constant at the product's scale
            d = self.ctx.scalar_mac([p.data], [two], lvl, c0_add=-int(round(p.scale)))
        else:
            k = int(round(p.scale / t1.scale))
            d = self.ctx.scalar_mac([p.data, t1.data], [two, [-k] * (lvl + 1)], lvl)
        return ckks.rescale(Ciphertext(d, p.scale, p.n, p.params), self.params)

    def lincomb(self, terms: list[tuple[Ciphertext, float]], c0: float, level: int, scale: float) -> Ciphertext:
        """c0 + sum c_i t_i landing exactly on (level, scale): one scalar-MAC
        over the level-dropped prefixes at level+1, one rescale."""
        lvl = level + 1
        q = self.params.q_mods[lvl].q
        srcs = [t.data for t, _ in terms]
        consts = [[int(round(c * scale * q / t.scale))] * (lvl + 1) for t, c in terms]
        acc = self.ctx.scalar_mac(srcs, consts, lvl, c0_add=int(round(c0 * scale * q)))
        out = ckks.rescale(Ciphertext(acc, scale * q, terms[0][0].n, terms[0][0].params), self.params)
        return Ciphertext(out.data, scale, out.n, out.params)


def cheb_divide(c: np.ndarray, m: int) -> tuple[np.ndarray, np.ndarray]:
    """p = r + T_m q for deg p < 2m (T_m T_j = (T_{m+j} + T_{m-j})/2)."""
    d = len(c) - 1
    q = np.zeros(d - m + 1)
    q[0] = c[m]
    q[1:] = 2.0 * c[m + 1:]
    r = np.array(c[:m], dtype=np.float64)
    for i in range(1, m):
        if 2 * m - i <= d:
            r[i] -= c[2 * m - i]
    return q, r


def _trim(c: np.ndarray, tol: float) -> np.ndarray:
    d = len(c) - 1
    while d > 0 and abs(c[d]) <= tol:
        d -= 1
    return np.asarray(c[: d + 1], dtype=np.float64)


def bsgs_split(c: np.ndarray, baby: int, tol: float = 1e-14):
    """The recursion tree of the baby-step giant-step evaluation: a leaf is
    the coefficient vector itself (degree < baby), a node is
    (m, q_tree, r_tree) with p = r + T_m q."""
    c = _trim(c, tol)
    d = len(c) - 1
    if d < baby:
        return c
    m = baby
    while 2 * m <= d:
        m *= 2
    q, r = cheb_divide(c, m)
    return (m, bsgs_split(q, baby, tol), bsgs_split(r, baby, tol))


def bsgs_eval_plain(tree, y: np.ndarray) -> np.ndarray:
    """Host mirror of the homomorphic evaluation order (tests)."""
    if isinstance(tree, np.ndarray):
        return npcheb.chebval(y, tree)
    m, q, r = tree
    tm = npcheb.chebval(y, np.eye(m + 1)[m])
    return bsgs_eval_plain(r, y) + tm * bsgs_eval_plain(q, y)


def bsgs_powers(tree, baby: int) -> set[int]:
    if isinstance(tree, np.ndarray):
        return set(range(1, len(tree)))
    m, q, r = tree
    return {m} | bsgs_powers(q, baby) | bsgs_powers(r, baby)


def eval_chebyshev(ev: _Exact, y: Ciphertext, coeffs: np.ndarray, target_scale: float,
                   baby: int = 8, tol: float = 1e-14) -> Ciphertext:
    """p(y) = sum c_i T_i(y) by baby-step giant-step: T_1..T_{baby-1} and the
    giants T_{baby 2^j} (each T one hmult with the 2x and T_1 correction
    fused), then p = r + T_m q recursively; every leaf is one scalar-MAC and
    one rescale, every split one hmult.  Depth ceil(log2(d+1)) + 1, about
    2 sqrt(d) + log d ciphertext products instead of d."""
    tree = bsgs_split(coeffs, baby, tol)
    T: dict[int, Ciphertext] = {1: y}

    def power(i: int) -> Ciphertext:
        if i not in T:
            a, b = i // 2, i - i // 2
            T[i] = ev.cheb_product(power(a), power(b), None if a == b else T[1])
        return T[i]

    for i in sorted(bsgs_powers(tree, baby)):
        power(i)

    def top(t) -> int:  # highest output level the subtree can land on
        if isinstance(t, np.ndarray):
            return min((T[i].level for i in range(1, len(t))), default=y.level) - 1
        m, q, r = t
        return min(T[m].level - 1, top(q) - 1, top(r))

    def run(t, level: int, scale: float) -> Ciphertext:
        if isinstance(t, np.ndarray):
            terms = [(T[i], float(t[i])) for i in range(1, len(t))] or [(T[1], 0.0)]
            return ev.lincomb(terms, float(t[0]), level, scale)
        m, q, r = t
        lvl = level + 1
        qp = ev.params.q_mods[lvl].q
        tm = T[m]
        qv = run(q, lvl, scale * qp / tm.scale)
        prod = ckks.rescale(ckks.hmult(ev.drop(tm, lvl), qv, ev.ks), ev.params)
        return ev.add(Ciphertext(prod.data, scale, prod.n, prod.params), run(r, level, scale))

    level = top(tree)
    if level < 0:
        raise LevelError("bootstrap evaluator ran out of levels")
    return run(tree, level, target_scale)


# ---------------------------------------------------------------------------
# bootstrapper
# ---------------------------------------------------------------------------

class Bootstrapper:
    """Precomputed CtS/StC diagonal plans, EvalMod coefficients and the
    level schedule for one parameter set; ``bootstrap(ct)`` refreshes a
    ciphertext of any level to ``output_level``.

    Constants are applied as exact scale relabels (a ciphertext with scale
    S and slots z is the same ciphertext as scale S/c with slots c z), so
    every diagonal has unit-magnitude entries and linear levels keep the
    scale (plaintext scale = the level's prime)."""

    def __init__(self, params: CkksParams, cfg: BootConfig = BootConfig()):
        self.params, self.cfg = params, cfg
        n = params.slots
        self.q0 = params.q_mods[0].q
        self.B = cfg.k_bound + 1
        self.cts_plans = [diag_plan(m, cfg.bsgs_baby) for m in cts_groups(n, cfg.cts_stages, 1.0)]
        self.stc_plans = [diag_plan(m, cfg.bsgs_baby) for m in stc_groups(n, cfg.stc_stages, 1.0)]
        self.cheb = evalmod_coeffs(cfg)
        self.output_level = params.max_level - cfg.depth()
        if self.output_level < 0:
            raise ParameterError(f"chain too short: bootstrapping needs {cfg.depth()} levels, "
                                 f"have {params.max_level}")
        # EvalMod works at the scale of the first EvalMod level's prime
        self.eval_scale = float(params.q_mods[params.max_level - len(cfg.cts_stages)].q)
        self._masks: dict = {}
        self.phase_hook = None  # optional callable(phase name) between pipeline phases (profiling)
        pprod = 1
        for m in params.p_mods:
            pprod *= m.q
        self._pmod_q = [pprod % m.q for m in params.q_mods]

    # -- keys ---------------------------------------------------------------
    def rotation_steps(self) -> set[int]:
        # + slots/2: X -> -X, unpacks two even-polynomial messages (bootstrap_pairs)
        return plan_rotations(self.cts_plans) | plan_rotations(self.stc_plans) | {self.params.slots // 2}

    def keygen(self, rng: np.random.Generator, rotations=()) -> KeySet:
        steps = sorted(set(rotations) | self.rotation_steps())
        ks = ckks.keygen(self.params, rng, rotations=steps, secret_weight=self.cfg.secret_weight,
                         conjugation=True)
        ks.bootstrapper = self
        return ks

    # -- linear transforms ----------------------------------------------------
    def _scale_bits(self, in_scale: float) -> int:
        """integer scale-up exponent e: q0 / (in_scale 2^e) ~ 2^message_ratio_bits"""
        e = int(round(math.log2(self.q0 / in_scale))) - self.cfg.message_ratio_bits
        return max(0, e)

    def _mask(self, tag, values: np.ndarray, level: int, scale: float):
        key = (tag, level, scale)
        m = self._masks.get(key)
        if m is None:
            pt = ckks.encode(values, self.params, level, scale)
            m = self.params.ctx.unop("to_mont", pt.data, level + 1)
            self._masks[key] = m
        return m

    def _mask_ext(self, tag, values: np.ndarray, level: int, scale: float):
        """diagonal encoded over Q_level || P, Montgomery evaluation rows"""
        key = ("ext", tag, level, scale)
        m = self._masks.get(key)
        if m is None:
            ctx = self.params.ctx
            coeffs = ckks.encode_coeffs(values, self.params, level, scale)
            rows = torch.from_numpy(np.ascontiguousarray(coeffs[None, :])).to(ctx.torch_device)
            t = ctx.from_signed(rows, level + 1, ctx.K, mont=True)[0]
            ctx.ntt(t, level + 1, ctx.K)
            self._masks[key] = m = t
        return m

    def _lift_ext(self, ct: Ciphertext) -> torch.Tensor:
        """(P c0, P c1) over Q_l || P (zero P limbs): the identity baby step"""
        ctx = self.params.ctx
        nq = ct.level + 1
        pmod = [self._pmod_q[i] for i in range(nq)]
        up = ctx.scalar_mul(ct.data, pmod, nq)
        zeros = torch.zeros(*ct.data.shape[:-2], ctx.K, ct.n, dtype=up.dtype, device=up.device)
        return torch.cat([up, zeros], dim=-2).contiguous()

    def _apply_dh(self, ct: Ciphertext, plans: list[DiagPlan], ks: KeySet, tag,
                  final_scale: float | None = None) -> Ciphertext:
        """Double-hoisted BSGS: baby rotations stay in Q||P (one shared ModUp,
        no ModDown), each giant group is MAC'd in Q||P, ModDown'd once and
        rotated without ModDown into a Q||P accumulator; one final ModDown
        per level matrix.  Same scale schedule as _apply."""
        ctx = self.params.ctx
        K = ctx.K
        nlev = len(plans)
        ratio = 1.0 if final_scale is None else (final_scale / ct.scale) ** (1.0 / nlev)
        for li, p in enumerate(plans):
            lvl = ct.level
            if lvl < 1:
                raise LevelError("linear transform ran out of levels")
            nq = lvl + 1
            q = self.params.q_mods[lvl].q
            tgt = final_scale if (li == nlev - 1 and final_scale is not None) else ct.scale * ratio
            s_d = tgt * q / ct.scale
            babies = [b for b in p.babies if b]
            keys = [(ks.gks[b].rows_b, ks.gks[b].rows_a) for b in babies]
            ext = dict(zip(babies, ctx.rotate_hoisted_ext(ct.data, lvl, [ckks.galois_element(b, ct.n) for b in babies],
                                                          keys)))
            if 0 in p.babies:
                ext[0] = self._lift_ext(ct)
            acc = None
            for gamt, terms in sorted(p.giants.items()):
                cts = [ext[b] for b, _ in terms]
                masks = [self._mask_ext((tag, li, gamt, b), pre, lvl, s_d) for b, pre in terms]
                part = ctx.mac_terms_ext(cts, masks, lvl)
                if gamt:
                    inner = ctx.moddown(part, lvl)
                    part = ctx.rotate_hoisted_ext(inner, lvl, [ckks.galois_element(gamt, ct.n)],
                                                  [(ks.gks[gamt].rows_b, ks.gks[gamt].rows_a)])[0]
                acc = part if acc is None else ctx.binop("add", acc, part, nq, K)
            if self.cfg.fused_moddown_rescale:
                # ModDown and the rescale in one base conversion: divide by P q_l at once
                out = ctx.moddown_rescale(acc, lvl)
                ct = Ciphertext(out, ct.scale * s_d / q, ct.n, ct.params)
            else:
                out = ctx.moddown(acc, lvl)
                ct = ckks.rescale(Ciphertext(out, ct.scale * s_d, ct.n, ct.params), self.params)
        return ct

    def _apply(self, ct: Ciphertext, plans: list[DiagPlan], ks: KeySet, tag,
               final_scale: float | None = None) -> Ciphertext:
        if self.cfg.double_hoist and self.params.ctx.K:
            return self._apply_dh(ct, plans, ks, tag, final_scale)
        return self._apply_sh(ct, plans, ks, tag, final_scale)

    def _apply_sh(self, ct: Ciphertext, plans: list[DiagPlan], ks: KeySet, tag,
                  final_scale: float | None = None) -> Ciphertext:
        """Apply the level matrices.  The scale moves geometrically from the
        input scale to final_scale (None: keep) so every level's plaintext
        scale stays close to its prime -- the precision of the product."""
        ctx = self.params.ctx
        nlev = len(plans)
        ratio = 1.0 if final_scale is None else (final_scale / ct.scale) ** (1.0 / nlev)
        for li, p in enumerate(plans):
            lvl = ct.level
            if lvl < 1:
                raise LevelError("linear transform ran out of levels")
            q = self.params.q_mods[lvl].q
            tgt = final_scale if (li == nlev - 1 and final_scale is not None) else ct.scale * ratio
            s_d = tgt * q / ct.scale
            rots = dict(zip(p.babies, ckks.rotate_many(ct, p.babies, ks)))
            acc = None
            for gamt, terms in sorted(p.giants.items()):
                cts = [rots[b].data for b, _ in terms]
                masks = [self._mask((tag, li, gamt, b), pre, lvl, s_d) for b, pre in terms]
                inner = Ciphertext(ctx.mac_terms(cts, masks, lvl), ct.scale * s_d, ct.n, ct.params)
                if gamt:
                    inner = ckks.rotate(inner, gamt, ks)
                acc = inner if acc is None else Ciphertext(ctx.binop("add", acc.data, inner.data, lvl + 1),
                                                          acc.scale, acc.n, acc.params)
            ct = ckks.rescale(acc, self.params)
        return ct

    @staticmethod
    def _relabel(ct: Ciphertext, scale: float) -> Ciphertext:
        return Ciphertext(ct.data, scale, ct.n, ct.params)

    def coeff_to_slot(self, ct: Ciphertext, ks: KeySet) -> tuple[Ciphertext, float]:
        """level-0 ct -> (ct with slots BR((t_lo + i t_hi)) / (2 q0 B), Delta1)."""
        x = ckks.mod_drop(ct, 0)
        e = self._scale_bits(x.scale)
        if e:
            x = ckks.mul_int(x, 1 << e)
        delta1 = x.scale
        x = ckks.mod_raise(x)
        # slots become U0 (t_lo + i t_hi) / (2 n q0 B); CtS multiplies by n BR U0^-1
        x = self._relabel(x, 2.0 * self.params.slots * self.q0 * self.B)
        u = self._apply(x, self.cts_plans, ks, "cts", final_scale=self.eval_scale)
        return u, delta1

    def eval_mod(self, y: Ciphertext, ks: KeySet) -> Ciphertext:
        """slots y = x/B (x = t/q0) -> sin(2 pi x)."""
        ev = _Exact(self.params, ks, fused=self.cfg.fused_moddown_rescale)
        c = eval_chebyshev(ev, y, self.cheb, self.eval_scale)
        for _ in range(self.cfg.double_angle):
            c = ev.cheb_product(c, c, None)  # cos(2t) = 2 cos(t)^2 - 1
        return c

    # -- the pipeline -----------------------------------------------------------
    def bootstrap(self, ct: Ciphertext, ks: KeySet, out_scale: float | None = None) -> Ciphertext:
        params = self.params
        if ks.conj is None:
            raise KeyError_("bootstrapping needs the conjugation key (Bootstrapper.keygen)")
        out_scale = ct.scale if out_scale is None else out_scale
        ev = _Exact(params, ks)
        hook = self.phase_hook or (lambda name: None)
        hook("start")
        u, delta1 = self.coeff_to_slot(ct, ks)
        hook("coeff_to_slot")
        uc = ckks.conjugate(u, ks)
        y_lo = ev.add(u, uc)                                                   # t_lo / (q0 B)
        y_hi = ckks.mul_monomial(ev.add(u, uc, sub=True), 3 * params.n // 2)  # -i * 2i Im u
        # both halves (of every batch entry) through one EvalMod pass
        both = torch.cat([y_lo.data, y_hi.data]) if u.batch is not None else torch.stack([y_lo.data, y_hi.data])
        hook("conjugate_split")
        vb = self.eval_mod(Ciphertext(both, y_lo.scale, y_lo.n, y_lo.params), ks)
        hook("eval_mod")
        h = vb.data.shape[0] // 2
        v_lo = Ciphertext(vb.data[:h] if u.batch is not None else vb.data[0], vb.scale, vb.n, vb.params)
        v_hi = Ciphertext(vb.data[h:] if u.batch is not None else vb.data[1], vb.scale, vb.n, vb.params)
        v = ev.add(v_lo, ckks.mul_monomial(v_hi, params.n // 2))              # 2 pi (m_lo + i m_hi) / q0
        # StC computes U0 BR; slots of the message are U0 m / Delta1 = v q0 / (2 pi Delta1)
        v = self._relabel(v, v.scale * (2.0 * math.pi * delta1) / self.q0)
        out = self._apply(v, self.stc_plans, ks, "stc", final_scale=out_scale)
        if out.level > self.output_level:
            out = ckks.mod_drop(out, self.output_level)
        hook("slot_to_coeff")
        return out

    def bootstrap_many(self, cts: list[Ciphertext], ks: KeySet, max_batch: int = 16,
                       out_scale_factor: float = 1.0) -> list[Ciphertext]:
        """Bootstrap several ciphertexts; members sharing (level, scale) run
        as one batch (every kernel covers the batch, key and diagonal loads
        are shared).  Entry-wise identical to ``bootstrap``."""
        out: list[Ciphertext | None] = [None] * len(cts)
        groups: dict = {}
        for i, c in enumerate(cts):
            groups.setdefault((c.level, c.scale), []).append(i)
        for idx in groups.values():
            for s0 in range(0, len(idx), max_batch):
                part = idx[s0:s0 + max_batch]
                osc = cts[part[0]].scale * out_scale_factor
                if len(part) == 1:
                    out[part[0]] = self.bootstrap(cts[part[0]], ks, osc)
                    continue
                res = ckks.unstack(self.bootstrap(ckks.stack([cts[i] for i in part]), ks, osc))
                for i, r in zip(part, res):
                    out[i] = r
        return out

    def bootstrap_pairs(self, pairs: list[tuple[Ciphertext, Ciphertext]], ks: KeySet) -> list[tuple[Ciphertext, Ciphertext]]:
        """Two ciphertexts per bootstrap.  Both members must encrypt even
        polynomials (slot vectors invariant under rotation by slots/2, see
        packing.slot_period) at one level and scale.  m = a + X b is
        bootstrapped once (at half the scale); then with s: X -> -X (the
        rotation by slots/2), a = (m + s(m))/2 and b = X^-1 (m - s(m))/2 --
        no level, one rotation for the whole batch."""
        if not pairs:
            return []
        n = self.params.n
        packed = [ckks.hadd(a, ckks.mul_monomial(b, 1)) for a, b in pairs]
        outs = self.bootstrap_many(packed, ks, out_scale_factor=0.5)
        res: list = [None] * len(pairs)
        groups: dict = {}
        for i, o in enumerate(outs):
            groups.setdefault((o.level, o.scale), []).append(i)
        ctx = self.params.ctx
        for idx in groups.values():
            o = outs[idx[0]] if len(idx) == 1 else ckks.stack([outs[i] for i in idx])
            r = ckks.rotate(o, self.params.slots // 2, ks)
            lvl = o.level
            even = Ciphertext(ctx.binop("add", o.data, r.data, lvl + 1), 2.0 * o.scale, o.n, o.params)
            odd = ckks.mul_monomial(Ciphertext(ctx.binop("sub", o.data, r.data, lvl + 1), 2.0 * o.scale, o.n, o.params),
                                    2 * n - 1)
            for k, a_out, b_out in zip(idx, ckks.unstack(even), ckks.unstack(odd)):
                res[k] = (a_out, b_out)
        return res
