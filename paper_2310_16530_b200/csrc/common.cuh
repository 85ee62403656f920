// Shared device/host definitions for the hcnn-b200 RNS-CKKS engine.
//
// Residues are uint64 < q < 2^62, held limb-major exactly like the
// reference's RnsPoly.coeffs ([nlimbs][N], /root/reference/pkg/src/hcnn/ring.py:204-213).
// Every kernel returns canonical residues in [0, q): the reference's REDC
// ends in a conditional subtract (kernels.py:177-188), so any exact modular
// method (Shoup, Montgomery, 128-bit lazy accumulation) reproduces its
// outputs bit for bit.
#pragma once

#include <cstdint>
#include <cstddef>
#include <cuda_runtime.h>

typedef uint64_t u64;
typedef unsigned int u32;

#define HCNN_MAX_MODS 128

// ---------------------------------------------------------------------------
// Per-modulus constants, one entry per modulus index.  Modulus indices:
// 0..Lq-1 are the q chain, Lq..Lq+K-1 the special primes (ckks.py:144-145).
// ---------------------------------------------------------------------------
struct ModConsts {
  u64 q;        // the prime
  u64 ninv;     // -q^-1 mod 2^64 (Montgomery, ring.py:48-50)
  u64 r2;       // 2^128 mod q
  u64 one_m;    // 2^64 mod q (Montgomery one)
  u64 ninvN;    // N^-1 mod q (standard form)
  u64 ninvN_sh; // Shoup companion floor(ninvN * 2^64 / q)
  u64 two_q;
  u64 ilast;    // inverse twiddle itw[1] * N^-1 mod q (last GS stage, N^-1 folded)
  u64 ilast_sh;
  u64 four_q;   // lazy bound of the approximate-quotient NTT (ntt2.cu)
  u64 one_sh;   // floor(2^64 / q): Shoup companion of 1 (exact reduction of any u64)
};

// A basis is (nq, np): limbs 0..nq-1 live over q_0..q_{nq-1}, limbs
// nq..nq+np-1 over p_0..p_{np-1} (the extended basis Q_l||P of ckks.py:144).
struct Basis {
  u32 nq, np, Lq;  // Lq = modulus index of p_0
  __host__ __device__ __forceinline__ u32 nlimbs() const { return nq + np; }
  __host__ __device__ __forceinline__ u32 mod_of(u32 r) const { return r < nq ? r : Lq + (r - nq); }
};

// ---------------------------------------------------------------------------
// 64-bit modular arithmetic (integer pipe; no native 64x64->128, the
// compiler emits IMAD.WIDE chains for __umul64hi).
// ---------------------------------------------------------------------------
__device__ __forceinline__ u64 add_mod(u64 a, u64 b, u64 q) {
  u64 t = a + b;
  return t >= q ? t - q : t;
}
__device__ __forceinline__ u64 sub_mod(u64 a, u64 b, u64 q) {
  return a >= b ? a - b : a + (q - b);
}
__device__ __forceinline__ u64 neg_mod(u64 a, u64 q) { return a == 0 ? 0 : q - a; }

// Montgomery REDC of a*b, b in Montgomery form (b = x*2^64 mod q):
// returns a*x mod q in [0,q).  Valid for a*b < q*2^64.
__device__ __forceinline__ u64 mont_mul(u64 a, u64 b, u64 q, u64 ninv) {
  u64 lo = a * b;
  u64 hi = __umul64hi(a, b);
  u64 m = lo * ninv;
  u64 t = hi + __umul64hi(m, q) + (lo != 0ull);
  return t >= q ? t - q : t;
}

// REDC of a 128-bit accumulator (hi:lo) < q*2^64 -> (hi:lo)*2^-64 mod q.
__device__ __forceinline__ u64 redc128(u64 hi, u64 lo, u64 q, u64 ninv) {
  u64 m = lo * ninv;
  u64 t = hi + __umul64hi(m, q) + (lo != 0ull);
  return t >= q ? t - q : t;
}

// Shoup product with a precomputed companion wp = floor(w*2^64/q).
// Lazy form returns a value in [0, 2q) for any a < 2^64, w < q.
__device__ __forceinline__ u64 shoup_lazy(u64 a, u64 w, u64 wp, u64 q) {
  u64 qh = __umul64hi(a, wp);
  return a * w - qh * q;
}
__device__ __forceinline__ u64 shoup_mul(u64 a, u64 w, u64 wp, u64 q) {
  u64 r = shoup_lazy(a, w, wp, q);
  return r >= q ? r - q : r;
}

// floor(a*b / 2^64) - e, e in {0,1,2}: the lo*lo partial product and the
// middle carries are dropped (3 IMAD.WIDE instead of 4 plus carry chain).
__device__ __forceinline__ u64 mulhi_approx(u64 a, u64 b) {
  const u32 alo = (u32)a, ahi = (u32)(a >> 32), blo = (u32)b, bhi = (u32)(b >> 32);
  const u64 m1 = (u64)alo * bhi, m2 = (u64)ahi * blo, hh = (u64)ahi * bhi;
  return hh + (m1 >> 32) + (m2 >> 32);
}
// Shoup product with the approximate quotient: a*w - qhat*q lies in [0, 4q)
// for any a < 2^64, w < q (qhat is at most 2 below the true quotient).
__device__ __forceinline__ u64 shoup_approx(u64 a, u64 w, u64 wp, u64 q) {
  return a * w - mulhi_approx(a, wp) * q;
}

// 128-bit accumulate of a*b into (hi:lo), keeping hi < q so the total stays
// below q*2^64 (subtracting q*2^64 does not change T*2^-64 mod q).
// Requires a*b < q*2^64 (true for a < 2^64, b < q).
__device__ __forceinline__ void mac128(u64& hi, u64& lo, u64 a, u64 b, u64 q) {
  u64 plo = a * b;
  u64 phi = __umul64hi(a, b);
  u64 nlo = lo + plo;
  hi = hi + phi + (nlo < lo ? 1ull : 0ull);
  lo = nlo;
  if (hi >= q) hi -= q;
}

// Lazy 128-bit multiply-accumulate: (hi:lo) += a*b with no per-step
// reduction.  Each product is below
// 2^124 (a < 2^64, b < q < 2^60 ... 2^62), so up to kLazyTerms products fit
// before hi must be folded (fold_hi); fold once more before redc128.
// Folding subtracts multiples of q*2^64, which REDC ignores: outputs stay
// canonical and bit-identical with mac128.
constexpr int kLazyTerms = 8;
__device__ __forceinline__ void mac128_lazy(u64& hi, u64& lo, u64 a, u64 b) {
  // the __int128 form compiles to ~11 SASS ops per product (IMAD.WIDE.U32
  // chains with carry), vs ~25 for mac128 and ~13 for mad.lo.cc/madc.hi
  unsigned __int128 acc = ((unsigned __int128)hi << 64) | lo;
  acc += (unsigned __int128)a * b;
  hi = (u64)(acc >> 64);
  lo = (u64)acc;
}
// hi mod q for any hi < 2^64 (Shoup with w = 1, one_sh = floor(2^64/q))
__device__ __forceinline__ u64 fold_hi(u64 hi, u64 q, u64 one_sh) {
  const u64 r = hi - __umul64hi(hi, one_sh) * q;
  return r >= q ? r - q : r;
}

// bit reversal of the low `logn` bits
__device__ __forceinline__ u32 brev_bits(u32 x, u32 logn) { return __brev(x) >> (32 - logn); }

// Eval-domain Galois permutation: NTT output index k holds a(psi^(2 brv(k)+1))
// (SURVEY §0.2); X -> X^g maps it to index brv(((2 brv(k)+1) g mod 2N - 1)/2).
// out[k] = in[galois_src(k)].
__device__ __forceinline__ u32 galois_src(u32 k, u64 g, u32 logn) {
  u32 n2mask = (2u << logn) - 1u;  // 2N - 1
  u32 e = (2u * brev_bits(k, logn) + 1u);
  u32 eg = (u32)(((u64)e * g) & n2mask);
  return brev_bits((eg - 1u) >> 1, logn);
}

// host helpers --------------------------------------------------------------
static inline u64 h_mulmod(u64 a, u64 b, u64 q) {
  return (u64)(((unsigned __int128)a * b) % q);
}
static inline u64 h_powmod(u64 a, u64 e, u64 q) {
  u64 r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = h_mulmod(r, a, q);
    a = h_mulmod(a, a, q);
    e >>= 1;
  }
  return r;
}
static inline u64 h_invmod(u64 a, u64 q) { return h_powmod(a, q - 2, q); }  // q prime
static inline u64 h_to_mont(u64 a, u64 q) {
  return (u64)((((unsigned __int128)(a % q)) << 64) % q);
}
static inline u64 h_shoup(u64 w, u64 q) {
  return (u64)((((unsigned __int128)w) << 64) / q);
}
