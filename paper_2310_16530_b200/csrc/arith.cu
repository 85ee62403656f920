// Element-wise, base-conversion, key-switch and rescale kernels (sm_100a).
//
// All of these are HBM-bound streaming kernels over [poly][limb][N] u64
// residues.  Each maps one CTA row to one (poly, limb) pair so the modulus
// constants are warp-uniform, and moves 16 B per thread per access.
#include <mutex>
#include <set>
#include <tuple>

#include "common.cuh"
#include "kernels.cuh"
#include "arith.cuh"
#include "tma.cuh"

namespace hcnn {

// Per-device side stream + fork/join events for kernels that run next to
// another launch of the same call (created once per device, never freed).
// The caller holds *mu across record-fork / wait / launch / record-join /
// wait so host threads sharing a device cannot interleave their forks.
int g_fbc_fork = 1;  // ModUp: the partial last digit's FBC on the side stream

cudaError_t side_stream(cudaStream_t* s, cudaEvent_t* fork, cudaEvent_t* join, std::mutex** mu) {
  static std::mutex init_mu;
  static std::mutex use_mu[64];
  static cudaStream_t ss[64] = {};
  static cudaEvent_t ef[64] = {}, ej[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(init_mu);
  if (!ss[dev]) {
    e = cudaStreamCreateWithFlags(&ss[dev], cudaStreamNonBlocking);
    if (!e) e = cudaEventCreateWithFlags(&ef[dev], cudaEventDisableTiming);
    if (!e) e = cudaEventCreateWithFlags(&ej[dev], cudaEventDisableTiming);
    if (e) return e;
  }
  *s = ss[dev];
  *fork = ef[dev];
  *join = ej[dev];
  *mu = &use_mu[dev];
  return cudaSuccess;
}


// 96-bit carry-chain MAC for operands below 2^42 (a = a1 2^32 + a0, m = m1 2^32 + m0,
// a1, m1 < 2^10): a m = a0 m0 + (a0 m1 + a1 m0) 2^32 + a1 m1 2^64 accumulated as
// T = lh + mid 2^32 -- 5 IMADs per product instead of the 128-bit product's ~11
__device__ __forceinline__ void mac96(u64& lh, u64& mid, u32 a0, u32 a1, u32 m0, u32 m1) {
  asm("{\n\t.reg .u32 lo, hi, ml, mh;\n\t"
      "mov.b64 {lo, hi}, %0;\n\t"
      "mov.b64 {ml, mh}, %1;\n\t"
      "mad.lo.cc.u32 lo, %2, %4, lo;\n\t"
      "madc.hi.cc.u32 hi, %2, %4, hi;\n\t"
      "madc.lo.u32 mh, %3, %5, mh;\n\t"
      "mov.b64 %0, {lo, hi};\n\t"
      "mov.b64 %1, {ml, mh};\n\t"
      "mad.wide.u32 %1, %2, %5, %1;\n\t"
      "mad.wide.u32 %1, %3, %4, %1;\n\t"
      "}"
      : "+l"(lh), "+l"(mid)
      : "r"(a0), "r"(a1), "r"(m0), "r"(m1));
}
// T = lh + mid 2^32 (< 2^90) -> T R^-1 mod q
// Signed Montgomery form of the reduction: with m = L2 q^-1 (q^-1 = -ninv mod
// 2^64) the low word of m q equals L2, so (T - m q) / 2^64 = H - hi(m q)
// exactly, in (-q, q) because H < q (T < 2^90) and hi(m q) < q: one
// correction and no carry-in term -- fewer ALU operations than redc128's
// H + hi + (L2 != 0) with its [0, 2q) result (the same canonical residue).
__device__ __forceinline__ u64 redc96(u64 lh, u64 mid, u64 q, u64 ninv) {
  const u64 L2 = lh + (mid << 32);
  const u64 H = (mid >> 32) + (L2 < lh ? 1ull : 0ull);
  const u64 mh = __umul64hi(L2 * (0ull - ninv), q);
  return H >= mh ? H - mh : H - mh + q;
}

// FBC: the 96-bit path for conversions whose sources and target are all below 2^42
__constant__ bool g_fbc_fast_dev = true;
// key-switch inner product (k_ks_inner_tma2 / _rots): 96-bit rows for q < 2^42
__constant__ bool g_ks96_dev = true;
cudaError_t set_ks96(int on) {
  const bool v = on != 0;
  return cudaMemcpyToSymbol(g_ks96_dev, &v, sizeof(v));
}
cudaError_t set_fbc_fast(int on) {
  const bool v = on != 0;
  return cudaMemcpyToSymbol(g_fbc_fast_dev, &v, sizeof(v));
}

static inline dim3 row_grid(u32 work_per_row, u32 rows, u32 threads) {
  u32 x = (work_per_row + threads - 1) / threads;
  if (x == 0) x = 1;
  if (x > 1024) x = 1024;
  return dim3(x, rows, 1);
}

// ---------------------------------------------------------------------------
// element-wise (ring.py:264-314, kernels.py:190-230)
// grid: x over N/(2*blockDim), y over rows = npolys*nlimbs
// ---------------------------------------------------------------------------
struct RowCtx {
  u32 row, z, r, mod;
};
__device__ __forceinline__ RowCtx row_ctx(const Basis& b) {
  RowCtx c;
  c.row = blockIdx.y;
  u32 nl = b.nlimbs();
  c.z = c.row / nl;
  c.r = c.row - c.z * nl;
  c.mod = b.mod_of(c.r);
  return c;
}

__global__ void k_ew_binary(int op, u64* __restrict__ out, const u64* __restrict__ a, const u64* __restrict__ b,
                            Basis basis, u32 logN, int b_bcast, const ModConsts* __restrict__ mc) {
  RowCtx rc = row_ctx(basis);
  const u32 N = 1u << logN;
  const ModConsts C = mc[rc.mod];
  const size_t off = (size_t)rc.row * N;
  const size_t boff = (size_t)(b_bcast ? rc.r : rc.row) * N;
  const ulonglong2* A = reinterpret_cast<const ulonglong2*>(a + off);
  const ulonglong2* B = reinterpret_cast<const ulonglong2*>(b + boff);
  ulonglong2* O = reinterpret_cast<ulonglong2*>(out + off);
  // b_bcast == 2 (ciphertext + plaintext): b goes into the even polys (c0 of
  // every ciphertext), the odd ones (c1) are copied -- one pass, no clone
  if (b_bcast == 2 && (rc.z & 1u)) {
    for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < N / 2; i += gridDim.x * blockDim.x) O[i] = A[i];
    return;
  }
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < N / 2; i += gridDim.x * blockDim.x) {
    ulonglong2 x = A[i], y = B[i], o;
    switch (op) {
      case EW_ADD:
        o.x = add_mod(x.x, y.x, C.q);
        o.y = add_mod(x.y, y.y, C.q);
        break;
      case EW_SUB:
        o.x = sub_mod(x.x, y.x, C.q);
        o.y = sub_mod(x.y, y.y, C.q);
        break;
      case EW_MUL_MONT:  // a * b_mont * 2^-64  (pmult_mont, _mul_rows_mont)
        o.x = mont_mul(x.x, y.x, C.q, C.ninv);
        o.y = mont_mul(x.y, y.y, C.q, C.ninv);
        break;
      case EW_MUL:  // both ordinary residues (poly_mul_pointwise)
        o.x = mont_mul(mont_mul(x.x, y.x, C.q, C.ninv), C.r2, C.q, C.ninv);
        o.y = mont_mul(mont_mul(x.y, y.y, C.q, C.ninv), C.r2, C.q, C.ninv);
        break;
      default:  // EW_MAC_MONT: out += a * b_mont
      {
        ulonglong2 acc = O[i];
        o.x = add_mod(acc.x, mont_mul(x.x, y.x, C.q, C.ninv), C.q);
        o.y = add_mod(acc.y, mont_mul(x.y, y.y, C.q, C.ninv), C.q);
      }
    }
    O[i] = o;
  }
}

__global__ void k_ew_unary(int op, u64* __restrict__ out, const u64* __restrict__ a, Basis basis, u32 logN,
                           const ModConsts* __restrict__ mc, const u64* __restrict__ consts,
                           const u64* __restrict__ consts_sh) {
  RowCtx rc = row_ctx(basis);
  const u32 N = 1u << logN;
  const ModConsts C = mc[rc.mod];
  const size_t off = (size_t)rc.row * N;
  const ulonglong2* A = reinterpret_cast<const ulonglong2*>(a + off);
  ulonglong2* O = reinterpret_cast<ulonglong2*>(out + off);
  u64 w = 0, wp = 0;
  if (op == EW_SCALAR || op == EW_SCALAR_ADD) {
    w = consts[rc.r];
    wp = consts_sh[rc.r];
  }
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < N / 2; i += gridDim.x * blockDim.x) {
    ulonglong2 x = A[i], o;
    switch (op) {
      case EW_NEG:
        o.x = neg_mod(x.x, C.q);
        o.y = neg_mod(x.y, C.q);
        break;
      case EW_TO_MONT:
        o.x = mont_mul(x.x, C.r2, C.q, C.ninv);
        o.y = mont_mul(x.y, C.r2, C.q, C.ninv);
        break;
      case EW_FROM_MONT:
        o.x = mont_mul(x.x, 1ull, C.q, C.ninv);
        o.y = mont_mul(x.y, 1ull, C.q, C.ninv);
        break;
      case EW_SCALAR_ADD:  // + per-limb constant (constant polynomial in the eval domain)
        o.x = add_mod(x.x, w, C.q);
        o.y = add_mod(x.y, w, C.q);
        break;
      default:  // EW_SCALAR
        o.x = shoup_mul(x.x, w, wp, C.q);
        o.y = shoup_mul(x.y, w, wp, C.q);
    }
    O[i] = o;
  }
}

// per-limb scalar multiply / add with the constants passed by value
// (capture-safe: no host->device copy), up to kScalarMax limbs
__global__ void k_scalar(int add, u64* __restrict__ out, const u64* __restrict__ a, Basis basis, u32 logN,
                         const ModConsts* __restrict__ mc, ScalarArgs args) {
  RowCtx rc = row_ctx(basis);
  const u32 N = 1u << logN;
  const u64 q = mc[rc.mod].q;
  const u64 w = args.w[rc.r], wp = args.wp[rc.r];
  const size_t off = (size_t)rc.row * N;
  const ulonglong2* A = reinterpret_cast<const ulonglong2*>(a + off);
  ulonglong2* O = reinterpret_cast<ulonglong2*>(out + off);
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < N / 2; i += gridDim.x * blockDim.x) {
    ulonglong2 x = A[i], o;
    if (add) {
      o.x = add_mod(x.x, w, q);
      o.y = add_mod(x.y, w, q);
    } else {
      o.x = shoup_mul(x.x, w, wp, q);
      o.y = shoup_mul(x.y, w, wp, q);
    }
    O[i] = o;
  }
}

cudaError_t launch_scalar(int add, u64* out, const u64* a, Basis basis, u32 logN, u32 npolys, const ModConsts* mc,
                          const ScalarArgs& args, cudaStream_t st) {
  u32 rows = npolys * basis.nlimbs();
  if (!rows) return cudaSuccess;
  k_scalar<<<row_grid((1u << logN) / 2, rows, 256), 256, 0, st>>>(add, out, a, basis, logN, mc, args);
  return cudaGetLastError();
}

// linear combination with per-limb integer constants (bootstrapping's
// Chebyshev leaves and fused T_{a+b} = 2 T_a T_b - T_{a-b}): one pass over
// the sources, fully reduced Shoup products summed mod q
__global__ void __launch_bounds__(256) k_scalar_mac(int nt, u64* __restrict__ out, u32 nl, u32 logN, int accumulate,
                                                    const ModConsts* __restrict__ mc, ScalarMacArgs A) {
  const u32 N = 1u << logN;
  const u32 r = blockIdx.y % nl, z = blockIdx.y / nl;
  const u64 q = mc[r].q;
  ulonglong2* O = reinterpret_cast<ulonglong2*>(out + ((size_t)z * nl + r) * N);
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < N / 2; i += gridDim.x * blockDim.x) {
    ulonglong2 acc = accumulate ? O[i] : make_ulonglong2(0, 0);
    for (int t = 0; t < nt; ++t) {
      const ulonglong2 x =
          reinterpret_cast<const ulonglong2*>(A.src[t] + ((size_t)z * A.src_limbs[t] + r) * N)[i];
      const u64 w = A.w[t][r], wp = A.wp[t][r];
      acc.x = add_mod(acc.x, shoup_mul(x.x, w, wp, q), q);
      acc.y = add_mod(acc.y, shoup_mul(x.y, w, wp, q), q);
    }
    if (A.has_add0 && (z & 1) == 0) {
      acc.x = add_mod(acc.x, A.add0[r], q);
      acc.y = add_mod(acc.y, A.add0[r], q);
    }
    O[i] = acc;
  }
}

cudaError_t launch_scalar_mac(const ScalarMacArgs& A, int nt, u64* out, u32 nl, u32 logN, u32 npolys,
                              int accumulate, const ModConsts* mc, cudaStream_t st) {
  if (!nl || !npolys) return cudaSuccess;
  k_scalar_mac<<<row_grid((1u << logN) / 2, nl * npolys, 256), 256, 0, st>>>(nt, out, nl, logN, accumulate, mc, A);
  return cudaGetLastError();
}

// signed int64 coefficients (one row of N per poly) -> residues in every
// limb (ring.py:446-468 replication, ckks.py:284-288 encode reduction)
__global__ void k_from_signed(u64* __restrict__ out, const long long* __restrict__ in, Basis basis, u32 logN,
                              const ModConsts* __restrict__ mc, int mont) {
  RowCtx rc = row_ctx(basis);
  const u32 N = 1u << logN;
  const ModConsts C = mc[rc.mod];
  const long long* src = in + (size_t)rc.z * N;
  u64* O = out + (size_t)rc.row * N;
  const u64 k = mont ? C.r2 : C.one_m;  // |v| R mod q (Montgomery form) or |v| mod q
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    long long v = src[i];
    u64 mag = v >= 0 ? (u64)v : (u64)(-(v + 1)) + 1ull;
    u64 red = mont_mul(mag, k, C.q, C.ninv);
    O[i] = v >= 0 ? red : neg_mod(red, C.q);
  }
}

// Galois automorphisms.  Eval domain: pure permutation.
// Coefficient domain: out[i*g mod 2N] = +-in[i] (ring.py:405-439).
__global__ void k_automorph(int eval_domain, u64* __restrict__ out, const u64* __restrict__ in, Basis basis,
                            u32 logN, u64 g, const ModConsts* __restrict__ mc) {
  RowCtx rc = row_ctx(basis);
  const u32 N = 1u << logN;
  const u64 q = mc[rc.mod].q;
  const u64* I = in + (size_t)rc.row * N;
  u64* O = out + (size_t)rc.row * N;
  for (u32 k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
    if (eval_domain) {
      O[k] = I[galois_src(k, g, logN)];
    } else {
      u64 j = ((u64)k * g) & ((2ull << logN) - 1);
      u64 v = I[k];
      if (j < N) O[j] = v;
      else O[j - N] = neg_mod(v, q);
    }
  }
}

// hmult tensor product (ckks.py:609-611): d0=a0b0, d1=a0b1+a1b0, d2=a1b1
__global__ void k_tensor(u64* __restrict__ d0, u64* __restrict__ d1, u64* __restrict__ d2,
                         const u64* __restrict__ a, const u64* __restrict__ b, u32 nlimbs, u32 logN,
                         const ModConsts* __restrict__ mc) {
  const u32 r = blockIdx.y;
  const u32 N = 1u << logN;
  const ModConsts C = mc[r];
  const size_t pst = (size_t)nlimbs * N;
  const size_t off = (size_t)r * N;
  // rows with q < 2^42: the three products through 96-bit carry chains (one
  // REDC each, the d1 sum in one chain) -- the same canonical residues
  const bool f96 = g_ks96_dev && C.q < (1ull << 42);
  for (u32 k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
    u64 a0 = a[off + k], a1 = a[pst + off + k];
    u64 b0 = b[off + k], b1 = b[pst + off + k];
    if (f96) {
      const u32 a00 = (u32)a0, a01 = (u32)(a0 >> 32), a10 = (u32)a1, a11 = (u32)(a1 >> 32);
      u64 l0 = 0, m0 = 0, l1 = 0, m1 = 0, l2 = 0, m2 = 0;
      mac96(l0, m0, a00, a01, (u32)b0, (u32)(b0 >> 32));
      mac96(l1, m1, a00, a01, (u32)b1, (u32)(b1 >> 32));
      mac96(l1, m1, a10, a11, (u32)b0, (u32)(b0 >> 32));
      mac96(l2, m2, a10, a11, (u32)b1, (u32)(b1 >> 32));
      d0[off + k] = mont_mul(redc96(l0, m0, C.q, C.ninv), C.r2, C.q, C.ninv);
      d1[off + k] = mont_mul(redc96(l1, m1, C.q, C.ninv), C.r2, C.q, C.ninv);
      d2[off + k] = mont_mul(redc96(l2, m2, C.q, C.ninv), C.r2, C.q, C.ninv);
      continue;
    }
    u64 t0 = mont_mul(a0, b0, C.q, C.ninv);
    u64 t2 = mont_mul(a1, b1, C.q, C.ninv);
    u64 hi = 0, lo = 0;
    mac128(hi, lo, a0, b1, C.q);
    mac128(hi, lo, a1, b0, C.q);
    u64 t1 = redc128(hi, lo, C.q, C.ninv);
    d0[off + k] = mont_mul(t0, C.r2, C.q, C.ninv);
    d1[off + k] = mont_mul(t1, C.r2, C.q, C.ninv);
    d2[off + k] = mont_mul(t2, C.r2, C.q, C.ninv);
  }
}

// ---------------------------------------------------------------------------
// centred fast base conversion (ring.py:378-398, kernels.py:283-301)
// ---------------------------------------------------------------------------
#define FBC_MAX_SRC 64
constexpr u32 kFbcTG = 128;  // targets per CTA in k_fbc_t (splitting measured slower)

__device__ __forceinline__ void fbc_point(const FbcDev& T, const ModConsts* __restrict__ mc,
                                          const u64* __restrict__ src, size_t src_limb_stride,
                                          u64* __restrict__ dst, u32 k, u32 N, u32 nt) {
  u64 mag[FBC_MAX_SRC];
  u32 negmask_lo = 0, negmask_hi = 0;
  const u32 ns = T.ns;
  for (u32 i = 0; i < ns; ++i) {
    const u64 qi = mc[T.src_mod[i]].q;
    u64 y = shoup_mul(src[(size_t)i * src_limb_stride + k], T.inv_punc[i], T.inv_punc_sh[i], qi);
    bool neg = y > (qi >> 1);
    mag[i] = neg ? qi - y : y;
    if (neg) {
      if (i < 32) negmask_lo |= 1u << i;
      else negmask_hi |= 1u << (i - 32);
    }
  }
  for (u32 t = 0; t < nt; ++t) {
    const ModConsts C = mc[T.dst_mod[t]];
    const u64* row = T.tmat + (size_t)t * ns;
    u64 phi = 0, plo = 0, nhi = 0, nlo = 0;
    for (u32 i = 0; i < ns; ++i) {
      bool neg = i < 32 ? (negmask_lo >> i) & 1u : (negmask_hi >> (i - 32)) & 1u;
      if (neg) mac128(nhi, nlo, mag[i], row[i], C.q);
      else mac128(phi, plo, mag[i], row[i], C.q);
    }
    // (pos - neg) mod q*2^64, then one REDC
    u64 lo = plo - nlo;
    u64 borrow = plo < nlo ? 1ull : 0ull;
    long long hi = (long long)phi - (long long)nhi - (long long)borrow;
    if (hi < 0) hi += (long long)C.q;
    dst[(size_t)T.dst_pos[t] * N + k] = redc128((u64)hi, lo, C.q, C.ninv);
  }
}

// generic base_convert: poly z: src limbs at in + z*in_pst + i*N
__global__ void k_fbc(FbcDev T, const ModConsts* __restrict__ mc, const u64* __restrict__ in, size_t in_pst,
                      u64* __restrict__ out, size_t out_pst, u32 logN, u32 nt) {
  const u32 N = 1u << logN, z = blockIdx.y;
  for (u32 k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x)
    fbc_point(T, mc, in + (size_t)z * in_pst, N, out + (size_t)z * out_pst, k, N, nt);
}

// Specialised centred FBC for NS <= 6 source limbs.  Per-target constants
// (modulus, Montgomery inverse, output position, conversion row and the
// sign-mask correction table) are staged in shared memory; each output is
// one 128-bit sum of NS products of the raw y_i = x_i (Q/q_i)^-1 mod q_i,
// one REDC, and one subtraction of corr[mask] = sum over the limbs whose
// y_i exceeds q_i/2 of q_i (Q/q_i) mod t -- i.e. the centred lift of
// ring.py:378-398 without per-limb branches.
// z = blockIdx.y selects table tabs[z] (modup: one table per digit) or
// tabs[0] (tab_per_z == 0).
template <int NS>
__global__ void __launch_bounds__(256) k_fbc_t(const FbcDev* __restrict__ tabs, int tab_per_z,
                                               const ModConsts* __restrict__ mc, const u64* __restrict__ in,
                                               size_t in_pst, u64* __restrict__ out, size_t out_pst, u32 logN,
                                               u32 nt_override, u32 z0, u32 zdiv, size_t in_bst, size_t out_bst,
                                               u32 tg) {
  constexpr int NM = 1 << NS;
  extern __shared__ u64 sh[];
  // blockIdx.y = b * zdiv + j: poly/digit j of batch entry b
  const u32 N = 1u << logN, b = blockIdx.y / zdiv, z = blockIdx.y % zdiv + z0;
  const FbcDev& T = tabs[tab_per_z ? z : 0];
  const u32 nt_all = nt_override ? nt_override : T.nt;
  // blockIdx.z selects a group of tg targets (small conversions get more CTAs)
  const u32 t0 = blockIdx.z * tg;
  if (t0 >= nt_all) return;
  const u32 nt = nt_all - t0 < tg ? nt_all - t0 : tg;
  u64* s_q = sh;
  u64* s_ninv = s_q + nt;
  u64* s_pos = s_ninv + nt;
  u64* s_tm = s_pos + nt;        // [nt][NS]
  u64* s_corr = s_tm + nt * NS;  // [nt][NM]
  for (u32 t = threadIdx.x; t < nt; t += blockDim.x) {
    const u32 m = T.dst_mod[t0 + t];
    s_q[t] = mc[m].q;
    s_ninv[t] = mc[m].ninv;
    s_pos[t] = (u64)T.dst_pos[t0 + t] * N;
  }
  for (u32 e = threadIdx.x; e < nt * NS; e += blockDim.x) s_tm[e] = T.tmat[(size_t)t0 * NS + e];
  for (u32 e = threadIdx.x; e < nt * NM; e += blockDim.x) s_corr[e] = T.corr[(size_t)t0 * NM + e];
  u64 qi[NS], hq[NS], ip[NS], ips[NS];
  bool src_small = g_fbc_fast_dev;
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    qi[i] = mc[T.src_mod[i]].q;
    hq[i] = qi[i] >> 1;
    ip[i] = T.inv_punc[i];
    ips[i] = T.inv_punc_sh[i];
    src_small = src_small && qi[i] < (1ull << 42);
  }
  __syncthreads();
  const u64* src = in + (size_t)b * in_bst + (size_t)z * in_pst;
  u64* dst = out + (size_t)b * out_bst + (size_t)z * out_pst;
  // two adjacent coefficients per thread: every per-target constant read from
  // shared memory serves both, and loads / stores are 16 bytes
  for (u32 kv = blockIdx.x * blockDim.x + threadIdx.x; kv < N / 2; kv += gridDim.x * blockDim.x) {
    const u32 k = 2 * kv;
    u64 y0[NS], y1[NS];
    u32 m0 = 0, m1 = 0;
#pragma unroll
    for (int i = 0; i < NS; ++i) {
      const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(src + (size_t)i * N + k);
      y0[i] = shoup_mul(x.x, ip[i], ips[i], qi[i]);
      y1[i] = shoup_mul(x.y, ip[i], ips[i], qi[i]);
      m0 |= (y0[i] > hq[i] ? 1u : 0u) << i;
      m1 |= (y1[i] > hq[i] ? 1u : 0u) << i;
    }
#pragma unroll 2
    for (u32 t = 0; t < nt; ++t) {
      const u64 qt = s_q[t], ni = s_ninv[t];
      u64 v0, v1;
      if (src_small && qt < (1ull << 42)) {
        // every operand below 2^42: 96-bit carry-chain sums (5 IMADs per
        // product, T < 2^87 < q 2^64), the same canonical sum R^-1 mod q
        u64 L0 = 0, M0 = 0, L1 = 0, M1 = 0;
#pragma unroll
        for (int i = 0; i < NS; ++i) {
          const u64 b = s_tm[t * NS + i];
          mac96(L0, M0, (u32)y0[i], (u32)(y0[i] >> 32), (u32)b, (u32)(b >> 32));
          mac96(L1, M1, (u32)y1[i], (u32)(y1[i] >> 32), (u32)b, (u32)(b >> 32));
        }
        v0 = sub_mod(redc96(L0, M0, qt, ni), s_corr[t * NM + m0], qt);
        v1 = sub_mod(redc96(L1, M1, qt, ni), s_corr[t * NM + m1], qt);
      } else {
        u64 h0 = 0, l0 = 0, h1 = 0, l1 = 0;
#pragma unroll
        for (int i = 0; i < NS; ++i) {  // NS <= 6 < kLazyTerms
          const u64 b = s_tm[t * NS + i];
          mac128_lazy(h0, l0, y0[i], b);
          mac128_lazy(h1, l1, y1[i], b);
        }
        v0 = sub_mod(redc128(h0, l0, qt, ni), s_corr[t * NM + m0], qt);
        v1 = sub_mod(redc128(h1, l1, qt, ni), s_corr[t * NM + m1], qt);
      }
      *reinterpret_cast<ulonglong2*>(dst + s_pos[t] + k) = make_ulonglong2(v0, v1);
    }
  }
}

// ModUp of every digit of a key-switch input (ckks.py:563-578):
// digit j's limbs [j*alpha, ...) of xc are converted to the extended basis
// minus the digit, written into raised[j] at their basis positions.
__global__ void k_modup(const FbcDev* __restrict__ tabs, const ModConsts* __restrict__ mc,
                        const u64* __restrict__ xc, u64* __restrict__ raised, u32 alpha, u32 n_ext, u32 logN) {
  const u32 N = 1u << logN, j = blockIdx.y;
  const FbcDev T = tabs[j];
  const u64* src = xc + (size_t)j * alpha * N;
  u64* dst = raised + (size_t)j * n_ext * N;
  for (u32 k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x)
    fbc_point(T, mc, src, N, dst, k, N, T.nt);
}

// Key-switch inner product (ckks.py:579-586), fused over digits with one
// REDC per output: acc_{b,a}[r] = sum_j raised_j[r] * key_{b,a}[j][mod(r)]
// (key rows are Montgomery form, so the 128-bit sum REDCs straight to the
// ordinary residue).  g != 1 applies the eval-domain Galois permutation to
// the raised digits on the fly (hoisted rotation).
int g_mac_batch = 1;  // shared-mask MAC: 1 = entry-fastest CTA order, 4 = 4 entries per thread
int g_ks_batch = 1;  // measured: grid-batched entries share keys through L2; NB>1 costs occupancy

template <int NB, int VEC>
__global__ void __launch_bounds__(256, NB == 1 ? 4 : 1) k_ks_inner(u64* __restrict__ acc, const u64* __restrict__ x_eval,
                                                  const u64* __restrict__ raised, const u64* __restrict__ key_b,
                                                  const u64* __restrict__ key_a, Basis basis, u32 alpha, u32 ndig,
                                                  u32 logN, u64 g, const ModConsts* __restrict__ mc, u32 nb,
                                                  size_t x_bst, const u64* __restrict__ c0, size_t c0_bst,
                                                  const u64* __restrict__ pR, u32 key_lq) {
  // VEC adjacent coefficients x NB batch entries per thread (NB*VEC <= 4 keeps
  // the 128-bit accumulators at 16 registers pairs: full occupancy)
  const u32 N = 1u << logN, r = blockIdx.y;
  const u32 n_ext = basis.nlimbs();
  const u32 mod = basis.mod_of(r);
  const u64 q = mc[mod].q, ninv = mc[mod].ninv;
  // keys may be stored truncated to their first key_lq q-limbs (+ all specials)
  const u32 klq = key_lq ? key_lq : basis.Lq;
  const size_t key_dst = (size_t)(klq + basis.np) * N;  // per-digit key stride
  const u32 kmod = mod < basis.Lq ? mod : klq + (mod - basis.Lq);
  const u32 own = r < basis.nq ? r / alpha : 0xffffffffu;     // digit owning limb r
  // NB == 1: blockIdx.x = tile * nb + entry -- the nb CTAs reading one key
  // tile run back to back, so the key streams from HBM once per batch (L2
  // serves the rest).  NB > 1: NB entries per thread (blockIdx.z chunks).
  const u32 b0 = NB == 1 ? blockIdx.x % nb : blockIdx.z * NB;
  const u32 ne = nb - b0 < (u32)NB ? nb - b0 : (u32)NB;
  const size_t r_bst = (size_t)ndig * n_ext * N, a_bst = 2 * (size_t)n_ext * N;
  const u32 x0 = NB == 1 ? blockIdx.x / nb : blockIdx.x, xs = NB == 1 ? gridDim.x / nb : gridDim.x;
  for (u32 kv = x0 * blockDim.x + threadIdx.x; kv < N / VEC; kv += xs * blockDim.x) {
    const u32 k = VEC * kv;
    u64 bh[NB][VEC], bl[NB][VEC], ah[NB][VEC], al[NB][VEC];
#pragma unroll
    for (int e = 0; e < NB; ++e)
#pragma unroll
      for (int v = 0; v < VEC; ++v) bh[e][v] = bl[e][v] = ah[e][v] = al[e][v] = 0;
#pragma unroll(NB == 1 ? 1 : 2)
    for (u32 j = 0; j < ndig; ++j) {
      const size_t kofs = (size_t)j * key_dst + (size_t)kmod * N + k;
      u64 kb[VEC], ka[VEC];
      if (VEC == 2) {
        const ulonglong2 b2 = *reinterpret_cast<const ulonglong2*>(key_b + kofs);
        const ulonglong2 a2 = *reinterpret_cast<const ulonglong2*>(key_a + kofs);
        kb[0] = b2.x;
        kb[VEC - 1] = b2.y;
        ka[0] = a2.x;
        ka[VEC - 1] = a2.y;
      } else {
        kb[0] = key_b[kofs];
        ka[0] = key_a[kofs];
      }
#pragma unroll
      for (int e = 0; e < NB; ++e) {
        if ((u32)e >= ne) break;
        const u64* src = (j == own) ? x_eval + (size_t)(b0 + e) * x_bst + (size_t)r * N
                                    : raised + (size_t)(b0 + e) * r_bst + ((size_t)j * n_ext + r) * N;
        u64 x[VEC];
        if (g == 1) {
          if (VEC == 2) {
            const ulonglong2 x2 = *reinterpret_cast<const ulonglong2*>(src + k);
            x[0] = x2.x;
            x[VEC - 1] = x2.y;
          } else {
            x[0] = src[k];
          }
        } else {
#pragma unroll
          for (int v = 0; v < VEC; ++v) x[v] = src[galois_src(k + v, g, logN)];
        }
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          mac128(bh[e][v], bl[e][v], x[v], kb[v], q);
          mac128(ah[e][v], al[e][v], x[v], ka[v], q);
        }
      }
    }
    if (c0 && r < basis.nq) {  // extended-basis output: + P * sigma_g(c0) on the Q limbs
      const u64 w = pR[r];
#pragma unroll
      for (int e = 0; e < NB; ++e) {
        if ((u32)e >= ne) break;
        const u64* src = c0 + (size_t)(b0 + e) * c0_bst + (size_t)r * N;
#pragma unroll
        for (int v = 0; v < VEC; ++v) mac128(bh[e][v], bl[e][v], src[g == 1 ? k + v : galois_src(k + v, g, logN)], w, q);
      }
    }
#pragma unroll
    for (int e = 0; e < NB; ++e) {
      if ((u32)e >= ne) break;
      u64* A = acc + (size_t)(b0 + e) * a_bst;
      if (VEC == 2) {
        *reinterpret_cast<ulonglong2*>(A + (size_t)r * N + k) =
            make_ulonglong2(redc128(bh[e][0], bl[e][0], q, ninv), redc128(bh[e][VEC - 1], bl[e][VEC - 1], q, ninv));
        *reinterpret_cast<ulonglong2*>(A + ((size_t)n_ext + r) * N + k) =
            make_ulonglong2(redc128(ah[e][0], al[e][0], q, ninv), redc128(ah[e][VEC - 1], al[e][VEC - 1], q, ninv));
      } else {
        A[(size_t)r * N + k] = redc128(bh[e][0], bl[e][0], q, ninv);
        A[((size_t)n_ext + r) * N + k] = redc128(ah[e][0], al[e][0], q, ninv);
      }
    }
  }
}

// Software-pipelined form of k_ks_inner<1,2> for the single-poly-per-thread
// case: the key / digit loads of JB digits are issued before any of their
// MACs (more bytes in flight per SM: the kernel is HBM-latency bound), and
// the Galois source index is computed once per coefficient instead of once
// per digit.  Same sums, same single REDC: bit-identical outputs.
int g_ks_pipe = 2;  // digits per load batch (0: k_ks_inner<1,2>)

template <int JB>
__global__ void __launch_bounds__(256, JB >= 4 ? 2 : 3) k_ks_inner_p(
    u64* __restrict__ acc, const u64* __restrict__ x_eval, const u64* __restrict__ raised,
    const u64* __restrict__ key_b, const u64* __restrict__ key_a, Basis basis, u32 alpha, u32 ndig, u32 logN, u64 g,
    const ModConsts* __restrict__ mc, u32 nb, size_t x_bst, const u64* __restrict__ c0, size_t c0_bst,
    const u64* __restrict__ pR, u32 key_lq) {
  const u32 N = 1u << logN, r = blockIdx.y;
  const u32 n_ext = basis.nlimbs();
  const u32 mod = basis.mod_of(r);
  const u64 q = mc[mod].q, ninv = mc[mod].ninv, one_sh = mc[mod].one_sh;
  const bool f96 = g_ks96_dev && q < (1ull << 42);  // 96-bit carry chains (see k_ks_inner_tma2)
  const u32 klq = key_lq ? key_lq : basis.Lq;
  const size_t key_dst = (size_t)(klq + basis.np) * N;
  const u32 kmod = mod < basis.Lq ? mod : klq + (mod - basis.Lq);
  const u32 own = r < basis.nq ? r / alpha : 0xffffffffu;
  const u32 b = blockIdx.x % nb, x0 = blockIdx.x / nb, xs = gridDim.x / nb;
  static_assert(kLazyTerms % JB == 0, "fold cadence");
  const u64* xsrc = x_eval + (size_t)b * x_bst + (size_t)r * N;
  const u64* rsrc = raised + (size_t)b * ndig * n_ext * N + (size_t)r * N;
  const u64* kb_base = key_b + (size_t)kmod * N;
  const u64* ka_base = key_a + (size_t)kmod * N;
  const size_t rstep = (size_t)n_ext * N;
  for (u32 kv = x0 * blockDim.x + threadIdx.x; kv < N / 2; kv += xs * blockDim.x) {
    const u32 k = 2 * kv;
    const u32 p0 = g == 1 ? k : galois_src(k, g, logN), p1 = g == 1 ? k + 1 : galois_src(k + 1, g, logN);
    u64 bh0 = 0, bl0 = 0, bh1 = 0, bl1 = 0, ah0 = 0, al0 = 0, ah1 = 0, al1 = 0;
    // running pointers (one 64-bit add per digit instead of re-deriving
    // every address from the digit index)
    const u64* kbp = kb_base + k;
    const u64* kap = ka_base + k;
    const u64* rp = rsrc;
    for (u32 j0 = 0; j0 < ndig; j0 += JB) {
      ulonglong2 KB[JB], KA[JB], X[JB];
#pragma unroll
      for (int i = 0; i < JB; ++i) {
        const u32 j = j0 + i;
        if (j < ndig) {
          KB[i] = *reinterpret_cast<const ulonglong2*>(kbp);
          KA[i] = *reinterpret_cast<const ulonglong2*>(kap);
          const u64* src = j == own ? xsrc : rp;
          if (g == 1) {
            X[i] = *reinterpret_cast<const ulonglong2*>(src + k);
          } else {
            X[i].x = src[p0];
            X[i].y = src[p1];
          }
        } else {
          KB[i] = KA[i] = X[i] = make_ulonglong2(0, 0);
        }
        kbp += key_dst;
        kap += key_dst;
        rp += rstep;
      }
      if (f96) {
#pragma unroll
        for (int i = 0; i < JB; ++i) {
          const u32 x0 = (u32)X[i].x, x1 = (u32)(X[i].x >> 32), y0 = (u32)X[i].y, y1 = (u32)(X[i].y >> 32);
          mac96(bh0, bl0, x0, x1, (u32)KB[i].x, (u32)(KB[i].x >> 32));
          mac96(ah0, al0, x0, x1, (u32)KA[i].x, (u32)(KA[i].x >> 32));
          mac96(bh1, bl1, y0, y1, (u32)KB[i].y, (u32)(KB[i].y >> 32));
          mac96(ah1, al1, y0, y1, (u32)KA[i].y, (u32)(KA[i].y >> 32));
        }
        continue;
      }
#pragma unroll
      for (int i = 0; i < JB; ++i) {
        mac128_lazy(bh0, bl0, X[i].x, KB[i].x);
        mac128_lazy(ah0, al0, X[i].x, KA[i].x);
        mac128_lazy(bh1, bl1, X[i].y, KB[i].y);
        mac128_lazy(ah1, al1, X[i].y, KA[i].y);
      }
      if ((j0 + JB) % kLazyTerms == 0) {  // never more than kLazyTerms unfolded products
        bh0 = fold_hi(bh0, q, one_sh);
        bh1 = fold_hi(bh1, q, one_sh);
        ah0 = fold_hi(ah0, q, one_sh);
        ah1 = fold_hi(ah1, q, one_sh);
      }
    }
    if (c0 && r < basis.nq) {  // extended-basis output: + P * sigma_g(c0) on the Q limbs
      const u64 w = pR[r];
      const u64* src = c0 + (size_t)b * c0_bst + (size_t)r * N;
      const u64 s0 = src[p0], s1 = src[p1];
      if (f96) {
        mac96(bh0, bl0, (u32)s0, (u32)(s0 >> 32), (u32)w, (u32)(w >> 32));
        mac96(bh1, bl1, (u32)s1, (u32)(s1 >> 32), (u32)w, (u32)(w >> 32));
      } else {
        mac128_lazy(bh0, bl0, s0, w);
        mac128_lazy(bh1, bl1, s1, w);
      }
    }
    if (f96) {
      u64* A = acc + (size_t)b * 2 * n_ext * N;
      *reinterpret_cast<ulonglong2*>(A + (size_t)r * N + k) =
          make_ulonglong2(redc96(bh0, bl0, q, ninv), redc96(bh1, bl1, q, ninv));
      *reinterpret_cast<ulonglong2*>(A + ((size_t)n_ext + r) * N + k) =
          make_ulonglong2(redc96(ah0, al0, q, ninv), redc96(ah1, al1, q, ninv));
      continue;
    }
    bh0 = fold_hi(bh0, q, one_sh);
    bh1 = fold_hi(bh1, q, one_sh);
    ah0 = fold_hi(ah0, q, one_sh);
    ah1 = fold_hi(ah1, q, one_sh);
    u64* A = acc + (size_t)b * 2 * n_ext * N;
    *reinterpret_cast<ulonglong2*>(A + (size_t)r * N + k) =
        make_ulonglong2(redc128(bh0, bl0, q, ninv), redc128(bh1, bl1, q, ninv));
    *reinterpret_cast<ulonglong2*>(A + ((size_t)n_ext + r) * N + k) =
        make_ulonglong2(redc128(ah0, al0, q, ninv), redc128(ah1, al1, q, ninv));
  }
}

// ModDown combine (ckks.py:593-601): out_z[r] = add_z[perm(k)] + (acc_z[r] - lift_z[r]) * P^-1
__global__ void __launch_bounds__(256) k_moddown_combine(u64* __restrict__ out0, u64* __restrict__ out1,
                                                         const u64* __restrict__ acc, const u64* __restrict__ lift,
                                                         const u64* __restrict__ add0, const u64* __restrict__ add1,
                                                         u64 g_add, u32 nq, u32 n_ext, u32 logN,
                                                         const u64* __restrict__ pinv, const u64* __restrict__ pinv_sh,
                                                         const ModConsts* __restrict__ mc, size_t out_bst,
                                                         size_t add_bst) {
  // z = 2 b + p: poly p of batch entry b (acc [nb][2][n_ext], lift [nb][2][nq])
  const u32 N = 1u << logN, r = blockIdx.y, z = blockIdx.z, b = z >> 1, p = z & 1;
  const u64 q = mc[r].q;
  const u64 w = pinv[r], wp = pinv_sh[r];
  const u64* A = acc + ((size_t)z * n_ext + r) * N;
  const u64* L = lift + ((size_t)z * nq + r) * N;
  const u64* ADD = p == 0 ? add0 : add1;
  if (ADD) ADD += (size_t)b * add_bst;
  u64* O = (p == 0 ? out0 : out1) + (size_t)b * out_bst + (size_t)r * N;
  for (u32 k2 = blockIdx.x * blockDim.x + threadIdx.x; k2 < N / 2; k2 += gridDim.x * blockDim.x) {
    const u32 k = 2 * k2;
    const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(A + k);
    const ulonglong2 l = *reinterpret_cast<const ulonglong2*>(L + k);
    u64 v0 = shoup_mul(sub_mod(a.x, l.x, q), w, wp, q);
    u64 v1 = shoup_mul(sub_mod(a.y, l.y, q), w, wp, q);
    if (ADD) {
      const u64* ar = ADD + (size_t)r * N;
      if (g_add == 1) {
        const ulonglong2 d = *reinterpret_cast<const ulonglong2*>(ar + k);
        v0 = add_mod(v0, d.x, q);
        v1 = add_mod(v1, d.y, q);
      } else {
        v0 = add_mod(v0, ar[galois_src(k, g_add, logN)], q);
        v1 = add_mod(v1, ar[galois_src(k + 1, g_add, logN)], q);
      }
    }
    *reinterpret_cast<ulonglong2*>(O + k) = make_ulonglong2(v0, v1);
  }
}

// The same for the rotations of one hoisted group done together: acc / lift
// hold [n_rot][nb][2][..]; z = (s*nb + b)*2 + p; each step s writes its own
// output batch and gathers c0 with its own Galois element.
__global__ void __launch_bounds__(256) k_moddown_combine_steps(ComboSteps S, const u64* __restrict__ acc,
                                                               const u64* __restrict__ lift,
                                                               const u64* __restrict__ add0, u32 nb, u32 nq,
                                                               u32 n_ext, u32 logN, const u64* __restrict__ pinv,
                                                               const u64* __restrict__ pinv_sh,
                                                               const ModConsts* __restrict__ mc, size_t out_bst,
                                                               size_t add_bst) {
  const u32 N = 1u << logN, r = blockIdx.y, z = blockIdx.z, p = z & 1, sb = z >> 1, s = sb / nb, b = sb % nb;
  const u64 q = mc[r].q;
  const u64 w = pinv[r], wp = pinv_sh[r];
  const u64 g_add = S.g[s];
  const u64* A = acc + ((size_t)z * n_ext + r) * N;
  const u64* L = lift + ((size_t)z * nq + r) * N;
  const u64* ADD = (p == 0 && add0) ? add0 + (size_t)b * add_bst + (size_t)r * N : nullptr;
  u64* O = S.out[s] + (size_t)b * out_bst + (size_t)p * nq * N + (size_t)r * N;
  for (u32 k2 = blockIdx.x * blockDim.x + threadIdx.x; k2 < N / 2; k2 += gridDim.x * blockDim.x) {
    const u32 k = 2 * k2;
    const ulonglong2 av = *reinterpret_cast<const ulonglong2*>(A + k);
    const ulonglong2 lv = *reinterpret_cast<const ulonglong2*>(L + k);
    u64 v0 = shoup_mul(sub_mod(av.x, lv.x, q), w, wp, q);
    u64 v1 = shoup_mul(sub_mod(av.y, lv.y, q), w, wp, q);
    if (ADD) {
      v0 = add_mod(v0, ADD[g_add == 1 ? k : galois_src(k, g_add, logN)], q);
      v1 = add_mod(v1, ADD[g_add == 1 ? k + 1 : galois_src(k + 1, g_add, logN)], q);
    }
    *reinterpret_cast<ulonglong2*>(O + k) = make_ulonglong2(v0, v1);
  }
}

// k_moddown_combine for rows r0.. of the lift from an NttCombine
// descriptor (the rows whose lift NTT ran on the integer network)
__global__ void __launch_bounds__(256) k_combine_rows(NttCombine C, const u64* __restrict__ lift, u32 nq, u32 r0,
                                                     u32 logN, const ModConsts* __restrict__ mc) {
  const u32 N = 1u << logN, r = blockIdx.y + r0, z = blockIdx.z, p = z & 1, sb = z >> 1, s = sb / C.nb,
            b = sb % C.nb;
  const u64 q = mc[r].q;
  const u64 w = C.pinv[r], wp = C.pinv_sh[r];
  const u64 g_add = C.g[s];
  const u64* A = C.acc + (size_t)z * C.acc_pst + (size_t)r * N;
  const u64* L = lift + ((size_t)z * nq + r) * N;
  const u64* ADD = C.add[p] ? C.add[p] + (size_t)b * C.add_bst + (size_t)r * N : nullptr;
  u64* O = C.out[s] + (size_t)b * C.out_bst + (size_t)p * C.out_pst + (size_t)r * N;
  for (u32 k2 = blockIdx.x * blockDim.x + threadIdx.x; k2 < N / 2; k2 += gridDim.x * blockDim.x) {
    const u32 k = 2 * k2;
    const ulonglong2 av = *reinterpret_cast<const ulonglong2*>(A + k);
    const ulonglong2 lv = *reinterpret_cast<const ulonglong2*>(L + k);
    u64 v0 = shoup_mul(sub_mod(av.x, lv.x, q), w, wp, q);
    u64 v1 = shoup_mul(sub_mod(av.y, lv.y, q), w, wp, q);
    if (ADD) {
      v0 = add_mod(v0, ADD[g_add == 1 ? k : galois_src(k, g_add, logN)], q);
      v1 = add_mod(v1, ADD[g_add == 1 ? k + 1 : galois_src(k + 1, g_add, logN)], q);
    }
    *reinterpret_cast<ulonglong2*>(O + k) = make_ulonglong2(v0, v1);
  }
}

cudaError_t launch_combine_rows(const NttCombine& C, const u64* lift, u32 nq, u32 r0, u32 nrows, u32 npolys,
                                u32 logN, const ModConsts* mc, cudaStream_t st) {
  if (nrows == 0 || npolys == 0) return cudaSuccess;
  dim3 g = row_grid((1u << logN) / 2, nrows, 256);
  g.z = npolys;
  k_combine_rows<<<g, 256, 0, st>>>(C, lift, nq, r0, logN, mc);
  return cudaGetLastError();
}

// acc_{b,p}[r] += P * d_{b,p}[r] mod q_r on the Q limbs of nb extended-basis
// accumulators ([nb][2][n_ext]); d is [nb][2][nq] (the tensor product's d0,
// d1), pR = P R mod q_r (Montgomery form, so one REDC gives P d).  Fused
// hmult + rescale: the key-switch sum and P (d0, d1) share one ModDown.
__global__ void __launch_bounds__(256) k_add_pmul(u64* __restrict__ acc, const u64* __restrict__ d, u32 nq,
                                                  u32 n_ext, u32 logN, const u64* __restrict__ pR,
                                                  const ModConsts* __restrict__ mc) {
  const u32 N = 1u << logN, r = blockIdx.y, z = blockIdx.z;
  const u64 q = mc[r].q, ninv = mc[r].ninv, w = pR[r];
  u64* A = acc + ((size_t)z * n_ext + r) * N;
  const u64* D = d + ((size_t)z * nq + r) * N;
  for (u32 k2 = blockIdx.x * blockDim.x + threadIdx.x; k2 < N / 2; k2 += gridDim.x * blockDim.x) {
    const u32 k = 2 * k2;
    const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(A + k);
    const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(D + k);
    *reinterpret_cast<ulonglong2*>(A + k) =
        make_ulonglong2(add_mod(a.x, mont_mul(x.x, w, q, ninv), q), add_mod(a.y, mont_mul(x.y, w, q, ninv), q));
  }
}

cudaError_t launch_add_pmul(u64* acc, const u64* d, u32 nb, u32 nq, u32 n_ext, u32 logN, const u64* pR,
                            const ModConsts* mc, cudaStream_t st) {
  dim3 g = row_grid((1u << logN) / 2, nq, 256);
  g.z = 2 * nb;
  k_add_pmul<<<g, 256, 0, st>>>(acc, d, nq, n_ext, logN, pR, mc);
  return cudaGetLastError();
}

cudaError_t launch_moddown_combine_steps(const ComboSteps& S, u32 n_rot, const u64* acc, const u64* lift,
                                         const u64* add0, u32 nb, u32 nq, u32 n_ext, u32 logN, const u64* pinv,
                                         const u64* pinv_sh, const ModConsts* mc, size_t out_bst, size_t add_bst,
                                         cudaStream_t st) {
  dim3 g = row_grid((1u << logN) / 2, nq, 256);
  g.z = 2 * nb * n_rot;
  k_moddown_combine_steps<<<g, 256, 0, st>>>(S, acc, lift, add0, nb, nq, n_ext, logN, pinv, pinv_sh, mc, out_bst,
                                             add_bst);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// plane MAC of the HyPHEN conv (packing.py:600-604 / :520-525):
// out_z = sum_t ct_t,z (.) mask_t over up to kMacMax terms, masks in
// Montgomery form -> one 128-bit sum and one REDC per residue (bit-exact
// with the reference's hadd(pmult_mont) chain since every partial result
// is canonical).  accumulate: out += sum.
// ---------------------------------------------------------------------------
template <int NB, int VEC>
__global__ void __launch_bounds__(256) k_mac_terms(MacTerms T, int nt, u64* __restrict__ out, u32 nq, u32 logN,
                                                   int accumulate, const ModConsts* __restrict__ mc, u32 nb, u32 nl,
                                                   u32 Lq) {
  // one thread: VEC adjacent coefficients of both polys of NB batch entries
  // (ciphertexts 2*nl*N apart, nl = nq or nq + K limbs for Q||P); each mask
  // load feeds all of them
  // NB == 1: blockIdx.x = tile * nb + entry (entries sharing a mask tile run
  // back to back: the mask streams once per batch)
  const u32 N = 1u << logN, r = blockIdx.y, b0 = NB == 1 ? blockIdx.x % nb : blockIdx.z * NB;
  const u32 ne = nb - b0 < (u32)NB ? nb - b0 : (u32)NB;
  const u32 x0 = NB == 1 ? blockIdx.x / nb : blockIdx.x, xs = NB == 1 ? gridDim.x / nb : gridDim.x;
  const u32 mod = r < nq ? r : Lq + (r - nq);
  const u64 q = mc[mod].q, ninv = mc[mod].ninv, one_sh = mc[mod].one_sh;
  // rows with q < 2^42: 96-bit carry chains (see k_ks_inner_tma2; nt <= 48 keeps T < 2^90)
  const bool f96 = g_ks96_dev && q < (1ull << 42) && nt <= 48;
  const size_t bst = 2 * (size_t)nl * N, pst = (size_t)nl * N;
  const size_t off = (size_t)r * N + (size_t)b0 * bst, moff = (size_t)r * N;
  for (u32 kv = x0 * blockDim.x + threadIdx.x; kv < N / VEC; kv += xs * blockDim.x) {
    const u32 k = kv * VEC;
    u64 hi[NB][2][VEC], lo[NB][2][VEC];
#pragma unroll
    for (int e = 0; e < NB; ++e)
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int v = 0; v < VEC; ++v) hi[e][p][v] = lo[e][p][v] = 0;
#pragma unroll 2
    for (int t = 0; t < nt; ++t) {
      u64 m[VEC];
      if (VEC == 2) {
        const ulonglong2 m2 = *reinterpret_cast<const ulonglong2*>(T.mask[t] + moff + k);
        m[0] = m2.x;
        m[VEC - 1] = m2.y;
      } else {
        m[0] = T.mask[t][moff + k];
      }
#pragma unroll
      for (int e = 0; e < NB; ++e) {
        if ((u32)e >= ne) break;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const u64* src = T.ct[t] + off + e * bst + p * pst + k;
          u64 x[VEC];
          if (VEC == 2) {
            const ulonglong2 x2 = *reinterpret_cast<const ulonglong2*>(src);
            x[0] = x2.x;
            x[VEC - 1] = x2.y;
          } else {
            x[0] = *src;
          }
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            if (f96) mac96(hi[e][p][v], lo[e][p][v], (u32)x[v], (u32)(x[v] >> 32), (u32)m[v], (u32)(m[v] >> 32));
            else mac128_lazy(hi[e][p][v], lo[e][p][v], x[v], m[v]);
          }
        }
      }
      if (!f96 && ((t + 1) % kLazyTerms == 0 || t + 1 == nt)) {
#pragma unroll
        for (int e = 0; e < NB; ++e)
#pragma unroll
          for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int v = 0; v < VEC; ++v) hi[e][p][v] = fold_hi(hi[e][p][v], q, one_sh);
      }
    }
#pragma unroll
    for (int e = 0; e < NB; ++e) {
      if ((u32)e >= ne) break;
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        u64* dst = out + off + e * bst + p * pst + k;
        u64 y[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v)
          y[v] = f96 ? redc96(hi[e][p][v], lo[e][p][v], q, ninv) : redc128(hi[e][p][v], lo[e][p][v], q, ninv);
        if (VEC == 2) {
          if (accumulate) {
            const ulonglong2 o = *reinterpret_cast<const ulonglong2*>(dst);
            y[0] = add_mod(y[0], o.x, q);
            y[VEC - 1] = add_mod(y[VEC - 1], o.y, q);
          }
          *reinterpret_cast<ulonglong2*>(dst) = make_ulonglong2(y[0], y[VEC - 1]);
        } else {
          if (accumulate) y[0] = add_mod(y[0], *dst, q);
          *dst = y[0];
        }
      }
    }
  }
}

cudaError_t launch_mac_terms(const MacTerms& T, int nt, u64* out, u32 nq, u32 logN, int accumulate,
                             const ModConsts* mc, cudaStream_t st, u32 nb, u32 np, u32 Lq) {
  const u32 nl = nq + np;
  if (nb <= 1 || g_mac_batch <= 1) {
    dim3 g = row_grid((1u << logN) / 2, nl, 256);
    g.x *= (nb ? nb : 1);
    k_mac_terms<1, 2><<<g, 256, 0, st>>>(T, nt, out, nq, logN, accumulate, mc, nb ? nb : 1, nl, Lq);
  } else {
    dim3 g = row_grid(1u << logN, nl, 256);
    g.z = (nb + 3) / 4;
    k_mac_terms<4, 1><<<g, 256, 0, st>>>(T, nt, out, nq, logN, accumulate, mc, nb, nl, Lq);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// rescale (ckks.py:506-528)
// ---------------------------------------------------------------------------
// centred lift of the (coefficient-domain) top limb into limbs 0..l-1
__global__ void k_rescale_lift(u64* __restrict__ out, const u64* __restrict__ top, u32 l, u32 logN,
                               const u64* __restrict__ qtop_mod, const ModConsts* __restrict__ mc) {
  const u32 N = 1u << logN, i = blockIdx.y, z = blockIdx.z;
  const ModConsts C = mc[i];
  const u64 qt = mc[l].q;
  const u64 qt_mod = qtop_mod[i];  // q_l mod q_i (host table)
  const u64* T = top + (size_t)z * N;
  u64* O = out + ((size_t)z * l + i) * N;
  for (u32 k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
    u64 t = T[k];
    u64 rr = mont_mul(t, C.one_m, C.q, C.ninv);  // t mod q_i
    if (t > (qt >> 1)) rr = sub_mod(rr, qt_mod, C.q);
    O[k] = rr;
  }
}

// out = (body - lift) * q_l^-1 ; lift already NTT'd in `out`
__global__ void k_rescale_combine(u64* __restrict__ out, const u64* __restrict__ in, u32 l, u32 logN,
                                  const u64* __restrict__ inv, const u64* __restrict__ inv_sh,
                                  const ModConsts* __restrict__ mc) {
  const u32 N = 1u << logN, i = blockIdx.y, z = blockIdx.z;
  const u64 q = mc[i].q, w = inv[i], wp = inv_sh[i];
  const u64* B = in + ((size_t)z * (l + 1) + i) * N;
  u64* O = out + ((size_t)z * l + i) * N;
  for (u32 k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x)
    O[k] = shoup_mul(sub_mod(B[k], O[k], q), w, wp, q);
}

// copy the top limb (index l) of each poly into a packed [npolys][N] buffer
__global__ void k_gather_limb(u64* __restrict__ out, const u64* __restrict__ in, u32 limb, u32 nlimbs, u32 logN) {
  const u32 N = 1u << logN, z = blockIdx.y;
  const u64* I = in + ((size_t)z * nlimbs + limb) * N;
  for (u32 k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) out[(size_t)z * N + k] = I[k];
}

template <int G, int VEC>
__global__ void __launch_bounds__(256) k_mac_multi(MacMulti M, int nt, u32 nq, u32 logN, int accumulate,
                                                   const ModConsts* __restrict__ mc) {
  // VEC adjacent coefficients of both polys for G outputs per thread: each
  // ciphertext load feeds every output that has a mask for it
  const u32 N = 1u << logN, r = blockIdx.y;
  const u64 q = mc[r].q, ninv = mc[r].ninv;
  const size_t pst = (size_t)nq * N, off = (size_t)r * N;
  for (u32 kv = blockIdx.x * blockDim.x + threadIdx.x; kv < N / VEC; kv += gridDim.x * blockDim.x) {
    const u32 k = VEC * kv;
    // byte offsets of this thread's coefficient in a packed mask's planes (limb r > 0)
    const size_t lo_off = 8 * (size_t)N + 4 * ((size_t)(r - 1) * N + k);
    const unsigned hb = r > 0 ? packed_hb(r, M.wide) : 2u;
    const size_t hi_plane = r > 0 ? packed_hi_off(r, nq, N, M.wide) : 0;
    u64 hi[G][2][VEC], lo[G][2][VEC];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int v = 0; v < VEC; ++v) hi[g][p][v] = lo[g][p][v] = 0;
#pragma unroll 2
    for (int t = 0; t < nt; ++t) {
      // all loads of the term first (null masks predicated to zero) so the
      // unrolled iterations keep several loads in flight
      u64 x[2][VEC], m[G][VEC];
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const u64* src = M.ct[t] + p * pst + off + k;
        if (VEC == 2) {
          const ulonglong2 v2 = *reinterpret_cast<const ulonglong2*>(src);
          x[p][0] = v2.x;
          x[p][VEC - 1] = v2.y;
        } else {
          x[p][0] = *src;
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const u64* mp = M.mask[g][t];
        if (mp && M.packed[g][t] && r > 0) {  // 48-bit packed limb: u32 low plane + u16 high plane
          const char* b = reinterpret_cast<const char*>(mp);
          const unsigned char* hp = reinterpret_cast<const unsigned char*>(b + hi_plane);
          if (VEC == 2) {
            const uint2 l2 = *reinterpret_cast<const uint2*>(b + lo_off);
            m[g][0] = (u64)l2.x | (packed_hi(hp, k, hb) << 32);
            m[g][VEC - 1] = (u64)l2.y | (packed_hi(hp, k + 1, hb) << 32);
          } else {
            m[g][0] = (u64)*reinterpret_cast<const unsigned*>(b + lo_off) | (packed_hi(hp, k, hb) << 32);
          }
          continue;
        }
        const u64* src = (mp && M.packed[g][t]) ? mp + k : mp + off + k;  // packed limb 0 sits first
        if (VEC == 2) {
          const ulonglong2 m2 = mp ? *reinterpret_cast<const ulonglong2*>(src) : make_ulonglong2(0, 0);
          m[g][0] = m2.x;
          m[g][VEC - 1] = m2.y;
        } else {
          m[g][0] = mp ? *src : 0ull;
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
          for (int v = 0; v < VEC; ++v) mac128(hi[g][p][v], lo[g][p][v], x[p][v], m[g][v], q);
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        u64* dst = M.out[g] + p * pst + off + k;
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          u64 y = redc128(hi[g][p][v], lo[g][p][v], q, ninv);
          if (accumulate) y = add_mod(y, dst[v], q);
          dst[v] = y;
        }
      }
    }
  }
}

__global__ void k_pack_masks(unsigned char* __restrict__ out, const u64* __restrict__ in, u32 nq, u32 logN,
                             unsigned long long wide, size_t mbytes) {
  const u32 N = 1u << logN, r = blockIdx.y, m = blockIdx.z;
  unsigned char* base = out + (size_t)m * mbytes;
  const u64* src = in + ((size_t)m * nq + r) * N;
  const unsigned hb = r > 0 ? packed_hb(r, wide) : 0u;
  unsigned char* hp = r > 0 ? base + packed_hi_off(r, nq, N, wide) : nullptr;
  for (u32 k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
    const u64 v = src[k];
    if (r == 0) {
      reinterpret_cast<u64*>(base)[k] = v;
    } else {
      reinterpret_cast<unsigned*>(base + 8 * (size_t)N)[(size_t)(r - 1) * N + k] = (unsigned)v;
      if (hb == 2) reinterpret_cast<unsigned short*>(hp)[k] = (unsigned short)(v >> 32);
      else hp[k] = (unsigned char)(v >> 32);
    }
  }
}

__global__ void k_unpack_mask(u64* __restrict__ out, const unsigned char* __restrict__ in, u32 nq, u32 logN,
                              unsigned long long wide) {
  const u32 N = 1u << logN, r = blockIdx.y;
  const unsigned hb = r > 0 ? packed_hb(r, wide) : 0u;
  const unsigned char* hp = r > 0 ? in + packed_hi_off(r, nq, N, wide) : nullptr;
  for (u32 k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
    u64 v;
    if (r == 0) {
      v = reinterpret_cast<const u64*>(in)[k];
    } else {
      v = (u64)reinterpret_cast<const unsigned*>(in + 8 * (size_t)N)[(size_t)(r - 1) * N + k] |
          (packed_hi(hp, k, hb) << 32);
    }
    out[(size_t)r * N + k] = v;
  }
}

static size_t packed_bytes(u32 nq, size_t N, unsigned long long wide) {
  return nq > 1 ? packed_hi_off(nq, nq, N, wide) : 8 * N;  // offset one past the last limb's high plane
}

cudaError_t launch_pack_masks(unsigned char* out, const u64* in, u32 nm, u32 nq, u32 logN, unsigned long long wide,
                              cudaStream_t st) {
  if (!nm || !nq) return cudaSuccess;
  dim3 g = row_grid(1u << logN, nq, 256);
  g.z = nm;
  k_pack_masks<<<g, 256, 0, st>>>(out, in, nq, logN, wide, packed_bytes(nq, 1u << logN, wide));
  return cudaGetLastError();
}

cudaError_t launch_unpack_mask(u64* out, const unsigned char* in, u32 nq, u32 logN, unsigned long long wide,
                               cudaStream_t st) {
  k_unpack_mask<<<row_grid(1u << logN, nq, 256), 256, 0, st>>>(out, in, nq, logN, wide);
  return cudaGetLastError();
}

// One lane per (output g, coefficient pair): the 4 lanes of a pair sit in one
// warp, so each ciphertext load is one broadcast transaction feeding all
// outputs, while every lane keeps only its own 8 accumulator words (high
// occupancy, many loads in flight).
__global__ void __launch_bounds__(256) k_mac_multi_lanes(MacMulti M, int ng, int nt, u32 nq, u32 logN,
                                                         int accumulate, const ModConsts* __restrict__ mc) {
  const u32 N = 1u << logN, r = blockIdx.y;
  const u32 g = threadIdx.x & 3u;
  const u32 kp = blockIdx.x * (blockDim.x >> 2) + (threadIdx.x >> 2);  // coefficient pair
  if (kp >= N / 2 || (int)g >= ng) return;
  const u32 k = 2 * kp;
  const u64 q = mc[r].q, ninv = mc[r].ninv;
  const size_t pst = (size_t)nq * N, off = (size_t)r * N;
  const size_t lo_off = 8 * (size_t)N + 4 * ((size_t)(r - 1) * N + k);
  const unsigned hb = r > 0 ? packed_hb(r, M.wide) : 2u;
  const size_t hi_plane = r > 0 ? packed_hi_off(r, nq, N, M.wide) : 0;
  u64 h00 = 0, l00 = 0, h01 = 0, l01 = 0, h10 = 0, l10 = 0, h11 = 0, l11 = 0;
#pragma unroll 4
  for (int t = 0; t < nt; ++t) {
    const u64* mp = M.mask[g][t];
    if (!mp) continue;
    u64 m0, m1;
    if (M.packed[g][t] && r > 0) {
      const char* b = reinterpret_cast<const char*>(mp);
      const unsigned char* hp = reinterpret_cast<const unsigned char*>(b + hi_plane);
      const uint2 l2 = *reinterpret_cast<const uint2*>(b + lo_off);
      m0 = (u64)l2.x | (packed_hi(hp, k, hb) << 32);
      m1 = (u64)l2.y | (packed_hi(hp, k + 1, hb) << 32);
    } else {
      const ulonglong2 m2 = *reinterpret_cast<const ulonglong2*>(M.packed[g][t] ? mp + k : mp + off + k);
      m0 = m2.x;
      m1 = m2.y;
    }
    const ulonglong2 x0 = *reinterpret_cast<const ulonglong2*>(M.ct[t] + off + k);
    const ulonglong2 x1 = *reinterpret_cast<const ulonglong2*>(M.ct[t] + pst + off + k);
    mac128(h00, l00, x0.x, m0, q);
    mac128(h01, l01, x0.y, m1, q);
    mac128(h10, l10, x1.x, m0, q);
    mac128(h11, l11, x1.y, m1, q);
  }
  u64* d0 = M.out[g] + off + k;
  u64* d1 = M.out[g] + pst + off + k;
  u64 y00 = redc128(h00, l00, q, ninv), y01 = redc128(h01, l01, q, ninv);
  u64 y10 = redc128(h10, l10, q, ninv), y11 = redc128(h11, l11, q, ninv);
  if (accumulate) {
    const ulonglong2 o0 = *reinterpret_cast<const ulonglong2*>(d0);
    const ulonglong2 o1 = *reinterpret_cast<const ulonglong2*>(d1);
    y00 = add_mod(y00, o0.x, q);
    y01 = add_mod(y01, o0.y, q);
    y10 = add_mod(y10, o1.x, q);
    y11 = add_mod(y11, o1.y, q);
  }
  *reinterpret_cast<ulonglong2*>(d0) = make_ulonglong2(y00, y01);
  *reinterpret_cast<ulonglong2*>(d1) = make_ulonglong2(y10, y11);
}


// ---------------------------------------------------------------------------
// Shared-term MAC with a cp.async pipeline: a CTA owns a 256-coefficient
// tile of one limb for up to 4 outputs; per term it stages the ciphertext
// tile (2 polys) and the outputs' mask tiles (u64, or the 48-bit packed
// planes) into shared memory kMacStages terms ahead, so HBM latency overlaps
// the 8 mac128 per coefficient of the current term.
// ---------------------------------------------------------------------------
constexpr int kMacStages = 4;
constexpr int kMacTile = 256;
struct MacStage {
  u64 ct[2][kMacTile];
  u64 mask[kMultiG][kMacTile];  // unpacked rows, or lo u32 [256] + hi u16 [256] when packed
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void mac_stage_issue(MacStage& S, const MacMulti& M, int t, int ng, u32 r, u32 nq, u32 N,
                                                u32 k0) {
  const u32 tid = threadIdx.x;
  const size_t off = (size_t)r * N + k0, pst = (size_t)nq * N;
  // ciphertext: 2 polys x 2 KB = 256 chunks of 16 B
  {
    const u32 p = tid >> 7, c = tid & 127u;
    cp_async16(&S.ct[p][2 * c], M.ct[t] + p * pst + off + 2 * c);
  }
  for (int g = 0; g < ng; ++g) {
    const u64* mp = M.mask[g][t];
    if (!mp) continue;
    if (M.packed[g][t] && r > 0) {
      const char* b = reinterpret_cast<const char*>(mp);
      const char* lo = b + 8 * (size_t)N + 4 * ((size_t)(r - 1) * N + k0);
      const unsigned hb = packed_hb(r, M.wide);
      const char* hi = b + packed_hi_off(r, nq, N, M.wide) + (size_t)hb * k0;
      char* dst = reinterpret_cast<char*>(S.mask[g]);
      const u32 nhi = 16 * hb;  // 16-byte chunks of the 256-coefficient high plane
      if (tid < 64) cp_async16(dst + 16 * tid, lo + 16 * tid);                            // 1 KB low words
      else if (tid < 64 + nhi) cp_async16(dst + 1024 + 16 * (tid - 64), hi + 16 * (tid - 64));  // 256 / 512 B high
    } else {
      const u64* src = M.packed[g][t] ? mp + k0 : mp + off;  // packed limb 0 is a plain u64 row
      if (tid < 128) cp_async16(&S.mask[g][2 * tid], src + 2 * tid);
    }
  }
}

__global__ void __launch_bounds__(256) k_mac_multi_async(MacMulti M, int ng, int nt, u32 nq, u32 logN,
                                                         int accumulate, const ModConsts* __restrict__ mc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MacStage* S = reinterpret_cast<MacStage*>(smem_raw);
  const u32 N = 1u << logN, r = blockIdx.y, k0 = blockIdx.x * kMacTile, tid = threadIdx.x;
  const u64 q = mc[r].q, ninv = mc[r].ninv, one_sh = mc[r].one_sh;
  for (int s = 0; s < kMacStages - 1; ++s) {
    if (s < nt) mac_stage_issue(S[s], M, s, ng, r, nq, N, k0);
    cp_async_commit();
  }
  u64 h[kMultiG][2], l[kMultiG][2];
#pragma unroll
  for (int g = 0; g < kMultiG; ++g) h[g][0] = h[g][1] = l[g][0] = l[g][1] = 0;
  for (int t = 0; t < nt; ++t) {
    cp_async_wait<kMacStages - 2>();
    __syncthreads();
    {  // refill the slot consumed last iteration
      const int tn = t + kMacStages - 1;
      if (tn < nt) mac_stage_issue(S[tn % kMacStages], M, tn, ng, r, nq, N, k0);
      cp_async_commit();
    }
    const MacStage& C = S[t % kMacStages];
    const u64 x0 = C.ct[0][tid], x1 = C.ct[1][tid];
#pragma unroll
    for (int g = 0; g < kMultiG; ++g) {
      if (g >= ng || !M.mask[g][t]) continue;
      u64 m;
      if (M.packed[g][t] && r > 0) {
        const unsigned* lo = reinterpret_cast<const unsigned*>(C.mask[g]);
        m = (u64)lo[tid] | (packed_hi(reinterpret_cast<const unsigned char*>(C.mask[g]) + 1024, tid,
                                      packed_hb(r, M.wide)) << 32);
      } else {
        m = C.mask[g][tid];
      }
      mac128_lazy(h[g][0], l[g][0], x0, m);
      mac128_lazy(h[g][1], l[g][1], x1, m);
    }
    if ((t + 1) % kLazyTerms == 0 || t + 1 == nt) {
#pragma unroll
      for (int g = 0; g < kMultiG; ++g) {
        h[g][0] = fold_hi(h[g][0], q, one_sh);
        h[g][1] = fold_hi(h[g][1], q, one_sh);
      }
    }
  }
  cp_async_wait<0>();
  const size_t pst = (size_t)nq * N, off = (size_t)r * N + k0 + tid;
#pragma unroll
  for (int g = 0; g < kMultiG; ++g) {
    if (g >= ng) break;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      u64* d = M.out[g] + p * pst + off;
      u64 y = redc128(h[g][p], l[g][p], q, ninv);
      if (accumulate) y = add_mod(y, *d, q);
      *d = y;
    }
  }
}

// ---------------------------------------------------------------------------
// The same shared-term MAC with the staging done by the bulk-copy engine
// (TMA, cp.async.bulk): per term one elected thread arms the stage's
// mbarrier with the byte count and issues <= 10 contiguous row copies
// (2 ciphertext polys of 2 KB, each output's mask row: 2 KB, or the 1 KB
// low + 512 B high planes of a packed limb).  The other 255 threads spend
// no instructions on address generation or copy issue; they wait on the
// stage's mbarrier phase and run the 8 lazy MACs per term.  Branches on
// mask presence / packing read one flag byte per term staged in smem.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mac_stage_bulk(MacStage& S, u64* bar, const MacMulti& M, int t, u32 fl, u32 r,
                                               u32 nq, u32 N, u32 k0) {
  const size_t off = (size_t)r * N + k0, pst = (size_t)nq * N;
  u32 bytes = 2 * kMacTile * 8;
  const u32 pk = kMacTile * (4 + (r > 0 ? packed_hb(r, M.wide) : 2u));  // packed tile bytes of this limb
  for (int g = 0; g < kMultiG; ++g)
    if (fl >> g & 1u) bytes += (fl >> (4 + g) & 1u) ? pk : kMacTile * 8;
  mbar_expect_tx(bar, bytes);
  bulk_g2s(S.ct[0], M.ct[t] + off, kMacTile * 8, bar);
  bulk_g2s(S.ct[1], M.ct[t] + pst + off, kMacTile * 8, bar);
  for (int g = 0; g < kMultiG; ++g) {
    if (!(fl >> g & 1u)) continue;
    const u64* mp = M.mask[g][t];
    if (fl >> (4 + g) & 1u) {
      const char* b = reinterpret_cast<const char*>(mp);
      char* dst = reinterpret_cast<char*>(S.mask[g]);
      const unsigned hb = packed_hb(r, M.wide);
      bulk_g2s(dst, b + 8 * (size_t)N + 4 * ((size_t)(r - 1) * N + k0), kMacTile * 4, bar);
      bulk_g2s(dst + kMacTile * 4, b + packed_hi_off(r, nq, N, M.wide) + (size_t)hb * k0, kMacTile * hb, bar);
    } else {
      bulk_g2s(S.mask[g], M.packed[g][t] ? mp + k0 : mp + off, kMacTile * 8, bar);  // packed limb 0: u64 row
    }
  }
}

template <int ST>
__global__ void __launch_bounds__(256) k_mac_multi_tma(MacMulti M, int ng, int nt, u32 nq, u32 logN,
                                                       int accumulate, const ModConsts* __restrict__ mc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MacStage* S = reinterpret_cast<MacStage*>(smem_raw);
  __shared__ __align__(8) u64 full[ST];
  __shared__ unsigned char flags[kMultiT];
  const u32 N = 1u << logN, r = blockIdx.y, k0 = blockIdx.x * kMacTile, tid = threadIdx.x;
  const u64 q = mc[r].q, ninv = mc[r].ninv, one_sh = mc[r].one_sh;
  const unsigned hb = r > 0 ? packed_hb(r, M.wide) : 2u;
  if (tid < (u32)nt) {
    u32 fl = 0;
    for (int g = 0; g < ng; ++g)
      if (M.mask[g][tid]) fl |= (1u << g) | ((M.packed[g][tid] && r > 0) ? (16u << g) : 0u);
    flags[tid] = (unsigned char)fl;
  }
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < ST - 1 && s < nt; ++s) mac_stage_bulk(S[s], &full[s], M, s, flags[s], r, nq, N, k0);
  u64 h[kMultiG][2], l[kMultiG][2];
#pragma unroll
  for (int g = 0; g < kMultiG; ++g) h[g][0] = h[g][1] = l[g][0] = l[g][1] = 0;
  for (int t = 0; t < nt; ++t) {
    if (t > 0) __syncthreads();  // every thread is done with slot (t-1) % ST
    if (tid == 0) {
      const int tn = t + ST - 1;
      if (tn < nt) mac_stage_bulk(S[tn % ST], &full[tn % ST], M, tn, flags[tn], r, nq, N, k0);
    }
    const u32 fl = flags[t];
    mbar_wait(&full[t % ST], (u32)(t / ST) & 1u);
    const MacStage& C = S[t % ST];
    const u64 x0 = C.ct[0][tid], x1 = C.ct[1][tid];
#pragma unroll
    for (int g = 0; g < kMultiG; ++g) {
      if (!(fl >> g & 1u)) continue;
      u64 m;
      if (fl >> (4 + g) & 1u) {
        const unsigned* lo = reinterpret_cast<const unsigned*>(C.mask[g]);
        m = (u64)lo[tid] | (packed_hi(reinterpret_cast<const unsigned char*>(C.mask[g]) + kMacTile * 4, tid, hb) << 32);
      } else {
        m = C.mask[g][tid];
      }
      mac128_lazy(h[g][0], l[g][0], x0, m);
      mac128_lazy(h[g][1], l[g][1], x1, m);
    }
    if ((t + 1) % kLazyTerms == 0 || t + 1 == nt) {
#pragma unroll
      for (int g = 0; g < kMultiG; ++g) {
        h[g][0] = fold_hi(h[g][0], q, one_sh);
        h[g][1] = fold_hi(h[g][1], q, one_sh);
      }
    }
  }
  const size_t pst = (size_t)nq * N, off = (size_t)r * N + k0 + tid;
#pragma unroll
  for (int g = 0; g < kMultiG; ++g) {
    if (g >= ng) break;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      u64* d = M.out[g] + p * pst + off;
      u64 y = redc128(h[g][p], l[g][p], q, ninv);
      if (accumulate) y = add_mod(y, *d, q);
      *d = y;
    }
  }
}

// k_mac_multi_tma with TPB threads per CTA, kMacTile / TPB coefficients per thread (TPB = 128:
// two independent coefficient chains per thread, a cheaper CTA barrier and
// more resident CTAs per SM for the same ring).  MINB = 1 leaves the
// minimum-blocks hint at 0: ptxas then settles at 96 registers (5 CTAs of
// 128 per SM) where an explicit 1 lets it take 166 (measured 25 % slower).
template <int ST, int TPB, int MINB = 1>
__global__ void __launch_bounds__(TPB, MINB > 1 ? MINB : 0) k_mac_multi_tma2(MacMulti M, int ng, int nt, u32 nq, u32 logN,
                                                       int accumulate, const ModConsts* __restrict__ mc) {
  constexpr int CPT = kMacTile / TPB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MacStage* S = reinterpret_cast<MacStage*>(smem_raw);
  __shared__ __align__(8) u64 full[ST];
  __shared__ unsigned char flags[kMultiT];
  const u32 N = 1u << logN, r = blockIdx.y, k0 = blockIdx.x * kMacTile, tid = threadIdx.x;
  const u64 q = mc[r].q, ninv = mc[r].ninv, one_sh = mc[r].one_sh;
  const unsigned hb = r > 0 ? packed_hb(r, M.wide) : 2u;
  for (u32 i = tid; i < (u32)nt; i += TPB) {
    u32 fl = 0;
    for (int g = 0; g < ng; ++g)
      if (M.mask[g][i]) fl |= (1u << g) | ((M.packed[g][i] && r > 0) ? (16u << g) : 0u);
    flags[i] = (unsigned char)fl;
  }
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < ST - 1 && s < nt; ++s) mac_stage_bulk(S[s], &full[s], M, s, flags[s], r, nq, N, k0);
  u64 h[kMultiG][2 * CPT], l[kMultiG][2 * CPT];
#pragma unroll
  for (int g = 0; g < kMultiG; ++g)
#pragma unroll
    for (int p = 0; p < 2 * CPT; ++p) h[g][p] = l[g][p] = 0;
  for (int t = 0; t < nt; ++t) {
    if (t > 0) __syncthreads();  // every thread is done with slot (t-1) % ST
    if (tid == 0) {
      const int tn = t + ST - 1;
      if (tn < nt) mac_stage_bulk(S[tn % ST], &full[tn % ST], M, tn, flags[tn], r, nq, N, k0);
    }
    const u32 fl = flags[t];
    mbar_wait(&full[t % ST], (u32)(t / ST) & 1u);
    const MacStage& C = S[t % ST];
    u64 x[2 * CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      x[2 * c] = C.ct[0][tid + c * TPB];
      x[2 * c + 1] = C.ct[1][tid + c * TPB];
    }
#pragma unroll
    for (int g = 0; g < kMultiG; ++g) {
      if (!(fl >> g & 1u)) continue;
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const u32 i = tid + c * TPB;
        u64 m;
        if (fl >> (4 + g) & 1u) {
          const unsigned* lo = reinterpret_cast<const unsigned*>(C.mask[g]);
          m = (u64)lo[i] | (packed_hi(reinterpret_cast<const unsigned char*>(C.mask[g]) + kMacTile * 4, i, hb) << 32);
        } else {
          m = C.mask[g][i];
        }
        mac128_lazy(h[g][2 * c], l[g][2 * c], x[2 * c], m);
        mac128_lazy(h[g][2 * c + 1], l[g][2 * c + 1], x[2 * c + 1], m);
      }
    }
    if ((t + 1) % kLazyTerms == 0 || t + 1 == nt) {
#pragma unroll
      for (int g = 0; g < kMultiG; ++g)
#pragma unroll
        for (int p = 0; p < 2 * CPT; ++p) h[g][p] = fold_hi(h[g][p], q, one_sh);
    }
  }
  const size_t pst = (size_t)nq * N;
#pragma unroll
  for (int g = 0; g < kMultiG; ++g) {
    if (g >= ng) break;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const size_t off = (size_t)r * N + k0 + tid + c * TPB;
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        u64* d = M.out[g] + p * pst + off;
        u64 y = redc128(h[g][2 * c + p], l[g][2 * c + p], q, ninv);
        if (accumulate) y = add_mod(y, *d, q);
        *d = y;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k_mac_multi_tma3: the plane MAC with a full / empty mbarrier ring (no
// CTA-wide barrier per term: warps run up to ST terms apart, the producer
// thread refills a slot once every warp has arrived on its "empty"
// barrier) and, for limbs with q < 2^42 (FAST: the 40-bit application
// primes), a 96-bit carry-chain accumulator fed by 32-bit halves:
//   a m = a0 m0 + (a0 m1 + a1 m0) 2^32 + a1 m1 2^64   (a1, m1 < 2^10)
// into T = (hi:lo) + mid 2^32 -- 5 IMADs per product instead of the 128-bit
// product's ~11, no lazy folds (T < 2^90 < q 2^64 for <= 48 terms), one
// REDC at the end: the same canonical sum * R^-1 mod q as mac128.
// ---------------------------------------------------------------------------
template <int ST, int TPB, bool FAST>
__global__ void __launch_bounds__(TPB + 32) k_mac_multi_tma3(MacMulti M, int ng, int nt, u32 nq, u32 logN, u32 r0,
                                                             int accumulate, const ModConsts* __restrict__ mc) {
  // TPB consumer threads + one producer warp (warp TPB/32) that only issues the bulk copies
  constexpr int CPT = kMacTile / TPB, NW = TPB / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MacStage* S = reinterpret_cast<MacStage*>(smem_raw);
  __shared__ __align__(8) u64 full[ST];
  __shared__ __align__(8) u64 empty[ST];
  __shared__ unsigned char flags[kMultiT];
  const u32 N = 1u << logN, r = blockIdx.y + r0, k0 = blockIdx.x * kMacTile, tid = threadIdx.x;
  const u64 q = mc[r].q, ninv = mc[r].ninv, one_sh = mc[r].one_sh;
  const unsigned hb = r > 0 ? packed_hb(r, M.wide) : 2u;
  for (u32 i = tid; i < (u32)nt; i += TPB + 32) {
    u32 fl = 0;
    for (int g = 0; g < ng; ++g)
      if (M.mask[g][i]) fl |= (1u << g) | ((M.packed[g][i] && r > 0) ? (16u << g) : 0u);
    flags[i] = (unsigned char)fl;
  }
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid >= (u32)TPB) {  // producer warp
    if (tid == (u32)TPB) {
      for (int t = 0; t < nt; ++t) {
        const int slot = t % ST;
        if (t >= ST) mbar_wait(&empty[slot], (u32)(t / ST - 1) & 1u);  // consumers released term t - ST
        mac_stage_bulk(S[slot], &full[slot], M, t, flags[t], r, nq, N, k0);
      }
    }
    return;
  }
  // per output poly-coefficient: FAST (lh, mid) of the 96-bit sum; generic
  // the lazy 128-bit (l, h)
  u64 AL[kMultiG][2 * CPT], AH[kMultiG][2 * CPT];
#pragma unroll
  for (int g = 0; g < kMultiG; ++g)
#pragma unroll
    for (int p = 0; p < 2 * CPT; ++p) AL[g][p] = AH[g][p] = 0;
  for (int t = 0; t < nt; ++t) {
    const int slot = t % ST;
    const u32 fl = flags[t];
    mbar_wait(&full[slot], (u32)(t / ST) & 1u);
    const MacStage& C = S[slot];
    u64 x[2 * CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      x[2 * c] = C.ct[0][tid + c * TPB];
      x[2 * c + 1] = C.ct[1][tid + c * TPB];
    }
#pragma unroll
    for (int g = 0; g < kMultiG; ++g) {
      if (!(fl >> g & 1u)) continue;
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const u32 i = tid + c * TPB;
        u32 m0, m1;
        if (fl >> (4 + g) & 1u) {
          m0 = reinterpret_cast<const unsigned*>(C.mask[g])[i];
          m1 = (u32)packed_hi(reinterpret_cast<const unsigned char*>(C.mask[g]) + kMacTile * 4, i, hb);
        } else {
          const u64 m = C.mask[g][i];
          m0 = (u32)m;
          m1 = (u32)(m >> 32);
        }
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const u64 a = x[2 * c + p];
          if constexpr (FAST) mac96(AL[g][2 * c + p], AH[g][2 * c + p], (u32)a, (u32)(a >> 32), m0, m1);
          else mac128_lazy(AH[g][2 * c + p], AL[g][2 * c + p], a, ((u64)m1 << 32) | m0);
        }
      }
    }
    if constexpr (!FAST) {
      if ((t + 1) % kLazyTerms == 0 || t + 1 == nt) {
#pragma unroll
        for (int g = 0; g < kMultiG; ++g)
#pragma unroll
          for (int p = 0; p < 2 * CPT; ++p) AH[g][p] = fold_hi(AH[g][p], q, one_sh);
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[slot]);
  }
  const size_t pst = (size_t)nq * N;
#pragma unroll
  for (int g = 0; g < kMultiG; ++g) {
    if (g >= ng) break;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const size_t off = (size_t)r * N + k0 + tid + c * TPB;
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        u64* d = M.out[g] + p * pst + off;
        const int k = 2 * c + p;
        u64 y = FAST ? redc96(AL[g][k], AH[g][k], q, ninv) : redc128(AH[g][k], AL[g][k], q, ninv);
        if (accumulate) y = add_mod(y, *d, q);
        *d = y;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k_mac_multi_img2: k_mac_multi_tma3 over two images that share every mask
// (image-batched execution, graph.stack_images): per term the producer warp
// bulk-copies both images' ciphertext tiles and each output's mask tile
// ONCE; 256 consumer threads (one coefficient each) accumulate the two
// images' sums with 96-bit carry chains.  Rows with q < 2^42 only (the
// generic limb-0 rows run as two single-image launches).
// ---------------------------------------------------------------------------
struct MacStage2 {
  u64 ct[2][2][kMacTile];        // [image][poly][coefficient]
  u64 mask[kMultiG][kMacTile];
};

__device__ __forceinline__ void mac_stage_bulk2(MacStage2& S, u64* bar, const MacMulti& M, int t, u32 fl, u32 r,
                                                u32 nq, u32 N, u32 k0) {
  const size_t off = (size_t)r * N + k0, pst = (size_t)nq * N;
  u32 bytes = 4 * kMacTile * 8;
  const u32 pk = kMacTile * (4 + packed_hb(r, M.wide));
  for (int g = 0; g < kMultiG; ++g)
    if (fl >> g & 1u) bytes += (fl >> (4 + g) & 1u) ? pk : kMacTile * 8;
  mbar_expect_tx(bar, bytes);
  for (int b = 0; b < 2; ++b) {
    const u64* c = M.ct[t] + (size_t)b * M.img_stride;
    bulk_g2s(S.ct[b][0], c + off, kMacTile * 8, bar);
    bulk_g2s(S.ct[b][1], c + pst + off, kMacTile * 8, bar);
  }
  for (int g = 0; g < kMultiG; ++g) {
    if (!(fl >> g & 1u)) continue;
    const u64* mp = M.mask[g][t];
    if (fl >> (4 + g) & 1u) {
      const char* bb = reinterpret_cast<const char*>(mp);
      char* dst = reinterpret_cast<char*>(S.mask[g]);
      const unsigned hb = packed_hb(r, M.wide);
      bulk_g2s(dst, bb + 8 * (size_t)N + 4 * ((size_t)(r - 1) * N + k0), kMacTile * 4, bar);
      bulk_g2s(dst + kMacTile * 4, bb + packed_hi_off(r, nq, N, M.wide) + (size_t)hb * k0, kMacTile * hb, bar);
    } else {
      bulk_g2s(S.mask[g], M.packed[g][t] ? mp + k0 : mp + off, kMacTile * 8, bar);
    }
  }
}

template <int ST>
__global__ void __launch_bounds__(kMacTile + 32, 2) k_mac_multi_img2(MacMulti M, int ng, int nt, u32 nq, u32 logN,
                                                                  u32 r0, int accumulate,
                                                                  const ModConsts* __restrict__ mc) {
  constexpr int NW = kMacTile / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MacStage2* S = reinterpret_cast<MacStage2*>(smem_raw);
  __shared__ __align__(8) u64 full[ST];
  __shared__ __align__(8) u64 empty[ST];
  __shared__ unsigned char flags[kMultiT];
  const u32 N = 1u << logN, r = blockIdx.y + r0, k0 = blockIdx.x * kMacTile, tid = threadIdx.x;
  const u64 q = mc[r].q, ninv = mc[r].ninv;
  const unsigned hb = packed_hb(r, M.wide);
  for (u32 i = tid; i < (u32)nt; i += kMacTile + 32) {
    u32 fl = 0;
    for (int g = 0; g < ng; ++g)
      if (M.mask[g][i]) fl |= (1u << g) | (M.packed[g][i] ? (16u << g) : 0u);
    flags[i] = (unsigned char)fl;
  }
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid >= (u32)kMacTile) {  // producer warp
    if (tid == (u32)kMacTile) {
      for (int t = 0; t < nt; ++t) {
        const int slot = t % ST;
        if (t >= ST) mbar_wait(&empty[slot], (u32)(t / ST - 1) & 1u);
        mac_stage_bulk2(S[slot], &full[slot], M, t, flags[t], r, nq, N, k0);
      }
    }
    return;
  }
  u64 AL[kMultiG][2][2], AH[kMultiG][2][2];  // [output][image][poly]
#pragma unroll
  for (int g = 0; g < kMultiG; ++g)
#pragma unroll
    for (int b = 0; b < 2; ++b) AL[g][b][0] = AL[g][b][1] = AH[g][b][0] = AH[g][b][1] = 0;
  for (int t = 0; t < nt; ++t) {
    const int slot = t % ST;
    const u32 fl = flags[t];
    mbar_wait(&full[slot], (u32)(t / ST) & 1u);
    const MacStage2& C = S[slot];
    u64 x[2][2];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      x[b][0] = C.ct[b][0][tid];
      x[b][1] = C.ct[b][1][tid];
    }
#pragma unroll
    for (int g = 0; g < kMultiG; ++g) {
      if (!(fl >> g & 1u)) continue;
      u32 m0, m1;
      if (fl >> (4 + g) & 1u) {
        m0 = reinterpret_cast<const unsigned*>(C.mask[g])[tid];
        m1 = (u32)packed_hi(reinterpret_cast<const unsigned char*>(C.mask[g]) + kMacTile * 4, tid, hb);
      } else {
        const u64 m = C.mask[g][tid];
        m0 = (u32)m;
        m1 = (u32)(m >> 32);
      }
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int p = 0; p < 2; ++p) mac96(AL[g][b][p], AH[g][b][p], (u32)x[b][p], (u32)(x[b][p] >> 32), m0, m1);
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[slot]);
  }
  const size_t pst = (size_t)nq * N, off = (size_t)r * N + k0 + tid;
#pragma unroll
  for (int g = 0; g < kMultiG; ++g) {
    if (g >= ng) break;
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        u64* d = M.out[g] + (size_t)b * M.img_stride + p * pst + off;
        u64 y = redc96(AL[g][b][p], AH[g][b][p], q, ninv);
        if (accumulate) y = add_mod(y, *d, q);
        *d = y;
      }
  }
}

// ---------------------------------------------------------------------------
// Key-switch inner product with TMA-staged operands.  A CTA owns one
// 256-coefficient tile of one output limb r for up to kKsEntries batch
// entries; per digit j one elected thread bulk-copies the two key rows'
// tiles (2 x 2 KB) and every entry's raised-digit tile (2 KB each) into a
// ring of ST stages tracked by mbarriers, so each key tile leaves
// HBM once per kKsEntries entries and no thread spends instructions on
// address generation.  The Galois permutation maps an aligned 256-block of
// outputs onto one aligned 256-block of sources (the low log2(N)-8 bits of
// the natural index fix the block), so the source tile is fetched whole and
// permuted on the shared-memory read.  Extended-basis outputs (c0 != null)
// take one more stage: P * sigma_g(c0) on the Q limbs.  Lazy 128-bit sums,
// one REDC: bit-identical with k_ks_inner.
// ---------------------------------------------------------------------------
constexpr int kKsEntries = 4;
struct KsStage {
  u64 kb[kMacTile];
  u64 ka[kMacTile];
  u64 x[kKsEntries][kMacTile];
};
int g_ks_tma = 1;
int g_ks_tma_min = 2;  // smallest batch routed to the TMA inner product (measured: 2 beats 1 and 3 with k_ks_inner_tma2)
int g_ks_tpb = 128;    // threads per key-switch inner-product CTA: 128 (k_ks_inner_tma2, two coefficients per thread) or 256
int g_ks_stages = 3;   // ring depth of k_ks_inner_tma2 (3 or 4)

template <int ST>
__global__ void __launch_bounds__(256) k_ks_inner_tma(u64* __restrict__ acc, const u64* __restrict__ x_eval,
                                                      const u64* __restrict__ raised, const u64* __restrict__ key_b,
                                                      const u64* __restrict__ key_a, Basis basis, u32 alpha,
                                                      u32 ndig, u32 logN, u64 g, const ModConsts* __restrict__ mc,
                                                      u32 nb, size_t x_bst, const u64* __restrict__ c0,
                                                      size_t c0_bst, const u64* __restrict__ pR, u32 key_lq) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  KsStage* S = reinterpret_cast<KsStage*>(smem_raw);
  __shared__ __align__(8) u64 full[ST];
  const u32 N = 1u << logN, r = blockIdx.y, tile = blockIdx.x, tid = threadIdx.x;
  const u32 b0 = blockIdx.z * kKsEntries;
  const u32 ne = nb - b0 < (u32)kKsEntries ? nb - b0 : (u32)kKsEntries;
  const u32 n_ext = basis.nlimbs();
  const u32 mod = basis.mod_of(r);
  const u64 q = mc[mod].q, ninv = mc[mod].ninv, one_sh = mc[mod].one_sh;
  const u32 klq = key_lq ? key_lq : basis.Lq;
  const size_t key_dst = (size_t)(klq + basis.np) * N;
  const u32 kmod = mod < basis.Lq ? mod : klq + (mod - basis.Lq);
  const u32 own = r < basis.nq ? r / alpha : 0xffffffffu;
  const u32 k = tile * kMacTile + tid;
  const u32 src = g == 1 ? k : galois_src(k, g, logN);
  const u32 s_in = src & (kMacTile - 1);                      // position inside the source tile
  const size_t t_src = (size_t)(src & ~(u32)(kMacTile - 1));  // same block for the whole CTA
  const size_t r_bst = (size_t)ndig * n_ext * N;
  const bool ext = c0 != nullptr && r < basis.nq;
  const u32 nst = ndig + (ext ? 1u : 0u);
  auto issue = [&](u32 j) {
    KsStage& T = S[j % ST];
    u64* bar = &full[j % ST];
    if (j < ndig) {
      mbar_expect_tx(bar, (2 + ne) * kMacTile * 8);
      const size_t kofs = (size_t)j * key_dst + (size_t)kmod * N + (size_t)tile * kMacTile;
      bulk_g2s(T.kb, key_b + kofs, kMacTile * 8, bar);
      bulk_g2s(T.ka, key_a + kofs, kMacTile * 8, bar);
      for (u32 e = 0; e < ne; ++e) {
        const u64* sp = j == own ? x_eval + (size_t)(b0 + e) * x_bst + (size_t)r * N
                                 : raised + (size_t)(b0 + e) * r_bst + ((size_t)j * n_ext + r) * N;
        bulk_g2s(T.x[e], sp + t_src, kMacTile * 8, bar);
      }
    } else {  // extended-basis term: c0 tiles
      mbar_expect_tx(bar, ne * kMacTile * 8);
      for (u32 e = 0; e < ne; ++e)
        bulk_g2s(T.x[e], c0 + (size_t)(b0 + e) * c0_bst + (size_t)r * N + t_src, kMacTile * 8, bar);
    }
  };
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (u32 j = 0; j < (u32)ST - 1 && j < nst; ++j) issue(j);
  u64 bh[kKsEntries], bl[kKsEntries], ah[kKsEntries], al[kKsEntries];
#pragma unroll
  for (int e = 0; e < kKsEntries; ++e) bh[e] = bl[e] = ah[e] = al[e] = 0;
  for (u32 j = 0; j < nst; ++j) {
    if (j > 0) __syncthreads();  // slot (j-1) % ST is free
    if (tid == 0 && j + ST - 1 < nst) issue(j + ST - 1);
    mbar_wait(&full[j % ST], (j / ST) & 1u);
    const KsStage& T = S[j % ST];
    if (j < ndig) {
      const u64 kb = T.kb[tid], ka = T.ka[tid];
#pragma unroll
      for (int e = 0; e < kKsEntries; ++e) {
        if ((u32)e >= ne) break;
        const u64 x = T.x[e][s_in];
        mac128_lazy(bh[e], bl[e], x, kb);
        mac128_lazy(ah[e], al[e], x, ka);
      }
    } else {
      const u64 w = pR[r];
#pragma unroll
      for (int e = 0; e < kKsEntries; ++e) {
        if ((u32)e >= ne) break;
        mac128_lazy(bh[e], bl[e], T.x[e][s_in], w);
      }
    }
    if ((j + 1) % kLazyTerms == 0 || j + 1 == nst) {
#pragma unroll
      for (int e = 0; e < kKsEntries; ++e) {
        bh[e] = fold_hi(bh[e], q, one_sh);
        ah[e] = fold_hi(ah[e], q, one_sh);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < kKsEntries; ++e) {
    if ((u32)e >= ne) break;
    u64* A = acc + (size_t)(b0 + e) * 2 * n_ext * N;
    A[(size_t)r * N + k] = redc128(bh[e], bl[e], q, ninv);
    A[((size_t)n_ext + r) * N + k] = redc128(ah[e], al[e], q, ninv);
  }
}

// k_ks_inner_tma with TPB threads per CTA and kMacTile / TPB output
// coefficients per thread (independent MAC chains per thread).  The body
// serves one rotation's output tile `tile` of limb row blockIdx.y.
template <int ST, int TPB>
__device__ __forceinline__ void ks_inner_tma2_body(u64* __restrict__ acc, const u64* __restrict__ x_eval,
                                                   const u64* __restrict__ raised, const u64* __restrict__ key_b,
                                                   const u64* __restrict__ key_a, const Basis& basis, u32 alpha,
                                                   u32 ndig, u32 logN, u64 g, const ModConsts* __restrict__ mc,
                                                   u32 nb, size_t x_bst, const u64* __restrict__ c0,
                                                   size_t c0_bst, const u64* __restrict__ pR, u32 key_lq,
                                                   u32 tile) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  KsStage* S = reinterpret_cast<KsStage*>(smem_raw);
  __shared__ __align__(8) u64 full[ST];
  const u32 N = 1u << logN, r = blockIdx.y, tid = threadIdx.x;
  const u32 b0 = blockIdx.z * kKsEntries;
  const u32 ne = nb - b0 < (u32)kKsEntries ? nb - b0 : (u32)kKsEntries;
  const u32 n_ext = basis.nlimbs();
  const u32 mod = basis.mod_of(r);
  const u64 q = mc[mod].q, ninv = mc[mod].ninv, one_sh = mc[mod].one_sh;
  // rows whose modulus is below 2^42 (the 40-bit primes): residues and key
  // words fit 42 bits, so each product accumulates through a 96-bit carry
  // chain (5 IMADs instead of ~11, no lazy folds; T < 2^90) -- CTA-uniform
  const bool f96 = g_ks96_dev && q < (1ull << 42);
  const u32 klq = key_lq ? key_lq : basis.Lq;
  const size_t key_dst = (size_t)(klq + basis.np) * N;
  const u32 kmod = mod < basis.Lq ? mod : klq + (mod - basis.Lq);
  const u32 own = r < basis.nq ? r / alpha : 0xffffffffu;
  constexpr int CPT = kMacTile / TPB;
  const u32 k = tile * kMacTile + tid;
  const u32 src = g == 1 ? k : galois_src(k, g, logN);
  u32 s_in[CPT];  // positions inside the source tile
  s_in[0] = src & (kMacTile - 1);
#pragma unroll
  for (int c = 1; c < CPT; ++c) s_in[c] = (g == 1 ? k + c * TPB : galois_src(k + c * TPB, g, logN)) & (kMacTile - 1);
  const size_t t_src = (size_t)(src & ~(u32)(kMacTile - 1));  // same block for the whole CTA
  const size_t r_bst = (size_t)ndig * n_ext * N;
  const bool ext = c0 != nullptr && r < basis.nq;
  const u32 nst = ndig + (ext ? 1u : 0u);
  auto issue = [&](u32 j) {
    KsStage& T = S[j % ST];
    u64* bar = &full[j % ST];
    if (j < ndig) {
      mbar_expect_tx(bar, (2 + ne) * kMacTile * 8);
      const size_t kofs = (size_t)j * key_dst + (size_t)kmod * N + (size_t)tile * kMacTile;
      bulk_g2s(T.kb, key_b + kofs, kMacTile * 8, bar);
      bulk_g2s(T.ka, key_a + kofs, kMacTile * 8, bar);
      for (u32 e = 0; e < ne; ++e) {
        const u64* sp = j == own ? x_eval + (size_t)(b0 + e) * x_bst + (size_t)r * N
                                 : raised + (size_t)(b0 + e) * r_bst + ((size_t)j * n_ext + r) * N;
        bulk_g2s(T.x[e], sp + t_src, kMacTile * 8, bar);
      }
    } else {  // extended-basis term: c0 tiles
      mbar_expect_tx(bar, ne * kMacTile * 8);
      for (u32 e = 0; e < ne; ++e)
        bulk_g2s(T.x[e], c0 + (size_t)(b0 + e) * c0_bst + (size_t)r * N + t_src, kMacTile * 8, bar);
    }
  };
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (u32 j = 0; j < (u32)ST - 1 && j < nst; ++j) issue(j);
  u64 bh[kKsEntries][CPT], bl[kKsEntries][CPT], ah[kKsEntries][CPT], al[kKsEntries][CPT];
#pragma unroll
  for (int e = 0; e < kKsEntries; ++e)
#pragma unroll
    for (int c = 0; c < CPT; ++c) bh[e][c] = bl[e][c] = ah[e][c] = al[e][c] = 0;
  for (u32 j = 0; j < nst; ++j) {
    if (j > 0) __syncthreads();  // slot (j-1) % ST is free
    if (tid == 0 && j + ST - 1 < nst) issue(j + ST - 1);
    mbar_wait(&full[j % ST], (j / ST) & 1u);
    const KsStage& T = S[j % ST];
    if (j < ndig) {
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const u64 kb = T.kb[tid + c * TPB], ka = T.ka[tid + c * TPB];
#pragma unroll
        for (int e = 0; e < kKsEntries; ++e) {
          if ((u32)e >= ne) break;
          const u64 x = T.x[e][s_in[c]];
          if (f96) {
            mac96(bh[e][c], bl[e][c], (u32)x, (u32)(x >> 32), (u32)kb, (u32)(kb >> 32));
            mac96(ah[e][c], al[e][c], (u32)x, (u32)(x >> 32), (u32)ka, (u32)(ka >> 32));
          } else {
            mac128_lazy(bh[e][c], bl[e][c], x, kb);
            mac128_lazy(ah[e][c], al[e][c], x, ka);
          }
        }
      }
    } else {
      const u64 w = pR[r];
#pragma unroll
      for (int c = 0; c < CPT; ++c)
#pragma unroll
        for (int e = 0; e < kKsEntries; ++e) {
          if ((u32)e >= ne) break;
          const u64 x = T.x[e][s_in[c]];
          if (f96) mac96(bh[e][c], bl[e][c], (u32)x, (u32)(x >> 32), (u32)w, (u32)(w >> 32));
          else mac128_lazy(bh[e][c], bl[e][c], x, w);
        }
    }
    if (!f96 && ((j + 1) % kLazyTerms == 0 || j + 1 == nst)) {
#pragma unroll
      for (int e = 0; e < kKsEntries; ++e)
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          bh[e][c] = fold_hi(bh[e][c], q, one_sh);
          ah[e][c] = fold_hi(ah[e][c], q, one_sh);
        }
    }
  }
#pragma unroll
  for (int e = 0; e < kKsEntries; ++e) {
    if ((u32)e >= ne) break;
    u64* A = acc + (size_t)(b0 + e) * 2 * n_ext * N;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const u32 kc = k + c * TPB;
      A[(size_t)r * N + kc] = f96 ? redc96(bh[e][c], bl[e][c], q, ninv) : redc128(bh[e][c], bl[e][c], q, ninv);
      A[((size_t)n_ext + r) * N + kc] = f96 ? redc96(ah[e][c], al[e][c], q, ninv) : redc128(ah[e][c], al[e][c], q, ninv);
    }
  }
}

template <int ST, int TPB>
__global__ void __launch_bounds__(TPB) k_ks_inner_tma2(u64* __restrict__ acc, const u64* __restrict__ x_eval,
                                                      const u64* __restrict__ raised, const u64* __restrict__ key_b,
                                                      const u64* __restrict__ key_a, Basis basis, u32 alpha,
                                                      u32 ndig, u32 logN, u64 g, const ModConsts* __restrict__ mc,
                                                      u32 nb, size_t x_bst, const u64* __restrict__ c0,
                                                      size_t c0_bst, const u64* __restrict__ pR, u32 key_lq) {
  ks_inner_tma2_body<ST, TPB>(acc, x_eval, raised, key_b, key_a, basis, alpha, ndig, logN, g, mc, nb, x_bst, c0,
                              c0_bst, pR, key_lq, blockIdx.x);
}

// Every rotation of a hoisted group in one launch: blockIdx.x = tile * n +
// rotation, so the CTAs resident at any time cover a few limb rows for all
// rotations and the raised digits of those rows (shared by every rotation,
// each read through its own Galois block remap) come from L2 after the
// first rotation touches them -- one HBM pass over the raised digits per
// group instead of one per rotation.  Same arithmetic per output as
// k_ks_inner_tma2 (bit-identical).
template <int ST, int TPB>
__global__ void __launch_bounds__(TPB) k_ks_inner_tma2_rots(const __grid_constant__ KsRots R, u32 nrot,
                                                           const u64* __restrict__ x_eval,
                                                           const u64* __restrict__ raised, Basis basis, u32 alpha,
                                                           u32 ndig, u32 logN, const ModConsts* __restrict__ mc,
                                                           u32 nb, size_t x_bst, const u64* __restrict__ c0,
                                                           size_t c0_bst, const u64* __restrict__ pR) {
  const u32 rot = blockIdx.x % nrot, tile = blockIdx.x / nrot;
  ks_inner_tma2_body<ST, TPB>(R.acc[rot], x_eval, raised, R.kb[rot], R.ka[rot], basis, alpha, ndig, logN, R.g[rot],
                              mc, nb, x_bst, c0, c0_bst, pR, R.klq[rot], tile);
}

// k_ks_inner_tma3: k_ks_inner_tma2 with a dedicated producer warp and a
// full / empty mbarrier ring (consumer warps run up to ST digits apart, no
// CTA-wide barrier per digit); FAST rows (Q limbs with q < 2^42) accumulate
// with the 96-bit carry chains of k_mac_multi_tma3.  Rows r0 .. r0+gridDim.y-1.
template <int ST, int TPB, bool FAST>
__global__ void __launch_bounds__(TPB + 32) k_ks_inner_tma3(u64* __restrict__ acc, const u64* __restrict__ x_eval,
                                                            const u64* __restrict__ raised, const u64* __restrict__ key_b,
                                                            const u64* __restrict__ key_a, Basis basis, u32 alpha,
                                                            u32 ndig, u32 logN, u64 g, const ModConsts* __restrict__ mc,
                                                            u32 nb, size_t x_bst, const u64* __restrict__ c0,
                                                            size_t c0_bst, const u64* __restrict__ pR, u32 key_lq,
                                                            u32 r0) {
  constexpr int NW = TPB / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  KsStage* S = reinterpret_cast<KsStage*>(smem_raw);
  __shared__ __align__(8) u64 full[ST];
  __shared__ __align__(8) u64 empty[ST];
  const u32 N = 1u << logN, r = blockIdx.y + r0, tile = blockIdx.x, tid = threadIdx.x;
  const u32 b0 = blockIdx.z * kKsEntries;
  const u32 ne = nb - b0 < (u32)kKsEntries ? nb - b0 : (u32)kKsEntries;
  const u32 n_ext = basis.nlimbs();
  const u32 mod = basis.mod_of(r);
  const u64 q = mc[mod].q, ninv = mc[mod].ninv, one_sh = mc[mod].one_sh;
  const u32 klq = key_lq ? key_lq : basis.Lq;
  const size_t key_dst = (size_t)(klq + basis.np) * N;
  const u32 kmod = mod < basis.Lq ? mod : klq + (mod - basis.Lq);
  const u32 own = r < basis.nq ? r / alpha : 0xffffffffu;
  constexpr int CPT = kMacTile / TPB;
  const u32 k = tile * kMacTile + (tid < (u32)TPB ? tid : 0);
  const u32 src = g == 1 ? k : galois_src(k, g, logN);
  const size_t t_src = (size_t)(src & ~(u32)(kMacTile - 1));  // same block for the whole CTA
  const size_t r_bst = (size_t)ndig * n_ext * N;
  const bool ext = c0 != nullptr && r < basis.nq;
  const u32 nst = ndig + (ext ? 1u : 0u);
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid >= (u32)TPB) {  // producer warp
    if (tid == (u32)TPB) {
      for (u32 j = 0; j < nst; ++j) {
        const u32 slot = j % ST;
        if (j >= (u32)ST) mbar_wait(&empty[slot], (j / ST - 1) & 1u);
        KsStage& T = S[slot];
        u64* bar = &full[slot];
        if (j < ndig) {
          mbar_expect_tx(bar, (2 + ne) * kMacTile * 8);
          const size_t kofs = (size_t)j * key_dst + (size_t)kmod * N + (size_t)tile * kMacTile;
          bulk_g2s(T.kb, key_b + kofs, kMacTile * 8, bar);
          bulk_g2s(T.ka, key_a + kofs, kMacTile * 8, bar);
          for (u32 e = 0; e < ne; ++e) {
            const u64* sp = j == own ? x_eval + (size_t)(b0 + e) * x_bst + (size_t)r * N
                                     : raised + (size_t)(b0 + e) * r_bst + ((size_t)j * n_ext + r) * N;
            bulk_g2s(T.x[e], sp + t_src, kMacTile * 8, bar);
          }
        } else {  // extended-basis term: c0 tiles
          mbar_expect_tx(bar, ne * kMacTile * 8);
          for (u32 e = 0; e < ne; ++e)
            bulk_g2s(T.x[e], c0 + (size_t)(b0 + e) * c0_bst + (size_t)r * N + t_src, kMacTile * 8, bar);
        }
      }
    }
    return;
  }
  u32 s_in[CPT];  // positions inside the source tile
  s_in[0] = src & (kMacTile - 1);
#pragma unroll
  for (int c = 1; c < CPT; ++c) s_in[c] = (g == 1 ? k + c * TPB : galois_src(k + c * TPB, g, logN)) & (kMacTile - 1);
  // FAST: (lh, mid) 96-bit sums; generic: lazy 128-bit (l, h)
  u64 bL[kKsEntries][CPT], bH[kKsEntries][CPT], aL[kKsEntries][CPT], aH[kKsEntries][CPT];
#pragma unroll
  for (int e = 0; e < kKsEntries; ++e)
#pragma unroll
    for (int c = 0; c < CPT; ++c) bL[e][c] = bH[e][c] = aL[e][c] = aH[e][c] = 0;
  for (u32 j = 0; j < nst; ++j) {
    const u32 slot = j % ST;
    mbar_wait(&full[slot], (j / ST) & 1u);
    const KsStage& T = S[slot];
    if (j < ndig) {
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const u64 kb = T.kb[tid + c * TPB], ka = T.ka[tid + c * TPB];
#pragma unroll
        for (int e = 0; e < kKsEntries; ++e) {
          if ((u32)e >= ne) break;
          const u64 x = T.x[e][s_in[c]];
          if constexpr (FAST) {
            mac96(bL[e][c], bH[e][c], (u32)x, (u32)(x >> 32), (u32)kb, (u32)(kb >> 32));
            mac96(aL[e][c], aH[e][c], (u32)x, (u32)(x >> 32), (u32)ka, (u32)(ka >> 32));
          } else {
            mac128_lazy(bH[e][c], bL[e][c], x, kb);
            mac128_lazy(aH[e][c], aL[e][c], x, ka);
          }
        }
      }
    } else {
      const u64 w = pR[r];
#pragma unroll
      for (int c = 0; c < CPT; ++c)
#pragma unroll
        for (int e = 0; e < kKsEntries; ++e) {
          if ((u32)e >= ne) break;
          const u64 x = T.x[e][s_in[c]];
          if constexpr (FAST) mac96(bL[e][c], bH[e][c], (u32)x, (u32)(x >> 32), (u32)w, (u32)(w >> 32));
          else mac128_lazy(bH[e][c], bL[e][c], x, w);
        }
    }
    if constexpr (!FAST) {
      if ((j + 1) % kLazyTerms == 0 || j + 1 == nst) {
#pragma unroll
        for (int e = 0; e < kKsEntries; ++e)
#pragma unroll
          for (int c = 0; c < CPT; ++c) {
            bH[e][c] = fold_hi(bH[e][c], q, one_sh);
            aH[e][c] = fold_hi(aH[e][c], q, one_sh);
          }
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[slot]);
  }
#pragma unroll
  for (int e = 0; e < kKsEntries; ++e) {
    if ((u32)e >= ne) break;
    u64* A = acc + (size_t)(b0 + e) * 2 * n_ext * N;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const u32 kc = k + c * TPB;
      A[(size_t)r * N + kc] = FAST ? redc96(bL[e][c], bH[e][c], q, ninv) : redc128(bH[e][c], bL[e][c], q, ninv);
      A[((size_t)n_ext + r) * N + kc] = FAST ? redc96(aL[e][c], aH[e][c], q, ninv) : redc128(aH[e][c], aL[e][c], q, ninv);
    }
  }
}

// 0: off -- measured slower than k_ks_inner_tma2 (tools/ks_bench.py: 3.7 vs 4.3 TB/s
// at level 14 nb 4, 4.0 vs 4.6 at level 30 nb 8; three row launches, 3 CTAs/SM)
int g_ks_tma3 = 0;     // 1: k_ks_inner_tma3 (warp-specialised, 96-bit rows split out), 2: one generic launch
int g_ks3_stages = 3;  // its ring depth (2, 3, 4)

int g_mac_tma = 3;    // 1: bulk-copy (TMA) staged k_mac_multi_tma(2), 3: warp-specialised k_mac_multi_tma3
int g_mac3_stages = 4;  // k_mac_multi_tma3 ring depth (2, 3, 4, 6); tools/mac_probe.py: 4 = 3 < 2, 6
int g_mac3_tpb = 128;   // k_mac_multi_tma3 threads per CTA (128 or 256)
int g_mac3_fork = 1;    // run the generic (limb 0) rows on a forked side stream
int g_mac_minb = 1;  // minimum resident CTAs per SM (register cap) of k_mac_multi_tma: 1, 4, 5, 6
int g_mac_tpb = 128;  // threads per plane-MAC CTA: 128 (k_mac_multi_tma2, two coefficients per thread) or 256
int g_tma_stages = 3;  // ring depth of the TMA-staged plane MAC (128 threads: 2, 3, 4; 256: 4, 6, 8; the 256-thread key-switch kernel takes max(4, this))
int g_mac_async = 1;  // 1: cp.async pipeline (k_mac_multi_async), 0: k_mac_multi_lanes

int g_mac_lanes = 1;  // 1: k_mac_multi_lanes, 0: register-blocked k_mac_multi

cudaError_t launch_mac_multi(const MacMulti& M, int ng, int nt, u32 nq, u32 logN, int accumulate,
                             const ModConsts* mc, cudaStream_t st) {
  if (ng < 1 || ng > kMultiG) return cudaErrorInvalidValue;
  if (M.nimg == 2) {
    // two images sharing the masks: FAST rows in one k_mac_multi_img2 launch,
    // the generic rows (limb 0) as one single-image launch per image
    if ((1u << logN) % kMacTile || nt > kMultiT) return cudaErrorInvalidValue;
    const u32 ff = M.fast_from < 1 ? 1 : (M.fast_from > nq ? nq : M.fast_from);
    for (int b = 0; b < 2; ++b) {
      MacMulti M1 = M;
      M1.nimg = 1;
      M1.fast_from = nq;  // every row generic in this helper call: only rows < ff are launched below
      for (int t = 0; t < nt; ++t) M1.ct[t] = M.ct[t] + (size_t)b * M.img_stride;
      for (int g = 0; g < kMultiG; ++g) M1.out[g] = M.out[g] ? M.out[g] + (size_t)b * M.img_stride : nullptr;
      const size_t sm = sizeof(MacStage) * 3;
      cudaError_t e = ensure_smem((const void*)k_mac_multi_tma3<3, 128, false>, sm);
      if (e) return e;
      k_mac_multi_tma3<3, 128, false><<<dim3((1u << logN) / kMacTile, ff, 1), 160, sm, st>>>(M1, ng, nt, nq, logN, 0,
                                                                                           accumulate, mc);
      e = cudaGetLastError();
      if (e) return e;
    }
    if (ff < nq) {
      constexpr int ST = 3;
      const size_t sm = sizeof(MacStage2) * ST;
      cudaError_t e = ensure_smem((const void*)k_mac_multi_img2<ST>, sm);
      if (e) return e;
      k_mac_multi_img2<ST><<<dim3((1u << logN) / kMacTile, nq - ff, 1), kMacTile + 32, sm, st>>>(
          M, ng, nt, nq, logN, ff, accumulate, mc);
      return cudaGetLastError();
    }
    return cudaSuccess;
  }
  if (g_mac_tma == 3 && (1u << logN) % kMacTile == 0 && nt <= kMultiT) {
    // rows [0, fast_from): generic 128-bit MACs; [fast_from, nq): 96-bit carry chains
    const int stages = g_mac3_stages, tpb = g_mac3_tpb;
    auto go3 = [&](auto kern, int fast, u32 r0, u32 rows, int kst, int ktpb, cudaStream_t ls) -> cudaError_t {
      (void)fast;
      if (rows == 0) return cudaSuccess;
      const size_t sm = sizeof(MacStage) * kst;
      cudaError_t e = ensure_smem((const void*)kern, sm);
      if (e) return e;
      kern<<<dim3((1u << logN) / kMacTile, rows, 1), ktpb + 32, sm, ls>>>(M, ng, nt, nq, logN, r0, accumulate, mc);
      return cudaGetLastError();
    };
    const u32 ff = M.fast_from < 1 ? 1 : (M.fast_from > nq ? nq : M.fast_from);
    // the generic rows (limb 0: 256 CTAs, latency-bound) run on a side
    // stream forked from st, concurrently with the FAST rows, and join back
    // before the call returns (also inside a CUDA-graph capture: a fork /
    // join branch of the captured graph)
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    std::mutex* fmu = nullptr;
    const bool par = g_mac3_fork && ff < nq && side_stream(&side, &fork, &join, &fmu) == cudaSuccess;
    std::unique_lock<std::mutex> flk;
    if (par) flk = std::unique_lock<std::mutex>(*fmu);
    cudaStream_t gst = st;
    if (par) {
      cudaError_t e = cudaEventRecord(fork, st);
      if (!e) e = cudaStreamWaitEvent(side, fork, 0);
      if (e) return e;
      gst = side;
    }
    {
      cudaError_t e = go3(k_mac_multi_tma3<3, 128, false>, 0, 0, ff, 3, 128, gst);
      if (e) return e;
    }
    cudaError_t e = cudaSuccess;
    bool done = false;
#define MAC3(ST, TPB) \
    if (!done && stages == ST && tpb == TPB) { e = go3(k_mac_multi_tma3<ST, TPB, true>, 1, ff, nq - ff, ST, TPB, st); done = true; }
    MAC3(2, 128) MAC3(4, 128) MAC3(6, 128) MAC3(2, 256) MAC3(3, 256) MAC3(4, 256) MAC3(6, 256)
#undef MAC3
    if (!done) e = go3(k_mac_multi_tma3<3, 128, true>, 1, ff, nq - ff, 3, 128, st);
    if (par) {
      cudaError_t e2 = cudaEventRecord(join, side);
      if (!e2) e2 = cudaStreamWaitEvent(st, join, 0);
      if (!e) e = e2;
    }
    return e;
  }
  if (g_mac_tma && (1u << logN) % kMacTile == 0 && nt <= kMultiT) {
    dim3 g((1u << logN) / kMacTile, nq, 1);
    auto go = [&](auto kern, int stages, int tpb) -> cudaError_t {
      const size_t sm = sizeof(MacStage) * stages;
      cudaError_t e = ensure_smem((const void*)kern, sm);
      if (e) return e;
      kern<<<g, tpb, sm, st>>>(M, ng, nt, nq, logN, accumulate, mc);
      return cudaGetLastError();
    };
    if (g_mac_tpb == 128) {
      if (g_tma_stages >= 4) return go(k_mac_multi_tma2<4, 128>, 4, 128);
      if (g_tma_stages == 2) return go(k_mac_multi_tma2<2, 128, 6>, 2, 128);
      switch (g_mac_minb) {
        case 4: return go(k_mac_multi_tma2<3, 128, 4>, 3, 128);
        case 5: return go(k_mac_multi_tma2<3, 128, 5>, 3, 128);
        case 6: return go(k_mac_multi_tma2<3, 128, 6>, 3, 128);
        default: return go(k_mac_multi_tma2<3, 128>, 3, 128);
      }
    }
    if (g_tma_stages >= 8) return go(k_mac_multi_tma<8>, 8, 256);
    if (g_tma_stages >= 6) return go(k_mac_multi_tma<6>, 6, 256);
    if (g_mac_minb == 4) return go(k_mac_multi_tma2<4, 256, 4>, 4, 256);
    return go(k_mac_multi_tma<4>, 4, 256);
  }
  if (g_mac_async && (1u << logN) % kMacTile == 0) {
    const size_t sm = sizeof(MacStage) * kMacStages;
    cudaError_t e = ensure_smem((const void*)k_mac_multi_async, sm);
    if (e) return e;
    dim3 g((1u << logN) / kMacTile, nq, 1);
    k_mac_multi_async<<<g, 256, sm, st>>>(M, ng, nt, nq, logN, accumulate, mc);
    return cudaGetLastError();
  }
  if (g_mac_lanes) {
    dim3 g((((1u << logN) / 2) + 63) / 64, nq, 1);
    k_mac_multi_lanes<<<g, 256, 0, st>>>(M, ng, nt, nq, logN, accumulate, mc);
    return cudaGetLastError();
  }
  dim3 g2 = row_grid((1u << logN) / 2, nq, 256), g1 = row_grid(1u << logN, nq, 256);
  switch (ng) {
    case 1: k_mac_multi<1, 2><<<g2, 256, 0, st>>>(M, nt, nq, logN, accumulate, mc); break;
    case 2: k_mac_multi<2, 2><<<g2, 256, 0, st>>>(M, nt, nq, logN, accumulate, mc); break;
    case 3: k_mac_multi<3, 1><<<g1, 256, 0, st>>>(M, nt, nq, logN, accumulate, mc); break;
    default: k_mac_multi<4, 1><<<g1, 256, 0, st>>>(M, nt, nq, logN, accumulate, mc); break;
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------

cudaError_t launch_ew_binary(int op, u64* out, const u64* a, const u64* b, Basis basis, u32 logN, u32 npolys,
                             int b_bcast, const ModConsts* mc, cudaStream_t st) {
  u32 rows = npolys * basis.nlimbs();
  if (!rows) return cudaSuccess;
  u32 N = 1u << logN;
  k_ew_binary<<<row_grid(N / 2, rows, 256), 256, 0, st>>>(op, out, a, b, basis, logN, b_bcast, mc);
  return cudaGetLastError();
}

cudaError_t launch_ew_unary(int op, u64* out, const u64* a, Basis basis, u32 logN, u32 npolys,
                            const ModConsts* mc, const u64* consts, const u64* consts_sh, cudaStream_t st) {
  u32 rows = npolys * basis.nlimbs();
  if (!rows) return cudaSuccess;
  u32 N = 1u << logN;
  k_ew_unary<<<row_grid(N / 2, rows, 256), 256, 0, st>>>(op, out, a, basis, logN, mc, consts, consts_sh);
  return cudaGetLastError();
}

cudaError_t launch_from_signed(u64* out, const long long* in, Basis basis, u32 logN, u32 npolys,
                               const ModConsts* mc, int mont, cudaStream_t st) {
  u32 rows = npolys * basis.nlimbs();
  if (!rows) return cudaSuccess;
  k_from_signed<<<row_grid(1u << logN, rows, 256), 256, 0, st>>>(out, in, basis, logN, mc, mont);
  return cudaGetLastError();
}

cudaError_t launch_automorph(int eval_domain, u64* out, const u64* in, Basis basis, u32 logN, u32 npolys, u64 g,
                             const ModConsts* mc, cudaStream_t st) {
  u32 rows = npolys * basis.nlimbs();
  if (!rows) return cudaSuccess;
  k_automorph<<<row_grid(1u << logN, rows, 256), 256, 0, st>>>(eval_domain, out, in, basis, logN, g, mc);
  return cudaGetLastError();
}

cudaError_t launch_tensor(u64* d0, u64* d1, u64* d2, const u64* a, const u64* b, u32 nlimbs, u32 logN,
                          const ModConsts* mc, cudaStream_t st) {
  k_tensor<<<row_grid(1u << logN, nlimbs, 256), 256, 0, st>>>(d0, d1, d2, a, b, nlimbs, logN, mc);
  return cudaGetLastError();
}

static size_t fbc_smem(u32 nt, int ns) {
  if (nt > kFbcTG) nt = kFbcTG;
  return (size_t)nt * (3 + ns + (1u << ns)) * 8;
}

// targets per CTA: all of them (up to kFbcTG) unless the conversion is too
// small to fill the GPU, then split so there are >= ~8 CTAs per SM
static u32 fbc_group(u32 nt, u32 base_ctas) {
  u32 tg = nt < (u32)kFbcTG ? nt : (u32)kFbcTG;
  const u32 want = 148u * 8u;
  if (base_ctas < want && tg > 1) {
    u32 split = (want + base_ctas - 1) / base_ctas;
    if (split > tg) split = tg;
    tg = (tg + split - 1) / split;
  }
  return tg ? tg : 1;
}

template <int NS>
static cudaError_t launch_fbc_t(const FbcDev* tabs, int tab_per_z, const ModConsts* mc, const u64* in,
                                size_t in_pst, u64* out, size_t out_pst, u32 logN, u32 nz, u32 z0, u32 nt,
                                u32 nt_override, u32 nb, size_t in_bst, size_t out_bst, cudaStream_t st) {
  dim3 g = row_grid((1u << logN) / 2, nz * nb, 256);  // two coefficients per thread
  const u32 tg = fbc_group(nt, g.x * g.y);
  size_t sm = fbc_smem(tg, NS);
  if (sm > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_fbc_t<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e) return e;
  }
  g.z = (nt + tg - 1) / tg;
  k_fbc_t<NS><<<g, 256, sm, st>>>(tabs, tab_per_z, mc, in, in_pst, out, out_pst, logN, nt_override, z0, nz, in_bst,
                                  out_bst, tg);
  return cudaGetLastError();
}

static cudaError_t dispatch_fbc_t(int ns, const FbcDev* tabs, int tab_per_z, const ModConsts* mc, const u64* in,
                                  size_t in_pst, u64* out, size_t out_pst, u32 logN, u32 nz, u32 z0, u32 nt,
                                  u32 nt_override, cudaStream_t st, u32 nb = 1, size_t in_bst = 0,
                                  size_t out_bst = 0) {
  switch (ns) {
    case 1: return launch_fbc_t<1>(tabs, tab_per_z, mc, in, in_pst, out, out_pst, logN, nz, z0, nt, nt_override, nb, in_bst, out_bst, st);
    case 2: return launch_fbc_t<2>(tabs, tab_per_z, mc, in, in_pst, out, out_pst, logN, nz, z0, nt, nt_override, nb, in_bst, out_bst, st);
    case 3: return launch_fbc_t<3>(tabs, tab_per_z, mc, in, in_pst, out, out_pst, logN, nz, z0, nt, nt_override, nb, in_bst, out_bst, st);
    case 4: return launch_fbc_t<4>(tabs, tab_per_z, mc, in, in_pst, out, out_pst, logN, nz, z0, nt, nt_override, nb, in_bst, out_bst, st);
    case 5: return launch_fbc_t<5>(tabs, tab_per_z, mc, in, in_pst, out, out_pst, logN, nz, z0, nt, nt_override, nb, in_bst, out_bst, st);
    case 6: return launch_fbc_t<6>(tabs, tab_per_z, mc, in, in_pst, out, out_pst, logN, nz, z0, nt, nt_override, nb, in_bst, out_bst, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_fbc(const FbcDev& T, const FbcDev* dT, const ModConsts* mc, const u64* in, size_t in_pst,
                       u64* out, size_t out_pst, u32 logN, u32 npolys, u32 nt, cudaStream_t st) {
  if (dT && T.corr && T.nored && T.ns <= 6)
    return dispatch_fbc_t(T.ns, dT, 0, mc, in, in_pst, out, out_pst, logN, npolys, 0, nt, nt, st);
  if (T.ns > FBC_MAX_SRC) return cudaErrorInvalidValue;
  k_fbc<<<row_grid(1u << logN, npolys, 128), 128, 0, st>>>(T, mc, in, in_pst, out, out_pst, logN, nt);
  return cudaGetLastError();
}

cudaError_t launch_modup(const FbcDev* tabs, const FbcDev* htabs, u32 ndig, const ModConsts* mc, const u64* xc,
                         u64* raised, u32 alpha, u32 n_ext, u32 logN, cudaStream_t st, u32 nb, size_t xc_bst) {
  if (alpha > FBC_MAX_SRC) return cudaErrorInvalidValue;
  bool fast = true;
  for (u32 j = 0; j < ndig; ++j) fast = fast && htabs[j].corr && htabs[j].nored && htabs[j].ns <= 6;
  const size_t r_bst = (size_t)ndig * n_ext * (1u << logN);
  if (!fast) {
    for (u32 b = 0; b < nb; ++b)
      k_modup<<<row_grid(1u << logN, ndig, 128), 128, 0, st>>>(tabs, mc, xc + b * xc_bst, raised + b * r_bst, alpha,
                                                                n_ext, logN);
    return cudaGetLastError();
  }
  // full digits share one launch; a partial last digit gets its own, on the
  // side stream next to it (independent outputs; joined before returning)
  u32 nfull = ndig;
  if (htabs[ndig - 1].ns != alpha) nfull = ndig - 1;
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  std::mutex* fmu = nullptr;
  const bool par = g_fbc_fork && nfull && nfull < ndig && side_stream(&side, &fork, &join, &fmu) == cudaSuccess;
  std::unique_lock<std::mutex> flk;
  cudaStream_t pst = st;
  if (par) {
    flk = std::unique_lock<std::mutex>(*fmu);
    cudaError_t e0 = cudaEventRecord(fork, st);
    if (!e0) e0 = cudaStreamWaitEvent(side, fork, 0);
    if (e0) return e0;
    pst = side;
  }
  cudaError_t e = cudaSuccess;
  if (nfull < ndig)
    e = dispatch_fbc_t((int)htabs[ndig - 1].ns, tabs, 1, mc, xc, (size_t)alpha * (1u << logN), raised,
                       (size_t)n_ext * (1u << logN), logN, 1, nfull, htabs[ndig - 1].nt, 0, pst, nb, xc_bst, r_bst);
  if (!e && nfull)
    e = dispatch_fbc_t((int)alpha, tabs, 1, mc, xc, (size_t)alpha * (1u << logN), raised,
                       (size_t)n_ext * (1u << logN), logN, nfull, 0, htabs[0].nt, 0, st, nb, xc_bst, r_bst);
  if (par) {
    cudaError_t e2 = cudaEventRecord(join, side);
    if (!e2) e2 = cudaStreamWaitEvent(st, join, 0);
    if (!e) e = e2;
  }
  return e;
}

cudaError_t launch_ks_inner(u64* acc, const u64* x_eval, const u64* raised, const u64* key_b, const u64* key_a,
                            Basis basis, u32 alpha, u32 ndig, u32 logN, u64 g, const ModConsts* mc,
                            cudaStream_t st, u32 nb, size_t x_bst, const u64* c0, size_t c0_bst, const u64* pR,
                            u32 key_lq, u32 fast_from) {
  // batches of g_ks_tma_min (2) or more entries take the TMA-staged inner
  // product, single entries the register-pipelined kernel (measured with
  // tools/ks_bench.py and interleaved ResNet20 A/B runs)
  if (g_ks_tma && g_ks_tma3 && nb >= (u32)g_ks_tma_min && (1u << logN) % kMacTile == 0) {
    // rows [0, ff) and [nq, n_ext): generic; [ff, nq): 96-bit carry chains
    const u32 nbb = nb ? nb : 1, nq = basis.nq, nl = basis.nlimbs();
    const u32 ff = fast_from < 1 ? 1 : (fast_from > nq ? nq : fast_from);
    const int stages = g_ks3_stages >= 2 && g_ks3_stages <= 4 ? g_ks3_stages : 3;
    auto go3 = [&](auto kern, int fast, u32 r0, u32 rows) -> cudaError_t {
      (void)fast;
      if (rows == 0) return cudaSuccess;
      const size_t sm = sizeof(KsStage) * stages;
      cudaError_t e = ensure_smem((const void*)kern, sm);
      if (e) return e;
      dim3 grid((1u << logN) / kMacTile, rows, (nbb + kKsEntries - 1) / kKsEntries);
      kern<<<grid, 128 + 32, sm, st>>>(acc, x_eval, raised, key_b, key_a, basis, alpha, ndig, logN, g, mc, nbb, x_bst,
                                      c0, c0_bst, pR, key_lq, r0);
      return cudaGetLastError();
    };
    cudaError_t e;
#define KS3(ST)                                                                          \
    if (stages == ST && g_ks_tma3 == 2) return go3(k_ks_inner_tma3<ST, 128, false>, 0, 0, nl); \
    if (stages == ST) {                                                                  \
      e = go3(k_ks_inner_tma3<ST, 128, false>, 0, 0, ff);                                \
      if (!e) e = go3(k_ks_inner_tma3<ST, 128, true>, 1, ff, nq - ff);                   \
      if (!e) e = go3(k_ks_inner_tma3<ST, 128, false>, 0, nq, nl - nq);                  \
      return e;                                                                          \
    }
    KS3(2) KS3(3) KS3(4)
#undef KS3
  }
  if (g_ks_tma && nb >= (u32)g_ks_tma_min && (1u << logN) % kMacTile == 0) {
    const u32 nbb = nb ? nb : 1;
    dim3 grid((1u << logN) / kMacTile, basis.nlimbs(), (nbb + kKsEntries - 1) / kKsEntries);
    const int tpb = g_ks_tpb == 128 ? 128 : 256;
    auto go = [&](auto kern, int stages) -> cudaError_t {
      const size_t sm = sizeof(KsStage) * stages;
      cudaError_t e = ensure_smem((const void*)kern, sm);
      if (e) return e;
      kern<<<grid, tpb, sm, st>>>(acc, x_eval, raised, key_b, key_a, basis, alpha, ndig, logN, g, mc, nbb, x_bst, c0,
                                  c0_bst, pR, key_lq);
      return cudaGetLastError();
    };
    cudaError_t e = tpb == 128 ? (g_ks_stages == 3 ? go(k_ks_inner_tma2<3, 128>, 3) : go(k_ks_inner_tma2<4, 128>, 4))
                    : g_tma_stages >= 8 ? go(k_ks_inner_tma<8>, 8)
                    : g_tma_stages >= 6 ? go(k_ks_inner_tma<6>, 6) : go(k_ks_inner_tma<4>, 4);
    if (e) return e;
  } else if ((nb <= 1 || g_ks_batch <= 1) && g_ks_pipe > 0) {
    dim3 grid = row_grid((1u << logN) / 2, basis.nlimbs(), 256);
    grid.x *= (nb ? nb : 1);
    if (g_ks_pipe >= 4)
      k_ks_inner_p<4><<<grid, 256, 0, st>>>(acc, x_eval, raised, key_b, key_a, basis, alpha, ndig, logN, g, mc,
                                            nb ? nb : 1, x_bst, c0, c0_bst, pR, key_lq);
    else
      k_ks_inner_p<2><<<grid, 256, 0, st>>>(acc, x_eval, raised, key_b, key_a, basis, alpha, ndig, logN, g, mc,
                                            nb ? nb : 1, x_bst, c0, c0_bst, pR, key_lq);
  } else if (nb <= 1 || g_ks_batch <= 1) {
    dim3 grid = row_grid((1u << logN) / 2, basis.nlimbs(), 256);
    grid.x *= (nb ? nb : 1);
    k_ks_inner<1, 2><<<grid, 256, 0, st>>>(acc, x_eval, raised, key_b, key_a, basis, alpha, ndig, logN, g, mc,
                                           nb ? nb : 1, x_bst, c0, c0_bst, pR, key_lq);
  } else if (nb == 2 || g_ks_batch == 2) {
    dim3 grid = row_grid(1u << logN, basis.nlimbs(), 256);
    grid.z = (nb + 1) / 2;
    k_ks_inner<2, 1><<<grid, 256, 0, st>>>(acc, x_eval, raised, key_b, key_a, basis, alpha, ndig, logN, g, mc, nb,
                                           x_bst, c0, c0_bst, pR, key_lq);
  } else {
    dim3 grid = row_grid(1u << logN, basis.nlimbs(), 256);
    grid.z = (nb + 3) / 4;
    k_ks_inner<4, 1><<<grid, 256, 0, st>>>(acc, x_eval, raised, key_b, key_a, basis, alpha, ndig, logN, g, mc, nb,
                                           x_bst, c0, c0_bst, pR, key_lq);
  }
  return cudaGetLastError();
}


int g_ks_rots = 1;         // hoisted groups: every rotation's inner product in one launch (k_ks_inner_tma2_rots)
int g_ks_rots_min_nb = 1;  // ... for batches of at least this many entries

bool ks_rots_ok(u32 nb, u32 nrot, u32 logN) {
  return g_ks_rots && g_ks_tma && !g_ks_tma3 && g_ks_tpb == 128 && nrot >= 2 && nb >= (u32)g_ks_rots_min_nb &&
         (1u << logN) % kMacTile == 0;
}

cudaError_t launch_ks_inner_rots(const KsRots& R, u32 nrot, const u64* x_eval, const u64* raised, Basis basis,
                                 u32 alpha, u32 ndig, u32 logN, const ModConsts* mc, cudaStream_t st, u32 nb,
                                 size_t x_bst, const u64* c0, size_t c0_bst, const u64* pR) {
  if (nrot == 0) return cudaSuccess;
  if (nrot > (u32)kKsRotMax) return cudaErrorInvalidValue;
  const u32 nbb = nb ? nb : 1;
  dim3 grid((1u << logN) / kMacTile * nrot, basis.nlimbs(), (nbb + kKsEntries - 1) / kKsEntries);
  auto go = [&](auto kern, int stages) -> cudaError_t {
    const size_t sm = sizeof(KsStage) * stages;
    cudaError_t e = ensure_smem((const void*)kern, sm);
    if (e) return e;
    kern<<<grid, 128, sm, st>>>(R, nrot, x_eval, raised, basis, alpha, ndig, logN, mc, nbb, x_bst, c0, c0_bst, pR);
    return cudaGetLastError();
  };
  return g_ks_stages == 4 ? go(k_ks_inner_tma2_rots<4, 128>, 4) : go(k_ks_inner_tma2_rots<3, 128>, 3);
}

cudaError_t launch_moddown_combine(u64* out0, u64* out1, const u64* acc, const u64* lift, const u64* add0,
                                   const u64* add1, u64 g_add, u32 nq, u32 n_ext, u32 logN, const u64* pinv,
                                   const u64* pinv_sh, const ModConsts* mc, cudaStream_t st, u32 nb,
                                   size_t out_bst, size_t add_bst) {
  dim3 g = row_grid((1u << logN) / 2, nq, 256);
  g.z = 2 * nb;
  k_moddown_combine<<<g, 256, 0, st>>>(out0, out1, acc, lift, add0, add1, g_add, nq, n_ext, logN, pinv, pinv_sh,
                                       mc, out_bst, add_bst);
  return cudaGetLastError();
}

cudaError_t launch_rescale_lift(u64* out, const u64* top, u32 l, u32 logN, u32 npolys, const u64* qtop_mod,
                                const ModConsts* mc, cudaStream_t st) {
  dim3 g = row_grid(1u << logN, l, 256);
  g.z = npolys;
  k_rescale_lift<<<g, 256, 0, st>>>(out, top, l, logN, qtop_mod, mc);
  return cudaGetLastError();
}

cudaError_t launch_rescale_combine(u64* out, const u64* in, u32 l, u32 logN, u32 npolys, const u64* inv,
                                   const u64* inv_sh, const ModConsts* mc, cudaStream_t st) {
  dim3 g = row_grid(1u << logN, l, 256);
  g.z = npolys;
  k_rescale_combine<<<g, 256, 0, st>>>(out, in, l, logN, inv, inv_sh, mc);
  return cudaGetLastError();
}

cudaError_t launch_gather_limb(u64* out, const u64* in, u32 limb, u32 nlimbs, u32 logN, u32 npolys,
                               cudaStream_t st) {
  k_gather_limb<<<row_grid(1u << logN, npolys, 256), 256, 0, st>>>(out, in, limb, nlimbs, logN);
  return cudaGetLastError();
}

}  // namespace hcnn
