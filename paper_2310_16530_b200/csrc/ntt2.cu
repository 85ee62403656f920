// Register-resident radix-16 NTT passes for 2^12 <= N <= 2^16 (sm_100a).
//
// Same contract as ntt.cu (bit-exact with the reference's CT / GS
// transforms, kernels.py:232-281), restructured for the integer pipe:
//   N = N1 * 256.  Pass "cols" runs the N1-point network down columns
//   (rows k*256), pass "chunks" the 256-point network inside each
//   contiguous chunk.  Every thread keeps 16 residues in registers and runs
//   4 butterfly stages per register group; groups exchange data through
//   one shared-memory transpose (conflict-free: lanes map to columns in the
//   column pass, a 16x17 padded tile per chunk in the chunk pass), so a
//   256-point network costs 8 stages of register butterflies and a single
//   smem round trip instead of a barrier per stage.
//   Chunk twiddles are pre-gathered per chunk (255 Shoup pairs, contiguous,
//   16-byte loads); column twiddles (first N1 entries of the standard
//   table) are staged in shared memory.
// Forward keeps Harvey-lazy values in [0,4q) between passes and fully
// reduces at the end; inverse keeps [0,2q) and folds N^-1 into the last
// Gentleman-Sande stage.
#include <atomic>

#include "common.cuh"
#include "kernels.cuh"
#include "tma.cuh"

namespace hcnn {

NttTuning g_ntt_tuning;


// L2 policy: keep twiddle tables resident (evict_last), stream the data
__device__ __forceinline__ u64 keep_policy() {
  u64 pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
template <bool HINT>
__device__ __forceinline__ ulonglong2 ld_tw(const ulonglong2* p, u64 pol) {
  if constexpr (HINT) {
    ulonglong2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;"
                 : "=l"(v.x), "=l"(v.y) : "l"(p), "l"(pol));
    return v;
  } else {
    return __ldg(p);
  }
}
template <bool HINT>
__device__ __forceinline__ u64 ld_last(const u64* p) {  // data read for the last time
  if constexpr (HINT) return __ldcs(p);
  else return *p;
}

// Harvey butterflies with the approximate Shoup quotient.  Forward keeps
// values in [0, 8q) (qb = 4q): X is folded to [0,4q), T in [0,4q).
// Inverse keeps [0, 4q).  Requires q < 2^61.
__device__ __forceinline__ void ct_bfly(u64& X, u64& Y, u64 w, u64 wp, u64 q, u64 qb) {
  u64 x = X >= qb ? X - qb : X;
  u64 t = shoup_approx(Y, w, wp, q);
  X = x + t;
  Y = x - t + qb;
}

__device__ __forceinline__ void gs_bfly(u64& X, u64& Y, u64 w, u64 wp, u64 q, u64 qb) {
  u64 s = X + Y;
  s = s >= qb ? s - qb : s;
  u64 t = X - Y + qb;
  X = s;
  Y = shoup_approx(t, w, wp, q);
}

// Unreduced butterflies for q < 2^47 (24 of the 29 moduli of config 2): the
// 64-bit word has room for the growth, so the per-stage conditional
// subtractions (the ALU-pipe bottleneck) disappear.  Forward: values grow by
// < 4q per stage (T = Shoup output in [0,4q)), < 65q after 16 stages.
// Inverse: the sum doubles per stage, values < q 2^(s+1) after stage s;
// C_s = q 2^(s+1) keeps X - Y + C_s positive.
__device__ __forceinline__ void ct_bfly_fast(u64& X, u64& Y, u64 w, u64 wp, u64 q, u64 q4) {
  u64 t = shoup_approx(Y, w, wp, q);
  u64 x = X;
  X = x + t;
  Y = x + q4 - t;
}
__device__ __forceinline__ void gs_bfly_fast(u64& X, u64& Y, u64 w, u64 wp, u64 q, u64 c) {
  u64 x = X, y = Y;
  X = x + y;
  Y = shoup_approx(x - y + c, w, wp, q);
}

// Shoup product with the quotient estimated on the FP64 pipe (q < 2^47,
// a < 2^51): wq = fl(w / q); qhat = trunc(fl(a) * wq - 1) is Q-2..Q of the
// true quotient Q = floor(a w / q), so a*w - qhat*q (exact, low 64 bits) lies
// in [0, 3q).  Moves the 3 IMAD.WIDE of the high product onto the DFMA and
// conversion units.
__device__ __forceinline__ u64 shoup_fp(u64 a, u64 w, double wq, u64 q) {
  const double qf = fma(__ull2double_rn(a), wq, -1.0);
  const u64 qhat = __double2ull_rz(qf);
  return a * w - qhat * q;
}
// Same with magic-number conversions (no XU ops): for 0 <= a < 2^52,
// double(a) = bits(2^52 | a) - 2^52 (one DADD), and fma(.., 2^52) rounds the
// quotient estimate to the nearest integer in the low mantissa bits.
// qr = round(a wq) is Q-1..Q+1, so a*w - qr*q + q lies in [0, 3q).
__device__ __forceinline__ u64 shoup_fp2(u64 a, u64 w, double wq, u64 q) {
  const double two52 = 4503599627370496.0;
  const double ad = __longlong_as_double((long long)(a | 0x4330000000000000ull)) - two52;
  const double qf = fma(ad, wq, two52);
  const u64 qr = (u64)__double_as_longlong(qf) & 0x000FFFFFFFFFFFFFull;
  return a * w - qr * q + q;
}
__device__ __forceinline__ void ct_bfly_fp2(u64& X, u64& Y, u64 w, double wq, u64 q, u64 q4) {
  u64 t = shoup_fp2(Y, w, wq, q);
  u64 x = X;
  X = x + t;
  Y = x + q4 - t;
}
__device__ __forceinline__ void ct_bfly_fp(u64& X, u64& Y, u64 w, double wq, u64 q, u64 q4) {
  u64 t = shoup_fp(Y, w, wq, q);
  u64 x = X;
  X = x + t;
  Y = x + q4 - t;
}

// One CT stage d of a 16-point network held in x[0..15]: pairs k with
// k + (8>>d) inside sub-block b = k >> (4-d).  Stages are template
// parameters so every register index is a compile-time constant.
template <int d, class TW>
__device__ __forceinline__ void ct_stage(u64 (&x)[16], u64 q, u64 q2, TW& tw) {
  constexpr int h = 8 >> d;
#pragma unroll
  for (int b = 0; b < (1 << d); ++b) {
    ulonglong2 W = tw(d, b);
#pragma unroll
    for (int r = 0; r < h; ++r) ct_bfly(x[2 * h * b + r], x[2 * h * b + r + h], W.x, W.y, q, q2);
  }
}

template <int d, class TW>
__device__ __forceinline__ void ct_stage_fast(u64 (&x)[16], u64 q, u64 q4, TW& tw) {
  constexpr int h = 8 >> d;
#pragma unroll
  for (int b = 0; b < (1 << d); ++b) {
    ulonglong2 W = tw(d, b);
#pragma unroll
    for (int r = 0; r < h; ++r) ct_bfly_fast(x[2 * h * b + r], x[2 * h * b + r + h], W.x, W.y, q, q4);
  }
}

template <int d, class TW>
__device__ __forceinline__ void ct_stage_fp(u64 (&x)[16], u64 q, u64 q4, TW& tw) {
  constexpr int h = 8 >> d;
#pragma unroll
  for (int b = 0; b < (1 << d); ++b) {
    ulonglong2 W = tw(d, b);
    const double wq = __longlong_as_double((long long)W.y);
#pragma unroll
    for (int r = 0; r < h; ++r) ct_bfly_fp(x[2 * h * b + r], x[2 * h * b + r + h], W.x, wq, q, q4);
  }
}

// CT stages d in [D0,4); FAST selects the unreduced butterflies (q < 2^47),
// FP the unreduced butterflies with the FP64 quotient (q < 2^44; twiddle
// companions hold double(w/q) bits)
template <int D0, bool FAST = false, class TW, bool FP = false>
__device__ __forceinline__ void ct16(u64 (&x)[16], u64 q, u64 q2, TW tw) {
  if constexpr (FP) {
    if constexpr (D0 <= 0) ct_stage_fp<0>(x, q, q2, tw);
    if constexpr (D0 <= 1) ct_stage_fp<1>(x, q, q2, tw);
    if constexpr (D0 <= 2) ct_stage_fp<2>(x, q, q2, tw);
    if constexpr (D0 <= 3) ct_stage_fp<3>(x, q, q2, tw);
  } else if constexpr (FAST) {
    if constexpr (D0 <= 0) ct_stage_fast<0>(x, q, q2, tw);
    if constexpr (D0 <= 1) ct_stage_fast<1>(x, q, q2, tw);
    if constexpr (D0 <= 2) ct_stage_fast<2>(x, q, q2, tw);
    if constexpr (D0 <= 3) ct_stage_fast<3>(x, q, q2, tw);
  } else {
    if constexpr (D0 <= 0) ct_stage<0>(x, q, q2, tw);
    if constexpr (D0 <= 1) ct_stage<1>(x, q, q2, tw);
    if constexpr (D0 <= 2) ct_stage<2>(x, q, q2, tw);
    if constexpr (D0 <= 3) ct_stage<3>(x, q, q2, tw);
  }
}

struct Fold {
  u64 ninvN, ninvN_sh, ilast, ilast_sh;
};

// One GS stage d: pairs k with k + (1<<d) inside sub-block b = k >> (d+1).
template <int d, class TW>
__device__ __forceinline__ void gs_stage(u64 (&x)[16], u64 q, u64 q2, TW& tw) {
  constexpr int h = 1 << d;
#pragma unroll
  for (int b = 0; b < (8 >> d); ++b) {
    ulonglong2 W = tw(d, b);
#pragma unroll
    for (int r = 0; r < h; ++r) gs_bfly(x[2 * h * b + r], x[2 * h * b + r + h], W.x, W.y, q, q2);
  }
}

template <int d, class TW>
__device__ __forceinline__ void gs_stage_fast(u64 (&x)[16], u64 q, u64 c, TW& tw) {
  constexpr int h = 1 << d;
#pragma unroll
  for (int b = 0; b < (8 >> d); ++b) {
    ulonglong2 W = tw(d, b);
#pragma unroll
    for (int r = 0; r < h; ++r) gs_bfly_fast(x[2 * h * b + r], x[2 * h * b + r + h], W.x, W.y, q, c);
  }
}

// GS stages d in [D0,4).  FOLD: stage 3 is the transform's last one
// (twiddle itw[1]) and also applies N^-1.  FAST: unreduced butterflies;
// s0 is the global index of stage d = 0 (sets C_s = q 2^(s+1)).
template <int D0, bool FOLD, bool FAST = false, class TW>
__device__ __forceinline__ void gs16(u64 (&x)[16], u64 q, u64 q2, TW tw, Fold C, u32 s0 = 0) {
  if constexpr (FAST) {
    if constexpr (D0 <= 0) gs_stage_fast<0>(x, q, q << (s0 + 1), tw);
    if constexpr (D0 <= 1) gs_stage_fast<1>(x, q, q << (s0 + 2), tw);
    if constexpr (D0 <= 2) gs_stage_fast<2>(x, q, q << (s0 + 3), tw);
  } else {
    if constexpr (D0 <= 0) gs_stage<0>(x, q, q2, tw);
    if constexpr (D0 <= 1) gs_stage<1>(x, q, q2, tw);
    if constexpr (D0 <= 2) gs_stage<2>(x, q, q2, tw);
  }
  if constexpr (FOLD) {
    const u64 c3 = FAST ? (q << (s0 + 4)) : q2;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      u64 s = x[r] + x[r + 8];
      u64 t = x[r] - x[r + 8] + c3;
      x[r] = shoup_mul(s, C.ninvN, C.ninvN_sh, q);
      x[r + 8] = shoup_mul(t, C.ilast, C.ilast_sh, q);
    }
  } else if constexpr (FAST) {
    gs_stage_fast<3>(x, q, q << (s0 + 4), tw);
  } else {
    gs_stage<3>(x, q, q2, tw);
  }
}

__device__ __forceinline__ bool limb_skipped2(const LimbMap& m, u32 r, u32 z) {
  if (m.skip_alpha == 0) return false;
  r += m.first_limb;
  if (m.zmod) z %= m.zmod;
  u32 lo = z * m.skip_alpha;
  u32 hi = lo + m.skip_alpha;
  if (hi > m.basis.nq) hi = m.basis.nq;
  return r >= lo && r < hi;
}

// ---------------------------------------------------------------------------
// column pass (N1 = 2^LOGN1 points, 16 <= N1 <= 256), 256 threads,
// COLS = 256/T1 columns per CTA, T1 = N1/16 threads per column
// ---------------------------------------------------------------------------
template <int LOGN1, bool HINT, int MINB, int MODE>
__global__ void __launch_bounds__(256, MINB) ntt2_fwd_cols(LimbMap map, const ModConsts* __restrict__ mc,
                                                     const u64* __restrict__ tw, const u64* __restrict__ twp,
                                                     u32 logN) {
  constexpr int N1 = 1 << LOGN1, T1 = N1 / 16, COLS = 256 / T1, NSB = LOGN1 - 4;
  __shared__ u64 tile[N1 * COLS];
  __shared__ ulonglong2 sw[N1];
  const u32 r = blockIdx.y + map.r0, z = blockIdx.z + map.z0;
  if (limb_skipped2(map, r, z)) return;
  const u32 N = 1u << logN, N2 = N >> LOGN1;
  const u32 mod = map.basis.mod_of(r + map.first_limb);
  const u64 q = mc[mod].q, q2 = mc[mod].four_q;
  u64* a = map.base + (size_t)z * map.poly_stride + (size_t)r * N + blockIdx.x * COLS;
  const int tid = threadIdx.x, c = tid % COLS, j = tid / COLS;
  // MODE 0: full-width, 1: q < 2^47 integer fast path, 3: FP64-quotient
  // path (q < 2^kFpBits), 2: chosen per limb at run time
  const bool fast = MODE == 2 ? (q < (1ull << 47)) : (MODE == 1 || MODE == 3);
  const bool fp = MODE == 3;  // (unused: class-2 limbs launch the FP64 kernels)
  for (int i = tid; i < N1; i += 256) {
    const u64 wp = twp[(size_t)mod * N + i];
    sw[i] = make_ulonglong2(tw[(size_t)mod * N + i], fp ? (u64)__double_as_longlong(__ull2double_rn(wp) * 0x1p-64) : wp);
  }
  u64 x[16];
  if (map.sin) {
    const long long* s = map.sin + (size_t)z * N + blockIdx.x * COLS;
    const u64 kr = map.smont ? mc[mod].r2 : mc[mod].one_m, ninv = mc[mod].ninv;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      long long v = s[(size_t)(j + T1 * k) * N2 + c];
      if (map.sin_center) {  // centred lift of a residue mod sin_center (fused rescale, ckks.py:506-528)
        const u64 t = (u64)v;
        v = t > (map.sin_center >> 1) ? (long long)(t - map.sin_center) : (long long)t;
      }
      const u64 mag = v >= 0 ? (u64)v : (u64)(-(v + 1)) + 1ull;
      const u64 red = mont_mul(mag, kr, q, ninv);
      x[k] = v >= 0 ? red : neg_mod(red, q);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = ld_last<HINT>(&a[(size_t)(j + T1 * k) * N2 + c]);
  }
  __syncthreads();
  auto twA = [&](int d, int b) { return sw[(1 << d) + b]; };
  if (fp) ct16<0, true, decltype(twA), true>(x, q, q2, twA);
  else if (fast) ct16<0, true>(x, q, q2, twA);
  else ct16<0, false>(x, q, q2, twA);
  if (NSB > 0) {
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[(j + T1 * k) * COLS + c] = x[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = tile[(16 * j + k) * COLS + c];
    auto twB = [&](int d, int b) { return sw[(1 << (d + NSB)) + (j << d) + b]; };
    if (fp) ct16<4 - NSB, true, decltype(twB), true>(x, q, q2, twB);
    else if (fast) ct16<4 - NSB, true>(x, q, q2, twB);
    else ct16<4 - NSB, false>(x, q, q2, twB);
#pragma unroll
    for (int k = 0; k < 16; ++k) a[(size_t)(16 * j + k) * N2 + c] = x[k];
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k) a[(size_t)(j + T1 * k) * N2 + c] = x[k];
  }
}

template <int LOGN1, bool HINT, int MINB, int MODE>
__global__ void __launch_bounds__(256, MINB) ntt2_inv_cols(LimbMap map, const ModConsts* __restrict__ mc,
                                                     const u64* __restrict__ itw, const u64* __restrict__ itwp,
                                                     u32 logN) {
  constexpr int N1 = 1 << LOGN1, T1 = N1 / 16, COLS = 256 / T1, NSA = LOGN1 - 4;
  __shared__ u64 tile[N1 * COLS];
  __shared__ ulonglong2 sw[N1];
  const u32 r = blockIdx.y + map.r0, z = blockIdx.z + map.z0;
  if (limb_skipped2(map, r, z)) return;
  const u32 N = 1u << logN, N2 = N >> LOGN1;
  const u32 mod = map.basis.mod_of(r + map.first_limb);
  const u64 q = mc[mod].q, q2 = mc[mod].four_q;
  const Fold C{mc[mod].ninvN, mc[mod].ninvN_sh, mc[mod].ilast, mc[mod].ilast_sh};
  u64* a = map.base + (size_t)z * map.poly_stride + (size_t)r * N + blockIdx.x * COLS;
  const int tid = threadIdx.x, c = tid % COLS, j = tid / COLS;
  for (int i = tid; i < N1; i += 256) sw[i] = make_ulonglong2(itw[(size_t)mod * N + i], itwp[(size_t)mod * N + i]);
  u64 x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = ld_last<HINT>(&a[(size_t)(16 * j + k) * N2 + c]);
  __syncthreads();
  // stages t = 1..8 rows: contiguous groups of 16 rows; twiddle itw[H + i],
  // H = N1 >> (d+1) blocks, i = j*(8>>d) + b
  const bool fast = MODE == 2 ? (q < (1ull << 47)) : (MODE == 1 || MODE == 3);
  auto twB = [&](int d, int b) { return sw[(N1 >> (d + 1)) + j * (8 >> d) + b]; };
  auto twA = [&](int d, int b) { return sw[(8 >> d) + b]; };
  if (NSA == 0) {
    if (fast) gs16<0, true, true>(x, q, q2, twB, C, 8);
    else gs16<0, true, false>(x, q, q2, twB, C);
#pragma unroll
    for (int k = 0; k < 16; ++k) a[(size_t)(16 * j + k) * N2 + c] = x[k];
  } else {
    if (fast) gs16<0, false, true>(x, q, q2, twB, C, 8);
    else gs16<0, false, false>(x, q, q2, twB, C);
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[(16 * j + k) * COLS + c] = x[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = tile[(j + T1 * k) * COLS + c];
    if (fast) gs16<4 - NSA, true, true>(x, q, q2, twA, C, 8 + NSA);
    else gs16<4 - NSA, true, false>(x, q, q2, twA, C);
#pragma unroll
    for (int k = 0; k < 16; ++k) a[(size_t)(j + T1 * k) * N2 + c] = x[k];
  }
}

// ---------------------------------------------------------------------------
// chunk pass: 8 chunks of 256 per CTA (128 threads), 16 threads (half a
// warp) per chunk.  All loads are issued up front: the 16 residues, the
// chunk's 15 shared first-group twiddles (into smem) and this thread's 15
// second-group twiddles (into registers), so their latency overlaps the
// first group's butterflies instead of stalling mid-network.
// ---------------------------------------------------------------------------
constexpr int kChunksPerCta = 8;

template <bool HINT, int MINB, int MODE>
__global__ void __launch_bounds__(128, MINB) ntt2_fwd_chunks(LimbMap map, const ModConsts* __restrict__ mc,
                                                       const ulonglong2* __restrict__ ctw, u32 logN) {
  __shared__ u64 tile[kChunksPerCta][16 * 17];
  __shared__ ulonglong2 twa[kChunksPerCta][16];
  const u32 r = blockIdx.y + map.r0, z = blockIdx.z + map.z0;
  if (limb_skipped2(map, r, z)) return;
  const u32 N = 1u << logN, N1 = N >> 8;
  const u32 mod = map.basis.mod_of(r + map.first_limb);
  const u64 q = mc[mod].q, q2 = mc[mod].four_q;
  const int tid = threadIdx.x, cc = tid >> 4, j = tid & 15;
  const u32 g = blockIdx.x * kChunksPerCta + cc;
  u64* a = map.base + (size_t)z * map.poly_stride + (size_t)r * N + (size_t)g * 256;
  const ulonglong2* T = ctw + ((size_t)mod * N1 + g) * 256;
  u64* tl = tile[cc];
  const u64 pol = HINT ? keep_policy() : 0;
  u64 x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = ld_last<HINT>(&a[j + 16 * k]);
  if (j < 15) twa[cc][j] = ld_tw<HINT>(&T[j], pol);
  // second-group twiddles: stage 4+d, block (j<<d)+b -> e = (16<<d)-1+(j<<d)+b
  ulonglong2 tb[15];
#pragma unroll
  for (int d = 0; d < 4; ++d)
#pragma unroll
    for (int b = 0; b < (1 << d); ++b) tb[(1 << d) - 1 + b] = ld_tw<HINT>(&T[(16 << d) - 1 + (j << d) + b], pol);
  __syncwarp();
  const bool fast = MODE == 2 ? (q < (1ull << 47)) : (MODE == 1 || MODE == 3);
  const bool fp = MODE == 3;  // (unused: class-2 limbs launch the FP64 kernels)
  auto twA = [&](int d, int b) { return twa[cc][(1 << d) - 1 + b]; };
  if (fp) ct16<0, true, decltype(twA), true>(x, q, q2, twA);
  else if (fast) ct16<0, true>(x, q, q2, twA);
  else ct16<0, false>(x, q, q2, twA);
#pragma unroll
  for (int k = 0; k < 16; ++k) tl[17 * k + j] = x[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = tl[17 * j + k];
  auto twB = [&](int d, int b) { return tb[(1 << d) - 1 + b]; };
  if (fast) {
    if (fp) ct16<0, true, decltype(twB), true>(x, q, q2, twB);
    else ct16<0, true>(x, q, q2, twB);
    const u64 one_sh = mc[mod].one_sh;
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = shoup_mul(x[k], 1, one_sh, q);  // < 65q -> [0, q)
  } else {
    ct16<0, false>(x, q, q2, twB);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      u64 v = x[k];
      v = v >= q2 ? v - q2 : v;              // [0, 4q)
      v = v >= 2 * q ? v - 2 * q : v;        // [0, 2q)
      x[k] = v >= q ? v - q : v;
    }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) tl[17 * j + k] = x[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) a[j + 16 * k] = tl[17 * k + j];
}

template <bool HINT, int MINB, int MODE>
__global__ void __launch_bounds__(128, MINB) ntt2_inv_chunks(LimbMap map, const ModConsts* __restrict__ mc,
                                                       const ulonglong2* __restrict__ ctw, u32 logN) {
  __shared__ u64 tile[kChunksPerCta][16 * 17];
  __shared__ ulonglong2 twa[kChunksPerCta][16];
  const u32 r = blockIdx.y + map.r0, z = blockIdx.z + map.z0;
  if (limb_skipped2(map, r, z)) return;
  const u32 N = 1u << logN, N1 = N >> 8;
  const u32 mod = map.basis.mod_of(r + map.first_limb);
  const u64 q = mc[mod].q, q2 = mc[mod].four_q;
  const Fold C{0, 0, 0, 0};
  const int tid = threadIdx.x, cc = tid >> 4, j = tid & 15;
  const u32 g = blockIdx.x * kChunksPerCta + cc;
  u64* a = map.base + (size_t)z * map.poly_stride + (size_t)r * N + (size_t)g * 256;
  const ulonglong2* T = ctw + ((size_t)mod * N1 + g) * 256;
  u64* tl = tile[cc];
  const u64 pol = HINT ? keep_policy() : 0;
  u64 x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = ld_last<HINT>(&a[j + 16 * k]);
  // first group (local stages 0..3): nb = 128>>d blocks, i = j*(8>>d)+b
  ulonglong2 tb[15];
#pragma unroll
  for (int d = 0; d < 4; ++d)
#pragma unroll
    for (int b = 0; b < (8 >> d); ++b)
      tb[16 - (16 >> d) + b] = ld_tw<HINT>(&T[(128 >> d) - 1 + j * (8 >> d) + b], pol);
  // second group (local stages 4..7): nb = 8>>d, i = b -> e = (8>>d)-1+b, shared
  if (j < 15) twa[cc][j] = ld_tw<HINT>(&T[j], pol);
#pragma unroll
  for (int k = 0; k < 16; ++k) tl[17 * k + j] = x[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = tl[17 * j + k];
  const bool fast = MODE == 2 ? (q < (1ull << 47)) : (MODE == 1 || MODE == 3);
  auto twB = [&](int d, int b) { return tb[16 - (16 >> d) + b]; };
  if (fast) gs16<0, false, true>(x, q, q2, twB, C, 0);
  else gs16<0, false, false>(x, q, q2, twB, C);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) tl[17 * j + k] = x[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = tl[17 * k + j];
  auto twA = [&](int d, int b) { return twa[cc][(8 >> d) - 1 + b]; };
  if (fast) gs16<0, false, true>(x, q, q2, twA, C, 4);
  else gs16<0, false, false>(x, q, q2, twA, C);
#pragma unroll
  for (int k = 0; k < 16; ++k) a[j + 16 * k] = x[k];
}

// ---------------------------------------------------------------------------
// FP64 network for the moduli below 2^kFpBits (the 40/41-bit application
// primes): residues live as signed integer-valued doubles between the load
// and the final store, so every butterfly runs on the FP64 pipe alone.
//   t = a*w mod q:  hi = fl(a w), lo = fma(a, w, -hi)  (a w = hi + lo exactly),
//   qe = round(a * fl(w/q)) by the 1.5*2^52 magic constant, t = fma(-qe, q, hi) + lo.
// For |a| < 2^51 and q < 2^44: |a fl(w/q) - a w/q| < 1/4, so t lies in
// (-3q/4, 3q/4) and both the fma and the final add are exact (integers
// below 2^53).  Forward CT values grow by < 3q/4 per stage (|x| < 7q after
// a pass of 8 stages from [0,q), < 13q after the second); inverse GS values
// double per stage (< 2^8 q after a pass) and are centred between passes.
// The final canonical reduction returns exactly the residues of the
// integer networks (kernels.py:232-281), so outputs are bit-identical.
// ---------------------------------------------------------------------------
constexpr double kMagicRound = 6755399441055744.0;  // 1.5 * 2^52
constexpr double kTwo52 = 4503599627370496.0;

__device__ __forceinline__ double u2d(u64 v) {  // 0 <= v < 2^52
  return __longlong_as_double((long long)(v | 0x4330000000000000ull)) - kTwo52;
}
__device__ __forceinline__ u64 d2u(double d) {  // integer 0 <= d < 2^52
  return (u64)__double_as_longlong(d + kTwo52) & 0x000FFFFFFFFFFFFFull;
}
__device__ __forceinline__ double bits_d(u64 b) { return __longlong_as_double((long long)b); }
__device__ __forceinline__ u64 d_bits(double d) { return (u64)__double_as_longlong(d); }

__device__ __forceinline__ double fmulmod(double a, double w, double wq, double q) {
  const double hi = a * w;
  const double lo = fma(a, w, -hi);
  const double qe = fma(a, wq, kMagicRound) - kMagicRound;
  return fma(-qe, q, hi) + lo;
}
// |v| < 2^51 -> (-q/2 - 1, q/2 + 1)
__device__ __forceinline__ double fcentre(double v, double q, double qinv) {
  return fma(-(fma(v, qinv, kMagicRound) - kMagicRound), q, v);
}
// |v| < 2^51 -> [0, q)
__device__ __forceinline__ double fcanon(double v, double q, double qinv) {
  const double r = fcentre(v, q, qinv);
  return r < 0.0 ? r + q : (r >= q ? r - q : r);
}

template <int d, class TW>
__device__ __forceinline__ void ct_stage_f64(double (&x)[16], double q, TW& tw) {
  constexpr int h = 8 >> d;
#pragma unroll
  for (int b = 0; b < (1 << d); ++b) {
    const ulonglong2 W = tw(d, b);
    const double w = bits_d(W.x), wq = bits_d(W.y);
#pragma unroll
    for (int r = 0; r < h; ++r) {
      double& X = x[2 * h * b + r];
      double& Y = x[2 * h * b + r + h];
      const double t = fmulmod(Y, w, wq, q);
      const double u = X;
      X = u + t;
      Y = u - t;
    }
  }
}
template <int D0, class TW>
__device__ __forceinline__ void ct16_f64(double (&x)[16], double q, TW tw) {
  if constexpr (D0 <= 0) ct_stage_f64<0>(x, q, tw);
  if constexpr (D0 <= 1) ct_stage_f64<1>(x, q, tw);
  if constexpr (D0 <= 2) ct_stage_f64<2>(x, q, tw);
  if constexpr (D0 <= 3) ct_stage_f64<3>(x, q, tw);
}
template <int d, class TW>
__device__ __forceinline__ void gs_stage_f64(double (&x)[16], double q, TW& tw) {
  constexpr int h = 1 << d;
#pragma unroll
  for (int b = 0; b < (8 >> d); ++b) {
    const ulonglong2 W = tw(d, b);
    const double w = bits_d(W.x), wq = bits_d(W.y);
#pragma unroll
    for (int r = 0; r < h; ++r) {
      double& X = x[2 * h * b + r];
      double& Y = x[2 * h * b + r + h];
      const double u = X, v = Y;
      X = u + v;
      Y = fmulmod(u - v, w, wq, q);
    }
  }
}
struct FoldF {
  double ninvN, ninvN_q, ilast, ilast_q;
};
// GS stages d in [D0,4); FOLD: stage 3 is the transform's last (N^-1 folded)
template <int D0, bool FOLD, class TW>
__device__ __forceinline__ void gs16_f64(double (&x)[16], double q, TW tw, const FoldF& C) {
  if constexpr (D0 <= 0) gs_stage_f64<0>(x, q, tw);
  if constexpr (D0 <= 1) gs_stage_f64<1>(x, q, tw);
  if constexpr (D0 <= 2) gs_stage_f64<2>(x, q, tw);
  if constexpr (FOLD) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const double u = x[r], v = x[r + 8];
      x[r] = fmulmod(u + v, C.ninvN, C.ninvN_q, q);
      x[r + 8] = fmulmod(u - v, C.ilast, C.ilast_q, q);
    }
  } else {
    gs_stage_f64<3>(x, q, tw);
  }
}
__device__ __forceinline__ FoldF fold_f64(const ModConsts& m) {
  return FoldF{(double)m.ninvN, (double)m.ninvN_sh * 0x1p-64, (double)m.ilast, (double)m.ilast_sh * 0x1p-64};
}
// twiddle staging for the column passes: (w, w/q) as double bit patterns
__device__ __forceinline__ ulonglong2 tw_f64(u64 w, u64 wp) {
  return make_ulonglong2(d_bits((double)w), d_bits((double)wp * 0x1p-64));
}

template <int LOGN1, bool HINT, int MINB>
__global__ void __launch_bounds__(256, MINB) ntt2_fwd_cols_f64(LimbMap map, const ModConsts* __restrict__ mc,
                                                           const u64* __restrict__ tw, const u64* __restrict__ twp,
                                                           u32 logN) {
  constexpr int N1 = 1 << LOGN1, T1 = N1 / 16, COLS = 256 / T1, NSB = LOGN1 - 4;
  __shared__ u64 tile[N1 * COLS];
  __shared__ ulonglong2 sw[N1];
  const u32 r = blockIdx.y + map.r0, z = blockIdx.z + map.z0;
  if (limb_skipped2(map, r, z)) return;
  const u32 N = 1u << logN, N2 = N >> LOGN1;
  const u32 mod = map.basis.mod_of(r + map.first_limb);
  const u64 qi = mc[mod].q;
  const double q = (double)qi;
  u64* a = map.base + (size_t)z * map.poly_stride + (size_t)r * N + blockIdx.x * COLS;
  const int tid = threadIdx.x, c = tid % COLS, j = tid / COLS;
  for (int i = tid; i < N1; i += 256) sw[i] = tw_f64(tw[(size_t)mod * N + i], twp[(size_t)mod * N + i]);
  double x[16];
  if (map.sin) {
    const long long* s = map.sin + (size_t)z * N + blockIdx.x * COLS;
    const u64 kr = map.smont ? mc[mod].r2 : mc[mod].one_m, ninv = mc[mod].ninv;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      long long v = s[(size_t)(j + T1 * k) * N2 + c];
      if (map.sin_center) {  // centred lift of a residue mod sin_center (fused rescale, ckks.py:506-528)
        const u64 t = (u64)v;
        v = t > (map.sin_center >> 1) ? (long long)(t - map.sin_center) : (long long)t;
      }
      const u64 mag = v >= 0 ? (u64)v : (u64)(-(v + 1)) + 1ull;
      const u64 red = mont_mul(mag, kr, qi, ninv);
      x[k] = u2d(v >= 0 ? red : neg_mod(red, qi));
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = u2d(ld_last<HINT>(&a[(size_t)(j + T1 * k) * N2 + c]));
  }
  __syncthreads();
  auto twA = [&](int d, int b) { return sw[(1 << d) + b]; };
  ct16_f64<0>(x, q, twA);
  if (NSB > 0) {
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[(j + T1 * k) * COLS + c] = d_bits(x[k]);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = bits_d(tile[(16 * j + k) * COLS + c]);
    auto twB = [&](int d, int b) { return sw[(1 << (d + NSB)) + (j << d) + b]; };
    ct16_f64<4 - NSB>(x, q, twB);
#pragma unroll
    for (int k = 0; k < 16; ++k) a[(size_t)(16 * j + k) * N2 + c] = d_bits(x[k]);  // |x| < 7q, double bits
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k) a[(size_t)(j + T1 * k) * N2 + c] = d_bits(x[k]);
  }
}

template <bool HINT, int MINB>
__global__ void __launch_bounds__(128, MINB) ntt2_fwd_chunks_f64(LimbMap map, const ModConsts* __restrict__ mc,
                                                             const ulonglong2* __restrict__ ctw, u32 logN) {
  __shared__ u64 tile[kChunksPerCta][16 * 17];
  __shared__ ulonglong2 twa[kChunksPerCta][16];
  const u32 r = blockIdx.y + map.r0, z = blockIdx.z + map.z0;
  if (limb_skipped2(map, r, z)) return;
  const u32 N = 1u << logN, N1 = N >> 8;
  const u32 mod = map.basis.mod_of(r + map.first_limb);
  const double q = (double)mc[mod].q, qinv = 1.0 / q;
  const int tid = threadIdx.x, cc = tid >> 4, j = tid & 15;
  const u32 g = blockIdx.x * kChunksPerCta + cc;
  u64* a = map.base + (size_t)z * map.poly_stride + (size_t)r * N + (size_t)g * 256;
  const ulonglong2* T = ctw + ((size_t)mod * N1 + g) * 256;
  u64* tl = tile[cc];
  const u64 pol = HINT ? keep_policy() : 0;
  double x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = bits_d(ld_last<HINT>(&a[j + 16 * k]));
  if (j < 15) twa[cc][j] = ld_tw<HINT>(&T[j], pol);
  __syncwarp();
  auto twA = [&](int d, int b) { return twa[cc][(1 << d) - 1 + b]; };
  ct16_f64<0>(x, q, twA);
  // second-group twiddles loaded after the first group: not live across it
  // (fewer registers), their latency overlaps the transpose
  ulonglong2 tb[15];
#pragma unroll
  for (int d = 0; d < 4; ++d)
#pragma unroll
    for (int b = 0; b < (1 << d); ++b) tb[(1 << d) - 1 + b] = ld_tw<HINT>(&T[(16 << d) - 1 + (j << d) + b], pol);
#pragma unroll
  for (int k = 0; k < 16; ++k) tl[17 * k + j] = d_bits(x[k]);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = bits_d(tl[17 * j + k]);
  auto twB = [&](int d, int b) { return tb[(1 << d) - 1 + b]; };
  ct16_f64<0>(x, q, twB);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) tl[17 * j + k] = d2u(fcanon(x[k], q, qinv));  // |x| < 13q -> [0, q)
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) a[j + 16 * k] = tl[17 * k + j];
}

// Forward chunk pass of the FP64 network, pipelined over polys: a CTA owns
// chunk group blockIdx.x (8 chunks = 2048 contiguous coefficients) of one
// limb for a range of polys.  The chunk twiddles are loaded once per CTA,
// and each poly's 16 KB block is bulk-copied (cp.async.bulk + mbarrier)
// into a double-buffered shared ring while the previous poly computes, so
// the load latency that stalls the one-shot kernel (long_scoreboard ~50 %
// of samples, r02_ncu_summary.md) overlaps the butterflies.
constexpr u32 kChunkBlock = kChunksPerCta * 256;  // coefficients per CTA block
template <bool HINT, bool CB>
__global__ void __launch_bounds__(128) ntt2_fwd_chunks_f64p(LimbMap map, const ModConsts* __restrict__ mc,
                                                            const ulonglong2* __restrict__ ctw, u32 logN, u32 zper,
                                                            u32 nz, NttCombine cbv) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  u64* buf = reinterpret_cast<u64*>(smem_raw);  // [2][kChunkBlock]
  u64* tile = buf + 2 * kChunkBlock;             // [kChunksPerCta][16 * 17]
  __shared__ ulonglong2 twa[kChunksPerCta][16];
  __shared__ __align__(8) u64 full[2];
  const u32 r = blockIdx.y + map.r0;
  const u32 z_lo = map.z0 + blockIdx.z * zper;
  const u32 z_hi = z_lo + zper < map.z0 + nz ? z_lo + zper : map.z0 + nz;
  const u32 N = 1u << logN, N1 = N >> 8;
  const u32 mod = map.basis.mod_of(r + map.first_limb);
  const double q = (double)mc[mod].q, qinv = 1.0 / q;
  const int tid = threadIdx.x, cc = tid >> 4, j = tid & 15;
  const u32 g0 = blockIdx.x * kChunksPerCta, g = g0 + cc;
  const ulonglong2* T = ctw + ((size_t)mod * N1 + g) * 256;
  u64* tl = tile + cc * (16 * 17);
  const u64 pol = HINT ? keep_policy() : 0;
  if (j < 15) twa[cc][j] = ld_tw<HINT>(&T[j], pol);
  ulonglong2 tb[15];
#pragma unroll
  for (int d = 0; d < 4; ++d)
#pragma unroll
    for (int b = 0; b < (1 << d); ++b) tb[(1 << d) - 1 + b] = ld_tw<HINT>(&T[(16 << d) - 1 + (j << d) + b], pol);
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto blk = [&](u32 z) { return map.base + (size_t)z * map.poly_stride + (size_t)r * N + (size_t)g0 * 256; };
  auto next = [&](u32 z) {
    while (z < z_hi && limb_skipped2(map, r, z)) ++z;
    return z;
  };
  u32 z = next(z_lo);
  if (tid == 0 && z < z_hi) {
    mbar_expect_tx(&full[0], kChunkBlock * 8);
    bulk_g2s(buf, blk(z), kChunkBlock * 8, &full[0]);
  }
  auto twA = [&](int d, int b) { return twa[cc][(1 << d) - 1 + b]; };
  auto twB = [&](int d, int b) { return tb[(1 << d) - 1 + b]; };
  for (u32 it = 0; z < z_hi; ++it) {
    const u32 zn = next(z + 1), cur = it & 1u;
    if (tid == 0 && zn < z_hi) {  // buffer cur^1 was released by the previous iteration's barrier
      mbar_expect_tx(&full[cur ^ 1u], kChunkBlock * 8);
      bulk_g2s(buf + (cur ^ 1u) * kChunkBlock, blk(zn), kChunkBlock * 8, &full[cur ^ 1u]);
    }
    mbar_wait(&full[cur], (it >> 1) & 1u);
    const u64* B = buf + cur * kChunkBlock + cc * 256;
    double x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = bits_d(B[j + 16 * k]);
    ct16_f64<0>(x, q, twA);
#pragma unroll
    for (int k = 0; k < 16; ++k) tl[17 * k + j] = d_bits(x[k]);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = bits_d(tl[17 * j + k]);
    ct16_f64<0>(x, q, twB);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) tl[17 * j + k] = d2u(fcanon(x[k], q, qinv));  // |x| < 13q -> [0, q)
    __syncwarp();
    if constexpr (CB) {
      // fused ModDown combine: out = (acc_Q - lift) P^-1 (+ add), k_moddown_combine's arithmetic
      const u32 p = z & 1u, sb = z >> 1, s = sb / cbv.nb, b = sb % cbv.nb;
      const u64 qi = mc[mod].q, w = cbv.pinv[r], wp = cbv.pinv_sh[r], ga = cbv.g[s];
      const size_t k0 = (size_t)g * 256;
      const u64* A = cbv.acc + (size_t)z * cbv.acc_pst + (size_t)r * N + k0;
      const u64* ADD = cbv.add[p] ? cbv.add[p] + (size_t)b * cbv.add_bst + (size_t)r * N : nullptr;
      u64* O = cbv.out[s] + (size_t)b * cbv.out_bst + (size_t)p * cbv.out_pst + (size_t)r * N + k0;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const u32 e = j + 16 * k;
        u64 v = shoup_mul(sub_mod(A[e], tl[17 * k + j], qi), w, wp, qi);
        if (ADD) v = add_mod(v, ADD[ga == 1 ? (u32)k0 + e : galois_src((u32)k0 + e, ga, logN)], qi);
        O[e] = v;
      }
    } else {
      u64* a = blk(z) + (size_t)cc * 256;
#pragma unroll
      for (int k = 0; k < 16; ++k) a[j + 16 * k] = tl[17 * k + j];
    }
    __syncthreads();  // buf[cur] and the transpose tiles are free
    z = zn;
  }
}

template <bool HINT, int MINB>
__global__ void __launch_bounds__(128, MINB) ntt2_inv_chunks_f64(LimbMap map, const ModConsts* __restrict__ mc,
                                                             const ulonglong2* __restrict__ ctw, u32 logN) {
  __shared__ u64 tile[kChunksPerCta][16 * 17];
  __shared__ ulonglong2 twa[kChunksPerCta][16];
  const u32 r = blockIdx.y + map.r0, z = blockIdx.z + map.z0;
  if (limb_skipped2(map, r, z)) return;
  const u32 N = 1u << logN, N1 = N >> 8;
  const u32 mod = map.basis.mod_of(r + map.first_limb);
  const double q = (double)mc[mod].q, qinv = 1.0 / q;
  const FoldF C{0, 0, 0, 0};
  const int tid = threadIdx.x, cc = tid >> 4, j = tid & 15;
  const u32 g = blockIdx.x * kChunksPerCta + cc;
  u64* a = map.base + (size_t)z * map.poly_stride + (size_t)r * N + (size_t)g * 256;
  const ulonglong2* T = ctw + ((size_t)mod * N1 + g) * 256;
  u64* tl = tile[cc];
  const u64 pol = HINT ? keep_policy() : 0;
  u64 v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = ld_last<HINT>(&a[j + 16 * k]);
  ulonglong2 tb[15];
#pragma unroll
  for (int d = 0; d < 4; ++d)
#pragma unroll
    for (int b = 0; b < (8 >> d); ++b)
      tb[16 - (16 >> d) + b] = ld_tw<HINT>(&T[(128 >> d) - 1 + j * (8 >> d) + b], pol);
  if (j < 15) twa[cc][j] = ld_tw<HINT>(&T[j], pol);
#pragma unroll
  for (int k = 0; k < 16; ++k) tl[17 * k + j] = v[k];
  __syncwarp();
  double x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = u2d(tl[17 * j + k]);  // canonical input residues
  auto twB = [&](int d, int b) { return tb[16 - (16 >> d) + b]; };
  gs16_f64<0, false>(x, q, twB, C);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) tl[17 * j + k] = d_bits(x[k]);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = bits_d(tl[17 * k + j]);
  auto twA = [&](int d, int b) { return twa[cc][(8 >> d) - 1 + b]; };
  gs16_f64<0, false>(x, q, twA, C);
#pragma unroll
  for (int k = 0; k < 16; ++k) a[j + 16 * k] = d_bits(fcentre(x[k], q, qinv));  // |x| < 2^8 q -> centred, double bits
}

template <int LOGN1, bool HINT, int MINB>
__global__ void __launch_bounds__(256, MINB) ntt2_inv_cols_f64(LimbMap map, const ModConsts* __restrict__ mc,
                                                           const u64* __restrict__ itw, const u64* __restrict__ itwp,
                                                           u32 logN) {
  constexpr int N1 = 1 << LOGN1, T1 = N1 / 16, COLS = 256 / T1, NSA = LOGN1 - 4;
  __shared__ u64 tile[N1 * COLS];
  __shared__ ulonglong2 sw[N1];
  const u32 r = blockIdx.y + map.r0, z = blockIdx.z + map.z0;
  if (limb_skipped2(map, r, z)) return;
  const u32 N = 1u << logN, N2 = N >> LOGN1;
  const u32 mod = map.basis.mod_of(r + map.first_limb);
  const double q = (double)mc[mod].q, qinv = 1.0 / q;
  const FoldF C = fold_f64(mc[mod]);
  u64* a = map.base + (size_t)z * map.poly_stride + (size_t)r * N + blockIdx.x * COLS;
  const int tid = threadIdx.x, c = tid % COLS, j = tid / COLS;
  for (int i = tid; i < N1; i += 256) sw[i] = tw_f64(itw[(size_t)mod * N + i], itwp[(size_t)mod * N + i]);
  double x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = bits_d(ld_last<HINT>(&a[(size_t)(16 * j + k) * N2 + c]));
  __syncthreads();
  auto twB = [&](int d, int b) { return sw[(N1 >> (d + 1)) + j * (8 >> d) + b]; };
  auto twA = [&](int d, int b) { return sw[(8 >> d) + b]; };
  if (NSA == 0) {
    gs16_f64<0, true>(x, q, twB, C);
#pragma unroll
    for (int k = 0; k < 16; ++k) a[(size_t)(16 * j + k) * N2 + c] = d2u(fcanon(x[k], q, qinv));
  } else {
    gs16_f64<0, false>(x, q, twB, C);
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[(16 * j + k) * COLS + c] = d_bits(x[k]);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = bits_d(tile[(j + T1 * k) * COLS + c]);
    gs16_f64<4 - NSA, true>(x, q, twA, C);
#pragma unroll
    for (int k = 0; k < 16; ++k) a[(size_t)(j + T1 * k) * N2 + c] = d2u(fcanon(x[k], q, qinv));
  }
}

// ---------------------------------------------------------------------------
// Integer-pipe ceiling of the NTT: the same radix-16 register network
// (ct16, 32 butterflies per call, approximate-Shoup products) iterated on
// register-resident data with register twiddles -- no memory traffic, no
// shuffles.  Its butterfly rate is the roofline denominator of the NTT
// kernels ("int" bound, bench.py), measured on the box like the HBM peak.
// ---------------------------------------------------------------------------
template <bool FAST>
__global__ void __launch_bounds__(256) k_bfly_peak(u64* __restrict__ out, const ulonglong2* __restrict__ tws,
                                                   u64 q, int iters) {
  ulonglong2 tw[15];
#pragma unroll
  for (int i = 0; i < 15; ++i) tw[i] = tws[i];
  u64 x[16];
  const u64 t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = (t * 16 + k) % q;
  const u64 q2 = 4 * q;
  auto twf = [&](int d, int b) { return tw[(1 << d) - 1 + b]; };
  for (int it = 0; it < iters; ++it) ct16<0, FAST>(x, q, q2, twf);
  u64 acc = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) acc ^= x[k];
  out[t] = acc;
}

// FP64-quotient variants of the same network (probe only)
template <bool MAGIC>
__global__ void __launch_bounds__(256) k_bfly_peak_fp(u64* __restrict__ out, const ulonglong2* __restrict__ tws,
                                                      u64 q, int iters) {
  u64 tw[15];
  double wq[15];
#pragma unroll
  for (int i = 0; i < 15; ++i) {
    tw[i] = tws[i].x;
    wq[i] = (double)tws[i].x / (double)q;
  }
  u64 x[16];
  const u64 t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = (t * 16 + k) % q;
  const u64 q4 = 4 * q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const int h = 8 >> d;
#pragma unroll
      for (int b = 0; b < (1 << d); ++b)
#pragma unroll
        for (int r = 0; r < h; ++r)
          if (MAGIC) ct_bfly_fp2(x[2 * h * b + r], x[2 * h * b + r + h], tw[(1 << d) - 1 + b], wq[(1 << d) - 1 + b], q, q4);
          else ct_bfly_fp(x[2 * h * b + r], x[2 * h * b + r + h], tw[(1 << d) - 1 + b], wq[(1 << d) - 1 + b], q, q4);
    }
    // keep values bounded as in the real network (final reduction of each pass)
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = x[k] >= q4 ? x[k] - q4 : x[k];
  }
  u64 acc = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) acc ^= x[k];
  out[t] = acc;
}

// Pure FP64 network (probe): residues held as signed doubles, exact
// products by the FMA two-product (a*w = hi + lo), quotient by the magic
// round-to-integer constant, no integer ops in the butterfly.
__device__ __forceinline__ double f64_mulmod(double a, double w, double wq, double q) {
  const double C = 6755399441055744.0;  // 1.5 * 2^52
  const double hi = a * w;
  const double lo = fma(a, w, -hi);
  const double qe = fma(a, wq, C) - C;
  return fma(-qe, q, hi) + lo;
}
__global__ void __launch_bounds__(256) k_bfly_peak_f64(u64* __restrict__ out, const ulonglong2* __restrict__ tws,
                                                       u64 qi, int iters) {
  const double q = (double)qi;
  double tw[15], wq[15];
#pragma unroll
  for (int i = 0; i < 15; ++i) {
    tw[i] = (double)tws[i].x;
    wq[i] = (double)tws[i].x / q;
  }
  double x[16];
  const u64 t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = (double)((t * 16 + k) % qi);
  const double qinv = 1.0 / q, C = 6755399441055744.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const int h = 8 >> d;
#pragma unroll
      for (int b = 0; b < (1 << d); ++b)
#pragma unroll
        for (int r = 0; r < h; ++r) {
          double& X = x[2 * h * b + r];
          double& Y = x[2 * h * b + r + h];
          const double tt = f64_mulmod(Y, tw[(1 << d) - 1 + b], wq[(1 << d) - 1 + b], q);
          const double xx = X;
          X = xx + tt;
          Y = xx - tt;
        }
    }
    // centre every value once per 4 stages (the real network reduces per pass)
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] -= (fma(x[k], qinv, C) - C) * q;
  }
  u64 acc = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) acc ^= (u64)(long long)x[k];
  out[t] = acc;
}

// butterflies per second of k_bfly_peak (fast: q < 2^47 unreduced network)
int ntt_butterfly_peak(int fast, double* bfly_per_s) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const u64 q = fast >= 1 ? 1099511922689ull : 1152921504606584833ull;  // 40-bit / 60-bit NTT primes
  const int threads = 256, blocks = sms * 8, iters = 256;
  ulonglong2 h[15];
  for (int i = 0; i < 15; ++i) {
    const u64 w = (0x9E3779B97F4A7C15ull * (i + 1)) % q;
    h[i] = make_ulonglong2(w, (u64)((((unsigned __int128)w) << 64) / q));
  }
  u64* d_out = nullptr;
  ulonglong2* d_tw = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaError_t err = cudaMalloc(&d_out, (size_t)blocks * threads * 8);
  if (!err) err = cudaMalloc(&d_tw, sizeof(h));
  if (!err) err = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (!err) err = cudaMemcpyAsync(d_tw, h, sizeof(h), cudaMemcpyHostToDevice, st);
  if (!err) err = cudaEventCreate(&e0);
  if (!err) err = cudaEventCreate(&e1);
  float ms = 0.f;
  if (!err) {
    auto go = [&]() {
      if (fast == 4) k_bfly_peak_f64<<<blocks, threads, 0, st>>>(d_out, d_tw, q, iters);
      else if (fast == 3) k_bfly_peak_fp<true><<<blocks, threads, 0, st>>>(d_out, d_tw, q, iters);
      else if (fast == 2) k_bfly_peak_fp<false><<<blocks, threads, 0, st>>>(d_out, d_tw, q, iters);
      else if (fast) k_bfly_peak<true><<<blocks, threads, 0, st>>>(d_out, d_tw, q, iters);
      else k_bfly_peak<false><<<blocks, threads, 0, st>>>(d_out, d_tw, q, iters);
    };
    for (int w = 0; w < 3; ++w) go();  // warm-up (clocks ramp)
    cudaEventRecord(e0, st);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) go();
    cudaEventRecord(e1, st);
    err = cudaEventSynchronize(e1);
    if (!err) err = cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
  }
  if (!err) err = cudaGetLastError();
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (st) cudaStreamDestroy(st);
  cudaFree(d_out);
  cudaFree(d_tw);
  if (err) return (int)err;
  *bfly_per_s = (double)blocks * threads * iters * 32.0 / (ms * 1e-3);
  return 0;
}

// limbs transformed per class since the last read: [fwd fast, fwd full, inv fast, inv full]
unsigned long long g_ntt_limbs[4] = {0, 0, 0, 0};
std::atomic<unsigned long long> g_ntt_extra_launches{0};

static void count_limbs(const NttTables& T, const LimbMap& m, u32 ny, u32 nz, bool inverse) {
  for (u32 r = 0; r < ny; ++r) {
    const bool f = T.small && T.small[m.basis.mod_of(m.r0 + r + m.first_limb)] != 0;
    g_ntt_limbs[(inverse ? 2 : 0) + (f ? 0 : 1)] += nz;
  }
}

bool ntt2_supported(u32 logN) { return logN >= 12 && logN <= 16; }

template <int L, bool H, int OCC, int F>
static void launch_cols_t(bool inv, dim3 g, const LimbMap& map, const NttTables& T, cudaStream_t st) {
  if (inv) ntt2_inv_cols<L, H, OCC == 1 ? 3 : 1, F><<<g, 256, 0, st>>>(map, T.mc, T.itw, T.itwp, T.logN);
  else ntt2_fwd_cols<L, H, OCC == 1 ? 3 : 1, F><<<g, 256, 0, st>>>(map, T.mc, T.tw, T.twp, T.logN);
}

template <int L, bool H>
static void launch_cols_f64(bool inv, dim3 g, const LimbMap& map, const NttTables& T, cudaStream_t st) {
  if (inv) ntt2_inv_cols_f64<L, H, 1><<<g, 256, 0, st>>>(map, T.mc, T.itw, T.itwp, T.logN);
  else ntt2_fwd_cols_f64<L, H, 1><<<g, 256, 0, st>>>(map, T.mc, T.tw, T.twp, T.logN);
}

// FP64-network pass pair (class-2 moduli, both directions)
template <bool H>
static cudaError_t launch_pair_f64(const NttTables& T, const LimbMap& map, u32 ny, u32 nz, bool inverse,
                                   cudaStream_t st) {
  const u32 logN = T.logN, logN1 = logN - 8, N1 = 1u << logN1;
  const u32 cols = 256 / (N1 / 16);
  dim3 gc(256 / cols, ny, nz);
  dim3 gk(N1 / kChunksPerCta, ny, nz);
  auto cols_launch = [&](bool inv) -> bool {
    switch (logN1) {
      case 4: launch_cols_f64<4, H>(inv, gc, map, T, st); return true;
      case 5: launch_cols_f64<5, H>(inv, gc, map, T, st); return true;
      case 6: launch_cols_f64<6, H>(inv, gc, map, T, st); return true;
      case 7: launch_cols_f64<7, H>(inv, gc, map, T, st); return true;
      case 8: launch_cols_f64<8, H>(inv, gc, map, T, st); return true;
      default: return false;
    }
  };
  const int mb = g_ntt_tuning.f64_minb;
  if (!inverse && g_ntt_tuning.pipe) {
    if (!cols_launch(false)) return cudaErrorInvalidValue;
    // polys per CTA: enough CTAs for ~2 waves of 4 per SM, the rest pipelined
    const u32 want = 2u * 148u * 4u, per_z = gk.x * ny;
    u32 zsplit = (want + per_z - 1) / per_z;
    zsplit = zsplit < 1 ? 1 : (zsplit > nz ? nz : zsplit);
    const u32 zper = (nz + zsplit - 1) / zsplit;
    zsplit = (nz + zper - 1) / zper;
    const size_t sm = (2 * kChunkBlock + kChunksPerCta * 16 * 17) * 8;
    if (map.cb) {
      cudaError_t e = ensure_smem((const void*)ntt2_fwd_chunks_f64p<H, true>, sm);
      if (e) return e;
      ntt2_fwd_chunks_f64p<H, true><<<dim3(gk.x, ny, zsplit), 128, sm, st>>>(map, T.mc, T.ctw, logN, zper, nz, *map.cb);
    } else {
      cudaError_t e = ensure_smem((const void*)ntt2_fwd_chunks_f64p<H, false>, sm);
      if (e) return e;
      ntt2_fwd_chunks_f64p<H, false><<<dim3(gk.x, ny, zsplit), 128, sm, st>>>(map, T.mc, T.ctw, logN, zper, nz,
                                                                             NttCombine{});
    }
    return cudaGetLastError();
  }
  if (!inverse) {
    if (!cols_launch(false)) return cudaErrorInvalidValue;
    if (mb == 5) ntt2_fwd_chunks_f64<H, 5><<<gk, 128, 0, st>>>(map, T.mc, T.ctw, logN);
    else if (mb == 6) ntt2_fwd_chunks_f64<H, 6><<<gk, 128, 0, st>>>(map, T.mc, T.ctw, logN);
    else ntt2_fwd_chunks_f64<H, 1><<<gk, 128, 0, st>>>(map, T.mc, T.ctw, logN);
  } else {
    if (mb == 5) ntt2_inv_chunks_f64<H, 5><<<gk, 128, 0, st>>>(map, T.mc, T.ictw, logN);
    else if (mb == 6) ntt2_inv_chunks_f64<H, 6><<<gk, 128, 0, st>>>(map, T.mc, T.ictw, logN);
    else ntt2_inv_chunks_f64<H, 1><<<gk, 128, 0, st>>>(map, T.mc, T.ictw, logN);
    if (!cols_launch(true)) return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <bool H, int OCC, int F>
static cudaError_t launch_pair(const NttTables& T, const LimbMap& map, u32 ny, u32 nz, bool inverse,
                               cudaStream_t st) {
  if constexpr (F == 3) return launch_pair_f64<H>(T, map, ny, nz, inverse, st);
  const u32 logN = T.logN, logN1 = logN - 8, N1 = 1u << logN1;
  const u32 cols = 256 / (N1 / 16);
  dim3 gc(256 / cols, ny, nz);
  dim3 gk(N1 / kChunksPerCta, ny, nz);
  auto cols_launch = [&](bool inv) -> bool {
    switch (logN1) {
      case 4: launch_cols_t<4, H, OCC, F>(inv, gc, map, T, st); return true;
      case 5: launch_cols_t<5, H, OCC, F>(inv, gc, map, T, st); return true;
      case 6: launch_cols_t<6, H, OCC, F>(inv, gc, map, T, st); return true;
      case 7: launch_cols_t<7, H, OCC, F>(inv, gc, map, T, st); return true;
      case 8: launch_cols_t<8, H, OCC, F>(inv, gc, map, T, st); return true;
      default: return false;
    }
  };
  if (!inverse) {
    if (!cols_launch(false)) return cudaErrorInvalidValue;
    ntt2_fwd_chunks<H, OCC == 1 ? 5 : OCC == 2 ? 4 : 1, F><<<gk, 128, 0, st>>>(map, T.mc, T.ctw, logN);
  } else {
    ntt2_inv_chunks<H, OCC == 1 ? 5 : OCC == 2 ? 4 : 1, F><<<gk, 128, 0, st>>>(map, T.mc, T.ictw, logN);
    if (!cols_launch(true)) return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// The two passes of a batch run back to back on L2-sized groups of limbs so
// the intermediate between passes is re-read from L2, not HBM.
cudaError_t launch_ntt2(const NttTables& T, const LimbMap& map, u32 nlimbs, u32 npolys, bool inverse,
                        cudaStream_t st) {
  if (nlimbs == 0 || npolys == 0) return cudaSuccess;
  const bool hint = g_ntt_tuning.hints != 0;
  const bool occ = g_ntt_tuning.occupancy == 1;
  // split: one launch pair per run of limbs of one modulus class (uniform
  // kernels); otherwise one launch pair dispatching per limb at run time
  // split 1: per-class launches both directions, 2: forward only (the
  // forward variants differ -- FP64 vs integer quotient -- so per-class
  // kernels are smaller; the inverse keeps one run-time-dispatch launch)
  // FP64-network moduli (class 2) always launch their own kernels: their
  // chunk twiddles are stored as doubles
  const bool split = g_ntt_tuning.split == 1 || (g_ntt_tuning.split == 2 && !inverse) ||
                     (kNttFp && T.small != nullptr);
  auto one = [&](const LimbMap& m, u32 ny, u32 nz, int mode, cudaStream_t s) -> cudaError_t {
    if (mode == 0) return g_ntt_tuning.occupancy == 2 ? launch_pair<true, 2, 0>(T, m, ny, nz, inverse, s)
                          : occ ? launch_pair<true, 1, 0>(T, m, ny, nz, inverse, s)
                                : launch_pair<true, 0, 0>(T, m, ny, nz, inverse, s);
    if (mode == 1) return occ ? launch_pair<true, 1, 1>(T, m, ny, nz, inverse, s)
                              : launch_pair<true, 0, 1>(T, m, ny, nz, inverse, s);
    // occupancy 2: chunk pass capped at 128 registers (4 CTAs of 128 threads per SM), cols unchanged
    if (mode == 3) return g_ntt_tuning.occupancy == 2 ? launch_pair<true, 2, 3>(T, m, ny, nz, inverse, s)
                                                      : launch_pair<true, 0, 3>(T, m, ny, nz, inverse, s);
    return occ ? launch_pair<true, 1, 2>(T, m, ny, nz, inverse, s) : launch_pair<true, 0, 2>(T, m, ny, nz, inverse, s);
  };
  auto pair = [&](const LimbMap& m, u32 ny, u32 nz) -> cudaError_t {
    if (!split || !T.small) {
      LimbMap mm = m;
      mm.cb = nullptr;
      cudaError_t err = one(mm, ny, nz, 2, st);
      if (!err && m.cb) {
        err = launch_combine_rows(*m.cb, m.base, m.basis.nq, m.r0 + m.first_limb, ny, nz, T.logN, T.mc, st);
        g_ntt_extra_launches += 1;
      }
      return err;
    }
    u32 r = 0;
    // launch class of a limb: the FP64 network (class 2) always alone; the
    // integer classes merge into one run-time-dispatch inverse unless split == 1
    auto cls = [&](u32 rr) -> int {
      const int f = T.small[m.basis.mod_of(m.r0 + rr + m.first_limb)];
      if (f == 2 && kNttFp) return 2;
      return inverse && g_ntt_tuning.split != 1 ? -1 : f;
    };
    // a mix of FP64-network and integer-network runs: the integer runs (q0's
    // single limb, the specials: small, latency-bound launches) go to the
    // side stream, forked before the first launch and joined after the last,
    // so they overlap the FP64 run instead of serialising behind it
    bool has_fp = false, has_int = false;
    for (u32 rr = 0; rr < ny; ++rr) (cls(rr) == 2 ? has_fp : has_int) = true;
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    std::mutex* fmu = nullptr;
    const bool par = g_ntt_tuning.fork && has_fp && has_int &&
                     side_stream(&side, &fork, &join, &fmu) == cudaSuccess;
    std::unique_lock<std::mutex> flk;
    if (par) {
      flk = std::unique_lock<std::mutex>(*fmu);
      cudaError_t e0 = cudaEventRecord(fork, st);
      if (!e0) e0 = cudaStreamWaitEvent(side, fork, 0);
      if (e0) return e0;
    }
    cudaError_t err = cudaSuccess;
    while (r < ny && !err) {
      const int f = cls(r);
      u32 e = r + 1;
      while (e < ny && cls(e) == f) ++e;
      LimbMap mm = m;
      mm.r0 = m.r0 + r;
      // class 2: the FP64 network both ways; other classes keep one
      // run-time-dispatch inverse launch unless split == 1
      const int mode = f == 2 ? 3 : f < 0 ? 2 : f;
      const cudaStream_t rs = par && mode != 3 ? side : st;
      // the fused ModDown combine runs inside the FP64 pipelined chunk pass;
      // integer-network rows get a plain NTT and the combine kernel after it
      const bool fuse_here = mm.cb && mode == 3 && !inverse && g_ntt_tuning.pipe;
      const NttCombine* cb = mm.cb;
      if (!fuse_here) mm.cb = nullptr;
      err = one(mm, e - r, nz, mode, rs);
      if (!err && cb && !fuse_here) {
        err = launch_combine_rows(*cb, m.base, m.basis.nq, mm.r0 + m.first_limb, e - r, nz, T.logN, T.mc, rs);
        g_ntt_extra_launches += 1;
      }
      if (r > 0) g_ntt_extra_launches += 2;  // launch accounting counts one pair per call
      r = e;
    }
    if (par) {  // join even after an error: the capture must not end with an open fork
      cudaError_t e2 = cudaEventRecord(join, side);
      if (!e2) e2 = cudaStreamWaitEvent(st, join, 0);
      if (!err) err = e2;
    }
    return err;
  };
  (void)hint;
  count_limbs(T, map, nlimbs, npolys, inverse);
  const u32 G = g_ntt_tuning.group_limbs > 0 ? (u32)g_ntt_tuning.group_limbs : 0;
  if (G == 0 || nlimbs * npolys <= G) return pair(map, nlimbs, npolys);
  cudaError_t e = cudaSuccess;
  if (nlimbs <= G) {
    const u32 gp = G / nlimbs;
    for (u32 z0 = 0; z0 < npolys && !e; z0 += gp) {
      LimbMap m = map;
      m.z0 = map.z0 + z0;
      e = pair(m, nlimbs, npolys - z0 < gp ? npolys - z0 : gp);
    }
  } else {
    for (u32 z = 0; z < npolys && !e; ++z)
      for (u32 r0 = 0; r0 < nlimbs && !e; r0 += G) {
        LimbMap m = map;
        m.z0 = map.z0 + z;
        m.r0 = map.r0 + r0;
        e = pair(m, nlimbs - r0 < G ? nlimbs - r0 : G, 1);
      }
  }
  return e;
}

}  // namespace hcnn
