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
#include "common.cuh"
#include "kernels.cuh"

namespace hcnn {

__device__ __forceinline__ void ct_bfly(u64& X, u64& Y, u64 w, u64 wp, u64 q, u64 q2) {
  u64 x = X >= q2 ? X - q2 : X;
  u64 t = shoup_lazy(Y, w, wp, q);
  X = x + t;
  Y = x - t + q2;
}

__device__ __forceinline__ void gs_bfly(u64& X, u64& Y, u64 w, u64 wp, u64 q, u64 q2) {
  u64 s = X + Y;
  s = s >= q2 ? s - q2 : s;
  u64 t = X - Y + q2;
  X = s;
  Y = shoup_lazy(t, w, wp, q);
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

// CT stages d in [D0,4)
template <int D0, class TW>
__device__ __forceinline__ void ct16(u64 (&x)[16], u64 q, u64 q2, TW tw) {
  if constexpr (D0 <= 0) ct_stage<0>(x, q, q2, tw);
  if constexpr (D0 <= 1) ct_stage<1>(x, q, q2, tw);
  if constexpr (D0 <= 2) ct_stage<2>(x, q, q2, tw);
  if constexpr (D0 <= 3) ct_stage<3>(x, q, q2, tw);
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

// GS stages d in [D0,4).  FOLD: stage 3 is the transform's last one
// (twiddle itw[1]) and also applies N^-1.
template <int D0, bool FOLD, class TW>
__device__ __forceinline__ void gs16(u64 (&x)[16], u64 q, u64 q2, TW tw, Fold C) {
  if constexpr (D0 <= 0) gs_stage<0>(x, q, q2, tw);
  if constexpr (D0 <= 1) gs_stage<1>(x, q, q2, tw);
  if constexpr (D0 <= 2) gs_stage<2>(x, q, q2, tw);
  if constexpr (FOLD) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      u64 s = x[r] + x[r + 8];
      u64 t = x[r] - x[r + 8] + q2;
      x[r] = shoup_mul(s, C.ninvN, C.ninvN_sh, q);
      x[r + 8] = shoup_mul(t, C.ilast, C.ilast_sh, q);
    }
  } else {
    gs_stage<3>(x, q, q2, tw);
  }
}

__device__ __forceinline__ bool limb_skipped2(const LimbMap& m, u32 r, u32 z) {
  if (m.skip_alpha == 0) return false;
  r += m.first_limb;
  u32 lo = z * m.skip_alpha;
  u32 hi = lo + m.skip_alpha;
  if (hi > m.basis.nq) hi = m.basis.nq;
  return r >= lo && r < hi;
}

// ---------------------------------------------------------------------------
// column pass (N1 = 2^LOGN1 points, 16 <= N1 <= 256), 256 threads,
// COLS = 256/T1 columns per CTA, T1 = N1/16 threads per column
// ---------------------------------------------------------------------------
template <int LOGN1>
__global__ void __launch_bounds__(256) ntt2_fwd_cols(LimbMap map, const ModConsts* __restrict__ mc,
                                                     const u64* __restrict__ tw, const u64* __restrict__ twp,
                                                     u32 logN) {
  constexpr int N1 = 1 << LOGN1, T1 = N1 / 16, COLS = 256 / T1, NSB = LOGN1 - 4;
  __shared__ u64 tile[N1 * COLS];
  __shared__ ulonglong2 sw[N1];
  const u32 r = blockIdx.y, z = blockIdx.z;
  if (limb_skipped2(map, r, z)) return;
  const u32 N = 1u << logN, N2 = N >> LOGN1;
  const u32 mod = map.basis.mod_of(r + map.first_limb);
  const u64 q = mc[mod].q, q2 = mc[mod].two_q;
  u64* a = map.base + (size_t)z * map.poly_stride + (size_t)r * N + blockIdx.x * COLS;
  const int tid = threadIdx.x, c = tid % COLS, j = tid / COLS;
  for (int i = tid; i < N1; i += 256) sw[i] = make_ulonglong2(tw[(size_t)mod * N + i], twp[(size_t)mod * N + i]);
  u64 x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = a[(size_t)(j + T1 * k) * N2 + c];
  __syncthreads();
  ct16<0>(x, q, q2, [&](int d, int b) { return sw[(1 << d) + b]; });
  if (NSB > 0) {
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[(j + T1 * k) * COLS + c] = x[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = tile[(16 * j + k) * COLS + c];
    ct16<4 - NSB>(x, q, q2, [&](int d, int b) { return sw[(1 << (d + NSB)) + (j << d) + b]; });
#pragma unroll
    for (int k = 0; k < 16; ++k) a[(size_t)(16 * j + k) * N2 + c] = x[k];
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k) a[(size_t)(j + T1 * k) * N2 + c] = x[k];
  }
}

template <int LOGN1>
__global__ void __launch_bounds__(256) ntt2_inv_cols(LimbMap map, const ModConsts* __restrict__ mc,
                                                     const u64* __restrict__ itw, const u64* __restrict__ itwp,
                                                     u32 logN) {
  constexpr int N1 = 1 << LOGN1, T1 = N1 / 16, COLS = 256 / T1, NSA = LOGN1 - 4;
  __shared__ u64 tile[N1 * COLS];
  __shared__ ulonglong2 sw[N1];
  const u32 r = blockIdx.y, z = blockIdx.z;
  if (limb_skipped2(map, r, z)) return;
  const u32 N = 1u << logN, N2 = N >> LOGN1;
  const u32 mod = map.basis.mod_of(r + map.first_limb);
  const u64 q = mc[mod].q, q2 = mc[mod].two_q;
  const Fold C{mc[mod].ninvN, mc[mod].ninvN_sh, mc[mod].ilast, mc[mod].ilast_sh};
  u64* a = map.base + (size_t)z * map.poly_stride + (size_t)r * N + blockIdx.x * COLS;
  const int tid = threadIdx.x, c = tid % COLS, j = tid / COLS;
  for (int i = tid; i < N1; i += 256) sw[i] = make_ulonglong2(itw[(size_t)mod * N + i], itwp[(size_t)mod * N + i]);
  u64 x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = a[(size_t)(16 * j + k) * N2 + c];
  __syncthreads();
  // stages t = 1..8 rows: contiguous groups of 16 rows; twiddle itw[H + i],
  // H = N1 >> (d+1) blocks, i = j*(8>>d) + b
  if (NSA == 0) {
    gs16<0, true>(x, q, q2, [&](int d, int b) { return sw[(N1 >> (d + 1)) + j * (8 >> d) + b]; }, C);
#pragma unroll
    for (int k = 0; k < 16; ++k) a[(size_t)(16 * j + k) * N2 + c] = x[k];
  } else {
    gs16<0, false>(x, q, q2, [&](int d, int b) { return sw[(N1 >> (d + 1)) + j * (8 >> d) + b]; }, C);
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[(16 * j + k) * COLS + c] = x[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = tile[(j + T1 * k) * COLS + c];
    gs16<4 - NSA, true>(x, q, q2, [&](int d, int b) { return sw[(8 >> d) + b]; }, C);
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

__global__ void __launch_bounds__(128) ntt2_fwd_chunks(LimbMap map, const ModConsts* __restrict__ mc,
                                                       const ulonglong2* __restrict__ ctw, u32 logN) {
  __shared__ u64 tile[kChunksPerCta][16 * 17];
  __shared__ ulonglong2 twa[kChunksPerCta][16];
  const u32 r = blockIdx.y, z = blockIdx.z;
  if (limb_skipped2(map, r, z)) return;
  const u32 N = 1u << logN, N1 = N >> 8;
  const u32 mod = map.basis.mod_of(r + map.first_limb);
  const u64 q = mc[mod].q, q2 = mc[mod].two_q;
  const int tid = threadIdx.x, cc = tid >> 4, j = tid & 15;
  const u32 g = blockIdx.x * kChunksPerCta + cc;
  u64* a = map.base + (size_t)z * map.poly_stride + (size_t)r * N + (size_t)g * 256;
  const ulonglong2* T = ctw + ((size_t)mod * N1 + g) * 256;
  u64* tl = tile[cc];
  u64 x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = a[j + 16 * k];
  if (j < 15) twa[cc][j] = __ldg(&T[j]);
  // second-group twiddles: stage 4+d, block (j<<d)+b -> e = (16<<d)-1+(j<<d)+b
  ulonglong2 tb[15];
#pragma unroll
  for (int d = 0; d < 4; ++d)
#pragma unroll
    for (int b = 0; b < (1 << d); ++b) tb[(1 << d) - 1 + b] = __ldg(&T[(16 << d) - 1 + (j << d) + b]);
  __syncwarp();
  ct16<0>(x, q, q2, [&](int d, int b) { return twa[cc][(1 << d) - 1 + b]; });
#pragma unroll
  for (int k = 0; k < 16; ++k) tl[17 * k + j] = x[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = tl[17 * j + k];
  ct16<0>(x, q, q2, [&](int d, int b) { return tb[(1 << d) - 1 + b]; });
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    u64 v = x[k];
    v = v >= q2 ? v - q2 : v;
    x[k] = v >= q ? v - q : v;
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) tl[17 * j + k] = x[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) a[j + 16 * k] = tl[17 * k + j];
}

__global__ void __launch_bounds__(128) ntt2_inv_chunks(LimbMap map, const ModConsts* __restrict__ mc,
                                                       const ulonglong2* __restrict__ ctw, u32 logN) {
  __shared__ u64 tile[kChunksPerCta][16 * 17];
  __shared__ ulonglong2 twa[kChunksPerCta][16];
  const u32 r = blockIdx.y, z = blockIdx.z;
  if (limb_skipped2(map, r, z)) return;
  const u32 N = 1u << logN, N1 = N >> 8;
  const u32 mod = map.basis.mod_of(r + map.first_limb);
  const u64 q = mc[mod].q, q2 = mc[mod].two_q;
  const Fold C{0, 0, 0, 0};
  const int tid = threadIdx.x, cc = tid >> 4, j = tid & 15;
  const u32 g = blockIdx.x * kChunksPerCta + cc;
  u64* a = map.base + (size_t)z * map.poly_stride + (size_t)r * N + (size_t)g * 256;
  const ulonglong2* T = ctw + ((size_t)mod * N1 + g) * 256;
  u64* tl = tile[cc];
  u64 x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = a[j + 16 * k];
  // first group (local stages 0..3): nb = 128>>d blocks, i = j*(8>>d)+b
  ulonglong2 tb[15];
#pragma unroll
  for (int d = 0; d < 4; ++d)
#pragma unroll
    for (int b = 0; b < (8 >> d); ++b) tb[16 - (16 >> d) + b] = __ldg(&T[(128 >> d) - 1 + j * (8 >> d) + b]);
  // second group (local stages 4..7): nb = 8>>d, i = b -> e = (8>>d)-1+b, shared
  if (j < 15) twa[cc][j] = __ldg(&T[j]);
#pragma unroll
  for (int k = 0; k < 16; ++k) tl[17 * k + j] = x[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = tl[17 * j + k];
  gs16<0, false>(x, q, q2, [&](int d, int b) { return tb[16 - (16 >> d) + b]; }, C);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) tl[17 * j + k] = x[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = tl[17 * k + j];
  gs16<0, false>(x, q, q2, [&](int d, int b) { return twa[cc][(8 >> d) - 1 + b]; }, C);
#pragma unroll
  for (int k = 0; k < 16; ++k) a[j + 16 * k] = x[k];
}

// ---------------------------------------------------------------------------
bool ntt2_supported(u32 logN) { return logN >= 12 && logN <= 16; }

template <int L>
static void launch_cols(bool inv, dim3 g, const LimbMap& map, const NttTables& T, cudaStream_t st) {
  if (inv) ntt2_inv_cols<L><<<g, 256, 0, st>>>(map, T.mc, T.itw, T.itwp, T.logN);
  else ntt2_fwd_cols<L><<<g, 256, 0, st>>>(map, T.mc, T.tw, T.twp, T.logN);
}

cudaError_t launch_ntt2(const NttTables& T, const LimbMap& map, u32 nlimbs, u32 npolys, bool inverse,
                        cudaStream_t st) {
  if (nlimbs == 0 || npolys == 0) return cudaSuccess;
  const u32 logN = T.logN, logN1 = logN - 8, N1 = 1u << logN1;
  const u32 cols = 256 / (N1 / 16);
  dim3 gc(256 / cols, nlimbs, npolys);
  dim3 gk(N1 / kChunksPerCta, nlimbs, npolys);
  if (!inverse) {
    switch (logN1) {
      case 4: launch_cols<4>(false, gc, map, T, st); break;
      case 5: launch_cols<5>(false, gc, map, T, st); break;
      case 6: launch_cols<6>(false, gc, map, T, st); break;
      case 7: launch_cols<7>(false, gc, map, T, st); break;
      case 8: launch_cols<8>(false, gc, map, T, st); break;
      default: return cudaErrorInvalidValue;
    }
    ntt2_fwd_chunks<<<gk, 128, 0, st>>>(map, T.mc, T.ctw, logN);
  } else {
    ntt2_inv_chunks<<<gk, 128, 0, st>>>(map, T.mc, T.ictw, logN);
    switch (logN1) {
      case 4: launch_cols<4>(true, gc, map, T, st); break;
      case 5: launch_cols<5>(true, gc, map, T, st); break;
      case 6: launch_cols<6>(true, gc, map, T, st); break;
      case 7: launch_cols<7>(true, gc, map, T, st); break;
      case 8: launch_cols<8>(true, gc, map, T, st); break;
      default: return cudaErrorInvalidValue;
    }
  }
  return cudaGetLastError();
}

}  // namespace hcnn
