// Negacyclic NTT / inverse NTT for sm_100a.
//
// Contract (reference kernels.py:232-281 / ring.py:317-336):
// forward output index k holds a(psi^(2*brv(k)+1)) mod q, fully reduced, for
// the reference's psi (smallest generator r in [2,1000), ring.py:160-167);
// inverse is the exact inverse including the N^-1 scaling.
//
// Structure: N = N1 * N2.  The Cooley-Tukey network's first log2(N1) stages
// only pair elements N2 or more apart, so they run as N1-point networks down
// "columns" (pass 1, k*N2 + col); the remaining log2(N2) stages run inside
// contiguous chunks of N2 (pass 2).  The inverse (Gentleman-Sande) runs the
// same two passes in the opposite order.  Each pass stages its tile in shared
// memory; butterflies are Harvey-lazy (values in [0,4q) forward / [0,2q)
// inverse between stages, q < 2^62) with Shoup twiddle products, and the
// final pass reduces to [0,q).  Small rings (N <= 4096) run a single pass.
#include "common.cuh"
#include "kernels.cuh"

namespace hcnn {

__device__ __forceinline__ bool limb_skipped(const LimbMap& m, u32 r, u32 z) {
  if (m.skip_alpha == 0) return false;
  r += m.first_limb;
  if (m.zmod) z %= m.zmod;
  u32 lo = z * m.skip_alpha;
  u32 hi = lo + m.skip_alpha;
  if (hi > m.basis.nq) hi = m.basis.nq;
  return r >= lo && r < hi;
}

// ---------------------------------------------------------------------------
// forward, pass 1: N1-point CT networks over COLS adjacent columns
// ---------------------------------------------------------------------------
template <int COLS>
__global__ void __launch_bounds__(256) ntt_fwd_cols(LimbMap map, const ModConsts* __restrict__ mc,
                                                    const u64* __restrict__ tw, const u64* __restrict__ twp,
                                                    u32 logN, u32 logN1) {
  extern __shared__ u64 sm[];
  const u32 r = blockIdx.y + map.r0, z = blockIdx.z + map.z0;
  if (limb_skipped(map, r, z)) return;
  const u32 N = 1u << logN, N1 = 1u << logN1, N2 = N >> logN1;
  const u32 mod = map.basis.mod_of(r + map.first_limb);
  const u64 q = mc[mod].q, q2 = mc[mod].two_q;
  u64* a = map.base + (size_t)z * map.poly_stride + (size_t)r * N;
  const u32 col0 = blockIdx.x * COLS;
  u64* s_w = sm + N1 * COLS;
  u64* s_wp = s_w + N1;
  const u64* twm = tw + (size_t)mod * N;
  const u64* twpm = twp + (size_t)mod * N;
  for (u32 j = threadIdx.x; j < N1; j += blockDim.x) {
    s_w[j] = twm[j];
    s_wp[j] = twpm[j];
  }
  for (u32 idx = threadIdx.x; idx < N1 * COLS; idx += blockDim.x) {
    u32 k = idx / COLS, c = idx % COLS;
    sm[idx] = a[(size_t)k * N2 + col0 + c];
  }
  __syncthreads();
  const u32 nb = (N1 / 2) * COLS;
  for (u32 s = 0; s < logN1; ++s) {
    const u32 lh = logN1 - 1 - s;  // log2(half)
    for (u32 b = threadIdx.x; b < nb; b += blockDim.x) {
      u32 c = b % COLS, p = b / COLS;
      u32 i = p >> lh, rr = p & ((1u << lh) - 1);
      u32 k1 = (i << (lh + 1)) + rr, k2 = k1 + (1u << lh);
      u64 w = s_w[(1u << s) + i], wp = s_wp[(1u << s) + i];
      u64 X = sm[k1 * COLS + c], Y = sm[k2 * COLS + c];
      X = X >= q2 ? X - q2 : X;
      u64 T = shoup_lazy(Y, w, wp, q);
      sm[k1 * COLS + c] = X + T;
      sm[k2 * COLS + c] = X - T + q2;
    }
    __syncthreads();
  }
  for (u32 idx = threadIdx.x; idx < N1 * COLS; idx += blockDim.x) {
    u32 k = idx / COLS, c = idx % COLS;
    a[(size_t)k * N2 + col0 + c] = sm[idx];
  }
}

// ---------------------------------------------------------------------------
// forward, pass 2 (or the whole transform when N1 == 1): chunks of M=N2
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) ntt_fwd_chunks(LimbMap map, const ModConsts* __restrict__ mc,
                                                      const u64* __restrict__ tw, const u64* __restrict__ twp,
                                                      u32 logN, u32 logN1, u32 CH) {
  extern __shared__ u64 sm[];
  const u32 r = blockIdx.y + map.r0, z = blockIdx.z + map.z0;
  if (limb_skipped(map, r, z)) return;
  const u32 N = 1u << logN, N1 = 1u << logN1;
  const u32 logM = logN - logN1, M = 1u << logM;
  const u32 mod = map.basis.mod_of(r + map.first_limb);
  const u64 q = mc[mod].q, q2 = mc[mod].two_q;
  u64* a = map.base + (size_t)z * map.poly_stride + (size_t)r * N;
  const u32 g0 = blockIdx.x * CH;  // first global chunk
  const u64* twm = tw + (size_t)mod * N;
  const u64* twpm = twp + (size_t)mod * N;
  const u32 tot = CH * M;
  u64* ag = a + (size_t)g0 * M;
  for (u32 idx = threadIdx.x; idx < tot; idx += blockDim.x) sm[idx] = ag[idx];
  __syncthreads();
  const u32 nb = tot / 2;
  for (u32 s = 0; s < logM; ++s) {
    const u32 lh = logM - 1 - s;
    for (u32 b = threadIdx.x; b < nb; b += blockDim.x) {
      u32 c = b >> (logM - 1), p = b & ((M >> 1) - 1);
      u32 i = p >> lh, rr = p & ((1u << lh) - 1);
      u32 k1 = c * M + (i << (lh + 1)) + rr, k2 = k1 + (1u << lh);
      u32 widx = ((N1 + g0 + c) << s) + i;
      u64 w = twm[widx], wp = twpm[widx];
      u64 X = sm[k1], Y = sm[k2];
      X = X >= q2 ? X - q2 : X;
      u64 T = shoup_lazy(Y, w, wp, q);
      sm[k1] = X + T;
      sm[k2] = X - T + q2;
    }
    __syncthreads();
  }
  for (u32 idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    u64 x = sm[idx];
    x = x >= q2 ? x - q2 : x;
    x = x >= q ? x - q : x;
    ag[idx] = x;
  }
}

// ---------------------------------------------------------------------------
// inverse, pass 1 (or whole transform when N1 == 1): GS inside chunks of M
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) ntt_inv_chunks(LimbMap map, const ModConsts* __restrict__ mc,
                                                      const u64* __restrict__ itw, const u64* __restrict__ itwp,
                                                      u32 logN, u32 logN1, u32 CH) {
  extern __shared__ u64 sm[];
  const u32 r = blockIdx.y + map.r0, z = blockIdx.z + map.z0;
  if (limb_skipped(map, r, z)) return;
  const u32 N = 1u << logN, N1 = 1u << logN1;
  const u32 logM = logN - logN1, M = 1u << logM;
  const u32 mod = map.basis.mod_of(r + map.first_limb);
  const ModConsts C = mc[mod];
  const u64 q = C.q, q2 = C.two_q;
  u64* a = map.base + (size_t)z * map.poly_stride + (size_t)r * N;
  const u32 g0 = blockIdx.x * CH;
  const u64* twm = itw + (size_t)mod * N;
  const u64* twpm = itwp + (size_t)mod * N;
  const u32 tot = CH * M;
  u64* ag = a + (size_t)g0 * M;
  for (u32 idx = threadIdx.x; idx < tot; idx += blockDim.x) sm[idx] = ag[idx];
  __syncthreads();
  const u32 nb = tot / 2;
  for (u32 u = 0; u < logM; ++u) {
    const u32 lhl = logM - 1 - u;  // log2(h_local)
    for (u32 b = threadIdx.x; b < nb; b += blockDim.x) {
      u32 c = b >> (logM - 1), p = b & ((M >> 1) - 1);
      u32 i = p >> u, rr = p & ((1u << u) - 1);
      u32 k1 = c * M + (i << (u + 1)) + rr, k2 = k1 + (1u << u);
      u32 widx = ((N1 + g0 + c) << lhl) + i;
      u64 w = twm[widx], wp = twpm[widx];
      u64 X = sm[k1], Y = sm[k2];
      u64 S = X + Y;
      S = S >= q2 ? S - q2 : S;
      u64 T = X - Y + q2;
      sm[k1] = S;
      sm[k2] = shoup_lazy(T, w, wp, q);
    }
    __syncthreads();
  }
  if (N1 == 1) {
    for (u32 idx = threadIdx.x; idx < tot; idx += blockDim.x)
      ag[idx] = shoup_mul(sm[idx], C.ninvN, C.ninvN_sh, q);
  } else {
    for (u32 idx = threadIdx.x; idx < tot; idx += blockDim.x) ag[idx] = sm[idx];
  }
}

// ---------------------------------------------------------------------------
// inverse, pass 2: N1-point GS networks over columns, N^-1 folded into the
// last stage
// ---------------------------------------------------------------------------
template <int COLS>
__global__ void __launch_bounds__(256) ntt_inv_cols(LimbMap map, const ModConsts* __restrict__ mc,
                                                    const u64* __restrict__ itw, const u64* __restrict__ itwp,
                                                    u32 logN, u32 logN1) {
  extern __shared__ u64 sm[];
  const u32 r = blockIdx.y + map.r0, z = blockIdx.z + map.z0;
  if (limb_skipped(map, r, z)) return;
  const u32 N = 1u << logN, N1 = 1u << logN1, N2 = N >> logN1;
  const u32 mod = map.basis.mod_of(r + map.first_limb);
  const ModConsts C = mc[mod];
  const u64 q = C.q, q2 = C.two_q;
  u64* a = map.base + (size_t)z * map.poly_stride + (size_t)r * N;
  const u32 col0 = blockIdx.x * COLS;
  u64* s_w = sm + N1 * COLS;
  u64* s_wp = s_w + N1;
  const u64* twm = itw + (size_t)mod * N;
  const u64* twpm = itwp + (size_t)mod * N;
  for (u32 j = threadIdx.x; j < N1; j += blockDim.x) {
    s_w[j] = twm[j];
    s_wp[j] = twpm[j];
  }
  for (u32 idx = threadIdx.x; idx < N1 * COLS; idx += blockDim.x) {
    u32 k = idx / COLS, c = idx % COLS;
    sm[idx] = a[(size_t)k * N2 + col0 + c];
  }
  __syncthreads();
  const u32 nb = (N1 / 2) * COLS;
  for (u32 u = 0; u + 1 < logN1; ++u) {
    const u32 lh = logN1 - 1 - u;  // log2(h)
    for (u32 b = threadIdx.x; b < nb; b += blockDim.x) {
      u32 c = b % COLS, p = b / COLS;
      u32 i = p >> u, rr = p & ((1u << u) - 1);
      u32 k1 = (i << (u + 1)) + rr, k2 = k1 + (1u << u);
      u64 w = s_w[(1u << lh) + i], wp = s_wp[(1u << lh) + i];
      u64 X = sm[k1 * COLS + c], Y = sm[k2 * COLS + c];
      u64 S = X + Y;
      S = S >= q2 ? S - q2 : S;
      u64 T = X - Y + q2;
      sm[k1 * COLS + c] = S;
      sm[k2 * COLS + c] = shoup_lazy(T, w, wp, q);
    }
    __syncthreads();
  }
  {  // last stage: h = 1, t = N1/2, twiddle itw[1]; scale by N^-1
    const u32 u = logN1 - 1;
    for (u32 b = threadIdx.x; b < nb; b += blockDim.x) {
      u32 c = b % COLS, p = b / COLS;
      u32 k1 = p, k2 = p + (1u << u);
      u64 X = sm[k1 * COLS + c], Y = sm[k2 * COLS + c];
      u64 S = X + Y;  // < 4q
      u64 T = X - Y + q2;
      sm[k1 * COLS + c] = shoup_mul(S, C.ninvN, C.ninvN_sh, q);
      sm[k2 * COLS + c] = shoup_mul(T, C.ilast, C.ilast_sh, q);
    }
    __syncthreads();
  }
  for (u32 idx = threadIdx.x; idx < N1 * COLS; idx += blockDim.x) {
    u32 k = idx / COLS, c = idx % COLS;
    a[(size_t)k * N2 + col0 + c] = sm[idx];
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static const int kCols = 16;
static const u32 kChunkElems = 2048;

void ntt_split(u32 logN, u32* logN1) {
  *logN1 = logN <= 12 ? 0 : logN / 2;
}

cudaError_t launch_ntt(const NttTables& T, const LimbMap& map, u32 nlimbs, u32 npolys, bool inverse,
                       cudaStream_t st) {
  if (nlimbs == 0 || npolys == 0) return cudaSuccess;
  if (T.ctw) return launch_ntt2(T, map, nlimbs, npolys, inverse, st);
  if (map.cb) {  // small rings: plain NTT, then the ModDown combine kernel
    LimbMap m = map;
    m.cb = nullptr;
    cudaError_t e = launch_ntt(T, m, nlimbs, npolys, inverse, st);
    if (e) return e;
    return launch_combine_rows(*map.cb, map.base, map.basis.nq, map.r0 + map.first_limb, nlimbs, npolys, T.logN,
                               T.mc, st);
  }
  u32 logN = T.logN, logN1;
  ntt_split(logN, &logN1);
  const u32 N = 1u << logN;
  const u32 M = N >> logN1;
  u32 CH = (logN1 == 0) ? 1 : (kChunkElems / M > 0 ? kChunkElems / M : 1);
  if (CH > (1u << logN1)) CH = 1u << logN1;
  dim3 gchunk((1u << logN1) / CH, nlimbs, npolys);
  size_t smem_chunk = (size_t)CH * M * sizeof(u64);
  dim3 gcols(M / kCols, nlimbs, npolys);
  size_t smem_cols = ((size_t)(1u << logN1) * kCols + 2 * (1u << logN1)) * sizeof(u64);
  if (!inverse) {
    if (logN1 > 0) {
      ntt_fwd_cols<kCols><<<gcols, 256, smem_cols, st>>>(map, T.mc, T.tw, T.twp, logN, logN1);
    }
    ntt_fwd_chunks<<<gchunk, 256, smem_chunk, st>>>(map, T.mc, T.tw, T.twp, logN, logN1, CH);
  } else {
    ntt_inv_chunks<<<gchunk, 256, smem_chunk, st>>>(map, T.mc, T.itw, T.itwp, logN, logN1, CH);
    if (logN1 > 0) {
      ntt_inv_cols<kCols><<<gcols, 256, smem_cols, st>>>(map, T.mc, T.itw, T.itwp, logN, logN1);
    }
  }
  return cudaGetLastError();
}

cudaError_t ntt_configure_smem() {
  cudaError_t e;
  e = cudaFuncSetAttribute(ntt_fwd_chunks, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  if (e) return e;
  e = cudaFuncSetAttribute(ntt_inv_chunks, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  if (e) return e;
  e = cudaFuncSetAttribute(ntt_fwd_cols<kCols>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  if (e) return e;
  e = cudaFuncSetAttribute(ntt_inv_cols<kCols>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  return e;
}

}  // namespace hcnn
