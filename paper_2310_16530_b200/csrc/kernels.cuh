// Kernel-level interfaces shared between the .cu translation units.
#pragma once
#include <atomic>
#include <mutex>

#include "common.cuh"

namespace hcnn {

// A batch of polynomials over one basis: poly z, limb r lives at
// base + z*poly_stride + r*N.  skip_alpha != 0 marks the key-switch ModUp
// layout: poly z is digit z and its own limbs [z*alpha, min(z*alpha+alpha, nq))
// are left untouched (they are taken from the eval-domain input instead).
struct LimbMap {
  u64* base;          // address of (poly 0, limb first_limb)
  size_t poly_stride;
  Basis basis;
  u32 skip_alpha;
  u32 first_limb;     // basis position of the first processed limb
  u32 r0, z0;         // sub-batch offsets (limb / poly) added to blockIdx.y / blockIdx.z
  u32 zmod;           // skip_alpha digit = z % zmod (batched ModUp: [nb][ndig] polys); 0 = z
  // forward NTT only: read signed int64 coefficients (one row of N per poly,
  // shared by every limb) and reduce them on load instead of reading base;
  // smont: Montgomery form (v R mod q).  Fuses from_signed into the NTT.
  const long long* sin;
  int smont;
  // sin_center != 0: the row holds residues mod sin_center (a rescale's top
  // limb after its iNTT), read as the centred lift t > q/2 ? t - q : t
  u64 sin_center;
  // forward NTT only, host pointer (null: plain NTT): the transform is the
  // ModDown lift and its store is fused with the combine (NttCombine)
  const struct NttCombine* cb;
};

// ModDown combine fused into the lift's forward NTT (ckks.py:548-602): for
// poly z = 2 (s nb + b) + p of the lift, out = (acc_Q - lift) P^-1 (+ add),
// exactly k_moddown_combine(_steps)'s arithmetic.  out[s] + b out_bst +
// p out_pst + r N; add[p] + b add_bst + r N gathered through Galois g[s].
constexpr int kCombineMax = 32;
struct NttCombine {
  const u64* acc;
  size_t acc_pst;  // poly stride of acc (n_ext N)
  const u64* pinv;
  const u64* pinv_sh;
  u32 nb;
  size_t out_bst, out_pst, add_bst;
  const u64* add[2];
  u64* out[kCombineMax];
  u64 g[kCombineMax];
};
// the combine for rows [r0, r0 + nrows) of an npolys-poly lift (the rows the
// NTT did not fuse)
cudaError_t launch_combine_rows(const NttCombine& C, const u64* lift, u32 nq, u32 r0, u32 nrows, u32 npolys,
                                u32 logN, const ModConsts* mc, cudaStream_t st);

// tuning knobs (hcnn_set_option): NTT sub-batch size in limbs (0 = one
// launch pair for the whole batch) and L2 cache-policy hints
struct NttTuning {
  int group_limbs = 0;
  int hints = 1;
  // 1: register-capped integer-network kernels (more resident warps): 3 interleaved
  // ResNet20 A/B pairs 331.8 vs 333.4 ms/image, each pair lower (profiles/r02_ntt_occ_ab.txt)
  int occupancy = 1;
  int split = 1;      // 1: separate launches per modulus class (measured: inverse 0.778 -> 0.758 us/limb), 2: forward only
  int f64_minb = 1;   // FP64 chunk passes: min CTAs per SM hint (1, 5 or 6)
  int pipe = 1;       // FP64 forward chunk pass pipelined over polys (ntt2_fwd_chunks_f64p)
  // ModDown combine fused into the lift NTT's FP64 chunk pass: off -- measured
  // slower (tools/ks_bench.py: hoisted rotations at level 14, 2.21 -> 2.86 ms;
  // the epilogue's acc / c0 loads are not prefetched and stall every poly)
  int md_fuse = 0;
  // integer-network class runs of a mixed launch (q0, the wide bootstrapping
  // primes, the specials) on a side stream forked from the caller's, next
  // to the FP64-network run (a fork / join branch inside a graph capture)
  int fork = 1;
};
extern NttTuning g_ntt_tuning;

// per-device side stream + fork / join events (arith.cu); the caller holds
// *mu from the fork record to the join wait
cudaError_t side_stream(cudaStream_t* s, cudaEvent_t* fork, cudaEvent_t* join, std::mutex** mu);

struct NttTables {
  u32 logN;
  const ModConsts* mc;
  const u64* tw;    // [mod][N] psi^brv(j)
  const u64* twp;   // Shoup companions
  const u64* itw;   // [mod][N] psi^-brv(j)
  const u64* itwp;
  const ulonglong2* ctw;   // [mod][N/256][256] per-chunk forward twiddles (ntt2.cu)
  const ulonglong2* ictw;  // [mod][N/256][256] per-chunk inverse twiddles
  const unsigned char* small;  // host: per modulus index, 2: q < 2^kFpBits, 1: q < 2^47, 0: full width
};

void ntt_split(u32 logN, u32* logN1);
cudaError_t launch_ntt(const NttTables& T, const LimbMap& map, u32 nlimbs, u32 npolys, bool inverse,
                       cudaStream_t st);
cudaError_t ntt_configure_smem();
bool ntt2_supported(u32 logN);
int ntt_butterfly_peak(int fast, double* bfly_per_s);
// moduli below 2^kFpBits run both transforms on the FP64 network
// (ntt2.cu); their chunk twiddles are (double(w), double(w/q)) bit patterns.
// 2^41 keeps the unreduced inverse pass (inputs < 4q, 2^8 growth) and the
// forward pass pair inside the exact window (|operand| < 2^51).
constexpr int kFpBits = 41;
constexpr bool kNttFp = true;
extern unsigned long long g_ntt_limbs[4];
extern std::atomic<unsigned long long> g_ntt_extra_launches;  // split NTT launches beyond one pair per call
cudaError_t launch_ntt2(const NttTables& T, const LimbMap& map, u32 nlimbs, u32 npolys, bool inverse,
                        cudaStream_t st);

// --------------------------------------------------------------------------
// fast base conversion tables (ring.py:343-375): for one source set and a
// set of target moduli.
//   y_i = x_i * (Q/q_i)^-1 mod q_i  (inv_punc, Shoup form with companion)
//   out_t = sum_i [y_i]_centred * (Q/q_i mod t)   (tmat Montgomery form)
// --------------------------------------------------------------------------
struct FbcDev {
  u32 ns, nt;
  const u32* src_mod;     // [ns] modulus index of each source limb
  const u32* dst_mod;     // [nt] modulus index of each target limb
  const u32* dst_pos;     // [nt] output limb position of each target
  const u64* inv_punc;    // [ns]
  const u64* inv_punc_sh; // [ns]
  const u64* tmat;        // [nt][ns] Montgomery form of (Q/q_i) mod t
  const u64* corr;        // [nt][1<<ns] sum_{i in mask} q_i*(Q/q_i) mod t, or null (ns > 6)
  int nored;              // ns * max(q_i) < 2^64: 128-bit sums need no interim reduction
};

}  // namespace hcnn
