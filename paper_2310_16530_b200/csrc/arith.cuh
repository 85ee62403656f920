#pragma once
#include "kernels.cuh"

namespace hcnn {

enum { EW_ADD = 0, EW_SUB = 1, EW_MUL_MONT = 2, EW_MUL = 3, EW_MAC_MONT = 4 };
enum { EW_NEG = 0, EW_TO_MONT = 1, EW_FROM_MONT = 2, EW_SCALAR = 3, EW_SCALAR_ADD = 4 };

cudaError_t launch_ew_binary(int op, u64* out, const u64* a, const u64* b, Basis basis, u32 logN, u32 npolys,
                             int b_bcast, const ModConsts* mc, cudaStream_t st);
cudaError_t launch_ew_unary(int op, u64* out, const u64* a, Basis basis, u32 logN, u32 npolys,
                            const ModConsts* mc, const u64* consts, const u64* consts_sh, cudaStream_t st);
cudaError_t launch_from_signed(u64* out, const long long* in, Basis basis, u32 logN, u32 npolys,
                               const ModConsts* mc, int mont, cudaStream_t st);
cudaError_t launch_automorph(int eval_domain, u64* out, const u64* in, Basis basis, u32 logN, u32 npolys, u64 g,
                             const ModConsts* mc, cudaStream_t st);
cudaError_t launch_tensor(u64* d0, u64* d1, u64* d2, const u64* a, const u64* b, u32 nlimbs, u32 logN,
                          const ModConsts* mc, cudaStream_t st);
// T: host copy of the table (pointers are device addresses); dT: the same
// table in device memory (enables the specialised kernel), may be null
cudaError_t launch_fbc(const FbcDev& T, const FbcDev* dT, const ModConsts* mc, const u64* in, size_t in_pst,
                       u64* out, size_t out_pst, u32 logN, u32 npolys, u32 nt, cudaStream_t st);
// tabs: device array of per-digit tables; htabs: host copies of the same
// batched over nb ciphertexts: xc [nb] entries xc_bst apart, raised [nb][ndig][n_ext]
cudaError_t launch_modup(const FbcDev* tabs, const FbcDev* htabs, u32 ndig, const ModConsts* mc, const u64* xc,
                         u64* raised, u32 alpha, u32 n_ext, u32 logN, cudaStream_t st, u32 nb = 1,
                         size_t xc_bst = 0);
// acc [nb][2][n_ext]; x_eval entries x_bst apart; one key load feeds up to
// g_ks_batch (1, 2 or 4) entries (hcnn_set_option "ks_batch")
extern int g_ks_batch;
extern int g_fbc_fork;
cudaError_t set_ks96(int on);
extern int g_ks_pipe;
extern int g_ks_tma;
extern int g_ks_tma_min;
extern int g_mac_batch;
extern int g_mac_lanes;
extern int g_mac_async;
extern int g_mac_tma;
cudaError_t set_fbc_fast(int on);  // 96-bit FBC sums for all-small conversions (default on)
extern int g_ks_tma3;
extern int g_ks3_stages;
extern int g_mac3_stages;
extern int g_mac3_tpb;
extern int g_mac3_fork;
extern int g_mac_tpb;
extern int g_mac_minb;
extern int g_ks_tpb;
extern int g_ks_stages;
extern int g_tma_stages;
// c0 (nullable): adds P * sigma_g(c0) on the Q limbs (pR[i] = P R mod q_i) --
// the extended-basis (ModDown-free) rotation of double hoisting
cudaError_t launch_ks_inner(u64* acc, const u64* x_eval, const u64* raised, const u64* key_b, const u64* key_a,
                            Basis basis, u32 alpha, u32 ndig, u32 logN, u64 g, const ModConsts* mc,
                            cudaStream_t st, u32 nb = 1, size_t x_bst = 0, const u64* c0 = nullptr,
                            size_t c0_bst = 0, const u64* pR = nullptr, u32 key_lq = 0,
                            u32 fast_from = 0xffffffffu);  // Q rows >= fast_from: q < 2^42 (96-bit MACs)
// every rotation of a hoisted group in one inner-product launch (same
// arguments as launch_ks_inner, per-rotation acc / keys / Galois / key_lq)
constexpr int kKsRotMax = 16;
struct KsRots {
  u64* acc[kKsRotMax];
  const u64* kb[kKsRotMax];
  const u64* ka[kKsRotMax];
  u64 g[kKsRotMax];
  u32 klq[kKsRotMax];
};
extern int g_ks_rots;
extern int g_ks_rots_min_nb;
bool ks_rots_ok(u32 nb, u32 nrot, u32 logN);
cudaError_t launch_ks_inner_rots(const KsRots& R, u32 nrot, const u64* x_eval, const u64* raised, Basis basis,
                                 u32 alpha, u32 ndig, u32 logN, const ModConsts* mc, cudaStream_t st, u32 nb,
                                 size_t x_bst, const u64* c0 = nullptr, size_t c0_bst = 0,
                                 const u64* pR = nullptr);
// acc [nb][2][n_ext], lift [nb][2][nq]; outputs / addends of entry b at +b*out_bst / +b*add_bst
cudaError_t launch_moddown_combine(u64* out0, u64* out1, const u64* acc, const u64* lift, const u64* add0,
                                   const u64* add1, u64 g_add, u32 nq, u32 n_ext, u32 logN, const u64* pinv,
                                   const u64* pinv_sh, const ModConsts* mc, cudaStream_t st, u32 nb = 1,
                                   size_t out_bst = 0, size_t add_bst = 0);
cudaError_t launch_rescale_lift(u64* out, const u64* top, u32 l, u32 logN, u32 npolys, const u64* qtop_mod,
                                const ModConsts* mc, cudaStream_t st);
cudaError_t launch_rescale_combine(u64* out, const u64* in, u32 l, u32 logN, u32 npolys, const u64* inv,
                                   const u64* inv_sh, const ModConsts* mc, cudaStream_t st);
constexpr int kComboMax = 32;
struct ComboSteps {
  u64* out[kComboMax];
  u64 g[kComboMax];
};
cudaError_t launch_add_pmul(u64* acc, const u64* d, u32 nb, u32 nq, u32 n_ext, u32 logN, const u64* pR,
                            const ModConsts* mc, cudaStream_t st);
cudaError_t launch_moddown_combine_steps(const ComboSteps& S, u32 n_rot, const u64* acc, const u64* lift,
                                         const u64* add0, u32 nb, u32 nq, u32 n_ext, u32 logN, const u64* pinv,
                                         const u64* pinv_sh, const ModConsts* mc, size_t out_bst, size_t add_bst,
                                         cudaStream_t st);
constexpr int kScalarMax = 128;
struct ScalarArgs {
  u64 w[kScalarMax];
  u64 wp[kScalarMax];
};
cudaError_t launch_scalar(int add, u64* out, const u64* a, Basis basis, u32 logN, u32 npolys, const ModConsts* mc,
                          const ScalarArgs& args, cudaStream_t st);

// out (+)= sum_t k_t[limb] * src_t over q-limbs; sources may be level-dropped
// views of longer ciphertexts (per-source poly stride in limbs)
constexpr int kSMacTerms = 16;
constexpr int kSMacLimbs = 48;
struct ScalarMacArgs {
  const u64* src[kSMacTerms];
  u32 src_limbs[kSMacTerms];
  u64 w[kSMacTerms][kSMacLimbs];
  u64 wp[kSMacTerms][kSMacLimbs];
  u64 add0[kSMacLimbs];  // per-limb constant added to every c0 (even poly index); has_add0
  int has_add0;
};
cudaError_t launch_scalar_mac(const ScalarMacArgs& A, int nt, u64* out, u32 nl, u32 logN, u32 npolys,
                              int accumulate, const ModConsts* mc, cudaStream_t st);

constexpr int kMacMax = 64;
struct MacTerms {
  const u64* ct[kMacMax];
  const u64* mask[kMacMax];
};
// nb > 1: ct[t] / out are batches of nb ciphertexts (2*nq*N apart) sharing the masks
// np > 0: ciphertexts / masks over Q_l||P (nq + np limbs; P moduli at Lq..)
cudaError_t launch_mac_terms(const MacTerms& T, int nt, u64* out, u32 nq, u32 logN, int accumulate,
                             const ModConsts* mc, cudaStream_t st, u32 nb = 1, u32 np = 0, u32 Lq = 0);
// several outputs sharing one term list (HyPHEN conv planes): each rotated
// ciphertext is read once per launch for up to kMultiG outputs; masks may be
// null (the output has no such term)
constexpr int kMultiG = 4;
constexpr int kMultiT = 48;
struct MacMulti {
  const u64* ct[kMultiT];
  const u64* mask[kMultiG][kMultiT];
  u64* out[kMultiG];
  unsigned char packed[kMultiG][kMultiT];  // 1: mask in the packed layout (launch_pack_masks)
  unsigned fast_from;  // limbs r >= fast_from (>= 1) have q < 2^42: 96-bit carry-chain MACs (k_mac_multi_tma3)
  unsigned nimg;       // image batches: ct[t] / out[g] hold nimg images img_stride apart (1: single)
  size_t img_stride;
  unsigned long long wide;                 // packed layout: bit r set = limb r needs a 16-bit high plane
};
// Packed resident masks: limb 0 as u64 [N]; limbs 1..nq-1 as u32 low words
// [nq-1][N]; then each limb's high bits as its own plane, u8 for moduli
// below 2^40 and u16 up to 2^48 (`wide` bit r) -- (8 + 4 (nq-1) + sum hb) N
// bytes, lossless.  Byte offset of limb r's high plane and its width:
__host__ __device__ __forceinline__ unsigned packed_hb(unsigned r, unsigned long long wide) {
  return ((wide >> r) & 1ull) ? 2u : 1u;
}
__host__ __device__ __forceinline__ size_t packed_hi_off(unsigned r, unsigned nq, size_t N, unsigned long long wide) {
  unsigned hb = 0;
#ifdef __CUDA_ARCH__
  hb = (r - 1) + __popcll(wide & ((1ull << r) - 2ull));
#else
  hb = (r - 1) + (unsigned)__builtin_popcountll(wide & ((1ull << r) - 2ull));
#endif
  return 8 * N + 4 * (size_t)(nq - 1) * N + (size_t)hb * N;
}
// the high bits of coefficient k of limb r (u8 or u16 plane)
__device__ __forceinline__ u64 packed_hi(const unsigned char* plane, size_t k, unsigned hb) {
  return hb == 2 ? (u64)reinterpret_cast<const unsigned short*>(plane)[k] : (u64)plane[k];
}
// packing (chains whose q_1..q_{nq-1} are < 2^48, the application primes)
cudaError_t launch_pack_masks(unsigned char* out, const u64* in, u32 nm, u32 nq, u32 logN, unsigned long long wide,
                              cudaStream_t st);
cudaError_t launch_unpack_mask(u64* out, const unsigned char* in, u32 nq, u32 logN, unsigned long long wide,
                               cudaStream_t st);
cudaError_t launch_mac_multi(const MacMulti& M, int ng, int nt, u32 nq, u32 logN, int accumulate,
                             const ModConsts* mc, cudaStream_t st);
cudaError_t launch_gather_limb(u64* out, const u64* in, u32 limb, u32 nlimbs, u32 logN, u32 npolys,
                               cudaStream_t st);

}  // namespace hcnn
