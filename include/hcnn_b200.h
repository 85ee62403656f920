/*
 * hcnn-b200: C ABI of the B200-native RNS-CKKS engine.
 *
 * Drop-in boundary for the hot path of the reference package `hcnn`
 * (/root/reference/pkg/src/hcnn).  The reference has no FFI: its seams are
 * the kernel function table of kernels.py:339-371 (per-row modular kernels)
 * and the ckks.* object API of ckks.py.  Every entry point below
 * replaces one of those, over DEVICE pointers to residues laid out exactly
 * like RnsPoly.coeffs (uint64 [nlimbs][N], limb-major, ring.py:204-213).
 *
 * Conventions
 *  - Plain C types only; device buffers are passed as uint64_t*, streams as
 *    void* (a cudaStream_t; NULL = legacy default stream).
 *  - A "basis" is (nq, np): limbs 0..nq-1 over q_0..q_{nq-1}, then np limbs
 *    over the special primes p_0..p_{np-1} (ckks.py:139-145 mods_at/ext_mods).
 *  - A batch of `npolys` polynomials over one basis is contiguous:
 *    poly z starts at base + z*(nq+np)*N.  A ciphertext is a batch of 2
 *    (c0 then c1), always in the evaluation domain (ckks.py:215-218).
 *  - Switch keys are two device arrays (rows_b, rows_a) of shape
 *    [dnum][Lq+K][N] in Montgomery form, as SwitchKey holds them
 *    (ckks.py:315-324, 392-393).
 *  - All results are canonical residues in [0,q): bit-exact with the
 *    reference for every integer operation.
 *  - Return value: HCNN_OK or an hcnn_status; hcnn_last_error() gives text.
 *    Codes map 1:1 onto the reference's exception taxonomy (errors.py:8-53).
 *  - Calls are asynchronous on `stream`; a context is reentrant across
 *    streams except for the lazily built conversion tables, which are
 *    created under a lock.
 */
#ifndef HCNN_B200_H
#define HCNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hcnn_ctx hcnn_ctx;

typedef enum hcnn_status {
  HCNN_OK = 0,
  HCNN_E_PARAMETER = 1, /* ParameterError  errors.py:12 */
  HCNN_E_DOMAIN = 2,    /* DomainError     errors.py:16 */
  HCNN_E_BASIS = 3,     /* BasisError      errors.py:20 */
  HCNN_E_LEVEL = 4,     /* LevelError      errors.py:24 */
  HCNN_E_SCALE = 5,     /* ScaleError      errors.py:28 */
  HCNN_E_KEY = 6,       /* KeyError_       errors.py:32 */
  HCNN_E_CUDA = 100,    /* CUDA runtime failure */
  HCNN_E_NOMEM = 101
} hcnn_status;

const char* hcnn_last_error(void);
int hcnn_abi_version(void);

/* ---- context: CkksParams on the device (ckks.py:65-161, ring.py:32-72,
 *      ring.py:141-197 twiddles from the reference's psi) ------------------ */
int hcnn_ctx_create(hcnn_ctx** out, int device, uint32_t n, const uint64_t* q_moduli, uint32_t n_q,
                    const uint64_t* p_moduli, uint32_t n_p);
void hcnn_ctx_destroy(hcnn_ctx* ctx);
/* psi chosen for modulus index i (q's then p's): TwiddleTable.psi ring.py:141-157 */
int hcnn_ctx_psi(const hcnn_ctx* ctx, uint32_t mod_index, uint64_t* psi);

/* ---- ring.py / kernels.py row-level ops over a batch --------------------- */
/* ntt_forward ring.py:317-325 (kernels.ntt_inplace kernels.py:232-253) */
int hcnn_ntt_forward(hcnn_ctx* ctx, uint64_t* data, uint32_t nq, uint32_t np, uint32_t npolys, void* stream);
/* ntt_inverse ring.py:328-336 (kernels.intt_inplace kernels.py:255-281) */
int hcnn_ntt_inverse(hcnn_ctx* ctx, uint64_t* data, uint32_t nq, uint32_t np, uint32_t npolys, void* stream);
/* poly_add / poly_sub / poly_neg ring.py:264-284 (kernels.addmod/submod/negmod kernels.py:208-230).
 * b_broadcast == 1: b is a single poly applied to every poly of a; == 2 (add / sub): a holds
 * ciphertexts (c0, c1 pairs), b is applied to every c0 and every c1 is copied (padd, ckks.py:477-479). */
int hcnn_poly_add(hcnn_ctx* ctx, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t nq, uint32_t np,
                  uint32_t npolys, int b_broadcast, void* stream);
int hcnn_poly_sub(hcnn_ctx* ctx, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t nq, uint32_t np,
                  uint32_t npolys, int b_broadcast, void* stream);
int hcnn_poly_neg(hcnn_ctx* ctx, uint64_t* out, const uint64_t* a, uint32_t nq, uint32_t np, uint32_t npolys,
                  void* stream);
/* poly_mul_pointwise ring.py:287-296: both operands ordinary residues */
int hcnn_poly_mul(hcnn_ctx* ctx, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t nq, uint32_t np,
                  uint32_t npolys, int b_broadcast, void* stream);
/* poly_mul_mont_rows ring.py:307-314, pmult_mont ckks.py:499-503
 * (kernels.mulmod_mont kernels.py:190-193): b in Montgomery form */
int hcnn_poly_mul_mont(hcnn_ctx* ctx, uint64_t* out, const uint64_t* a, const uint64_t* b_mont, uint32_t nq,
                       uint32_t np, uint32_t npolys, int b_broadcast, void* stream);
/* kernels.muladd_mont kernels.py:200-206: out += a * b_mont */
int hcnn_poly_mac_mont(hcnn_ctx* ctx, uint64_t* out, const uint64_t* a, const uint64_t* b_mont, uint32_t nq,
                       uint32_t np, uint32_t npolys, int b_broadcast, void* stream);
/* to_mont_rows ring.py:299-304 / its inverse */
int hcnn_to_mont(hcnn_ctx* ctx, uint64_t* out, const uint64_t* a, uint32_t nq, uint32_t np, uint32_t npolys,
                 void* stream);
int hcnn_from_mont(hcnn_ctx* ctx, uint64_t* out, const uint64_t* a, uint32_t nq, uint32_t np, uint32_t npolys,
                   void* stream);
/* _scalar_mul_rows ckks.py:350-356: limb i times consts[i] (host array, any value, reduced here) */
int hcnn_scalar_mul(hcnn_ctx* ctx, uint64_t* out, const uint64_t* a, const uint64_t* consts, uint32_t nq,
                    uint32_t np, uint32_t npolys, void* stream);
/* + consts[i] on every residue of limb i: adds the constant polynomial
 * (evaluation domain), used for exact constant terms in polynomial evaluation */
int hcnn_scalar_add(hcnn_ctx* ctx, uint64_t* out, const uint64_t* a, const uint64_t* consts, uint32_t nq,
                    uint32_t np, uint32_t npolys, void* stream);
/* signed int64 coefficient rows [npolys][N] (device) -> residues in every limb:
 * sample_poly replication ring.py:463-467, encode reduction ckks.py:284-288 */
int hcnn_from_signed(hcnn_ctx* ctx, uint64_t* out, const int64_t* in, uint32_t nq, uint32_t np, uint32_t npolys,
                     void* stream);
/* as hcnn_from_signed, output in Montgomery form (v R mod q): NTT-linear, so
 * NTT(from_signed_mont(v)) == to_mont(NTT(from_signed(v))) bit for bit --
 * the mask path's to_mont pass folded away (packing.py _mask_pt rows) */
int hcnn_from_signed_mont(hcnn_ctx* ctx, uint64_t* out, const int64_t* in, uint32_t nq, uint32_t np,
                          uint32_t npolys, void* stream);
/* forward NTT of signed int64 coefficient rows ([npolys][N], one row shared
 * by all nq limbs) into out [npolys][nq][N], Montgomery form if mont:
 * == hcnn_from_signed(_mont) + hcnn_ntt_forward, fused into the first NTT
 * pass (compact-mask materialisation, packing.py _mask_pt rows) */
int hcnn_ntt_from_signed(hcnn_ctx* ctx, uint64_t* out, const int64_t* in, uint32_t nq, uint32_t npolys, int mont,
                         void* stream);
/* automorphism X -> X^g.  eval_domain=0: ring.automorphism ring.py:427-439
 * (coefficient domain, signed permutation); eval_domain=1: the equivalent
 * index permutation of the bit-reversed NTT output. */
int hcnn_automorphism(hcnn_ctx* ctx, uint64_t* out, const uint64_t* in, uint64_t g, int eval_domain, uint32_t nq,
                      uint32_t np, uint32_t npolys, void* stream);
/* base_convert ring.py:378-398 (centred FBC, kernels.fbc_row kernels.py:283-301).
 * Source/target limbs are given as modulus indices (q's 0..Lq-1, p's Lq..). */
int hcnn_base_convert(hcnn_ctx* ctx, uint64_t* out, const uint64_t* in, const uint32_t* src_mods, uint32_t n_src,
                      const uint32_t* dst_mods, uint32_t n_dst, uint32_t npolys, void* stream);

/* ---- ckks.py scheme ops --------------------------------------------------- */
/* scratch needed by keyswitch/hmult/rotate at `level` */
size_t hcnn_ks_workspace_bytes(const hcnn_ctx* ctx, uint32_t level);
/* _keyswitch_coeff ckks.py:548-602 applied to iNTT(x_eval): x_eval is an
 * eval-domain poly over q_0..q_level; out0/out1 eval-domain over the same basis */
int hcnn_keyswitch(hcnn_ctx* ctx, uint64_t* out0, uint64_t* out1, const uint64_t* x_eval, uint32_t level,
                   const uint64_t* key_b, const uint64_t* key_a, void* ws, void* stream);
/* hmult ckks.py:605-613 (tensor product + relinearisation; caller rescales) */
int hcnn_hmult(hcnn_ctx* ctx, uint64_t* out_ct, const uint64_t* a_ct, const uint64_t* b_ct, uint32_t level,
               const uint64_t* rlk_b, const uint64_t* rlk_a, void* ws, void* stream);
/* n_rot single-key rotations of one ciphertext sharing one ModUp (hoisted);
 * rotation i applies galois[i] with key (keys_b[i], keys_a[i]) and is
 * bit-exact with ckks._apply_step ckks.py:620-625.  outs[i] are ct buffers. */
int hcnn_rotate_hoisted(hcnn_ctx* ctx, uint64_t* const* outs, const uint64_t* ct, uint32_t level, uint32_t n_rot,
                        const uint64_t* galois, const uint64_t* const* keys_b, const uint64_t* const* keys_a,
                        void* ws, void* stream);
/* Several MAC outputs over one shared term list (the HyPHEN conv's planes:
 * every output plane of a layer sums masks against the same rotated input
 * ciphertexts).  outs[g] (+)= sum_t cts[t] (.) masks[g * n_terms + t]; a null
 * mask means output g has no term t.  Each ciphertext is read once per 4
 * outputs instead of once per output; results equal hcnn_mac_terms on each
 * output's non-null terms (packing.py:600-604 / :520-525). */
int hcnn_mac_terms_multi(hcnn_ctx* ctx, uint64_t* const* outs, const uint64_t* const* cts,
                         const uint64_t* const* masks_mont, uint32_t n_out, uint32_t n_terms, uint32_t level,
                         int accumulate, void* stream);

/* as hcnn_mac_terms_multi; packed[g*n_terms+t] = 1 marks a mask stored in
 * the packed layout of hcnn_pack_masks (nullable: none packed) */
int hcnn_mac_terms_multi_packed(hcnn_ctx* ctx, uint64_t* const* outs, const uint64_t* const* cts,
                                const uint64_t* const* masks_mont, const unsigned char* packed, uint32_t n_out,
                                uint32_t n_terms, uint32_t level, int accumulate, void* stream);
/* hcnn_mac_terms_multi_packed over image batches (no reference counterpart:
 * the reference runs one image at a time): cts[t] and outs[g] each hold
 * n_images (1 or 2) ciphertexts 2 (level+1) N words apart that share every
 * mask; each mask tile is read once for both images.  Per image the residues
 * equal hcnn_mac_terms_multi_packed's. */
int hcnn_mac_terms_multi_images(hcnn_ctx* ctx, uint64_t* const* outs, const uint64_t* const* cts,
                                const uint64_t* const* masks, const unsigned char* packed, uint32_t n_out,
                                uint32_t n_terms, uint32_t level, uint32_t n_images, int accumulate, void* stream);
/* Resident mask compaction: n_masks Montgomery rows [n][level+1][N] ->
 * (8 + 4 level + sum_r hb_r) N bytes each: limb 0 as u64, limbs 1.. as u32
 * low-word planes, then one high plane per limb, u8 when q_r < 2^40 and u16
 * otherwise (hb_r = 1 or 2); only for chains whose q_1..q_level are < 2^48
 * (HCNN_E_BASIS otherwise).  Lossless; hcnn_unpack_mask restores one mask's rows. */
int hcnn_pack_masks(hcnn_ctx* ctx, void* out, const uint64_t* in, uint32_t n_masks, uint32_t level, void* stream);
int hcnn_unpack_mask(hcnn_ctx* ctx, uint64_t* out, const void* in, uint32_t level, void* stream);

/* ---- batched ciphertext ops ---------------------------------------------
 * A batch is nb ciphertexts stored back to back ([nb][2][level+1][N]); every
 * kernel of the op covers the whole batch and each key / mask load feeds
 * several entries.  Entry-wise bit-exact with the single-ciphertext calls. */
size_t hcnn_ks_workspace_bytes_batch(const hcnn_ctx* ctx, uint32_t level, uint32_t nb);
/* workspace for hcnn_rotate_hoisted_batch with n_rot steps (all steps share
 * one ModDown chain: ks inner products for every step, then one iNTT / FBC /
 * NTT / combine launch each for the whole group) */
size_t hcnn_ks_workspace_bytes_rot(const hcnn_ctx* ctx, uint32_t level, uint32_t nb, uint32_t n_rot);
int hcnn_hmult_batch(hcnn_ctx* ctx, uint64_t* out_cts, const uint64_t* a_cts, const uint64_t* b_cts, uint32_t level,
                     uint32_t nb, const uint64_t* rlk_b, const uint64_t* rlk_a, void* ws, void* stream);
/* outs[i]: batch buffer receiving rotation i of every entry.  key_lqs
 * (nullable): key i is stored truncated to its first key_lqs[i] q-limbs
 * (rows [ceil(key_lqs[i]/K)][key_lqs[i]+K][N], same residues as the full
 * key's prefix) -- enough for every level < key_lqs[i]; 0 = full key. */
int hcnn_rotate_hoisted_batch(hcnn_ctx* ctx, uint64_t* const* outs, const uint64_t* cts, uint32_t level,
                              uint32_t nb, uint32_t n_rot, const uint64_t* galois, const uint64_t* const* keys_b,
                              const uint64_t* const* keys_a, const uint32_t* key_lqs, void* ws, void* stream);
/* hcnn_mac_terms over batches: cts[t] and out_cts are batches, the masks are
 * shared by every entry (bootstrapping's CtS/StC diagonals) */
int hcnn_mac_terms_batch(hcnn_ctx* ctx, uint64_t* out_cts, const uint64_t* const* cts,
                         const uint64_t* const* masks_mont, uint32_t n_terms, uint32_t level, uint32_t nb,
                         int accumulate, void* stream);

/* ---- extended-basis (double-hoisted) linear transforms ---------------------
 * Bootstrapping's baby-step/giant-step products keep rotations in Q_l||P
 * (no ModDown per rotation): out = (P sigma_g(c0) + <d, key_b>, <d, key_a>)
 * over nq + K limbs ([nb][2][nq+K][N] per rotation), MAC'd against masks
 * encoded over Q_l||P, and brought back with one ModDown per sum.  No
 * reference counterpart (the reference has no bootstrapping). */
int hcnn_rotate_hoisted_ext_batch(hcnn_ctx* ctx, uint64_t* const* outs_ext, const uint64_t* cts, uint32_t level,
                                  uint32_t nb, uint32_t n_rot, const uint64_t* galois,
                                  const uint64_t* const* keys_b, const uint64_t* const* keys_a,
                                  const uint32_t* key_lqs, void* ws, void* stream);
int hcnn_mac_terms_ext_batch(hcnn_ctx* ctx, uint64_t* out_ext, const uint64_t* const* cts_ext,
                             const uint64_t* const* masks_mont_ext, uint32_t n_terms, uint32_t level, uint32_t nb,
                             int accumulate, void* stream);
/* out [nb][2][nq][N] = ModDown(in_ext [nb][2][nq+K][N]); in_ext's P limbs are
 * clobbered; ws: hcnn_ks_workspace_bytes_batch(level, nb) */
int hcnn_moddown_batch(hcnn_ctx* ctx, uint64_t* out, uint64_t* in_ext, uint32_t level, uint32_t nb, void* ws,
                       void* stream);
/* ModDown and the following rescale fused: Q_level||P ciphertexts ->
 * round(x / (P q_level)) over Q_{level-1} with one centred base conversion
 * from the K+1 limbs (q_level, P).  One rounding instead of two, so residues
 * differ from hcnn_moddown_batch + hcnn_rescale (no reference counterpart;
 * bootstrapping's linear transforms).  out [nb][2][level][N]; in_ext's limbs
 * level..level+K are clobbered; ws: hcnn_ks_workspace_bytes_batch(level, nb) */
int hcnn_moddown_rescale_batch(hcnn_ctx* ctx, uint64_t* out, uint64_t* in_ext, uint32_t level, uint32_t nb, void* ws,
                               void* stream);
/* hmult + relinearisation + rescale with one ModDown (the key-switch sum and
 * P (d0, d1) are divided by P q_level together): out [nb][2][level][N].
 * Residues differ from hcnn_hmult_batch + hcnn_rescale (one rounding);
 * bootstrapping's EvalMod products.  ws: hcnn_hmult_rescale_workspace_bytes */
size_t hcnn_hmult_rescale_workspace_bytes(const hcnn_ctx* ctx, uint32_t level, uint32_t nb);
int hcnn_hmult_rescale_batch(hcnn_ctx* ctx, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t level,
                             uint32_t nb, const uint64_t* kb, const uint64_t* ka, void* ws, void* stream);

/* rescale ckks.py:506-528 for npolys polys at `level` -> level-1 */
size_t hcnn_rescale_workspace_bytes(const hcnn_ctx* ctx, uint32_t npolys);
int hcnn_rescale(hcnn_ctx* ctx, uint64_t* out, const uint64_t* in, uint32_t level, uint32_t npolys, void* ws,
                 void* stream);

/* plane MAC of the HyPHEN convolution (packing.py:600-604, 520-525):
 * out = [accumulate ? out : 0] + sum_t cts[t] (.) masks[t], ciphertexts at
 * `level` (2 polys each), masks Montgomery-form [level+1][N] like the
 * reference's _mask_pt rows; cts/masks are host arrays of device pointers */
int hcnn_mac_terms(hcnn_ctx* ctx, uint64_t* out_ct, const uint64_t* const* cts, const uint64_t* const* masks_mont,
                   uint32_t n_terms, uint32_t level, int accumulate, void* stream);

/* out[npolys][nq][N] (+)= sum_t consts[t][r] * srcs[t] limb-wise (integer
 * constants, reduced per limb).  srcs[t] has src_limbs[t] >= nq limbs per
 * poly (a longer ciphertext is read as its level-dropped prefix).  Replaces
 * the per-coefficient mul_const / add chain of a Chebyshev evaluation
 * (no reference counterpart: the reference has no bootstrapping,
 * ckks.py:667-690 debug_refresh); any number of terms (batched by 16).
 * c0_add (nullable, one per limb) is added to every even poly (the c0 of
 * each ciphertext): a plaintext constant joins the same pass. */
int hcnn_scalar_mac(hcnn_ctx* ctx, uint64_t* out, const uint64_t* const* srcs, const uint32_t* src_limbs,
                    const uint64_t* consts, uint32_t n_terms, uint32_t nq, uint32_t npolys, int accumulate,
                    const uint64_t* c0_add, void* stream);

/* ---- instrumentation ------------------------------------------------------ */
/* count of engine kernels launched since load (all contexts) */
unsigned long long hcnn_kernel_launches(void);
/* Compute ceiling of the NTT: butterflies/s of a radix-16 register network
 * run on register-resident data (no memory traffic) on `device`.  fast:
 * 0 full-width integer network, 1 unreduced q < 2^47 integer network,
 * 2 FP64-quotient network, 3 its magic-constant variant, 4 the pure FP64
 * network the q < 2^41 limbs run.  No reference counterpart (roofline
 * denominator for bench.py). */
int hcnn_ntt_butterfly_peak(int device, int fast, double* bfly_per_s);
/* limbs transformed since the last reset, by class:
 * [forward q<2^47, forward full, inverse q<2^47, inverse full] */
void hcnn_ntt_limb_counts(unsigned long long* out4, int reset);
/* key-switch accounting since the last reset (bench roofline row, no
 * reference counterpart): [key switches, minimal HBM bytes (digits read
 * once + switch keys + outputs), forward limb-NTTs, inverse limb-NTTs] */
void hcnn_ks_counters(unsigned long long* out4, int reset);
/* process-wide tuning knobs: "ntt_group_limbs" (NTT pass pairs run on groups
 * of this many limbs so the inter-pass data stays in L2; 0 = whole batch),
 * "ntt_hints" (1 = evict-last twiddles / streaming data loads) */
int hcnn_set_option(const char* name, long long value);
/* when enabled, every launch is bracketed by CUDA events on its stream */
void hcnn_profile_enable(int on);
/* per-kernel totals as JSON {"name": [launches, ms, algorithmic_bytes, kernels]};
 * returns the JSON length (buf may be NULL to size it) */
int hcnn_profile_read(char* buf, size_t len, int reset);

#ifdef __cplusplus
}
#endif
#endif /* HCNN_B200_H */
