// C ABI: device context (CkksParams in HBM) and the scheme-level
// orchestration of keyswitch / hmult / rotate / rescale.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hcnn_b200.h"
#include "arith.cuh"
#include "common.cuh"
#include "kernels.cuh"

using namespace hcnn;

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(expr)                                                                              \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      return fail(HCNN_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));           \
  } while (0)

// host-resident FBC table with its device copy
struct FbcStore {
  FbcDev dev{};            // host copy (pointers into `mem`)
  FbcDev* d_dev = nullptr;  // the same struct in device memory
  void* mem = nullptr;
};

struct ModupSet {
  std::vector<FbcStore> digits;
  std::vector<FbcDev> host;  // host copies, one per digit
  FbcDev* d_tabs = nullptr;  // device array of FbcDev, one per digit
};

struct hcnn_ctx {
  int device = 0;
  u32 n = 0, logN = 0, Lq = 0, K = 0, nmods = 0, alpha = 0, dnum = 0;
  std::vector<u64> mods, psi;
  std::vector<ModConsts> hmc;
  ModConsts* d_mc = nullptr;
  u64 *d_tw = nullptr, *d_twp = nullptr, *d_itw = nullptr, *d_itwp = nullptr;
  ulonglong2 *d_ctw = nullptr, *d_ictw = nullptr;
  bool ntt2_ok = false;
  std::vector<unsigned char> small;  // NTT modulus class per modulus (see ctx_create)
  unsigned long long wide = 0;       // packed masks: bit r = q_r >= 2^40 (16-bit high plane)
  FbcStore moddown;                  // P -> q_0..q_{Lq-1}
  u64 *d_pinv = nullptr, *d_pinv_sh = nullptr;  // P^-1 mod q_i
  u64* d_pR = nullptr;                            // P R mod q_i (Montgomery form of P)
  u64 *d_rinv = nullptr, *d_rinv_sh = nullptr;  // [l][i] q_l^-1 mod q_i
  u64* d_qmod = nullptr;                         // [l][i] q_l mod q_i
  std::mutex mu;
  std::map<u32, ModupSet> modup;
  // fused ModDown + rescale at level l: FBC from (q_l, P) to q_0..q_{l-1},
  // (P q_l)^-1 mod q_i (+ Shoup companions)
  struct MdrSet {
    FbcStore fbc;
    u64 *d_inv = nullptr, *d_inv_sh = nullptr;
  };
  std::map<u32, MdrSet> mdr;
  std::map<std::vector<u32>, FbcStore> generic;
  NttTables tables() const {
    NttTables T;
    T.logN = logN;
    T.mc = d_mc;
    T.tw = d_tw;
    T.twp = d_twp;
    T.itw = d_itw;
    T.itwp = d_itwp;
    T.ctw = d_ctw;
    T.ictw = d_ictw;
    T.small = small.data();
    return T;
  }
  Basis basis(u32 nq, u32 np) const {
    Basis b;
    b.nq = nq;
    b.np = np;
    b.Lq = Lq;
    return b;
  }
};

static u32 bitrev(u32 x, u32 bits) {
  u32 r = 0;
  for (u32 i = 0; i < bits; ++i) {
    r = (r << 1) | (x & 1);
    x >>= 1;
  }
  return r;
}

// _find_psi (ring.py:160-167): smallest r in [2,1000) whose (q-1)/2N power
// is a primitive 2N-th root
static bool find_psi(u64 q, u32 n, u64* out) {
  if ((q - 1) % (2ull * n) != 0) return false;
  for (u64 r = 2; r < 1000; ++r) {
    u64 psi = h_powmod(r, (q - 1) / (2ull * n), q);
    if (psi != 1 && h_powmod(psi, n, q) == q - 1) {
      *out = psi;
      return true;
    }
  }
  return false;
}

static int build_fbc(hcnn_ctx* c, const std::vector<u32>& src, const std::vector<u32>& dst,
                     const std::vector<u32>& dst_pos, FbcStore* st) {
  const u32 ns = (u32)src.size(), nt = (u32)dst.size();
  std::vector<u32> u32buf;
  u32buf.insert(u32buf.end(), src.begin(), src.end());
  u32buf.insert(u32buf.end(), dst.begin(), dst.end());
  u32buf.insert(u32buf.end(), dst_pos.begin(), dst_pos.end());
  while (u32buf.size() % 2) u32buf.push_back(0);
  const bool with_corr = ns <= 6;
  std::vector<u64> u64buf(2 * ns + (size_t)nt * ns + (with_corr ? (size_t)nt << ns : 0));
  for (u32 i = 0; i < ns; ++i) {
    u64 qi = c->mods[src[i]];
    u64 prod = 1;
    for (u32 j = 0; j < ns; ++j)
      if (j != i) prod = h_mulmod(prod, c->mods[src[j]] % qi, qi);
    u64 inv = h_invmod(prod, qi);
    u64buf[i] = inv;
    u64buf[ns + i] = h_shoup(inv, qi);
  }
  for (u32 t = 0; t < nt; ++t) {
    u64 qt = c->mods[dst[t]];
    for (u32 i = 0; i < ns; ++i) {
      u64 prod = 1 % qt;
      for (u32 j = 0; j < ns; ++j)
        if (j != i) prod = h_mulmod(prod, c->mods[src[j]] % qt, qt);
      u64buf[2 * ns + (size_t)t * ns + i] = h_to_mont(prod, qt);
    }
    if (with_corr) {
      // corr[t][mask] = sum_{i in mask} q_i * (Q/q_i) mod t: the centred
      // lift subtracts q_i for every limb whose y_i exceeds q_i/2
      for (u32 mask = 0; mask < (1u << ns); ++mask) {
        u64 acc = 0;
        for (u32 i = 0; i < ns; ++i) {
          if (!((mask >> i) & 1)) continue;
          u64 prod = c->mods[src[i]] % qt;
          for (u32 j = 0; j < ns; ++j)
            if (j != i) prod = h_mulmod(prod, c->mods[src[j]] % qt, qt);
          acc = (acc + prod) % qt;
        }
        u64buf[2 * ns + (size_t)nt * ns + ((size_t)t << ns) + mask] = acc;
      }
    }
  }
  unsigned __int128 bound = 0;
  for (u32 i = 0; i < ns; ++i) bound += c->mods[src[i]];
  size_t b32 = u32buf.size() * 4, b64 = u64buf.size() * 8;
  CK(cudaMalloc(&st->mem, b32 + b64));
  CK(cudaMemcpy(st->mem, u32buf.data(), b32, cudaMemcpyHostToDevice));
  CK(cudaMemcpy((char*)st->mem + b32, u64buf.data(), b64, cudaMemcpyHostToDevice));
  u32* d32 = (u32*)st->mem;
  u64* d64 = (u64*)((char*)st->mem + b32);
  st->dev.ns = ns;
  st->dev.nt = nt;
  st->dev.src_mod = d32;
  st->dev.dst_mod = d32 + ns;
  st->dev.dst_pos = d32 + ns + nt;
  st->dev.inv_punc = d64;
  st->dev.inv_punc_sh = d64 + ns;
  st->dev.tmat = d64 + 2 * ns;
  st->dev.corr = with_corr ? d64 + 2 * ns + (size_t)nt * ns : nullptr;
  st->dev.nored = bound < ((unsigned __int128)1 << 64) ? 1 : 0;
  CK(cudaMalloc(&st->d_dev, sizeof(FbcDev)));
  CK(cudaMemcpy(st->d_dev, &st->dev, sizeof(FbcDev), cudaMemcpyHostToDevice));
  return HCNN_OK;
}

// Fused ModDown + rescale tables for level l >= 1: the K special limbs and
// q_l together are the modulus divided away (no reference counterpart:
// bootstrapping only, where one rounding instead of two is fine)
static int get_mdr(hcnn_ctx* c, u32 level, hcnn_ctx::MdrSet** out) {
  std::lock_guard<std::mutex> lk(c->mu);
  auto it = c->mdr.find(level);
  if (it != c->mdr.end()) {
    *out = &it->second;
    return HCNN_OK;
  }
  hcnn_ctx::MdrSet set;
  std::vector<u32> src{level}, dst, pos;
  for (u32 j = 0; j < c->K; ++j) src.push_back(c->Lq + j);
  for (u32 i = 0; i < level; ++i) {
    dst.push_back(i);
    pos.push_back(i);
  }
  int rc = build_fbc(c, src, dst, pos, &set.fbc);
  if (rc) return rc;
  std::vector<u64> inv(level), inv_sh(level);
  for (u32 i = 0; i < level; ++i) {
    const u64 qi = c->mods[i];
    u64 prod = c->mods[level] % qi;
    for (u32 j = 0; j < c->K; ++j) prod = h_mulmod(prod, c->mods[c->Lq + j] % qi, qi);
    inv[i] = h_invmod(prod, qi);
    inv_sh[i] = h_shoup(inv[i], qi);
  }
  CK(cudaMalloc(&set.d_inv, level * 8));
  CK(cudaMalloc(&set.d_inv_sh, level * 8));
  CK(cudaMemcpy(set.d_inv, inv.data(), level * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(set.d_inv_sh, inv_sh.data(), level * 8, cudaMemcpyHostToDevice));
  auto res = c->mdr.emplace(level, set);
  *out = &res.first->second;
  return HCNN_OK;
}

// ModUp tables for level l (ckks.py:563-571): digit j = q limbs
// [j*alpha, min(j*alpha+alpha, nq)), targets = Q_l||P minus the digit
static int get_modup(hcnn_ctx* c, u32 level, ModupSet** out) {
  std::lock_guard<std::mutex> lk(c->mu);
  auto it = c->modup.find(level);
  if (it != c->modup.end()) {
    *out = &it->second;
    return HCNN_OK;
  }
  ModupSet set;
  const u32 nq = level + 1, n_ext = nq + c->K, nd = (nq + c->alpha - 1) / c->alpha;
  Basis b = c->basis(nq, c->K);
  std::vector<FbcDev> devs;
  for (u32 j = 0; j < nd; ++j) {
    u32 lo = j * c->alpha, hi = std::min(lo + c->alpha, nq);
    std::vector<u32> src, dst, pos;
    for (u32 i = lo; i < hi; ++i) src.push_back(i);
    for (u32 r = 0; r < n_ext; ++r) {
      if (r >= lo && r < hi) continue;
      dst.push_back(b.mod_of(r));
      pos.push_back(r);
    }
    FbcStore st;
    int rc = build_fbc(c, src, dst, pos, &st);
    if (rc) return rc;
    set.digits.push_back(st);
    devs.push_back(st.dev);
    set.host.push_back(st.dev);
  }
  CK(cudaMalloc(&set.d_tabs, sizeof(FbcDev) * devs.size()));
  CK(cudaMemcpy(set.d_tabs, devs.data(), sizeof(FbcDev) * devs.size(), cudaMemcpyHostToDevice));
  auto res = c->modup.emplace(level, set);
  *out = &res.first->second;
  return HCNN_OK;
}


// ---------------------------------------------------------------------------
// launch accounting + optional per-launch CUDA-event profiling
// ---------------------------------------------------------------------------
#include <atomic>
#include <array>
struct ProfRec {
  std::string name;
  cudaEvent_t a, b;
  double bytes;
  int nk;
};
static std::mutex g_pm;
static std::atomic<bool> g_prof{false};
static std::vector<ProfRec> g_pending;
static std::map<std::string, std::array<double, 4>> g_acc;  // launches, ms, bytes, kernels
static std::atomic<unsigned long long> g_kernels{0};

#define PK(name, bytes, nk, st, expr)                                                 \
  do {                                                                                \
    cudaEvent_t _a = nullptr, _b = nullptr;                                           \
    const bool _p = g_prof.load();                                                    \
    if (_p) {                                                                         \
      cudaEventCreate(&_a);                                                           \
      cudaEventCreate(&_b);                                                           \
      cudaEventRecord(_a, st);                                                        \
    }                                                                                 \
    CK(expr);                                                                         \
    g_kernels += (nk);                                                                \
    if (_p) {                                                                         \
      cudaEventRecord(_b, st);                                                        \
      std::lock_guard<std::mutex> _lk(g_pm);                                          \
      g_pending.push_back(ProfRec{name, _a, _b, (double)(bytes), (int)(nk)});         \
    }                                                                                 \
  } while (0)

static int ntt_nk(const hcnn_ctx* c) { return c->logN > 12 ? 2 : 1; }

// key-switch accounting for the bench's key-switch roofline:
// [key switches, minimal HBM bytes (digits read once + keys + outputs),
//  forward limb-NTTs, inverse limb-NTTs] -- ModUp, inner product, ModDown
static std::atomic<unsigned long long> g_ks_acc[4];
static inline void ks_acc(int i, double v) { g_ks_acc[i] += (unsigned long long)v; }

extern "C" {

const char* hcnn_last_error(void) { return g_err.c_str(); }
int hcnn_abi_version(void) { return 1; }

int hcnn_ctx_create(hcnn_ctx** out, int device, uint32_t n, const uint64_t* q_moduli, uint32_t n_q,
                    const uint64_t* p_moduli, uint32_t n_p) {
  if (!out) return fail(HCNN_E_PARAMETER, "null output handle");
  if (n < 4 || (n & (n - 1))) return fail(HCNN_E_PARAMETER, "ring degree must be a power of two >= 4");
  if (n > (1u << 17)) return fail(HCNN_E_PARAMETER, "ring degree above 2^17 unsupported");
  if (n_q == 0) return fail(HCNN_E_BASIS, "empty q chain");
  if (n_q + n_p > HCNN_MAX_MODS) return fail(HCNN_E_PARAMETER, "too many moduli");
  CK(cudaSetDevice(device));
  hcnn_ctx* c = new hcnn_ctx();
  c->device = device;
  c->n = n;
  c->logN = 0;
  while ((1u << c->logN) < n) ++c->logN;
  c->Lq = n_q;
  c->K = n_p;
  c->nmods = n_q + n_p;
  c->alpha = n_p ? n_p : 1;
  c->dnum = (n_q + c->alpha - 1) / c->alpha;
  for (u32 i = 0; i < n_q; ++i) c->mods.push_back(q_moduli[i]);
  for (u32 i = 0; i < n_p; ++i) c->mods.push_back(p_moduli[i]);
  for (u32 i = 0; i < c->nmods; ++i) {
    u64 q = c->mods[i];
    if (q <= 2 || q >= (1ull << 62)) {
      delete c;
      return fail(HCNN_E_PARAMETER, "modulus outside (2, 2^62)");
    }
    for (u32 j = 0; j < i; ++j)
      if (c->mods[j] == q) {
        delete c;
        return fail(HCNN_E_PARAMETER, "moduli must be pairwise distinct");
      }
    u64 psi;
    if (!find_psi(q, n, &psi)) {
      delete c;
      return fail(HCNN_E_PARAMETER, "modulus is not 1 mod 2N or has no primitive 2N-th root");
    }
    c->psi.push_back(psi);
  }
  const size_t N = n;
  std::vector<u64> tw(c->nmods * N), twp(c->nmods * N), itw(c->nmods * N), itwp(c->nmods * N);
  std::vector<u64> pf(N), pi(N);
  for (u32 m = 0; m < c->nmods; ++m) {
    u64 q = c->mods[m], psi = c->psi[m], psi_inv = h_invmod(psi, q);
    u64 f = 1, g = 1;
    for (size_t j = 0; j < N; ++j) {
      pf[j] = f;
      pi[j] = g;
      f = h_mulmod(f, psi, q);
      g = h_mulmod(g, psi_inv, q);
    }
    for (size_t j = 0; j < N; ++j) {
      u32 b = bitrev((u32)j, c->logN);
      tw[m * N + j] = pf[b];
      twp[m * N + j] = h_shoup(pf[b], q);
      itw[m * N + j] = pi[b];
      itwp[m * N + j] = h_shoup(pi[b], q);
    }
    ModConsts mc{};
    mc.q = q;
    u64 x = q;  // q^-1 mod 2^64 by Newton (3 correct bits, doubling)
    for (int it = 0; it < 6; ++it) x *= 2 - q * x;
    mc.ninv = (u64)(0 - x);
    mc.r2 = (u64)(((unsigned __int128)1 << 127) % q);
    mc.r2 = h_mulmod(mc.r2, 2, q);
    mc.one_m = h_to_mont(1, q);
    mc.ninvN = h_invmod(n % q, q);
    mc.ninvN_sh = h_shoup(mc.ninvN, q);
    mc.two_q = 2 * q;
    mc.four_q = 4 * q;
    mc.one_sh = h_shoup(1, q);
    u64 w1 = itw[m * N + (N > 1 ? 1 : 0)];
    mc.ilast = h_mulmod(w1, mc.ninvN, q);
    mc.ilast_sh = h_shoup(mc.ilast, q);
    c->hmc.push_back(mc);
  }
  size_t tb = c->nmods * N * sizeof(u64);
  CK(cudaMalloc(&c->d_mc, sizeof(ModConsts) * c->nmods));
  CK(cudaMemcpy(c->d_mc, c->hmc.data(), sizeof(ModConsts) * c->nmods, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&c->d_tw, tb));
  CK(cudaMalloc(&c->d_twp, tb));
  CK(cudaMalloc(&c->d_itw, tb));
  CK(cudaMalloc(&c->d_itwp, tb));
  CK(cudaMemcpy(c->d_tw, tw.data(), tb, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_twp, twp.data(), tb, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_itw, itw.data(), tb, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_itwp, itwp.data(), tb, cudaMemcpyHostToDevice));
  for (u32 r = 0; r < c->Lq && r < 64; ++r)
    if (c->mods[r] >> 40) c->wide |= 1ull << r;
  u64 qmax = 0;
  for (u64 q : c->mods) {
    qmax = q > qmax ? q : qmax;
    // NTT modulus class: 2 = FP64 network, 1 = q < 2^47 integer fast path, 0 = full width
    c->small.push_back(q < (1ull << kFpBits) ? 2 : q < (1ull << 47) ? 1 : 0);
  }
  c->ntt2_ok = ntt2_supported(c->logN) && qmax < (1ull << 61);  // 8q < 2^64 (approximate-quotient NTT)
  if (c->ntt2_ok) {
    // per-chunk twiddles for the radix-16 chunk pass (ntt2.cu): chunk g of
    // 256 owns 255 Shoup pairs, forward e = 2^s-1+i -> tw[(N1+g)*2^s + i],
    // inverse e = nb-1+i -> itw[nb*(N1+g) + i] (nb = 128>>u blocks)
    const u32 N1 = n >> 8;
    std::vector<ulonglong2> ctw((size_t)c->nmods * N), ictw((size_t)c->nmods * N);
    for (u32 m = 0; m < c->nmods; ++m) {
      // FP64 network (ntt2.cu, q < 2^kFpBits), both directions: a twiddle
      // is the pair (double(w), double(wp * 2^-64) ~ w/q) as bit patterns
      const bool fp = kNttFp && c->mods[m] < (1ull << kFpBits);
      auto dbits = [](double d) -> u64 {
        u64 bits;
        std::memcpy(&bits, &d, 8);
        return bits;
      };
      auto pair_of = [&](u64 w, u64 wp) -> ulonglong2 {
        return fp ? make_ulonglong2(dbits((double)w), dbits((double)wp * 0x1p-64)) : make_ulonglong2(w, wp);
      };
      for (u32 g = 0; g < N1; ++g) {
        ulonglong2* F = &ctw[((size_t)m * N1 + g) * 256];
        ulonglong2* I = &ictw[((size_t)m * N1 + g) * 256];
        F[255] = make_ulonglong2(0, 0);
        I[255] = make_ulonglong2(0, 0);
        for (u32 s = 0; s < 8; ++s)
          for (u32 i = 0; i < (1u << s); ++i) {
            size_t src = (size_t)(N1 + g) * (1u << s) + i;
            F[(1u << s) - 1 + i] = pair_of(tw[m * N + src], twp[m * N + src]);
            u32 nb = 1u << s;  // inverse stage with nb blocks
            size_t isrc = (size_t)nb * (N1 + g) + i;
            I[nb - 1 + i] = pair_of(itw[m * N + isrc], itwp[m * N + isrc]);
          }
      }
    }
    CK(cudaMalloc(&c->d_ctw, ctw.size() * sizeof(ulonglong2)));
    CK(cudaMalloc(&c->d_ictw, ictw.size() * sizeof(ulonglong2)));
    CK(cudaMemcpy(c->d_ctw, ctw.data(), ctw.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_ictw, ictw.data(), ictw.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice));
  }
  // rescale table: q_l^-1 mod q_i
  std::vector<u64> rinv((size_t)n_q * n_q, 0), rinv_sh((size_t)n_q * n_q, 0), qmod((size_t)n_q * n_q, 0);
  for (u32 l = 1; l < n_q; ++l)
    for (u32 i = 0; i < l; ++i) {
      u64 qi = c->mods[i];
      u64 v = h_invmod(c->mods[l] % qi, qi);
      rinv[(size_t)l * n_q + i] = v;
      rinv_sh[(size_t)l * n_q + i] = h_shoup(v, qi);
      qmod[(size_t)l * n_q + i] = c->mods[l] % qi;
    }
  CK(cudaMalloc(&c->d_qmod, qmod.size() * 8));
  CK(cudaMemcpy(c->d_qmod, qmod.data(), qmod.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&c->d_rinv, rinv.size() * 8));
  CK(cudaMalloc(&c->d_rinv_sh, rinv.size() * 8));
  CK(cudaMemcpy(c->d_rinv, rinv.data(), rinv.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_rinv_sh, rinv_sh.data(), rinv.size() * 8, cudaMemcpyHostToDevice));
  if (n_p) {
    // ModDown tables: P -> every q (ckks.py:593-601)
    std::vector<u32> src, dst, pos;
    for (u32 k = 0; k < n_p; ++k) src.push_back(n_q + k);
    for (u32 i = 0; i < n_q; ++i) {
      dst.push_back(i);
      pos.push_back(i);
    }
    int rc = build_fbc(c, src, dst, pos, &c->moddown);
    if (rc) return rc;
    std::vector<u64> pinv(n_q), pinv_sh(n_q), pR(n_q);
    for (u32 i = 0; i < n_q; ++i) {
      u64 qi = c->mods[i], prod = 1;
      for (u32 k = 0; k < n_p; ++k) prod = h_mulmod(prod, c->mods[n_q + k] % qi, qi);
      pinv[i] = h_invmod(prod, qi);
      pinv_sh[i] = h_shoup(pinv[i], qi);
      pR[i] = h_to_mont(prod, qi);
    }
    CK(cudaMalloc(&c->d_pR, n_q * 8));
    CK(cudaMemcpy(c->d_pR, pR.data(), n_q * 8, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&c->d_pinv, n_q * 8));
    CK(cudaMalloc(&c->d_pinv_sh, n_q * 8));
    CK(cudaMemcpy(c->d_pinv, pinv.data(), n_q * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_pinv_sh, pinv_sh.data(), n_q * 8, cudaMemcpyHostToDevice));
  }
  CK(ntt_configure_smem());
  *out = c;
  return HCNN_OK;
}

void hcnn_ctx_destroy(hcnn_ctx* c) {
  if (!c) return;
  cudaFree(c->d_mc);
  cudaFree(c->d_tw);
  cudaFree(c->d_twp);
  cudaFree(c->d_itw);
  cudaFree(c->d_itwp);
  cudaFree(c->d_ctw);
  cudaFree(c->d_ictw);
  cudaFree(c->d_pinv);
  cudaFree(c->d_pinv_sh);
  cudaFree(c->d_pR);
  cudaFree(c->d_rinv);
  cudaFree(c->d_rinv_sh);
  cudaFree(c->d_qmod);
  cudaFree(c->moddown.mem);
  cudaFree(c->moddown.d_dev);
  for (auto& kv : c->modup) {
    for (auto& d : kv.second.digits) {
      cudaFree(d.mem);
      cudaFree(d.d_dev);
    }
    cudaFree(kv.second.d_tabs);
  }
  for (auto& kv : c->generic) {
    cudaFree(kv.second.mem);
    cudaFree(kv.second.d_dev);
  }
  delete c;
}

int hcnn_ctx_psi(const hcnn_ctx* c, uint32_t i, uint64_t* psi) {
  if (!c || i >= c->nmods) return fail(HCNN_E_PARAMETER, "bad modulus index");
  *psi = c->psi[i];
  return HCNN_OK;
}

static int check_basis(const hcnn_ctx* c, u32 nq, u32 np) {
  if (!c) return fail(HCNN_E_PARAMETER, "null context");
  if (nq > c->Lq || np > c->K) return fail(HCNN_E_BASIS, "basis exceeds the context's chain");
  if (nq + np == 0) return fail(HCNN_E_BASIS, "empty basis");
  return HCNN_OK;
}

#define STREAM(s) ((cudaStream_t)(s))

static int ntt_common(hcnn_ctx* c, uint64_t* data, u32 nq, u32 np, u32 npolys, void* s, bool inv) {
  int rc = check_basis(c, nq, np);
  if (rc) return rc;
  LimbMap m{};
  m.base = data;
  m.poly_stride = (size_t)(nq + np) * c->n;
  m.basis = c->basis(nq, np);
  PK(inv ? "ntt_inv" : "ntt_fwd", 16.0 * (nq + np) * npolys * c->n, ntt_nk(c), STREAM(s),
     launch_ntt(c->tables(), m, nq + np, npolys, inv, STREAM(s)));
  return HCNN_OK;
}

int hcnn_ntt_forward(hcnn_ctx* c, uint64_t* data, uint32_t nq, uint32_t np, uint32_t npolys, void* s) {
  return ntt_common(c, data, nq, np, npolys, s, false);
}
int hcnn_ntt_inverse(hcnn_ctx* c, uint64_t* data, uint32_t nq, uint32_t np, uint32_t npolys, void* s) {
  return ntt_common(c, data, nq, np, npolys, s, true);
}

static int binop(hcnn_ctx* c, int op, uint64_t* out, const uint64_t* a, const uint64_t* b, u32 nq, u32 np,
                 u32 npolys, int bc, void* s) {
  int rc = check_basis(c, nq, np);
  if (rc) return rc;
  PK("ew_binary", 24.0 * (nq + np) * npolys * c->n, 1, STREAM(s),
     launch_ew_binary(op, out, a, b, c->basis(nq, np), c->logN, npolys, bc, c->d_mc, STREAM(s)));
  return HCNN_OK;
}
int hcnn_poly_add(hcnn_ctx* c, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t nq, uint32_t np,
                  uint32_t npolys, int bc, void* s) {
  return binop(c, EW_ADD, out, a, b, nq, np, npolys, bc, s);
}
int hcnn_poly_sub(hcnn_ctx* c, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t nq, uint32_t np,
                  uint32_t npolys, int bc, void* s) {
  return binop(c, EW_SUB, out, a, b, nq, np, npolys, bc, s);
}
int hcnn_poly_mul(hcnn_ctx* c, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t nq, uint32_t np,
                  uint32_t npolys, int bc, void* s) {
  return binop(c, EW_MUL, out, a, b, nq, np, npolys, bc, s);
}
int hcnn_poly_mul_mont(hcnn_ctx* c, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t nq, uint32_t np,
                       uint32_t npolys, int bc, void* s) {
  return binop(c, EW_MUL_MONT, out, a, b, nq, np, npolys, bc, s);
}
int hcnn_poly_mac_mont(hcnn_ctx* c, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t nq, uint32_t np,
                       uint32_t npolys, int bc, void* s) {
  return binop(c, EW_MAC_MONT, out, a, b, nq, np, npolys, bc, s);
}

static int unop(hcnn_ctx* c, int op, uint64_t* out, const uint64_t* a, u32 nq, u32 np, u32 npolys, void* s) {
  int rc = check_basis(c, nq, np);
  if (rc) return rc;
  PK("ew_unary", 16.0 * (nq + np) * npolys * c->n, 1, STREAM(s),
     launch_ew_unary(op, out, a, c->basis(nq, np), c->logN, npolys, c->d_mc, nullptr, nullptr, STREAM(s)));
  return HCNN_OK;
}
int hcnn_poly_neg(hcnn_ctx* c, uint64_t* out, const uint64_t* a, uint32_t nq, uint32_t np, uint32_t npolys,
                  void* s) {
  return unop(c, EW_NEG, out, a, nq, np, npolys, s);
}
int hcnn_to_mont(hcnn_ctx* c, uint64_t* out, const uint64_t* a, uint32_t nq, uint32_t np, uint32_t npolys,
                 void* s) {
  return unop(c, EW_TO_MONT, out, a, nq, np, npolys, s);
}
int hcnn_from_mont(hcnn_ctx* c, uint64_t* out, const uint64_t* a, uint32_t nq, uint32_t np, uint32_t npolys,
                   void* s) {
  return unop(c, EW_FROM_MONT, out, a, nq, np, npolys, s);
}

static int scalar_op(hcnn_ctx* c, int op, uint64_t* out, const uint64_t* a, const uint64_t* consts, uint32_t nq,
                     uint32_t np, uint32_t npolys, void* s);

int hcnn_scalar_mul(hcnn_ctx* c, uint64_t* out, const uint64_t* a, const uint64_t* consts, uint32_t nq,
                    uint32_t np, uint32_t npolys, void* s) {
  return scalar_op(c, EW_SCALAR, out, a, consts, nq, np, npolys, s);
}

int hcnn_scalar_add(hcnn_ctx* c, uint64_t* out, const uint64_t* a, const uint64_t* consts, uint32_t nq,
                    uint32_t np, uint32_t npolys, void* s) {
  return scalar_op(c, EW_SCALAR_ADD, out, a, consts, nq, np, npolys, s);
}

static int scalar_op(hcnn_ctx* c, int op, uint64_t* out, const uint64_t* a, const uint64_t* consts, uint32_t nq,
                     uint32_t np, uint32_t npolys, void* s) {
  int rc = check_basis(c, nq, np);
  if (rc) return rc;
  Basis b = c->basis(nq, np);
  const u32 nl = nq + np;
  if (nl > (u32)kScalarMax) return fail(HCNN_E_BASIS, "too many limbs for a scalar op");
  ScalarArgs args;  // by value: capture-safe, no host->device copy
  for (u32 r = 0; r < nl; ++r) {
    u64 q = c->mods[b.mod_of(r)];
    args.w[r] = consts[r] % q;
    args.wp[r] = h_shoup(args.w[r], q);
  }
  PK(op == EW_SCALAR ? "ew_scalar" : "ew_scalar_add", 16.0 * nl * npolys * c->n, 1, STREAM(s),
     launch_scalar(op == EW_SCALAR_ADD ? 1 : 0, out, a, b, c->logN, npolys, c->d_mc, args, STREAM(s)));
  return HCNN_OK;
}

int hcnn_scalar_mac(hcnn_ctx* c, uint64_t* out, const uint64_t* const* srcs, const uint32_t* src_limbs,
                    const uint64_t* consts, uint32_t nterms, uint32_t nq, uint32_t npolys, int accumulate,
                    const uint64_t* c0_add, void* s) {
  int rc = check_basis(c, nq, 0);
  if (rc) return rc;
  if (nq > (u32)kSMacLimbs) return fail(HCNN_E_BASIS, "too many limbs for scalar_mac");
  if (nterms == 0 && accumulate && !c0_add) return HCNN_OK;
  ScalarMacArgs A;  // by value: capture-safe
  u32 t0 = 0;
  do {
    const u32 nt = nterms - t0 < (u32)kSMacTerms ? nterms - t0 : (u32)kSMacTerms;
    for (u32 t = 0; t < nt; ++t) {
      if (src_limbs[t0 + t] < nq) return fail(HCNN_E_BASIS, "scalar_mac source has fewer limbs than the output");
      A.src[t] = srcs[t0 + t];
      A.src_limbs[t] = src_limbs[t0 + t];
      for (u32 r = 0; r < nq; ++r) {
        const u64 q = c->mods[r];
        A.w[t][r] = consts[(size_t)(t0 + t) * nq + r] % q;
        A.wp[t][r] = h_shoup(A.w[t][r], q);
      }
    }
    A.has_add0 = (c0_add && t0 == 0) ? 1 : 0;  // the constant joins the first launch only
    if (A.has_add0)
      for (u32 r = 0; r < nq; ++r) A.add0[r] = c0_add[r] % c->mods[r];
    const int acc = accumulate || t0 > 0;
    PK("scalar_mac", 8.0 * (nt + 1 + (acc ? 1 : 0)) * nq * npolys * c->n, 1, STREAM(s),
       launch_scalar_mac(A, (int)nt, out, nq, c->logN, npolys, acc, c->d_mc, STREAM(s)));
    t0 += nt;
  } while (t0 < nterms);
  return HCNN_OK;
}

static int from_signed(hcnn_ctx* c, uint64_t* out, const int64_t* in, uint32_t nq, uint32_t np, uint32_t npolys,
                       int mont, void* s) {
  int rc = check_basis(c, nq, np);
  if (rc) return rc;
  PK("from_signed", 8.0 * (nq + np + 1) * npolys * c->n, 1, STREAM(s),
     launch_from_signed(out, (const long long*)in, c->basis(nq, np), c->logN, npolys, c->d_mc, mont, STREAM(s)));
  return HCNN_OK;
}

static int from_signed(hcnn_ctx* c, uint64_t* out, const int64_t* in, uint32_t nq, uint32_t np, uint32_t npolys,
                       int mont, void* s);

int hcnn_ntt_from_signed(hcnn_ctx* c, uint64_t* out, const int64_t* in, uint32_t nq, uint32_t npolys, int mont,
                         void* s) {
  int rc = check_basis(c, nq, 0);
  if (rc) return rc;
  LimbMap m{};
  m.base = out;
  m.poly_stride = (size_t)nq * c->n;
  m.basis = c->basis(nq, 0);
  if (c->tables().ctw) {  // fused: the column pass reduces the int64 rows on load
    m.sin = (const long long*)in;
    m.smont = mont;
    PK("ntt_fwd_signed", 8.0 * (1 + 2 * (double)nq) * npolys * c->n, ntt_nk(c), STREAM(s),
       launch_ntt(c->tables(), m, nq, npolys, false, STREAM(s)));
    return HCNN_OK;
  }
  rc = from_signed(c, out, in, nq, 0, npolys, mont, s);
  if (rc) return rc;
  PK("ntt_fwd_signed", 16.0 * nq * npolys * c->n, ntt_nk(c), STREAM(s),
     launch_ntt(c->tables(), m, nq, npolys, false, STREAM(s)));
  return HCNN_OK;
}

int hcnn_from_signed(hcnn_ctx* c, uint64_t* out, const int64_t* in, uint32_t nq, uint32_t np, uint32_t npolys,
                     void* s) {
  return from_signed(c, out, in, nq, np, npolys, 0, s);
}

int hcnn_from_signed_mont(hcnn_ctx* c, uint64_t* out, const int64_t* in, uint32_t nq, uint32_t np,
                          uint32_t npolys, void* s) {
  return from_signed(c, out, in, nq, np, npolys, 1, s);
}

int hcnn_automorphism(hcnn_ctx* c, uint64_t* out, const uint64_t* in, uint64_t g, int eval_domain, uint32_t nq,
                      uint32_t np, uint32_t npolys, void* s) {
  int rc = check_basis(c, nq, np);
  if (rc) return rc;
  if ((g & 1) == 0) return fail(HCNN_E_PARAMETER, "automorphism exponent must be odd");
  g %= 2ull * c->n;
  PK("automorph", 16.0 * (nq + np) * npolys * c->n, 1, STREAM(s),
     launch_automorph(eval_domain, out, in, c->basis(nq, np), c->logN, npolys, g, c->d_mc, STREAM(s)));
  return HCNN_OK;
}

int hcnn_base_convert(hcnn_ctx* c, uint64_t* out, const uint64_t* in, const uint32_t* src_mods, uint32_t n_src,
                      const uint32_t* dst_mods, uint32_t n_dst, uint32_t npolys, void* s) {
  if (!c) return fail(HCNN_E_PARAMETER, "null context");
  if (n_src == 0 || n_dst == 0) return fail(HCNN_E_BASIS, "empty basis");
  if (n_src > 64) return fail(HCNN_E_BASIS, "at most 64 source limbs");
  std::vector<u32> key;
  key.push_back(n_src);
  for (u32 i = 0; i < n_src; ++i) {
    if (src_mods[i] >= c->nmods) return fail(HCNN_E_BASIS, "bad source modulus index");
    key.push_back(src_mods[i]);
  }
  for (u32 i = 0; i < n_dst; ++i) {
    if (dst_mods[i] >= c->nmods) return fail(HCNN_E_BASIS, "bad target modulus index");
    key.push_back(dst_mods[i]);
  }
  FbcStore* st;
  {
    std::lock_guard<std::mutex> lk(c->mu);
    auto it = c->generic.find(key);
    if (it == c->generic.end()) {
      std::vector<u32> src(src_mods, src_mods + n_src), dst(dst_mods, dst_mods + n_dst), pos(n_dst);
      for (u32 i = 0; i < n_dst; ++i) pos[i] = i;
      FbcStore fs;
      int rc = build_fbc(c, src, dst, pos, &fs);
      if (rc) return rc;
      it = c->generic.emplace(key, fs).first;
    }
    st = &it->second;
  }
  PK("fbc", 8.0 * (n_src + n_dst) * npolys * c->n, 1, STREAM(s),
     launch_fbc(st->dev, st->d_dev, c->d_mc, in, (size_t)n_src * c->n, out, (size_t)n_dst * c->n, c->logN, npolys, n_dst,
                STREAM(s)));
  return HCNN_OK;
}

// ---------------------------------------------------------------------------
// key switching
// workspace: xc [nq] | raised [d][n_ext] | acc [2][n_ext] | lift [2][nq]  (limbs of N u64)
// ---------------------------------------------------------------------------
struct KsWs {
  u64 *xc, *raised, *acc, *lift;
};
// batched layout: xc [nb][nq] | raised [nb][d][n_ext] | acc [nb][2][n_ext] | lift [nb][2][nq]
static KsWs ks_layout(const hcnn_ctx* c, u32 level, void* ws, u32 nb = 1, u32 n_steps = 1) {
  const u32 nq = level + 1, n_ext = nq + c->K, nd = (nq + c->alpha - 1) / c->alpha;
  const size_t N = c->n;
  KsWs w;
  w.xc = (u64*)ws;
  w.raised = w.xc + (size_t)nb * nq * N;
  w.acc = w.raised + (size_t)nb * nd * n_ext * N;
  w.lift = w.acc + (size_t)n_steps * nb * 2 * n_ext * N;
  return w;
}

size_t hcnn_ks_workspace_bytes(const hcnn_ctx* c, uint32_t level) {
  const u32 nq = level + 1, n_ext = nq + c->K, nd = (nq + c->alpha - 1) / c->alpha;
  return ((size_t)nq + (size_t)nd * n_ext + 2 * (size_t)n_ext + 2 * (size_t)nq) * c->n * 8;
}

size_t hcnn_ks_workspace_bytes_batch(const hcnn_ctx* c, uint32_t level, uint32_t nb) {
  return hcnn_ks_workspace_bytes(c, level) * (nb ? nb : 1);
}

int g_merge_moddown = 1;  // rotations of a hoisted group share one ModDown chain

// steps of a hoisted group that share one ModDown chain: bounded so the
// extra acc/lift workspace stays under 1 GiB
static u32 merge_chunk(const hcnn_ctx* c, u32 level, u32 nb, u32 n_rot) {
  if (!g_merge_moddown || n_rot < 2) return 1;
  const u32 nq = level + 1, n_ext = nq + c->K;
  const size_t per_step = (size_t)(nb ? nb : 1) * (2 * (size_t)n_ext + 2 * (size_t)nq) * c->n * 8;
  size_t chunk = (1ull << 30) / (per_step ? per_step : 1);
  if (chunk > n_rot) chunk = n_rot;
  if (chunk > (size_t)kComboMax) chunk = kComboMax;
  return chunk < 1 ? 1 : (u32)chunk;
}

// hoisted rotation groups finish chunks of steps together: acc / lift for merge_chunk steps
size_t hcnn_ks_workspace_bytes_rot(const hcnn_ctx* c, uint32_t level, uint32_t nb, uint32_t n_rot) {
  const u32 nq = level + 1, n_ext = nq + c->K, ch = merge_chunk(c, level, nb, n_rot);
  const size_t extra = (size_t)(ch - 1) * (nb ? nb : 1) * (2 * (size_t)n_ext + 2 * (size_t)nq);
  return hcnn_ks_workspace_bytes_batch(c, level, nb) + extra * c->n * 8;
}

// first Q row from which every modulus of the first nq is below 2^42: the
// key-switch inner product runs those rows with 96-bit carry-chain MACs
static u32 ks_fast_from(const hcnn_ctx* c, u32 nq) {
  u32 ff = nq;
  while (ff > 1 && c->mods[ff - 1] < (1ull << 42)) --ff;
  return ff;
}

// ModUp of nb polys (entry b at x_eval + b*x_bst): iNTT a copy, convert
// every digit to Q_l||P, NTT the new limbs -- one launch per step for the batch
static int ks_modup(hcnn_ctx* c, u32 level, const u64* x_eval, const KsWs& w, cudaStream_t st, u32 nb = 1,
                    size_t x_bst = 0) {
  const u32 nq = level + 1, n_ext = nq + c->K, nd = (nq + c->alpha - 1) / c->alpha;
  const size_t N = c->n;
  ModupSet* mu;
  int rc = get_modup(c, level, &mu);
  if (rc) return rc;
  if (nb == 1 || x_bst == nq * N)
    CK(cudaMemcpyAsync(w.xc, x_eval, (size_t)nb * nq * N * 8, cudaMemcpyDeviceToDevice, st));
  else
    CK(cudaMemcpy2DAsync(w.xc, nq * N * 8, x_eval, x_bst * 8, nq * N * 8, nb, cudaMemcpyDeviceToDevice, st));
  LimbMap m{};
  m.base = w.xc;
  m.poly_stride = nq * N;
  m.basis = c->basis(nq, 0);
  ks_acc(1, 8.0 * nb * nq * N);
  ks_acc(2, (double)nb * ((double)nd * n_ext - nq));
  ks_acc(3, (double)nb * nq);
  PK("ntt_inv_modup", 16.0 * nb * nq * N, ntt_nk(c), st, launch_ntt(c->tables(), m, nq, nb, true, st));
  PK("modup", 8.0 * nb * (nq + (double)nd * (n_ext - c->alpha)) * N, 1, st,
     launch_modup(mu->d_tabs, mu->host.data(), nd, c->d_mc, w.xc, w.raised, c->alpha, n_ext, c->logN, st, nb,
                  nq * N));
  LimbMap r{};
  r.base = w.raised;
  r.poly_stride = (size_t)n_ext * N;
  r.basis = c->basis(nq, c->K);
  r.skip_alpha = c->alpha;
  r.zmod = nd;
  PK("ntt_fwd_modup", 16.0 * nb * ((double)nd * n_ext - nq) * N, ntt_nk(c), st,
     launch_ntt(c->tables(), r, n_ext, nd * nb, false, st));
  return HCNN_OK;
}

// ModDown of nb extended-basis ciphertexts acc [nb][2][n_ext] (P limbs are
// clobbered by the in-place iNTT) + combine: out = (acc_Q - lift) P^-1 (+ add)
static int ks_moddown(hcnn_ctx* c, u32 level, u64* acc, u64* lift, u64* out0, u64* out1, const u64* add0,
                      const u64* add1, u64 g_add, cudaStream_t st, u32 nb, size_t out_bst, size_t add_bst) {
  const u32 nq = level + 1, n_ext = nq + c->K;
  const size_t N = c->n;
  LimbMap m{};
  m.base = acc + nq * N;
  m.poly_stride = (size_t)n_ext * N;
  m.basis = c->basis(nq, c->K);
  m.first_limb = nq;
  ks_acc(2, 2.0 * nb * nq);
  ks_acc(3, 2.0 * nb * c->K);
  PK("ntt_inv_moddown", 16.0 * 2 * nb * c->K * N, ntt_nk(c), st, launch_ntt(c->tables(), m, c->K, 2 * nb, true, st));
  PK("moddown_fbc", 8.0 * 2 * nb * (c->K + nq) * N, 1, st,
     launch_fbc(c->moddown.dev, c->moddown.d_dev, c->d_mc, acc + nq * N, (size_t)n_ext * N, lift, nq * N,
                c->logN, 2 * nb, nq, st));
  LimbMap l{};
  l.base = lift;
  l.poly_stride = nq * N;
  l.basis = c->basis(nq, 0);
  // the combine rides on the lift NTT's store when the outputs are laid out
  // [c0 | c1] (out1 = out0 + nq N, add1 = add0 + nq N or absent)
  NttCombine cb{};
  const bool fuse = g_ntt_tuning.md_fuse && g_ntt_tuning.group_limbs == 0 && out1 == out0 + (size_t)nq * N &&
                    (!add1 || (add0 && add1 == add0 + (size_t)nq * N));
  if (fuse) {
    cb.acc = acc;
    cb.acc_pst = (size_t)n_ext * N;
    cb.pinv = c->d_pinv;
    cb.pinv_sh = c->d_pinv_sh;
    cb.nb = nb;
    cb.out_bst = out_bst;
    cb.out_pst = (size_t)nq * N;
    cb.add_bst = add_bst;
    cb.add[0] = add0;
    cb.add[1] = add1;
    cb.out[0] = out0;
    cb.g[0] = g_add;
    l.cb = &cb;
  }
  PK("ntt_fwd_moddown", 16.0 * 2 * nb * nq * N, ntt_nk(c), st, launch_ntt(c->tables(), l, nq, 2 * nb, false, st));
  if (!fuse)
    PK("moddown_combine", 8.0 * 2 * nb * (3 * nq + (add0 ? nq : 0)) * N, 1, st,
       launch_moddown_combine(out0, out1, acc, lift, add0, add1, g_add, nq, n_ext, c->logN, c->d_pinv,
                              c->d_pinv_sh, c->d_mc, st, nb, out_bst, add_bst));
  return HCNN_OK;
}

// inner product with one key (optionally Galois-permuted) + ModDown + combine,
// for nb entries: outputs / addends of entry b at +b*out_bst / +b*add_bst
static int ks_finish(hcnn_ctx* c, u32 level, const u64* x_eval, const KsWs& w, u64 g, const u64* kb,
                     const u64* ka, u64* out0, u64* out1, const u64* add0, const u64* add1, u64 g_add,
                     cudaStream_t st, u32 nb = 1, size_t x_bst = 0, size_t out_bst = 0, size_t add_bst = 0,
                     u32 key_lq = 0) {
  const u32 nq = level + 1, n_ext = nq + c->K, nd = (nq + c->alpha - 1) / c->alpha;
  const size_t N = c->n;
  ks_acc(0, nb);
  ks_acc(1, 8.0 * (2.0 * nd * n_ext + 2.0 * nb * nq) * N);
  PK("ks_inner", 8.0 * ((double)nd * n_ext * (2 + nb) + 2.0 * nb * n_ext) * N, 1, st,
     launch_ks_inner(w.acc, x_eval, w.raised, kb, ka, c->basis(nq, c->K), c->alpha, nd, c->logN, g, c->d_mc, st,
                     nb, x_bst, nullptr, 0, nullptr, key_lq, ks_fast_from(c, nq)));
  return ks_moddown(c, level, w.acc, w.lift, out0, out1, add0, add1, g_add, st, nb, out_bst, add_bst);
}

static int check_level(const hcnn_ctx* c, u32 level) {
  if (!c) return fail(HCNN_E_PARAMETER, "null context");
  if (level >= c->Lq) return fail(HCNN_E_LEVEL, "level outside chain");
  if (c->K == 0) return fail(HCNN_E_KEY, "no special primes: key switching unavailable");
  return HCNN_OK;
}

int hcnn_keyswitch(hcnn_ctx* c, uint64_t* out0, uint64_t* out1, const uint64_t* x_eval, uint32_t level,
                   const uint64_t* kb, const uint64_t* ka, void* ws, void* s) {
  int rc = check_level(c, level);
  if (rc) return rc;
  KsWs w = ks_layout(c, level, ws);
  rc = ks_modup(c, level, x_eval, w, STREAM(s));
  if (rc) return rc;
  return ks_finish(c, level, x_eval, w, 1, kb, ka, out0, out1, nullptr, nullptr, 1, STREAM(s));
}

int hcnn_hmult_batch(hcnn_ctx* c, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t level, uint32_t nb,
                     const uint64_t* kb, const uint64_t* ka, void* ws, void* s) {
  int rc = check_level(c, level);
  if (rc) return rc;
  if (nb == 0) return HCNN_OK;
  const u32 nq = level + 1;
  const size_t N = c->n, ct = 2 * (size_t)nq * N;
  KsWs w = ks_layout(c, level, ws, nb);
  // d2 of entry e parked in the first half of its ModDown scratch until the inner product
  for (u32 e = 0; e < nb; ++e)
    PK("tensor", 8.0 * 7 * nq * N, 1, STREAM(s),
       launch_tensor(out + e * ct, out + e * ct + nq * N, w.lift + e * ct, a + e * ct, b + e * ct, nq, c->logN,
                     c->d_mc, STREAM(s)));
  rc = ks_modup(c, level, w.lift, w, STREAM(s), nb, ct);
  if (rc) return rc;
  return ks_finish(c, level, w.lift, w, 1, kb, ka, out, out + nq * N, out, out + nq * N, 1, STREAM(s), nb, ct, ct,
                   ct);
}

int hcnn_hmult(hcnn_ctx* c, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t level,
               const uint64_t* kb, const uint64_t* ka, void* ws, void* s) {
  return hcnn_hmult_batch(c, out, a, b, level, 1, kb, ka, ws, s);
}

static int key_lq_ok(const hcnn_ctx* c, const uint32_t* key_lqs, uint32_t n, uint32_t level) {
  for (uint32_t i = 0; key_lqs && i < n; ++i)
    if (key_lqs[i] && (key_lqs[i] <= level || key_lqs[i] > c->Lq))
      return fail(HCNN_E_KEY, "rotation key truncated below the ciphertext level");
  return HCNN_OK;
}

int hcnn_rotate_hoisted_batch(hcnn_ctx* c, uint64_t* const* outs, const uint64_t* cts, uint32_t level, uint32_t nb,
                              uint32_t n_rot, const uint64_t* galois, const uint64_t* const* kbs,
                              const uint64_t* const* kas, const uint32_t* key_lqs, void* ws, void* s) {
  int rc = check_level(c, level);
  if (rc) return rc;
  if (nb == 0) return HCNN_OK;
  const u32 nq = level + 1;
  const size_t N = c->n, ct = 2 * (size_t)nq * N;
  for (u32 i = 0; i < n_rot; ++i)
    if ((galois[i] % (2ull * c->n) & 1) == 0) return fail(HCNN_E_PARAMETER, "galois element must be odd");
  rc = key_lq_ok(c, key_lqs, n_rot, level);
  if (rc) return rc;
  const u32 chunk = merge_chunk(c, level, nb, n_rot);
  KsWs w = ks_layout(c, level, ws, nb, chunk);
  const u64* c1 = cts + nq * N;
  rc = ks_modup(c, level, c1, w, STREAM(s), nb, ct);
  if (rc) return rc;
  if (chunk < 2) {
    for (u32 i = 0; i < n_rot; ++i) {
      u64 g = galois[i] % (2ull * c->n);
      rc = ks_finish(c, level, c1, w, g, kbs[i], kas[i], outs[i], outs[i] + nq * N, cts, nullptr, g, STREAM(s), nb,
                     ct, ct, ct, key_lqs ? key_lqs[i] : 0);
      if (rc) return rc;
    }
    return HCNN_OK;
  }
  // per chunk: inner products of every step into acc[step], then one ModDown chain
  const u32 n_ext = nq + c->K, nd = (nq + c->alpha - 1) / c->alpha;
  const size_t a_step = (size_t)nb * 2 * n_ext * N;
  for (u32 i0 = 0; i0 < n_rot; i0 += chunk) {
    const u32 nr = n_rot - i0 < chunk ? n_rot - i0 : chunk;
    ComboSteps S;
    // the chunk's inner products: one launch for all its rotations when
    // ks_rots_ok (raised digits read from HBM once per chunk), else one each
    // (sub-groups of up to kKsRotMax rotations per launch)
    const bool rots = ks_rots_ok(nb, nr, c->logN);
    for (u32 j0 = 0; j0 < nr; j0 += (u32)kKsRotMax) {
      const u32 nj = nr - j0 < (u32)kKsRotMax ? nr - j0 : (u32)kKsRotMax;
      KsRots R{};
      for (u32 jj = 0; jj < nj; ++jj) {
        const u32 j = j0 + jj, i = i0 + j;
        const u64 g = galois[i] % (2ull * c->n);
        S.out[j] = outs[i];
        S.g[j] = g;
        ks_acc(0, nb);
        ks_acc(1, 8.0 * (2.0 * nd * n_ext + 2.0 * nb * nq) * N);
        if (rots && nj >= 2) {
          R.acc[jj] = w.acc + j * a_step;
          R.kb[jj] = kbs[i];
          R.ka[jj] = kas[i];
          R.g[jj] = g;
          R.klq[jj] = key_lqs ? key_lqs[i] : 0;
          continue;
        }
        PK("ks_inner", 8.0 * ((double)nd * n_ext * (2 + nb) + 2.0 * nb * n_ext) * N, 1, STREAM(s),
           launch_ks_inner(w.acc + j * a_step, c1, w.raised, kbs[i], kas[i], c->basis(nq, c->K), c->alpha, nd,
                           c->logN, g, c->d_mc, STREAM(s), nb, ct, nullptr, 0, nullptr, key_lqs ? key_lqs[i] : 0,
                           ks_fast_from(c, nq)));
      }
      if (rots && nj >= 2)
        PK("ks_inner", 8.0 * nj * ((double)nd * n_ext * (2 + nb) + 2.0 * nb * n_ext) * N, 1, STREAM(s),
           launch_ks_inner_rots(R, nj, c1, w.raised, c->basis(nq, c->K), c->alpha, nd, c->logN, c->d_mc,
                                STREAM(s), nb, ct));
    }
    const u32 np = 2 * nb * nr;
    LimbMap m{};
    m.base = w.acc + nq * N;
    m.poly_stride = (size_t)n_ext * N;
    m.basis = c->basis(nq, c->K);
    m.first_limb = nq;
    ks_acc(2, (double)np * nq);
    ks_acc(3, (double)np * c->K);
    PK("ntt_inv_moddown", 16.0 * np * c->K * N, ntt_nk(c), STREAM(s),
       launch_ntt(c->tables(), m, c->K, np, true, STREAM(s)));
    PK("moddown_fbc", 8.0 * np * (c->K + nq) * N, 1, STREAM(s),
       launch_fbc(c->moddown.dev, c->moddown.d_dev, c->d_mc, w.acc + nq * N, (size_t)n_ext * N, w.lift, nq * N,
                  c->logN, np, nq, STREAM(s)));
    LimbMap l{};
    l.base = w.lift;
    l.poly_stride = nq * N;
    l.basis = c->basis(nq, 0);
    NttCombine cb{};
    const bool fuse = g_ntt_tuning.md_fuse && g_ntt_tuning.group_limbs == 0 && nr <= (u32)kCombineMax;
    if (fuse) {
      cb.acc = w.acc;
      cb.acc_pst = (size_t)n_ext * N;
      cb.pinv = c->d_pinv;
      cb.pinv_sh = c->d_pinv_sh;
      cb.nb = nb;
      cb.out_bst = ct;
      cb.out_pst = (size_t)nq * N;
      cb.add_bst = ct;
      cb.add[0] = cts;
      cb.add[1] = nullptr;
      for (u32 j = 0; j < nr; ++j) {
        cb.out[j] = S.out[j];
        cb.g[j] = S.g[j];
      }
      l.cb = &cb;
    }
    PK("ntt_fwd_moddown", 16.0 * np * nq * N, ntt_nk(c), STREAM(s),
       launch_ntt(c->tables(), l, nq, np, false, STREAM(s)));
    if (!fuse)
      PK("moddown_combine", 8.0 * np * 4 * nq * N, 1, STREAM(s),
         launch_moddown_combine_steps(S, nr, w.acc, w.lift, cts, nb, nq, n_ext, c->logN, c->d_pinv, c->d_pinv_sh,
                                      c->d_mc, ct, ct, STREAM(s)));
  }
  return HCNN_OK;
}

int hcnn_rotate_hoisted_ext_batch(hcnn_ctx* c, uint64_t* const* outs, const uint64_t* cts, uint32_t level,
                                  uint32_t nb, uint32_t n_rot, const uint64_t* galois, const uint64_t* const* kbs,
                                  const uint64_t* const* kas, const uint32_t* key_lqs, void* ws, void* s) {
  int rc = check_level(c, level);
  if (rc) return rc;
  if (nb == 0) return HCNN_OK;
  const u32 nq = level + 1, n_ext = nq + c->K, nd = (nq + c->alpha - 1) / c->alpha;
  const size_t N = c->n, ct = 2 * (size_t)nq * N;
  for (u32 i = 0; i < n_rot; ++i)
    if ((galois[i] % (2ull * c->n) & 1) == 0) return fail(HCNN_E_PARAMETER, "galois element must be odd");
  rc = key_lq_ok(c, key_lqs, n_rot, level);
  if (rc) return rc;
  KsWs w = ks_layout(c, level, ws, nb);
  const u64* c1 = cts + nq * N;
  rc = ks_modup(c, level, c1, w, STREAM(s), nb, ct);
  if (rc) return rc;
  // groups of up to kKsRotMax rotations in one launch when ks_rots_ok
  for (u32 i0 = 0; i0 < n_rot; i0 += (u32)kKsRotMax) {
    const u32 nr = n_rot - i0 < (u32)kKsRotMax ? n_rot - i0 : (u32)kKsRotMax;
    const bool rots = ks_rots_ok(nb, nr, c->logN);
    KsRots R{};
    for (u32 j = 0; j < nr; ++j) {
      const u32 i = i0 + j;
      const u64 g = galois[i] % (2ull * c->n);
      ks_acc(0, nb);
      ks_acc(1, 8.0 * (2.0 * nd * n_ext + 2.0 * nb * n_ext + nb * nq) * N);
      if (rots) {
        R.acc[j] = outs[i];
        R.kb[j] = kbs[i];
        R.ka[j] = kas[i];
        R.g[j] = g;
        R.klq[j] = key_lqs ? key_lqs[i] : 0;
        continue;
      }
      PK("ks_inner", 8.0 * ((double)nd * n_ext * (2 + nb) + 2.0 * nb * n_ext + nb * nq) * N, 1, STREAM(s),
         launch_ks_inner(outs[i], c1, w.raised, kbs[i], kas[i], c->basis(nq, c->K), c->alpha, nd, c->logN, g,
                         c->d_mc, STREAM(s), nb, ct, cts, ct, c->d_pR, key_lqs ? key_lqs[i] : 0, ks_fast_from(c, nq)));
    }
    if (rots)
      PK("ks_inner", 8.0 * nr * ((double)nd * n_ext * (2 + nb) + 2.0 * nb * n_ext + nb * nq) * N, 1, STREAM(s),
         launch_ks_inner_rots(R, nr, c1, w.raised, c->basis(nq, c->K), c->alpha, nd, c->logN, c->d_mc, STREAM(s),
                              nb, ct, cts, ct, c->d_pR));
  }
  return HCNN_OK;
}

// (Q_l||P ciphertexts) -> round(x / (P q_l)) over Q_{l-1}: ModDown and the
// following rescale with one base conversion -- iNTT of the K+1 limbs
// (q_l, P), centred FBC to q_0..q_{l-1}, NTT of l limbs, combine.
static int moddown_rescale(hcnn_ctx* c, u32 level, u64* in_ext, u64* lift, u64* out, u32 nb, cudaStream_t st) {
  if (c->K + 1 > 6) return fail(HCNN_E_PARAMETER, "fused ModDown+rescale needs K + 1 <= 6");
  hcnn_ctx::MdrSet* md;
  int rc = get_mdr(c, level, &md);
  if (rc) return rc;
  const u32 nq = level + 1, n_ext = nq + c->K, l = level;
  const size_t N = c->n;
  LimbMap m{};
  m.base = in_ext + (size_t)l * N;
  m.poly_stride = (size_t)n_ext * N;
  m.basis = c->basis(nq, c->K);
  m.first_limb = l;
  ks_acc(2, 2.0 * nb * l);
  ks_acc(3, 2.0 * nb * (c->K + 1));
  PK("ntt_inv_moddown", 16.0 * 2 * nb * (c->K + 1) * N, ntt_nk(c), st,
     launch_ntt(c->tables(), m, c->K + 1, 2 * nb, true, st));
  PK("moddown_fbc", 8.0 * 2 * nb * (c->K + 1 + l) * N, 1, st,
     launch_fbc(md->fbc.dev, md->fbc.d_dev, c->d_mc, in_ext + (size_t)l * N, (size_t)n_ext * N, lift, (size_t)l * N,
                c->logN, 2 * nb, l, st));
  LimbMap f{};
  f.base = lift;
  f.poly_stride = (size_t)l * N;
  f.basis = c->basis(l, 0);
  PK("ntt_fwd_moddown", 16.0 * 2 * nb * l * N, ntt_nk(c), st, launch_ntt(c->tables(), f, l, 2 * nb, false, st));
  PK("moddown_combine", 8.0 * 2 * nb * 3 * l * N, 1, st,
     launch_moddown_combine(out, out + (size_t)l * N, in_ext, lift, nullptr, nullptr, 1, l, n_ext, c->logN,
                            md->d_inv, md->d_inv_sh, c->d_mc, st, nb, 2 * (size_t)l * N, 0));
  return HCNN_OK;
}

// (Q_l||P ciphertexts) -> round(x / (P q_l)) over Q_{l-1}: ModDown and the
// following rescale with one base conversion -- iNTT of the K+1 limbs
// (q_l, P), centred FBC to q_0..q_{l-1}, NTT of l limbs, combine.
int hcnn_moddown_rescale_batch(hcnn_ctx* c, uint64_t* out, uint64_t* in_ext, uint32_t level, uint32_t nb, void* ws,
                               void* s) {
  int rc = check_level(c, level);
  if (rc) return rc;
  if (level == 0) return fail(HCNN_E_LEVEL, "no limb left to rescale away");
  if (nb == 0) return HCNN_OK;
  KsWs w = ks_layout(c, level, ws, nb);
  return moddown_rescale(c, level, in_ext, w.lift, out, nb, STREAM(s));
}

size_t hcnn_hmult_rescale_workspace_bytes(const hcnn_ctx* c, uint32_t level, uint32_t nb) {
  return hcnn_ks_workspace_bytes_batch(c, level, nb) + 2ull * (nb ? nb : 1) * (level + 1) * c->n * 8;
}

// tensor + relinearisation + rescale with one ModDown: the key-switch sum and
// P (d0, d1) are accumulated over Q_l||P and divided by P q_l at once
// (bootstrapping's EvalMod products; no reference counterpart).
int hcnn_hmult_rescale_batch(hcnn_ctx* c, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t level,
                             uint32_t nb, const uint64_t* kb, const uint64_t* ka, void* ws, void* s) {
  int rc = check_level(c, level);
  if (rc) return rc;
  if (level == 0) return fail(HCNN_E_LEVEL, "no limb left to rescale away");
  if (nb == 0) return HCNN_OK;
  const u32 nq = level + 1, n_ext = nq + c->K, nd = (nq + c->alpha - 1) / c->alpha;
  const size_t N = c->n, ct = 2 * (size_t)nq * N;
  KsWs w = ks_layout(c, level, ws, nb);
  u64* d01 = (u64*)((char*)ws + hcnn_ks_workspace_bytes_batch(c, level, nb));  // [nb][2][nq]
  for (u32 e = 0; e < nb; ++e)
    PK("tensor", 8.0 * 7 * nq * N, 1, STREAM(s),
       launch_tensor(d01 + e * ct, d01 + e * ct + nq * N, w.lift + e * ct, a + e * ct, b + e * ct, nq, c->logN,
                     c->d_mc, STREAM(s)));
  rc = ks_modup(c, level, w.lift, w, STREAM(s), nb, ct);
  if (rc) return rc;
  ks_acc(0, nb);
  ks_acc(1, 8.0 * (2.0 * nd * n_ext + 2.0 * nb * nq) * N);
  PK("ks_inner", 8.0 * ((double)nd * n_ext * (2 + nb) + 2.0 * nb * n_ext) * N, 1, STREAM(s),
     launch_ks_inner(w.acc, w.lift, w.raised, kb, ka, c->basis(nq, c->K), c->alpha, nd, c->logN, 1, c->d_mc,
                     STREAM(s), nb, ct, nullptr, 0, nullptr, 0, ks_fast_from(c, nq)));
  PK("add_pmul", 8.0 * 2 * nb * 3 * nq * N, 1, STREAM(s),
     launch_add_pmul(w.acc, d01, nb, nq, n_ext, c->logN, c->d_pR, c->d_mc, STREAM(s)));
  return moddown_rescale(c, level, w.acc, w.lift, out, nb, STREAM(s));
}

int hcnn_moddown_batch(hcnn_ctx* c, uint64_t* out, uint64_t* in_ext, uint32_t level, uint32_t nb, void* ws, void* s) {
  int rc = check_level(c, level);
  if (rc) return rc;
  if (nb == 0) return HCNN_OK;
  const u32 nq = level + 1;
  const size_t N = c->n, ct = 2 * (size_t)nq * N;
  KsWs w = ks_layout(c, level, ws, nb);
  return ks_moddown(c, level, in_ext, w.lift, out, out + nq * N, nullptr, nullptr, 1, STREAM(s), nb, ct, 0);
}

int hcnn_rotate_hoisted(hcnn_ctx* c, uint64_t* const* outs, const uint64_t* ct, uint32_t level, uint32_t n_rot,
                        const uint64_t* galois, const uint64_t* const* kbs, const uint64_t* const* kas, void* ws,
                        void* s) {
  return hcnn_rotate_hoisted_batch(c, outs, ct, level, 1, n_rot, galois, kbs, kas, nullptr, ws, s);
}

int hcnn_mac_terms_batch(hcnn_ctx* c, uint64_t* out, const uint64_t* const* cts, const uint64_t* const* masks,
                         uint32_t n_terms, uint32_t level, uint32_t nb, int accumulate, void* s);

int hcnn_mac_terms(hcnn_ctx* c, uint64_t* out, const uint64_t* const* cts, const uint64_t* const* masks,
                   uint32_t n_terms, uint32_t level, int accumulate, void* s) {
  return hcnn_mac_terms_batch(c, out, cts, masks, n_terms, level, 1, accumulate, s);
}

static int mac_terms_impl(hcnn_ctx* c, uint64_t* out, const uint64_t* const* cts, const uint64_t* const* masks,
                          uint32_t n_terms, uint32_t level, uint32_t nb, uint32_t np, int accumulate, void* s);

int hcnn_mac_terms_batch(hcnn_ctx* c, uint64_t* out, const uint64_t* const* cts, const uint64_t* const* masks,
                         uint32_t n_terms, uint32_t level, uint32_t nb, int accumulate, void* s) {
  return mac_terms_impl(c, out, cts, masks, n_terms, level, nb, 0, accumulate, s);
}

int hcnn_mac_terms_ext_batch(hcnn_ctx* c, uint64_t* out, const uint64_t* const* cts, const uint64_t* const* masks,
                             uint32_t n_terms, uint32_t level, uint32_t nb, int accumulate, void* s) {
  if (c && c->K == 0) return fail(HCNN_E_KEY, "no special primes");
  return mac_terms_impl(c, out, cts, masks, n_terms, level, nb, c ? c->K : 0, accumulate, s);
}

static int mac_terms_impl(hcnn_ctx* c, uint64_t* out, const uint64_t* const* cts, const uint64_t* const* masks,
                          uint32_t n_terms, uint32_t level, uint32_t nb, uint32_t np, int accumulate, void* s) {
  if (!c) return fail(HCNN_E_PARAMETER, "null context");
  if (level >= c->Lq) return fail(HCNN_E_LEVEL, "level outside chain");
  const u32 nq = level + 1;
  if (nb == 0) return HCNN_OK;
  if (n_terms == 0) {
    if (!accumulate) CK(cudaMemsetAsync(out, 0, 2ull * nb * (nq + np) * c->n * 8, STREAM(s)));
    return HCNN_OK;
  }
  for (u32 t0 = 0; t0 < n_terms; t0 += kMacMax) {
    MacTerms T;
    u32 nt = std::min<u32>(kMacMax, n_terms - t0);
    for (u32 t = 0; t < nt; ++t) {
      T.ct[t] = cts[t0 + t];
      T.mask[t] = masks[t0 + t];
    }
    PK("mac_terms", 8.0 * ((2.0 * nb + 1) * nt + nb * (2 + (accumulate || t0 ? 2 : 0))) * (nq + np) * c->n, 1,
       STREAM(s), launch_mac_terms(T, (int)nt, out, nq, c->logN, accumulate || t0 > 0, c->d_mc, STREAM(s), nb, np,
                                   c->Lq));
  }
  return HCNN_OK;
}

static int masks_packable(const hcnn_ctx* c, u32 nq) {
  if (nq > 63) return 0;  // packed_hb / packed_hi_off shift 1ull << nq
  for (u32 r = 1; r < nq; ++r)
    if (c->mods[r] >> 48) return 0;
  return 1;
}

int hcnn_pack_masks(hcnn_ctx* c, void* out, const uint64_t* in, uint32_t n_masks, uint32_t level, void* s) {
  if (!c) return fail(HCNN_E_PARAMETER, "null context");
  if (level >= c->Lq) return fail(HCNN_E_LEVEL, "level outside chain");
  if (!masks_packable(c, level + 1)) return fail(HCNN_E_BASIS, "a modulus above 2^48: masks not packable");
  PK("pack_masks", (8.0 * (level + 1) + packed_hi_off(level + 1, level + 1, 1, c->wide)) * n_masks * c->n, 1,
     STREAM(s), launch_pack_masks((unsigned char*)out, in, n_masks, level + 1, c->logN, c->wide, STREAM(s)));
  return HCNN_OK;
}

int hcnn_unpack_mask(hcnn_ctx* c, uint64_t* out, const void* in, uint32_t level, void* s) {
  if (!c) return fail(HCNN_E_PARAMETER, "null context");
  if (level >= c->Lq) return fail(HCNN_E_LEVEL, "level outside chain");
  PK("unpack_mask", (8.0 * (level + 1) + packed_hi_off(level + 1, level + 1, 1, c->wide)) * c->n, 1, STREAM(s),
     launch_unpack_mask(out, (const unsigned char*)in, level + 1, c->logN, c->wide, STREAM(s)));
  return HCNN_OK;
}

int hcnn_mac_terms_multi(hcnn_ctx* c, uint64_t* const* outs, const uint64_t* const* cts,
                         const uint64_t* const* masks, uint32_t n_out, uint32_t n_terms, uint32_t level, int accumulate,
                         void* s) {
  return hcnn_mac_terms_multi_packed(c, outs, cts, masks, nullptr, n_out, n_terms, level, accumulate, s);
}

int hcnn_mac_terms_multi_packed(hcnn_ctx* c, uint64_t* const* outs, const uint64_t* const* cts,
                                const uint64_t* const* masks, const unsigned char* packed, uint32_t n_out,
                                uint32_t n_terms, uint32_t level, int accumulate, void* s) {
  return hcnn_mac_terms_multi_images(c, outs, cts, masks, packed, n_out, n_terms, level, 1, accumulate, s);
}

int hcnn_mac_terms_multi_images(hcnn_ctx* c, uint64_t* const* outs, const uint64_t* const* cts,
                                const uint64_t* const* masks, const unsigned char* packed, uint32_t n_out,
                                uint32_t n_terms, uint32_t level, uint32_t n_images, int accumulate, void* s) {
  if (!c) return fail(HCNN_E_PARAMETER, "null context");
  if (level >= c->Lq) return fail(HCNN_E_LEVEL, "level outside chain");
  if (n_images != 1 && n_images != 2) return fail(HCNN_E_PARAMETER, "n_images must be 1 or 2");
  if (n_images == 2 && c->n % 256) return fail(HCNN_E_PARAMETER, "two-image MAC needs N % 256 == 0");
  const u32 nq = level + 1;
  for (u32 g0 = 0; g0 < n_out; g0 += kMultiG) {
    const u32 ng = std::min<u32>(kMultiG, n_out - g0);
    if (n_terms == 0) {
      if (!accumulate)
        for (u32 g = 0; g < ng; ++g)
          CK(cudaMemsetAsync(outs[g0 + g], 0, 2ull * n_images * nq * c->n * 8, STREAM(s)));
      continue;
    }
    for (u32 t0 = 0; t0 < n_terms; t0 += kMultiT) {
      const u32 nt = std::min<u32>(kMultiT, n_terms - t0);
      MacMulti M;
      M.wide = c->wide;
      M.nimg = n_images;
      M.img_stride = 2ull * nq * c->n;
      M.fast_from = nq;
      while (M.fast_from > 1 && c->mods[M.fast_from - 1] < (1ull << 42)) --M.fast_from;
      for (u32 t = 0; t < nt; ++t) M.ct[t] = cts[t0 + t];
      // packed bytes relative to u64 rows, averaged over the limbs
      const double pf = nq > 1 ? (double)packed_hi_off(nq, nq, 1, c->wide) / (8.0 * nq) : 1.0;
      double used = 0;
      for (u32 g = 0; g < (u32)kMultiG; ++g) {
        M.out[g] = g < ng ? outs[g0 + g] : nullptr;
        for (u32 t = 0; t < nt; ++t) {
          const size_t idx = (size_t)(g0 + g) * n_terms + t0 + t;
          M.mask[g][t] = g < ng ? masks[idx] : nullptr;
          M.packed[g][t] = (g < ng && packed) ? packed[idx] : 0;
          used += M.mask[g][t] ? (M.packed[g][t] ? pf : 1.0) : 0.0;
        }
      }
      PK("mac_multi", 8.0 * (2.0 * nt * n_images + used + 2.0 * ng * n_images * (accumulate || t0 ? 2 : 1)) * nq * c->n,
         n_images == 2 ? 3 : 1, STREAM(s),
         launch_mac_multi(M, (int)ng, (int)nt, nq, c->logN, accumulate || t0 > 0, c->d_mc, STREAM(s)));
    }
  }
  return HCNN_OK;
}

size_t hcnn_rescale_workspace_bytes(const hcnn_ctx* c, uint32_t npolys) { return (size_t)npolys * c->n * 8; }

int hcnn_rescale(hcnn_ctx* c, uint64_t* out, const uint64_t* in, uint32_t level, uint32_t npolys, void* ws,
                 void* s) {
  if (!c) return fail(HCNN_E_PARAMETER, "null context");
  if (level == 0) return fail(HCNN_E_LEVEL, "no limb left to rescale away");
  if (level >= c->Lq) return fail(HCNN_E_LEVEL, "level outside chain");
  const u32 l = level;
  u64* top = (u64*)ws;
  PK("rescale_gather", 16.0 * npolys * c->n, 1, STREAM(s), launch_gather_limb(top, in, l, l + 1, c->logN, npolys, STREAM(s)));
  LimbMap m{};
  m.base = top;
  m.poly_stride = c->n;
  m.basis = c->basis(l + 1, 0);
  m.first_limb = l;
  PK("ntt_inv_rescale", 16.0 * npolys * c->n, ntt_nk(c), STREAM(s), launch_ntt(c->tables(), m, 1, npolys, true, STREAM(s)));
  LimbMap o{};
  o.base = out;
  o.poly_stride = (size_t)l * c->n;
  o.basis = c->basis(l, 0);
  if (c->tables().ctw) {
    // the column pass lifts the (centred) top limb into every q_i on load:
    // no lift kernel, one shared row per poly instead of l lifted rows
    o.sin = (const long long*)top;
    o.smont = 0;
    o.sin_center = c->hmc[l].q;
    PK("ntt_fwd_rescale", 8.0 * (1 + 2.0 * l) * npolys * c->n, ntt_nk(c), STREAM(s),
       launch_ntt(c->tables(), o, l, npolys, false, STREAM(s)));
  } else {
    PK("rescale_lift", 8.0 * (l + 1) * npolys * c->n, 1, STREAM(s), launch_rescale_lift(out, top, l, c->logN, npolys, c->d_qmod + (size_t)l * c->Lq, c->d_mc, STREAM(s)));
    PK("ntt_fwd_rescale", 16.0 * l * npolys * c->n, ntt_nk(c), STREAM(s), launch_ntt(c->tables(), o, l, npolys, false, STREAM(s)));
  }
  PK("rescale_combine", 24.0 * l * npolys * c->n, 1, STREAM(s), launch_rescale_combine(out, in, l, c->logN, npolys, c->d_rinv + (size_t)l * c->Lq,
                            c->d_rinv_sh + (size_t)l * c->Lq, c->d_mc, STREAM(s)));
  return HCNN_OK;
}


void hcnn_profile_enable(int on) { g_prof.store(on != 0); }

int hcnn_set_option(const char* name, long long value) {
  std::string k = name ? name : "";
  if (k == "ntt_group_limbs") g_ntt_tuning.group_limbs = (int)value;
  else if (k == "ntt_hints") g_ntt_tuning.hints = (int)value;
  else if (k == "ntt_occupancy") g_ntt_tuning.occupancy = (int)value;
  else if (k == "ntt_split") g_ntt_tuning.split = (int)value;
  else if (k == "ntt_f64_minb") g_ntt_tuning.f64_minb = (int)value;
  else if (k == "ntt_pipe") g_ntt_tuning.pipe = (int)value;
  else if (k == "ntt_fork") g_ntt_tuning.fork = (int)value;
  else if (k == "fbc_fork") g_fbc_fork = (int)value;
  else if (k == "ks_rots") g_ks_rots = (int)value;
  else if (k == "ks_rots_min_nb") g_ks_rots_min_nb = (int)value;
  else if (k == "md_fuse") g_ntt_tuning.md_fuse = (int)value;
  else if (k == "fbc_fast") CK(set_fbc_fast((int)value));
  else if (k == "ks96") CK(set_ks96((int)value));
  else if (k == "ks_batch") g_ks_batch = (int)value;
  else if (k == "ks_pipe") g_ks_pipe = (int)value;
  else if (k == "ks_tma") g_ks_tma = (int)value;
  else if (k == "ks_tma_min") g_ks_tma_min = (int)value;
  else if (k == "mac_batch") g_mac_batch = (int)value;
  else if (k == "mac_lanes") g_mac_lanes = (int)value;
  else if (k == "mac_async") g_mac_async = (int)value;
  else if (k == "mac_tma") g_mac_tma = (int)value;
  else if (k == "ks_tma3") g_ks_tma3 = (int)value;
  else if (k == "ks3_stages") g_ks3_stages = (int)value;
  else if (k == "mac3_stages") g_mac3_stages = (int)value;
  else if (k == "mac3_tpb") g_mac3_tpb = (int)value;
  else if (k == "mac3_fork") g_mac3_fork = (int)value;
  else if (k == "tma_stages") g_tma_stages = (int)value;
  else if (k == "ks_tpb") g_ks_tpb = value == 128 ? 128 : 256;
  else if (k == "ks_stages") g_ks_stages = (int)value;
  else if (k == "mac_minb") g_mac_minb = (int)value;
  else if (k == "mac_tpb") g_mac_tpb = value == 128 ? 128 : 256;
  else if (k == "merge_moddown") g_merge_moddown = (int)value;
  else return fail(HCNN_E_PARAMETER, "unknown option " + k);
  return HCNN_OK;
}

unsigned long long hcnn_kernel_launches(void) { return g_kernels.load() + g_ntt_extra_launches.load(); }

int hcnn_ntt_butterfly_peak(int device, int fast, double* bfly_per_s) {
  if (!bfly_per_s) return fail(HCNN_E_PARAMETER, "null output");
  CK(cudaSetDevice(device));
  CK((cudaError_t)ntt_butterfly_peak(fast, bfly_per_s));
  return HCNN_OK;
}

void hcnn_ks_counters(unsigned long long* out4, int reset) {
  for (int i = 0; i < 4; ++i) {
    if (out4) out4[i] = g_ks_acc[i].load();
    if (reset) g_ks_acc[i] = 0;
  }
}

void hcnn_ntt_limb_counts(unsigned long long* out4, int reset) {
  for (int i = 0; i < 4; ++i) {
    if (out4) out4[i] = g_ntt_limbs[i];
    if (reset) g_ntt_limbs[i] = 0;
  }
}

// Drain pending event pairs into per-name totals and render them as JSON:
// {"name": [launches, total_ms, algorithmic_bytes, kernels], ...}
int hcnn_profile_read(char* buf, size_t len, int reset) {
  std::lock_guard<std::mutex> lk(g_pm);
  for (auto& r : g_pending) {
    float ms = 0.f;
    cudaEventSynchronize(r.b);
    cudaEventElapsedTime(&ms, r.a, r.b);
    auto& a = g_acc[r.name];
    a[0] += 1;
    a[1] += ms;
    a[2] += r.bytes;
    a[3] += r.nk;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_pending.clear();
  std::string js = "{";
  bool first = true;
  for (auto& kv : g_acc) {
    char tmp[256];
    snprintf(tmp, sizeof tmp, "%s\"%s\": [%.0f, %.6f, %.0f, %.0f]", first ? "" : ", ", kv.first.c_str(),
             kv.second[0], kv.second[1], kv.second[2], kv.second[3]);
    js += tmp;
    first = false;
  }
  js += "}";
  if (reset) g_acc.clear();
  if (buf && len) {
    size_t n = js.size() < len - 1 ? js.size() : len - 1;
    memcpy(buf, js.data(), n);
    buf[n] = 0;
  }
  return (int)js.size();
}

}  // extern "C"
