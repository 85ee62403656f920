/*
 * TEST INFRASTRUCTURE -- the CPU checker, never the product.
 *
 * Plain-C restatement of the reference's modular kernels
 * (/root/reference/pkg/src/hcnn/kernels.py), used by oracle/ckks_oracle.py
 * to recompute residues the CUDA engine must reproduce bit for bit, and as
 * the CPU baseline arm of bench.py.  Each function follows the numba kernel
 * cited beside it; 64x64->128 products use unsigned __int128 instead of the
 * reference's 32-bit splits (same integers).  Row-batched entry points run
 * rows in parallel with OpenMP (the reference is single-threaded).
 */
#include <stddef.h>
#include <stdint.h>

typedef unsigned __int128 u128;

/* _redc kernels.py:177-188: a*b*2^-64 mod q, a,b < 2^62 */
static inline uint64_t redc(uint64_t a, uint64_t b, uint64_t q, uint64_t ninv) {
  u128 p = (u128)a * b;
  uint64_t lo = (uint64_t)p, hi = (uint64_t)(p >> 64);
  uint64_t m = lo * ninv;
  uint64_t t = hi + (uint64_t)(((u128)m * q) >> 64) + (lo != 0);
  return t >= q ? t - q : t;
}

/* _k_mulmod kernels.py:190-193 / _k_mulmod_scalar_b :195-198 */
void o_mulmod(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t len, int b_scalar, uint64_t q,
              uint64_t ninv) {
  for (size_t i = 0; i < len; ++i) out[i] = redc(a[i], b_scalar ? b[0] : b[i], q, ninv);
}

/* _k_muladd kernels.py:200-206 */
void o_muladd(uint64_t* acc, const uint64_t* a, const uint64_t* b, size_t len, uint64_t q, uint64_t ninv) {
  for (size_t i = 0; i < len; ++i) {
    uint64_t t = acc[i] + redc(a[i], b[i], q, ninv);
    acc[i] = t >= q ? t - q : t;
  }
}

/* _k_addmod / _k_submod / _k_negmod kernels.py:208-230 */
void o_addmod(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t len, uint64_t q) {
  for (size_t i = 0; i < len; ++i) {
    uint64_t t = a[i] + b[i];
    out[i] = t >= q ? t - q : t;
  }
}
void o_submod(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t len, uint64_t q) {
  for (size_t i = 0; i < len; ++i) out[i] = a[i] >= b[i] ? a[i] - b[i] : a[i] + (q - b[i]);
}
void o_negmod(uint64_t* out, const uint64_t* a, size_t len, uint64_t q) {
  for (size_t i = 0; i < len; ++i) out[i] = a[i] == 0 ? 0 : q - a[i];
}

/* _k_ntt kernels.py:232-253: Cooley-Tukey, natural -> bit-reversed,
 * stage m uses wtab[m+i] (Montgomery-form twiddles) */
void o_ntt(uint64_t* a, size_t n, const uint64_t* wtab, uint64_t q, uint64_t ninv) {
  size_t t = n;
  for (size_t m = 1; m < n; m <<= 1) {
    t >>= 1;
    for (size_t i = 0; i < m; ++i) {
      uint64_t s = wtab[m + i];
      size_t j1 = 2 * i * t;
      for (size_t j = j1; j < j1 + t; ++j) {
        uint64_t u = a[j];
        uint64_t v = redc(a[j + t], s, q, ninv);
        uint64_t hi = u + v;
        a[j] = hi >= q ? hi - q : hi;
        a[j + t] = u >= v ? u - v : u + (q - v);
      }
    }
  }
}

/* _k_intt kernels.py:255-281: Gentleman-Sande, bit-reversed -> natural, x N^-1 */
void o_intt(uint64_t* a, size_t n, const uint64_t* iwtab, uint64_t q, uint64_t ninv, uint64_t n_inv_mont) {
  size_t t = 1;
  for (size_t m = n; m > 1; m >>= 1) {
    size_t h = m >> 1, j1 = 0;
    for (size_t i = 0; i < h; ++i) {
      uint64_t s = iwtab[h + i];
      for (size_t j = j1; j < j1 + t; ++j) {
        uint64_t u = a[j], v = a[j + t];
        uint64_t hi = u + v;
        a[j] = hi >= q ? hi - q : hi;
        uint64_t d = u >= v ? u - v : u + (q - v);
        a[j + t] = redc(d, s, q, ninv);
      }
      j1 += 2 * t;
    }
    t <<= 1;
  }
  for (size_t j = 0; j < n; ++j) a[j] = redc(a[j], n_inv_mont, q, ninv);
}

/* _k_fbc_row kernels.py:283-301: centred fast-base-conversion row */
void o_fbc_row(uint64_t* out, const uint64_t* ys, size_t ns, size_t n, const uint64_t* src_qs,
               const uint64_t* src_halves, const uint64_t* tcol_mont, uint64_t q, uint64_t ninv) {
  for (size_t i = 0; i < ns; ++i) {
    uint64_t qi = src_qs[i], half = src_halves[i], tm = tcol_mont[i];
    const uint64_t* y = ys + i * n;
    for (size_t k = 0; k < n; ++k) {
      uint64_t term;
      if (y[k] <= half) {
        term = redc(y[k], tm, q, ninv);
      } else {
        term = redc(qi - y[k], tm, q, ninv);
        if (term != 0) term = q - term;
      }
      uint64_t acc = out[k] + term;
      out[k] = acc >= q ? acc - q : acc;
    }
  }
}

/* ---- row-batched drivers (OpenMP over rows; rows are independent,
 *      ring.py:5-6) ------------------------------------------------------- */
void o_ntt_rows(uint64_t* a, size_t rows, size_t n, const uint64_t* wtabs, const uint64_t* qs,
                const uint64_t* ninvs) {
#pragma omp parallel for schedule(static)
  for (long r = 0; r < (long)rows; ++r) o_ntt(a + r * n, n, wtabs + r * n, qs[r], ninvs[r]);
}

void o_intt_rows(uint64_t* a, size_t rows, size_t n, const uint64_t* iwtabs, const uint64_t* qs,
                 const uint64_t* ninvs, const uint64_t* n_inv_monts) {
#pragma omp parallel for schedule(static)
  for (long r = 0; r < (long)rows; ++r)
    o_intt(a + r * n, n, iwtabs + r * n, qs[r], ninvs[r], n_inv_monts[r]);
}

/* out[r] = a[r] (*) b[r or 0] with row r's modulus */
void o_mulmod_rows(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t rows, size_t n, int b_bcast,
                   const uint64_t* qs, const uint64_t* ninvs) {
#pragma omp parallel for schedule(static)
  for (long r = 0; r < (long)rows; ++r)
    o_mulmod(out + r * n, a + r * n, b + (b_bcast ? 0 : r * n), n, 0, qs[r], ninvs[r]);
}

void o_muladd_rows(uint64_t* acc, const uint64_t* a, const uint64_t* b, size_t rows, size_t n,
                   const uint64_t* qs, const uint64_t* ninvs) {
#pragma omp parallel for schedule(static)
  for (long r = 0; r < (long)rows; ++r) o_muladd(acc + r * n, a + r * n, b + r * n, n, qs[r], ninvs[r]);
}

/* every target row t of base_convert (ring.py:393-397) */
void o_fbc_rows(uint64_t* out, const uint64_t* ys, size_t ns, size_t nt, size_t n, const uint64_t* src_qs,
                const uint64_t* src_halves, const uint64_t* tmat_mont, const uint64_t* dst_qs,
                const uint64_t* dst_ninvs) {
#pragma omp parallel for schedule(static)
  for (long t = 0; t < (long)nt; ++t)
    o_fbc_row(out + t * n, ys, ns, n, src_qs, src_halves, tmat_mont + t * ns, dst_qs[t], dst_ninvs[t]);
}

int o_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
