/* ols_oracle.c — CPU restatement of the reference's fused OLS path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle and the CPU
 * baseline ("port") of bench.py; nothing in the product package links or
 * calls it.  It restates, loop for loop, the numba kernels of the reference
 * (olsconv/_kernels_nb.py) in C so it can run on the GPU box, where the
 * reference does not exist:
 *
 *   tables        fft.py:70-78       tw[j] = exp(-2 pi i j / n) (fp64, rounded)
 *   dif_fwd       _kernels_nb.py:11-28
 *   dit_inv       _kernels_nb.py:31-51
 *   _gather       _kernels_nb.py:206-215
 *   _store k0/1   _kernels_nb.py:218-222
 *   fused_c2c     _kernels_nb.py:265-285
 *   oracle_conv   _kernels_nb.py:183-199
 *
 * Complex products use numba's formula (a c - b d, a d + b c) with FMA
 * contraction disabled (-ffp-contract=off), the same IEEE operations in the
 * same order as the reference's compiled loops, so the single-precision
 * output is pinned bit-for-bit against fixtures produced by the reference
 * itself (tests/golden, tests/test_oracle.py).  Segment ranges are split
 * over OpenMP threads like the reference's ThreadPoolExecutor (ols.py:212-225);
 * results do not depend on the split.
 */
#include <math.h>
#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#include <stdint.h>
#include <stdlib.h>
#include <pthread.h>
#include <string.h>
#include <unistd.h>

/* run fn(ctx, lo, hi) over `threads` contiguous chunks of [lo0, hi0) on
 * pthreads (the reference's _chunk_bounds + ThreadPoolExecutor). */
typedef void (*chunk_fn)(void* ctx, int64_t lo, int64_t hi);
typedef struct {
  chunk_fn fn;
  void* ctx;
  int64_t lo, hi;
} chunk_job;
static void* chunk_main(void* arg) {
  chunk_job* j = (chunk_job*)arg;
  if (j->lo < j->hi) j->fn(j->ctx, j->lo, j->hi);
  return NULL;
}
static void run_chunks(int threads, int64_t lo0, int64_t hi0, chunk_fn fn,
                       void* ctx) {
  const int64_t n = hi0 - lo0;
  if (n <= 0) return;
  if (threads < 1) threads = 1;
  if (threads > n) threads = (int)n;
  const int64_t step = (n + threads - 1) / threads;
  if (threads == 1) {
    fn(ctx, lo0, hi0);
    return;
  }
  chunk_job* jobs = (chunk_job*)malloc(sizeof(chunk_job) * (size_t)threads);
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int c = 0; c < threads; ++c) {
    jobs[c].fn = fn;
    jobs[c].ctx = ctx;
    jobs[c].lo = lo0 + (int64_t)c * step;
    jobs[c].hi = jobs[c].lo + step < hi0 ? jobs[c].lo + step : hi0;
    pthread_create(&tids[c], NULL, chunk_main, &jobs[c]);
  }
  for (int c = 0; c < threads; ++c) pthread_join(tids[c], NULL);
  free(jobs);
  free(tids);
}

#define DEFINE_OLS(R, SFX)                                                    \
  typedef struct {                                                            \
    R re, im;                                                                 \
  } cpx_##SFX;                                                                \
                                                                              \
  static inline cpx_##SFX cmul_##SFX(cpx_##SFX a, cpx_##SFX b) {              \
    cpx_##SFX r;                                                              \
    r.re = a.re * b.re - a.im * b.im;                                         \
    r.im = a.re * b.im + a.im * b.re;                                         \
    return r;                                                                 \
  }                                                                           \
                                                                              \
  void ols_tables_##SFX(int n, R* tw, R* twc) {                               \
    for (int j = 0; j < n / 2; ++j) {                                         \
      const double th = (-2.0 * M_PI * (double)j) / (double)n;                \
      tw[2 * j] = (R)cos(th);                                                 \
      tw[2 * j + 1] = (R)sin(th);                                             \
      twc[2 * j] = tw[2 * j];                                                 \
      twc[2 * j + 1] = -tw[2 * j + 1];                                        \
    }                                                                         \
  }                                                                           \
                                                                              \
  void ols_dif_fwd_##SFX(R* ar, int n, const R* twr) {                        \
    cpx_##SFX* a = (cpx_##SFX*)ar;                                            \
    const cpx_##SFX* tw = (const cpx_##SFX*)twr;                              \
    int span = n >> 1, step = 1;                                              \
    while (span >= 1) {                                                       \
      for (int start = 0; start < n; start += span << 1) {                    \
        int tj = 0;                                                           \
        for (int j = start; j < start + span; ++j) {                          \
          const cpx_##SFX u = a[j], v = a[j + span];                          \
          cpx_##SFX s, d;                                                     \
          s.re = u.re + v.re;                                                 \
          s.im = u.im + v.im;                                                 \
          d.re = u.re - v.re;                                                 \
          d.im = u.im - v.im;                                                 \
          a[j] = s;                                                           \
          a[j + span] = cmul_##SFX(d, tw[tj]);                                \
          tj += step;                                                         \
        }                                                                     \
      }                                                                       \
      span >>= 1;                                                             \
      step <<= 1;                                                             \
    }                                                                         \
  }                                                                           \
                                                                              \
  void ols_dit_inv_##SFX(R* ar, int n, const R* twcr) {                       \
    cpx_##SFX* a = (cpx_##SFX*)ar;                                            \
    const cpx_##SFX* twc = (const cpx_##SFX*)twcr;                            \
    int span = 1, step = n >> 1;                                              \
    while (span < n) {                                                        \
      for (int start = 0; start < n; start += span << 1) {                    \
        int tj = 0;                                                           \
        for (int j = start; j < start + span; ++j) {                          \
          const cpx_##SFX u = a[j];                                           \
          const cpx_##SFX v = cmul_##SFX(a[j + span], twc[tj]);               \
          a[j].re = u.re + v.re;                                              \
          a[j].im = u.im + v.im;                                              \
          a[j + span].re = u.re - v.re;                                       \
          a[j + span].im = u.im - v.im;                                       \
          tj += step;                                                         \
        }                                                                     \
      }                                                                       \
      span <<= 1;                                                             \
      step >>= 1;                                                             \
    }                                                                         \
    /* a[i] * (1.0 / n): 1/n is a power of two, exact in either precision */ \
    const double inv = 1.0 / (double)n;                                       \
    for (int i = 0; i < n; ++i) {                                             \
      a[i].re = (R)((double)a[i].re * inv);                                   \
      a[i].im = (R)((double)a[i].im * inv);                                   \
    }                                                                         \
  }                                                                           \
                                                                              \
  void ols_dif_fwd_batch_##SFX(R* mat, int rows, int n, const R* tw) {        \
    for (int r = 0; r < rows; ++r) ols_dif_fwd_##SFX(mat + 2 * (size_t)r * n, \
                                                     n, tw);                  \
  }                                                                           \
                                                                              \
  void ols_dit_inv_batch_##SFX(R* mat, int rows, int n, const R* twc) {       \
    for (int r = 0; r < rows; ++r) ols_dit_inv_##SFX(mat + 2 * (size_t)r * n, \
                                                     n, twc);                 \
  }                                                                           \
                                                                              \
  static void fused_range_##SFX(const cpx_##SFX* x, int64_t n_s,              \
                                const cpx_##SFX* spectra, int n_fil, int n,   \
                                const R* tw, const R* twc, int64_t l_eff,     \
                                int64_t t0, int64_t win_off, int64_t seg_lo,  \
                                int64_t seg_hi, int pp_kind, double pp_c,     \
                                cpx_##SFX* out, cpx_##SFX* buf,               \
                                cpx_##SFX* spec_buf) {                        \
    for (int64_t s = seg_lo; s < seg_hi; ++s) {                               \
      const int64_t g0 = s * l_eff;                                           \
      const int64_t w0 = g0 + win_off;                                        \
      for (int t = 0; t < n; ++t) { /* _gather */                             \
        const int64_t idx = w0 + t;                                           \
        if (idx >= 0 && idx < n_s) {                                          \
          buf[t] = x[idx];                                                    \
        } else {                                                              \
          buf[t].re = 0;                                                      \
          buf[t].im = 0;                                                      \
        }                                                                     \
      }                                                                       \
      ols_dif_fwd_##SFX((R*)buf, n, tw);                                      \
      memcpy(spec_buf, buf, sizeof(cpx_##SFX) * (size_t)n);                   \
      int64_t span = l_eff;                                                   \
      if (g0 + span > n_s) span = n_s - g0;                                   \
      for (int f = 0; f < n_fil; ++f) {                                       \
        const cpx_##SFX* h = spectra + (size_t)f * n;                         \
        for (int t = 0; t < n; ++t) buf[t] = cmul_##SFX(spec_buf[t], h[t]);   \
        ols_dit_inv_##SFX((R*)buf, n, twc);                                   \
        cpx_##SFX* row = out + (size_t)f * (size_t)n_s;                       \
        if (pp_kind == 0) {                                                   \
          for (int64_t j = 0; j < span; ++j) row[g0 + j] = buf[t0 + j];       \
        } else {                                                              \
          /* _store kind 1: Python-float pp_c x complex64 promotes to     \
             complex128, rounded once into the output (ols.py _store) */  \
          for (int64_t j = 0; j < span; ++j) {                                \
            row[g0 + j].re = (R)(pp_c * (double)buf[t0 + j].re);              \
            row[g0 + j].im = (R)(pp_c * (double)buf[t0 + j].im);              \
          }                                                                   \
        }                                                                     \
      }                                                                       \
    }                                                                         \
  }                                                                           \
                                                                              \
  typedef struct {                                                            \
    const R *x, *spectra, *tw, *twc;                                          \
    int64_t n_s, l_eff, t0, win_off;                                          \
    int n_fil, n, pp_kind;                                                    \
    double pp_c;                                                              \
    R* out;                                                                   \
  } fused_ctx_##SFX;                                                          \
                                                                              \
  static void fused_chunk_##SFX(void* vc, int64_t lo, int64_t hi) {           \
    const fused_ctx_##SFX* c = (const fused_ctx_##SFX*)vc;                    \
    cpx_##SFX* scratch =                                                      \
        (cpx_##SFX*)malloc(2 * sizeof(cpx_##SFX) * (size_t)c->n);             \
    fused_range_##SFX((const cpx_##SFX*)c->x, c->n_s,                         \
                      (const cpx_##SFX*)c->spectra, c->n_fil, c->n, c->tw,    \
                      c->twc, c->l_eff, c->t0, c->win_off, lo, hi,            \
                      c->pp_kind, c->pp_c, (cpx_##SFX*)c->out, scratch,       \
                      scratch + c->n);                                        \
    free(scratch);                                                            \
  }                                                                           \
                                                                              \
  /* K.fused_c2c over [seg_lo, seg_hi), split into `threads` contiguous   */  \
  /* chunks (ols.py:212-225).  spectra: reference permuted layout.        */  \
  void ols_fused_c2c_##SFX(const R* x, int64_t n_s, const R* spectra,         \
                           int n_fil, int n, const R* tw, const R* twc,       \
                           int64_t l_eff, int64_t t0, int64_t win_off,        \
                           int64_t seg_lo, int64_t seg_hi, int pp_kind,       \
                           double pp_c, R* out, int threads) {                \
    fused_ctx_##SFX c = {x,     spectra, tw,      twc,     n_s, l_eff,        \
                         t0,    win_off, n_fil,   n,       pp_kind,           \
                         pp_c,  out};                                         \
    run_chunks(threads, seg_lo, seg_hi, fused_chunk_##SFX, &c);               \
  }

DEFINE_OLS(float, f)
DEFINE_OLS(double, d)

/* Direct time-domain convolution, complex128 accumulate (oracle_conv,
 * _kernels_nb.py:183-199): out[f, i] = sum_k taps[f, k] x[i - k + origin]. */
typedef struct {
  const cpx_d *x, *taps;
  cpx_d* out;
  int64_t n_s;
  int n_fil, m, origin;
} direct_ctx;

static void direct_chunk(void* vc, int64_t lo, int64_t hi) {
  const direct_ctx* c = (const direct_ctx*)vc;
  for (int64_t w = lo; w < hi; ++w) {
    const int f = (int)(w / c->n_s);
    const int64_t i = w - (int64_t)f * c->n_s;
    int64_t klo = i + c->origin - c->n_s + 1;
    if (klo < 0) klo = 0;
    int64_t khi = i + c->origin;
    if (khi > c->m - 1) khi = c->m - 1;
    cpx_d acc = {0.0, 0.0};
    for (int64_t k = klo; k <= khi; ++k) {
      const cpx_d p =
          cmul_d(c->taps[(size_t)f * c->m + k], c->x[i - k + c->origin]);
      acc.re += p.re;
      acc.im += p.im;
    }
    c->out[w] = acc;
  }
}

void ols_direct_d(const double* xr, int64_t n_s, const double* tapsr,
                  int n_fil, int m, int origin, double* outr, int threads) {
  direct_ctx c = {(const cpx_d*)xr, (const cpx_d*)tapsr, (cpx_d*)outr, n_s,
                  n_fil, m, origin};
  run_chunks(threads, 0, (int64_t)n_fil * n_s, direct_chunk, &c);
}

int ols_oracle_max_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}
