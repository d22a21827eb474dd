// olsb_kernels.cu — launchers and the C ABI of the OLS engine (include/olsb.h).
//
// Device code lives in olsb_engine.cuh / olsb_fft.cuh.  Every entry point
// validates its arguments, dispatches the runtime FFT length and precision to
// a template instantiation and launches on the caller's stream.  Kernel
// shapes (policies) are chosen per N from measurements;
// OLSB_VARIANT=k overrides the fp32 policy for tuning sweeps.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "olsb.h"
#include "olsb_launch.cuh"

// the per-length launchers live in olsb_inst.cu objects
#define OLSB_EXTERN_ALL(L) OLSB_LAUNCHERS_ALL(extern, L)
OLSB_EXTERN_ALL(2)
OLSB_EXTERN_ALL(3)
OLSB_EXTERN_ALL(4)
OLSB_EXTERN_ALL(5)
OLSB_EXTERN_ALL(6)
OLSB_EXTERN_ALL(7)
OLSB_EXTERN_ALL(8)
OLSB_EXTERN_ALL(9)
OLSB_EXTERN_ALL(10)
OLSB_EXTERN_ALL(11)
OLSB_EXTERN_ALL(12)

namespace olsb {

int g_filter_chunk = 0;

// (kernel, device) -> resident CTAs, for prepare() (olsb_launch.cuh)
struct Prepared {
  const void* kernel;
  int dev, resident;
};
static std::mutex g_prep_mu;
static Prepared g_prep[512];
static int g_prep_n = 0;

int prepared_lookup(const void* kernel, int* resident) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_prep_mu);
  for (int i = 0; i < g_prep_n; ++i) {
    if (g_prep[i].kernel == kernel && g_prep[i].dev == dev) {
      *resident = g_prep[i].resident;
      return 1;
    }
  }
  return 0;
}

void prepared_store(const void* kernel, int resident) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_prep_mu);
  if (g_prep_n < 512) g_prep[g_prep_n++] = Prepared{kernel, dev, resident};
}

// Texture objects over engine-layout spectra (H_TEX), cached per
// (device, base, size); creating one costs microseconds, so a FilterSet
// reused across calls pays it once.  Entries are never destroyed: a launch
// still in flight on any stream, or a CUDA graph captured by
// Executor.graph(), may hold the handle, and destroying it would need a
// device-wide sync that is illegal during stream capture.  A linear texture
// is only a (pointer, size) descriptor, so an entry stays valid when its
// allocation is freed and the address reused; the cache grows by one small
// descriptor per distinct spectra range a process ever launches with.
struct TexKey {
  int dev;
  const void* ptr;
  size_t bytes;
  cudaTextureObject_t tex;
};
static std::mutex g_tex_mu;
static std::vector<TexKey> g_tex_cache;

int spectra_texture(const void* ptr, size_t bytes,
                           cudaTextureObject_t* out) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_tex_mu);
  for (const TexKey& k : g_tex_cache) {
    if (k.dev == dev && k.ptr == ptr && k.bytes == bytes) {
      *out = k.tex;
      return 0;
    }
  }
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = const_cast<void*>(ptr);
  rd.res.linear.desc = cudaCreateChannelDesc<float4>();
  rd.res.linear.sizeInBytes = bytes;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex = 0;
  cudaError_t e = cudaCreateTextureObject(&tex, &rd, &td, nullptr);
  if (e != cudaSuccess) return int(e);
  g_tex_cache.push_back(TexKey{dev, ptr, bytes, tex});
  *out = tex;
  return 0;
}

inline int log2_of(int n) {
  if (n < 4 || n > 4096 || (n & (n - 1))) return -1;
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

// runtime N -> template instantiation
template <class R, class F>
int dispatch_n(int logn, F&& f) {
  switch (logn) {
    case 2: return f(IC<2>{});
    case 3: return f(IC<3>{});
    case 4: return f(IC<4>{});
    case 5: return f(IC<5>{});
    case 6: return f(IC<6>{});
    case 7: return f(IC<7>{});
    case 8: return f(IC<8>{});
    case 9: return f(IC<9>{});
    case 10: return f(IC<10>{});
    case 11: return f(IC<11>{});
    case 12: return f(IC<12>{});
    default: return OLSB_E_BAD_LENGTH;
  }
}

template <class F>
int dispatch_prec(int precision, F&& f) {
  if (precision == 0) return f(float{});
  if (precision == 1) return f(double{});
  return OLSB_E_BAD_PRECISION;
}

}  // namespace olsb

using namespace olsb;

extern "C" {

int olsb_version(void) { return 100; }

const char* olsb_error_string(int code) {
  switch (code) {
    case OLSB_OK: return "ok";
    case OLSB_E_BAD_LENGTH: return "FFT length must be a power of two in [4, 4096]";
    case OLSB_E_BAD_ARG: return "invalid argument";
    case OLSB_E_BAD_PRECISION: return "precision must be 0 (single) or 1 (double)";
    case OLSB_E_UNSUPPORTED: return "post-processing kind not supported";
    case OLSB_E_GEOMETRY: return "inconsistent segment geometry";
    default:
      return code > 0 ? cudaGetErrorString(cudaError_t(code)) : "unknown error";
  }
}

int olsb_spectra_dev_len(int n) { return log2_of(n) < 0 ? OLSB_E_BAD_LENGTH : n; }

int olsb_set_filter_chunk(int filters_per_item) {
  if (filters_per_item < 0) return OLSB_E_BAD_ARG;
  g_filter_chunk = filters_per_item;
  return 0;
}

int olsb_dif_fwd_batch(const void* in, void* out, int rows, int n,
                       int precision, void* stream) {
  const int logn = log2_of(n);
  if (logn < 0) return OLSB_E_BAD_LENGTH;
  if (rows < 0 || (rows > 0 && (!in || !out))) return OLSB_E_BAD_ARG;
  if (rows == 0) return 0;
  return dispatch_prec(precision, [&](auto rv) {
    using R = decltype(rv);
    return dispatch_n<R>(logn, [&](auto lc) {
      RowsArgs<R> a{static_cast<const Cpx<R>*>(in), n, n, rows,
                    static_cast<Cpx<R>*>(out), nullptr};
      return launch_fwd_rows<R, decltype(lc)::value>(
          a, static_cast<cudaStream_t>(stream));
    });
  });
}

int olsb_dit_inv_batch(const void* in, void* out, int rows, int n,
                       int precision, void* stream) {
  const int logn = log2_of(n);
  if (logn < 0) return OLSB_E_BAD_LENGTH;
  if (rows < 0 || (rows > 0 && (!in || !out))) return OLSB_E_BAD_ARG;
  if (rows == 0) return 0;
  return dispatch_prec(precision, [&](auto rv) {
    using R = decltype(rv);
    return dispatch_n<R>(logn, [&](auto lc) {
      return launch_inv_rows<R, decltype(lc)::value>(
          static_cast<const Cpx<R>*>(in), static_cast<Cpx<R>*>(out), rows,
          static_cast<cudaStream_t>(stream));
    });
  });
}

int olsb_filter_spectra_c2c(const void* taps, int n_fil, int m, int n,
                            void* spectra_perm, void* spectra_dev,
                            int precision, void* stream) {
  const int logn = log2_of(n);
  if (logn < 0) return OLSB_E_BAD_LENGTH;
  if (n_fil < 0 || m < 1 || m > n || (n_fil > 0 && !taps))
    return OLSB_E_BAD_ARG;
  if (n_fil == 0 || (!spectra_perm && !spectra_dev)) return 0;
  return dispatch_prec(precision, [&](auto rv) {
    using R = decltype(rv);
    return dispatch_n<R>(logn, [&](auto lc) {
      RowsArgs<R> a{static_cast<const Cpx<R>*>(taps), m, m, n_fil,
                    static_cast<Cpx<R>*>(spectra_perm),
                    static_cast<typename V16<R>::type*>(spectra_dev)};
      return launch_fwd_rows<R, decltype(lc)::value>(
          a, static_cast<cudaStream_t>(stream));
    });
  });
}

int olsb_filter_spectra_c2c_ref(const void* taps, int n_fil, int m, int n,
                                const void* tw, void* spectra_perm,
                                void* spectra_dev, int precision,
                                void* stream) {
  const int logn = log2_of(n);
  if (logn < 0) return OLSB_E_BAD_LENGTH;
  if (n_fil < 0 || m < 1 || m > n || (n_fil > 0 && !taps) || !tw)
    return OLSB_E_BAD_ARG;
  if (n_fil == 0 || (!spectra_perm && !spectra_dev)) return 0;
  return dispatch_prec(precision, [&](auto rv) {
    using R = decltype(rv);
    return dispatch_n<R>(logn, [&](auto lc) {
      RowsArgs<R> a{static_cast<const Cpx<R>*>(taps), m, m, n_fil,
                    static_cast<Cpx<R>*>(spectra_perm),
                    static_cast<typename V16<R>::type*>(spectra_dev),
                    static_cast<const Cpx<R>*>(tw)};
      return launch_fwd_rows<R, decltype(lc)::value>(
          a, static_cast<cudaStream_t>(stream));
    });
  });
}

int olsb_spectra_perm_to_dev(const void* spectra_perm, int n_fil, int n,
                             void* spectra_dev, int precision, void* stream) {
  const int logn = log2_of(n);
  if (logn < 0) return OLSB_E_BAD_LENGTH;
  if (n_fil < 0 || (n_fil > 0 && (!spectra_perm || !spectra_dev)))
    return OLSB_E_BAD_ARG;
  return dispatch_prec(precision, [&](auto rv) {
    using R = decltype(rv);
    return dispatch_n<R>(logn, [&](auto lc) {
      return launch_perm_to_dev<R, decltype(lc)::value>(
          static_cast<const Cpx<R>*>(spectra_perm), spectra_dev, n_fil,
          static_cast<cudaStream_t>(stream));
    });
  });
}

// Engine segment grid for the reference geometry (t0, l_eff) at length n:
// valid in-place samples [t0, t0 + l_eff) of every segment.  For n >= 512
// the engine discards up to the next multiple of 32 and keeps a multiple of
// 32 samples, so every warp store writes one aligned 256-byte chunk; the grid
// is anchored at sample 0, so any split of the output range is bit-identical.
static void engine_grid(int n, int t0, long long l_eff, int* t0e,
                        long long* le) {
  *t0e = t0;
  *le = l_eff;
  if (n < 512) return;
  const int ta = (t0 + 31) & ~31;
  const long long la = ((long long)t0 + l_eff - ta) & ~31LL;
  if (la >= 32 && la * 100 >= l_eff * 97) {
    *t0e = ta;
    *le = la;
  }
}

// mode: FMODE_C2C (complex x / out), FMODE_R2R (real x / out, segment
// pairs), FMODE_ABS2 (complex x, real |y|^2 out)
static int fused_range(int mode, const void* x, int64_t x_base, int64_t n_s,
                       const void* spectra_dev, int n_fil, int n, int t0,
                       int origin, int64_t l_eff, int64_t g_lo, int64_t g_hi,
                       int pp_kind, double pp_c, void* out, int64_t out_ld,
                       int64_t out_base, int precision, void* stream,
                       const void* xtw = nullptr) {
  const int logn = log2_of(n);
  if (logn < 0) return OLSB_E_BAD_LENGTH;
  const bool pp_ok =
      xtw ? (mode == FMODE_C2C && (pp_kind == OLSB_PP_NONE ||
                                   pp_kind == OLSB_PP_SCALE)) ||
                (mode == FMODE_ABS2 && pp_kind == OLSB_PP_NONE)
          : pp_kind == OLSB_PP_NONE || pp_kind == OLSB_PP_SCALE ||
                (mode == FMODE_R2R && pp_kind == OLSB_PP_MAG2) ||
                (mode != FMODE_ABS2 && pp_kind == OLSB_PP_DERIV && t0 >= 1 &&
                 t0 + l_eff <= n - 1);
  if (!pp_ok) return OLSB_E_UNSUPPORTED;
  if (n_s < 1 || n_fil < 0 || g_lo < 0 || g_hi < g_lo) return OLSB_E_BAD_ARG;
  if (l_eff < 1 || t0 < 0 || t0 + l_eff > n) return OLSB_E_GEOMETRY;
  if (g_hi > n_s) g_hi = n_s;
  if (n_fil == 0 || g_hi <= g_lo) return 0;
  if (!x || !spectra_dev || !out) return OLSB_E_BAD_ARG;
  int t0e = t0;
  long long le = l_eff;
  // exact mode keeps the reference's segment grid
  if (!xtw) engine_grid(n, t0, l_eff, &t0e, &le);
  return dispatch_prec(precision, [&](auto rv) {
    using R = decltype(rv);
    return dispatch_n<R>(logn, [&](auto lc) {
      FusedArgs<R> a = {};
      a.xtw = static_cast<const Cpx<R>*>(xtw);
      a.x = static_cast<const Cpx<R>*>(x);
      a.xr = static_cast<const R*>(x);
      a.x_base = x_base;
      a.n_s = n_s;
      a.spec = static_cast<const typename V16<R>::type*>(spectra_dev);
      a.n_fil = n_fil;
      a.fchunk = n_fil;
      a.pp_kind = pp_kind;
      a.t0 = t0e;
      a.origin = origin;
      a.seg_len = le;
      a.k_lo = g_lo / le;
      a.k_hi = (g_hi + le - 1) / le;
      if (mode == FMODE_R2R) {  // segment pairs {2k, 2k + 1}
        a.k_lo /= 2;
        a.k_hi = (a.k_hi + 1) / 2;
      }
      a.g_lo = g_lo;
      a.g_hi = g_hi;
      a.pp_c = R(pp_c);
      a.pp_cd = pp_c;
      a.out = static_cast<Cpx<R>*>(out);
      a.outr = static_cast<R*>(out);
      a.out_ld = out_ld;
      a.out_base = out_base;
      a.dbg = debug_env();
      return launch_fused<R, decltype(lc)::value>(
          a, mode, static_cast<cudaStream_t>(stream));
    });
  });
}

static int check_ref_geometry(int64_t n_s, int n_fil, int n, int m, int origin,
                              int64_t l_eff, int t0, int64_t win_off,
                              int64_t seg_lo, int64_t seg_hi) {
  if (n_s < 1 || n_fil < 0 || m < 1 || m > n || origin < 0 || origin >= m ||
      seg_lo < 0 || seg_hi < seg_lo)
    return OLSB_E_BAD_ARG;
  if (l_eff < 1 || t0 < 0 || t0 + l_eff > n || win_off != origin - t0)
    return OLSB_E_GEOMETRY;
  return 0;
}

int olsb_fused_c2c(const void* x, int64_t x_base, int64_t n_s,
                   const void* spectra_dev, int n_fil, int n, int m,
                   int origin, int64_t l_eff, int t0, int64_t win_off,
                   int64_t seg_lo, int64_t seg_hi, int pp_kind, double pp_c,
                   void* out, int64_t out_ld, int64_t out_base,
                   int precision, void* stream) {
  const int rc = check_ref_geometry(n_s, n_fil, n, m, origin, l_eff, t0,
                                    win_off, seg_lo, seg_hi);
  if (rc) return rc;
  // the reference segments [seg_lo, seg_hi) own outputs
  // [seg_lo * l_eff, min(seg_hi * l_eff, n_s))
  return fused_range(FMODE_C2C, x, x_base, n_s, spectra_dev, n_fil, n, t0,
                     origin, l_eff, seg_lo * l_eff,
                     std::min<int64_t>(seg_hi * l_eff, n_s), pp_kind, pp_c,
                     out, out_ld, out_base, precision, stream);
}

int olsb_fused_c2c_ref(const void* x, int64_t x_base, int64_t n_s,
                       const void* spectra_dev, int n_fil, int n, int m,
                       int origin, int64_t l_eff, int t0, int64_t win_off,
                       int64_t seg_lo, int64_t seg_hi, int pp_kind,
                       double pp_c, const void* tw, void* out, int64_t out_ld,
                       int64_t out_base, int precision, void* stream) {
  const int rc = check_ref_geometry(n_s, n_fil, n, m, origin, l_eff, t0,
                                    win_off, seg_lo, seg_hi);
  if (rc) return rc;
  if (!tw) return OLSB_E_BAD_ARG;
  return fused_range(FMODE_C2C, x, x_base, n_s, spectra_dev, n_fil, n, t0,
                     origin, l_eff, seg_lo * l_eff,
                     std::min<int64_t>(seg_hi * l_eff, n_s), pp_kind, pp_c,
                     out, out_ld, out_base, precision, stream, tw);
}

int olsb_fused_c2c_abs2_ref(const void* x, int64_t x_base, int64_t n_s,
                            const void* spectra_dev, int n_fil, int n, int m,
                            int origin, int64_t l_eff, int t0, int64_t win_off,
                            int64_t seg_lo, int64_t seg_hi, const void* tw,
                            void* out, int64_t out_ld, int64_t out_base,
                            int precision, void* stream) {
  const int rc = check_ref_geometry(n_s, n_fil, n, m, origin, l_eff, t0,
                                    win_off, seg_lo, seg_hi);
  if (rc) return rc;
  if (!tw) return OLSB_E_BAD_ARG;
  return fused_range(FMODE_ABS2, x, x_base, n_s, spectra_dev, n_fil, n, t0,
                     origin, l_eff, seg_lo * l_eff,
                     std::min<int64_t>(seg_hi * l_eff, n_s), OLSB_PP_NONE, 1.0,
                     out, out_ld, out_base, precision, stream, tw);
}

int olsb_fused_c2c_abs2(const void* x, int64_t x_base, int64_t n_s,
                        const void* spectra_dev, int n_fil, int n, int m,
                        int origin, int64_t l_eff, int t0, int64_t win_off,
                        int64_t seg_lo, int64_t seg_hi, void* out,
                        int64_t out_ld, int64_t out_base, int precision,
                        void* stream) {
  const int rc = check_ref_geometry(n_s, n_fil, n, m, origin, l_eff, t0,
                                    win_off, seg_lo, seg_hi);
  if (rc) return rc;
  return fused_range(FMODE_ABS2, x, x_base, n_s, spectra_dev, n_fil, n, t0,
                     origin, l_eff, seg_lo * l_eff,
                     std::min<int64_t>(seg_hi * l_eff, n_s), OLSB_PP_NONE, 1.0,
                     out, out_ld, out_base, precision, stream);
}

int olsb_fused_r2r(const void* x, int64_t x_base, int64_t n_s,
                   const void* spectra_dev, int n_fil, int n, int m,
                   int origin, int64_t l_eff, int t0, int64_t win_off,
                   int64_t seg_lo, int64_t seg_hi, int pp_kind, double pp_c,
                   void* out, int64_t out_ld, int64_t out_base,
                   int precision, void* stream) {
  const int rc = check_ref_geometry(n_s, n_fil, n, m, origin, l_eff, t0,
                                    win_off, seg_lo, seg_hi);
  if (rc) return rc;
  return fused_range(FMODE_R2R, x, x_base, n_s, spectra_dev, n_fil, n, t0,
                     origin, l_eff, seg_lo * l_eff,
                     std::min<int64_t>(seg_hi * l_eff, n_s), pp_kind, pp_c,
                     out, out_ld, out_base, precision, stream);
}

// Segment geometry of the range entries: the plain one (t0 = m - 1, L = n -
// m + 1), or for the derivative the halo geometry (t0 = m, L = n - m - 1):
// every output's neighbours are then in-place samples of its own segment
// (ols.py:137-146 with halo 1; for m = 1 too, where the reference instead
// recomputes seam neighbours from the input)
static int range_geometry(int pp_kind, int n, int m, int* t0, int64_t* l_eff) {
  *t0 = m - 1;
  *l_eff = n - m + 1;
  if (pp_kind == OLSB_PP_DERIV) {
    *t0 = m;
    *l_eff = n - m - 1;
    if (*l_eff < 1) return OLSB_E_GEOMETRY;
  }
  return 0;
}

int olsb_fused_c2c_range(const void* x, int64_t x_base, int64_t n_s,
                         const void* spectra_dev, int n_fil, int n, int m,
                         int origin, int64_t g_lo, int64_t g_hi, int pp_kind,
                         double pp_c, void* out, int64_t out_ld,
                         int64_t out_base, int precision, void* stream) {
  if (m < 1 || m > n || origin < 0 || origin >= m) return OLSB_E_BAD_ARG;
  int t0;
  int64_t le;
  if (int rc = range_geometry(pp_kind, n, m, &t0, &le)) return rc;
  // magnitude_squared: the |y|^2 epilogue into a REAL out
  if (pp_kind == OLSB_PP_MAG2)
    return fused_range(FMODE_ABS2, x, x_base, n_s, spectra_dev, n_fil, n,
                       m - 1, origin, n - m + 1, g_lo, g_hi, OLSB_PP_NONE, 1.0,
                       out, out_ld, out_base, precision, stream);
  return fused_range(FMODE_C2C, x, x_base, n_s, spectra_dev, n_fil, n, t0,
                     origin, le, g_lo, g_hi, pp_kind, pp_c, out, out_ld,
                     out_base, precision, stream);
}

int olsb_fused_r2r_range(const void* x, int64_t x_base, int64_t n_s,
                         const void* spectra_dev, int n_fil, int n, int m,
                         int origin, int64_t g_lo, int64_t g_hi, int pp_kind,
                         double pp_c, void* out, int64_t out_ld,
                         int64_t out_base, int precision, void* stream) {
  if (m < 1 || m > n || origin < 0 || origin >= m) return OLSB_E_BAD_ARG;
  int t0;
  int64_t le;
  if (int rc = range_geometry(pp_kind, n, m, &t0, &le)) return rc;
  return fused_range(FMODE_R2R, x, x_base, n_s, spectra_dev, n_fil, n, t0,
                     origin, le, g_lo, g_hi, pp_kind, pp_c, out, out_ld,
                     out_base, precision, stream);
}

static int input_extent(int mode, int n, int m, int origin, int64_t g_lo,
                        int64_t g_hi, int64_t* x_lo, int64_t* x_hi,
                        int pp_kind = OLSB_PP_NONE) {
  if (log2_of(n) < 0) return OLSB_E_BAD_LENGTH;
  if (m < 1 || m > n || origin < 0 || origin >= m || g_hi < g_lo || !x_lo ||
      !x_hi)
    return OLSB_E_BAD_ARG;
  int t0;
  int64_t l_eff;
  if (int rc = range_geometry(pp_kind, n, m, &t0, &l_eff)) return rc;
  int t0e;
  long long le;
  engine_grid(n, t0, l_eff, &t0e, &le);
  long long k_lo = g_lo / le, k_hi = (g_hi + le - 1) / le;
  if (mode == FMODE_R2R) {  // whole segment pairs {2k, 2k + 1}
    k_lo = (k_lo / 2) * 2;
    k_hi = ((k_hi + 1) / 2) * 2;
  }
  *x_lo = k_lo * le - t0e + origin;
  *x_hi = (k_hi - 1) * le - t0e + origin + n;
  return 0;
}

int olsb_input_extent(int n, int m, int origin, int64_t g_lo, int64_t g_hi,
                      int64_t* x_lo, int64_t* x_hi) {
  return input_extent(FMODE_C2C, n, m, origin, g_lo, g_hi, x_lo, x_hi);
}

int olsb_input_extent_r2r(int n, int m, int origin, int64_t g_lo,
                          int64_t g_hi, int64_t* x_lo, int64_t* x_hi) {
  return input_extent(FMODE_R2R, n, m, origin, g_lo, g_hi, x_lo, x_hi);
}

int olsb_input_extent_pp(int mode, int n, int m, int origin, int pp_kind,
                         int64_t g_lo, int64_t g_hi, int64_t* x_lo,
                         int64_t* x_hi) {
  if (mode != FMODE_C2C && mode != FMODE_R2R) return OLSB_E_BAD_ARG;
  return input_extent(mode, n, m, origin, g_lo, g_hi, x_lo, x_hi, pp_kind);
}

int olsb_copy2d_async(void* dst, int64_t dst_pitch_bytes, const void* src,
                      int64_t src_pitch_bytes, int64_t width_bytes,
                      int64_t height, int kind, void* stream) {
  if (kind != 0 || width_bytes < 0 || height < 0) return OLSB_E_BAD_ARG;
  if (width_bytes == 0 || height == 0) return 0;
  if (!dst || !src) return OLSB_E_BAD_ARG;
  return int(cudaMemcpy2DAsync(dst, size_t(dst_pitch_bytes), src,
                               size_t(src_pitch_bytes), size_t(width_bytes),
                               size_t(height), cudaMemcpyDefault,
                               static_cast<cudaStream_t>(stream)));
}

}  // extern "C"
