// olsb_kernels.cu — sm_100a kernels and the C ABI of the OLS engine.
//
// Kernels
//   fused_c2c_kernel  the hot path: segment staging -> forward FFT -> per
//                     filter {multiply, inverse FFT, valid-sample writeback}
//                     (reference: _kernels_nb.py:265-285, ols.py:319-360)
//   fwd_rows_kernel   forward transform of rows (filter spectra,
//                     fft_forward_permuted); same passes as the fused kernel
//   inv_rows_kernel   inverse transform of rows (fft_inverse_permuted)
//   perm_to_dev_kernel  reference permuted layout -> engine layout
//
// One thread owns E = 16 samples of a segment; T = N / 16 threads form a
// segment group, SEGS groups a CTA of 256 threads.  Samples move between
// 4-bit windows through padded, bank-conflict-free shared memory (see
// olsb_fft.cuh).  The whole filter loop runs with the segment spectrum held
// in registers; filter spectra stream from L2 through L1 (every segment
// group of the CTA reads the same spectrum in lockstep).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>

#include "olsb.h"
#include "olsb_fft.cuh"

namespace olsb {

constexpr int kThreads = 256;

// 16-byte vector type holding two complex<float> or one complex<double>
template <class R>
struct V16;
template <>
struct V16<float> {
  using type = float4;
  static constexpr int per = 2;  // complex per vector
};
template <>
struct V16<double> {
  using type = double2;
  static constexpr int per = 1;
};

template <class R, int LOGN>
struct Cfg {
  using G = Geo<LOGN>;
  using L = SmemLayout<R, LOGN>;
  static constexpr bool dbl = std::is_same<R, double>::value;
  static constexpr int E = G::E, T = G::T, P = G::P, LOGE = G::LOGE;
  static constexpr int SEGS = (kThreads / T) > 0 ? (kThreads / T) : 1;
  static constexpr int THREADS = SEGS * T;
  static constexpr int NBUF = dbl ? 1 : 2;
  static constexpr int VPT = E / V16<R>::per;  // 16-B vectors per thread (J)
  // top-window twiddles kept in registers (float only; 30 registers)
  static constexpr bool TOPREG = !dbl && P >= 2;
  static constexpr int tab_elems = G::tw_total();
  static constexpr size_t tab_bytes =
      ((size_t(tab_elems) * sizeof(Tw<R>)) + 127) & ~size_t(127);
  static constexpr size_t buf_elems = size_t(SEGS) * L::stride;
  static constexpr size_t smem_bytes =
      tab_bytes + (P >= 2 ? NBUF * buf_elems * sizeof(Cpx<R>) : 0);
};

// ---------------------------------------------------------------------------
// shared-memory window I/O (addresses = per-thread base + immediates)
// ---------------------------------------------------------------------------
template <class R, int LOGN, int Q>
__device__ __forceinline__ void smem_store(Cpx<R>* __restrict__ seg_buf, int t,
                                           const Cpx<R>* x) {
  using C = Cfg<R, LOGN>;
  using G = typename C::G;
  using L = typename C::L;
  Cpx<R>* b = seg_buf + L::pos(G::thread_part(Q, t));
  if constexpr (Q == 0 && !C::dbl && C::E >= 2) {
    sfor<0, C::E / 2>([&](auto ec) {
      constexpr int e = 2 * decltype(ec)::value;
      constexpr int off = L::pos(G::elem_part(Q, e));
      *reinterpret_cast<float4*>(b + off) =
          make_float4(x[e].re, x[e].im, x[e + 1].re, x[e + 1].im);
    });
  } else {
    sfor<0, C::E>([&](auto ec) {
      constexpr int e = decltype(ec)::value;
      constexpr int off = L::pos(G::elem_part(Q, e));
      b[off] = x[e];
    });
  }
}

template <class R, int LOGN, int Q>
__device__ __forceinline__ void smem_load(const Cpx<R>* __restrict__ seg_buf,
                                          int t, Cpx<R>* x) {
  using C = Cfg<R, LOGN>;
  using G = typename C::G;
  using L = typename C::L;
  const Cpx<R>* b = seg_buf + L::pos(G::thread_part(Q, t));
  if constexpr (Q == 0 && !C::dbl && C::E >= 2) {
    sfor<0, C::E / 2>([&](auto ec) {
      constexpr int e = 2 * decltype(ec)::value;
      constexpr int off = L::pos(G::elem_part(Q, e));
      const float4 v = *reinterpret_cast<const float4*>(b + off);
      x[e] = Cpx<R>{v.x, v.y};
      x[e + 1] = Cpx<R>{v.z, v.w};
    });
  } else {
    sfor<0, C::E>([&](auto ec) {
      constexpr int e = decltype(ec)::value;
      constexpr int off = L::pos(G::elem_part(Q, e));
      x[e] = b[off];
    });
  }
}

// twiddle tables for windows 1..P-1 (double-precision math, rounded once)
template <class R, int LOGN>
__device__ void build_tables(Tw<R>* tab) {
  using G = Geo<LOGN>;
  sfor<1, G::P>([&](auto qc) {
    constexpr int q = decltype(qc)::value;
    constexpr int lo = G::lo(q);
    constexpr int cnt = G::tw_entries(q);
    constexpr int off = G::tw_offset(q);
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      double c, t;
      twiddle_entry(lo, i >> lo, i & ((1 << lo) - 1), &c, &t);
      tab[off + i] = Tw<R>{R(c), R(t)};
    }
  });
}

// accessor of the thread's 15 runtime twiddles of window q
template <class R>
struct TwSmem {
  const Tw<R>* base;  // tab + off + l
  int lstride;        // 2^lo
  __device__ __forceinline__ Tw<R> operator()(int idx) const {
    return base[idx * lstride];
  }
};
template <class R>
struct TwRegs {
  const Tw<R>* r;
  __device__ __forceinline__ Tw<R> operator()(int idx) const { return r[idx]; }
};

// exchange: write window QW, barrier, read window QR
template <class R, int LOGN, int QW, int QR>
__device__ __forceinline__ void exchange(Cpx<R>* bufs, int& xc, int sl, int t,
                                         Cpx<R>* x) {
  using C = Cfg<R, LOGN>;
  Cpx<R>* buf = bufs + (C::NBUF == 2 ? (xc & 1) * C::buf_elems : 0) +
                size_t(sl) * C::L::stride;
  if constexpr (C::NBUF == 1) __syncthreads();
  smem_store<R, LOGN, QW>(buf, t, x);
  __syncthreads();
  smem_load<R, LOGN, QR>(buf, t, x);
  ++xc;
}

// full forward transform: x holds window P-1 on entry, window 0 (J) on exit
template <class R, int LOGN>
__device__ __forceinline__ void forward_fft(Cpx<R>* x, const Tw<R>* tab,
                                            Cpx<R>* bufs, int& xc, int sl,
                                            int t) {
  using C = Cfg<R, LOGN>;
  using G = typename C::G;
  sfor<0, G::P>([&](auto qr) {
    constexpr int q = G::P - 1 - decltype(qr)::value;
    if constexpr (q < G::P - 1) exchange<R, LOGN, q + 1, q>(bufs, xc, sl, t, x);
    if constexpr (q == 0) {
      dif_pass_static<R, C::LOGE, G::G0>(x);
    } else {
      constexpr int lo = G::lo(q);
      const TwSmem<R> tw{tab + G::tw_offset(q) + G::low_bits(q, t), 1 << lo};
      dif_pass_rt<R>(x, tw);
    }
  });
}

// ---------------------------------------------------------------------------
// fused OLS kernel
// ---------------------------------------------------------------------------
template <class R>
struct FusedArgs {
  const Cpx<R>* x;
  long long x_base, n_s;
  const typename V16<R>::type* spec;  // engine layout
  int n_fil, fchunk, t0, pp_kind;
  long long l_eff, win_off, seg_lo, seg_hi;
  R pp_c;
  Cpx<R>* out;
  long long out_ld, out_base;
};

template <class R, int LOGN>
__global__ void __launch_bounds__(Cfg<R, LOGN>::THREADS)
    fused_c2c_kernel(const FusedArgs<R> a) {
  using C = Cfg<R, LOGN>;
  using G = typename C::G;
  constexpr int E = C::E, T = C::T, P = C::P;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Tw<R>* tab = reinterpret_cast<Tw<R>*>(smem_raw);
  Cpx<R>* bufs = reinterpret_cast<Cpx<R>*>(smem_raw + C::tab_bytes);

  const int tid = threadIdx.x;
  const int sl = tid / T;
  const int t = tid % T;

  build_tables<R, LOGN>(tab);
  __syncthreads();

  // top-window (inverse) twiddles: fixed per thread for the kernel lifetime
  Tw<R> twr[15];
  if constexpr (C::TOPREG) {
    constexpr int q = P - 1;
    const Tw<R>* base = tab + G::tw_offset(q) + G::low_bits(q, t);
#pragma unroll
    for (int i = 0; i < 15; ++i) twr[i] = base[i << G::lo(q)];
  }

  const long long nseg = a.seg_hi - a.seg_lo;
  const long long ngroups = (nseg + C::SEGS - 1) / C::SEGS;
  const int nfch = (a.n_fil + a.fchunk - 1) / a.fchunk;
  const long long nitems = ngroups * nfch;
  const R inv_n = R(1) / R(G::N);
  int xc = 0;

  for (long long it = blockIdx.x; it < nitems; it += gridDim.x) {
    const long long grp = it / nfch;
    const int fc = int(it - grp * nfch);
    const long long s = a.seg_lo + grp * C::SEGS + sl;
    const bool live = s < a.seg_hi;
    const long long g0 = s * a.l_eff;
    const long long span =
        live ? (a.l_eff < a.n_s - g0 ? a.l_eff : a.n_s - g0) : 0;
    const long long w0 = g0 + a.win_off;

    // ---- segment staging: zero-extended window, top-window layout
    // (_gather, _kernels_nb.py:206-215)
    Cpx<R> x[E];
    {
      constexpr int q = P - 1;
      const long long pb = w0 + G::thread_part(q, t);
      sfor<0, E>([&](auto ec) {
        constexpr int e = decltype(ec)::value;
        const long long gi = pb + G::elem_part(q, e);
        if (live && gi >= 0 && gi < a.n_s) {
          x[e] = a.x[gi - a.x_base];
        } else {
          x[e] = Cpx<R>{R(0), R(0)};
        }
      });
    }
    // ---- forward FFT (dif_fwd, _kernels_nb.py:11-28), spectrum kept in
    // registers with the inverse's 1/N folded in
    forward_fft<R, LOGN>(x, tab, bufs, xc, sl, t);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      x[e].re *= inv_n;
      x[e].im *= inv_n;
    }

    const int f_lo = fc * a.fchunk;
    const int f_hi = min(a.n_fil, f_lo + a.fchunk);
    for (int f = f_lo; f < f_hi; ++f) {
      // ---- pointwise multiply, both operands bit-reversed
      // (_kernels_nb.py:280-282)
      Cpx<R> y[E];
      const typename V16<R>::type* hs =
          a.spec + (size_t(f) * C::VPT) * T + t;
      if constexpr (!C::dbl) {
        sfor<0, C::VPT>([&](auto uc) {
          constexpr int u = decltype(uc)::value;
          const float4 h = __ldg(reinterpret_cast<const float4*>(hs) + u * T);
          const Cpx<R> s0 = x[2 * u], s1 = x[2 * u + 1];
          y[2 * u] = Cpx<R>{fmaR(s0.re, h.x, -s0.im * h.y),
                            fmaR(s0.re, h.y, s0.im * h.x)};
          y[2 * u + 1] = Cpx<R>{fmaR(s1.re, h.z, -s1.im * h.w),
                                fmaR(s1.re, h.w, s1.im * h.z)};
        });
      } else {
        sfor<0, C::VPT>([&](auto uc) {
          constexpr int u = decltype(uc)::value;
          const double2 h = __ldg(reinterpret_cast<const double2*>(hs) + u * T);
          const Cpx<R> s0 = x[u];
          y[u] = Cpx<R>{fmaR(s0.re, h.x, -s0.im * h.y),
                        fmaR(s0.re, h.y, s0.im * h.x)};
        });
      }
      // ---- inverse FFT (dit_inv, _kernels_nb.py:31-51)
      dit_pass_static<R, C::LOGE, G::G0>(y);
      sfor<1, P>([&](auto qc) {
        constexpr int q = decltype(qc)::value;
        exchange<R, LOGN, q - 1, q>(bufs, xc, sl, t, y);
        if constexpr (q == P - 1 && C::TOPREG) {
          dit_pass_rt<R>(y, TwRegs<R>{twr});
        } else {
          constexpr int lo = G::lo(q);
          const TwSmem<R> tw{tab + G::tw_offset(q) + G::low_bits(q, t),
                             1 << lo};
          dit_pass_rt<R>(y, tw);
        }
      });
      // ---- valid-sample writeback (_store kind 0/1, _kernels_nb.py:218-222)
      {
        constexpr int q = P - 1;
        const long long ob = G::thread_part(q, t) - a.t0;
        Cpx<R>* orow = a.out + f * a.out_ld + g0 - a.out_base;
        const bool scale = a.pp_kind == OLSB_PP_SCALE;
        sfor<0, E>([&](auto ec) {
          constexpr int e = decltype(ec)::value;
          const long long o = ob + G::elem_part(q, e);
          if (live && o >= 0 && o < span) {
            Cpx<R> v = y[e];
            if (scale) {
              v.re *= a.pp_c;
              v.im *= a.pp_c;
            }
            if constexpr (!C::dbl) {
              __stcs(reinterpret_cast<float2*>(orow + o),
                     make_float2(v.re, v.im));
            } else {
              __stcs(reinterpret_cast<double2*>(orow + o),
                     make_double2(v.re, v.im));
            }
          }
        });
      }
    }
  }
}

// ---------------------------------------------------------------------------
// row transforms
// ---------------------------------------------------------------------------
template <class R>
struct RowsArgs {
  const Cpx<R>* in;
  long long in_ld;  // row stride of `in` (elements)
  int len;          // valid input columns (zero-padded to N)
  int rows;
  Cpx<R>* out_perm;  // may be null
  typename V16<R>::type* out_dev;  // may be null
};

template <class R, int LOGN>
__global__ void __launch_bounds__(Cfg<R, LOGN>::THREADS)
    fwd_rows_kernel(const RowsArgs<R> a) {
  using C = Cfg<R, LOGN>;
  using G = typename C::G;
  constexpr int E = C::E, T = C::T, P = C::P;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Tw<R>* tab = reinterpret_cast<Tw<R>*>(smem_raw);
  Cpx<R>* bufs = reinterpret_cast<Cpx<R>*>(smem_raw + C::tab_bytes);
  const int sl = threadIdx.x / T, t = threadIdx.x % T;
  build_tables<R, LOGN>(tab);
  __syncthreads();
  int xc = 0;
  const int ngroups = (a.rows + C::SEGS - 1) / C::SEGS;
  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const int r = grp * C::SEGS + sl;
    const bool live = r < a.rows;
    Cpx<R> x[E];
    {
      constexpr int q = P - 1;
      const int pb = G::thread_part(q, t);
      sfor<0, E>([&](auto ec) {
        constexpr int e = decltype(ec)::value;
        const int p = pb + G::elem_part(q, e);
        x[e] = (live && p < a.len) ? a.in[size_t(r) * a.in_ld + p]
                                   : Cpx<R>{R(0), R(0)};
      });
    }
    // every load of the group precedes any store (in-place safety)
    __syncthreads();
    forward_fft<R, LOGN>(x, tab, bufs, xc, sl, t);
    if (live) {
      if (a.out_perm) {
        Cpx<R>* o = a.out_perm + size_t(r) * G::N + G::thread_part(0, t);
#pragma unroll
        for (int e = 0; e < E; ++e) o[e] = x[e];
      }
      if (a.out_dev) {
        typename V16<R>::type* o = a.out_dev + size_t(r) * C::VPT * T + t;
        if constexpr (!C::dbl) {
#pragma unroll
          for (int u = 0; u < C::VPT; ++u)
            o[u * T] = make_float4(x[2 * u].re, x[2 * u].im, x[2 * u + 1].re,
                                   x[2 * u + 1].im);
        } else {
#pragma unroll
          for (int u = 0; u < C::VPT; ++u) o[u * T] = make_double2(x[u].re, x[u].im);
        }
      }
    }
  }
}

template <class R, int LOGN>
__global__ void __launch_bounds__(Cfg<R, LOGN>::THREADS)
    inv_rows_kernel(const Cpx<R>* in, Cpx<R>* out, int rows) {
  using C = Cfg<R, LOGN>;
  using G = typename C::G;
  constexpr int E = C::E, T = C::T, P = C::P;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Tw<R>* tab = reinterpret_cast<Tw<R>*>(smem_raw);
  Cpx<R>* bufs = reinterpret_cast<Cpx<R>*>(smem_raw + C::tab_bytes);
  const int sl = threadIdx.x / T, t = threadIdx.x % T;
  build_tables<R, LOGN>(tab);
  __syncthreads();
  int xc = 0;
  const R inv_n = R(1) / R(G::N);
  const int ngroups = (rows + C::SEGS - 1) / C::SEGS;
  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const int r = grp * C::SEGS + sl;
    const bool live = r < rows;
    Cpx<R> y[E];
    const Cpx<R>* src = in + size_t(r) * G::N + G::thread_part(0, t);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const Cpx<R> v = live ? src[e] : Cpx<R>{R(0), R(0)};
      y[e] = Cpx<R>{v.re * inv_n, v.im * inv_n};
    }
    __syncthreads();
    dit_pass_static<R, C::LOGE, G::G0>(y);
    sfor<1, P>([&](auto qc) {
      constexpr int q = decltype(qc)::value;
      exchange<R, LOGN, q - 1, q>(bufs, xc, sl, t, y);
      const TwSmem<R> tw{tab + G::tw_offset(q) + G::low_bits(q, t),
                         1 << G::lo(q)};
      dit_pass_rt<R>(y, tw);
    });
    if (live) {
      constexpr int q = P - 1;
      Cpx<R>* o = out + size_t(r) * G::N + G::thread_part(q, t);
      sfor<0, E>([&](auto ec) {
        constexpr int e = decltype(ec)::value;
        o[G::elem_part(q, e)] = y[e];
      });
    }
  }
}

template <class R, int LOGN>
__global__ void perm_to_dev_kernel(const Cpx<R>* perm,
                                   typename V16<R>::type* dev, int rows) {
  using C = Cfg<R, LOGN>;
  constexpr int T = C::T, VPT = C::VPT, per = V16<R>::per;
  const long long total = (long long)rows * VPT * T;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
       i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / (VPT * T);
    const int rem = int(i - r * VPT * T);
    const int u = rem / T, t = rem % T;
    const Cpx<R>* s = perm + r * Geo<LOGN>::N + t * C::E + u * per;
    if constexpr (per == 2) {
      dev[i] = make_float4(s[0].re, s[0].im, s[1].re, s[1].im);
    } else {
      dev[i] = make_double2(s[0].re, s[0].im);
    }
  }
}

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------
inline int num_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 1;
}

template <class K>
int prepare(K kernel, size_t smem, int threads, int* resident) {
  cudaError_t e = cudaFuncSetAttribute(
      kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return int(e);
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads,
                                                    smem);
  if (e != cudaSuccess) return int(e);
  *resident = std::max(1, occ) * num_sms();
  return 0;
}

static int g_filter_chunk = 0;

template <class R, int LOGN>
int launch_fused(FusedArgs<R> a, cudaStream_t st) {
  using C = Cfg<R, LOGN>;
  auto kern = fused_c2c_kernel<R, LOGN>;
  int resident = 0;
  int rc = prepare(kern, C::smem_bytes, C::THREADS, &resident);
  if (rc) return rc;
  a.fchunk = (g_filter_chunk > 0 && g_filter_chunk < a.n_fil) ? g_filter_chunk
                                                              : a.n_fil;
  const long long nseg = a.seg_hi - a.seg_lo;
  const long long ngroups = (nseg + C::SEGS - 1) / C::SEGS;
  const long long nitems = ngroups * ((a.n_fil + a.fchunk - 1) / a.fchunk);
  const int grid = int(std::min<long long>(nitems, resident));
  if (grid <= 0) return 0;
  kern<<<grid, C::THREADS, C::smem_bytes, st>>>(a);
  return int(cudaGetLastError());
}

template <class R, int LOGN>
int launch_fwd_rows(RowsArgs<R> a, cudaStream_t st) {
  using C = Cfg<R, LOGN>;
  auto kern = fwd_rows_kernel<R, LOGN>;
  int resident = 0;
  int rc = prepare(kern, C::smem_bytes, C::THREADS, &resident);
  if (rc) return rc;
  const int ngroups = (a.rows + C::SEGS - 1) / C::SEGS;
  const int grid = std::min(ngroups, resident);
  if (grid <= 0) return 0;
  kern<<<grid, C::THREADS, C::smem_bytes, st>>>(a);
  return int(cudaGetLastError());
}

template <class R, int LOGN>
int launch_inv_rows(const Cpx<R>* in, Cpx<R>* out, int rows, cudaStream_t st) {
  using C = Cfg<R, LOGN>;
  auto kern = inv_rows_kernel<R, LOGN>;
  int resident = 0;
  int rc = prepare(kern, C::smem_bytes, C::THREADS, &resident);
  if (rc) return rc;
  const int ngroups = (rows + C::SEGS - 1) / C::SEGS;
  const int grid = std::min(ngroups, resident);
  if (grid <= 0) return 0;
  kern<<<grid, C::THREADS, C::smem_bytes, st>>>(in, out, rows);
  return int(cudaGetLastError());
}

template <class R, int LOGN>
int launch_perm_to_dev(const Cpx<R>* perm, void* dev, int rows,
                       cudaStream_t st) {
  const long long total =
      (long long)rows * Cfg<R, LOGN>::VPT * Cfg<R, LOGN>::T;
  if (total == 0) return 0;
  const int grid = int(std::min<long long>((total + 255) / 256, 4096));
  perm_to_dev_kernel<R, LOGN><<<grid, 256, 0, st>>>(
      perm, reinterpret_cast<typename V16<R>::type*>(dev), rows);
  return int(cudaGetLastError());
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

int olsb_fused_c2c(const void* x, int64_t x_base, int64_t n_s,
                   const void* spectra_dev, int n_fil, int n, int m,
                   int origin, int64_t l_eff, int t0, int64_t win_off,
                   int64_t seg_lo, int64_t seg_hi, int pp_kind, double pp_c,
                   void* out, int64_t out_ld, int64_t out_base,
                   int precision, void* stream) {
  const int logn = log2_of(n);
  if (logn < 0) return OLSB_E_BAD_LENGTH;
  if (pp_kind != OLSB_PP_NONE && pp_kind != OLSB_PP_SCALE)
    return OLSB_E_UNSUPPORTED;
  if (n_s < 1 || n_fil < 0 || m < 1 || m > n || origin < 0 || origin >= m ||
      seg_lo < 0 || seg_hi < seg_lo)
    return OLSB_E_BAD_ARG;
  if (l_eff < 1 || t0 < 0 || t0 + l_eff > n) return OLSB_E_GEOMETRY;
  if (n_fil == 0 || seg_hi == seg_lo) return 0;
  if (!x || !spectra_dev || !out) return OLSB_E_BAD_ARG;
  return dispatch_prec(precision, [&](auto rv) {
    using R = decltype(rv);
    return dispatch_n<R>(logn, [&](auto lc) {
      FusedArgs<R> a;
      a.x = static_cast<const Cpx<R>*>(x);
      a.x_base = x_base;
      a.n_s = n_s;
      a.spec = static_cast<const typename V16<R>::type*>(spectra_dev);
      a.n_fil = n_fil;
      a.fchunk = n_fil;
      a.t0 = t0;
      a.pp_kind = pp_kind;
      a.l_eff = l_eff;
      a.win_off = win_off;
      a.seg_lo = seg_lo;
      a.seg_hi = seg_hi;
      a.pp_c = R(pp_c);
      a.out = static_cast<Cpx<R>*>(out);
      a.out_ld = out_ld;
      a.out_base = out_base;
      return launch_fused<R, decltype(lc)::value>(
          a, static_cast<cudaStream_t>(stream));
    });
  });
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
