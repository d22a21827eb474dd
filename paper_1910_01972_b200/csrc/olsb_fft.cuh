// olsb_fft.cuh — register-resident radix-2 FFT passes for the B200 OLS engine.
//
// The reference transforms (olsconv/_kernels_nb.py) are in-place radix-2:
//   dif_fwd  (:11-28)  spans N/2 -> 1, natural in -> bit-reversed out, unscaled
//   dit_inv  (:31-51)  spans 1 -> N/2, bit-reversed in -> natural out, x 1/N
// Here the same stage sequence is executed in "windows" of 4 index bits: each
// thread owns E = 16 samples whose in-place indices differ only in the window
// bits, runs the 4 radix-2 stages of that window in registers, and the segment
// moves to the next window through shared memory.  Because the stages and the
// in-place positions are exactly the reference's, the forward output sits in
// the reference's bit-reversed ("permuted") order, the multiply needs no
// reordering, and the inverse writes natural order — the reorder-free pairing
// of SURVEY §7.3.
//
// Everything in this header is plain C++ usable on the host as well, so the
// per-thread pass arithmetic is unit-tested on CPU (tests/test_fft_host.py).
#pragma once

#include <cmath>
#include <cstdint>
#include <type_traits>
#include <utility>

#if defined(__CUDACC__)
#define OLSB_HD __host__ __device__ __forceinline__
#else
#define OLSB_HD inline
#endif

namespace olsb {

template <class R>
struct alignas(2 * sizeof(R)) Cpx {
  R re, im;
};

// A twiddle in one of two encodings (see "butterfly forms" below):
//   STD : (cos theta, sin theta)
//   GOOD: (cos theta, tan theta)                 |tan| <= 1
//   ROT : (sin theta, -cot theta) = (cos, tan) of theta - pi/2, |.| <= 1
template <class R>
struct alignas(2 * sizeof(R)) Tw {
  R c, t;
};

OLSB_HD float fmaR(float a, float b, float c) { return fmaf(a, b, c); }
OLSB_HD double fmaR(double a, double b, double c) { return fma(a, b, c); }

// ---------------------------------------------------------------------------
// compile-time loops
// ---------------------------------------------------------------------------
template <int V>
using IC = std::integral_constant<int, V>;

template <int I, int N, class F>
OLSB_HD void sfor(F&& f) {
  if constexpr (I < N) {
    f(IC<I>{});
    sfor<I + 1, N>(f);
  }
}

// ---------------------------------------------------------------------------
// geometry
// ---------------------------------------------------------------------------
// N = 2^LOGN.  E = min(16, N) samples per thread, T = N / E threads per
// segment, P windows.  Window 0 ("J", the junction) holds index bits
// [0, G0) (plus G0..3 as batch bits); window q >= 1 holds bits [lo, lo+4).
template <int LOGN_>
struct Geo {
  static constexpr int LOGN = LOGN_;
  static constexpr int N = 1 << LOGN;
  static constexpr int LOGE = LOGN < 4 ? LOGN : 4;
  static constexpr int E = 1 << LOGE;
  static constexpr int LOGT = LOGN - LOGE;
  static constexpr int T = 1 << LOGT;
  static constexpr int P = (LOGN + 3) / 4;
  static constexpr int G0 = LOGN - 4 * (P - 1);
  static constexpr int lo(int q) { return q == 0 ? 0 : LOGN - 4 * (P - q); }
  static constexpr int g(int q) { return q == 0 ? G0 : 4; }
  // number of runtime twiddle entries of window q (15 per low-bit value l)
  static constexpr int tw_entries(int q) { return q == 0 ? 0 : 15 << lo(q); }
  static constexpr int tw_offset(int q) {
    int off = 0;
    for (int i = 1; i < q; ++i) off += tw_entries(i);
    return off;
  }
  static constexpr int tw_total() { return tw_offset(P); }
  // thread part / element part of the in-place index in window q (disjoint
  // bit fields, so p = thread_part + elem_part)
  static OLSB_HD int thread_part(int q, int t) {
    const int l = lo(q);
    return ((t >> l) << (l + LOGE)) | (t & ((1 << l) - 1));
  }
  static constexpr int elem_part(int q, int e) { return e << lo(q); }
  static OLSB_HD int low_bits(int q, int t) { return t & ((1 << lo(q)) - 1); }
};

// ---------------------------------------------------------------------------
// shared-memory exchange layout: pos(p) = p + P1*(p>>K1) + P2*(p>>K2).
// Linear over disjoint bit fields, so every address is a per-thread base plus
// a compile-time immediate.  Parameters found by tools/smem_layout_search.py
// (zero bank conflicts for every access of both transforms).
// ---------------------------------------------------------------------------
struct Pad {
  int k1, p1, k2, p2, stride;
};

constexpr Pad pad_for(bool dbl, int logn) {
  constexpr Pad f[13] = {{2, 0, 2, 0, 2},    {2, 0, 2, 0, 2},
                         {2, 0, 2, 0, 6},    {2, 0, 2, 0, 10},
                         {2, 0, 2, 0, 18},   {2, 0, 4, 8, 42},
                         {4, 2, 5, 4, 76},   {2, 0, 4, 2, 152},
                         {2, 0, 4, 2, 286},  {4, 2, 7, 2, 580},
                         {4, 2, 7, 4, 1178}, {4, 2, 7, 8, 2422},
                         {2, 0, 4, 2, 4606}};
  constexpr Pad d[13] = {{2, 0, 2, 0, 1},    {2, 0, 2, 0, 1},
                         {2, 0, 2, 0, 5},    {2, 0, 2, 0, 9},
                         {2, 0, 2, 0, 17},   {2, 0, 4, 1, 34},
                         {2, 0, 4, 1, 68},   {2, 0, 4, 1, 135},
                         {2, 0, 4, 1, 271},  {2, 0, 4, 1, 543},
                         {2, 0, 4, 1, 1087}, {2, 0, 4, 1, 2175},
                         {2, 0, 4, 1, 4351}};
  return dbl ? d[logn] : f[logn];
}

template <class R, int LOGN>
struct SmemLayout {
  static constexpr Pad pd = pad_for(std::is_same<R, double>::value, LOGN);
  static OLSB_HD constexpr int pos(int p) {
    return p + pd.p1 * (p >> pd.k1) + pd.p2 * (p >> pd.k2);
  }
  static constexpr int stride = pd.stride;  // per segment, in Cpx<R> units
};

// ---------------------------------------------------------------------------
// static twiddles of the junction window: theta = pi * m / 8, m in [0, 8)
// ---------------------------------------------------------------------------
// forms: 0 = one, 1 = i, 2 = GOOD, 3 = ROT
constexpr double kCos8[8] = {1.0,
                             0.92387953251128675613,
                             0.70710678118654752440,
                             0.38268343236508977173,
                             0.0,
                             -0.38268343236508977173,
                             -0.70710678118654752440,
                             -0.92387953251128675613};
constexpr double kSin8[8] = {0.0,
                             0.38268343236508977173,
                             0.70710678118654752440,
                             0.92387953251128675613,
                             1.0,
                             0.92387953251128675613,
                             0.70710678118654752440,
                             0.38268343236508977173};
constexpr int static_form(int m) {
  return m == 0 ? 0 : m == 4 ? 1 : (m == 3 || m == 5) ? 3 : 2;
}
constexpr double static_c(int m) {
  return static_form(m) == 3 ? kSin8[m] : kCos8[m];
}
constexpr double static_t(int m) {
  return static_form(m) == 3 ? -kCos8[m] / kSin8[m] : kSin8[m] / kCos8[m];
}
// runtime-window stages j >= 2 have a static form per k (SURVEY-free
// derivation in DESIGN.md §3): theta in [pi k/2^j, pi (k+1)/2^j)
constexpr bool rot_static(int j, int k) {
  return 4 * k >= (1 << j) && 4 * (k + 1) <= 3 * (1 << j);
}

// ---------------------------------------------------------------------------
// butterfly forms.  Inverse (DIT): a = u + w v, b = u - w v, w = e^{+i theta}.
// Forward (DIF): a = u + v, b = (u - v) conj(w).
// GOOD/ROT are the FMA ("tangent") forms: w v = c (v + i t v) is 2 FMA, and
// the scale c fuses into the butterfly adds, so a twiddled DIT butterfly is
// 6 FFMA instead of 4 mul + 4 add.  ROT handles |tan| > 1 by rotating w by
// -pi/2 (the +i is a free swap/negate).
// ---------------------------------------------------------------------------
template <class R>
OLSB_HD void dit_one(Cpx<R>& u, Cpx<R>& v) {
  const Cpx<R> a{u.re + v.re, u.im + v.im};
  v = Cpx<R>{u.re - v.re, u.im - v.im};
  u = a;
}
template <class R>
OLSB_HD void dit_i(Cpx<R>& u, Cpx<R>& v) {  // w = i: w v = (-v.im, v.re)
  const Cpx<R> a{u.re - v.im, u.im + v.re};
  v = Cpx<R>{u.re + v.im, u.im - v.re};
  u = a;
}
template <class R>
OLSB_HD void dit_good(Cpx<R>& u, Cpx<R>& v, R c, R t) {
  const R pr = fmaR(-t, v.im, v.re);
  const R pi = fmaR(t, v.re, v.im);
  const Cpx<R> a{fmaR(c, pr, u.re), fmaR(c, pi, u.im)};
  v = Cpx<R>{fmaR(-c, pr, u.re), fmaR(-c, pi, u.im)};
  u = a;
}
template <class R>
OLSB_HD void dit_rot(Cpx<R>& u, Cpx<R>& v, R c, R t) {
  // w = i c (1 + i t): w v = i c p = (-c p.im, c p.re)
  const R pr = fmaR(-t, v.im, v.re);
  const R pi = fmaR(t, v.re, v.im);
  const Cpx<R> a{fmaR(-c, pi, u.re), fmaR(c, pr, u.im)};
  v = Cpx<R>{fmaR(c, pi, u.re), fmaR(-c, pr, u.im)};
  u = a;
}
template <class R>
OLSB_HD void dit_std(Cpx<R>& u, Cpx<R>& v, R c, R s) {
  const R wr = fmaR(v.re, c, -v.im * s);
  const R wi = fmaR(v.re, s, v.im * c);
  const Cpx<R> a{u.re + wr, u.im + wi};
  v = Cpx<R>{u.re - wr, u.im - wi};
  u = a;
}

template <class R>
OLSB_HD void dif_one(Cpx<R>& u, Cpx<R>& v) { dit_one(u, v); }
template <class R>
OLSB_HD void dif_i(Cpx<R>& u, Cpx<R>& v) {  // conj(w) = -i: b = (d.im, -d.re)
  const R dr = u.re - v.re, di = u.im - v.im;
  u = Cpx<R>{u.re + v.re, u.im + v.im};
  v = Cpx<R>{di, -dr};
}
template <class R>
OLSB_HD void dif_good(Cpx<R>& u, Cpx<R>& v, R c, R t) {
  // conj(w) = c (1 - i t): b = c (d.re + t d.im, d.im - t d.re)
  const R dr = u.re - v.re, di = u.im - v.im;
  u = Cpx<R>{u.re + v.re, u.im + v.im};
  v = Cpx<R>{c * fmaR(t, di, dr), c * fmaR(-t, dr, di)};
}
template <class R>
OLSB_HD void dif_rot(Cpx<R>& u, Cpx<R>& v, R c, R t) {
  // conj(w) = -i c (1 - i t): q = (d.re + t d.im, d.im - t d.re), b = -i c q
  const R dr = u.re - v.re, di = u.im - v.im;
  u = Cpx<R>{u.re + v.re, u.im + v.im};
  const R qr = fmaR(t, di, dr), qi = fmaR(-t, dr, di);
  v = Cpx<R>{c * qi, -c * qr};
}
template <class R>
OLSB_HD void dif_std(Cpx<R>& u, Cpx<R>& v, R c, R s) {
  const R dr = u.re - v.re, di = u.im - v.im;
  u = Cpx<R>{u.re + v.re, u.im + v.im};
  v = Cpx<R>{fmaR(dr, c, di * s), fmaR(di, c, -dr * s)};
}

// ---------------------------------------------------------------------------
// window passes.  x[E] are the thread's samples; local index a <-> window bits.
// ---------------------------------------------------------------------------
// Junction window (lo = 0, l = 0): all twiddles are compile-time constants.
template <class R, int LOGE, int G>
OLSB_HD void dit_pass_static(Cpx<R>* x) {
  constexpr int E = 1 << LOGE;
  sfor<0, G>([&](auto jc) {
    constexpr int j = decltype(jc)::value;
    sfor<0, E / 2>([&](auto bc) {
      constexpr int b = decltype(bc)::value;
      // b-th pair: insert a 0 at bit j
      constexpr int a = ((b >> j) << (j + 1)) | (b & ((1 << j) - 1));
      constexpr int k = a & ((1 << j) - 1);
      constexpr int m = k << (3 - j);
      constexpr int form = static_form(m);
      if constexpr (form == 0) {
        dit_one(x[a], x[a | (1 << j)]);
      } else if constexpr (form == 1) {
        dit_i(x[a], x[a | (1 << j)]);
      } else if constexpr (form == 2) {
        dit_good(x[a], x[a | (1 << j)], R(static_c(m)), R(static_t(m)));
      } else {
        dit_rot(x[a], x[a | (1 << j)], R(static_c(m)), R(static_t(m)));
      }
    });
  });
}

template <class R, int LOGE, int G>
OLSB_HD void dif_pass_static(Cpx<R>* x) {
  constexpr int E = 1 << LOGE;
  sfor<0, G>([&](auto jr) {
    constexpr int j = G - 1 - decltype(jr)::value;
    sfor<0, E / 2>([&](auto bc) {
      constexpr int b = decltype(bc)::value;
      constexpr int a = ((b >> j) << (j + 1)) | (b & ((1 << j) - 1));
      constexpr int k = a & ((1 << j) - 1);
      constexpr int m = k << (3 - j);
      constexpr int form = static_form(m);
      if constexpr (form == 0) {
        dif_one(x[a], x[a | (1 << j)]);
      } else if constexpr (form == 1) {
        dif_i(x[a], x[a | (1 << j)]);
      } else if constexpr (form == 2) {
        dif_good(x[a], x[a | (1 << j)], R(static_c(m)), R(static_t(m)));
      } else {
        dif_rot(x[a], x[a | (1 << j)], R(static_c(m)), R(static_t(m)));
      }
    });
  });
}

// Runtime windows (lo > 0): twiddle (j, k) is entry 2^j - 1 + k of the
// thread's 15-entry set `tw(idx)`.  Stages j < 2 use STD entries, j >= 2 the
// static GOOD/ROT form.
template <class R, class TW>
OLSB_HD void dit_pass_rt(Cpx<R>* x, const TW& tw) {
  sfor<0, 4>([&](auto jc) {
    constexpr int j = decltype(jc)::value;
    sfor<0, (1 << j)>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      const Tw<R> w = tw((1 << j) - 1 + k);
      sfor<0, (8 >> j)>([&](auto hc) {
        constexpr int a = (decltype(hc)::value << (j + 1)) | k;
        if constexpr (j < 2) {
          dit_std(x[a], x[a | (1 << j)], w.c, w.t);
        } else if constexpr (rot_static(j, k)) {
          dit_rot(x[a], x[a | (1 << j)], w.c, w.t);
        } else {
          dit_good(x[a], x[a | (1 << j)], w.c, w.t);
        }
      });
    });
  });
}

template <class R, class TW>
OLSB_HD void dif_pass_rt(Cpx<R>* x, const TW& tw) {
  sfor<0, 4>([&](auto jr) {
    constexpr int j = 3 - decltype(jr)::value;
    sfor<0, (1 << j)>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      const Tw<R> w = tw((1 << j) - 1 + k);
      sfor<0, (8 >> j)>([&](auto hc) {
        constexpr int a = (decltype(hc)::value << (j + 1)) | k;
        if constexpr (j < 2) {
          dif_std(x[a], x[a | (1 << j)], w.c, w.t);
        } else if constexpr (rot_static(j, k)) {
          dif_rot(x[a], x[a | (1 << j)], w.c, w.t);
        } else {
          dif_good(x[a], x[a | (1 << j)], w.c, w.t);
        }
      });
    });
  });
}

// Value of runtime twiddle entry idx (j, k) for low bits l of window lo, in
// double precision (theta / pi = (k 2^lo + l) / 2^(lo + j)).  Used to build
// the shared-memory tables; forward uses conj implicitly.
OLSB_HD void twiddle_entry(int lo, int idx, int l, double* c, double* t) {
  int j = 0;
  while ((2 << j) - 1 <= idx) ++j;  // idx in [2^j - 1, 2^(j+1) - 1)
  const int k = idx - ((1 << j) - 1);
  const double num = double(k) * double(1 << lo) + double(l);
  const double den = double(1 << (lo + j));
  double s, co;
#if defined(__CUDA_ARCH__)
  sincospi(num / den, &s, &co);
#else
  const double th = 3.14159265358979323846 * (num / den);
  s = std::sin(th);
  co = std::cos(th);
#endif
  if (j < 2) {
    *c = co;
    *t = s;
  } else if (rot_static(j, k)) {
    *c = s;
    *t = -co / s;
  } else {
    *c = co;
    *t = s / co;
  }
}

}  // namespace olsb
