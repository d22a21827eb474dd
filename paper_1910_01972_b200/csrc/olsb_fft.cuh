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
#ifndef OLSB_MID_REMAP
#define OLSB_MID_REMAP 1
#endif

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
  // runtime twiddle entries of window q: 8 pair slots (16 entries, one
  // unused) per low-bit value l, see twiddle_slot()
  static constexpr int tw_entries(int q) { return q == 0 ? 0 : 16 << lo(q); }
  // Thread-bit remap of window q: its low bits l = p & (2^lo - 1) pick the
  // tangent form of stages 0-1 through their top two bits ("hb", index bits
  // lo-2 and lo-1).  Those must be warp bits for the choice to be uniform.
  // With the plain mapping (thread bit i -> index bit i for i < lo) that
  // holds iff lo >= 7; a lower window with at least two warp bits to spare
  // swaps thread bits (lo-2, lo-1) with the top two thread bits instead.
  // Not at N = 4096: there the plain mapping makes the first inverse
  // exchange warp-local (warp bits = index bits 9-11 in both windows), which
  // saves one of its two 8-warp barriers per filter and outweighs the plain
  // (non-tangent) forms of window 1's first two stages (-4% on the cfg5
  // shard); at N = 2048 the remap wins (+5% without it).
  static constexpr bool remap(int q) {
    return OLSB_MID_REMAP && LOGN != 12 && q >= 1 && lo(q) >= 2 && lo(q) < 7 &&
           LOGT >= 7 && lo(q) <= LOGT - 2;
  }
  // windows whose first two stages use the FMA (tangent) forms
  static constexpr bool tan01(int q) {
    return q >= 1 && (lo(q) >= 7 || remap(q));
  }
  static OLSB_HD constexpr int perm(int q, int t) {
    if (!remap(q)) return t;
    const int a = remap(q) ? lo(q) - 2 : 0, b = remap(q) ? LOGT - 2 : 0;
    const int x = ((t >> a) ^ (t >> b)) & 3;  // swap two 2-bit fields
    return t ^ (x << a) ^ (x << b);
  }
  static constexpr int tw_offset(int q) {
    int off = 0;
    for (int i = 1; i < q; ++i) off += tw_entries(i);
    return off;
  }
  static constexpr int tw_total() { return tw_offset(P); }
  // thread part / element part of the in-place index in window q (disjoint
  // bit fields, so p = thread_part + elem_part)
  static OLSB_HD constexpr int thread_part(int q, int t) {
    const int l = lo(q);
    const int u = perm(q, t);
    return ((u >> l) << (l + LOGE)) | (u & ((1 << l) - 1));
  }
  static constexpr int elem_part(int q, int e) { return e << lo(q); }
  static OLSB_HD int low_bits(int q, int t) {
    return perm(q, t) & ((1 << lo(q)) - 1);
  }
  // Exchange x (windows x <-> x+1) is warp-local when every warp bit (thread
  // bits 5 .. LOGT-1) maps to the same index bit in both windows: each warp
  // then reads back only what it wrote, and a warp-level sync suffices.
  static constexpr bool warp_local(int x) {
    for (int b = 5; b < LOGT; ++b)
      if (thread_part(x, 1 << b) != thread_part(x + 1, 1 << b)) return false;
    return true;
  }
};

// ---------------------------------------------------------------------------
// shared-memory exchange layout: pos(p) = p + P1*(p>>K1) + P2*(p>>K2) +
// P3*(p>>K3).
// Linear over disjoint bit fields, so every address is a per-thread base plus
// a compile-time immediate.  Parameters found by tools/smem_layout_search.py
// (zero bank conflicts for every access of both transforms).
// ---------------------------------------------------------------------------
struct Pad {
  int k1, p1, k2, p2, k3, p3, stride;
};

constexpr Pad pad_for(bool dbl, int logn) {
  // LOGN 11 carries the Geo::remap thread-bit swap of the middle window
  constexpr Pad f[13] = {{2, 0, 2, 0, 2, 0, 2},    {2, 0, 2, 0, 2, 0, 2},
                         {2, 0, 2, 0, 2, 0, 6},    {2, 0, 2, 0, 2, 0, 10},
                         {2, 0, 2, 0, 2, 0, 18},   {2, 0, 4, 8, 4, 0, 42},
                         {4, 2, 5, 4, 5, 0, 76},   {2, 0, 4, 2, 4, 0, 152},
                         {2, 0, 4, 2, 4, 0, 286},  {4, 2, 7, 2, 7, 0, 580},
                         {4, 2, 7, 4, 7, 0, 1178}, {4, 2, 7, 2, 10, 4, 2336},
                         {2, 0, 4, 2, 4, 0, 4606}};
  constexpr Pad d[13] = {{2, 0, 2, 0, 2, 0, 1},    {2, 0, 2, 0, 2, 0, 1},
                         {2, 0, 2, 0, 2, 0, 5},    {2, 0, 2, 0, 2, 0, 9},
                         {2, 0, 2, 0, 2, 0, 17},   {2, 0, 4, 1, 4, 0, 34},
                         {2, 0, 4, 1, 4, 0, 68},   {2, 0, 4, 1, 4, 0, 135},
                         {2, 0, 4, 1, 4, 0, 271},  {2, 0, 4, 1, 4, 0, 543},
                         {2, 0, 4, 1, 4, 0, 1087}, {4, 1, 9, 2, 9, 0, 2181},
                         {2, 0, 4, 1, 4, 0, 4351}};
#if !OLSB_MID_REMAP
  // A/B builds without the middle-window remap: the round-1 layouts
  if (!dbl && logn == 11) return Pad{4, 2, 7, 8, 7, 0, 2422};
#endif
  return dbl ? d[logn] : f[logn];
}

// Per-exchange layouts (exchange X moves a segment between windows X and
// X+1).  fp32, N = 512..2048: index bit `rb` becomes address bit 0, so a
// 128-bit access pairs two samples that differ in that bit; plo / phi are the
// element bits paired on the lower / upper window side (-1: 64-bit access).
// Exchange 0 pairs on an index bit both windows hold in registers (the
// junction's batch bits), so both sides are 128-bit; exchange 1 pairs on the
// upper window's element bit 0.  Found by tools/smem_layout_search.py
// (xsearch), zero bank conflicts; other cases use pad_for with the junction
// side paired on bit 0.
struct XPad {
  int rb, k1, p1, k2, p2, k3, p3, plo, phi, span;
};
constexpr XPad xpad_for(bool dbl, int logn, int x) {
  if (!dbl && logn == 9)
    return x == 0 ? XPad{1, 4, 2, 4, 0, 4, 0, 1, 0, 574}
                  : XPad{5, 6, 4, 6, 0, 6, 0, -1, 0, 540};
  if (!dbl && logn == 10)
    return x == 0 ? XPad{2, 4, 2, 4, 0, 4, 0, 2, 0, 1150}
                  : XPad{6, 7, 8, 7, 0, 7, 0, -1, 0, 1080};
  if (!dbl && logn == 11)
    return x == 0 ? XPad{3, 4, 2, 9, 4, 9, 0, 3, 0, 2314}
                  : XPad{7, 9, 4, 9, 0, 9, 0, -1, 0, 2060};
  const Pad pd = pad_for(dbl, logn);
  return XPad{0,     pd.k1, pd.p1, pd.k2, pd.p2, pd.k3, pd.p3,
              (!dbl && x == 0) ? 0 : -1, -1, pd.stride};
}

template <class R, int LOGN, int X>
struct XLayout {
  static constexpr XPad xp = xpad_for(std::is_same<R, double>::value, LOGN, X);
  static OLSB_HD constexpr int rot(int p) {
    return xp.rb == 0 ? p
                      : ((p >> (xp.rb + 1)) << (xp.rb + 1)) |
                            ((p & ((1 << xp.rb) - 1)) << 1) | ((p >> xp.rb) & 1);
  }
  static OLSB_HD constexpr int pos(int p) {
    return rot(p) + xp.p1 * (rot(p) >> xp.k1) + xp.p2 * (rot(p) >> xp.k2) +
           xp.p3 * (rot(p) >> xp.k3);
  }
  // paired element bit for an access from window q (X or X+1)
  static constexpr int pair_bit(int q) { return q == X ? xp.plo : xp.phi; }
};

template <class R, int LOGN>
struct SmemLayout {
  // buffer stride per segment (Cpx<R> units): the largest exchange layout
  static constexpr int stride =
      xpad_for(std::is_same<R, double>::value, LOGN, 0).span >
              xpad_for(std::is_same<R, double>::value, LOGN, 1).span
          ? xpad_for(std::is_same<R, double>::value, LOGN, 0).span
          : xpad_for(std::is_same<R, double>::value, LOGN, 1).span;
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
// runtime-window stages j >= 2 have a static form per k (derivation in
// DESIGN.md §3): theta in [pi k/2^j, pi (k+1)/2^j)
constexpr bool rot_static(int j, int k) {
  return 4 * k >= (1 << j) && 4 * (k + 1) <= 3 * (1 << j);
}

// ---------------------------------------------------------------------------
// packed fp32x2 arithmetic (sm_100a FADD2 / FMUL2 / FFMA2).  A complex<float>
// is one aligned register pair; ptxas folds half swaps, per-half negation and
// scalar broadcasts (`pk(x, x)`) into the instruction's operand modifiers, so
// a complex butterfly costs half the issue slots of scalar code.  Device only;
// the host (tests) and fp64 paths use the scalar formulas below.
// ---------------------------------------------------------------------------
#if defined(__CUDA_ARCH__)
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ u64 pk(Cpx<float> v) { return pk(v.re, v.im); }
__device__ __forceinline__ Cpx<float> upk(u64 r) {
  Cpx<float> v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.re), "=f"(v.im) : "l"(r));
  return v;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
#define OLSB_PACKED(R) (std::is_same<R, float>::value)
#else
#define OLSB_PACKED(R) false
#endif

// complex product a * b
template <class R>
OLSB_HD Cpx<R> cmul(Cpx<R> a, Cpx<R> b) {
#if defined(__CUDA_ARCH__)
  if constexpr (OLSB_PACKED(R)) {
    // a.re (b.re, b.im) + a.im (-b.im, b.re)
    return upk(fma2(pk(-b.im, b.re), pk(a.im, a.im),
                    mul2(pk(b.re, b.im), pk(a.re, a.re))));
  }
#endif
  return Cpx<R>{fmaR(a.re, b.re, -a.im * b.im), fmaR(a.re, b.im, a.im * b.re)};
}

template <class R>
OLSB_HD Cpx<R> cscale(Cpx<R> a, R s) {
#if defined(__CUDA_ARCH__)
  if constexpr (OLSB_PACKED(R)) return upk(mul2(pk(a), pk(s, s)));
#endif
  return Cpx<R>{a.re * s, a.im * s};
}

// ---------------------------------------------------------------------------
// butterfly forms.  Inverse (DIT): a = u + w v, b = u - w v, w = e^{+i theta}.
// Forward (DIF): a = u + v, b = (u - v) conj(w).
// GOOD/ROT are the FMA ("tangent") forms: w v = c (v + i t v) is one FMA per
// component, and the scale c fuses into the butterfly adds, so a twiddled
// DIT butterfly is 6 FFMA (3 FFMA2) instead of 4 mul + 4 add.  ROT handles
// |tan| > 1 by rotating w by -pi/2 (the +i is a free swap/negate).
// ---------------------------------------------------------------------------
template <class R>
OLSB_HD void dit_one(Cpx<R>& u, Cpx<R>& v) {
#if defined(__CUDA_ARCH__)
  if constexpr (OLSB_PACKED(R)) {
    const u64 U = pk(u), V = pk(v);
    u = upk(add2(U, V));
    v = upk(sub2(U, V));
    return;
  }
#endif
  const Cpx<R> a{u.re + v.re, u.im + v.im};
  v = Cpx<R>{u.re - v.re, u.im - v.im};
  u = a;
}
template <class R>
OLSB_HD void dit_i(Cpx<R>& u, Cpx<R>& v) {  // w = i: w v = (-v.im, v.re)
#if defined(__CUDA_ARCH__)
  if constexpr (OLSB_PACKED(R)) {
    const u64 U = pk(u), IV = pk(-v.im, v.re);
    u = upk(add2(U, IV));
    v = upk(sub2(U, IV));
    return;
  }
#endif
  const Cpx<R> a{u.re - v.im, u.im + v.re};
  v = Cpx<R>{u.re + v.im, u.im - v.re};
  u = a;
}
template <class R>
OLSB_HD void dit_good(Cpx<R>& u, Cpx<R>& v, R c, R t) {
#if defined(__CUDA_ARCH__)
  if constexpr (OLSB_PACKED(R)) {
    const u64 U = pk(u);
    const u64 P = fma2(pk(v.im, v.re), pk(-t, t), pk(v));  // v + i t v
    u = upk(fma2(P, pk(c, c), U));
    v = upk(fma2(P, pk(-c, -c), U));
    return;
  }
#endif
  const R pr = fmaR(-t, v.im, v.re);
  const R pi = fmaR(t, v.re, v.im);
  const Cpx<R> a{fmaR(c, pr, u.re), fmaR(c, pi, u.im)};
  v = Cpx<R>{fmaR(-c, pr, u.re), fmaR(-c, pi, u.im)};
  u = a;
}
template <class R>
OLSB_HD void dit_rot(Cpx<R>& u, Cpx<R>& v, R c, R t) {
  // w = i c (1 + i t): w v = i c p = (-c p.im, c p.re)
#if defined(__CUDA_ARCH__)
  if constexpr (OLSB_PACKED(R)) {
    const u64 U = pk(u);
    const Cpx<float> p =
        upk(fma2(pk(v.im, v.re), pk(-t, t), pk(v)));  // v + i t v
    u = upk(fma2(pk(-p.im, p.re), pk(c, c), U));
    v = upk(fma2(pk(p.im, -p.re), pk(c, c), U));
    return;
  }
#endif
  const R pr = fmaR(-t, v.im, v.re);
  const R pi = fmaR(t, v.re, v.im);
  const Cpx<R> a{fmaR(-c, pi, u.re), fmaR(c, pr, u.im)};
  v = Cpx<R>{fmaR(c, pi, u.re), fmaR(-c, pr, u.im)};
  u = a;
}
template <class R>
OLSB_HD void dit_std(Cpx<R>& u, Cpx<R>& v, R c, R s) {
#if defined(__CUDA_ARCH__)
  if constexpr (OLSB_PACKED(R)) {
    const u64 U = pk(u);
    // v.re (c, s) + v.im (-s, c)
    const u64 W = fma2(pk(-s, c), pk(v.im, v.im), mul2(pk(c, s), pk(v.re, v.re)));
    u = upk(add2(U, W));
    v = upk(sub2(U, W));
    return;
  }
#endif
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
#if defined(__CUDA_ARCH__)
  if constexpr (OLSB_PACKED(R)) {
    const u64 U = pk(u), V = pk(v);
    const Cpx<float> d = upk(sub2(U, V));
    u = upk(add2(U, V));
    v = Cpx<float>{d.im, -d.re};
    return;
  }
#endif
  const R dr = u.re - v.re, di = u.im - v.im;
  u = Cpx<R>{u.re + v.re, u.im + v.im};
  v = Cpx<R>{di, -dr};
}
template <class R>
OLSB_HD void dif_good(Cpx<R>& u, Cpx<R>& v, R c, R t) {
  // conj(w) = c (1 - i t): b = c (d.re + t d.im, d.im - t d.re)
#if defined(__CUDA_ARCH__)
  if constexpr (OLSB_PACKED(R)) {
    const u64 U = pk(u), V = pk(v);
    const u64 D = sub2(U, V);
    const Cpx<float> d = upk(D);
    u = upk(add2(U, V));
    v = upk(mul2(fma2(pk(d.im, -d.re), pk(t, t), D), pk(c, c)));
    return;
  }
#endif
  const R dr = u.re - v.re, di = u.im - v.im;
  u = Cpx<R>{u.re + v.re, u.im + v.im};
  v = Cpx<R>{c * fmaR(t, di, dr), c * fmaR(-t, dr, di)};
}
template <class R>
OLSB_HD void dif_rot(Cpx<R>& u, Cpx<R>& v, R c, R t) {
  // conj(w) = -i c (1 - i t): q = (d.re + t d.im, d.im - t d.re), b = -i c q
#if defined(__CUDA_ARCH__)
  if constexpr (OLSB_PACKED(R)) {
    const u64 U = pk(u), V = pk(v);
    const u64 D = sub2(U, V);
    const Cpx<float> d = upk(D);
    u = upk(add2(U, V));
    const Cpx<float> q = upk(fma2(pk(d.im, -d.re), pk(t, t), D));
    v = upk(mul2(pk(q.im, -q.re), pk(c, c)));
    return;
  }
#endif
  const R dr = u.re - v.re, di = u.im - v.im;
  u = Cpx<R>{u.re + v.re, u.im + v.im};
  const R qr = fmaR(t, di, dr), qi = fmaR(-t, dr, di);
  v = Cpx<R>{c * qi, -c * qr};
}
template <class R>
OLSB_HD void dif_std(Cpx<R>& u, Cpx<R>& v, R c, R s) {
#if defined(__CUDA_ARCH__)
  if constexpr (OLSB_PACKED(R)) {
    const u64 U = pk(u), V = pk(v);
    const u64 D = sub2(U, V);
    const Cpx<float> d = upk(D);
    u = upk(add2(U, V));
    // d conj(w) = d.re (c, -s) + d.im (s, c)
    v = upk(fma2(pk(s, c), pk(d.im, d.im), mul2(pk(c, -s), pk(d.re, d.re))));
    return;
  }
#endif
  const R dr = u.re - v.re, di = u.im - v.im;
  u = Cpx<R>{u.re + v.re, u.im + v.im};
  v = Cpx<R>{fmaR(dr, c, di * s), fmaR(di, c, -dr * s)};
}

// ---------------------------------------------------------------------------
// Radix-4 DIT group over stages (j, j + 1) of a runtime window: samples x0..x3
// at a, a + 2^j, a + 2^(j+1), a + 3 2^j.  With v the stage-(j+1) twiddle of k
// (and w = v^2 the stage-j twiddle, i v the stage-(j+1) twiddle of k + 2^j):
//   A, B = x0 +- w x1,   C = v x2,   D = v^3 x3
//   z0, z2 = A +- (C + D),   z1, z3 = B +- i (C - D)
// which is the reference's two radix-2 stages exactly (same outputs at the
// same in-place positions).  In the FMA tangent forms (w x = rho c (x + i t x),
// rho = 1 GOOD / i ROT) and with C + D = c1 (rho1 P2 + r rho3 P3), r = c3 / c1,
// a group costs 11 FFMA2 instead of 4 x 3 (Linzer & Feig's radix-4 FMA
// count).  Table entries: w = (c_w, t_w), v = (c1, t1), v3 = (r, t3); the
// rho's are compile-time (RW, RV, R3 = ROT).
// ---------------------------------------------------------------------------
template <class R>
OLSB_HD Cpx<R> mul_i(Cpx<R> x) { return Cpx<R>{-x.im, x.re}; }
// x * i^Q (Q mod 4): a half swap and / or negations, which ptxas folds into
// the operand modifiers of an FFMA2 multiplicand
template <int Q, class R>
OLSB_HD Cpx<R> rot_q(Cpx<R> x) {
  constexpr int q = ((Q % 4) + 4) % 4;
  if constexpr (q == 0) return x;
  if constexpr (q == 1) return Cpx<R>{-x.im, x.re};
  if constexpr (q == 2) return Cpx<R>{-x.re, -x.im};
  return Cpx<R>{x.im, -x.re};
}

// (the rotations rho are kept on FFMA2 multiplicands only -- an addend cannot
// carry swap / negate modifiers:  C + D = c1 rho1 (P2 + r (rho3 / rho1) P3))
template <bool RW, bool RV, bool R3, class R>
OLSB_HD void dit_r4(Cpx<R>& x0, Cpx<R>& x1, Cpx<R>& x2, Cpx<R>& x3, Tw<R> w,
                    Tw<R> v, Tw<R> v3) {
  constexpr int QW = RW ? 1 : 0, Q1 = RV ? 1 : 0, Q3 = (R3 ? 1 : 0) - Q1;
#if defined(__CUDA_ARCH__)
  if constexpr (OLSB_PACKED(R)) {
    const u64 X0 = pk(x0);
    const Cpx<float> p1 = upk(fma2(pk(x1.im, x1.re), pk(-w.t, w.t), pk(x1)));
    const Cpx<float> p2 = upk(fma2(pk(x2.im, x2.re), pk(-v.t, v.t), pk(x2)));
    const Cpx<float> p3 = upk(fma2(pk(x3.im, x3.re), pk(-v3.t, v3.t), pk(x3)));
    const u64 A = fma2(pk(rot_q<QW>(p1)), pk(w.c, w.c), X0);
    const u64 B = fma2(pk(rot_q<QW>(p1)), pk(-w.c, -w.c), X0);
    const Cpx<float> sp = upk(fma2(pk(rot_q<Q3>(p3)), pk(v3.c, v3.c), pk(p2)));
    const Cpx<float> dm = upk(fma2(pk(rot_q<Q3>(p3)), pk(-v3.c, -v3.c), pk(p2)));
    x0 = upk(fma2(pk(rot_q<Q1>(sp)), pk(v.c, v.c), A));
    x2 = upk(fma2(pk(rot_q<Q1>(sp)), pk(-v.c, -v.c), A));
    x1 = upk(fma2(pk(rot_q<Q1 + 1>(dm)), pk(v.c, v.c), B));
    x3 = upk(fma2(pk(rot_q<Q1 + 1>(dm)), pk(-v.c, -v.c), B));
    return;
  }
#endif
  auto tanf = [](Cpx<R> x, R t) {
    return Cpx<R>{fmaR(-t, x.im, x.re), fmaR(t, x.re, x.im)};
  };
  auto axpy = [](R c, Cpx<R> x, Cpx<R> y) {
    return Cpx<R>{fmaR(c, x.re, y.re), fmaR(c, x.im, y.im)};
  };
  const Cpx<R> p1 = rot_q<QW>(tanf(x1, w.t));
  const Cpx<R> p2 = tanf(x2, v.t);
  const Cpx<R> p3 = rot_q<Q3>(tanf(x3, v3.t));
  const Cpx<R> A = axpy(w.c, p1, x0), B = axpy(-w.c, p1, x0);
  const Cpx<R> sp = axpy(v3.c, p3, p2), dm = axpy(-v3.c, p3, p2);
  x0 = axpy(v.c, rot_q<Q1>(sp), A);
  x2 = axpy(-v.c, rot_q<Q1>(sp), A);
  x1 = axpy(v.c, rot_q<Q1 + 1>(dm), B);
  x3 = axpy(-v.c, rot_q<Q1 + 1>(dm), B);
}

// DIF butterfly with the twiddle i W, W = (c, t) in form ROT_BASE: i W is
// ROT with the same (c, t) when W is GOOD, GOOD with (-c, t) when W is ROT
// (used where a table slot holds radix-4 data instead of i W)
template <bool ROT_BASE, class R>
OLSB_HD void dif_times_i(Cpx<R>& u, Cpx<R>& v, R c, R t) {
  if constexpr (ROT_BASE) {
    dif_good(u, v, -c, t);
  } else {
    dif_rot(u, v, c, t);
  }
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

// Runtime windows (lo > 0).  Twiddle (j, k) of a thread is entry
// idx = 2^j - 1 + k of its 15-entry set; accessors hand them out as idx 0
// (get0) and pairs (2p - 1, 2p), p = 1..7 (get2) so a shared-memory table is
// read with 128-bit loads.  Stages j >= 2 use the static GOOD/ROT form.
// Stages j < 2 use STD, or with TAN01 the FMA forms, picked by `hb` = the top
// two bits of l (warp-uniform where TAN01 is enabled):
//   j = 0     : ROT iff hb in {1, 2}  (theta = pi x, x = l / 2^lo)
//   j = 1, k=0: ROT iff hb >= 2       (theta = pi x / 2)
//   j = 1, k=1: ROT iff hb <  2       (theta = pi (1 + x) / 2)
template <class R>
struct TwPair {
  Tw<R> a, b;
};

template <class R, bool TAN01, class TW>
OLSB_HD void dit_pass_rt(Cpx<R>* x, const TW& tw, int hb) {
  // stages 0, 1: radix-4 groups {a, a+1, a+2, a+3} with w = idx 0, v = idx 1,
  // v^3 data = idx 2 (forms by hb, warp-uniform under TAN01); without the
  // tangent forms: radix-2 STD butterflies with idx 0, 1, 2
  if constexpr (TAN01) {
    const Tw<R> w = tw.get0();
    const TwPair<R> p = tw.get2(1);
    auto groups = [&](auto rw, auto rv, auto r3) {
      sfor<0, 4>([&](auto gc) {
        constexpr int a = 4 * decltype(gc)::value;
        dit_r4<decltype(rw)::value != 0, decltype(rv)::value != 0,
               decltype(r3)::value != 0>(x[a], x[a + 1], x[a + 2], x[a + 3],
                                         w, p.a, p.b);
      });
    };
    // w: ROT iff hb in {1, 2}; v: ROT iff hb >= 2; v^3: ROT iff hb odd
    if (hb == 0) {
      groups(IC<0>{}, IC<0>{}, IC<0>{});
    } else if (hb == 1) {
      groups(IC<1>{}, IC<0>{}, IC<1>{});
    } else if (hb == 2) {
      groups(IC<1>{}, IC<1>{}, IC<0>{});
    } else {
      groups(IC<0>{}, IC<1>{}, IC<1>{});
    }
  } else {
    {
      const Tw<R> w = tw.get0();
      sfor<0, 8>([&](auto hc) {
        constexpr int a = 2 * decltype(hc)::value;
        dit_std(x[a], x[a + 1], w.c, w.t);
      });
    }
    {
      const TwPair<R> w = tw.get2(1);
      sfor<0, 4>([&](auto hc) {
        constexpr int a = 4 * decltype(hc)::value;
        dit_std(x[a], x[a + 2], w.a.c, w.a.t);
        dit_std(x[a + 1], x[a + 3], w.b.c, w.b.t);
      });
    }
  }
  // stages 2, 3: radix-4 groups {k, k+4, k+8, k+12}, k < 4: w = idx 3 + k,
  // v = idx 7 + k, v^3 data = idx 11 + k; static forms
  const TwPair<R> w01 = tw.get2(2), w23 = tw.get2(3);
  const TwPair<R> v01 = tw.get2(4), v23 = tw.get2(5);
  const TwPair<R> t01 = tw.get2(6), t23 = tw.get2(7);
  sfor<0, 4>([&](auto kc) {
    constexpr int k = decltype(kc)::value;
    const Tw<R> w = k == 0 ? w01.a : k == 1 ? w01.b : k == 2 ? w23.a : w23.b;
    const Tw<R> v = k == 0 ? v01.a : k == 1 ? v01.b : k == 2 ? v23.a : v23.b;
    const Tw<R> t = k == 0 ? t01.a : k == 1 ? t01.b : k == 2 ? t23.a : t23.b;
    dit_r4<rot_static(2, k), rot_static(3, k), (k & 1) != 0>(
        x[k], x[k + 4], x[k + 8], x[k + 12], w, v, t);
  });
}

template <class R, bool TAN01, class TW>
OLSB_HD void dif_pass_rt(Cpx<R>* x, const TW& tw, int hb) {
  // j = 3, 2: static forms.  Stage-3 twiddles of k >= 4 are i times those
  // of k - 4 (their table slots hold the inverse's radix-4 data)
  sfor<0, 2>([&](auto jr) {
    constexpr int j = 3 - decltype(jr)::value;
    sfor<(1 << (j - 1)), (1 << j)>([&](auto pc) {
      constexpr int pp = decltype(pc)::value;
      const TwPair<R> w = tw.get2(j == 3 && pp >= 6 ? pp - 2 : pp);
      sfor<0, 2>([&](auto hc2) {
        constexpr int idx = 2 * pp - 1 + decltype(hc2)::value;
        constexpr int k = idx - ((1 << j) - 1);
        const Tw<R> ww = decltype(hc2)::value == 0 ? w.a : w.b;
        sfor<0, (8 >> j)>([&](auto hc) {
          constexpr int a = (decltype(hc)::value << (j + 1)) | k;
          if constexpr (j == 3 && k >= 4) {
            dif_times_i<rot_static(3, k - 4)>(x[a], x[a | (1 << j)], ww.c, ww.t);
          } else if constexpr (rot_static(j, k)) {
            dif_rot(x[a], x[a | (1 << j)], ww.c, ww.t);
          } else {
            dif_good(x[a], x[a | (1 << j)], ww.c, ww.t);
          }
        });
      });
    });
  });
  // j = 1 (k = 1: i times the k = 0 twiddle; its slot holds radix-4 data)
  {
    const TwPair<R> w = tw.get2(1);
    if constexpr (TAN01) {
      if (hb >= 2) {
        sfor<0, 4>([&](auto hc) {
          constexpr int a = 4 * decltype(hc)::value;
          dif_rot(x[a], x[a + 2], w.a.c, w.a.t);
          dif_times_i<true>(x[a + 1], x[a + 3], w.a.c, w.a.t);
        });
      } else {
        sfor<0, 4>([&](auto hc) {
          constexpr int a = 4 * decltype(hc)::value;
          dif_good(x[a], x[a + 2], w.a.c, w.a.t);
          dif_times_i<false>(x[a + 1], x[a + 3], w.a.c, w.a.t);
        });
      }
    } else {
      sfor<0, 4>([&](auto hc) {
        constexpr int a = 4 * decltype(hc)::value;
        dif_std(x[a], x[a + 2], w.a.c, w.a.t);
        dif_std(x[a + 1], x[a + 3], w.b.c, w.b.t);
      });
    }
  }
  // j = 0
  {
    const Tw<R> w = tw.get0();
    if constexpr (TAN01) {
      if (hb == 1 || hb == 2) {
        sfor<0, 8>([&](auto hc) {
          constexpr int a = 2 * decltype(hc)::value;
          dif_rot(x[a], x[a + 1], w.c, w.t);
        });
      } else {
        sfor<0, 8>([&](auto hc) {
          constexpr int a = 2 * decltype(hc)::value;
          dif_good(x[a], x[a + 1], w.c, w.t);
        });
      }
    } else {
      sfor<0, 8>([&](auto hc) {
        constexpr int a = 2 * decltype(hc)::value;
        dif_std(x[a], x[a + 1], w.c, w.t);
      });
    }
  }
}

// ---------------------------------------------------------------------------
// Reference-arithmetic passes (exact mode).  The same stage / element pairing
// as the fast passes (the reference's in-place radix-2 positions), but every
// butterfly is the reference's: an explicit complex product by the fp32
// table entry w = tw[(p mod 2^b) * (N >> (b + 1))] (dif_fwd, dit_inv with
// twc = conj(tw), _kernels_nb.py:11-51), written with non-contracting
// round-to-nearest intrinsics so no FMA is formed.  Tw fields hold (re, im)
// of w here.  Results are bit-identical to the reference's fp32 (and fp64)
// kernels.
// ---------------------------------------------------------------------------
#if defined(__CUDACC__)
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// a * b as the reference computes complex products (oracle cmul)
template <class R>
__device__ __forceinline__ Cpx<R> cmul_ref(Cpx<R> a, Cpx<R> b) {
  return Cpx<R>{sub_rn(mul_rn(a.re, b.re), mul_rn(a.im, b.im)),
                add_rn(mul_rn(a.re, b.im), mul_rn(a.im, b.re))};
}
// dit_inv butterfly: v' = v * conj(w); u, v <- u + v', u - v'
template <class R>
__device__ __forceinline__ void dit_ref(Cpx<R>& u, Cpx<R>& v, Tw<R> w) {
  const Cpx<R> p = cmul_ref(v, Cpx<R>{w.c, -w.t});
  const Cpx<R> a{add_rn(u.re, p.re), add_rn(u.im, p.im)};
  v = Cpx<R>{sub_rn(u.re, p.re), sub_rn(u.im, p.im)};
  u = a;
}
// dif_fwd butterfly: u, v <- u + v, (u - v) * w
template <class R>
__device__ __forceinline__ void dif_ref(Cpx<R>& u, Cpx<R>& v, Tw<R> w) {
  const Cpx<R> d{sub_rn(u.re, v.re), sub_rn(u.im, v.im)};
  u = Cpx<R>{add_rn(u.re, v.re), add_rn(u.im, v.im)};
  v = cmul_ref(d, Cpx<R>{w.c, w.t});
}

// runtime window (4 stages over 16 elements), entries idx = 2^j - 1 + k
template <class R, bool INV, class TW>
__device__ __forceinline__ void pass_ref(Cpx<R>* x, const TW& tw) {
  auto stage = [&](auto jc) {
    constexpr int j = decltype(jc)::value;
    auto bf = [&](Tw<R> w, auto kc) {
      constexpr int k = decltype(kc)::value;
      sfor<0, (8 >> j)>([&](auto hc) {
        constexpr int a = (decltype(hc)::value << (j + 1)) | k;
        if constexpr (INV) {
          dit_ref(x[a], x[a | (1 << j)], w);
        } else {
          dif_ref(x[a], x[a | (1 << j)], w);
        }
      });
    };
    if constexpr (j == 0) {
      bf(tw.get0(), IC<0>{});
    } else {
      sfor<(1 << (j - 1)), (1 << j)>([&](auto pc) {
        constexpr int pp = decltype(pc)::value;
        const TwPair<R> w = tw.get2(pp);
        bf(w.a, IC<2 * pp - 1 - ((1 << j) - 1)>{});
        bf(w.b, IC<2 * pp - ((1 << j) - 1)>{});
      });
    }
  };
  if constexpr (INV) {
    sfor<0, 4>([&](auto jc) { stage(jc); });
  } else {
    sfor<0, 4>([&](auto jr) { stage(IC<3 - decltype(jr)::value>{}); });
  }
}

// junction window (lo = 0): G stages, entries jt[2^j - 1 + k] (broadcast)
template <class R, int LOGE, int G, bool INV>
__device__ __forceinline__ void pass_static_ref(Cpx<R>* x, const Tw<R>* jt) {
  constexpr int E = 1 << LOGE;
  auto stage = [&](auto jc) {
    constexpr int j = decltype(jc)::value;
    sfor<0, E / 2>([&](auto bc) {
      constexpr int b = decltype(bc)::value;
      constexpr int a = ((b >> j) << (j + 1)) | (b & ((1 << j) - 1));
      constexpr int k = a & ((1 << j) - 1);
      const Tw<R> w = jt[(1 << j) - 1 + k];
      if constexpr (INV) {
        dit_ref(x[a], x[a | (1 << j)], w);
      } else {
        dif_ref(x[a], x[a | (1 << j)], w);
      }
    });
  };
  if constexpr (INV) {
    sfor<0, G>([&](auto jc) { stage(jc); });
  } else {
    sfor<0, G>([&](auto jr) { stage(IC<G - 1 - decltype(jr)::value>{}); });
  }
}
#endif

// Table slot of twiddle idx: slot s = (idx + 1) / 2 holds the pair
// (2s - 1, 2s) (slot 0: idx 0 and an unused half); half = 1 for even idx > 0.
OLSB_HD constexpr int twiddle_slot(int idx) { return (idx + 1) >> 1; }
OLSB_HD constexpr int twiddle_half(int idx) { return idx == 0 ? 0 : ((idx + 1) & 1); }

// Value of runtime twiddle entry idx (j, k) for low bits l of window lo, in
// double precision (theta / pi = (k 2^lo + l) / 2^(lo + j)).  Used to build
// the tables; the forward transform uses conj implicitly.  idx < 0 = unused.
OLSB_HD void twiddle_entry(int lo, int idx, int l, bool tan01, double* c,
                           double* t) {
  if (idx < 0) {
    *c = 0.0;
    *t = 0.0;
    return;
  }
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
  bool rot;
  if (j < 2) {
    if (!tan01) {
      *c = co;
      *t = s;
      return;
    }
    const int hb = lo >= 2 ? (l >> (lo - 2)) & 3 : 0;
    rot = (j == 0) ? (hb == 1 || hb == 2) : (k == 0 ? hb >= 2 : hb < 2);
  } else {
    rot = rot_static(j, k);
  }
  if (rot) {
    *c = s;
    *t = -co / s;
  } else {
    *c = co;
    *t = s / co;
  }
}

// Runtime-window table entry idx for the radix-4 inverse (dit_pass_rt): as
// twiddle_entry, except the slots of the stage-(j+1) twiddles i v of
// k + 2^j, which the radix-4 groups do not need, hold the groups' v^3 data
// (r = c3 / c1, t3): idx 11 + k for the stage-(2, 3) group k, and idx 2 for
// the stage-(0, 1) group when the tangent forms are on.  v^3's form is static
// (ROT iff k, or hb, is odd), |t3| <= tan(3 pi / 8).
OLSB_HD void twiddle_entry_r4(int lo, int idx, int l, bool tan01, double* c,
                              double* t) {
  const bool g23 = idx >= 11 && idx <= 14;
  const bool g01 = idx == 2 && tan01;
  if (!g23 && !g01) {
    twiddle_entry(lo, idx, l, tan01, c, t);
    return;
  }
  const int k = g23 ? idx - 11 : 0;
  const int j1 = g23 ? 3 : 1;                      // stage of v
  const int hb = lo >= 2 ? (l >> (lo - 2)) & 3 : 0;
  const double num = double(k) * double(1 << lo) + double(l);
  const double den = double(1 << (lo + j1));
  double s1, c1, s3, c3;
#if defined(__CUDA_ARCH__)
  sincospi(num / den, &s1, &c1);
  sincospi(3.0 * num / den, &s3, &c3);
#else
  const double th = 3.14159265358979323846 * (num / den);
  s1 = std::sin(th);
  c1 = std::cos(th);
  s3 = std::sin(3.0 * th);
  c3 = std::cos(3.0 * th);
#endif
  const bool rot_v = g23 ? rot_static(3, k) : hb >= 2;
  const bool rot_3 = ((g23 ? k : hb) & 1) != 0;
  const double cv = rot_v ? s1 : c1;
  *c = (rot_3 ? s3 : c3) / cv;
  *t = rot_3 ? -c3 / s3 : s3 / c3;
}

// entry i of window lo's table -> (idx or -1, l)
// Table entry i of a window -> (idx, l).  fp32 tables are [slot][l][half]
// (a thread's pair is one 16-byte load); fp64 tables are [slot][half][l]
// (`split`: consecutive l are consecutive 16-byte entries, so a warp's
// 128-bit loads are bank-conflict free).
OLSB_HD void twiddle_decode(int lo, int i, int* idx, int* l, bool split = false) {
  int h, sl;
  if (split) {
    *l = i & ((1 << lo) - 1);
    h = (i >> lo) & 1;
    sl = i >> (lo + 1);
  } else {
    h = i & 1;
    const int rest = i >> 1;
    *l = rest & ((1 << lo) - 1);
    sl = rest >> lo;
  }
  *idx = sl == 0 ? (h == 0 ? 0 : -1) : 2 * sl - 1 + h;
}

}  // namespace olsb
