// Host emulation of the engine's window-pass FFT (tests only).
//
// Runs the exact per-thread pass functions of csrc/olsb_fft.cuh for every
// thread of one segment sequentially, with a plain array standing in for
// shared memory (threads of a window touch disjoint samples, so sequential
// execution is exact).  Lets the CPU test suite check the decomposition,
// twiddle forms and in-place index maps against numpy without a GPU.
#include <vector>

#include "olsb_fft.cuh"

using namespace olsb;

template <class R, int LOGN>
static void run(const R* in, R* out, bool inverse) {
  using G = Geo<LOGN>;
  const Cpx<R>* src = reinterpret_cast<const Cpx<R>*>(in);
  std::vector<Cpx<R>> a(src, src + G::N);
  auto window = [&](auto qc) {
    constexpr int q = decltype(qc)::value;
    for (int t = 0; t < G::T; ++t) {
      Cpx<R> x[G::E];
      const int base = G::thread_part(q, t);
      for (int e = 0; e < G::E; ++e) x[e] = a[base + G::elem_part(q, e)];
      if constexpr (q == 0) {
        if (inverse)
          dit_pass_static<R, G::LOGE, G::G0>(x);
        else
          dif_pass_static<R, G::LOGE, G::G0>(x);
      } else {
        struct Acc {
          Tw<R> tw[15];
          Tw<R> get0() const { return tw[0]; }
          TwPair<R> get2(int p) const { return TwPair<R>{tw[2 * p - 1], tw[2 * p]}; }
        } acc;
        const int l = G::low_bits(q, t);
        for (int i = 0; i < 15; ++i) {
          double c, tt;
          twiddle_entry_r4(G::lo(q), i, l, G::tan01(q), &c, &tt);
          acc.tw[i] = Tw<R>{R(c), R(tt)};
        }
        const int hb = G::lo(q) >= 2 ? (l >> (G::lo(q) - 2)) & 3 : 0;
        if (inverse)
          dit_pass_rt<R, G::tan01(q)>(x, acc, hb);
        else
          dif_pass_rt<R, G::tan01(q)>(x, acc, hb);
      }
      for (int e = 0; e < G::E; ++e) a[base + G::elem_part(q, e)] = x[e];
    }
  };
  if (inverse) {
    sfor<0, G::P>([&](auto qc) { window(qc); });
    for (auto& v : a) {
      v.re /= R(G::N);
      v.im /= R(G::N);
    }
  } else {
    sfor<0, G::P>([&](auto qr) { window(IC<G::P - 1 - decltype(qr)::value>{}); });
  }
  Cpx<R>* dst = reinterpret_cast<Cpx<R>*>(out);
  for (int i = 0; i < G::N; ++i) dst[i] = a[i];
}

template <class R>
static int dispatch(int logn, const R* in, R* out, bool inverse) {
  switch (logn) {
    case 2: run<R, 2>(in, out, inverse); return 0;
    case 3: run<R, 3>(in, out, inverse); return 0;
    case 4: run<R, 4>(in, out, inverse); return 0;
    case 5: run<R, 5>(in, out, inverse); return 0;
    case 6: run<R, 6>(in, out, inverse); return 0;
    case 7: run<R, 7>(in, out, inverse); return 0;
    case 8: run<R, 8>(in, out, inverse); return 0;
    case 9: run<R, 9>(in, out, inverse); return 0;
    case 10: run<R, 10>(in, out, inverse); return 0;
    case 11: run<R, 11>(in, out, inverse); return 0;
    case 12: run<R, 12>(in, out, inverse); return 0;
  }
  return -1;
}

extern "C" {
int emu_fft_f(int logn, const float* in, float* out, int inverse) {
  return dispatch<float>(logn, in, out, inverse != 0);
}
int emu_fft_d(int logn, const double* in, double* out, int inverse) {
  return dispatch<double>(logn, in, out, inverse != 0);
}
// shared-memory layout probe for the layout tests:
// k1, p1, k2, p2, k3, p3, stride
void emu_pad(int dbl, int logn, int* out7) {
  const Pad pd = pad_for(dbl != 0, logn);
  out7[0] = pd.k1;
  out7[1] = pd.p1;
  out7[2] = pd.k2;
  out7[3] = pd.p2;
  out7[4] = pd.k3;
  out7[5] = pd.p3;
  out7[6] = pd.stride;
}
// per-exchange layout probe: rb, k1, p1, k2, p2, k3, p3, plo, phi, span
void emu_xpad(int dbl, int logn, int x, int* out10) {
  const XPad p = xpad_for(dbl != 0, logn, x);
  const int v[10] = {p.rb, p.k1, p.p1, p.k2, p.p2, p.k3, p.p3, p.plo, p.phi, p.span};
  for (int i = 0; i < 10; ++i) out10[i] = v[i];
}
}
