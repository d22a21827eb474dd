// olsb_w64.cuh — warp-per-segment fused OLS kernel for N = 2048 (fp32).
//
// Same computation as fused_c2c_kernel (olsb_engine.cuh) — the reference's
// per-segment pipeline of _kernels_nb.py:265-285: gather, dif_fwd, then per
// filter multiply / dit_inv / _store — with a different decomposition of the
// 2048-point transforms:
//
//   * one WARP owns a segment: each lane holds E = 64 samples in registers,
//     so the 11 radix-2 stages split into two register windows,
//       window A = index bits 0..5  (lane L holds p = 64 L + e, e < 64)
//       window B = index bits 6..10 (+ bit 5 as a batch bit: lane l holds
//                  p = 64 h + 32 b + l, h < 32, b < 2)
//     and a transform needs ONE exchange through shared memory instead of
//     two, and that exchange is warp-local (__syncwarp, no CTA barrier):
//     segments never wait for each other;
//   * window A's six stages have compile-time twiddles (theta = pi m / 32):
//     FMA tangent forms with immediate operands, no twiddle registers;
//   * window B's twiddles depend on the lane only: 62 (c, t) pairs per lane,
//     parked in tensor memory (tcgen05.ld, off the shared-memory pipe),
//     shared by every warp of a lane quadrant;
//   * the segment spectrum (64 complex per lane) lives in tensor memory for
//     the whole filter loop; filter spectra stream through the TEX path,
//     16 complex per lane at a time, fetched ahead of use.
//
// Per filter-segment this moves 32 KB through shared memory (the E = 16
// kernel: 64 KB) with no cross-warp barrier.  Stage pairings and in-place
// positions are the reference's (radix-2 DIT / DIF), so the forward output
// is in the reference's bit-reversed order and the inverse ends in natural
// order, exactly as in olsb_fft.cuh.
#pragma once

#include "olsb_engine.cuh"

// compile-time ablation bits for bottleneck analysis (results wrong when
// set): 2 no exchange shared-memory traffic, 4 no output staging; build with
// OLSB_NVCC_EXTRA=-DOLSB_W64_ABL=k (output writes: OLSB_DEBUG=1 at run time)
#ifndef OLSB_W64_ABL
#define OLSB_W64_ABL 0
#endif

namespace olsb {
namespace w64 {

constexpr int LOGN = 11, N = 2048, E = 64;
constexpr int STRIDE = 66;           // padded 64-sample row (complex units)
constexpr int BUF = 32 * STRIDE;     // per-warp exchange buffer (complex)

// cos(pi m / 32), m = 0..16 (exactly 0 at 16); other angles by symmetry
constexpr double kC16[17] = {1.0,
                             0.99518472667219688624,
                             0.98078528040323044913,
                             0.95694033573220886494,
                             0.92387953251128675613,
                             0.88192126434835502971,
                             0.83146961230254523708,
                             0.77301045336273696081,
                             0.70710678118654752440,
                             0.63439328416364549822,
                             0.55557023301960222474,
                             0.47139673682599764856,
                             0.38268343236508977173,
                             0.29028467725446236764,
                             0.19509032201612826785,
                             0.09801714032956060199,
                             0.0};
constexpr double cos32(int m) {  // cos(pi m / 32), any m
  m = ((m % 64) + 64) % 64;
  return m <= 16 ? kC16[m] : m <= 32 ? -kC16[32 - m] : m <= 48 ? -kC16[m - 32]
                                                                : kC16[64 - m];
}
constexpr double sin32(int m) { return cos32(m - 16); }
// static twiddle forms (olsb_fft.cuh): 0 one, 1 i, 2 GOOD, 3 ROT
constexpr int form32(int m) {
  return m == 0 ? 0 : m == 16 ? 1 : (m <= 8 || m >= 24) ? 2 : 3;
}
constexpr double c32(int m) { return form32(m) == 3 ? sin32(m) : cos32(m); }
constexpr double t32(int m) {
  return form32(m) == 3 ? -cos32(m) / sin32(m) : sin32(m) / cos32(m);
}

// DIT stage J over NE register samples: pairs (a, a + 2^J), theta =
// pi (a mod 2^J) / 2^J = pi m / 32
template <int J, int NE>
__device__ __forceinline__ void dit_stage_static(Cpx<float>* x) {
  sfor<0, NE / 2>([&](auto bc) {
    constexpr int b = decltype(bc)::value;
    constexpr int a = ((b >> J) << (J + 1)) | (b & ((1 << J) - 1));
    constexpr int m = (a & ((1 << J) - 1)) << (5 - J);
    constexpr int fm = form32(m);
    if constexpr (fm == 0) {
      dit_one(x[a], x[a | (1 << J)]);
    } else if constexpr (fm == 1) {
      dit_i(x[a], x[a | (1 << J)]);
    } else if constexpr (fm == 2) {
      dit_good(x[a], x[a | (1 << J)], float(c32(m)), float(t32(m)));
    } else {
      dit_rot(x[a], x[a | (1 << J)], float(c32(m)), float(t32(m)));
    }
  });
}
template <int J, int NE>
__device__ __forceinline__ void dif_stage_static(Cpx<float>* x) {
  sfor<0, NE / 2>([&](auto bc) {
    constexpr int b = decltype(bc)::value;
    constexpr int a = ((b >> J) << (J + 1)) | (b & ((1 << J) - 1));
    constexpr int m = (a & ((1 << J) - 1)) << (5 - J);
    constexpr int fm = form32(m);
    if constexpr (fm == 0) {
      dif_one(x[a], x[a | (1 << J)]);
    } else if constexpr (fm == 1) {
      dif_i(x[a], x[a | (1 << J)]);
    } else if constexpr (fm == 2) {
      dif_good(x[a], x[a | (1 << J)], float(c32(m)), float(t32(m)));
    } else {
      dif_rot(x[a], x[a | (1 << J)], float(c32(m)), float(t32(m)));
    }
  });
}

// Window-B runtime stage j on the 32 samples z[0..32) of batch B: pairs
// (h, h + 2^j), twiddle entry idx = 2^j - 1 + k, k = h mod 2^j.  Forms:
// j = 0 STD (its GOOD/ROT choice would depend on lane bit 4), j = 1 fixed per
// (B, k) because index bit 5 is the batch bit, j >= 2 rot_static(j, k).
template <int J, int B>
constexpr bool rot_b(int k) {
  return J == 1 ? (k == 0 ? B == 1 : B == 0) : rot_static(J, k);
}
// (butterflies b in [BLO, BHI); the twiddle of k comes from tw(IC<k>))
template <int J, int B, bool INV, int BLO = 0, int BHI = 16, class TWF>
__device__ __forceinline__ void stage_rt(Cpx<float>* z, const TWF& tw) {
  sfor<BLO, BHI>([&](auto bc) {
    constexpr int b = decltype(bc)::value;
    constexpr int a = ((b >> J) << (J + 1)) | (b & ((1 << J) - 1));
    constexpr int k = a & ((1 << J) - 1);
    const Tw<float> w = tw(IC<k>{});
    Cpx<float>& u = z[a];
    Cpx<float>& v = z[a | (1 << J)];
    if constexpr (J == 0) {
      if constexpr (INV) dit_std(u, v, w.c, w.t); else dif_std(u, v, w.c, w.t);
    } else if constexpr (rot_b<J, B>(k)) {
      if constexpr (INV) dit_rot(u, v, w.c, w.t); else dif_rot(u, v, w.c, w.t);
    } else {
      if constexpr (INV) dit_good(u, v, w.c, w.t); else dif_good(u, v, w.c, w.t);
    }
  });
}

// 16 consecutive columns of the thread's lane -> r[0..16), no wait
__device__ __forceinline__ void tm_ld16(uint32_t ta, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,"
      "%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]),
        "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
        "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15])
      : "r"(ta));
}
// wait for every outstanding tcgen05.ld; the 32 registers are tied to the
// wait so no consumer can be scheduled above it
__device__ __forceinline__ void tm_wait32(uint32_t* r) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]),
                 "+r"(r[5]), "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]),
                 "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),
                 "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]),
                 "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]),
                 "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]),
                 "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

// TMA bulk copy shared -> global (one elected lane) and its completion
__device__ __forceinline__ void bulk_store(void* g, const void* sm, uint32_t bytes) {
  asm volatile(
      "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
      "cp.async.bulk.commit_group;" ::"l"(g),
      "r"(smem_u32(sm)), "r"(bytes)
      : "memory");
}
// the smem source of every committed bulk store has been read
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// generic-proxy smem writes -> visible to the async (TMA) proxy
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// TMEM columns (per lane): [slot * 128, +128) segment spectrum of the warp in
// that slot (chunk c of 16 samples at 32 c), then the window-B twiddles:
// batch b at TW_COL + 64 b, stage j's 2^j (c, t) pairs contiguous at
// tw_col(j) + 2 k, so every stage is read with aligned 16-column loads
template <int WPC>
struct Cols {
  static constexpr int SLOTS = WPC / 4;
  static constexpr int TW_COL = SLOTS * 128;
  static constexpr int USED = TW_COL + 128;
  static constexpr int ALLOC = USED <= 256 ? 256 : 512;
};
__host__ __device__ constexpr int tw_col(int j) {
  return j == 4 ? 0 : j == 3 ? 32 : j == 2 ? 48 : j == 1 ? 56 : 60;
}

__device__ __forceinline__ Tw<float> tw_of(const uint32_t* r, int i) {
  return Tw<float>{__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])};
}

// Window B of the inverse for batch B (5 stages; twiddles from TMEM at `tt`,
// this batch's 64 columns).  `mid` runs while the stage-4 twiddle loads are
// in flight.
template <int B, class MID>
__device__ __forceinline__ void inv_window_b(Cpx<float>* z, uint32_t tt,
                                             MID&& mid) {
  // (tcgen05.ld latency is ~12 cycles: loads are issued right before use)
  uint32_t r[32];
  tm_ld16(tt + tw_col(2), r);       // stages 0, 1, 2
  tm_ld16(tt + tw_col(3), r + 16);  // stage 3
  mid();
  tm_wait32(r);
  stage_rt<0, B, true>(z, [&](auto kc) { return tw_of(r + 12, decltype(kc)::value); });
  stage_rt<1, B, true>(z, [&](auto kc) { return tw_of(r + 8, decltype(kc)::value); });
  stage_rt<2, B, true>(z, [&](auto kc) { return tw_of(r, decltype(kc)::value); });
  stage_rt<3, B, true>(z, [&](auto kc) { return tw_of(r + 16, decltype(kc)::value); });
  tm_ld16(tt + tw_col(4), r);
  tm_ld16(tt + tw_col(4) + 16, r + 16);
  tm_wait32(r);
  stage_rt<4, B, true>(z, [&](auto kc) { return tw_of(r, decltype(kc)::value); });
}
template <int B>
__device__ __forceinline__ void fwd_window_b(Cpx<float>* z, uint32_t tt) {
  uint32_t r[32];
  tm_ld16(tt + tw_col(4), r);
  tm_ld16(tt + tw_col(4) + 16, r + 16);
  tm_wait32(r);
  stage_rt<4, B, false>(z, [&](auto kc) { return tw_of(r, decltype(kc)::value); });
  tm_ld16(tt + tw_col(2), r);
  tm_ld16(tt + tw_col(3), r + 16);
  tm_wait32(r);
  stage_rt<3, B, false>(z, [&](auto kc) { return tw_of(r + 16, decltype(kc)::value); });
  stage_rt<2, B, false>(z, [&](auto kc) { return tw_of(r, decltype(kc)::value); });
  stage_rt<1, B, false>(z, [&](auto kc) { return tw_of(r + 8, decltype(kc)::value); });
  stage_rt<0, B, false>(z, [&](auto kc) { return tw_of(r + 12, decltype(kc)::value); });
}

// Exchange layout: in-place p = 64 hi + 32 b + lo -> hi * STRIDE + 2 lo + b:
// both windows move 16-byte pairs (p, p + 32) (the only index bit both hold
// in registers), conflict-free (window A: lane rows 528 bytes apart; window
// B: lanes consecutive)
__device__ __forceinline__ void store_a(Cpx<float>* buf, int lane,
                                        const Cpx<float>* y) {
  float4* b = reinterpret_cast<float4*>(buf + lane * STRIDE);
  sfor<0, 32>([&](auto ec) {
    constexpr int e = decltype(ec)::value;
    b[e] = make_float4(y[e].re, y[e].im, y[e + 32].re, y[e + 32].im);
  });
}
__device__ __forceinline__ void load_a(const Cpx<float>* buf, int lane,
                                       Cpx<float>* y) {
  const float4* b = reinterpret_cast<const float4*>(buf + lane * STRIDE);
  sfor<0, 32>([&](auto ec) {
    constexpr int e = decltype(ec)::value;
    const float4 v = b[e];
    y[e] = Cpx<float>{v.x, v.y};
    y[e + 32] = Cpx<float>{v.z, v.w};
  });
}
__device__ __forceinline__ void store_b(Cpx<float>* buf, int lane,
                                        const Cpx<float>* z) {
  sfor<0, 32>([&](auto hc) {
    constexpr int h = decltype(hc)::value;
    *reinterpret_cast<float4*>(buf + h * STRIDE + 2 * lane) =
        make_float4(z[h].re, z[h].im, z[h + 32].re, z[h + 32].im);
  });
}
__device__ __forceinline__ void load_b(const Cpx<float>* buf, int lane,
                                       Cpx<float>* z) {
  sfor<0, 32>([&](auto hc) {
    constexpr int h = decltype(hc)::value;
    const float4 v = *reinterpret_cast<const float4*>(buf + h * STRIDE + 2 * lane);
    z[h] = Cpx<float>{v.x, v.y};
    z[h + 32] = Cpx<float>{v.z, v.w};
  });
}

// ---------------------------------------------------------------------------
// The kernel.  Per item (segment, filter range): gather + dif_fwd, spectrum
// to TMEM; per filter: window A (multiply + 6 static stages), exchange,
// window B per batch, valid outputs staged in natural order in the warp's
// exchange buffer (free after the exchange) and written by ONE TMA bulk copy
// (a segment's outputs of one filter are a contiguous row span): no
// per-lane store queue whose source registers stay locked while it drains
// at HBM speed.
// ---------------------------------------------------------------------------
template <int WPC, int MINB, int MODE>
__global__ void __launch_bounds__(WPC * 32, MINB)
    fused_w64_kernel(const FusedArgs<float> a) {
  using C = Cols<WPC>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  Cpx<float>* buf = reinterpret_cast<Cpx<float>*>(smem_raw) + size_t(w) * BUF;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem_raw + size_t(WPC) * BUF * 8);

  if (w == 0) tmem_alloc<C::ALLOC>(tslot);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t tlane = tbase + (uint32_t((w & 3) * 32) << 16);
  const uint32_t tx = tlane + uint32_t((w >> 2) * 128);  // segment spectrum
  const uint32_t tt = tlane + uint32_t(C::TW_COL);        // twiddles

  // window-B twiddles of this lane (the first warp of each quadrant): entry
  // (j, k) of batch b for low bits l = 32 b + lane, window lo = 6 (fp64 math,
  // rounded once, as twiddle_entry for the E = 16 windows)
  if (w < 4) {
#pragma unroll 1
    for (int b = 0; b < 2; ++b) {
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        uint32_t r[32];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          // pair column 32 half + 2 i -> stage j, k (tw_col)
          const int col = 32 * half + 2 * i;
          const int j = col < 32 ? 4 : col < 48 ? 3 : col < 56 ? 2 : col < 60 ? 1 : col < 62 ? 0 : -1;
          const int idx = j < 0 ? -1 : (1 << j) - 1 + (col - tw_col(j)) / 2;
          double c = 0.0, t = 0.0;
          if (idx >= 0) twiddle_entry(6, idx, 32 * b + lane, idx > 0, &c, &t);
          r[2 * i] = __float_as_uint(float(c));
          r[2 * i + 1] = __float_as_uint(float(t));
        }
        tmem_st32(tt + uint32_t(64 * b + 32 * half), r);
      }
    }
    tmem_wait_st();
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();

  // ---- items: (segment, filter range); warp-granular, balanced tail
  const long long nseg = a.k_hi - a.k_lo;
  const long long nw = (long long)gridDim.x * WPC;
  const long long gw = (long long)blockIdx.x * WPC + w;
  const int ntch = (a.n_fil + a.tchunk - 1) / a.tchunk;
  const long long nitems = a.full_items + (nseg - a.full_items) * ntch;
  auto item = [&](long long it, long long& s, int& f_lo, int& f_hi) {
    if (it < a.full_items) {
      s = it;
      f_lo = 0;
      f_hi = a.n_fil;
    } else {
      const long long r = it - a.full_items;
      s = a.full_items + r / ntch;
      f_lo = int(r % ntch) * a.tchunk;
      f_hi = min(a.n_fil, f_lo + a.tchunk);
    }
    s += a.k_lo;
  };

  // filter spectra (engine layout, spec_vec): chunk c of this lane (samples
  // 64 lane + 16 c + [0, 16)) is E = 16 thread t = 4 lane + c, vectors
  // v = 0..7 at f * 1024 + 128 v + t
  float4 h0[8], h1[8];
  auto fetch = [&](float4* h, int f, int c) {
    const int base = a.hoff + f * 1024 + 4 * lane + c;
#pragma unroll
    for (int v = 0; v < 8; ++v) h[v] = tex1Dfetch<float4>(a.htex, base + v * 128);
  };
  const float inv_n = 1.0f / float(N);
  constexpr int ESZ = MODE == FMODE_C2C ? 8 : 4, EPV = 16 / ESZ;
  char* const gbase = MODE == FMODE_C2C ? reinterpret_cast<char*>(a.out)
                                        : reinterpret_cast<char*>(a.outr);

  for (long long it = gw; it < nitems; it += nw) {
    long long s;
    int f_lo, f_hi;
    item(it, s, f_lo, f_hi);
    const long long g0 = s * a.seg_len;
    // L2 prefetch of the next item's input window (one lane)
    if (lane == 0 && it + nw < nitems) {
      long long sn;
      int fl_, fh_;
      item(it + nw, sn, fl_, fh_);
      long long lo = sn * a.seg_len - a.t0 + a.origin, hi = lo + N;
      lo = lo > 0 ? lo : 0;
      hi = hi < a.n_s ? hi : a.n_s;
      if (hi > lo) {
        const char* base = reinterpret_cast<const char*>(a.x);
        uintptr_t b0 = reinterpret_cast<uintptr_t>(base + (lo - a.x_base) * 8);
        uintptr_t b1 = reinterpret_cast<uintptr_t>(base + (hi - a.x_base) * 8);
        b0 = (b0 + 15) & ~uintptr_t(15);
        b1 &= ~uintptr_t(15);
        if (b1 > b0) l2_prefetch(reinterpret_cast<const void*>(b0), uint32_t(b1 - b0));
      }
    }
    // owned outputs o in [o_lo, o_hi) of this segment (output o is in-place
    // sample t0 + o)
    const long long o_lo = a.g_lo > g0 ? a.g_lo - g0 : 0;
    const long long o_hi = a.g_hi - g0 < a.seg_len ? a.g_hi - g0 : a.seg_len;
    const bool any = !(a.dbg & 1) && o_hi > o_lo;

    // ---- gather (window B layout: sample (b, h) of this lane is in-place
    // p = 64 h + 32 b + lane; _gather, _kernels_nb.py:206-215) and the
    // forward transform (dif_fwd, :11-28)
    {
      Cpx<float> z[E];
      const long long w0 = g0 - a.t0 + a.origin + lane;
      const Cpx<float>* xp = a.x + (w0 - a.x_base);
      sfor<0, 64>([&](auto rc) {
        constexpr int r = decltype(rc)::value;
        constexpr int off = 64 * (r & 31) + 32 * (r >> 5);
        z[r] = ld_nc_or0(xp + off, (unsigned long long)(w0 + off) <
                                       (unsigned long long)a.n_s);
      });
      fwd_window_b<0>(z, tt);
      fwd_window_b<1>(z + 32, tt + 64);
      if (lane == 0) bulk_wait_read();  // the buffer's last bulk store
      __syncwarp();
      store_b(buf, lane, z);
      __syncwarp();
      load_a(buf, lane, z);
      dif_stage_static<5, 64>(z);
      dif_stage_static<4, 32>(z);
      dif_stage_static<4, 32>(z + 32);
      const float sc = a.pp_kind == OLSB_PP_SCALE ? inv_n * a.pp_c : inv_n;
      sfor<0, 4>([&](auto cc) {
        constexpr int c = decltype(cc)::value;
        dif_pass_static<float, 4, 4>(z + 16 * c);
#pragma unroll
        for (int e = 0; e < 16; ++e) z[16 * c + e] = cscale(z[16 * c + e], sc);
        tmem_st_cpx(tx + 32 * c, z + 16 * c);
      });
      tmem_wait_st();
    }
    fetch(h0, f_lo, 0);
    fetch(h1, f_lo, 1);

    for (int f = f_lo; f < f_hi; ++f) {
      const bool more = f + 1 < f_hi;
      // ---- window A: multiply (both operands bit-reversed,
      // _kernels_nb.py:280-282) + stages 0..5 of dit_inv (:31-51).  Spectrum
      // chunks 0 / 1 were fetched during the previous filter, chunk c + 2 is
      // fetched once chunk c is consumed.
      Cpx<float> y[E];
      sfor<0, 4>([&](auto cc) {
        constexpr int c = decltype(cc)::value;
        float4* hb = (c & 1) ? h1 : h0;
        uint32_t xr[32];
        tm_ld16(tx + 32 * c, xr);
        tm_ld16(tx + 32 * c + 16, xr + 16);
        tm_wait32(xr);
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const Cpx<float> x0{__uint_as_float(xr[4 * v]), __uint_as_float(xr[4 * v + 1])};
          const Cpx<float> x1{__uint_as_float(xr[4 * v + 2]), __uint_as_float(xr[4 * v + 3])};
          y[16 * c + 2 * v] = cmul(x0, Cpx<float>{hb[v].x, hb[v].y});
          y[16 * c + 2 * v + 1] = cmul(x1, Cpx<float>{hb[v].z, hb[v].w});
        }
        if constexpr (c < 2) fetch(hb, f, c + 2);
        dit_pass_static<float, 4, 4>(y + 16 * c);
      });
      dit_stage_static<4, 32>(y);
      dit_stage_static<4, 32>(y + 32);
      dit_stage_static<5, 64>(y);
      // ---- the exchange (warp-local)
      if (lane == 0) bulk_wait_read();  // the previous filter's bulk store
      __syncwarp();
      if (!(OLSB_W64_ABL & 2)) store_a(buf, lane, y);  // ablation: no exchange
      __syncwarp();
      // ---- window B, batch by batch; outputs staged at natural position
      // p + delta, delta chosen so staged and global element addresses agree
      // modulo 16 bytes (_store, _kernels_nb.py:218-222)
      const long long rowbase = (long long)f * a.out_ld + (g0 - a.out_base);
      const int galign =
          int((reinterpret_cast<uintptr_t>(gbase + rowbase * ESZ) / ESZ) % EPV);
      const int delta = ((galign - a.t0) % EPV + EPV) % EPV;
      auto stage_out = [&](auto bc, const Cpx<float>* z) {
        constexpr int b = decltype(bc)::value;
        if (OLSB_W64_ABL & 4) return;  // ablation: no staging
        if constexpr (MODE == FMODE_C2C) {
          Cpx<float>* stg = buf + delta + 32 * b + lane;
          sfor<0, 32>([&](auto hc) {
            constexpr int h = decltype(hc)::value;
            *reinterpret_cast<float2*>(stg + 64 * h) = make_float2(z[h].re, z[h].im);
          });
        } else {
          float* stg = reinterpret_cast<float*>(buf) + delta + 32 * b + lane;
          sfor<0, 32>([&](auto hc) {
            constexpr int h = decltype(hc)::value;
            stg[64 * h] = fmaf(z[h].re, z[h].re, z[h].im * z[h].im);
          });
        }
      };
      Cpx<float>* y0 = y;
      Cpx<float>* y1 = y + 32;
      if (!(OLSB_W64_ABL & 2)) load_b(buf, lane, y);
      inv_window_b<0>(y0, tt, [&] { if (more) fetch(h0, f + 1, 0); });
      __syncwarp();  // every lane's exchange reads precede the staging
      stage_out(IC<0>{}, y0);
      inv_window_b<1>(y1, tt + 64, [&] { if (more) fetch(h1, f + 1, 1); });
      stage_out(IC<1>{}, y1);
      fence_proxy_async_smem();
      __syncwarp();
      if (any) {
        // element o of the row segment: staged at t0 + o + delta, global
        // rowbase + o; [q_lo, q_hi) is its 16-byte aligned part
        const long long q_lo = o_lo + ((EPV - (galign + o_lo) % EPV) % EPV);
        const long long q_hi = o_hi - ((galign + o_hi) % EPV);
        const char* sb = reinterpret_cast<const char*>(buf);
        if (lane == 0 && q_hi > q_lo)
          bulk_store(gbase + (rowbase + q_lo) * ESZ,
                     sb + (a.t0 + q_lo + delta) * ESZ, uint32_t((q_hi - q_lo) * ESZ));
        // the unaligned ends (< EPV samples each) by plain stores
        const bool split = q_hi > q_lo;
        const long long e = lane < 4 ? o_lo + lane : (split ? q_hi : o_lo + 4) + (lane - 4);
        const long long e_end = lane < 4 ? (split ? q_lo : o_hi) : o_hi;
        if (lane < 8 && e < e_end) {
          const char* src = sb + (a.t0 + e + delta) * ESZ;
          char* dst = gbase + (rowbase + e) * ESZ;
          if constexpr (ESZ == 8)
            *reinterpret_cast<float2*>(dst) = *reinterpret_cast<const float2*>(src);
          else
            *reinterpret_cast<float*>(dst) = *reinterpret_cast<const float*>(src);
        }
      }
    }
  }
  if (lane == 0) bulk_wait_read();
  tmem_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<C::ALLOC>(tbase);
}

}  // namespace w64
}  // namespace olsb
