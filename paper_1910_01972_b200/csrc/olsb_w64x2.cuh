// olsb_w64x2.cuh — fused OLS kernel for N = 4096 (fp32): two warps per
// segment, 64 samples per lane, ONE exchange per transform.
//
// The N = 2048 warp-per-segment kernel (olsb_w64.cuh) carried over to 12 index
// bits: a segment is a PAIR of warps (ws = 0, 1), each lane holding 64
// samples in registers,
//   window A = index bits 0..5  (lane l of warp ws holds row hi = l + 32 ws,
//              samples p = 64 hi + e, e < 64): six stages, compile-time
//              twiddles (theta = pi m / 32)
//   window B = index bits 6..11 (lane l of warp ws holds p = 64 h + 32 ws + l,
//              h < 64): six stages whose twiddles depend on (ws, lane) only,
//              126 words per lane in tensor memory
// so a transform needs one exchange through shared memory (the E = 16
// engine: two, each coupling the 8 warps of a segment) and it couples only
// the two warps of the segment (a 64-thread named barrier).  Valid outputs
// are staged in natural order in the segment's exchange buffer and written
// by one TMA bulk copy per (segment, filter), as in olsb_w64.cuh.  Stage
// pairings and in-place positions are the reference's (_kernels_nb.py:11-51).
#pragma once

#include "olsb_w64.cuh"

namespace olsb {
namespace w64x2 {

using namespace w64;

constexpr int LOGN = 12, N = 4096, E = 64;
constexpr int STRIDE = 66;          // padded 64-sample row (complex units)
constexpr int SBUF = 64 * STRIDE;   // per-segment exchange buffer (complex)

// TMEM columns per lane: [0, 128) the segment spectrum (chunk c of 16 samples
// at 32 c), [128, 256) the window-B twiddles, stage j's 2^j (c, t) pairs
// contiguous at 128 + tw_col12(j) + 2 k
__host__ __device__ constexpr int tw_col12(int j) {
  return j == 5 ? 0 : j == 4 ? 64 : j == 3 ? 96 : j == 2 ? 112 : j == 1 ? 120 : 124;
}

// Window-B stage J on 64 registers: pairs (h, h + 2^J), k = h mod 2^J,
// butterflies b in [BLO, BHI) (32 per stage).  Forms: J = 0 STD (lane bit 4
// would decide), J = 1 fixed by WS (index bit 5 = the warp-in-segment bit),
// J >= 2 rot_static(J, k).
template <int J, int WS, bool INV, int BLO = 0, int BHI = 32, class TWF>
__device__ __forceinline__ void stage_b(Cpx<float>* z, const TWF& tw) {
  sfor<BLO, BHI>([&](auto bc) {
    constexpr int b = decltype(bc)::value;
    constexpr int a = ((b >> J) << (J + 1)) | (b & ((1 << J) - 1));
    constexpr int k = a & ((1 << J) - 1);
    const Tw<float> w = tw(IC<k>{});
    Cpx<float>& u = z[a];
    Cpx<float>& v = z[a | (1 << J)];
    if constexpr (J == 0) {
      if constexpr (INV) dit_std(u, v, w.c, w.t); else dif_std(u, v, w.c, w.t);
    } else if constexpr (rot_b<J, WS>(k)) {
      if constexpr (INV) dit_rot(u, v, w.c, w.t); else dif_rot(u, v, w.c, w.t);
    } else {
      if constexpr (INV) dit_good(u, v, w.c, w.t); else dif_good(u, v, w.c, w.t);
    }
  });
}

// the six window-B stages, inverse (DIT, j = 0..5) or forward (DIF, 5..0)
template <bool INV, int WS>
__device__ __forceinline__ void window_b(Cpx<float>* z, uint32_t tt) {
  uint32_t r[32];
  auto tw = [&](int off) {
    return [&, off](auto kc) { return tw_of(r + off, decltype(kc)::value); };
  };
  auto low = [&] {  // stages 0, 1, 2 (cols 112..127) and 3 (96..111)
    tm_ld16(tt + tw_col12(2), r);
    tm_ld16(tt + tw_col12(3), r + 16);
    tm_wait32(r);
  };
  auto s4 = [&] {
    tm_ld16(tt + tw_col12(4), r);
    tm_ld16(tt + tw_col12(4) + 16, r + 16);
    tm_wait32(r);
    stage_b<4, WS, INV>(z, tw(0));
  };
  auto s5 = [&] {  // 32 pairs, in two halves of 16 twiddles
    tm_ld16(tt + tw_col12(5), r);
    tm_ld16(tt + tw_col12(5) + 16, r + 16);
    tm_wait32(r);
    stage_b<5, WS, INV, 0, 16>(z, tw(0));
    tm_ld16(tt + tw_col12(5) + 32, r);
    tm_ld16(tt + tw_col12(5) + 48, r + 16);
    tm_wait32(r);
    stage_b<5, WS, INV, 16, 32>(z, [&](auto kc) {
      return tw_of(r, decltype(kc)::value - 16);
    });
  };
  if constexpr (INV) {
    low();
    stage_b<0, WS, INV>(z, tw(12));
    stage_b<1, WS, INV>(z, tw(8));
    stage_b<2, WS, INV>(z, tw(0));
    stage_b<3, WS, INV>(z, tw(16));
    s4();
    s5();
  } else {
    s5();
    s4();
    low();
    stage_b<3, WS, INV>(z, tw(16));
    stage_b<2, WS, INV>(z, tw(0));
    stage_b<1, WS, INV>(z, tw(8));
    stage_b<0, WS, INV>(z, tw(12));
  }
}

__device__ __forceinline__ void seg_sync(int sl) {
  asm volatile("bar.sync %0, 64;" ::"r"(1 + sl) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(128, 2) fused_w64x2_kernel(const FusedArgs<float> a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  const int ws = w & 1, sl = w >> 1;  // warp in segment, segment slot
  Cpx<float>* buf = reinterpret_cast<Cpx<float>*>(smem_raw) + size_t(sl) * SBUF;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem_raw + size_t(2) * SBUF * 8);
  const bool issuer = ws == 0 && lane == 0;

  if (w == 0) tmem_alloc<256>(tslot);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t tx = tbase + (uint32_t(w * 32) << 16);  // segment spectrum
  const uint32_t tt = tx + 128u;                        // twiddles

  // window-B twiddles of this (ws, lane): entry (j, k) for low bits
  // l = 32 ws + lane of window lo = 6 (fp64 math, rounded once)
#pragma unroll 1
  for (int q = 0; q < 4; ++q) {
    uint32_t r[32];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int col = 32 * q + 2 * i;
      const int j = col < 64 ? 5 : col < 96 ? 4 : col < 112 ? 3 : col < 120 ? 2
                  : col < 124 ? 1 : col < 126 ? 0 : -1;
      const int idx = j < 0 ? -1 : (1 << j) - 1 + (col - tw_col12(j)) / 2;
      double c = 0.0, t = 0.0;
      if (idx >= 0) twiddle_entry(6, idx, 32 * ws + lane, idx > 0, &c, &t);
      r[2 * i] = __float_as_uint(float(c));
      r[2 * i + 1] = __float_as_uint(float(t));
    }
    tmem_st32(tt + uint32_t(32 * q), r);
  }
  tmem_wait_st();
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();

  // ---- items: (segment, filter range) per segment slot, balanced tail
  const long long nseg = a.k_hi - a.k_lo;
  const long long ng = (long long)gridDim.x * 2;
  const long long gg = (long long)blockIdx.x * 2 + sl;
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

  // filter spectra (engine layout, spec_vec, N = 4096): chunk c of row
  // hi = lane + 32 ws is E = 16 thread t = 4 hi + c, vectors v at
  // f * 2048 + 256 v + t
  float4 h0[8], h1[8];
  const int row = lane + 32 * ws;
  auto fetch = [&](float4* h, int f, int c) {
    const int base = a.hoff + f * 2048 + 4 * row + c;
#pragma unroll
    for (int v = 0; v < 8; ++v) h[v] = tex1Dfetch<float4>(a.htex, base + v * 256);
  };
  const float inv_n = 1.0f / float(N);
  constexpr int ESZ = MODE == FMODE_C2C ? 8 : 4, EPV = 16 / ESZ;
  char* const gbase = MODE == FMODE_C2C ? reinterpret_cast<char*>(a.out)
                                        : reinterpret_cast<char*>(a.outr);

  for (long long it = gg; it < nitems; it += ng) {
    long long s;
    int f_lo, f_hi;
    item(it, s, f_lo, f_hi);
    const long long g0 = s * a.seg_len;
    if (issuer && it + ng < nitems) {  // L2 prefetch of the next window
      long long sn;
      int fl_, fh_;
      item(it + ng, sn, fl_, fh_);
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
    const long long o_lo = a.g_lo > g0 ? a.g_lo - g0 : 0;
    const long long o_hi = a.g_hi - g0 < a.seg_len ? a.g_hi - g0 : a.seg_len;
    const bool any = !(a.dbg & 1) && o_hi > o_lo;

    // ---- gather (window B layout, _gather _kernels_nb.py:206-215) and the
    // forward transform (dif_fwd, :11-28)
    {
      Cpx<float> z[E];
      const long long w0 = g0 - a.t0 + a.origin + 32 * ws + lane;
      const Cpx<float>* xp = a.x + (w0 - a.x_base);
      sfor<0, 64>([&](auto hc) {
        constexpr int h = decltype(hc)::value;
        z[h] = ld_nc_or0(xp + 64 * h, (unsigned long long)(w0 + 64 * h) <
                                          (unsigned long long)a.n_s);
      });
      if (ws) window_b<false, 1>(z, tt); else window_b<false, 0>(z, tt);
      if (issuer) bulk_wait_read();  // the buffer's last bulk store
      seg_sync(sl);
      sfor<0, 64>([&](auto hc) {
        constexpr int h = decltype(hc)::value;
        *reinterpret_cast<float2*>(buf + h * STRIDE + 32 * ws + lane) =
            make_float2(z[h].re, z[h].im);
      });
      seg_sync(sl);
      {
        const float4* b = reinterpret_cast<const float4*>(buf + row * STRIDE);
        sfor<0, 32>([&](auto ec) {
          constexpr int e = decltype(ec)::value;
          const float4 v = b[e];
          z[2 * e] = Cpx<float>{v.x, v.y};
          z[2 * e + 1] = Cpx<float>{v.z, v.w};
        });
      }
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
      // _kernels_nb.py:280-282) + stages 0..5 of dit_inv (:31-51)
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
        if constexpr (c == 2) {
          if (more) fetch(h0, f + 1, 0);
        }
        if constexpr (c == 3) {
          if (more) fetch(h1, f + 1, 1);
        }
        dit_pass_static<float, 4, 4>(y + 16 * c);
      });
      dit_stage_static<4, 32>(y);
      dit_stage_static<4, 32>(y + 32);
      dit_stage_static<5, 64>(y);
      // ---- the exchange (the segment's two warps)
      if (issuer) bulk_wait_read();  // the previous filter's bulk store
      seg_sync(sl);
      {
        float4* b = reinterpret_cast<float4*>(buf + row * STRIDE);
        sfor<0, 32>([&](auto ec) {
          constexpr int e = decltype(ec)::value;
          b[e] = make_float4(y[2 * e].re, y[2 * e].im, y[2 * e + 1].re,
                             y[2 * e + 1].im);
        });
      }
      seg_sync(sl);
      sfor<0, 64>([&](auto hc) {
        constexpr int h = decltype(hc)::value;
        const float2 v =
            *reinterpret_cast<const float2*>(buf + h * STRIDE + 32 * ws + lane);
        y[h] = Cpx<float>{v.x, v.y};
      });
      // ---- window B, then the valid samples (_store, :218-222) staged at
      // natural position p + delta (staged and global addresses agree
      // modulo 16 bytes) and written by one bulk copy
      if (ws) window_b<true, 1>(y, tt); else window_b<true, 0>(y, tt);
      const long long rowbase = (long long)f * a.out_ld + (g0 - a.out_base);
      const int galign =
          int((reinterpret_cast<uintptr_t>(gbase + rowbase * ESZ) / ESZ) % EPV);
      const int delta = ((galign - a.t0) % EPV + EPV) % EPV;
      seg_sync(sl);  // both warps' exchange reads precede the staging
      if constexpr (MODE == FMODE_C2C) {
        Cpx<float>* stg = buf + delta + 32 * ws + lane;
        sfor<0, 64>([&](auto hc) {
          constexpr int h = decltype(hc)::value;
          *reinterpret_cast<float2*>(stg + 64 * h) = make_float2(y[h].re, y[h].im);
        });
      } else {
        float* stg = reinterpret_cast<float*>(buf) + delta + 32 * ws + lane;
        sfor<0, 64>([&](auto hc) {
          constexpr int h = decltype(hc)::value;
          stg[64 * h] = fmaf(y[h].re, y[h].re, y[h].im * y[h].im);
        });
      }
      fence_proxy_async_smem();
      seg_sync(sl);
      if (any && ws == 0) {
        const long long q_lo = o_lo + ((EPV - (galign + o_lo) % EPV) % EPV);
        const long long q_hi = o_hi - ((galign + o_hi) % EPV);
        const char* sb = reinterpret_cast<const char*>(buf);
        if (lane == 0 && q_hi > q_lo)
          bulk_store(gbase + (rowbase + q_lo) * ESZ,
                     sb + (a.t0 + q_lo + delta) * ESZ, uint32_t((q_hi - q_lo) * ESZ));
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
  if (issuer) bulk_wait_read();
  tmem_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<256>(tbase);
}

}  // namespace w64x2
}  // namespace olsb
