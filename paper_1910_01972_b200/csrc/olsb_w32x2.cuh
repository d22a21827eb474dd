// olsb_w32x2.cuh — fused OLS kernel for N = 2048 (fp32): two warps per
// segment, 32 samples per lane, 16 warps per SM.
//
// Index bits of the in-place position p (the reference's radix-2 stages,
// _kernels_nb.py:11-51) are split as
//   window A = bits 0..4   lane l of warp ws holds row r = l + 32 ws,
//                          p = 32 r + e, e < 32: five stages with
//                          compile-time twiddles
//   window B = bits 5..9   lane l of warp ws holds p = 1024 ws + 32 h + l,
//                          h < 32: five stages, twiddles per lane (TMEM)
//   stage  C = bit 10      pairs (p, p + 1024) sit in the segment's two
//                          warps: a HALF exchange (each warp sends 16 of its
//                          32 samples) gives warp 0 the pairs of h < 16 and
//                          warp 1 those of h >= 16
// so an inverse (and the forward) transform moves 16 KB + 8 KB through
// shared memory instead of 2 x 16 KB, the A <-> B exchange is warp-local,
// and only the half exchange couples the two warps (a 64-thread named
// barrier).  Registers: 32 complex of data per lane, 12 warps per SM (one
// 384-thread CTA, six segments; 3 warps per scheduler), where the 64-sample
// warp-per-segment engine (olsb_w64.cuh) ran at 2.
#pragma once

#include "olsb_w64.cuh"

namespace olsb {
namespace w32x2 {

using namespace w64;

constexpr int LOGN = 11, N = 2048, E = 32;
constexpr int RSTRIDE = 33;          // padded 32-sample row (complex units)
constexpr int SBUF = 64 * RSTRIDE;   // per-segment buffer (complex), >= N + 2

// TMEM columns per lane (quadrant q holds warp-in-segment ws = q >> 1; the
// three warps of a quadrant are in different segments):
//   [64 s, 64 s + 64)    segment spectrum of the quadrant's warp s = 0, 1, 2
//   [192, 256)           window-B twiddles (per lane, shared by the quadrant):
//                        stage j's 2^j (c, t) pairs at 192 + twc_b(j) + 2 k
//   [256, 288)           stage-C twiddles of this ws's 16 h values
__host__ __device__ constexpr int twc_b(int j) {
  return j == 4 ? 0 : j == 3 ? 32 : j == 2 ? 48 : j == 1 ? 56 : 60;
}

// window-B stage J (32 registers, 16 butterflies (h, h + 2^J)); forms: J < 2
// STD (their GOOD / ROT choice would depend on lane bits), else rot_static
template <int J, bool INV, int BLO = 0, int BHI = 16, class TWF>
__device__ __forceinline__ void stage_b(Cpx<float>* z, const TWF& tw) {
  sfor<BLO, BHI>([&](auto bc) {
    constexpr int b = decltype(bc)::value;
    constexpr int a = ((b >> J) << (J + 1)) | (b & ((1 << J) - 1));
    constexpr int k = a & ((1 << J) - 1);
    const Tw<float> w = tw(IC<k>{});
    Cpx<float>& u = z[a];
    Cpx<float>& v = z[a | (1 << J)];
    if constexpr (J < 2) {
      if constexpr (INV) dit_std(u, v, w.c, w.t); else dif_std(u, v, w.c, w.t);
    } else if constexpr (rot_static(J, k)) {
      if constexpr (INV) dit_rot(u, v, w.c, w.t); else dif_rot(u, v, w.c, w.t);
    } else {
      if constexpr (INV) dit_good(u, v, w.c, w.t); else dif_good(u, v, w.c, w.t);
    }
  });
}

template <bool INV>
__device__ __forceinline__ void window_b(Cpx<float>* z, uint32_t tt) {
  uint32_t r[32];
  auto tw = [&](int off) {
    return [&, off](auto kc) { return tw_of(r + off, decltype(kc)::value); };
  };
  auto low = [&] {  // stages 0, 1, 2 (cols 48..63) and 3 (32..47)
    tm_ld16(tt + twc_b(2), r);
    tm_ld16(tt + twc_b(3), r + 16);
    tm_wait32(r);
  };
  auto s4 = [&] {
    tm_ld16(tt + twc_b(4), r);
    tm_ld16(tt + twc_b(4) + 16, r + 16);
    tm_wait32(r);
    stage_b<4, INV>(z, tw(0));
  };
  if constexpr (INV) {
    low();
    stage_b<0, INV>(z, tw(12));
    stage_b<1, INV>(z, tw(8));
    stage_b<2, INV>(z, tw(0));
    stage_b<3, INV>(z, tw(16));
    s4();
  } else {
    s4();
    low();
    stage_b<3, INV>(z, tw(16));
    stage_b<2, INV>(z, tw(0));
    stage_b<1, INV>(z, tw(8));
    stage_b<0, INV>(z, tw(12));
  }
}

// stage C (bit 10) on 16 pairs (u[i], v[i]) = (p, p + 1024), p = 32 (h0 + i)
// + lane; twiddle of h = h0 + i from TMEM (forms rot_static(5, h))
template <bool INV, int H0>
__device__ __forceinline__ void stage_c(Cpx<float>* u, Cpx<float>* v, uint32_t tc) {
  uint32_t r[32];
  tm_ld16(tc, r);
  tm_ld16(tc + 16, r + 16);
  tm_wait32(r);
  sfor<0, 16>([&](auto ic) {
    constexpr int i = decltype(ic)::value;
    constexpr int h = H0 + i;
    const Tw<float> w = tw_of(r, i);
    if constexpr (rot_static(5, h)) {
      if constexpr (INV) dit_rot(u[i], v[i], w.c, w.t); else dif_rot(u[i], v[i], w.c, w.t);
    } else {
      if constexpr (INV) dit_good(u[i], v[i], w.c, w.t); else dif_good(u[i], v[i], w.c, w.t);
    }
  });
}

__device__ __forceinline__ void seg_sync(int sid) {
  asm volatile("bar.sync %0, 64;" ::"r"(1 + sid) : "memory");
}

constexpr int WARPS = 12, SEGS = 6;

template <int MODE>
__global__ void __launch_bounds__(WARPS * 32, 1) fused_w32x2_kernel(const FusedArgs<float> a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;     // 12 warps
  const int q = w & 3;                         // TMEM lane quadrant
  const int ws = q >> 1;                       // warp in segment
  const int slot = w >> 2;                     // this warp's slot in the quadrant
  const int sid = (q & 1) + 2 * slot;          // segment slot 0..5
  Cpx<float>* buf = reinterpret_cast<Cpx<float>*>(smem_raw) + size_t(sid) * SBUF;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem_raw + size_t(SEGS) * SBUF * 8);

  if (w == 0) tmem_alloc<512>(tslot);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t tl = tbase + (uint32_t(q * 32) << 16);
  const uint32_t tx = tl + uint32_t(64 * slot);  // segment spectrum
  const uint32_t tt = tl + 192u;                 // window-B twiddles
  const uint32_t tc = tl + 256u;                 // stage-C twiddles

  // twiddles (fp64 math, rounded once): window B of lo = 5 for low bits l =
  // lane (entries (j, k) at twc_b(j) + 2k), stage C (window lo = 5, j = 5,
  // k = h) for this ws's h = 16 ws + i; written by the first warp of each
  // quadrant
  if (slot == 0) {
#pragma unroll 1
    for (int part = 0; part < 3; ++part) {
      uint32_t r[32];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        int idx = -1;
        if (part < 2) {
          const int col = 32 * part + 2 * i;
          const int j = col < 32 ? 4 : col < 48 ? 3 : col < 56 ? 2 : col < 60 ? 1
                      : col < 62 ? 0 : -1;
          idx = j < 0 ? -1 : (1 << j) - 1 + (col - twc_b(j)) / 2;
        } else {
          idx = 31 + 16 * ws + i;
        }
        double c = 0.0, t = 0.0;
        if (idx >= 0) twiddle_entry(5, idx, lane, false, &c, &t);
        r[2 * i] = __float_as_uint(float(c));
        r[2 * i + 1] = __float_as_uint(float(t));
      }
      tmem_st32(tl + 192u + uint32_t(32 * part), r);
    }
    tmem_wait_st();
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();

  // ---- items: (segment, filter range) per segment slot, balanced tail
  const long long nseg = a.k_hi - a.k_lo;
  const long long ng = (long long)gridDim.x * SEGS;
  const long long gg = (long long)blockIdx.x * SEGS + sid;
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

  // filter spectra (engine layout, spec_vec, N = 2048): half c of row
  // r = lane + 32 ws (samples 32 r + 16 c + [0, 16)) is E = 16 thread
  // t = 2 r + c, vectors v at f * 1024 + 128 v + t
  const int row = lane + 32 * ws;
  float4 h0[8], h1[8];
  auto fetch = [&](float4* h, int f, int c) {
    const int base = a.hoff + f * 1024 + 2 * row + c;
#pragma unroll
    for (int v = 0; v < 8; ++v) h[v] = tex1Dfetch<float4>(a.htex, base + v * 128);
  };
  const float inv_n = 1.0f / float(N);
  // exchange layout (window A <-> B, within a warp): warp ws uses buffer rows
  // 32 ws .. 32 ws + 31, row r = p >> 5 at r * RSTRIDE, column p & 31
  Cpx<float>* wbuf = buf + 32 * ws * RSTRIDE;
  // half exchanges: each warp writes its outgoing 16 samples per lane into
  // rows 0..15 of its OWN region (its exchange reads are done, the partner
  // reads them after the segment barrier)
  const Cpx<float>* pbuf = buf + 32 * (1 - ws) * RSTRIDE;

  // the per-item work, compiled once per warp-in-segment (every exchange
  // role, stage-C half and output position is a compile-time constant)
  auto run = [&](auto wsc) __attribute__((always_inline)) {
    constexpr int WS = decltype(wsc)::value;
    for (long long it = gg; it < nitems; it += ng) {
      long long s;
      int f_lo, f_hi;
      item(it, s, f_lo, f_hi);
      const long long g0 = s * a.seg_len;
      if (WS == 0 && lane == 0 && it + ng < nitems) {  // L2 prefetch, next window
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
      // outputs of this lane after stage C: p = 32 h + lane (+ 1024) for h in
      // [16 ws, 16 ws + 16); output o = p - t0, kept iff o in [o_lo, o_hi)
      const long long o_lo = a.g_lo > g0 ? a.g_lo - g0 : 0;
      const long long o_hi = a.g_hi - g0 < a.seg_len ? a.g_hi - g0 : a.seg_len;
      const unsigned span = ((a.dbg & 1) || o_hi <= o_lo) ? 0u : unsigned(o_hi - o_lo);
      const int o0 = lane - a.t0 - int(o_lo);
      unsigned mlo = 0, mhi = 0;
  #pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int p = 32 * (16 * WS + i);
        mlo |= (unsigned(o0 + p) < span ? 1u : 0u) << i;
        mhi |= (unsigned(o0 + p + 1024) < span ? 1u : 0u) << i;
      }

      // ---- forward transform (dif_fwd, _kernels_nb.py:11-28) of the gathered
      // window (_gather, :206-215): this warp loads the stage-C pairs of its
      // 16 h, runs stage C, and the half exchange hands the other warp its
      // half; then window B, the A <-> B exchange, window A, 1/N, TMEM
      {
        Cpx<float> u[16], v[16];
        const long long w0 = g0 - a.t0 + a.origin + lane;
        const Cpx<float>* xp = a.x + (w0 - a.x_base);
        sfor<0, 16>([&](auto ic) {
          constexpr int i = decltype(ic)::value;
          constexpr int p = 32 * (16 * WS + i);
          u[i] = ld_nc_or0(xp + p, (unsigned long long)(w0 + p) < (unsigned long long)a.n_s);
          v[i] = ld_nc_or0(xp + p + 1024,
                           (unsigned long long)(w0 + p + 1024) < (unsigned long long)a.n_s);
        });
        stage_c<false, 16 * WS>(u, v, tc);
        Cpx<float> z[E];
        // half exchange: ws 0 keeps u (p < 1024) and sends v; ws 1 keeps v
        seg_sync(sid);  // the buffer's previous users are done
        {
          Cpx<float>* hb = wbuf;   // outgoing half: rows 0..15 of my own region
          sfor<0, 16>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            if constexpr (WS) {
              hb[i * RSTRIDE + lane] = u[i];
              z[16 + i] = v[i];
            } else {
              hb[i * RSTRIDE + lane] = v[i];
              z[i] = u[i];
            }
          });
        }
        seg_sync(sid);
        {
          const Cpx<float>* hb = pbuf;   // the partner's outgoing half
          sfor<0, 16>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            if constexpr (WS) z[i] = hb[i * RSTRIDE + lane]; else z[16 + i] = hb[i * RSTRIDE + lane];
          });
        }
        // z[h] = sample 1024 ws + 32 h + lane (window B layout)
        window_b<false>(z, tt);
        seg_sync(sid);  // both warps' half-exchange reads are done
        sfor<0, 32>([&](auto hc) {
          constexpr int h = decltype(hc)::value;
          wbuf[h * RSTRIDE + lane] = z[h];
        });
        __syncwarp();
        {
          const Cpx<float>* rb = wbuf + lane * RSTRIDE;
          sfor<0, 32>([&](auto ec) {
            constexpr int e = decltype(ec)::value;
            z[e] = rb[e];
          });
        }
        // z[e] = sample 32 (lane + 32 ws) + e (window A layout)
        dif_stage_static<4, 32>(z);
        const float sc = a.pp_kind == OLSB_PP_SCALE ? inv_n * a.pp_c : inv_n;
        sfor<0, 2>([&](auto cc) {
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
        // _kernels_nb.py:280-282) + stages 0..4 of dit_inv (:31-51)
        Cpx<float> y[E];
        sfor<0, 2>([&](auto cc) {
          constexpr int c = decltype(cc)::value;
          float4* hb = c ? h1 : h0;
          uint32_t xr[32];
          tm_ld16(tx + 32 * c, xr);
          tm_ld16(tx + 32 * c + 16, xr + 16);
          tm_wait32(xr);
  #pragma unroll
          for (int vv = 0; vv < 8; ++vv) {
            const Cpx<float> x0{__uint_as_float(xr[4 * vv]), __uint_as_float(xr[4 * vv + 1])};
            const Cpx<float> x1{__uint_as_float(xr[4 * vv + 2]), __uint_as_float(xr[4 * vv + 3])};
            y[16 * c + 2 * vv] = cmul(x0, Cpx<float>{hb[vv].x, hb[vv].y});
            y[16 * c + 2 * vv + 1] = cmul(x1, Cpx<float>{hb[vv].z, hb[vv].w});
          }

          dit_pass_static<float, 4, 4>(y + 16 * c);
        });
        dit_stage_static<4, 32>(y);
        // ---- A -> B exchange (within the warp)
        seg_sync(sid);  // the partner's half-exchange reads of the previous filter
        {
          Cpx<float>* rb = wbuf + lane * RSTRIDE;
          sfor<0, 32>([&](auto ec) {
            constexpr int e = decltype(ec)::value;
            rb[e] = y[e];
          });
        }
        __syncwarp();
        sfor<0, 32>([&](auto hc) {
          constexpr int h = decltype(hc)::value;
          y[h] = wbuf[h * RSTRIDE + lane];
        });
        if (more) fetch(h0, f + 1, 0);  // the next filter's half 0
        // ---- window B (bits 5..9)
        window_b<true>(y, tt);
        // ---- half exchange + stage C (bit 10): ws 0 takes the pairs of h < 16
        __syncwarp();  // this warp's exchange reads precede its half writes
        {
          Cpx<float>* hb = wbuf;
          sfor<0, 16>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            hb[i * RSTRIDE + lane] = WS ? y[i] : y[16 + i];
          });
        }
        seg_sync(sid);
        Cpx<float> u[16], v[16];
        {
          const Cpx<float>* hb = pbuf;
          sfor<0, 16>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            const Cpx<float> o = hb[i * RSTRIDE + lane];
            if constexpr (WS) {
              u[i] = o;
              v[i] = y[16 + i];
            } else {
              u[i] = y[i];
              v[i] = o;
            }
          });
        }
        stage_c<true, 16 * WS>(u, v, tc);
        if (more) fetch(h1, f + 1, 1);  // the next filter's half 1
        // ---- valid-sample writeback (_store, :218-222): u at p = 32 h + lane,
        // v at p + 1024, h = 16 ws + i
        if constexpr (MODE == FMODE_C2C) {
          Cpx<float>* orow = a.out + (long long)f * a.out_ld + (g0 - a.out_base) + o0 + o_lo;
          sfor<0, 16>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            constexpr int p = 32 * (16 * WS + i);
            st_cs_mask<(1u << i)>(orow + p, u[i], mlo);
            st_cs_mask<(1u << i)>(orow + p + 1024, v[i], mhi);
          });
        } else {
          float* orow = a.outr + (long long)f * a.out_ld + (g0 - a.out_base) + o0 + o_lo;
          sfor<0, 16>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            constexpr int p = 32 * (16 * WS + i);
            st_cs_mask_r<(1u << i)>(orow + p, fmaf(u[i].re, u[i].re, u[i].im * u[i].im), mlo);
            st_cs_mask_r<(1u << i)>(orow + p + 1024,
                                    fmaf(v[i].re, v[i].re, v[i].im * v[i].im), mhi);
          });
        }
      }
    }
  };
  if (ws) run(IC<1>{}); else run(IC<0>{});
  tmem_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tbase);
}

}  // namespace w32x2
}  // namespace olsb
