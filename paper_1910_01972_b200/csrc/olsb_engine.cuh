// olsb_engine.cuh — sm_100a kernels of the OLS engine (device code).
//
//   fused_c2c_kernel  the hot path: segment staging -> forward FFT -> per
//                     filter {multiply, inverse FFT, valid-sample writeback}
//                     (reference: _kernels_nb.py:265-285, ols.py:319-360)
//   fwd_rows_kernel   forward transform of rows (filter spectra,
//                     fft_forward_permuted); same passes as the fused kernel
//   inv_rows_kernel   inverse transform of rows (fft_inverse_permuted)
//   perm_to_dev_kernel  reference permuted layout -> engine layout
//
// One thread owns E = 16 samples of a segment; T = N / 16 threads form a
// segment group and SEGS groups a CTA.  Samples move between 4-bit windows
// through padded, bank-conflict-free shared memory (olsb_fft.cuh).  The
// segment spectrum stays in registers for the whole filter loop; the kernel
// shape (groups per CTA, exchange buffers, how filter spectra are staged,
// barrier scope) is a compile-time policy, tuned per N (olsb_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "olsb.h"
#include "olsb_fft.cuh"

namespace olsb {

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

// Engine layout of filter spectra: 16-byte vector u (in-place samples
// 16 t + 2u, +1) of E = 16 thread t at index f * N/2 + spec_vec(t, u) =
// u * T + t: the four threads of a texture quad read 64 contiguous bytes
// (the warp-per-segment kernel of olsb_w64.cuh reads the same layout).
template <class R, int LOGN>
__host__ __device__ constexpr int spec_vec(int t, int u) {
  return u * (Geo<LOGN>::T) + t;
}

// How the fused kernel fetches filter spectra:
enum HMode : int {
  H_LDG = 0,  // read through L1 with __ldg at the multiply (fp64 policy)
  H_TEX = 3,  // texture fetches: the TEX data path runs beside the LSU pipe
              // that carries the shared-memory exchanges (fp32 policies)
  H_TMA = 4,  // a CTA-shared two-slot ring in shared memory, filled by one
              // TMA bulk copy per filter one filter ahead (full / empty
              // mbarriers); no prefetch registers
};

// Kernel configuration.  SEGS segment groups per CTA, NBUF exchange buffers
// per group (2: one barrier per exchange, 1: two), HM spectrum staging, BAR
// barrier scope (0: CTA-wide __syncthreads, 1: named barrier per group),
// MINB target CTAs per SM (register cap).
template <class R_, int LOGN_, int SEGS_, int NBUF_, int HM_, int BAR_,
          int MINB_, int TMX_ = 0, int PREF_ = 0, int ABL_ = 0, int MB_ = 0>
struct KCfg {
  using R = R_;
  static constexpr int LOGN = LOGN_;
  using G = Geo<LOGN>;
  using L = SmemLayout<R, LOGN>;
  static constexpr bool dbl = std::is_same<R, double>::value;
  static constexpr int E = G::E, T = G::T, P = G::P, LOGE = G::LOGE;
  static constexpr int SEGS = SEGS_;
  static constexpr int THREADS = SEGS * T;
  static constexpr int NBUF = NBUF_;
  static constexpr int HM = HM_;
  static constexpr int BAR = (BAR_ && T >= 32 && SEGS > 1) ? 1 : 0;
  static constexpr int MINB = MINB_;
  static constexpr int VPT = E / V16<R>::per;  // 16-B vectors per thread (J)
  // top-window twiddles live in registers (float: 30 registers) and its
  // table is built inside the exchange buffers, which it only occupies until
  // the registers are loaded
  // Tensor-memory residency (fused kernel, fp32, whole warpgroups): every
  // thread parks per-thread state in its own TMEM lane instead of registers
  //   TMX = 1: segment spectrum (32 words) + top-window twiddles (30 words)
  //   TMX = 2: also the twiddles of the window below
  // TMEM is read by tcgen05.ld at ~400 B/clk/SM, off the LSU pipe that
  // carries the shared-memory exchanges (tools/mb_tmem.cu).
  static constexpr int TMX =
      (!dbl && P >= 2 && THREADS % 128 == 0) ? (P >= 3 ? TMX_ : (TMX_ ? 1 : 0))
                                             : 0;
  static constexpr int WG = THREADS / 128;     // warpgroups (TMEM lane sets)
  static constexpr int CPW = 32 * (1 + TMX);   // TMEM columns per warpgroup
  static constexpr int TCOLS = WG * CPW <= 32    ? 32
                               : WG * CPW <= 64  ? 64
                               : WG * CPW <= 128 ? 128
                               : WG * CPW <= 256 ? 256
                                                 : 512;
  // H_TEX only: the next filter's spectrum is fetched into registers while
  // the current one is transformed (hides the L2 latency of the fetch)
  static constexpr bool PREF = PREF_ && HM_ == H_TEX && !dbl;
  // H_TMA: spectrum ring in shared memory (fp32)
  static constexpr bool HT = HM_ == H_TMA && !dbl;
  // ablation switches for bottleneck analysis (results are wrong with any
  // bit set): 1 no output stores, 2 no shared-memory traffic in the inverse
  // exchanges, 4 no inverse exchange barriers, 8 spectra of filters f & 1
  // only (L1-resident: isolates the L2 traffic of the spectrum fetches)
  static constexpr int ABL = ABL_;
  // MB: the "buffer free" side of each exchange is an mbarrier per segment
  // group (every warp arrives after its loads; the next exchange's stores
  // wait on that phase) instead of a blocking barrier before the stores
  static constexpr bool MB = MB_ && NBUF_ == 1 && T > 32 && !(ABL_ & 4);
  static constexpr bool TOPREG = !dbl && P >= 2 && !TMX;
  // the top window's table is built in the exchange buffers (TOPREG / TMX)
  static constexpr bool TOPOUT = TOPREG || TMX;
  static constexpr size_t al(size_t b) { return (b + 127) & ~size_t(127); }
  static constexpr size_t buf_elems = size_t(SEGS) * L::stride;
  static constexpr size_t bufs_bytes =
      P >= 2 ? al(NBUF * buf_elems * sizeof(Cpx<R>)) : 0;
  // ---- row kernels: every twiddle table in shared memory, then buffers
  static constexpr size_t tab_bytes = al(size_t(G::tw_total()) * sizeof(Tw<R>));
  // exact mode: junction-window table (15 broadcast entries) at the end
  static constexpr size_t jt_bytes = al(16 * sizeof(Tw<R>));
  static constexpr size_t jt_off = tab_bytes + bufs_bytes;
  static constexpr size_t smem_bytes = jt_off + jt_bytes;
  // ---- fused kernel: [bufs (+ top table at init) | low tables | TMEM slot]
  static constexpr int lowtab_elems = TOPOUT ? G::tw_offset(P - 1) : G::tw_total();
  static constexpr size_t f_bufs_bytes =
      P >= 2 ? std::max(bufs_bytes,
                        TOPOUT ? al(size_t(G::tw_entries(P - 1)) * sizeof(Tw<R>))
                               : size_t(0))
             : 0;
  static constexpr size_t f_tab_off = f_bufs_bytes;
  static constexpr size_t f_tab_bytes = al(size_t(lowtab_elems) * sizeof(Tw<R>));
  static constexpr size_t f_slot_off = f_tab_off + f_tab_bytes;
  // [TMEM base address slot | MB: one mbarrier per segment group]
  static constexpr size_t f_mbar_off = f_slot_off + 16;
  static constexpr size_t f_jt_off = al(f_mbar_off + (MB ? 8 * SEGS : 0));
  // HT: [two spectrum slots | full[2], empty[2] mbarriers]
  static constexpr size_t h_slot_bytes = al(size_t(VPT) * T * 16);
  static constexpr size_t f_ring_off = al(f_jt_off + jt_bytes);
  static constexpr size_t f_hbar_off = f_ring_off + (HT ? 2 * h_slot_bytes : 0);
  static constexpr size_t f_smem_bytes = f_hbar_off + (HT ? 32 : 0);
};

// configuration of the row kernels (filter spectra, standalone transforms)
template <class R, int LOGN>
using RowCfg = KCfg<R, LOGN,
                    std::max(1, ((!std::is_same<R, double>::value && LOGN == 12)
                                     ? 512 : 256) >> Geo<LOGN>::LOGT),
                    std::is_same<R, double>::value ? 1 : 2, H_LDG, 0, 1>;

// ---------------------------------------------------------------------------
// barriers
// ---------------------------------------------------------------------------
template <class C>
__device__ __forceinline__ void group_sync(int sl) {
  if constexpr (C::T <= 32) {
    // a segment group lives inside one warp (N <= 512): warp-level sync
    // orders its shared-memory exchange; other warps are independent
    __syncwarp();
  } else if constexpr (C::BAR == 1) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + sl), "r"(C::T) : "memory");
  } else {
    __syncthreads();
  }
}

// mbarrier helpers (MB exchanges)
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a),
               "r"(bytes)
               : "memory");
}
// one-dimensional TMA bulk copy global -> shared, completion on `mbar`
__device__ __forceinline__ void tma_load_1d(uint32_t dst, const void* src,
                                            uint32_t bytes, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}
template <class C>
__device__ __forceinline__ uint32_t group_mbar(int sl) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  return uint32_t(__cvta_generic_to_shared(smem_raw + C::f_mbar_off)) + 8u * sl;
}

// ---------------------------------------------------------------------------
// shared-memory window I/O (addresses = per-thread base + immediates)
// ---------------------------------------------------------------------------
template <class C, int Q, int X>
__device__ __forceinline__ void smem_store(Cpx<typename C::R>* __restrict__ seg_buf,
                                           int t, const Cpx<typename C::R>* x) {
  using R = typename C::R;
  using G = typename C::G;
  using L = XLayout<R, C::LOGN, X>;
  constexpr int pb = L::pair_bit(Q);
  Cpx<R>* b = seg_buf + L::pos(G::thread_part(Q, t));
  if constexpr (pb >= 0 && !C::dbl && C::E >= 2) {
    // 128-bit: samples e and e | 2^pb are adjacent in shared memory
    sfor<0, C::E>([&](auto ec) {
      constexpr int e = decltype(ec)::value;
      if constexpr (!((e >> pb) & 1)) {
        constexpr int off = L::pos(G::elem_part(Q, e));
        constexpr int e1 = e | (1 << pb);
        *reinterpret_cast<float4*>(b + off) =
            make_float4(x[e].re, x[e].im, x[e1].re, x[e1].im);
      }
    });
  } else {
    sfor<0, C::E>([&](auto ec) {
      constexpr int e = decltype(ec)::value;
      constexpr int off = L::pos(G::elem_part(Q, e));
      b[off] = x[e];
    });
  }
}

template <class C, int Q, int X>
__device__ __forceinline__ void smem_load(const Cpx<typename C::R>* __restrict__ seg_buf,
                                          int t, Cpx<typename C::R>* x) {
  using R = typename C::R;
  using G = typename C::G;
  using L = XLayout<R, C::LOGN, X>;
  constexpr int pb = L::pair_bit(Q);
  const Cpx<R>* b = seg_buf + L::pos(G::thread_part(Q, t));
  if constexpr (pb >= 0 && !C::dbl && C::E >= 2) {
    sfor<0, C::E>([&](auto ec) {
      constexpr int e = decltype(ec)::value;
      if constexpr (!((e >> pb) & 1)) {
        constexpr int off = L::pos(G::elem_part(Q, e));
        constexpr int e1 = e | (1 << pb);
        const float4 v = *reinterpret_cast<const float4*>(b + off);
        x[e] = Cpx<R>{v.x, v.y};
        x[e1] = Cpx<R>{v.z, v.w};
      }
    });
  } else {
    sfor<0, C::E>([&](auto ec) {
      constexpr int e = decltype(ec)::value;
      constexpr int off = L::pos(G::elem_part(Q, e));
      x[e] = b[off];
    });
  }
}

// twiddle tables for windows 1..P-1 (double-precision math, rounded once).
// Window q's table goes to lowtab + tw_offset(q), except the top window's
// when `toptab` is given.
// Device-wide copy of every runtime-window table of length 2^LOGN, in the
// canonical layout (window q at tw_offset(q)); filled once per device by
// tw_table_kernel, which then raises g_twready.  Static device memory: the
// C ABI never allocates.
template <int LOGN>
struct TwTableSize {
  static constexpr int n = Geo<LOGN>::tw_total() > 0 ? Geo<LOGN>::tw_total() : 1;
};
template <class R, int LOGN>
__device__ Tw<R> g_twtab[TwTableSize<LOGN>::n];
template <class R, int LOGN>
__device__ int g_twready;

template <class R, int LOGN>
__device__ __forceinline__ Tw<R> twiddle_value(int q_lo, int i, bool tan01) {
  int idx, l;
  twiddle_decode(q_lo, i, &idx, &l, std::is_same<R, double>::value);
  double c, t;
  twiddle_entry_r4(q_lo, idx, l, tan01, &c, &t);
  return Tw<R>{R(c), R(t)};
}

template <class R, int LOGN>
__global__ void tw_table_kernel() {
  using G = Geo<LOGN>;
  sfor<1, G::P>([&](auto qc) {
    constexpr int q = decltype(qc)::value;
    for (int i = threadIdx.x; i < G::tw_entries(q); i += blockDim.x)
      g_twtab<R, LOGN>[G::tw_offset(q) + i] =
          twiddle_value<R, LOGN>(G::lo(q), i, G::tan01(q));
  });
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) atomicExch(&g_twready<R, LOGN>, 1);
}

// twiddle tables for windows 1..P-1 (double-precision math, rounded once).
// Window q's table goes to lowtab + tw_offset(q), except the top window's
// when `toptab` is given.  Copied from the device-wide table once it is
// ready, else computed here (same values bit for bit).
// exact mode: entry (idx = 2^j - 1 + k, l) of window lo is the caller's
// fp32 / fp64 table value tw[(l + k 2^lo) * (N >> (lo + j + 1))]
template <class R, int LOGN>
__device__ __forceinline__ Tw<R> ref_entry(const Cpx<R>* xtw, int lo, int idx,
                                           int l) {
  if (idx < 0) return Tw<R>{R(0), R(0)};
  int j = 0;
  while ((2 << j) - 1 <= idx) ++j;
  const int k = idx - ((1 << j) - 1);
  const Cpx<R> w = xtw[(l + (k << lo)) * ((1 << LOGN) >> (lo + j + 1))];
  return Tw<R>{w.re, w.im};
}
// exact mode: junction-window entries jt[2^j - 1 + k] = tw[k * (N >> (j + 1))]
template <class R, int LOGN>
__device__ void build_jt(Tw<R>* jt, const Cpx<R>* xtw) {
  constexpr int G0 = Geo<LOGN>::G0;
  for (int i = threadIdx.x; i < (1 << G0) - 1; i += blockDim.x)
    jt[i] = ref_entry<R, LOGN>(xtw, 0, i, 0);
}

template <class R, int LOGN>
__device__ void build_tables(Tw<R>* lowtab, Tw<R>* toptab,
                             const Cpx<R>* xtw = nullptr) {
  using G = Geo<LOGN>;
  if (xtw) {
    sfor<1, G::P>([&](auto qc) {
      constexpr int q = decltype(qc)::value;
      constexpr int lo = G::lo(q);
      Tw<R>* dst = (q == G::P - 1 && toptab) ? toptab : lowtab + G::tw_offset(q);
      for (int i = threadIdx.x; i < G::tw_entries(q); i += blockDim.x) {
        int idx, l;
        twiddle_decode(lo, i, &idx, &l, std::is_same<R, double>::value);
        dst[i] = ref_entry<R, LOGN>(xtw, lo, idx, l);
      }
    });
    return;
  }
  int ready;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];"
               : "=r"(ready)
               : "l"(&g_twready<R, LOGN>)
               : "memory");
  sfor<1, G::P>([&](auto qc) {
    constexpr int q = decltype(qc)::value;
    constexpr int lo = G::lo(q);
    constexpr int cnt = G::tw_entries(q);
    Tw<R>* dst = (q == G::P - 1 && toptab) ? toptab : lowtab + G::tw_offset(q);
    if (ready) {
      const Tw<R>* src = g_twtab<R, LOGN> + G::tw_offset(q);
      for (int i = threadIdx.x; i < cnt; i += blockDim.x) dst[i] = src[i];
    } else {
      for (int i = threadIdx.x; i < cnt; i += blockDim.x)
        dst[i] = twiddle_value<R, LOGN>(lo, i, G::tan01(q));
    }
  });
}

// ---- predicated read-only loads (zero when !ok): branch-free, so all loads
// of a segment window are in flight together
__device__ __forceinline__ Cpx<float> ld_nc_or0(const Cpx<float>* p, bool ok) {
  float re, im;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n"
      " mov.b32 %0, 0;\n mov.b32 %1, 0;\n"
      " @q ld.global.nc.v2.f32 {%0, %1}, [%2];\n}"
      : "=f"(re), "=f"(im)
      : "l"(p), "r"(int(ok)));
  return Cpx<float>{re, im};
}
__device__ __forceinline__ Cpx<double> ld_nc_or0(const Cpx<double>* p, bool ok) {
  double re, im;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n"
      " mov.b64 %0, 0;\n mov.b64 %1, 0;\n"
      " @q ld.global.nc.v2.f64 {%0, %1}, [%2];\n}"
      : "=d"(re), "=d"(im)
      : "l"(p), "r"(int(ok)));
  return Cpx<double>{re, im};
}
__device__ __forceinline__ float ld_nc_or0(const float* p, bool ok) {
  float v;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n mov.b32 %0, 0;\n"
      " @q ld.global.nc.f32 %0, [%1];\n}"
      : "=f"(v)
      : "l"(p), "r"(int(ok)));
  return v;
}
__device__ __forceinline__ double ld_nc_or0(const double* p, bool ok) {
  double v;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n mov.b64 %0, 0;\n"
      " @q ld.global.nc.f64 %0, [%1];\n}"
      : "=d"(v)
      : "l"(p), "r"(int(ok)));
  return v;
}

// ---- TMA prefetch of a global range into L2 (16-byte aligned / sized)
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes)
               : "memory");
}

// ---- shared-memory address for PTX operands
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// ---- tensor memory (tcgen05) as per-thread storage.  Thread i of warp w
// owns TMEM lane 32 (w % 4) + i; `ta` = allocation base + lane + column.
template <int COLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {
  asm volatile(
      "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
          smem_u32(slot)),
      "n"(COLS)
      : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::
                   : "memory");
}
template <int COLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base),
               "n"(COLS)
               : "memory");
}
__device__ __forceinline__ void tmem_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// 32 consecutive columns of the thread's lane <-> 32 registers
__device__ __forceinline__ void tmem_ld32(uint32_t ta, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,"
      "%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,"
      "%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]),
        "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
        "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(ta));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t ta, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,"
      "%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,"
      "%27,%28,%29,%30,%31,%32};" ::"r"(ta),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
      "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]),
      "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
      "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
      "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]),
      "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// 16 complex<float> (a thread's segment) <-> 32 TMEM columns
__device__ __forceinline__ void tmem_ld_cpx(uint32_t ta, Cpx<float>* v) {
  uint32_t r[32];
  tmem_ld32(ta, r);
#pragma unroll
  for (int i = 0; i < 16; ++i)
    v[i] = Cpx<float>{__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])};
}
__device__ __forceinline__ void tmem_st_cpx(uint32_t ta, const Cpx<float>* v) {
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    r[2 * i] = __float_as_uint(v[i].re);
    r[2 * i + 1] = __float_as_uint(v[i].im);
  }
  tmem_st32(ta, r);
}
// a thread's 15 runtime twiddles of one window (30 columns, 2 spare)
__device__ __forceinline__ void tmem_ld_tw(uint32_t ta, Tw<float>* w) {
  uint32_t r[32];
  tmem_ld32(ta, r);
#pragma unroll
  for (int i = 0; i < 15; ++i)
    w[i] = Tw<float>{__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])};
}
__device__ __forceinline__ void tmem_st_tw(uint32_t ta, const Tw<float>* w) {
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 15; ++i) {
    r[2 * i] = __float_as_uint(w[i].c);
    r[2 * i + 1] = __float_as_uint(w[i].t);
  }
  r[30] = r[31] = 0u;
  tmem_st32(ta, r);
}
// double-precision stubs (TMX is fp32-only; never instantiated for double)
__device__ __forceinline__ void tmem_ld_cpx(uint32_t, Cpx<double>*) {}
__device__ __forceinline__ void tmem_st_cpx(uint32_t, const Cpx<double>*) {}
__device__ __forceinline__ void tmem_ld_tw(uint32_t, Tw<double>*) {}
__device__ __forceinline__ void tmem_st_tw(uint32_t, const Tw<double>*) {}

// predicated streaming store of one complex sample: stores iff o < span
// (unsigned compare folds the o >= 0 test)
__device__ __forceinline__ void st_cs_if(Cpx<float>* p, Cpx<float> v,
                                         unsigned o, unsigned span) {
  asm volatile(
      "{\n .reg .pred q;\n setp.lt.u32 q, %3, %4;\n"
      " @q st.global.cs.v2.f32 [%0], {%1, %2};\n}" ::"l"(p),
      "f"(v.re), "f"(v.im), "r"(o), "r"(span)
      : "memory");
}
// streaming store of one complex sample iff (mask & bit)
template <unsigned BIT>
__device__ __forceinline__ void st_cs_mask(Cpx<float>* p, Cpx<float> v,
                                           unsigned mask) {
  asm volatile(
      "{\n .reg .pred q;\n .reg .b32 m;\n and.b32 m, %3, %4;\n"
      " setp.ne.u32 q, m, 0;\n"
      " @q st.global.cs.v2.f32 [%0], {%1, %2};\n}" ::"l"(p),
      "f"(v.re), "f"(v.im), "r"(mask), "n"(BIT)
      : "memory");
}
template <unsigned BIT>
__device__ __forceinline__ void st_cs_mask(Cpx<double>* p, Cpx<double> v,
                                           unsigned mask) {
  asm volatile(
      "{\n .reg .pred q;\n .reg .b32 m;\n and.b32 m, %3, %4;\n"
      " setp.ne.u32 q, m, 0;\n"
      " @q st.global.cs.v2.f64 [%0], {%1, %2};\n}" ::"l"(p),
      "d"(v.re), "d"(v.im), "r"(mask), "n"(BIT)
      : "memory");
}
__device__ __forceinline__ void st_cs_if(Cpx<double>* p, Cpx<double> v,
                                         unsigned o, unsigned span) {
  asm volatile(
      "{\n .reg .pred q;\n setp.lt.u32 q, %3, %4;\n"
      " @q st.global.cs.v2.f64 [%0], {%1, %2};\n}" ::"l"(p),
      "d"(v.re), "d"(v.im), "r"(o), "r"(span)
      : "memory");
}

// accessors of the thread's 15 runtime twiddles of window q (see
// dit_pass_rt): a shared-memory table read with 128-bit pair loads, or
// registers
template <class R>
struct TwSmem {
  // window table + 2 l (fp32, [slot][l][half]) or + l (fp64, [slot][half][l],
  // see twiddle_decode)
  const Tw<R>* base;
  int lo;
  static constexpr bool split = std::is_same<R, double>::value;
  __device__ __forceinline__ Tw<R> get0() const { return base[0]; }
  __device__ __forceinline__ TwPair<R> get2(int p) const {
    if constexpr (split)
      return TwPair<R>{base[size_t(2 * p) << lo], base[size_t(2 * p + 1) << lo]};
    else
      return *reinterpret_cast<const TwPair<R>*>(base + (size_t(p) << (lo + 1)));
  }
};
template <class R>
struct TwRegs {
  const Tw<R>* r;  // indexed by idx
  __device__ __forceinline__ Tw<R> get0() const { return r[0]; }
  __device__ __forceinline__ TwPair<R> get2(int p) const {
    return TwPair<R>{r[2 * p - 1], r[2 * p]};
  }
};

template <class R, int LOGN, int Q>
__device__ __forceinline__ TwSmem<R> tw_smem(const Tw<R>* tab, int t) {
  using G = Geo<LOGN>;
  return TwSmem<R>{tab + (TwSmem<R>::split ? 1 : 2) * G::low_bits(Q, t), G::lo(Q)};
}
template <int LOGN, int Q>
__device__ __forceinline__ int top_bits(int t) {
  using G = Geo<LOGN>;
  return G::lo(Q) >= 2 ? (G::low_bits(Q, t) >> (G::lo(Q) - 2)) & 3 : 0;
}


// some exchange of the transform is warp-local (Geo::warp_local)
template <class G>
constexpr bool any_warp_local() {
  bool r = false;
  for (int x = 0; x + 1 < G::P; ++x) r = r || G::warp_local(x);
  return r;
}
// exchange: write window QW, barrier, read window QR (ABL: ablation bits)
template <class C, int QW, int QR, int ABL = 0>
__device__ __forceinline__ void exchange(Cpx<typename C::R>* bufs, int& xc,
                                         int sl, int t, Cpx<typename C::R>* x,
                                         IC<ABL> = {}) {
  Cpx<typename C::R>* buf = bufs + (C::NBUF == 2 ? (xc & 1) * C::buf_elems : 0) +
                            size_t(sl) * C::L::stride;
  constexpr int X = QW < QR ? QW : QR;  // exchange between windows X, X+1
  // warp-local exchange (Geo::warp_local): a warp reads back only what it
  // wrote, so the store -> load sync is warp-level.  The sync BEFORE the
  // stores stays group-wide: the buffer's previous user may be a cross-warp
  // exchange whose loads other warps are still issuing.
  constexpr bool WL = C::G::warp_local(X);
  if constexpr (C::MB) {
    // the previous exchange's loads are done in every warp of the group
    if (xc > 0) mbar_wait(group_mbar<C>(sl), uint32_t(xc - 1) & 1u);
  } else if constexpr ((C::NBUF == 1 ||
                        (!WL && any_warp_local<typename C::G>())) &&
                       !(ABL & 4)) {
    // NBUF = 2 skips this barrier because the previous exchange's barrier
    // orders the loads of the one before it; a warp-local previous exchange
    // (only __syncwarp) does not, so cross-warp exchanges then keep it
    group_sync<C>(sl);
  }
  if constexpr (!(ABL & 2)) smem_store<C, QW, X>(buf, t, x);
  if constexpr (!(ABL & 4)) {
    if constexpr (WL) {
      __syncwarp();
    } else {
      group_sync<C>(sl);
    }
  }
  if constexpr (!(ABL & 2)) smem_load<C, QR, X>(buf, t, x);
  if constexpr (C::MB) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(group_mbar<C>(sl));
  }
  ++xc;
}

// full forward transform: x holds window P-1 on entry, window 0 (J) on exit.
// With TOPREG the top window's 15 twiddles come from `twr`; with TMX the
// runtime windows' twiddles are read from TMEM at `tb`.
template <class C, bool TOPREG, bool XR = false>
__device__ __forceinline__ void forward_fft(Cpx<typename C::R>* x,
                                            const Tw<typename C::R>* lowtab,
                                            const Tw<typename C::R>* twr,
                                            Cpx<typename C::R>* bufs, int& xc,
                                            int sl, int t, uint32_t tb = 0,
                                            const Tw<typename C::R>* jt = nullptr) {
  using R = typename C::R;
  using G = typename C::G;
  constexpr int LOGN = C::LOGN;
  sfor<0, G::P>([&](auto qr) {
    constexpr int q = G::P - 1 - decltype(qr)::value;
    if constexpr (q < G::P - 1) exchange<C, q + 1, q>(bufs, xc, sl, t, x);
    auto pass = [&](const auto& tws) {
      if constexpr (XR) {
        pass_ref<R, false>(x, tws);
      } else {
        dif_pass_rt<R, G::tan01(q)>(x, tws, top_bits<LOGN, q>(t));
      }
    };
    if constexpr (q == 0) {
      if constexpr (XR) {
        pass_static_ref<R, C::LOGE, G::G0, false>(x, jt);
      } else {
        dif_pass_static<R, C::LOGE, G::G0>(x);
      }
    } else {
      if constexpr (C::TMX && (q == G::P - 1 || (q == G::P - 2 && C::TMX == 2))) {
        Tw<R> tw[16];
        tmem_ld_tw(tb + (q == G::P - 1 ? 32u : 64u), tw);
        pass(TwRegs<R>{tw});
      } else if constexpr (q == G::P - 1 && TOPREG) {
        pass(TwRegs<R>{twr});
      } else {
        pass(tw_smem<R, LOGN, q>(lowtab + G::tw_offset(q), t));
      }
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
  cudaTextureObject_t htex;           // texture over `spec` (H_TEX)
  int hoff;  // float4 offset of `spec` from the texture base (alignment)
  int n_fil, fchunk, pp_kind;
  // balanced tail: the first full_items items take groups [0, full_items)
  // with every filter (fchunk = n_fil); the remaining groups are split into
  // items of tchunk filters, so the last wave ends within one small item
  // (0 = plain (group, fchunk) items)
  long long full_items;
  int tchunk;
  // segment grid (engine geometry, anchored at global sample 0): segment k
  // reads the zero-extended window x[k*seg_len - t0 + origin, + N) and owns
  // outputs [k*seg_len, (k+1)*seg_len) = in-place samples [t0, t0 + seg_len);
  // this call writes outputs [g_lo, g_hi) of segments [k_lo, k_hi)
  int t0, origin;
  long long seg_len, k_lo, k_hi, g_lo, g_hi;
  R pp_c;
  double pp_cd;  // pp_c as the caller passed it (exact mode's _store)
  Cpx<R>* out;
  long long out_ld, out_base;
  int dbg;  // tuning: bit 0 = predicate off the output stores
  // real-valued modes (FMODE_R2R: real signal and output; FMODE_ABS2:
  // real |y|^2 output)
  const R* xr;
  R* outr;
  // exact mode: the reference's twiddle table tw[j] = e^{-2 pi i j / N},
  // j < N/2, rounded to R (fft.py:70-78); null for the fast path
  const Cpx<R>* xtw;
};

// fused-kernel data modes
enum FMode : int {
  FMODE_C2C = 0,   // complex signal -> complex outputs (_kernels_nb.py:265)
  FMODE_R2R = 1,   // real signal, real taps -> real outputs; two segments per
                   // complex transform (re: segment 2k, im: segment 2k + 1)
  FMODE_ABS2 = 2,  // complex signal -> |y|^2 (fused_c2c_abs2, :288-309)
};

// streaming store of one real sample iff (mask & BIT)
template <unsigned BIT>
__device__ __forceinline__ void st_cs_mask_r(float* p, float v, unsigned mask) {
  asm volatile(
      "{\n .reg .pred q;\n .reg .b32 m;\n and.b32 m, %2, %3;\n"
      " setp.ne.u32 q, m, 0;\n"
      " @q st.global.cs.f32 [%0], %1;\n}" ::"l"(p),
      "f"(v), "r"(mask), "n"(BIT)
      : "memory");
}
template <unsigned BIT>
__device__ __forceinline__ void st_cs_mask_r(double* p, double v, unsigned mask) {
  asm volatile(
      "{\n .reg .pred q;\n .reg .b32 m;\n and.b32 m, %2, %3;\n"
      " setp.ne.u32 q, m, 0;\n"
      " @q st.global.cs.f64 [%0], %1;\n}" ::"l"(p),
      "d"(v), "r"(mask), "n"(BIT)
      : "memory");
}

// XR: exact mode (reference arithmetic, bit-identical to the reference's
// kernels; C2C and ABS2 only)
template <class C, int MODE = FMODE_C2C, bool XR = false>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
    fused_c2c_kernel(const FusedArgs<typename C::R> a) {
  using R = typename C::R;
  using G = typename C::G;
  constexpr int LOGN = C::LOGN;
  constexpr int E = C::E, T = C::T, P = C::P;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Cpx<R>* bufs = reinterpret_cast<Cpx<R>*>(smem_raw);
  Tw<R>* lowtab = reinterpret_cast<Tw<R>*>(smem_raw + C::f_tab_off);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem_raw + C::f_slot_off);

  const int tid = threadIdx.x;
  const int sl = tid / T;
  const int t = tid % T;

  // ---- work decomposition: items = (group of SEGS segments, filter chunk)
  const long long nseg = a.k_hi - a.k_lo;
  const long long ngroups = (nseg + C::SEGS - 1) / C::SEGS;
  const int nfch = (a.n_fil + a.fchunk - 1) / a.fchunk;
  // the balanced tail is compiled only into the <= 2 CTAs/SM policies (the
  // launcher never enables it for the others; keeping their item loop
  // minimal is worth 1.6% at cfg3)
  constexpr bool TS = C::MINB <= 2;
  const bool ts = TS && a.full_items > 0;
  const int ntch = ts ? (a.n_fil + a.tchunk - 1) / a.tchunk : 1;
  long long nitems = ngroups * nfch;
  if constexpr (TS) {
    if (ts) nitems = a.full_items + (ngroups - a.full_items) * ntch;
  }
  // item -> (segment group, first filter); filters [f_lo, f_lo + width)
  auto item = [&](long long it, long long& grp, int& f_lo, int& width) {
    if (TS && ts) {
      if (it < a.full_items) {
        grp = it;
        f_lo = 0;
        width = a.n_fil;
      } else {
        const long long r = it - a.full_items;
        grp = a.full_items + r / ntch;
        f_lo = int(r % ntch) * a.tchunk;
        width = a.tchunk;
      }
    } else {
      grp = it / nfch;
      f_lo = int(it - grp * nfch) * a.fchunk;
      width = a.fchunk;
    }
  };

  // L2 prefetch (TMA, one thread) of item `itn`'s input window: the live
  // segments of its group only, so it stays inside the input extent the
  // caller guarantees for [k_lo, k_hi)
  auto prefetch_window = [&](long long itn) {
    long long gn = itn / nfch;
    if constexpr (TS) {
      int fn_, wn_;
      item(itn, gn, fn_, wn_);
    }
    const long long sn = a.k_lo + gn * C::SEGS;
    const long long nl = a.k_hi - sn < C::SEGS ? a.k_hi - sn : C::SEGS;
    const long long segs = MODE == FMODE_R2R ? 2 * nl : nl;
    long long lo = (MODE == FMODE_R2R ? 2 * sn : sn) * a.seg_len - a.t0 + a.origin;
    long long hi = lo + (segs - 1) * a.seg_len + G::N;
    lo = lo > 0 ? lo : 0;
    hi = hi < a.n_s ? hi : a.n_s;
    const int esz = MODE == FMODE_R2R ? int(sizeof(R)) : int(sizeof(Cpx<R>));
    if (hi > lo) {
      const char* base = MODE == FMODE_R2R ? reinterpret_cast<const char*>(a.xr)
                                           : reinterpret_cast<const char*>(a.x);
      uintptr_t b0 = reinterpret_cast<uintptr_t>(base + (lo - a.x_base) * esz);
      uintptr_t b1 = reinterpret_cast<uintptr_t>(base + (hi - a.x_base) * esz);
      // stay inside the caller's buffer: whole 16-byte units only
      b0 = (b0 + 15) & ~uintptr_t(15);
      b1 &= ~uintptr_t(15);
      if (b1 > b0) l2_prefetch(reinterpret_cast<const void*>(b0), uint32_t(b1 - b0));
    }
  };

  // ---- filter-spectrum staging.  PREF: this thread's VPT vectors of the next filter, in registers
  float4 hn[C::PREF ? C::VPT : 1];
  auto fetch = [&](int f) {
    if constexpr (C::PREF) {
      const int hb = a.hoff + ((C::ABL & 8) ? (f & 1) : f) * (C::VPT * T);
      sfor<0, C::VPT>([&](auto uc) {
        constexpr int u = decltype(uc)::value;
        hn[u] = tex1Dfetch<float4>(a.htex, hb + spec_vec<R, LOGN>(t, u));
      });
    }
  };
  // the first item's spectrum and input window are requested before the
  // table build / TMEM allocation, so their latency overlaps the prologue
  // (the whole kernel is a few microseconds on small cells)
  if (blockIdx.x < nitems) {
    if (tid == 0) prefetch_window(blockIdx.x);
    int f0 = int(blockIdx.x % nfch) * a.fchunk;
    if constexpr (TS) {
      long long g_;
      int w_;
      item(blockIdx.x, g_, f0, w_);
    }
    fetch(f0);
    if constexpr (C::HT) {
      if (tid == 0) {
        const uint32_t hb0 = uint32_t(__cvta_generic_to_shared(smem_raw + C::f_hbar_off));
        mbar_init(hb0, 1);
        mbar_init(hb0 + 8, 1);
        mbar_init(hb0 + 16, C::THREADS / 32);
        mbar_init(hb0 + 24, C::THREADS / 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        constexpr uint32_t hbytes = uint32_t(C::VPT) * C::T * 16;
        mbar_expect_tx(hb0, hbytes);
        tma_load_1d(uint32_t(__cvta_generic_to_shared(smem_raw + C::f_ring_off)),
                    a.spec + size_t(f0) * (C::VPT * T), hbytes, hb0);
      }
    }
  }

  if constexpr (C::TMX) {
    if (tid < 32) tmem_alloc<C::TCOLS>(tslot);
    tmem_fence_before();
  }
  Tw<R>* jt = reinterpret_cast<Tw<R>*>(smem_raw + C::f_jt_off);
  build_tables<R, LOGN>(lowtab,
                        C::TOPOUT ? reinterpret_cast<Tw<R>*>(bufs) : nullptr,
                        XR ? a.xtw : nullptr);
  if constexpr (XR) build_jt<R, LOGN>(jt, a.xtw);
  if constexpr (C::MB) {
    if (tid < C::SEGS) mbar_init(group_mbar<C>(tid), T / 32);
  }
  __syncthreads();
  uint32_t tbase = 0, tb = 0;
  if constexpr (C::TMX) {
    tmem_fence_after();
    tbase = *tslot;
    const int w = tid / 32;
    tb = tbase + (uint32_t((w & 3) * 32) << 16) + uint32_t((w >> 2) * C::CPW);
  }

  // runtime-window twiddles: fixed per thread for the kernel lifetime, in
  // registers (TOPREG) or TMEM (TMX)
  Tw<R> twr[15];
  if constexpr (C::TMX == 2) {
    Tw<R> twm[15];
    constexpr int q = P - 2;
    const TwSmem<R> tt = tw_smem<R, LOGN, q>(lowtab + G::tw_offset(q), t);
    twm[0] = tt.get0();
#pragma unroll
    for (int pp = 1; pp < 8; ++pp) {
      const TwPair<R> w = tt.get2(pp);
      twm[2 * pp - 1] = w.a;
      twm[2 * pp] = w.b;
    }
    tmem_st_tw(tb + 64, twm);
  }
  if constexpr (C::TOPOUT) {
    constexpr int q = P - 1;
    const TwSmem<R> tt =
        tw_smem<R, LOGN, q>(reinterpret_cast<const Tw<R>*>(bufs), t);
    twr[0] = tt.get0();
#pragma unroll
    for (int pp = 1; pp < 8; ++pp) {
      const TwPair<R> w = tt.get2(pp);
      twr[2 * pp - 1] = w.a;
      twr[2 * pp] = w.b;
    }
    if constexpr (C::TMX) {
      tmem_st_tw(tb + 32, twr);
      tmem_wait_st();
    }
    __syncthreads();  // the exchange buffers are free from here on
  }

  const R inv_n = R(1) / R(G::N);
  int xc = 0;
  int hc = 0;  // HT: spectra consumed so far (ring slot hc & 1)

  for (long long it = blockIdx.x; it < nitems; it += gridDim.x) {
    long long grp = it / nfch;
    int f_lo = int(it - grp * nfch) * a.fchunk, f_w = a.fchunk;
    if constexpr (TS) item(it, grp, f_lo, f_w);
    // s = segment (R2R: segment pair {2s, 2s + 1}) of this thread's group
    const long long s = a.k_lo + grp * C::SEGS + sl;
    const bool live = s < a.k_hi;
    const long long g0 = (MODE == FMODE_R2R ? 2 * s : s) * a.seg_len;
    const int o0 = G::thread_part(P - 1, t) - a.t0;
    // owned outputs o in [o_lo, o_hi) of the segment starting at g (clipped
    // to this call's range) -> writeback mask (item-invariant): element e of
    // this thread is output o = o0 + elem_part(e), kept iff o_lo <= o < o_hi
    auto seg_mask = [&](long long g, long long& olo, unsigned& sp) {
      olo = a.g_lo > g ? a.g_lo - g : 0;
      const long long ohi = a.g_hi - g < a.seg_len ? a.g_hi - g : a.seg_len;
      sp = (!live || (a.dbg & 1) || (C::ABL & 1) || ohi <= olo)
               ? 0u
               : unsigned(ohi - olo);
      unsigned m = 0;
      sfor<0, E>([&](auto ec) {
        constexpr int e = decltype(ec)::value;
        const unsigned o = unsigned(o0 + G::elem_part(P - 1, e) - int(olo));
        m |= (o < sp ? 1u : 0u) << e;
      });
      return m;
    };
    long long o_lo, o_lo_b = 0;
    unsigned span, span_b = 0;
    const unsigned vmask = seg_mask(g0, o_lo, span);
    const unsigned vmask_b =
        MODE == FMODE_R2R ? seg_mask(g0 + a.seg_len, o_lo_b, span_b) : 0u;
    const long long w0 = g0 - a.t0 + a.origin;
    // L2 prefetch of the next item's input window (TMA, one thread): with
    // few filters per segment nothing else hides the DRAM latency of the
    // gather at the start of an item
    if (tid == 0 && it + gridDim.x < nitems) prefetch_window(it + gridDim.x);
    const int f_hi = min(a.n_fil, f_lo + f_w);
    const long long nit = it + gridDim.x;
    int f_next_item = nit < nitems ? int(nit % nfch) * a.fchunk : -1;
    if constexpr (TS) {
      if (nit < nitems) {
        long long gn2;
        int wn2;
        item(nit, gn2, f_next_item, wn2);
      }
    }

    // ---- segment staging: zero-extended window, top-window layout
    // (_gather, _kernels_nb.py:206-215)
    Cpx<R> x[E];
    if constexpr (MODE == FMODE_R2R) {
      // re <- segment 2s's window, im <- segment 2s + 1's.  Both halves are
      // always loaded (the partner's samples change the rounding of the
      // other half), so results are bit-identical for any split of the
      // output range; the caller provides the pair-aligned input extent
      // (olsb_input_extent_r2r)
      constexpr int q = P - 1;
      const long long pa = w0 + G::thread_part(q, t);
      const long long pbb = pa + a.seg_len;
      const bool la = live, lb = live;
      sfor<0, E>([&](auto ec) {
        constexpr int e = decltype(ec)::value;
        const long long ga = pa + G::elem_part(q, e);
        const long long gb = pbb + G::elem_part(q, e);
        const R ra = ld_nc_or0(a.xr + (ga - a.x_base),
                               la && (unsigned long long)ga < (unsigned long long)a.n_s);
        const R rb = ld_nc_or0(a.xr + (gb - a.x_base),
                               lb && (unsigned long long)gb < (unsigned long long)a.n_s);
        x[e] = Cpx<R>{ra, rb};
      });
    } else {
      constexpr int q = P - 1;
      const long long pb = w0 + G::thread_part(q, t);
      const Cpx<R>* xp = a.x + (pb - a.x_base);
      sfor<0, E>([&](auto ec) {
        constexpr int e = decltype(ec)::value;
        const long long gi = pb + G::elem_part(q, e);
        x[e] = ld_nc_or0(xp + G::elem_part(q, e),
                         live && (unsigned long long)gi < (unsigned long long)a.n_s);
      });
    }
    // ---- forward FFT (dif_fwd, _kernels_nb.py:11-28); the spectrum stays in
    // registers (or TMEM) with the inverse's 1/N and the scale post-process
    // folded in
    forward_fft<C, C::TOPREG, XR>(x, lowtab, twr, bufs, xc, sl, t, tb, jt);
    if constexpr (!XR) {
      const R sc = a.pp_kind == OLSB_PP_SCALE ? inv_n * a.pp_c : inv_n;
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = cscale(x[e], sc);
    }
    if constexpr (C::TMX) {
      tmem_st_cpx(tb, x);
      tmem_wait_st();
    }

    for (int f = f_lo; f < f_hi; ++f) {
      const int f_next = f + 1 < f_hi ? f + 1 : f_next_item;
      // ---- pointwise multiply, both operands bit-reversed
      // (_kernels_nb.py:280-282)
      Cpx<R> y[E];
      if constexpr (C::TMX) tmem_ld_cpx(tb, y);  // y = segment spectrum
      const Cpx<R>* xs = C::TMX ? y : x;
      auto mul1 = [&](Cpx<R> xv, Cpx<R> hv) {
        if constexpr (XR) {
          return cmul_ref(xv, hv);
        } else {
          return cmul(xv, hv);
        }
      };
      auto mulh = [&](int u, float4 h) {
        y[2 * u] = mul1(xs[2 * u], Cpx<R>{R(h.x), R(h.y)});
        y[2 * u + 1] = mul1(xs[2 * u + 1], Cpx<R>{R(h.z), R(h.w)});
      };
      if constexpr (C::PREF) {
        sfor<0, C::VPT>([&](auto uc) {
          constexpr int u = decltype(uc)::value;
          mulh(u, hn[u]);
        });
        if (f_next >= 0) fetch(f_next);
      } else if constexpr (C::HT) {
        const uint32_t hb0 = uint32_t(__cvta_generic_to_shared(smem_raw + C::f_hbar_off));
        constexpr uint32_t hbytes = uint32_t(C::VPT) * C::T * 16;
        if (tid == 0 && f_next >= 0) {
          // the next spectrum into the other slot, once every warp has
          // released that slot's previous contents (consumption hc - 1)
          const int sn = (hc + 1) & 1;
          if (hc >= 1) mbar_wait(hb0 + 16 + 8 * sn, uint32_t((hc - 1) >> 1) & 1u);
          mbar_expect_tx(hb0 + 8 * sn, hbytes);
          tma_load_1d(uint32_t(__cvta_generic_to_shared(smem_raw + C::f_ring_off)) +
                          uint32_t(sn) * uint32_t(C::h_slot_bytes),
                      a.spec + size_t(f_next) * (C::VPT * T), hbytes,
                      hb0 + 8 * sn);
        }
        const int sc = hc & 1;
        mbar_wait(hb0 + 8 * sc, uint32_t(hc >> 1) & 1u);
        const float4* hs = reinterpret_cast<const float4*>(
            smem_raw + C::f_ring_off + size_t(sc) * C::h_slot_bytes);
        sfor<0, C::VPT>([&](auto uc) {
          constexpr int u = decltype(uc)::value;
          mulh(u, hs[spec_vec<R, LOGN>(t, u)]);
        });
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(hb0 + 16 + 8 * sc);
        ++hc;
      } else if constexpr (C::HM == H_TEX) {
        const int hb = a.hoff + f * (C::VPT * T);
        sfor<0, C::VPT>([&](auto uc) {
          constexpr int u = decltype(uc)::value;
          mulh(u, tex1Dfetch<float4>(a.htex, hb + spec_vec<R, LOGN>(t, u)));
        });
      } else {
        const typename V16<R>::type* hs = a.spec + (size_t(f) * C::VPT) * T;
        sfor<0, C::VPT>([&](auto uc) {
          constexpr int u = decltype(uc)::value;
          const auto h = __ldg(hs + spec_vec<R, LOGN>(t, u));
          if constexpr (V16<R>::per == 2) {
            mulh(u, h);
          } else {
            y[u] = mul1(x[u], Cpx<R>{h.x, h.y});
          }
        });
      }
      // ---- inverse FFT (dit_inv, _kernels_nb.py:31-51)
      if constexpr (XR) {
        pass_static_ref<R, C::LOGE, G::G0, true>(y, jt);
      } else {
        dit_pass_static<R, C::LOGE, G::G0>(y);
      }
      sfor<1, P>([&](auto qc) {
        constexpr int q = decltype(qc)::value;
        exchange<C, q - 1, q>(bufs, xc, sl, t, y, IC<C::ABL>{});
        auto pass = [&](const auto& tws) {
          if constexpr (XR) {
            pass_ref<R, true>(y, tws);
          } else {
            dit_pass_rt<R, G::tan01(q)>(y, tws, top_bits<LOGN, q>(t));
          }
        };
        if constexpr (C::TMX && (q == P - 1 || (q == P - 2 && C::TMX == 2))) {
          Tw<R> tw[16];
          tmem_ld_tw(tb + (q == P - 1 ? 32u : 64u), tw);
          pass(TwRegs<R>{tw});
        } else if constexpr (q == P - 1 && C::TOPREG) {
          pass(TwRegs<R>{twr});
        } else {
          pass(tw_smem<R, LOGN, q>(lowtab + G::tw_offset(q), t));
        }
      });
      if constexpr (XR) {
        // dit_inv's final 1/N (exact: a power of two), then _store's pp_c:
        // the reference multiplies a Python float by the complex64 sample,
        // i.e. in double precision, and rounds once into the output
        // (_kernels_nb.py:223-225)
        const bool scl = a.pp_kind == OLSB_PP_SCALE;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          Cpx<R> v{mul_rn(y[e].re, inv_n), mul_rn(y[e].im, inv_n)};
          if (scl)
            v = Cpx<R>{R(__dmul_rn(a.pp_cd, double(v.re))),
                       R(__dmul_rn(a.pp_cd, double(v.im)))};
          y[e] = v;
        }
      }
      // ---- valid-sample writeback (_store kind 0/1, _kernels_nb.py:218-222):
      // in-place sample p is output o = p - t0 of this segment, kept iff
      // o_lo <= o < o_hi.  With the 32-aligned engine grid every warp store
      // covers one aligned 256-byte chunk of the output row.
      if constexpr (MODE != FMODE_ABS2) {
        if (a.pp_kind == OLSB_PP_DERIV) {
          // non-local epilogue (_store kind 3, _kernels_nb.py:224-262):
          // central difference of neighbouring samples, one-sided at the
          // signal ends.  The segment is staged in natural order in this
          // group's exchange buffer (free after the last exchange) and p +- 1
          // read back; the halo geometry keeps both inside the segment.
          const R half = R(0.5);
          auto dv = [&](long long g, R l, R c, R r) {
            return g == 0 ? r - c : (g == a.n_s - 1 ? c - l : half * (r - l));
          };
          const int pb = G::thread_part(P - 1, t);
          if constexpr (P == 1) {
            // one thread holds the whole segment in natural order
            Cpx<R> d[E];
            sfor<0, E>([&](auto ec) {
              constexpr int e = decltype(ec)::value;
              const Cpx<R> l = y[e > 0 ? e - 1 : 0];
              const Cpx<R> r = y[e + 1 < E ? e + 1 : E - 1];
              const long long g = g0 + (e - a.t0);
              const long long gi = MODE == FMODE_R2R ? g + a.seg_len : g;
              d[e] = Cpx<R>{dv(g, l.re, y[e].re, r.re),
                            dv(gi, l.im, y[e].im, r.im)};
            });
            sfor<0, E>([&](auto ec) { y[decltype(ec)::value] = d[decltype(ec)::value]; });
          } else {
            Cpx<R>* stg = bufs + size_t(sl) * C::L::stride;
            group_sync<C>(sl);
            sfor<0, E>([&](auto ec) {
              constexpr int e = decltype(ec)::value;
              stg[pb + G::elem_part(P - 1, e)] = y[e];
            });
            group_sync<C>(sl);
            sfor<0, E>([&](auto ec) {
              constexpr int e = decltype(ec)::value;
              const int p = pb + G::elem_part(P - 1, e);
              const Cpx<R> l = stg[p > 0 ? p - 1 : 0];
              const Cpx<R> r = stg[p + 1 < G::N ? p + 1 : G::N - 1];
              const long long g = g0 + (p - a.t0);
              const long long gi = MODE == FMODE_R2R ? g + a.seg_len : g;
              y[e] = Cpx<R>{dv(g, l.re, y[e].re, r.re),
                            dv(gi, l.im, y[e].im, r.im)};
            });
            if constexpr (C::NBUF >= 2 || C::MB) group_sync<C>(sl);  // next exchange
          }
        }
      }
      if constexpr (MODE == FMODE_C2C) {
        const long long goff = (long long)f * a.out_ld + (g0 - a.out_base);
        Cpx<R>* orow = a.out + goff + o0;
        sfor<0, E>([&](auto ec) {
          constexpr int e = decltype(ec)::value;
          constexpr int pe = G::elem_part(P - 1, e);
          st_cs_mask<(1u << e)>(orow + pe, y[e], vmask);
        });
      } else {
        // real outputs: |y|^2 (ABS2), or re -> segment 2s and im -> 2s + 1
        // (R2R, squared for magnitude_squared as fused_r2r pp_kind 2)
        const long long goff = (long long)f * a.out_ld + (g0 - a.out_base);
        R* orow = a.outr + goff + o0;
        const bool sq = a.pp_kind == OLSB_PP_MAG2;
        sfor<0, E>([&](auto ec) {
          constexpr int e = decltype(ec)::value;
          constexpr int pe = G::elem_part(P - 1, e);
          if constexpr (MODE == FMODE_ABS2 && XR) {
            st_cs_mask_r<(1u << e)>(
                orow + pe,
                add_rn(mul_rn(y[e].re, y[e].re), mul_rn(y[e].im, y[e].im)), vmask);
          } else if constexpr (MODE == FMODE_ABS2) {
            st_cs_mask_r<(1u << e)>(orow + pe,
                                    fmaR(y[e].re, y[e].re, y[e].im * y[e].im),
                                    vmask);
          } else {
            const R va = sq ? y[e].re * y[e].re : y[e].re;
            const R vb = sq ? y[e].im * y[e].im : y[e].im;
            st_cs_mask_r<(1u << e)>(orow + pe, va, vmask);
            st_cs_mask_r<(1u << e)>(orow + a.seg_len + pe, vb, vmask_b);
          }
        });
      }
    }
  }
  if constexpr (C::TMX) {
    tmem_fence_before();
    __syncthreads();
    if (tid < 32) tmem_dealloc<C::TCOLS>(tbase);
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
  Cpx<R>* out_perm;                // may be null
  typename V16<R>::type* out_dev;  // may be null
  const Cpx<R>* xtw;               // exact mode: the reference's tw table
};

template <class C, bool XR = false>
__global__ void __launch_bounds__(C::THREADS)
    fwd_rows_kernel(const RowsArgs<typename C::R> a) {
  using R = typename C::R;
  using G = typename C::G;
  constexpr int E = C::E, T = C::T, P = C::P;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Tw<R>* tab = reinterpret_cast<Tw<R>*>(smem_raw);
  Cpx<R>* bufs = reinterpret_cast<Cpx<R>*>(smem_raw + C::tab_bytes);
  Tw<R>* jt = reinterpret_cast<Tw<R>*>(smem_raw + C::jt_off);
  const int sl = threadIdx.x / T, t = threadIdx.x % T;
  build_tables<R, C::LOGN>(tab, nullptr, XR ? a.xtw : nullptr);
  if constexpr (XR) build_jt<R, C::LOGN>(jt, a.xtw);
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
    forward_fft<C, false, XR>(x, tab, nullptr, bufs, xc, sl, t, 0, jt);
    if (live) {
      if (a.out_perm) {
        Cpx<R>* o = a.out_perm + size_t(r) * G::N + G::thread_part(0, t);
#pragma unroll
        for (int e = 0; e < E; ++e) o[e] = x[e];
      }
      if (a.out_dev) {
        typename V16<R>::type* o = a.out_dev + size_t(r) * C::VPT * T;
        if constexpr (!C::dbl) {
#pragma unroll
          for (int u = 0; u < C::VPT; ++u)
            o[spec_vec<R, C::LOGN>(t, u)] = make_float4(x[2 * u].re, x[2 * u].im, x[2 * u + 1].re,
                                   x[2 * u + 1].im);
        } else {
#pragma unroll
          for (int u = 0; u < C::VPT; ++u)
            o[spec_vec<R, C::LOGN>(t, u)] = make_double2(x[u].re, x[u].im);
        }
      }
    }
  }
}

template <class C>
__global__ void __launch_bounds__(C::THREADS)
    inv_rows_kernel(const Cpx<typename C::R>* in, Cpx<typename C::R>* out,
                    int rows) {
  using R = typename C::R;
  using G = typename C::G;
  constexpr int LOGN = C::LOGN;
  constexpr int E = C::E, T = C::T, P = C::P;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Tw<R>* tab = reinterpret_cast<Tw<R>*>(smem_raw);
  Cpx<R>* bufs = reinterpret_cast<Cpx<R>*>(smem_raw + C::tab_bytes);
  const int sl = threadIdx.x / T, t = threadIdx.x % T;
  build_tables<R, LOGN>(tab, nullptr);
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
      exchange<C, q - 1, q>(bufs, xc, sl, t, y);
      dit_pass_rt<R, G::tan01(q)>(
          y, tw_smem<R, LOGN, q>(tab + G::tw_offset(q), t),
          top_bits<LOGN, q>(t));
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

template <class C>
__global__ void perm_to_dev_kernel(const Cpx<typename C::R>* perm,
                                   typename V16<typename C::R>::type* dev,
                                   int rows) {
  using R = typename C::R;
  constexpr int T = C::T, VPT = C::VPT, per = V16<R>::per;
  const long long total = (long long)rows * VPT * T;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
       i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / (VPT * T);
    const int rem = int(i - r * VPT * T);
    const int u = rem / T, t = rem % T;
    const Cpx<R>* s = perm + r * C::G::N + t * C::E + u * per;
    if constexpr (per == 2) {
      dev[r * (VPT * T) + spec_vec<R, C::LOGN>(t, u)] =
          make_float4(s[0].re, s[0].im, s[1].re, s[1].im);
    } else {
      dev[i] = make_double2(s[0].re, s[0].im);
    }
  }
}

}  // namespace olsb
