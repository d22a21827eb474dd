// olsb_launch.cuh — kernel policies and launchers of the OLS engine.
//
// The launch templates are instantiated once per FFT length in separate
// translation units (olsb_inst.cu compiled with -DOLSB_LOGN=L, in parallel by
// build.py); olsb_kernels.cu sees only the extern declarations below.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "olsb.h"
#include "olsb_engine.cuh"
#include "olsb_w64.cuh"
#include "olsb_w64x2.cuh"
#include "olsb_w32x2.cuh"

namespace olsb {

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------
inline int num_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 1;
}

// Kernel attributes + resident CTA count, done once per (kernel, device):
// the attribute call and the occupancy query cost microseconds, which is the
// whole budget of a small convolution (cache in olsb_kernels.cu).
int prepared_lookup(const void* kernel, int* resident);
void prepared_store(const void* kernel, int resident);

template <class K>
int prepare(K kernel, size_t smem, int threads, int* resident) {
  if (prepared_lookup(reinterpret_cast<const void*>(kernel), resident)) return 0;
  cudaError_t e = cudaFuncSetAttribute(
      kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return int(e);
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads,
                                                    smem);
  if (e != cudaSuccess) return int(e);
  *resident = std::max(1, occ) * num_sms();
  prepared_store(reinterpret_cast<const void*>(kernel), *resident);
  return 0;
}

extern int g_filter_chunk;

// texture object over engine-layout spectra (cached; olsb_kernels.cu)
int spectra_texture(const void* ptr, size_t bytes, cudaTextureObject_t* out);

// Bind the spectra of a launch: linear textures need a textureAlignment-
// aligned base, and callers may pass a sub-range of a filter bank (the
// streaming path's row chunks), so the texture starts at the aligned-down
// address and the kernel adds the float4 offset.
template <class R>
int bind_spectra(FusedArgs<R>& a, size_t bytes) {
  static int align = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrTextureAlignment, dev);
    return v > 0 ? v : 512;
  }();
  const uintptr_t p = reinterpret_cast<uintptr_t>(a.spec);
  const uintptr_t base = p & ~uintptr_t(align - 1);
  a.hoff = int((p - base) / 16);
  return spectra_texture(reinterpret_cast<const void*>(base), bytes + (p - base),
                         &a.htex);
}

// default fused-kernel policy per (precision, N)
template <class R, int LOGN>
struct DefaultPolicy {
  static constexpr bool dbl = std::is_same<R, double>::value;
  static constexpr int T = Geo<LOGN>::T;
  // fp32 (OLSB_VARIANT=2 / 3 of the sweep in DESIGN.md §5, plus BAR = 1): 128-thread CTAs,
  // 4 CTAs per SM, segment spectrum and runtime-window twiddles in TMEM, the
  // next filter's spectrum prefetched through the TEX path; N = 4096 double
  // buffers the exchanges: its first inverse exchange is warp-local (no
  // Geo::remap at N = 4096, only __syncwarp), the second keeps a barrier on
  // both sides (a third buffer would remove one, but the 113 KB of shared
  // memory per CTA leave too little L1 for the spectrum fetches: slower).
  // fp64: 128-thread CTAs (256 for N = 4096) at 3 CTAs/SM, 170 registers
  // (OLSB_DVARIANT sweep: cfg3 shape 5.65 vs 6.12 ms for 256-thread CTAs at
  // one CTA/SM)
  static constexpr int SEGS = std::max(1, 128 / T);
  // BAR = 1: named barrier per segment group, so only the warps of one
  // segment are coupled (matters for N = 1024: two 2-warp groups per CTA)
  // (The mbarrier "buffer free" exchanges of OLSB_VARIANT=8 are 4% faster at
  // N = 1024 but not default: compute-sanitizer racecheck does not model the
  // mbarrier wait and reports the exchange as a race.)
  using type = KCfg<R, LOGN, SEGS, (!dbl && LOGN == 12) ? 2 : 1,
                    dbl ? H_LDG : H_TEX, 1,
                    dbl ? (SEGS * T >= 256 ? 1 : 3)
                        : std::max(1, 512 / (SEGS * T)),
                    dbl ? 0 : 2,
                    dbl ? 0 : 1>;
};

// tuning variants for fp32 (OLSB_VARIANT).  A CTA holds SEGS x max(1,
// 128 / T) segments; MINB is the target number of 128-thread warpgroups per
// SM (CTAs per SM = MINB x 128 / CTA threads).
template <int LOGN, int V>
struct Variant {
  static constexpr int T = Geo<LOGN>::T;
  // {SEGS, NBUF, HM, BAR, MINB (warpgroups/SM), TMX, PREF, ABL, MB}
  static constexpr int tab[9][9] = {
      {1, 1, H_TEX, 0, 4, 0, 0, 0, 0}, {1, 1, H_TEX, 0, 4, 1, 1, 0, 0},
      {1, 1, H_TEX, 0, 4, 2, 1, 0, 0}, {1, 2, H_TEX, 0, 4, 2, 1, 0, 0},
      {1, 1, H_TEX, 0, 4, 2, 1, 1, 0}, {1, 1, H_TEX, 0, 4, 2, 1, 6, 0},
      {1, 1, H_TEX, 0, 4, 2, 1, 8, 0}, {1, 1, H_TEX, 0, 4, 2, 1, 14, 0},
      {1, 1, H_TEX, 1, 4, 2, 1, 0, 1}};
  static constexpr int segs = tab[V][0] * std::max(1, 128 / T);
  static constexpr int minb = std::max(1, tab[V][4] * 128 / (segs * T));
  using type = KCfg<float, LOGN, segs, tab[V][1], tab[V][2], tab[V][3], minb,
                    tab[V][5], tab[V][6], tab[V][7], tab[V][8]>;
};

inline int debug_env() {
  static int v = [] {
    const char* e = getenv("OLSB_DEBUG");
    return e ? atoi(e) : 0;
  }();
  return v;
}

inline int tail_env() {
  static int v = [] {
    const char* e = getenv("OLSB_TAIL_SPLIT");
    return e ? atoi(e) : 4;
  }();
  return v;
}
inline bool tail_forced() {
  static bool v = getenv("OLSB_TAIL_SPLIT") != nullptr;
  return v;
}

// experiment: filter spectra through the shared-memory TMA ring (H_TMA)
// instead of the TEX path (1: with the default TMEM residency, 2: TMX = 1)
inline int htma_env() {
  static int v = [] {
    const char* e = getenv("OLSB_HTMA");
    return e ? atoi(e) : 0;
  }();
  return v;
}
template <class R, int LOGN, int TMX>
using HtmaPolicy =
    KCfg<R, LOGN, DefaultPolicy<R, LOGN>::SEGS, 1, H_TMA, 1,
         DefaultPolicy<R, LOGN>::type::MINB, TMX, 0>;

// experiment: cap on CTAs per SM of the fused launch (0 = the policy's)
inline int grid_cap_env() {
  static int v = [] {
    const char* e = getenv("OLSB_GRID_CAP");
    return e ? atoi(e) : 0;
  }();
  return v;
}

inline int variant_env() {
  static int v = [] {
    const char* e = getenv("OLSB_VARIANT");
    return e ? atoi(e) : -1;
  }();
  return v;
}

// Fill the device-wide twiddle table of (R, LOGN) once per device, on the
// caller's stream (kernels that run before it completes compute their own).
template <class R, int LOGN>
int ensure_twiddle_table(cudaStream_t st) {
  constexpr int kMaxDev = 64;
  static std::atomic<int> filled[kMaxDev];
  if (Geo<LOGN>::tw_total() == 0) return 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDev) return 0;
  if (filled[dev].exchange(1) == 1) return 0;
  tw_table_kernel<R, LOGN><<<1, 1024, 0, st>>>();
  return int(cudaGetLastError());
}

template <class C, int MODE = FMODE_C2C, bool XR = false>
int launch_fused_cfg(FusedArgs<typename C::R> a, cudaStream_t st) {
  if (int rc = ensure_twiddle_table<typename C::R, C::LOGN>(st)) return rc;
  auto kern = fused_c2c_kernel<C, MODE, XR>;
  int resident = 0;
  int rc = prepare(kern, C::f_smem_bytes, C::THREADS, &resident);
  if (rc) return rc;
  // the occupancy API reports one CTA per SM for kernels that allocate
  // tensor memory; the TMEM policies size their columns for MINB CTAs/SM
  if constexpr (C::TMX) resident = std::max(resident, C::MINB * num_sms());
  if (grid_cap_env() > 0)
    resident = std::min(resident, grid_cap_env() * num_sms());
  if constexpr (C::HM == H_TEX) {
    rc = bind_spectra(a, size_t(a.n_fil) * C::VPT * C::T * 16);
    if (rc) return rc;
  }
  a.fchunk = (g_filter_chunk > 0 && g_filter_chunk < a.n_fil) ? g_filter_chunk
                                                              : a.n_fil;
  const long long nseg = a.k_hi - a.k_lo;
  const long long ngroups = (nseg + C::SEGS - 1) / C::SEGS;
  long long nitems = ngroups * ((a.n_fil + a.fchunk - 1) / a.fchunk);
  a.full_items = 0;
  a.tchunk = a.n_fil;
  // balanced tail: whole waves of full-filter items, then the leftover
  // groups in items of ~n_fil/4 filters.  It pays only where a CTA that runs
  // out of work leaves much of its SM idle (<= 2 CTAs/SM, N = 4096) and the
  // tail is a large part of the launch (< 6 waves): cfg2 N = 4096 0.416 ->
  // 0.390 ms; with 4 CTAs/SM the other CTAs absorb the idle share and the
  // extra forward transforms cost more (cfg3 1.72 -> 1.74 ms).
  // OLSB_TAIL_SPLIT overrides the divisor (0 disables).
  const int tdiv = tail_env();
  if (a.fchunk == a.n_fil && tdiv > 0 && a.n_fil >= 2 * tdiv &&
      C::MINB <= 2 && (tail_forced() || ngroups < 6LL * resident) &&
      ngroups > resident && ngroups % resident != 0) {
    a.full_items = (ngroups / resident) * resident;
    a.tchunk = (a.n_fil + tdiv - 1) / tdiv;
    nitems = a.full_items +
             (ngroups - a.full_items) * ((a.n_fil + a.tchunk - 1) / a.tchunk);
  }
  const int grid = int(std::min<long long>(nitems, resident));
  if (grid <= 0) return 0;
  kern<<<grid, C::THREADS, C::f_smem_bytes, st>>>(a);
  return int(cudaGetLastError());
}

// fp64 tuning variants (OLSB_DVARIANT): 128-thread CTAs (one segment group
// for N >= 2048) at 2 / 3 / 4 CTAs per SM (255 / 170 / 128 registers)
inline int dvariant_env() {
  static int v = [] {
    const char* e = getenv("OLSB_DVARIANT");
    return e ? atoi(e) : -1;
  }();
  return v;
}
template <int LOGN, int MINB>
using DVariant = KCfg<double, LOGN, std::max(1, 128 / Geo<LOGN>::T), 1, H_LDG, 1,
                      MINB>;

// One filter per item: the spectrum is used once, so parking it (and the
// twiddles) in TMEM and prefetching the next filter only add latency; the
// register policy is 2-11% faster on F = 1 cells (cfg1 9.7 -> 8.6 us kernel,
// tools/time_graph.py).
template <class R, int LOGN>
using SingleFilterPolicy =
    KCfg<R, LOGN, DefaultPolicy<R, LOGN>::SEGS,
         DefaultPolicy<R, LOGN>::type::NBUF, DefaultPolicy<R, LOGN>::type::HM,
         1, DefaultPolicy<R, LOGN>::type::MINB, 0, 0>;

// warp-per-segment engine for N = 2048 (olsb_w64.cuh), selected with
// OLSB_W64=1.  Not the default: at 8 warps/SM (252 registers) its FP core
// alone takes 1.32 ms on cfg3 against the E = 16 engine's 1.05 ms, so
// halving the exchange traffic and dropping the CTA barriers only reaches
// parity (1.68 ms)
inline int w64_env() {
  static int v = [] {
    const char* e = getenv("OLSB_W64");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <int WPC, int MINB, int MODE>
int launch_w64_cfg(FusedArgs<float> a, cudaStream_t st) {
  auto kern = w64::fused_w64_kernel<WPC, MINB, MODE>;
  constexpr size_t smem = size_t(WPC) * w64::BUF * sizeof(Cpx<float>) + 16;
  int resident = 0;
  int rc = prepare(kern, smem, WPC * 32, &resident);
  if (rc) return rc;
  // TMEM-allocating kernels: the occupancy API reports 1 CTA/SM
  resident = std::max(resident, MINB * num_sms());
  rc = bind_spectra(a, size_t(a.n_fil) * 1024 * 16);
  if (rc) return rc;
  const long long nseg = a.k_hi - a.k_lo;
  const long long warps = (long long)resident * WPC;
  // whole waves of full-filter items, then the leftover segments in items
  // of ~n_fil/8 filters so every warp finishes within one small item
  a.full_items = nseg;
  a.tchunk = a.n_fil;
  if (nseg % warps != 0 && a.n_fil >= 2) {
    a.full_items = (nseg / warps) * warps;
    const int tdiv = std::min(8, a.n_fil);
    a.tchunk = (a.n_fil + tdiv - 1) / tdiv;
  }
  const long long ntch = (a.n_fil + a.tchunk - 1) / a.tchunk;
  const long long nitems = a.full_items + (nseg - a.full_items) * ntch;
  const long long grid = std::min<long long>((nitems + WPC - 1) / WPC, resident);
  if (grid <= 0) return 0;
  kern<<<int(grid), WPC * 32, smem, st>>>(a);
  return int(cudaGetLastError());
}

// two-warps-per-segment engine for N = 4096 (olsb_w64x2.cuh), selected with
// OLSB_W64X2=1.  Not the default: parity green and equal to the E = 16
// engine on the cfg5 shard (21.0 vs 21.1 ms) but slower on cfg2 N = 4096
// (0.465 vs 0.395 ms, fewer segments than resident slots); like the N = 2048
// warp-per-segment engine it is held back by 8 warps/SM at 255 registers
// (profiles/r02_w64x2.log)
inline int w64x2_env() {
  static int v = [] {
    const char* e = getenv("OLSB_W64X2");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <int MODE>
int launch_w64x2(FusedArgs<float> a, cudaStream_t st) {
  auto kern = w64x2::fused_w64x2_kernel<MODE>;
  constexpr size_t smem = size_t(2) * w64x2::SBUF * sizeof(Cpx<float>) + 16;
  int resident = 0;
  int rc = prepare(kern, smem, 128, &resident);
  if (rc) return rc;
  resident = std::max(resident, 2 * num_sms());  // TMEM kernels: see above
  rc = bind_spectra(a, size_t(a.n_fil) * 2048 * 16);
  if (rc) return rc;
  const long long nseg = a.k_hi - a.k_lo;
  const long long slots = (long long)resident * 2;
  a.full_items = nseg;
  a.tchunk = a.n_fil;
  if (nseg % slots != 0 && a.n_fil >= 2) {
    a.full_items = (nseg / slots) * slots;
    const int tdiv = std::min(8, a.n_fil);
    a.tchunk = (a.n_fil + tdiv - 1) / tdiv;
  }
  const long long ntch = (a.n_fil + a.tchunk - 1) / a.tchunk;
  const long long nitems = a.full_items + (nseg - a.full_items) * ntch;
  const long long grid = std::min<long long>((nitems + 1) / 2, resident);
  if (grid <= 0) return 0;
  kern<<<int(grid), 128, smem, st>>>(a);
  return int(cudaGetLastError());
}

// two-warps-per-segment E = 32 engine for N = 2048 (olsb_w32x2.cuh),
// OLSB_W32X2=1
inline int w32x2_env() {
  static int v = [] {
    const char* e = getenv("OLSB_W32X2");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <int MODE>
int launch_w32x2(FusedArgs<float> a, cudaStream_t st) {
  auto kern = w32x2::fused_w32x2_kernel<MODE>;
  constexpr size_t smem = size_t(w32x2::SEGS) * w32x2::SBUF * sizeof(Cpx<float>) + 16;
  int resident = 0;
  int rc = prepare(kern, smem, w32x2::WARPS * 32, &resident);
  if (rc) return rc;
  resident = std::max(resident, num_sms());  // TMEM kernels: see above
  rc = bind_spectra(a, size_t(a.n_fil) * 1024 * 16);
  if (rc) return rc;
  const long long nseg = a.k_hi - a.k_lo;
  const long long slots = (long long)resident * w32x2::SEGS;
  a.full_items = nseg;
  a.tchunk = a.n_fil;
  if (nseg % slots != 0 && a.n_fil >= 2) {
    a.full_items = (nseg / slots) * slots;
    const int tdiv = std::min(8, a.n_fil);
    a.tchunk = (a.n_fil + tdiv - 1) / tdiv;
  }
  const long long ntch = (a.n_fil + a.tchunk - 1) / a.tchunk;
  const long long nitems = a.full_items + (nseg - a.full_items) * ntch;
  const long long grid =
      std::min<long long>((nitems + w32x2::SEGS - 1) / w32x2::SEGS, resident);
  if (grid <= 0) return 0;
  kern<<<int(grid), w32x2::WARPS * 32, smem, st>>>(a);
  return int(cudaGetLastError());
}

template <class R, int LOGN>
int launch_fused(FusedArgs<R> a, int mode, cudaStream_t st) {
  using D = typename DefaultPolicy<R, LOGN>::type;
  if constexpr (std::is_same<R, float>::value && LOGN == 12) {
    if (!a.xtw && variant_env() < 0 && w64x2_env() &&
        (a.pp_kind == OLSB_PP_NONE || a.pp_kind == OLSB_PP_SCALE)) {
      if (mode == FMODE_C2C) return launch_w64x2<FMODE_C2C>(a, st);
      if (mode == FMODE_ABS2) return launch_w64x2<FMODE_ABS2>(a, st);
    }
  }
  if constexpr (std::is_same<R, float>::value && LOGN == 11) {
    if (!a.xtw && variant_env() < 0 && w32x2_env() &&
        (a.pp_kind == OLSB_PP_NONE || a.pp_kind == OLSB_PP_SCALE)) {
      if (mode == FMODE_C2C) return launch_w32x2<FMODE_C2C>(a, st);
      if (mode == FMODE_ABS2) return launch_w32x2<FMODE_ABS2>(a, st);
    }
    if (!a.xtw && variant_env() < 0 && w64_env() &&
        (a.pp_kind == OLSB_PP_NONE || a.pp_kind == OLSB_PP_SCALE)) {
      if (mode == FMODE_C2C) return launch_w64_cfg<4, 2, FMODE_C2C>(a, st);
      if (mode == FMODE_ABS2) return launch_w64_cfg<4, 2, FMODE_ABS2>(a, st);
    }
  }
  if constexpr (std::is_same<R, float>::value) {
    if (!a.xtw && variant_env() < 0 && htma_env()) {
      if (a.n_fil == 1 || htma_env() == 3) {
        using S = HtmaPolicy<R, LOGN, 0>;
        if (mode == FMODE_R2R) return launch_fused_cfg<S, FMODE_R2R>(a, st);
        if (mode == FMODE_ABS2) return launch_fused_cfg<S, FMODE_ABS2>(a, st);
        return launch_fused_cfg<S>(a, st);
      }
      if (htma_env() == 2) {
        using S = HtmaPolicy<R, LOGN, 1>;
        if (mode == FMODE_R2R) return launch_fused_cfg<S, FMODE_R2R>(a, st);
        if (mode == FMODE_ABS2) return launch_fused_cfg<S, FMODE_ABS2>(a, st);
        return launch_fused_cfg<S>(a, st);
      }
      using S = HtmaPolicy<R, LOGN, 2>;
      if (mode == FMODE_R2R) return launch_fused_cfg<S, FMODE_R2R>(a, st);
      if (mode == FMODE_ABS2) return launch_fused_cfg<S, FMODE_ABS2>(a, st);
      return launch_fused_cfg<S>(a, st);
    }
    if (a.n_fil == 1 && !a.xtw && variant_env() < 0) {
      using S = SingleFilterPolicy<R, LOGN>;
      if (mode == FMODE_R2R) return launch_fused_cfg<S, FMODE_R2R>(a, st);
      if (mode == FMODE_ABS2) return launch_fused_cfg<S, FMODE_ABS2>(a, st);
      return launch_fused_cfg<S>(a, st);
    }
  }
  if (a.xtw) {  // exact mode (reference arithmetic), default policy
    if (mode == FMODE_ABS2) return launch_fused_cfg<D, FMODE_ABS2, true>(a, st);
    if (mode == FMODE_C2C) return launch_fused_cfg<D, FMODE_C2C, true>(a, st);
    return OLSB_E_UNSUPPORTED;
  }
  if constexpr (std::is_same<R, double>::value) {
    if (mode == FMODE_C2C) {
      switch (dvariant_env()) {
        case 2: return launch_fused_cfg<DVariant<LOGN, 2>>(a, st);
        case 3: return launch_fused_cfg<DVariant<LOGN, 3>>(a, st);
        case 4: return launch_fused_cfg<DVariant<LOGN, 4>>(a, st);
        default: break;
      }
    }
  }
  if (mode == FMODE_R2R) return launch_fused_cfg<D, FMODE_R2R>(a, st);
  if (mode == FMODE_ABS2) return launch_fused_cfg<D, FMODE_ABS2>(a, st);
  if constexpr (std::is_same<R, float>::value) {
    switch (variant_env()) {
      case 0: return launch_fused_cfg<typename Variant<LOGN, 0>::type>(a, st);
      case 1: return launch_fused_cfg<typename Variant<LOGN, 1>::type>(a, st);
      case 2: return launch_fused_cfg<typename Variant<LOGN, 2>::type>(a, st);
      case 3: return launch_fused_cfg<typename Variant<LOGN, 3>::type>(a, st);
      case 4: return launch_fused_cfg<typename Variant<LOGN, 4>::type>(a, st);
      case 5: return launch_fused_cfg<typename Variant<LOGN, 5>::type>(a, st);
      case 6: return launch_fused_cfg<typename Variant<LOGN, 6>::type>(a, st);
      case 7: return launch_fused_cfg<typename Variant<LOGN, 7>::type>(a, st);
      case 8: return launch_fused_cfg<typename Variant<LOGN, 8>::type>(a, st);
      default: break;
    }
  }
  return launch_fused_cfg<D>(a, st);
}

template <class R, int LOGN>
int launch_fwd_rows(RowsArgs<R> a, cudaStream_t st) {
  using C = RowCfg<R, LOGN>;
  auto kern = a.xtw ? fwd_rows_kernel<C, true> : fwd_rows_kernel<C, false>;
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
  using C = RowCfg<R, LOGN>;
  auto kern = inv_rows_kernel<C>;
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
  using C = RowCfg<R, LOGN>;
  const long long total = (long long)rows * C::VPT * C::T;
  if (total == 0) return 0;
  const int grid = int(std::min<long long>((total + 255) / 256, 4096));
  perm_to_dev_kernel<C><<<grid, 256, 0, st>>>(
      perm, reinterpret_cast<typename V16<R>::type*>(dev), rows);
  return int(cudaGetLastError());
}

}  // namespace olsb

#define OLSB_LAUNCHERS(EXT, R, L)                                            \
  EXT template int olsb::launch_fused<R, L>(olsb::FusedArgs<R>, int,         \
                                            cudaStream_t);                 \
  EXT template int olsb::launch_fwd_rows<R, L>(olsb::RowsArgs<R>,             \
                                               cudaStream_t);                 \
  EXT template int olsb::launch_inv_rows<R, L>(                               \
      const olsb::Cpx<R>*, olsb::Cpx<R>*, int, cudaStream_t);                 \
  EXT template int olsb::launch_perm_to_dev<R, L>(const olsb::Cpx<R>*, void*, \
                                                  int, cudaStream_t);
#define OLSB_LAUNCHERS_ALL(EXT, L) \
  OLSB_LAUNCHERS(EXT, float, L)    \
  OLSB_LAUNCHERS(EXT, double, L)
