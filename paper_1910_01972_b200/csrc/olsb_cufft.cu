// olsb_cufft.cu — the paper's cuFFT-based OLS comparison point (PAPER.md
// Algorithm 1; reference _pipelined, ols.py:363-410), written to be as fast
// as cuFFT allows without fusing the FFT itself:
//
//   per chunk of segments (the chunk's spectra X stay in L2):
//     pad     : the chunk's input span, zero-extended at the signal ends,
//               copied once (the only gather)
//     forward : ONE batched C2C whose input layout has idist = L < N, i.e.
//               cuFFT reads the overlapping segment windows in place
//     per chunk of filters:
//       multiply: Y[f, s, :] = X[s, :] * H[f, :]           (one kernel)
//       inverse : one batched C2C over (filter, segment), in place
//       store   : valid samples t >= M-1, times 1/N, into out[f, :]
//
// The paper's version moves the multiply into a cuFFT load callback and the
// discard into a store callback.  On this platform (cuFFT 11.4, sm_100a)
// legacy callbacks are accepted by cufftXtSetCallback but not applied (the
// transform still reads idata and writes every odata element), and LTO
// callbacks fail at plan creation (CUFFT_INTERNAL_ERROR): tools/mb_cufft_*.cu,
// profiles/r02_cufft_callbacks.log.  The explicit multiply / store kernels
// are the closest equivalent.
//
// Links the dynamic libcufft (whichever libcufft.so.11 the process has
// loaded, normally torch's); comparison point only, not the engine.
#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>

#include "olsb.h"

namespace {

// segment-chunk input span xs[i] = x[lo + i] (zero outside [0, n_s))
__global__ void pad_kernel(const float2* __restrict__ x, long long n_s,
                           long long lo, long long len, float2* __restrict__ xs) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len;
       i += (long long)gridDim.x * blockDim.x) {
    const long long g = lo + i;
    xs[i] = (g >= 0 && g < n_s) ? __ldg(x + g) : make_float2(0.f, 0.f);
  }
}

// Y[f, s, t] = X[s, t] * H[f0 + f, t]  (float4 = two complex)
__global__ void multiply_kernel(const float4* __restrict__ X,
                                const float4* __restrict__ H, int f0, int nf,
                                long long ns_c, int n2, float4* __restrict__ Y) {
  const long long per = ns_c * n2;
  const long long total = per * nf;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long f = i / per, r = i - f * per;
    const int t = int(r % n2);
    const float4 a = X[r];
    const float4 h = __ldg(H + (f0 + f) * (long long)n2 + t);
    Y[i] = make_float4(a.x * h.x - a.y * h.y, a.x * h.y + a.y * h.x,
                       a.z * h.z - a.w * h.w, a.z * h.w + a.w * h.z);
  }
}

// out[f0 + f, (s0 + s) L + j] = Y[f, s, t0 + j] / N for j < L, g < n_s
__global__ void store_kernel(const float2* __restrict__ Y, int f0, int nf,
                             long long s0, long long ns_c, int n, int t0,
                             long long L, long long n_s, float scale,
                             float2* __restrict__ out, long long out_ld) {
  const long long per = ns_c * L;
  const long long total = per * nf;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long f = i / per, r = i - f * per;
    const long long s = r / L, j = r - s * L;
    const long long g = (s0 + s) * L + j;
    if (g >= n_s) continue;
    const float2 v = Y[(f * ns_c + s) * n + t0 + j];
    __stcs(out + (f0 + f) * out_ld + g, make_float2(v.x * scale, v.y * scale));
  }
}

struct PlanKey {
  int dev, kind, n, batch;
  long long dist;
  bool operator<(const PlanKey& o) const {
    return std::tie(dev, kind, n, batch, dist) <
           std::tie(o.dev, o.kind, o.n, o.batch, o.dist);
  }
};
std::mutex g_mu;
std::map<PlanKey, cufftHandle> g_plans;

// kind 0: forward over overlapping windows (idist = L); kind 1: inverse,
// contiguous rows
int get_plan(int kind, int n, int batch, long long idist, cufftHandle* out) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  const PlanKey key{dev, kind, n, batch, idist};
  auto it = g_plans.find(key);
  if (it != g_plans.end()) {
    *out = it->second;
    return 0;
  }
  cufftHandle p;
  int nn = n, emb = n;
  const cufftResult r =
      kind == 0 ? cufftPlanMany(&p, 1, &nn, &emb, 1, int(idist), &emb, 1, n,
                                CUFFT_C2C, batch)
                : cufftPlanMany(&p, 1, &nn, nullptr, 1, n, nullptr, 1, n,
                                CUFFT_C2C, batch);
  if (r != CUFFT_SUCCESS) return OLSB_E_BAD_ARG;
  g_plans[key] = p;
  *out = p;
  return 0;
}

int grid_for(long long work) {
  return int(std::max<long long>(1, std::min<long long>((work + 255) / 256, 148 * 16)));
}

// working-set sizing: segment chunk and filter chunk (env-tunable)
long long env_ll(const char* name, long long dflt) {
  const char* e = getenv(name);
  return e ? atoll(e) : dflt;
}

}  // namespace

extern "C" {

// complex elements reserved for a chunk's padded input span (a multiple of
// 32, so X and Y that follow stay 256-byte aligned for the float4 kernels)
static long long span_alloc(long long sc, long long L, int n) {
  return ((sc * L + n) + 31) / 32 * 32;
}

// segments per chunk and filters per inverse launch for length n
static void chunking(int n, int n_fil, long long nseg, long long* sc, int* fc) {
  // X chunk 16 MiB (L2-resident while every filter reads it), product chunk
  // up to 1 GiB: measured on cfg3 / cfg2 N=1024 over {16, 64, 256} MiB x
  // {32, 256, 1024} MiB (profiles/r02_cufft_chunks.log), cuFFT launch count
  // matters more than keeping the product in L2 (cfg3: 11.9 ms at 32 MiB,
  // 8.3 ms at 1 GiB)
  *sc = std::min(nseg, std::max(1LL, env_ll("OLSB_CUFFT_XCHUNK", 16LL << 20) / (8LL * n)));
  *fc = int(std::max(1LL, std::min<long long>(
      n_fil, env_ll("OLSB_CUFFT_YCHUNK", 1LL << 30) / (8LL * n * *sc))));
}

// workspace bytes for olsb_cufft_ols_c2c (pad span + X + product)
size_t olsb_cufft_ols_workspace(int64_t n_s, int n_fil, int n, int m) {
  if (n < 4 || m < 1 || m > n || n_s < 1 || n_fil < 1) return 0;
  const long long L = n - m + 1, nseg = (n_s + L - 1) / L;
  long long sc;
  int fc;
  chunking(n, n_fil, nseg, &sc, &fc);
  return size_t(span_alloc(sc, L, n)) * 8 + size_t(sc) * n * 8 +
         size_t(fc) * sc * n * 8;
}

// out[f, g] for g in [0, n_s): c2c, the reference's plan geometry (L = n - m
// + 1, t0 = m - 1, window offset origin - (m - 1)).  spectra: natural-order
// filter spectra [n_fil][n] (fft of the zero-padded taps).  work:
// olsb_cufft_ols_workspace bytes of device memory (16-byte aligned).
int olsb_cufft_ols_c2c(const void* x, int64_t n_s, const void* spectra,
                       int n_fil, int n, int m, int origin, void* out,
                       int64_t out_ld, void* work, void* stream) {
  if (n < 4 || n > 16384 || (n & (n - 1)) || m < 1 || m > n || origin < 0 ||
      origin >= m || n_s < 1 || n_fil < 1 || !x || !spectra || !out || !work)
    return OLSB_E_BAD_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long long L = n - m + 1;
  const long long nseg = (n_s + L - 1) / L;
  const long long win_off = origin - (m - 1);
  long long sc;
  int fc;
  chunking(n, n_fil, nseg, &sc, &fc);
  float2* xs = static_cast<float2*>(work);
  float2* X = xs + span_alloc(sc, L, n);
  float2* Y = X + sc * n;
  const float scale = 1.0f / float(n);
  for (long long s0 = 0; s0 < nseg; s0 += sc) {
    const long long ns_c = std::min(sc, nseg - s0);
    const long long span = (ns_c - 1) * L + n;
    pad_kernel<<<grid_for(span), 256, 0, st>>>(static_cast<const float2*>(x),
                                               n_s, s0 * L + win_off, span, xs);
    cufftHandle fwd;
    if (int rc = get_plan(0, n, int(ns_c), L, &fwd)) return rc;
    cufftSetStream(fwd, st);
    if (cufftExecC2C(fwd, reinterpret_cast<cufftComplex*>(xs),
                     reinterpret_cast<cufftComplex*>(X), CUFFT_FORWARD) !=
        CUFFT_SUCCESS)
      return OLSB_E_BAD_ARG;
    for (int f0 = 0; f0 < n_fil; f0 += fc) {
      const int nf = std::min(fc, n_fil - f0);
      multiply_kernel<<<grid_for(nf * ns_c * n / 2), 256, 0, st>>>(
          reinterpret_cast<const float4*>(X),
          reinterpret_cast<const float4*>(spectra), f0, nf, ns_c, n / 2,
          reinterpret_cast<float4*>(Y));
      cufftHandle inv;
      if (int rc = get_plan(1, n, int(nf * ns_c), n, &inv)) return rc;
      cufftSetStream(inv, st);
      if (cufftExecC2C(inv, reinterpret_cast<cufftComplex*>(Y),
                       reinterpret_cast<cufftComplex*>(Y), CUFFT_INVERSE) !=
          CUFFT_SUCCESS)
        return OLSB_E_BAD_ARG;
      store_kernel<<<grid_for(nf * ns_c * L), 256, 0, st>>>(
          Y, f0, nf, s0, ns_c, n, m - 1, L, n_s, scale,
          static_cast<float2*>(out), out_ld);
    }
  }
  return int(cudaGetLastError());
}

}  // extern "C"
