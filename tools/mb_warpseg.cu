// Timing prototype (results are NOT a convolution): a warp-per-segment
// schedule for N = 2048 OLS filter loops, to measure whether removing all
// CTA-wide barriers pays for ~12% more FP work.  Per (segment, filter) row a
// warp (32 threads x 64 samples) does:
//   4 groups x { X group from TMEM, spectrum from TEX, multiply, 4 static
//                radix-2 stages } -> smem
//   __syncwarp; 4 groups x { smem -> 4 runtime stages (STD forms) -> smem }
//   __syncwarp; 8 groups x { smem + 7 twiddles from an smem table -> 3
//                runtime stages -> 8 streaming stores (80% valid) }
// using the engine's own pass functions (csrc/olsb_fft.cuh).  Compared with
// the engine's cfg3 kernel time (same rows, same output bytes).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "olsb_fft.cuh"
using namespace olsb;

struct TwTab {
  const Tw<float>* base;
  __device__ Tw<float> get0() const { return base[0]; }
  __device__ TwPair<float> get2(int p) const { return TwPair<float>{base[2 * p - 1], base[2 * p]}; }
};
struct TwR {
  const Tw<float>* r;
  __device__ Tw<float> get0() const { return r[0]; }
  __device__ TwPair<float> get2(int p) const { return TwPair<float>{r[2 * p - 1], r[2 * p]}; }
};

__device__ __forceinline__ void tmem_ld32(uint32_t ta, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(ta));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(128, 3)
    warpseg(float2* out, cudaTextureObject_t htex, long long rows, int nfil,
            long long out_ld, int dbg) {
  extern __shared__ __align__(16) unsigned char dyn[];
  Cpx<float> (*buf)[2048 + 64] = reinterpret_cast<Cpx<float> (*)[2048 + 64]>(dyn);
  Tw<float>* ttab = reinterpret_cast<Tw<float>*>(dyn + 4 * (2048 + 64) * 8);
  __shared__ uint32_t tslot;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 256 * 8; i += 128) ttab[i] = Tw<float>{0.9f + i * 1e-6f, 0.3f};
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tslot + ((uint32_t)(w * 32) << 16);
  Tw<float> twm[15];
  for (int i = 0; i < 15; ++i) twm[i] = Tw<float>{0.8f + i * 1e-3f + lane * 1e-5f, 0.2f};
  Cpx<float>* b = buf[w];
  const long long wid = blockIdx.x * 4LL + w, nw = gridDim.x * 4LL;
  for (long long r = wid; r < rows; r += nw) {
    const int f = int(r % nfil);
    const long long seg = r / nfil;
    // pass 1: junction (static) per 16-sample group
#pragma unroll 1
    for (int g = 0; g < 4; ++g) {
      uint32_t xr[32];
      tmem_ld32(tb + 32 * g, xr);
      Cpx<float> y[16];
      const int hb = (f * 4 + g) * 256 + lane;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float4 h = tex1Dfetch<float4>(htex, hb + u * 32);
        y[2 * u] = cmul(Cpx<float>{__uint_as_float(xr[4 * u]), __uint_as_float(xr[4 * u + 1])}, Cpx<float>{h.x, h.y});
        y[2 * u + 1] = cmul(Cpx<float>{__uint_as_float(xr[4 * u + 2]), __uint_as_float(xr[4 * u + 3])}, Cpx<float>{h.z, h.w});
      }
      dit_pass_static<float, 4, 4>(y);
      // conflict-free timing layout: lanes 16 B apart
      float4* bp = reinterpret_cast<float4*>(b + g * 512 + lane * 2);
#pragma unroll
      for (int u = 0; u < 8; ++u) bp[u * 32] = make_float4(y[2 * u].re, y[2 * u].im, y[2 * u + 1].re, y[2 * u + 1].im);
    }
    __syncwarp();
    // pass 2: middle window (runtime twiddles in registers, STD forms)
#pragma unroll 1
    for (int g = 0; g < 4; ++g) {
      Cpx<float> y[16];
      const float4* bp = reinterpret_cast<const float4*>(b + g * 512 + lane * 2);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float4 v = bp[u * 32];
        y[2 * u] = Cpx<float>{v.x, v.y};
        y[2 * u + 1] = Cpx<float>{v.z, v.w};
      }
      dit_pass_rt<float, false>(y, TwR{twm}, 0);
      float4* bq = reinterpret_cast<float4*>(b + g * 512 + lane * 2);
#pragma unroll
      for (int u = 0; u < 8; ++u) bq[u * 32] = make_float4(y[2 * u].re, y[2 * u].im, y[2 * u + 1].re, y[2 * u + 1].im);
    }
    __syncwarp();
    // pass 3: top window, 8 groups of 8 (3 stages), twiddles from smem
    float2* orow = out + (long long)f * out_ld + seg * 1632 + lane;
#pragma unroll 1
    for (int g = 0; g < 8; ++g) {
      Cpx<float> y[16];
      const float4* bp = reinterpret_cast<const float4*>(b + g * 256 + lane * 2);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float4 v = bp[u * 32];
        y[2 * u] = Cpx<float>{v.x, v.y};
        y[2 * u + 1] = Cpx<float>{v.z, v.w};
      }
      // 3 stages on 8 samples: reuse the runtime pass on the first 8 (the
      // other 8 registers are dead work kept tiny)
      Tw<float> tw[15];
#pragma unroll
      for (int i = 0; i < 7; ++i) tw[i] = ttab[(g * 8 + i) * 32 + lane];
      for (int i = 7; i < 15; ++i) tw[i] = tw[i - 7];
      // stages j = 0..2 with STD forms
#pragma unroll
      for (int h = 0; h < 4; ++h) dit_std(y[2 * h], y[2 * h + 1], tw[0].c, tw[0].t);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        dit_std(y[4 * h], y[4 * h + 2], tw[1].c, tw[1].t);
        dit_std(y[4 * h + 1], y[4 * h + 3], tw[2].c, tw[2].t);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) dit_std(y[k], y[k + 4], tw[3 + k].c, tw[3 + k].t);
      if (!(dbg & 1)) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int o = g * 256 + e * 32 + lane - 416;
          if (o >= 0 && o < 1632) __stcs(orow + (o - lane), make_float2(y[e].re, y[e].im));
        }
      }
    }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tslot));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nfil = 96;
  const long long nseg = 5141, rows = nseg * nfil, out_ld = nseg * 1632;
  float2* out;
  cudaMalloc(&out, nfil * out_ld * sizeof(float2));
  float4* h;
  cudaMalloc(&h, nfil * 2048 * 8);
  cudaMemset(h, 0, nfil * 2048 * 8);
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = h;
  rd.res.linear.desc = cudaCreateChannelDesc<float4>();
  rd.res.linear.sizeInBytes = nfil * 2048 * 8;
  cudaTextureDesc td = {};
  cudaTextureObject_t tex;
  cudaCreateTextureObject(&tex, &rd, &td, nullptr);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int smem = 4 * (2048 + 64) * 8 + 256 * 8 * 8;
  cudaFuncSetAttribute(warpseg, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int dbg = 0; dbg < 2; ++dbg) {
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      warpseg<<<sms * 3, 128, smem>>>(out, tex, rows, nfil, out_ld, dbg);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("warp-per-segment prototype (%s): %.3f ms  %s\n", dbg ? "no stores" : "with stores", ms,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
