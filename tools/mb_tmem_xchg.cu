// Microbenchmark: a warp-local 16-complex-per-thread exchange through TMEM
// round trips (tcgen05.st.32x32b + tcgen05.ld.16x256b / 16x32bx2, 3 trips as
// the N = 2048 first inverse exchange needs) against the same exchange
// through shared memory (8 x STS.128, __syncwarp, 8 x LDS.128), each between
// blocks of packed-FP work, at 4 CTAs x 4 warps per SM like the fused engine.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/mb_tmem_xchg tools/mb_tmem_xchg.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define R4(b) "=r"(r[b]), "=r"(r[b + 1]), "=r"(r[b + 2]), "=r"(r[b + 3])

__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void ld_a(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : R4(0), R4(4), R4(8), R4(12)
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void ld_d(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16], 16;"
      : R4(0), R4(4), R4(8), R4(12)
      : "r"(taddr)
      : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(128, 4) k(float* out, int iters, int fpw) {
  extern __shared__ float4 sm[];
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr_s + ((uint32_t)(warp * 32) << 16) + 96;  // scratch cols
  float2 x[16];
  for (int i = 0; i < 16; ++i) x[i] = make_float2(lane * 0.01f + i, i * 0.5f);
  float4* wb = sm + warp * 32 * 9;  // per-warp region, padded
  for (int it = 0; it < iters; ++it) {
    // FP block: fpw rounds of 16 packed FMAs
    for (int j = 0; j < fpw; ++j)
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        x[i].x = fmaf(x[i].x, 0.999f, x[(i + 1) & 15].y);
        x[i].y = fmaf(x[i].y, 0.999f, x[(i + 3) & 15].x);
      }
    if (MODE == 1) {  // shared memory, warp-local
#pragma unroll
      for (int i = 0; i < 8; ++i)
        wb[i * 36 + lane] = make_float4(x[2 * i].x, x[2 * i].y, x[2 * i + 1].x, x[2 * i + 1].y);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 v = wb[((i + lane) & 7) * 36 + (lane ^ i)];
        x[2 * i] = make_float2(v.x, v.y);
        x[2 * i + 1] = make_float2(v.z, v.w);
      }
      __syncwarp();
    } else if (MODE == 2) {  // TMEM: three round trips (A, A, D)
#pragma unroll
      for (int trip = 0; trip < 3; ++trip) {
        uint32_t r[32];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          r[2 * i] = __float_as_uint(x[i].x);
          r[2 * i + 1] = __float_as_uint(x[i].y);
        }
        st32(base, r);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        if (trip < 2) {
          ld_a(base, r);
          ld_a(base + (16u << 16), r + 16);
        } else {
          ld_d(base, r);
          ld_d(base + (16u << 16), r + 16);
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 16; ++i)
          x[i] = make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
      }
    }
  }
  float s = 0;
  for (int i = 0; i < 16; ++i) s += x[i].x + x[i].y;
  out[blockIdx.x * 128 + threadIdx.x] = s;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(taddr_s));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = 4 * sms, iters = 2000;
  float* out;
  cudaMalloc(&out, grid * 128 * 4);
  const int smem = 4 * 32 * 9 * 16;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[3] = {"FP only", "FP + smem exchange", "FP + TMEM 3 trips"};
  for (int fpw : {0, 4, 8}) {
    for (int mode = 0; mode < 3; ++mode) {
      auto run = [&] {
        if (mode == 0) k<0><<<grid, 128, smem>>>(out, iters, fpw);
        if (mode == 1) k<1><<<grid, 128, smem>>>(out, iters, fpw);
        if (mode == 2) k<2><<<grid, 128, smem>>>(out, iters, fpw);
      };
      run();
      cudaEventRecord(a);
      run();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      // per-SM cycles per warp-exchange at ~1.965 GHz
      const double per = ms * 1e-3 * 1.965e9 / iters;
      printf("fpw %d %-22s %.3f ms  %.0f SM-cycles per iteration (16 warps) [%s]\n", fpw,
             names[mode], ms, per, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
