// FP32 pipe microbenchmark: scalar FFMA vs packed FFMA2 vs a mix.
// Reports lane-ops (one fp32 FMA/add per lane) per SM-clock.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
template <int MODE>
__global__ void k(float* out, int iters, float s) {
  float a[16];
  u64 b[8];
  for (int i = 0; i < 16; i++) a[i] = threadIdx.x * 0.001f + i;
  for (int i = 0; i < 8; i++) b[i] = (u64)__float_as_uint(i * 0.5f) | ((u64)__float_as_uint(i * 0.25f) << 32);
  const u64 ss = (u64)__float_as_uint(s) | ((u64)__float_as_uint(s) << 32);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i++) {
      if (MODE == 0) a[i] = fmaf(a[i], s, a[(i + 3) & 15]);          // 16 FFMA
      if (MODE == 1) { if (i < 8) b[i] = fma2(b[i], ss, b[(i + 3) & 7]); }  // 8 FFMA2
      if (MODE == 2) {  // 8 FFMA2 + 16 FFMA, independent
        if (i < 8) b[i] = fma2(b[i], ss, b[(i + 3) & 7]);
        a[i] = fmaf(a[i], s, a[(i + 3) & 15]);
      }
      if (MODE == 3) {  // 8 FFMA2 + 8 FFMA
        if (i < 8) b[i] = fma2(b[i], ss, b[(i + 3) & 7]);
        if (i & 1) a[i] = fmaf(a[i], s, a[(i + 3) & 15]);
      }
    }
  }
  float r = 0;
  for (int i = 0; i < 16; i++) r += a[i];
  for (int i = 0; i < 8; i++) r += __uint_as_float((unsigned)b[i]) + __uint_as_float((unsigned)(b[i] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, sms * 4 * 512 * 4);
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double lane_ops_per_it[4] = {16, 16, 32, 24};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<sms * 4, 512>>>(out, iters, 1.0001f);
      if (mode == 1) k<1><<<sms * 4, 512>>>(out, iters, 1.0001f);
      if (mode == 2) k<2><<<sms * 4, 512>>>(out, iters, 1.0001f);
      if (mode == 3) k<3><<<sms * 4, 512>>>(out, iters, 1.0001f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double ops = double(sms) * 4 * 512 * iters * lane_ops_per_it[mode];
      if (rep)
        printf("mode %d: %.3f ms  %.1f lane-ops/clk/SM (clock %d MHz)\n", mode, ms,
               ops / sms / (ms * 1e-3 * clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
