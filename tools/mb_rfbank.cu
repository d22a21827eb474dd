// FFMA2 throughput vs operand register pattern (RF bank reads): 
//  A: d = a * b + c, three distinct 64-bit register pairs
//  B: d = a * s + c, s a 32-bit scalar broadcast to both halves
//  C: d = a * s + a, repeated operand
//  D: scalar FFMA with three distinct registers (same lane-ops as A)
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 fma2s(u64 a, float s, u64 c) {
  u64 d;
  asm volatile("{ .reg .b64 t; mov.b64 t, {%2, %2}; fma.rn.f32x2 %0, %1, t, %3; }"
               : "=l"(d) : "l"(a), "f"(s), "l"(c));
  return d;
}
template <int MODE>
__global__ void __launch_bounds__(128, 4) k(float* out, int iters, float sc) {
  u64 a[8], b[8], c[8];
  float fa[16], fb[16], fc[16];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x + i; b[i] = threadIdx.x * 3 + i + 1; c[i] = threadIdx.x * 7 + i + 5; }
  for (int i = 0; i < 16; ++i) { fa[i] = i; fb[i] = 2 * i + 1; fc[i] = 3 * i; }
  const float s = sc;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = fma2(a[i], b[i], c[i]);
      if (MODE == 1) a[i] = fma2s(a[i], s, c[i]);
      if (MODE == 2) a[i] = fma2s(a[i], s, a[i]);
      // E: the butterfly's u + c*P: pair, per-thread (vector) scalar, pair
      if (MODE == 4) a[i] = fma2s(a[i], __uint_as_float((unsigned)b[i]), c[i]);
    }
    if (MODE == 5) {  // the same lane-ops as E as scalar FFMAs
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float cc = __uint_as_float((unsigned)b[i]);
        fa[2 * i] = fmaf(fa[2 * i], cc, fc[2 * i]);
        fa[2 * i + 1] = fmaf(fa[2 * i + 1], cc, fc[2 * i + 1]);
      }
    }
    if (MODE == 3) {
#pragma unroll
      for (int i = 0; i < 16; ++i) fa[i] = fmaf(fa[i], fb[i], fc[i]);
    }
  }
  float r = 0;
  for (int i = 0; i < 8; ++i) r += __uint_as_float((unsigned)a[i]) + __uint_as_float((unsigned)c[i]) + __uint_as_float((unsigned)b[i]);
  for (int i = 0; i < 16; ++i) r += fa[i] + fb[i] + fc[i];
  out[blockIdx.x * 128 + threadIdx.x] = r;
}
int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, sms * 16 * 128 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 40000;
  const char* names[6] = {"A FFMA2 3 distinct pairs", "B FFMA2 a*s+c (uniform s)",
                          "C FFMA2 a*s+a", "D FFMA 3 distinct",
                          "E FFMA2 P*c+U (vector c)", "F 2x FFMA P*c+U (vector c)"};
  for (int mode = 0; mode < 6; ++mode) {
    for (int per : {4, 8}) {
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k<0><<<sms * per, 128>>>(out, iters, 1.0001f);
        if (mode == 1) k<1><<<sms * per, 128>>>(out, iters, 1.0001f);
        if (mode == 2) k<2><<<sms * per, 128>>>(out, iters, 1.0001f);
        if (mode == 3) k<3><<<sms * per, 128>>>(out, iters, 1.0001f);
        if (mode == 4) k<4><<<sms * per, 128>>>(out, iters, 1.0001f);
        if (mode == 5) k<5><<<sms * per, 128>>>(out, iters, 1.0001f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      const double lane_ops = double(sms) * per * 128 * iters * 16;
      printf("%-30s %d CTA/SM: %.1f lane-ops/clk/SM\n", names[mode], per,
             lane_ops / sms / (ms * 1e-3 * clk * 1e3));
    }
  }
  return 0;
}
