// Does SHFL share throughput with LDS?  mode 1: LDS.64 x8, 2: SHFL x16 (same bytes), 3: both
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(256) k(float* out, int iters) {
  __shared__ float2 sm[256 * 8 + 64];
  int t = threadIdx.x;
  for (int i = t; i < 256 * 8 + 64; i += 256) sm[i] = make_float2(i, t);
  __syncthreads();
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = t * 0.5f + i;
  float2 acc = make_float2(0, 0);
  for (int it = 0; it < iters; ++it) {
    if (MODE & 1) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float2 v = sm[u * 256 + ((t + it) & 255)];
        acc.x += v.x; acc.y += v.y;
      }
    }
    if (MODE & 2) {
#pragma unroll
      for (int u = 0; u < 16; ++u) a[u] = __shfl_xor_sync(0xffffffffu, a[u], (u + it) & 31) + 1.0f;
    }
  }
  float s = acc.x + acc.y;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * 256 + t] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 4000, grid = 148 * 8;
  for (int mode : {1, 2, 3}) for (int w = 0; w < 2; ++w) {
    cudaEventRecord(a);
    if (mode == 1) k<1><<<grid, 256>>>(out, iters);
    if (mode == 2) k<2><<<grid, 256>>>(out, iters);
    if (mode == 3) k<3><<<grid, 256>>>(out, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (w) printf("mode %d: %.3f ms (LDS 64 B/thr/iter, SHFL 64 B/thr/iter)\n", mode, ms);
  }
}
