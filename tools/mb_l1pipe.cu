// Does the TEX path share throughput with LDS (the LSU data pipe)?
// Each kernel runs `iters` rounds per thread of: LDS.64 x8 (mode&1) and/or
// 16-byte loads of L1-resident data via TEX (mode&2) or LDG (mode&4).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(256) k(const float4* __restrict__ g, cudaTextureObject_t tex,
                                         float* out, int iters) {
  __shared__ float2 sm[256 * 8 + 64];
  int t = threadIdx.x;
  for (int i = t; i < 256 * 8 + 64; i += 256) sm[i] = make_float2(i, t);
  __syncthreads();
  float2 acc = make_float2(0, 0);
  float4 acc4 = make_float4(0, 0, 0, 0);
  int base = (blockIdx.x & 7) * 1024;  // 8 x 16 KiB working sets -> L1 hits
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
      for (int u = 0; u < 4; ++u) {
        float4 v = tex1Dfetch<float4>(tex, base + u * 256 + ((t + it) & 255));
        acc4.x += v.x; acc4.w += v.w;
      }
    }
    if (MODE & 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float4 v = __ldg(g + base + u * 256 + ((t + it) & 255));
        acc4.x += v.x; acc4.w += v.w;
      }
    }
  }
  out[blockIdx.x * 256 + t] = acc.x + acc.y + acc4.x + acc4.w;
}
int main() {
  float4* g; cudaMalloc(&g, 8 * 1024 * 16 * 4);
  cudaMemset(g, 0, 8 * 1024 * 16 * 4);
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaResourceDesc rd = {}; rd.resType = cudaResourceTypeLinear; rd.res.linear.devPtr = g;
  rd.res.linear.desc = cudaCreateChannelDesc<float4>(); rd.res.linear.sizeInBytes = 8 * 1024 * 16 * 4;
  cudaTextureDesc td = {}; td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex; cudaCreateTextureObject(&tex, &rd, &td, nullptr);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 4000, grid = 148 * 8;
  const char* names[] = {"", "LDS64x8", "TEX128x4", "LDS+TEX", "LDG128x4", "LDS+LDG"};
  for (int mode : {1, 2, 3, 4, 5}) {
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(a);
      switch (mode) {
        case 1: k<1><<<grid, 256>>>(g, tex, out, iters); break;
        case 2: k<2><<<grid, 256>>>(g, tex, out, iters); break;
        case 3: k<3><<<grid, 256>>>(g, tex, out, iters); break;
        case 4: k<4><<<grid, 256>>>(g, tex, out, iters); break;
        case 5: k<5><<<grid, 256>>>(g, tex, out, iters); break;
      }
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double lds_b = (mode & 1) ? 8.0 * 8 : 0, tex_b = (mode & 6) ? 4.0 * 16 : 0;
      double thr = (double)grid * 256 * iters;
      if (w) printf("%-9s %.3f ms  LDS %.0f GB/s  TEX/LDG %.0f GB/s  (per SM per clk @1.9GHz: %.1f + %.1f B)\n",
                    names[mode], ms, thr * lds_b / ms / 1e6, thr * tex_b / ms / 1e6,
                    thr * lds_b / ms / 1e6 / 148 / 1.9, thr * tex_b / ms / 1e6 / 148 / 1.9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
