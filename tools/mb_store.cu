// Store-pattern microbenchmark for the OLS output writes (no FFT).
// Each CTA (128 threads) writes, per (segment, filter), L valid samples of
// out[f][s*L + o].  Modes vary what the fused kernel could do differently.
#include <cstdio>
#include <cuda_runtime.h>
// mode 0: fused pattern: p = t + 128 e (16 x 8 B per thread), o = p - t0
// mode 2: 16-byte stores: thread writes o = 2 t + 256 e, o + 1 (8 x 16 B)
template <int MODE>
__global__ void __launch_bounds__(128, 4) k(float2* out, long long ns, int L,
                                            int t0, int nseg, int F, long long ld) {
  int t = threadIdx.x;
  for (int s = blockIdx.x; s < nseg; s += gridDim.x) {
    long long g0 = (long long)s * L;
    unsigned span = (unsigned)min((long long)L, ns - g0);
    for (int f = 0; f < F; ++f) {
      if (MODE == 0) {
        float2* row = out + (long long)f * ld + g0 + t - t0;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          unsigned o = t + 128 * e - t0;
          if (o < span) __stcs(row + 128 * e, make_float2(s + e, f + t));
        }
      } else {
        float2* row = out + (long long)f * ld + g0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          unsigned o = 2 * t + 256 * e;
          if (o + 1 < span) __stcs(reinterpret_cast<float4*>(row + o), make_float4(s, e, f, t));
          else if (o < span) __stcs(row + o, make_float2(s, e));
        }
      }
    }
  }
}
int main() {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  long long total = (1LL << 23) * 96;
  float2* out; cudaMalloc(&out, total * 8 + 4096);
  struct Case { const char* name; long long ns; int F; int L; int mode; int grid; };
  Case cases[] = {
    {"fused F=96 L=1649 p592", 1 << 23, 96, 1649, 0, 592},
    {"fused F=96 L=1649 g5088", 1 << 23, 96, 1649, 0, 5088},
    {"one row L=1649 g5088", total, 1, 1649, 0, 1 << 20},
    {"F=96 L=2048 aligned g4096", 1 << 23, 96, 2048, 0, 4096},
    {"F=96 L=1649 16B g5088", 1 << 23, 96, 1649, 2, 5088},
    {"F=96 L=1648 16B g5091", 1 << 23, 96, 1648, 2, 5091},
    {"F=96 L=2048 16B g4096", 1 << 23, 96, 2048, 2, 4096},
  };
  for (auto& c : cases) {
    int nseg = int((c.ns + c.L - 1) / c.L);
    int t0 = 2048 - c.L;
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(a);
      if (c.mode == 0) k<0><<<c.grid, 128>>>(out, c.ns, c.L, t0, nseg, c.F, c.ns);
      else k<2><<<c.grid, 128>>>(out, c.ns, c.L, t0, nseg, c.F, c.ns);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (w) printf("%-28s %.3f ms  %.0f GB/s\n", c.name, ms, c.ns * c.F * 8 / ms / 1e6);
    }
  }
  cudaEventRecord(a); cudaMemsetAsync(out, 0, total * 8); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); printf("memset                       %.3f ms  %.0f GB/s\n", ms, total * 8 / ms / 1e6);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
