// Store-only patterns at the fused kernel's occupancy (4 x 128-thread CTAs
// per SM, 16 samples per thread per row of 2048 complex).
//  P0: element e of thread t -> row[e*128 + t]        (fused kernel today)
//  P1: warp-contiguous: warp w writes row[512w + 32e + lane]
//  P2: as P0 but v4 stores of pairs (lane owns 2 adjacent samples)
//  P3: as P0 with st.global (write-back) instead of .cs
#include <cstdio>
#include <cuda_runtime.h>
template <int P>
__global__ void __launch_bounds__(128, 4) k(float2* out, long long rows) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
    float2* row = out + r * 2048;
    if (P == 0 || P == 3) {
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        float2* p = row + e * 128 + t;
        if (P == 0)
          asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(1.f), "f"(2.f) : "memory");
        else
          asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(1.f), "f"(2.f) : "memory");
      }
    } else if (P == 1) {
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        float2* p = row + 512 * w + 32 * e + lane;
        asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(1.f), "f"(2.f) : "memory");
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float4* p = reinterpret_cast<float4*>(row + e * 256 + 2 * t);
        asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(2.f), "f"(3.f), "f"(4.f) : "memory");
      }
    }
  }
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long rows = 5141LL * 96;
  float2* out;
  cudaMalloc(&out, rows * 2048 * sizeof(float2));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* nm, auto kern, int per) {
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      kern<<<sms * per, 128>>>(out, rows);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("%-40s %d CTA/SM  %.3f ms  %.0f GB/s\n", nm, per, ms, rows * 2048 * 8.0 / ms / 1e6);
  };
  for (int per : {4, 8}) {
    run("P0 e*128+t st.cs.v2 (kernel today)", k<0>, per);
    run("P1 warp-contiguous st.cs.v2", k<1>, per);
    run("P2 pairs st.cs.v4", k<2>, per);
    run("P3 e*128+t st.v2 (write-back)", k<3>, per);
  }
  return 0;
}
