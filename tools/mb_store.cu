// Write-bandwidth microbenchmark for the OLS output stream: every warp writes
// aligned 256-byte chunks (32 lanes x 8 B), like the fused kernel's
// writeback.  Variants: store width / cache policy / TMA bulk store.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(128) wr(float2* out, long long n2, int iters) {
  // grid-stride over 256-B chunks; 16 chunks per warp per iteration like the
  // kernel's 16 stores per filter
  const long long nch = n2 / 32;
  const int lane = threadIdx.x & 31;
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32;
  const long long nw = (gridDim.x * (long long)blockDim.x) / 32;
  float2 v = make_float2(lane * 1.f, 2.f);
  for (long long c = w; c < nch; c += nw) {
    float2* p = out + c * 32 + lane;
    if (MODE == 0) {
      asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
    } else if (MODE == 1) {
      asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
    } else if (MODE == 2) {
      asm volatile("st.global.L1::no_allocate.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
    }
  }
}
// v4: each lane writes 16 B (two warps' worth of chunks per instruction)
__global__ void __launch_bounds__(128) wr4(float4* out, long long n4) {
  const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long st = gridDim.x * (long long)blockDim.x;
  for (long long i = i0; i < n4; i += st) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(out + i), "f"(1.f), "f"(2.f), "f"(3.f), "f"(4.f) : "memory");
  }
}
// TMA bulk store: each CTA writes 8 KB tiles from shared memory
__global__ void __launch_bounds__(128) wr_tma(char* out, long long bytes) {
  __shared__ __align__(128) float4 tile[512];  // 8 KB
  for (int i = threadIdx.x; i < 512; i += 128) tile[i] = make_float4(1, 2, 3, 4);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long ntile = bytes / 8192;
    for (long long tt = blockIdx.x; tt < ntile; tt += gridDim.x) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 8192;" ::"l"(out + tt * 8192),
                   "r"((uint32_t)__cvta_generic_to_shared(tile)) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long bytes = 6442450944LL;  // cfg3 output: 96 x 2^23 x 8 B
  char* buf;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("%-34s %.3f ms  %.0f GB/s  %s\n", name, ms, bytes / ms / 1e6,
                           cudaGetErrorString(cudaGetLastError()));
    }
  };
  const long long n2 = bytes / 8;
  for (int per : {4, 8, 16}) {
    char nm[64];
    snprintf(nm, 64, "st.cs.v2   %2d CTA/SM", per);
    run(nm, [&] { wr<0><<<sms * per, 128>>>((float2*)buf, n2, 1); });
    snprintf(nm, 64, "st.v2      %2d CTA/SM", per);
    run(nm, [&] { wr<1><<<sms * per, 128>>>((float2*)buf, n2, 1); });
    snprintf(nm, 64, "st.noalloc %2d CTA/SM", per);
    run(nm, [&] { wr<2><<<sms * per, 128>>>((float2*)buf, n2, 1); });
    snprintf(nm, 64, "st.cs.v4   %2d CTA/SM", per);
    run(nm, [&] { wr4<<<sms * per, 128>>>((float4*)buf, bytes / 16); });
  }
  run("tma bulk 8KB x 16 CTA/SM", [&] { wr_tma<<<sms * 16, 128>>>(buf, bytes); });
  run("cudaMemsetAsync", [&] { cudaMemsetAsync(buf, 0, bytes); });
  return 0;
}
