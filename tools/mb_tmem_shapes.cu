// Microbenchmark / decoder: which (TMEM lane, column) word each thread
// receives from the 16-lane tcgen05.ld shapes, after every thread of a warp
// stored its own 32 words with tcgen05.st.32x32b.x32 (word = lane*100+col).
// Used to build warp-local exchanges out of TMEM round trips.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o mb_tmem_shapes tools/mb_tmem_shapes.cu
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
      "r"(r[29]), "r"(r[30]), "r"(r[31]));
}

// 16x256b.x4: 16 registers (lanes base..base+15, columns 0..31)
__device__ __forceinline__ void ld_16x256b_x4(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : R4(0), R4(4), R4(8), R4(12)
      : "r"(taddr));
}
// 16x128b.x8: 16 registers
__device__ __forceinline__ void ld_16x128b_x8(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x128b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : R4(0), R4(4), R4(8), R4(12)
      : "r"(taddr));
}
// 16x64b.x16: 16 registers
__device__ __forceinline__ void ld_16x64b_x16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x64b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : R4(0), R4(4), R4(8), R4(12)
      : "r"(taddr));
}
// 16x32bx2.x16: 16 registers, second half at column offset 16
__device__ __forceinline__ void ld_16x32bx2_x16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16], 16;"
      : R4(0), R4(4), R4(8), R4(12)
      : "r"(taddr));
}

template <int SHAPE>
__global__ void __launch_bounds__(128) decode(uint32_t* out) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr_s + ((uint32_t)(warp * 32) << 16);
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = uint32_t(lane * 100 + i);
  st32(base, r);
  asm volatile("tcgen05.wait::st.sync.aligned;");
  uint32_t v[32];
  // two 16-lane halves: lane field +0 and +16
  for (int h = 0; h < 2; ++h) {
    const uint32_t a = base + ((uint32_t)(16 * h) << 16);
    if (SHAPE == 0) ld_16x256b_x4(a, v + 16 * h);
    if (SHAPE == 1) ld_16x128b_x8(a, v + 16 * h);
    if (SHAPE == 2) ld_16x64b_x16(a, v + 16 * h);
    if (SHAPE == 3) ld_16x32bx2_x16(a, v + 16 * h);
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  if (warp == 0)
    for (int i = 0; i < 32; ++i) out[lane * 32 + i] = v[i];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(taddr_s));
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 32 * 32 * 4);
  uint32_t h[32 * 32];
  const char* names[4] = {"16x256b.x4", "16x128b.x8", "16x64b.x16", "16x32bx2.x16(off16)"};
  for (int s = 0; s < 4; ++s) {
    cudaMemset(d, 0xff, sizeof(h));
    if (s == 0) decode<0><<<1, 128>>>(d);
    if (s == 1) decode<1><<<1, 128>>>(d);
    if (s == 2) decode<2><<<1, 128>>>(d);
    if (s == 3) decode<3><<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("== %s (%s): thread: reg -> lane.col\n", names[s], cudaGetErrorString(e));
    for (int t = 0; t < 32; ++t) {
      printf("t%02d:", t);
      for (int i = 0; i < 32; ++i) printf(" %d.%d", h[t * 32 + i] / 100, h[t * 32 + i] % 100);
      printf("\n");
    }
  }
  return 0;
}
