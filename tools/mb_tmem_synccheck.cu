// Minimal repro for compute-sanitizer --tool synccheck on tensor-memory
// kernels.  Every kernel follows the documented protocol (warp 0 allocates,
// relinquish, fence::before_thread_sync / bar.sync / fence::after_thread_sync,
// use, fence / bar.sync, warp 0 deallocates); the plain kernel does the same
// slot hand-off through shared memory without tcgen05.
//   ./mb_tmem_synccheck <0|1|2>   0 plain smem, 1 alloc+dealloc, 2 alloc+st+ld
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int MODE>
__global__ void k(uint32_t* out) {
  __shared__ uint32_t slot[4];
  const int w = threadIdx.x / 32;
  if (MODE == 0) {
    if (threadIdx.x == 0) slot[1] = 42u;
    __syncthreads();
    out[blockIdx.x * blockDim.x + threadIdx.x] = slot[1];
    return;
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;"
                 ::"r"(su32(&slot[1])) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = slot[1];
  uint32_t v = threadIdx.x;
  if (MODE == 2) {
    const uint32_t ta = base + (uint32_t(w * 32) << 16);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta), "r"(v) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = v;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(base) : "memory");
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 2;
  uint32_t* out;
  cudaMalloc(&out, 4 * 128 * sizeof(uint32_t));
  if (mode == 0) k<0><<<4, 128>>>(out);
  if (mode == 1) k<1><<<4, 128>>>(out);
  if (mode == 2) k<2><<<4, 128>>>(out);
  const cudaError_t e = cudaDeviceSynchronize();
  uint32_t h[128];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  printf("mode %d: %s, out[5] = %u\n", mode, cudaGetErrorString(e), h[5]);
  return 0;
}
