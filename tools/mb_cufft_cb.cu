// Diagnostic: does a batched C2C inverse with load + store callbacks write
// its odata buffer?  (sentinel check; built and run on the GPU box:
// nvcc -rdc=true ... -lcufft_static -lculibos)
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include <cufft.h>
#include <cufftXt.h>

struct P { const float2* X; int logn; };
__device__ cufftComplex ld(void*, size_t off, void* info, void*) {
  const P* p = (const P*)info;
  return p->X[off & ((1u << p->logn) - 1)];
}
__device__ void st(void* out, size_t off, cufftComplex v, void* info, void*) {
  // drop everything
}
__device__ cufftCallbackLoadC d_ld = ld;
__device__ cufftCallbackStoreC d_st = st;

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  for (int n : {64, 256, 2048, 4096}) {
    for (int batch : {16, 4096, 65536}) {
      cufftHandle plan; cufftCreate(&plan);
      size_t ws; cufftMakePlanMany(plan, 1, &n, nullptr, 1, n, nullptr, 1, n, CUFFT_C2C, batch, &ws);
      P hp; float2* X; cudaMalloc(&X, n * 8); cudaMemset(X, 0, n * 8);
      hp.X = X; int logn = 0; while ((1 << logn) < n) ++logn; hp.logn = logn;
      P* dp; cudaMalloc(&dp, sizeof(P)); cudaMemcpy(dp, &hp, sizeof(P), cudaMemcpyHostToDevice);
      cufftCallbackLoadC hl; cufftCallbackStoreC hs;
      cudaMemcpyFromSymbol(&hl, d_ld, sizeof(hl)); cudaMemcpyFromSymbol(&hs, d_st, sizeof(hs));
      void* info[1] = {dp};
      int r1 = cufftXtSetCallback(plan, (void**)&hl, CUFFT_CB_LD_COMPLEX, info);
      int r2 = cufftXtSetCallback(plan, (void**)&hs, CUFFT_CB_ST_COMPLEX, info);
      size_t tot = size_t(n) * batch;
      float2 *in, *out; cudaMalloc(&in, tot * 8); cudaMalloc(&out, tot * 8);
      cudaMemset(in, 0xff, tot * 8); cudaMemset(out, 0xff, tot * 8);
      int r3 = cufftExecC2C(plan, in, out, CUFFT_INVERSE);
      cudaDeviceSynchronize();
      std::vector<unsigned> hi(tot * 2), ho(tot * 2);
      cudaMemcpy(hi.data(), in, tot * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(ho.data(), out, tot * 8, cudaMemcpyDeviceToHost);
      size_t wi = 0, wo = 0;
      for (size_t i = 0; i < tot * 2; ++i) { wi += hi[i] != 0xffffffffu; wo += ho[i] != 0xffffffffu; }
      printf("n=%d batch=%d setcb=%d,%d exec=%d err=%s  in words changed %zu / %zu, out words changed %zu\n",
             n, batch, r1, r2, r3, cudaGetErrorString(cudaGetLastError()), wi, tot * 2, wo);
      cufftDestroy(plan); cudaFree(in); cudaFree(out); cudaFree(X); cudaFree(dp);
    }
  }
  return 0;
}
