// LTO callback routines for tools/mb_cufft_cb2.cu
#include <cufftXt.h>
struct P { const float2* X; int logn; };
extern "C" __device__ cufftComplex ld_lto(void*, unsigned long long off, void* info, void*) {
  const P* p = (const P*)info;
  return p->X[off & ((1ull << p->logn) - 1)];
}
extern "C" __device__ void st_lto(void*, unsigned long long, cufftComplex, void*, void*) {}
