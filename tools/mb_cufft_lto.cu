// Diagnostic 3: cuFFT LTO (JIT) callbacks, dynamic libcufft: does the store
// callback replace the odata writes?  usage: mb_cufft_lto <callback fatbin>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <vector>
#include <cuda_runtime.h>
#include <cufft.h>
#include <cufftXt.h>

struct P { const float2* X; int logn; };

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  int ver = 0; cufftGetVersion(&ver); printf("cufft version %d\n", ver);
  std::ifstream f(argv[1], std::ios::binary);
  std::vector<char> fb((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  printf("fatbin %zu bytes\n", fb.size());
  int n = 256, batch = 64;
  float2* X; cudaMalloc(&X, n * 8); cudaMemset(X, 0, n * 8);
  P hp{X, 8}; P* dp; cudaMalloc(&dp, sizeof(P));
  cudaMemcpy(dp, &hp, sizeof(P), cudaMemcpyHostToDevice);
  void* info[1] = {dp};
  cufftHandle plan; printf("create %d\n", cufftCreate(&plan));
  printf("set ld %d\n", cufftXtSetJITCallback(plan, "ld_lto", fb.data(), fb.size(), CUFFT_CB_LD_COMPLEX, info));
  printf("set st %d\n", cufftXtSetJITCallback(plan, "st_lto", fb.data(), fb.size(), CUFFT_CB_ST_COMPLEX, info));
  size_t ws = 0;
  const int pr = cufftMakePlanMany(plan, 1, &n, nullptr, 1, n, nullptr, 1, n, CUFFT_C2C, batch, &ws);
  printf("plan %d\n", pr);
  if (pr != 0) return 1;
  size_t tot = size_t(n) * batch;
  float2 *in, *out; cudaMalloc(&in, tot * 8); cudaMalloc(&out, tot * 8);
  cudaMemset(in, 0xff, tot * 8); cudaMemset(out, 0xff, tot * 8);
  printf("exec %d\n", cufftExecC2C(plan, in, out, CUFFT_INVERSE));
  printf("sync %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<unsigned> ho(tot * 2);
  cudaMemcpy(ho.data(), out, tot * 8, cudaMemcpyDeviceToHost);
  size_t wo = 0;
  for (size_t i = 0; i < tot * 2; ++i) wo += ho[i] != 0xffffffffu;
  printf("out words changed %zu / %zu (0 = store callback replaced the writes)\n", wo, tot * 2);
  return 0;
}
