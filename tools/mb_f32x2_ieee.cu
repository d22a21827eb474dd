// Are the packed f32x2 ops bit-identical to scalar IEEE round-to-nearest ops?
// Compares mul/add.rn.f32x2 lane by lane with __fmul_rn / __fadd_rn on
// random normals and on denormal inputs, and a mul2 -> add2 chain (which
// ptxas may contract into FFMA2) with the scalar chain.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) {
  u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r;
}
__device__ __forceinline__ void upk(u64 r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 d; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;
}

__global__ void k(const float* x, int n, unsigned* bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i + 3 >= n) return;
  float a = x[i], b = x[i + 1], c = x[i + 2], d = x[i + 3];
  float p0, p1, s0, s1, q0, q1;
  upk(mul2(pk(a, b), pk(c, d)), p0, p1);
  if (__float_as_uint(p0) != __float_as_uint(__fmul_rn(a, c)) ||
      __float_as_uint(p1) != __float_as_uint(__fmul_rn(b, d)))
    atomicAdd(&bad[0], 1u);
  upk(add2(pk(a, b), pk(c, d)), s0, s1);
  if (__float_as_uint(s0) != __float_as_uint(__fadd_rn(a, c)) ||
      __float_as_uint(s1) != __float_as_uint(__fadd_rn(b, d)))
    atomicAdd(&bad[1], 1u);
  // chain: (a*c + b*d, a*d + b*c) both ways
  upk(add2(mul2(pk(a, a), pk(c, d)), mul2(pk(b, b), pk(d, c))), q0, q1);
  const float r0 = __fadd_rn(__fmul_rn(a, c), __fmul_rn(b, d));
  const float r1 = __fadd_rn(__fmul_rn(a, d), __fmul_rn(b, c));
  if (__float_as_uint(q0) != __float_as_uint(r0) ||
      __float_as_uint(q1) != __float_as_uint(r1))
    atomicAdd(&bad[2], 1u);
}

int main() {
  const int n = 1 << 22;
  float* h = new float[n];
  uint32_t s = 12345;
  for (int pass = 0; pass < 2; ++pass) {
    for (int i = 0; i < n; ++i) {
      s = s * 1664525u + 1013904223u;
      float v = (float)((int)(s >> 8) - (1 << 23)) / (float)(1 << 20);
      h[i] = pass ? v * 1e-38f : v;  // pass 1: products / values denormal
    }
    float* d; unsigned* bad;
    cudaMalloc(&d, n * 4); cudaMalloc(&bad, 12);
    cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
    cudaMemset(bad, 0, 12);
    k<<<n / 256, 256>>>(d, n, bad);
    unsigned hb[3];
    cudaMemcpy(hb, bad, 12, cudaMemcpyDeviceToHost);
    printf("%s inputs: mul2 mismatches %u, add2 %u, mul2->add2 chain %u (of %d)\n",
           pass ? "tiny (denormal results)" : "normal", hb[0], hb[1], hb[2], n - 3);
    cudaFree(d); cudaFree(bad);
  }
  return 0;
}
