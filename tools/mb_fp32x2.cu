#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float2 add2(float2 a, float2 b){
  unsigned long long ra = *reinterpret_cast<unsigned long long*>(&a), rb = *reinterpret_cast<unsigned long long*>(&b), rd;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(rd) : "l"(ra), "l"(rb));
  return *reinterpret_cast<float2*>(&rd);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c){
  unsigned long long ra = *reinterpret_cast<unsigned long long*>(&a), rb = *reinterpret_cast<unsigned long long*>(&b), rc=*reinterpret_cast<unsigned long long*>(&c), rd;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  return *reinterpret_cast<float2*>(&rd);
}
template<int MODE>
__global__ void k(float* out, int iters, float s){
  float a[16]; float2 b[8];
  for(int i=0;i<16;i++) a[i]=threadIdx.x*0.001f+i;
  for(int i=0;i<8;i++) b[i]=make_float2(threadIdx.x*0.001f+i, i*0.5f);
  float2 ss = make_float2(s, s);
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<16;i++){
      if(MODE==0){ a[i] = a[i] + a[(i+1)&15]; }
      else if(MODE==1){ a[i] = fmaf(a[i], s, a[(i+3)&15]); }
      else if(MODE==2){ if(i<8) b[i] = add2(b[i], b[(i+1)&7]); }
      else if(MODE==3){ if(i<8) b[i] = fma2(b[i], ss, b[(i+3)&7]); }
    }
  }
  float r=0; for(int i=0;i<16;i++) r+=a[i]; for(int i=0;i<8;i++) r+=b[i].x+b[i].y;
  out[blockIdx.x*blockDim.x+threadIdx.x]=r;
}
int main(){
  float* out; cudaMalloc(&out, 148*8*1024*4);
  int iters=20000;
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for(int mode=0; mode<4; ++mode){
    for(int rep=0; rep<2; ++rep){
    cudaEventRecord(e0);
    if(mode==0) k<0><<<148*4,512>>>(out,iters,1.0001f);
    if(mode==1) k<1><<<148*4,512>>>(out,iters,1.0001f);
    if(mode==2) k<2><<<148*4,512>>>(out,iters,1.0001f);
    if(mode==3) k<3><<<148*4,512>>>(out,iters,1.0001f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double ops = 148.0*4*512*(double)iters*16; // scalar fp32 ops (MODE 2,3: 8 instr x2 lanes)
    double instr = (mode<2)? ops : ops/2;
    printf("mode %d: %.3f ms, %.2f Tflop-ops/s, %.2f Tinstr(thread)/s\n", mode, ms, ops/ms/1e9, instr/ms/1e9);
    }
  }
  return 0;
}
