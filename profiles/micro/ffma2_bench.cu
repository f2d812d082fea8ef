// Microbenchmark: FP32 FMA throughput of FFMA vs packed FFMA2 (sm_100a), and an
// LWPR-like mix with MUFU.EX2.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_bench ffma2_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b){ u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c){ u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ float ex2(float x){ float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

__global__ void k_ffma(float* out, float a, float b, int iters){
  float x[16];
  for(int i=0;i<16;i++) x[i]=threadIdx.x*1e-3f+i;
  for(int it=0; it<iters; it++){
#pragma unroll
    for(int i=0;i<16;i++) x[i]=fmaf(x[i],a,b);
  }
  float s=0; for(int i=0;i<16;i++) s+=x[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_ffma2(float* out, float a, float b, int iters){
  u64 x[8]; u64 A=pk(a,a), B=pk(b,b);
  for(int i=0;i<8;i++) x[i]=pk(threadIdx.x*1e-3f+i, i+0.5f);
  for(int it=0; it<iters; it++){
#pragma unroll
    for(int i=0;i<8;i++) x[i]=ffma2(x[i],A,B);
  }
  float s=0; for(int i=0;i<8;i++){ float lo,hi; asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[i])); s+=lo+hi; }
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
// 16 FFMA + 1 MUFU per "row-field" (8 rows), like the LWPR loop
__global__ void k_mix(float* out, const float4* __restrict__ p, int iters){
  float x[8], acc[8];
  for(int i=0;i<8;i++){ x[i]=threadIdx.x*1e-4f+i*0.01f; acc[i]=0; }
  for(int it=0; it<iters; it++){
    float4 q=p[it&63];
#pragma unroll
    for(int r=0;r<8;r++){
      float l=fmaf(fmaf(q.x,x[r],q.y),x[r],q.z);
      l=fmaf(fmaf(q.y,x[r],q.z),x[r],l);
      l=fmaf(fmaf(q.z,x[r],q.w),x[r],l);
      l=fmaf(fmaf(q.w,x[r],q.x),x[r],l);
      float e=ex2(l);
      float y=fmaf(q.x,x[r],q.w); y=fmaf(q.y,x[r],y); y=fmaf(q.z,x[r],y); y=fmaf(q.w,x[r],y);
      acc[r]=fmaf(e,y,acc[r]);
    }
  }
  float s=0; for(int i=0;i<8;i++) s+=acc[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks=sms*8, threads=256, iters=4096;
  float* out; cudaMalloc(&out, blocks*threads*4);
  float4* p; cudaMalloc(&p, 64*16); cudaMemset(p,0,64*16);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for(int rep=0;rep<2;rep++){
    cudaEventRecord(e0); k_ffma<<<blocks,threads>>>(out,0.999f,1e-3f,iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms,e0,e1); double f=2.0*16*iters*(double)blocks*threads; printf("FFMA : %.2f TFLOP/s (%.3f ms)\n", f/ms/1e9, ms);
    cudaEventRecord(e0); k_ffma2<<<blocks,threads>>>(out,0.999f,1e-3f,iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms,e0,e1); f=2.0*16*iters*(double)blocks*threads; printf("FFMA2: %.2f TFLOP/s (%.3f ms)\n", f/ms/1e9, ms);
    cudaEventRecord(e0); k_mix<<<blocks,threads>>>(out,p,iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms,e0,e1); f=2.0*13*8*iters*(double)blocks*threads; double mu=8.0*iters*blocks*threads;
    printf("MIX  : %.2f TFLOP/s FMA-part, %.2f Tex2/s (%.3f ms)\n", f/ms/1e9, mu/ms/1e9, ms);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
