// Microbenchmark: does MUFU.EX2 overlap with FFMA on sm_100a?
// Per iteration and per independent chain: N FFMA (register operands only) + 1 MUFU.EX2,
// for N in a sweep; plus the same with the FMA part as packed FFMA2, and a
// polynomial exp2 on the FMA/ALU pipes instead of MUFU.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_mix mufu_mix.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void upk(u64 v, float& a, float& b) { asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }

// polynomial 2^x for x in [-126, 0]: round-to-nearest split + degree-5 minimax on [-0.5, 0.5]
__device__ __forceinline__ float exp2_poly(float x) {
  const float j = __fadd_rn(__fadd_rn(x, 12582912.0f), -12582912.0f);  // rint(x)
  const float f = __fsub_rn(x, j);
  float p = fmaf(1.3333558146e-3f, f, 9.6181291076e-3f);
  p = fmaf(p, f, 5.5504108665e-2f);
  p = fmaf(p, f, 2.4022650696e-1f);
  p = fmaf(p, f, 6.9314718056e-1f);
  p = fmaf(p, f, 1.0f);
  const int e = __float2int_rn(j) << 23;
  return __int_as_float(__float_as_int(p) + e);
}

template <int N, int MODE>  // MODE 0: FFMA+MUFU, 1: FFMA2+MUFU, 2: FFMA+poly, 3: FFMA only, 4: MUFU only
__global__ void k(float* out, float a, float b, int iters) {
  constexpr int C = 8;
  float x[C], acc[C];
#pragma unroll
  for (int i = 0; i < C; ++i) { x[i] = -0.001f * (threadIdx.x & 7) - i * 0.01f; acc[i] = 0.0f; }
  const u64 A2 = pk(a, a), B2 = pk(b, b);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i) {
      if (MODE == 1) {
        if (i % 2) continue;
        u64 v = pk(x[i], x[i + 1]);
#pragma unroll
        for (int n = 0; n < N; ++n) v = ffma2(v, A2, B2);
        float u0, u1;
        upk(v, u0, u1);
        acc[i] += ex2(u0);
        acc[i + 1] += ex2(u1);
        x[i] = u0 * 1e-3f - 1.0f;
        x[i + 1] = u1 * 1e-3f - 1.0f;
      } else {
        float v = x[i];
        if (MODE != 4) {
#pragma unroll
          for (int n = 0; n < N; ++n) v = fmaf(v, a, b);
        }
        if (MODE == 0 || MODE == 1 || MODE == 4) acc[i] = ex2(v + acc[i] * 1e-30f);
        else if (MODE == 2) acc[i] = exp2_poly(v + acc[i] * 1e-30f);
        else acc[i] += v;
        x[i] = v;
      }
    }
  }
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < C; ++i) s += acc[i] + x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int N, int MODE>
void run(const char* name, float* out, int blocks, int threads, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<N, MODE><<<blocks, threads>>>(out, 0.999f, -1e-3f, 16);
  cudaEventRecord(e0);
  k<N, MODE><<<blocks, threads>>>(out, 0.999f, -1e-3f, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double lanes = (double)blocks * threads * iters * 8;
  const double fma = (MODE == 4) ? 0 : lanes * N, mufu = (MODE == 3) ? 0 : lanes;
  printf("%-26s N=%2d: %6.2f TFMA/s (%.0f%% of 37.2T)  %5.2f Tex2/s  %.3f ms\n", name, N, fma / ms / 1e9,
         100 * fma / ms / 1e9 / 37.2, mufu / ms / 1e9, ms);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 2048;
  float* out;
  cudaMalloc(&out, blocks * threads * 4);
  run<1, 4>("MUFU only", out, blocks, threads, iters);
  run<16, 3>("FFMA only", out, blocks, threads, iters);
  run<4, 0>("FFMA+MUFU", out, blocks, threads, iters);
  run<8, 0>("FFMA+MUFU", out, blocks, threads, iters);
  run<12, 0>("FFMA+MUFU", out, blocks, threads, iters);
  run<16, 0>("FFMA+MUFU", out, blocks, threads, iters);
  run<24, 0>("FFMA+MUFU", out, blocks, threads, iters);
  run<8, 1>("FFMA2+MUFU", out, blocks, threads, iters);
  run<16, 1>("FFMA2+MUFU", out, blocks, threads, iters);
  run<8, 2>("FFMA+poly exp2", out, blocks, threads, iters);
  run<16, 2>("FFMA+poly exp2", out, blocks, threads, iters);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
