// Rate of the LWPR exp phase alone (tc_fields8 over 64-field chunks read from a pre-filled
// TMEM buffer, the kernel's unrolled LD16 loop), with 1..4 co-resident CTAs of 4 warps per SM
// (= 1..4 warps per SM sub-partition): clocks per field per warp and the MUFU ex2 rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//          -I paper_1503_00330_b200/csrc -o exp_loop_rate profiles/micro/exp_loop_rate.cu
#include <cstdio>

#include "lwpr_tc.cuh"

// share of the 2^x on MUFU: (8 - 2 POLY) + (8 - 2 POLY_B) of 16 fields
#define VAR_SHARE(v) ((v) ? (16.0 - 2 * PI2_TC_POLY_VAR - 2 * PI2_TC_POLY_VAR_B) / 16.0 : (16.0 - 2 * PI2_TC_POLY_MEAN - 2 * PI2_TC_POLY_MEAN_B) / 16.0)

using namespace pi2;

template <bool VAR>
__global__ void __launch_bounds__(128, 4) exp_rate_kernel(int reps, float *out, unsigned long long *clk) {
  __shared__ __align__(16) float slv[64];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid < 64) slv[tid] = 0.01f * tid;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)), "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
  {  // fill: logits in [-8, 8], y' in [-1, 1]
    uint32_t v[16];
    for (int c = 0; c < 128; c += 16) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        v[j] = __float_as_uint(c < 64 ? -8.0f + 0.25f * ((tid + c + j) & 63) : 0.03f * ((tid * 7 + j) & 63) - 1.0f);
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
              tl + c),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
          "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  float2 den = make_float2(0.f, 0.f), num = den, m2 = den, lv = den;
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int b = 0; b < 8; b += 2) {
      uint32_t l16[16], y16[16];
      PI2_TMEM_LD16(l16, tl + 8 * b);
      PI2_TMEM_LD16(y16, tl + 64 + 8 * b);
      PI2_TMEM_WAIT16(l16, y16);
      PI2_TMEM_WAIT16(l16 + 8, y16 + 8);
      tc_fields8<VAR>(l16, y16, slv + 8 * b, den, num, m2, lv);
      tc_fields8<VAR, true>(l16 + 8, y16 + 8, slv + 8 * b + 8, den, num, m2, lv);
    }
  }
  const long long t1 = clock64();
  out[blockIdx.x * 128 + tid] = den.x + den.y + num.x + num.y + m2.x + m2.y + lv.x;
  if ((tid & 31) == 0) atomicAdd(clk, (unsigned long long)(t1 - t0));
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(128));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *out;
  unsigned long long *clk;
  cudaMalloc(&out, sms * 4 * 128 * 4);
  cudaMalloc(&clk, 8);
  const int reps = 2000;
  for (int var = 1; var >= 0; --var)
    for (int per = 1; per <= 4; ++per) {
      const int pad = 228 * 1024 / per - 1024 - 1024;
      auto *k = var ? exp_rate_kernel<true> : exp_rate_kernel<false>;
      cudaFuncSetAttribute((const void *)k, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
      cudaMemset(clk, 0, 8);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      k<<<sms * per, 128, pad>>>(reps, out, clk);  // warm
      cudaMemset(clk, 0, 8);
      cudaEventRecord(e0);
      k<<<sms * per, 128, pad>>>(reps, out, clk);
      cudaEventRecord(e1);
      cudaError_t e = cudaDeviceSynchronize();
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long h;
      cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
      const double fields = (double)sms * per * 128 * reps * 64;  // row-fields
      const double ex2 = fields * (VAR_SHARE(var));
      printf("%s warps/SMSP %d: %.1f clk per field per warp, %.2f T ex2/s on MUFU (%.0f%% of 4.6), %.2f T fields/s (%s)\n",
             var ? "variance " : "mean-only", per, (double)h / (sms * per * 4) / reps / 64, ex2 / (ms * 1e-3) / 1e12,
             100.0 * ex2 / (ms * 1e-3) / 4.6e12, fields / (ms * 1e-3) / 1e12, cudaGetErrorString(e));
    }
  return 0;
}
