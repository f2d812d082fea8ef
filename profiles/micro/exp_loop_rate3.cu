// [variant exp_loop_rate3: the variance loop with a third TMEM column z = y'^2 + var_l per field
// (what an MMA over quadratic features would produce): m2 += e z, no per-field variance loads.
// 40-field chunks (3 x 40 columns of 128).]
// Rate of the LWPR exp phase alone (tc_fields8 over 64-field chunks read from a pre-filled
// TMEM buffer, the kernel's unrolled LD16 loop), with 1..4 co-resident CTAs of 4 warps per SM
// (= 1..4 warps per SM sub-partition): clocks per field per warp and the MUFU ex2 rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//          -I paper_1503_00330_b200/csrc -o exp_loop_rate profiles/micro/exp_loop_rate.cu
#include <cstdio>

#include "lwpr_tc.cuh"
#ifndef ZPOLY
#define ZPOLY 0
#endif

// share of the 2^x on MUFU: (8 - 2 POLY) + (8 - 2 POLY_B) of 16 fields
#define VAR_SHARE(v) ((v) ? (16.0 - 2 * PI2_TC_POLY_VAR - 2 * PI2_TC_POLY_VAR_B) / 16.0 : (16.0 - 2 * PI2_TC_POLY_MEAN - 2 * PI2_TC_POLY_MEAN_B) / 16.0)

using namespace pi2;

__device__ __forceinline__ void fields8_z(const uint32_t *lg, const uint32_t *yy, const uint32_t *zz, float2 &den,
                                          float2 &num, float2 &m2) {
#pragma unroll
  for (int i = 0; i < 8; i += 2) {
    const float2 x = make_float2(__uint_as_float(lg[i]), __uint_as_float(lg[i + 1]));
    const float2 e = (i / 2 < ZPOLY) ? exp2_poly2(x) : make_float2(ex2_ftz(x.x), ex2_ftz(x.y));
    const float2 y = make_float2(__uint_as_float(yy[i]), __uint_as_float(yy[i + 1]));
    const float2 z = make_float2(__uint_as_float(zz[i]), __uint_as_float(zz[i + 1]));
    den = __fadd2_rn(den, e);
    num = __ffma2_rn(e, y, num);
    m2 = __ffma2_rn(e, z, m2);
  }
}

template <bool VAR>
__global__ void __launch_bounds__(128, 4) exp_rate_kernel(int reps, float *out, unsigned long long *clk) {
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
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
  {
    uint32_t v[16];
    for (int c = 0; c < 128; c += 16) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        v[j] = __float_as_uint(c < 48 ? -8.0f + 0.25f * ((tid + c + j) & 63) : 0.03f * ((tid * 7 + j) & 63) - 1.0f);
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
              tl + c),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
          "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  float2 den = make_float2(0.f, 0.f), num = den, m2 = den;
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int b = 0; b < 40; b += 8) {  // 40-field chunk: logits 0..39, y' 40..79, z 80..119
      uint32_t l8[8], y8[8], z8[8];
      PI2_TMEM_LD8(l8, tl + b);
      PI2_TMEM_LD8(y8, tl + 40 + b);
      PI2_TMEM_LD8(z8, tl + 80 + b);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      fields8_z(l8, y8, z8, den, num, m2);
    }
  }
  const long long t1 = clock64();
  out[blockIdx.x * 128 + tid] = den.x + den.y + num.x + num.y + m2.x + m2.y;
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
  for (int var = 1; var >= 1; --var)
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
      const double fields = (double)sms * per * 128 * reps * 40;  // row-fields
      const double ex2 = fields * (4.0 - ZPOLY) / 4.0;
      printf("%s warps/SMSP %d: %.1f clk per field per warp, %.2f T ex2/s on MUFU (%.0f%% of 4.6), %.2f T fields/s (%s)\n",
             "var+z ZPOLY", per, (double)h / (sms * per * 4) / reps / 40, ex2 / (ms * 1e-3) / 1e12,
             100.0 * ex2 / (ms * 1e-3) / 4.6e12, fields / (ms * 1e-3) / 1e12, cudaGetErrorString(e));
    }
  return 0;
}
