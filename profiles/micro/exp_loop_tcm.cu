// Rate of the exp phase of a "moments on the tensor cores" LWPR schedule, alone: per 16
// fields, tcgen05.ld the logits, e = 2^logit (TCM_POLY of 8 pairs on the FMA pipe, the rest
// on MUFU), the tf32 split lo = e - trunc_tf32(e), tcgen05.st e (in place) and lo -- no
// moment FMAs.  Same frame as exp_loop_rate.cu (1..4 CTAs of 4 warps per SM).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//          -I paper_1503_00330_b200/csrc -DPOLY=2 -o exp_loop_tcm profiles/micro/exp_loop_tcm.cu
#include <cstdio>

#include "lwpr_tc.cuh"

#ifndef TCM_POLY
#define TCM_POLY 2
#endif

using namespace pi2;

#define TMEM_ST16(addr, r)                                                                                  \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
               ::"r"(addr), "r"((r)[0]), "r"((r)[1]), "r"((r)[2]), "r"((r)[3]), "r"((r)[4]), "r"((r)[5]),       \
               "r"((r)[6]), "r"((r)[7]), "r"((r)[8]), "r"((r)[9]), "r"((r)[10]), "r"((r)[11]), "r"((r)[12]),   \
               "r"((r)[13]), "r"((r)[14]), "r"((r)[15]) : "memory")

__global__ void __launch_bounds__(128, 4) exp_tcm_kernel(int reps, float *out, unsigned long long *clk) {
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
  float acc = 0.0f;
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    {  // refill the 48 logit columns (the MMA's job in the kernel; not timed separately)
      uint32_t v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(-8.0f + 0.25f * ((tid + j + r) & 63));
#pragma unroll
      for (int c = 0; c < 48; c += 16) TMEM_ST16(tl + c, v);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
#pragma unroll
    for (int c = 0; c < 48; c += 16) {
      uint32_t l16[16], lo16[16];
      PI2_TMEM_LD16(l16, tl + c);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const float2 x = make_float2(__uint_as_float(l16[i]), __uint_as_float(l16[i + 1]));
        const float2 e = ((i / 2) % 8 < TCM_POLY) ? exp2_poly2(x) : make_float2(ex2_ftz(x.x), ex2_ftz(x.y));
        // -trunc_tf32(e) in one LOP3 each, lo = e - trunc_tf32(e) exactly
        const float2 nh = make_float2(__uint_as_float((__float_as_uint(e.x) & 0xFFFFE000u) ^ 0x80000000u),
                                      __uint_as_float((__float_as_uint(e.y) & 0xFFFFE000u) ^ 0x80000000u));
        const float2 lo = __fadd2_rn(e, nh);
        l16[i] = __float_as_uint(e.x);
        l16[i + 1] = __float_as_uint(e.y);
        lo16[i] = __float_as_uint(lo.x);
        lo16[i + 1] = __float_as_uint(lo.y);
      }
      TMEM_ST16(tl + c, l16);
      TMEM_ST16(tl + 48 + c, lo16);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  const long long t1 = clock64();
  {
    uint32_t l16[16];
    PI2_TMEM_LD16(l16, tl + 48);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 16; ++j) acc += __uint_as_float(l16[j]);
  }
  out[blockIdx.x * 128 + tid] = acc;
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
  const int reps = 4000;
  for (int per = 1; per <= 4; ++per) {
    const int pad = 228 * 1024 / per - 1024 - 1024;
    cudaFuncSetAttribute((const void *)exp_tcm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    exp_tcm_kernel<<<sms * per, 128, pad>>>(reps, out, clk);  // warm
    cudaMemset(clk, 0, 8);
    cudaEventRecord(e0);
    exp_tcm_kernel<<<sms * per, 128, pad>>>(reps, out, clk);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h;
    cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
    const double fields = (double)sms * per * 128 * reps * 48;
    const double ex2 = fields * (8.0 - TCM_POLY) / 8.0;
    printf("TCM_POLY %d/8 warps/SMSP %d: %.1f clk per field per warp (incl. refill), %.2f T ex2/s on MUFU (%.0f%% of 4.6), %.2f T fields/s (%s)\n",
           TCM_POLY, per, (double)h / (sms * per * 4) / reps / 48, ex2 / (ms * 1e-3) / 1e12, 100.0 * ex2 / (ms * 1e-3) / 4.6e12,
           fields / (ms * 1e-3) / 1e12, cudaGetErrorString(e));
  }
  return 0;
}
