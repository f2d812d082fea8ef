// Latency of the LWPR chunk MMA (3 x tcgen05.mma kind::tf32, M=128, N=2*Lc, K=8, SS operands,
// commit -> mbarrier) as the issuing thread sees it, with 1..4 co-resident CTAs per SM issuing
// back to back, and the wait cost of tcgen05.ld + wait::ld for 8/16/32 columns.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//          -I paper_1503_00330_b200/csrc -o mma_lat profiles/micro/mma_lat.cu
#include <cstdio>

#include "lwpr_tc.cuh"

using namespace pi2;

__global__ void __launch_bounds__(128) mma_lat_kernel(int n_mma, int ncols, int reps, unsigned long long *out) {
  __shared__ __align__(128) uint8_t sm[8192 + 2 * 8192];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (8192 + 16384) / 4; i += 128) reinterpret_cast<float *>(sm)[i] = 0.001f * (i & 7);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)), "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const uint32_t mbar_addr = (uint32_t)__cvta_generic_to_shared(&mbar);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_addr));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base, sa = (uint32_t)__cvta_generic_to_shared(sm);
  uint32_t phase = 0;
  long long t_mma = 0, t_ld = 0;
  float acc = 0.f;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    const long long t0 = clock64();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t idesc = umma_idesc_tf32(128, ncols);
      for (int i = 0; i < n_mma; ++i)
        mma_tf32(tmem, umma_smem_desc(sa + (i & 1) * 4096), umma_smem_desc(sa + 8192 + (i & 1) * 8192), idesc, i > 0);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar_addr));
    }
    mbar_wait(mbar_addr, phase);
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
    const long long t1 = clock64();
    uint32_t v[16];
    const uint32_t lane = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < ncols; c += 16) {
      PI2_TMEM_LD16(v, lane + c);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 16; ++j) acc += __uint_as_float(v[j]);
    }
    const long long t2 = clock64();
    asm volatile("tcgen05.fence::before_thread_sync;");
    t_mma += t1 - t0;
    t_ld += t2 - t1;
  }
  if ((tid & 31) == 0) {
    atomicAdd(&out[0], (unsigned long long)t_mma);
    atomicAdd(&out[1], (unsigned long long)t_ld);
    atomicAdd(&out[2], 1ull);
  }
  if (acc == 12345.f) out[3] = 1;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(128));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *d;
  cudaMalloc(&d, 32);
  // smem padding so that exactly `per` CTAs fit on an SM
  for (int per : {1, 2, 4}) {
    const int pad = 228 * 1024 / per - 1024 - 8192 - 16384 - 256;
    cudaFuncSetAttribute((const void *)mma_lat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
    for (int n_mma : {1, 3}) {
      for (int ncols : {64, 128}) {
        const int reps = 200;
        cudaMemset(d, 0, 32);
        mma_lat_kernel<<<sms * per, 128, pad>>>(n_mma, ncols, reps, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[4];
        cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
        printf("CTAs/SM %d  MMAs %d  N %3d: issue->mbarrier %6.0f clk, tcgen05.ld x16 + wait per 16 cols %5.0f clk (%s)\n", per,
               n_mma, ncols, (double)h[0] / h[2] / reps, (double)h[1] / h[2] / reps / (ncols / 16), cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
