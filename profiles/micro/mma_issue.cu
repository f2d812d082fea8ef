// Cost of ISSUING the LWPR chunk MMA (3 x tcgen05.mma kind::tf32 M=128 N=128 K=8 + commit) and its
// completion latency, while the CTA's other warps (a) idle, (b) stream tcgen05.ld x16 from the other
// TMEM buffer, (c) run MUFU ex2; 1 or 2 CTAs per SM, 256 TMEM columns per CTA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//          -I paper_1503_00330_b200/csrc -o mma_issue profiles/micro/mma_issue.cu
#include <cstdio>

#include "lwpr_tc.cuh"

using namespace pi2;

__global__ void __launch_bounds__(128) mma_issue_kernel(int mode, int reps, unsigned long long *out) {
  __shared__ __align__(128) uint8_t sm[8192 + 16384];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ volatile int stop;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (8192 + 16384) / 4; i += 128) reinterpret_cast<float *>(sm)[i] = 0.001f * (i & 7);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)), "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const uint32_t mbar_addr = (uint32_t)__cvta_generic_to_shared(&mbar);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_addr));
    asm volatile("fence.mbarrier_init.release.cluster;");
    stop = 0;
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base, sa = (uint32_t)__cvta_generic_to_shared(sm);
  float acc = 0.f;
  if (warp == 0) {
    uint32_t phase = 0;
    long long t_issue = 0, t_done = 0;
    for (int r = 0; r < reps; ++r) {
      if (tid == 0) {
        const long long t0 = clock64();
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t idesc = umma_idesc_tf32(128, 128);
        mma_tf32(tmem, umma_smem_desc(sa), umma_smem_desc(sa + 8192), idesc, 0);
        mma_tf32(tmem, umma_smem_desc(sa), umma_smem_desc(sa + 16384), idesc, 1);
        mma_tf32(tmem, umma_smem_desc(sa + 4096), umma_smem_desc(sa + 8192), idesc, 1);
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar_addr));
        const long long t1 = clock64();
        mbar_wait(mbar_addr, phase);
        const long long t2 = clock64();
        t_issue += t1 - t0;
        t_done += t2 - t0;
      }
      phase ^= 1;
      __syncwarp();
    }
    if (tid == 0) {
      atomicAdd(&out[0], (unsigned long long)t_issue);
      atomicAdd(&out[1], (unsigned long long)t_done);
      atomicAdd(&out[2], 1ull);
      stop = 1;
    }
  } else if (mode == 1) {  // stream TMEM reads of buffer 1 (this warp's lanes)
    const uint32_t lane = tmem + 128 + ((uint32_t)(warp * 32) << 16);
    uint32_t v[16];
    while (!stop) {
#pragma unroll
      for (int c = 0; c < 128; c += 16) {
        PI2_TMEM_LD16(v, lane + c);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        acc += __uint_as_float(v[0]) + __uint_as_float(v[15]);
      }
    }
  } else if (mode == 2) {  // MUFU ex2 flood
    float x = 0.001f * tid;
    while (!stop) {
#pragma unroll
      for (int k = 0; k < 64; ++k) x = ex2_ftz(x) * 0.5f;
    }
    acc = x;
  }
  if (acc == 12345.f) out[3] = 1;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *d;
  cudaMalloc(&d, 32);
  const char *names[3] = {"others idle", "others tcgen05.ld", "others MUFU"};
  for (int per : {1, 2})
    for (int mode = 0; mode < 3; ++mode) {
      const int pad = 228 * 1024 / per - 1024 - 8192 - 16384 - 512;
      cudaFuncSetAttribute((const void *)mma_issue_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
      cudaMemset(d, 0, 32);
      const int reps = 500;
      mma_issue_kernel<<<sms * per, 128, pad>>>(mode, reps, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[4];
      cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
      printf("CTAs/SM %d, %-18s: issue %5.0f clk, issue->complete %5.0f clk (%s)\n", per, names[mode],
             (double)h[0] / h[2] / reps, (double)h[1] / h[2] / reps, cudaGetErrorString(e));
    }
  return 0;
}
