// TMEM -> register bandwidth on sm_100a (tcgen05.ld.32x32b.x32): decides whether a
// FlashAttention-shaped tensor-core LWPR (logits in TMEM, exp on CUDA cores) can
// beat the CUDA-core kernel.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int COLS_PER_LD>
__global__ void __launch_bounds__(128, 1) tmem_ld(float *out, int iters) {
  __shared__ uint32_t taddr;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr + ((uint32_t)(warp * 32) << 16);
  // fill 256 columns of this warp's 32 lanes
  for (int c = 0; c < 256; c += 8) {
    const uint32_t v = __float_as_uint((float)(threadIdx.x + c));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(base + c), "r"(v));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  float acc = 0.0f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 256; c += COLS_PER_LD) {
      uint32_t r[32];
      if (COLS_PER_LD == 32) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
              "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
              "=r"(r[30]), "=r"(r[31])
            : "r"(base + c));
      } else {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                       "=r"(r[7])
                     : "r"(base + c));
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int i = 0; i < COLS_PER_LD; ++i) acc += __uint_as_float(r[i]);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(taddr));
}

template <int C>
void run(const char *name, int blocks, int iters, float *out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  tmem_ld<C><<<blocks, 128>>>(out, 2);
  cudaEventRecord(e0);
  tmem_ld<C><<<blocks, 128>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)blocks * 128 * 256 * 4 * iters;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("%-28s blocks %4d: %8.1f GB/s total, %6.1f B/clk/SM at 1.965 GHz (%.3f ms)\n", name, blocks,
         bytes / ms / 1e6, bytes / ms / 1e6 / sms / 1.965, ms);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *out;
  cudaMalloc(&out, 4 * sms * 128 * 4);
  run<32>("ld.32x32b.x32, 1 CTA/SM", sms, 2000, out);
  run<32>("ld.32x32b.x32, 2 CTA/SM", 2 * sms, 2000, out);
  run<8>("ld.32x32b.x8, 1 CTA/SM", sms, 2000, out);
  run<8>("ld.32x32b.x8, 2 CTA/SM", 2 * sms, 2000, out);
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
