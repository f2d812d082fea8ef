// Feasibility of the LWPR moments as a second tcgen05 GEMM with the A operand (the
// weights e of a row tile) in TMEM: D[128, N] += E[128, K] . V[K, N], kind::tf32,
// A = TMEM columns (lane = row), B = shared memory (K-major, no swizzle).
//  (1) correctness against a host fp64 GEMM of the tf32-truncated operands;
//  (2) issue cost and issue->complete latency of n back-to-back K=8 MMAs (N = 16 / 32),
//      1 or 4 CTAs per SM, A from TMEM vs A from shared memory;
//  (3) tcgen05.st x16 + wait::st cost.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//          -I paper_1503_00330_b200/csrc -o mma_tmem_a profiles/micro/mma_tmem_a.cu
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "lwpr_tc.cuh"

using namespace pi2;

__device__ __forceinline__ void mma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc, int acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}

#define TMEM_ST16(addr, r)                                                                                  \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
               ::"r"(addr), "r"((r)[0]), "r"((r)[1]), "r"((r)[2]), "r"((r)[3]), "r"((r)[4]), "r"((r)[5]),       \
               "r"((r)[6]), "r"((r)[7]), "r"((r)[8]), "r"((r)[9]), "r"((r)[10]), "r"((r)[11]), "r"((r)[12]),   \
               "r"((r)[13]), "r"((r)[14]), "r"((r)[15]) : "memory")

constexpr int NMAX = 32;
// B block s (k = 8s .. 8s+7) at s * NMAX * 32 bytes: rows n, k K-major (umma_kmajor_off)

__global__ void __launch_bounds__(128) check_kernel(const float *E, const float *V, int K, int N, float *D) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int s = 0; s < K / 8; ++s)
    for (int i = tid; i < N * 8; i += 128) {
      const int n = i / 8, k = i % 8;
      *reinterpret_cast<float *>(sm + s * NMAX * 32 + umma_kmajor_off(n, k)) = V[(8 * s + k) * N + n];
    }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)), "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const uint32_t mbar_addr = (uint32_t)__cvta_generic_to_shared(&mbar);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_addr));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base, lane = tmem + ((uint32_t)(warp * 32) << 16);
  for (int c = 0; c < K; c += 16) {
    uint32_t r[16];
    for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(E[tid * K + c + j]);
    TMEM_ST16(lane + c, r);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = umma_idesc_tf32(128, N);
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
    for (int s = 0; s < K / 8; ++s) mma_tf32_ta(tmem + 128, tmem + 8 * s, umma_smem_desc(sb + s * NMAX * 32), idesc, s > 0);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar_addr));
  }
  mbar_wait(mbar_addr, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16], z[16];
    PI2_TMEM_LD16(r, lane + 128 + c);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 16; ++j) D[tid * N + c + j] = __uint_as_float(r[j]);
    (void)z;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
}

// timing: warp 0 issues NM K=8 MMAs (A from TMEM if TA, else shared) N columns, commit, wait.
// ELECT: the warp stays converged and one lane is elected inside the asm (uniform operands,
// no divergent region around the UTCHMMA); else thread 0 issues in a divergent branch.
template <int NM, bool TA, bool ELECT>
__global__ void __launch_bounds__(128) time_kernel(int N, int reps, int do_st, unsigned long long *out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (16 * NMAX * 32 + 8192) / 4; i += 128) reinterpret_cast<float *>(sm)[i] = 0.001f * (i & 7);
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
  const uint32_t tmem = tmem_base, lane = tmem + ((uint32_t)(warp * 32) << 16);
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t idesc = umma_idesc_tf32(128, N);
  const uint64_t bd0 = umma_smem_desc(sb), ad0 = umma_smem_desc(sb + 16 * NMAX * 32);
  uint32_t phase = 0;
  long long t_iss = 0, t_done = 0, t_st = 0;
  for (int r = 0; r < reps; ++r) {
    if (do_st) {  // every warp stores 96 columns of its lanes (the e / e_lo of a 48-field chunk)
      const long long t0 = clock64();
      uint32_t v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(0.25f * j + r);
#pragma unroll
      for (int c = 0; c < 96; c += 16) TMEM_ST16(lane + c, v);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      t_st += clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) {
      const long long t0 = clock64();
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (ELECT) {
#pragma unroll
        for (int s = 0; s < NM; ++s) {
          const uint64_t bd = bd0 + (uint64_t)(((s & 15) * NMAX * 32) >> 4);
          if (TA)
            asm volatile(
                "{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + 96),
                "r"(tmem + 8 * (s % 12)), "l"(bd), "r"(idesc), "r"(s)
                : "memory");
          else
            asm volatile(
                "{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + 96),
                "l"(ad0), "l"(bd), "r"(idesc), "r"(s)
                : "memory");
        }
        asm volatile(
            "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(mbar_addr)
            : "memory");
      } else if (tid == 0) {
#pragma unroll
        for (int s = 0; s < NM; ++s) {
          const uint64_t bd = bd0 + (uint64_t)(((s & 15) * NMAX * 32) >> 4);
          if (TA) mma_tf32_ta(tmem + 96, tmem + 8 * (s % 12), bd, idesc, s > 0);
          else mma_tf32(tmem + 96, ad0, bd, idesc, s > 0);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar_addr));
      }
      __syncwarp();
      const long long t1 = clock64();
      mbar_wait(mbar_addr, phase);
      const long long t2 = clock64();
      t_iss += t1 - t0;
      t_done += t2 - t0;
    } else {
      mbar_wait(mbar_addr, phase);
    }
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  if (tid == 0) {
    atomicAdd(&out[0], (unsigned long long)t_iss);
    atomicAdd(&out[1], (unsigned long long)t_done);
    atomicAdd(&out[2], 1ull);
  }
  if (tid == 32) atomicAdd(&out[3], (unsigned long long)t_st);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(128));
}

template <int NM, bool TA, bool ELECT>
void run_time(int sms, unsigned long long *d) {
  for (int per : {1, 4})
    for (int N : {16, 32, 128}) {
      const int smem = 228 * 1024 / per - 1024 - 512;
      auto fn = time_kernel<NM, TA, ELECT>;
      cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaMemset(d, 0, 64);
      const int reps = 400;
      const int tmemN = N > 32 ? 32 : N;  // N=128 only with A from SMEM (D would overlap A)
      if (TA && N > 32) continue;
      fn<<<sms * per, 128, smem>>>(N > 32 ? N : tmemN, reps, per == 4, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[4];
      cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
      printf("%s CTAs/SM %d N %3d A=%s MMAs %2d: issue %6.0f clk, issue->complete %6.0f clk", ELECT ? "elect " : "tid==0",
             per, N, TA ? "TMEM" : "SMEM", NM, (double)h[0] / h[2] / reps, (double)h[1] / h[2] / reps);
      if (per == 4) printf(", st 6 x16 + wait %5.0f clk", (double)h[3] / h[2] / reps);
      printf(" (%s)\n", cudaGetErrorString(e));
    }
}

static float trunc_tf32(float v) {
  uint32_t b;
  std::memcpy(&b, &v, 4);
  b &= 0xFFFFE000u;
  std::memcpy(&v, &b, 4);
  return v;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // (1) correctness
  for (int N : {16, 32}) {
    const int K = 96;
    std::vector<float> E(128 * K), V(K * N), D(128 * N);
    unsigned s = 12345;
    auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (float)((s >> 8) & 0xFFFFFF) / 16777216.0f - 0.5f; };
    for (auto &v : E) v = rnd();
    for (auto &v : V) v = rnd();
    float *dE, *dV, *dD;
    cudaMalloc(&dE, E.size() * 4);
    cudaMalloc(&dV, V.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dE, E.data(), E.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dV, V.data(), V.size() * 4, cudaMemcpyHostToDevice);
    const int smem = 16 * NMAX * 32;
    cudaFuncSetAttribute((const void *)check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    check_kernel<<<1, 128, smem>>>(dE, dV, K, N, dD);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr_t = 0, maxerr_f = 0, scale = 0;
    for (int r = 0; r < 128; ++r)
      for (int n = 0; n < N; ++n) {
        double st = 0, sf = 0;
        for (int k = 0; k < K; ++k) {
          st += (double)trunc_tf32(E[r * K + k]) * (double)trunc_tf32(V[k * N + n]);
          sf += (double)E[r * K + k] * (double)V[k * N + n];
        }
        maxerr_t = std::fmax(maxerr_t, std::fabs(st - D[r * N + n]));
        maxerr_f = std::fmax(maxerr_f, std::fabs(sf - D[r * N + n]));
        scale = std::fmax(scale, std::fabs(sf));
      }
    printf("check A=TMEM K=%d N=%d: max |D - tf32-trunc GEMM| %.3e, max |D - fp32 GEMM| %.3e (scale %.2f) (%s)\n", K,
           N, maxerr_t, maxerr_f, scale, cudaGetErrorString(e));
  }
  // (2)/(3) timing
  unsigned long long *d;
  cudaMalloc(&d, 64);
  run_time<2, true, false>(sms, d);
  run_time<8, true, false>(sms, d);
  run_time<24, true, false>(sms, d);
  run_time<2, true, true>(sms, d);
  run_time<8, true, true>(sms, d);
  run_time<24, true, true>(sms, d);
  run_time<40, true, true>(sms, d);
  run_time<2, false, true>(sms, d);
  run_time<8, false, true>(sms, d);
  run_time<24, false, true>(sms, d);
  return 0;
}
