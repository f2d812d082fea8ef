// Co-scheduling study: can the issue-bound rollout work run on the SMs NEXT TO the
// MUFU-bound LWPR kernel?  lwpr_tc_kernel is launched persistent with kTcCtasPerSm CTAs
// per SM (build with -DPI2_TC_CTAS=3 to leave a quarter of the register file free), a
// rollout-like filler (Philox4x32-10 + Box-Muller + the integration/cost FP32 mix, one
// thread per sub-rollout, 50 steps) on a second stream.  Times: LWPR alone, filler alone,
// both launched together (CUDA events around both streams).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//          -I paper_1503_00330_b200/csrc -DPI2_TC_CTAS=3 -o lwpr_corun profiles/micro/lwpr_corun.cu
#include <cstdio>
#include <vector>

#include "lwpr_tc.cuh"

using namespace pi2;

static uint64_t s_rng = 88172645463325252ull;
static double urand() {
  s_rng ^= s_rng << 13; s_rng ^= s_rng >> 7; s_rng ^= s_rng << 17;
  return (s_rng >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void __launch_bounds__(256) filler_kernel(int64_t n, int steps, const float *planes, int64_t plane, float *out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float cs[3] = {0.f, 0.f, 0.f}, ccs[3] = {0.f, 0.f, 0.f}, q = 0.f;
  const int64_t k = i >> 2;
  for (int t = 0; t < steps; ++t) {
    const float4 z = normals4((uint64_t)i * steps + t, 0x1234567887654321ull, 0x0badf00dcafef00dull);
    const float d[3] = {z.x, z.y, z.z};
    const int64_t row = (int64_t)t * (n >> 2) + k;
    float pos[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float mn = __ldcg(planes + c * plane + row), sd = __ldcg(planes + (3 + c) * plane + row);
      const float acc = __fadd_rn(__fmul_rn(sd, d[c]), mn);
      cs[c] = __fadd_rn(cs[c], acc);
      ccs[c] = __fadd_rn(ccs[c], cs[c]);
      pos[c] = __fadd_rn(__fmul_rn(__fsub_rn(ccs[c], cs[c]), 1e-4f), __fmul_rn(cs[c], 0.01f));
    }
    float o = __fmul_rn(pos[0], pos[0]);
    o = __fadd_rn(o, __fmul_rn(pos[1], pos[1]));
    o = __fadd_rn(o, __fmul_rn(__fmul_rn(pos[2], pos[2]), 10.0f));
#pragma unroll
    for (int ob = 0; ob < 3; ++ob) {
      const float dx = __fsub_rn(pos[0], 0.3f * ob), dy = __fsub_rn(pos[1], -0.2f * ob);
      const float tt = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
      o = __fadd_rn(o, __fmul_rn(ex2_ftz(__fmul_rn(tt, -14.4269504f)), 100.0f));
    }
    // the M-mean butterfly of 4 lanes
    o = __fmul_rn(0.5f, __fadd_rn(o, __shfl_xor_sync(0xffffffffu, o, 1)));
    o = __fmul_rn(0.5f, __fadd_rn(o, __shfl_xor_sync(0xffffffffu, o, 2)));
    q = __fadd_rn(q, o);
  }
  out[i] = q;
}

int main(int argc, char **argv) {
  const int64_t rows = 65536ll * 50;
  const int L = 100;
  const int64_t nfill = argc > 1 ? atoll(argv[1]) : 65536ll * 4;  // sub-rollouts (C2: K x M)
  AxisRaw ax[3];
  const double lo[4] = {-0.35, -0.35, -0.35, 0.10}, hi[4] = {0.35, 0.35, 0.35, 0.28};
  const double md[4] = {30, 30, 30, 1500};
  for (auto &a : ax) {
    a.L = L; a.d = 4;
    for (int l = 0; l < L; ++l) {
      for (int i = 0; i < 4; ++i) a.centers.push_back(lo[i] + (hi[i] - lo[i]) * urand());
      for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) a.metrics.push_back(i == j ? md[i] : 0.0);
      for (int i = 0; i < 5; ++i) a.coefs.push_back(4.0 * (urand() - 0.5));
      a.lvar.push_back(0.01 + 0.09 * urand());
    }
  }
  std::vector<float> rec;
  AxisHeader hdr[3];
  for (int i = 0; i < 3; ++i) fold_axis(ax[i], kLayShared, rec, hdr[i]);
  std::vector<float> blob;
  LwprTcArgs ta{};
  if (!build_tc_weights(ax, blob, ta)) { printf("not tc-eligible\n"); return 1; }
  std::vector<float4> hx(rows);
  for (auto &v : hx)
    v = make_float4(0.8 * (urand() - 0.5), 0.8 * (urand() - 0.5), 0.8 * (urand() - 0.5), 0.05 + 0.3 * urand());
  float4 *dx; float *dparams, *dblob, *m2, *s2, *planes, *fout;
  cudaMalloc(&dx, rows * 16); cudaMalloc(&m2, rows * 16); cudaMalloc(&s2, rows * 16);
  cudaMalloc(&dparams, rec.size() * 4); cudaMalloc(&dblob, blob.size() * 4);
  cudaMalloc(&planes, rows * 6 * 4); cudaMalloc(&fout, nfill * 4);
  cudaMemset(planes, 0, rows * 24);
  cudaMemcpy(dx, hx.data(), rows * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(dparams, rec.data(), rec.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dblob, blob.data(), blob.size() * 4, cudaMemcpyHostToDevice);
  ta.params = dparams;
  for (int i = 0; i < 3; ++i) ta.axis[i] = hdr[i];
  ta.w = dblob; ta.rows = rows; ta.x = dx; ta.mean_out = m2; ta.sd_out = s2; ta.plane = rows; ta.sqrt_out = 1;
  int64_t wmax = 0;
  for (int i = 0; i < 3; ++i) {
    const int64_t we = i < 2 ? ta.axis_off[i + 1] : ta.w_floats;
    wmax = std::max<int64_t>(wmax, we - ta.axis_off[i] + (int64_t)ta.nchunks[i] * kTcChunk);
  }
  auto *k2 = lwpr_tc_kernel<true, false, false, 5>;
  // this axis' W + variances + two A operands, no padding: the persistent grid of
  // kTcCtasPerSm x SMs keeps the LWPR CTAs at kTcCtasPerSm per SM
  const int smem2 = (int)((wmax * 4 + 127) / 128 * 128 + 2 * kTcABytes);
  cudaFuncSetAttribute((const void *)k2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int per_sm = argc > 2 ? atoi(argv[2]) : kTcCtasPerSm;  // LWPR CTAs launched per SM
  const unsigned g2 = (per_sm * sms) / 3 * 3;
  cudaFuncAttributes fa{}, fb{};
  cudaFuncGetAttributes(&fa, (const void *)k2);
  cudaFuncGetAttributes(&fb, (const void *)filler_kernel);
  printf("LWPR CTAs/SM %d (built for %d), %d regs, smem %d B; filler %d regs, %lld threads\n", per_sm, kTcCtasPerSm, fa.numRegs, smem2, fb.numRegs,
         (long long)nfill);
  cudaStream_t sa, sb; cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, ea, eb; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&ea); cudaEventCreate(&eb);
  const unsigned gf = (unsigned)((nfill + 255) / 256);
  auto run = [&](int mode) {  // 1 LWPR, 2 filler, 3 both (LWPR first), 4 both sequential
    cudaEventRecord(e0, sa);
    cudaStreamWaitEvent(sb, e0);
    if (mode == 4) {
      k2<<<g2, kTcThreads, smem2, sa>>>(ta);
      filler_kernel<<<gf, 256, 0, sa>>>(nfill, 50, planes, rows, fout);
    } else {
      if (mode & 1) k2<<<g2, kTcThreads, smem2, sa>>>(ta);
      if (mode & 2) filler_kernel<<<gf, 256, 0, sb>>>(nfill, 50, planes, rows, fout);
    }
    cudaEventRecord(eb, sb);
    cudaStreamWaitEvent(sa, eb);
    cudaEventRecord(e1, sa);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
  };
  for (int r = 0; r < 2; ++r) {
    for (int mode : {1, 2, 4, 3}) {
      run(mode);
      float best = 1e9;
      for (int i = 0; i < 5; ++i) best = std::min(best, run(mode));
      printf("  %-26s %8.1f us\n", mode == 1 ? "LWPR alone" : mode == 2 ? "filler alone" : mode == 4 ? "LWPR then filler (1 stream)" : "LWPR || filler (2 streams)", best * 1e3);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
