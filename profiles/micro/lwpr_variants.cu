// Sweep of lwpr_kernel variants (record layout, rows per thread, block size,
// min blocks/SM) on a C2-sized batch: 65536 x 50 rows, L=100 fields per axis,
// 3 axes, variance on.  Prints device time and algorithmic FP32 TFLOP/s
// (32 flops per (row, axis, field)).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//          -I paper_1503_00330_b200/csrc -o lwpr_variants profiles/micro/lwpr_variants.cu
#include <cstdio>
#include <vector>

#include "fold.h"
#include "kernels.cuh"

using namespace pi2;

static uint64_t s_rng = 88172645463325252ull;
static double urand() {
  s_rng ^= s_rng << 13; s_rng ^= s_rng >> 7; s_rng ^= s_rng << 17;
  return (s_rng >> 11) * (1.0 / 9007199254740992.0);
}

struct Setup {
  int layout;
  std::vector<float> rec;
  AxisHeader hdr[3];
};

static Setup make(int layout_override, int L) {
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
  Setup s;
  s.layout = layout_override >= 0 ? layout_override : choose_layout(ax, 3);
  for (int i = 0; i < 3; ++i) fold_axis(ax[i], s.layout, s.rec, s.hdr[i]);
  return s;
}

template <int LAY, bool VAR, int R, int BLOCK, int MINB>
float run(const Setup &s, const float *dparams, const float4 *dx, float *dm, float *ds, int64_t rows,
          const char *name, float *ref_m = nullptr) {
  LwprArgs a{};
  a.params = dparams;
  for (int i = 0; i < 3; ++i) a.axis[i] = s.hdr[i];
  a.a_begin = 0; a.a_end = 3; a.layout = LAY; a.resident = 1; a.tile = 0;
  a.rows = rows; a.x = dx; a.mean_out = dm; a.sd_out = VAR ? ds : nullptr; a.out_stride = 4; a.sqrt_out = 1;
  const int smem = (int)(s.rec.size() * sizeof(float));
  auto *fn = lwpr_kernel<LAY, VAR, R, BLOCK, MINB>;
  cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int64_t grid = (rows + (int64_t)BLOCK * R - 1) / ((int64_t)BLOCK * R);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  fn<<<(unsigned)grid, BLOCK, smem>>>(a);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) fn<<<(unsigned)grid, BLOCK, smem>>>(a);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const double flops = (double)rows * 3 * s.hdr[0].num_fields * 32;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, (const void *)fn);
  float maxdiff = 0;
  if (ref_m) {
    std::vector<float> h(rows * 4), r(rows * 4);
    cudaMemcpy(h.data(), dm, rows * 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(r.data(), ref_m, rows * 16, cudaMemcpyDeviceToHost);
    for (int64_t i = 0; i < rows * 4; ++i)
      if (i % 4 != 3) maxdiff = fmaxf(maxdiff, fabsf(h[i] - r[i]));
  }
  printf("%-34s regs %3d  %8.1f us  %6.2f TFLOP/s  (%.1f%% of 74.4)  maxdiff %.2e\n", name, fa.numRegs,
         ms * 1e3, flops / ms / 1e9, 100 * flops / ms / 1e9 / 74.45, maxdiff);
  return ms;
}

int main() {
  const int64_t rows = 65536ll * 50;
  const int L = 100;
  std::vector<float4> hx(rows);
  for (auto &v : hx)
    v = make_float4(0.8 * (urand() - 0.5), 0.8 * (urand() - 0.5), 0.8 * (urand() - 0.5), 0.05 + 0.3 * urand());
  float4 *dx;
  float *dm, *ds, *dref;
  cudaMalloc(&dx, rows * 16);
  cudaMalloc(&dm, rows * 16);
  cudaMalloc(&ds, rows * 16);
  cudaMalloc(&dref, rows * 16);
  cudaMemcpy(dx, hx.data(), rows * 16, cudaMemcpyHostToDevice);
  const uint64_t seed = s_rng;
  Setup diag = make(kLayDiag, L);
  s_rng = seed;  // same fields for both layouts
  Setup shared = make(-1, L);
  float *pd, *ps;
  cudaMalloc(&pd, diag.rec.size() * 4);
  cudaMalloc(&ps, shared.rec.size() * 4);
  cudaMemcpy(pd, diag.rec.data(), diag.rec.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(ps, shared.rec.data(), shared.rec.size() * 4, cudaMemcpyHostToDevice);
  printf("shared layout chosen: %d\n", shared.layout);

  run<kLayDiag, true, 8, 128, 4>(diag, pd, dx, dref, ds, rows, "diag  VAR R8  B128 m4 (prev)");
  run<kLayShared, true, 8, 128, 4>(shared, ps, dx, dm, ds, rows, "shared VAR R8  B128 m4", dref);
  run<kLayShared, true, 4, 128, 8>(shared, ps, dx, dm, ds, rows, "shared VAR R4  B128 m8", dref);
  run<kLayShared, true, 4, 256, 4>(shared, ps, dx, dm, ds, rows, "shared VAR R4  B256 m4", dref);
  run<kLayShared, true, 6, 128, 5>(shared, ps, dx, dm, ds, rows, "shared VAR R6  B128 m5", dref);
  run<kLayShared, true, 8, 256, 2>(shared, ps, dx, dm, ds, rows, "shared VAR R8  B256 m2", dref);
  run<kLayShared, true, 8, 64, 8>(shared, ps, dx, dm, ds, rows, "shared VAR R8  B64 m8", dref);
  run<kLayShared, true, 12, 128, 3>(shared, ps, dx, dm, ds, rows, "shared VAR R12 B128 m3", dref);
  run<kLayShared, true, 16, 128, 2>(shared, ps, dx, dm, ds, rows, "shared VAR R16 B128 m2", dref);
  run<kLayShared, true, 2, 128, 8>(shared, ps, dx, dm, ds, rows, "shared VAR R2  B128 m8", dref);
  run<kLayDiag, false, 8, 128, 4>(diag, pd, dx, dref, ds, rows, "diag  mean R8  B128 m4");
  run<kLayShared, false, 8, 128, 4>(shared, ps, dx, dm, ds, rows, "shared mean R8 B128 m4", dref);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
