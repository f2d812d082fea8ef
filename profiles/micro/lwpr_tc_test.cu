// Tensor-core LWPR (lwpr_tc_kernel) vs the CUDA-core kernel on a C2-sized batch:
// max |diff| of mean/std and device time of both.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//          -I paper_1503_00330_b200/csrc -o lwpr_tc_test profiles/micro/lwpr_tc_test.cu
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <vector>

#include "lwpr_tc.cuh"

using namespace pi2;

static uint64_t s_rng = 88172645463325252ull;
static uint64_t fnv(const std::vector<float> &v, int64_t n) {  // bit hash of the first n floats
  uint64_t h = 1469598103934665603ull;
  for (int64_t i = 0; i < n; ++i) {
    uint32_t b;
    memcpy(&b, &v[i], 4);
    h = (h ^ b) * 1099511628211ull;
  }
  return h;
}
static double urand() {
  s_rng ^= s_rng << 13; s_rng ^= s_rng >> 7; s_rng ^= s_rng << 17;
  return (s_rng >> 11) * (1.0 / 9007199254740992.0);
}

int main(int argc, char **argv) {
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 65536ll * 50;
  const int L = argc > 2 ? atoi(argv[2]) : 100;
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
  float4 *dx; float *dparams, *dblob, *m1, *s1, *m2, *s2;
  cudaMalloc(&dx, rows * 16); cudaMalloc(&m1, rows * 16); cudaMalloc(&s1, rows * 16);
  cudaMalloc(&m2, rows * 16); cudaMalloc(&s2, rows * 16);
  cudaMalloc(&dparams, rec.size() * 4); cudaMalloc(&dblob, blob.size() * 4);
  cudaMemcpy(dx, hx.data(), rows * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(dparams, rec.data(), rec.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dblob, blob.data(), blob.size() * 4, cudaMemcpyHostToDevice);

  LwprArgs la{};
  la.params = dparams;
  for (int i = 0; i < 3; ++i) la.axis[i] = hdr[i];
  la.a_begin = 0; la.a_end = 3; la.layout = kLayShared; la.resident = 1;
  la.rows = rows; la.x = dx; la.mean_out = m1; la.sd_out = s1; la.row_stride = 1; la.axis_stride = rows; la.sqrt_out = 1;
  const int smem1 = (int)(rec.size() * 4);
  auto *k1 = lwpr_kernel<kLayShared, true, 8>;
  cudaFuncSetAttribute((const void *)k1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem1);
  const unsigned g1 = (unsigned)((rows + 1023) / 1024);

  ta.params = dparams;
  for (int i = 0; i < 3; ++i) ta.axis[i] = hdr[i];
  ta.w = dblob; ta.rows = rows; ta.x = dx; ta.mean_out = m2; ta.sd_out = s2; ta.plane = rows; ta.sqrt_out = 1;
  int64_t wmax = 0;
  for (int i = 0; i < 3; ++i) {
    const int64_t we = i < 2 ? ta.axis_off[i + 1] : ta.w_floats;
    wmax = std::max<int64_t>(wmax, we - ta.axis_off[i] + (int64_t)ta.nchunks[i] * kTcChunk);
  }
  // at most kTcCtasPerSm co-resident CTAs (their TMEM allocations must all fit)
  int64_t lvmax = 0;
  for (int i = 0; i < 3; ++i) lvmax = std::max<int64_t>(lvmax, (int64_t)ta.nchunks[i] * kTcChunk);
  // the product's resident instantiation: remainder chunk unrolled at its batch count
  using Fn = void (*)(LwprTcArgs);
  const Fn kv[8] = {lwpr_tc_kernel<true, false, false, 0>, lwpr_tc_kernel<true, false, false, 1>,
                    lwpr_tc_kernel<true, false, false, 2>, lwpr_tc_kernel<true, false, false, 3>,
                    lwpr_tc_kernel<true, false, false, 4>, lwpr_tc_kernel<true, false, false, 5>,
                    lwpr_tc_kernel<true, false, false, 6>, lwpr_tc_kernel<true, false, false, 7>};
  const Fn km[8] = {lwpr_tc_kernel<false, false, false, 0>, lwpr_tc_kernel<false, false, false, 1>,
                    lwpr_tc_kernel<false, false, false, 2>, lwpr_tc_kernel<false, false, false, 3>,
                    lwpr_tc_kernel<false, false, false, 4>, lwpr_tc_kernel<false, false, false, 5>,
                    lwpr_tc_kernel<false, false, false, 6>, lwpr_tc_kernel<false, false, false, 7>};
  const int remb = getenv("REMB0") ? 0 : tc_remainder_batches(ta);
  auto *k2 = kv[remb];
  auto *k4 = km[remb];
  int smem2 = tc_smem_bytes(wmax, (const void *)k2);
  const bool stream = smem2 < 0 || getenv("STREAM");
  if (stream) {  // W streamed per chunk
    k2 = lwpr_tc_kernel<true, true>;
    k4 = lwpr_tc_kernel<false, true>;
    smem2 = tc_smem_bytes(2 * kTcWSlotFloats + lvmax, (const void *)k2);
  }
  const int tc_threads = kTcThreads, tc_per_sm = kTcCtasPerSm;
  printf("W %s\n", stream ? "streamed" : "resident");
  if (smem2 < 0) { printf("does not fit %d CTAs/SM\n", tc_per_sm); return 1; }
  cudaFuncSetAttribute((const void *)k2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const unsigned g2 = (tc_per_sm * sms) / 3 * 3;
  printf("CTAS %d CHUNK %d\n", PI2_TC_CTAS, PI2_TC_CHUNK);
  printf("rows %lld L %d: W %lld floats, lv %lld, smem tc %d B, chunks %d pad %d\n", (long long)rows, L,
         (long long)ta.w_floats, (long long)ta.lv_floats, smem2, ta.nchunks[0], ta.chunk_pad[0][0]);

  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms1, ms2;
  k1<<<g1, 128, smem1>>>(la);
  k2<<<g2, tc_threads, smem2>>>(ta);
  cudaError_t err = cudaDeviceSynchronize();
  printf("first run: %s\n", cudaGetErrorString(err));
  if (err != cudaSuccess) return 2;
  cudaEventRecord(e0); for (int r = 0; r < 5; ++r) k1<<<g1, 128, smem1>>>(la); cudaEventRecord(e1);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms1, e0, e1);
  cudaEventRecord(e0); for (int r = 0; r < 5; ++r) k2<<<g2, tc_threads, smem2>>>(ta); cudaEventRecord(e1);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms2, e0, e1);
#ifdef PI2_TC_TRACE
  {  // one traced launch: per SM sub-partition (hw warp slot % 4), time share with n warps in the exp phase
    const int on = 1;
    unsigned zero = 0;
    void *tbuf;
    cudaGetSymbolAddress(&tbuf, g_tc_trace);
    cudaMemset(tbuf, 0, sizeof(unsigned long long) * 64 * kTcTraceCap);
    cudaMemcpyToSymbol(g_tc_trace_n, &zero, 4);
    cudaMemcpyToSymbol(g_tc_trace_on, &on, 4);
    k2<<<g2, tc_threads, smem2>>>(ta);
    cudaDeviceSynchronize();
    const int off = 0;
    cudaMemcpyToSymbol(g_tc_trace_on, &off, 4);
    std::vector<unsigned long long> all(64 * kTcTraceCap), ev;
    cudaMemcpy(all.data(), tbuf, all.size() * 8, cudaMemcpyDeviceToHost);
    for (auto e : all)
      if (e) ev.push_back(e);
    const unsigned n = (unsigned)ev.size();
    std::sort(ev.begin(), ev.end());
    // per warp slot: last event clock; interval (last, now] is the phase that ended now
    std::vector<long long> last(64, -1);
    std::vector<int> inexp(4, 0);
    std::vector<int> cur(64, -1);  // phase the warp is in (known only after its event) -- use end-labelled intervals
    // build intervals
    struct Iv { long long a, b; int w, ph; };
    std::vector<Iv> iv;
    for (auto e : ev) {
      const long long c = (long long)(e >> 20);
      const int w = (int)((e >> 4) & 63), ph = (int)(e & 15);
      if (last[w] >= 0) iv.push_back({last[w], c, w, ph});
      last[w] = c;
    }
    long long t0 = 1LL << 62, t1 = 0;
    for (auto &v : iv) { t0 = std::min(t0, v.a); t1 = std::max(t1, v.b); }
    for (int sp = 0; sp < 4; ++sp) {
      std::vector<std::pair<long long, int>> d;
      double ph_tot[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (auto &v : iv)
        if (v.w % 4 == sp) {
          ph_tot[v.ph] += (double)(v.b - v.a);
          if (v.ph == 3) { d.push_back({v.a, 1}); d.push_back({v.b, -1}); }
        }
      std::sort(d.begin(), d.end());
      double hist[9] = {0};
      int k = 0; long long prev = t0;
      for (auto &x : d) { hist[std::min(k, 8)] += (double)(x.first - prev); prev = x.first; k += x.second; }
      hist[0] += (double)(t1 - prev);
      const double T = (double)(t1 - t0);
      printf("SMSP %d (%.0f clk): time with n warps in exp:", sp, T);
      for (int i = 0; i < 6; ++i) printf(" %d:%.2f", i, hist[i] / T);
      printf("   phase clk: ph0 %.0f ph1 %.0f mma %.0f exp %.0f ph5 %.0f ph6 %.0f ph7 %.0f\n", ph_tot[0], ph_tot[1], ph_tot[2], ph_tot[3], ph_tot[5], ph_tot[6], ph_tot[7]);
    }
    printf("events %u\n", n);
    // timeline sample: every warp of SM 0, a window after the start
    const long long w0 = getenv("TRACE_FROM") ? atoll(getenv("TRACE_FROM")) : 100000, w1 = w0 + 12000;
    int shown = 0;
    for (auto &v : iv)
      if (v.a - t0 >= w0 && v.a - t0 < w1 && shown < 400) {
        printf("  w%02d %7lld-%7lld ph%d (%lld)\n", v.w, v.a - t0, v.b - t0, v.ph, v.b - v.a);
        ++shown;
      }
  }
#endif
#ifdef PI2_TC_PROF
  {
    unsigned long long pr[5];
    cudaMemcpyFromSymbol(pr, g_tc_prof, sizeof(pr));
    double tot = 0;
    for (auto v : pr) tot += (double)v;
    const double n = 6.0 * ((rows + 127) / 128) * 3 * 4;  // warp-tile-axes over 6 launches (4 row warps per CTA)
    printf("clocks per warp-tile-axis: features+finalize %.0f  barrier %.0f  mma-wait %.0f  exp %.0f  tail %.0f  total %.0f\n",
           pr[0] / n, pr[1] / n, pr[2] / n, pr[3] / n, pr[4] / n, tot / n);
  }
#endif
  std::vector<float> a1(rows * 4), b1(rows * 4), a2(rows * 4), b2(rows * 4);
  cudaMemcpy(a1.data(), m1, rows * 16, cudaMemcpyDeviceToHost); cudaMemcpy(b1.data(), s1, rows * 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(a2.data(), m2, rows * 16, cudaMemcpyDeviceToHost); cudaMemcpy(b2.data(), s2, rows * 16, cudaMemcpyDeviceToHost);
  double dm = 0, ds = 0, mm = 0;
  int64_t bad = 0;
  for (int64_t i = 0; i < rows * 4; ++i) {
    const double d1 = fabs(a1[i] - a2[i]), d2 = fabs(b1[i] - b2[i]) / fmax(1e-6, fabs(b1[i]));
    if (!(d1 <= 1e30)) ++bad;
    dm = fmax(dm, d1); ds = fmax(ds, d2); mm = fmax(mm, fabs(a1[i]));
  }
  const double flops = (double)rows * 3 * L * 32;
  printf("cuda-core: %8.1f us (%.1f TFLOP/s alg)   tensor-core: %8.1f us (%.1f TFLOP/s alg)\n", ms1 / 5 * 1e3,
         flops / (ms1 / 5) / 1e9, ms2 / 5 * 1e3, flops / (ms2 / 5) / 1e9);
  printf("max |dmean| %.3e (max |mean| %.2f), max rel dstd %.3e, nan/inf %lld\n", dm, mm, ds, (long long)bad);
  printf("sample: cc %f %f tc %f %f\n", a1[0], b1[0], a2[0], b2[0]);
  printf("tc output hash: mean %016llx std %016llx\n", (unsigned long long)fnv(a2, rows * 3), (unsigned long long)fnv(b2, rows * 3));
  {  // mean only (M = 1 rollouts)
    auto *k3 = lwpr_kernel<kLayShared, false, 8>;
    cudaFuncSetAttribute((const void *)k3, cudaFuncAttributeMaxDynamicSharedMemorySize, smem1);
    cudaFuncSetAttribute((const void *)k4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    la.sd_out = nullptr;
    ta.sd_out = nullptr;
    k3<<<g1, 128, smem1>>>(la);
    k4<<<g2, tc_threads, smem2>>>(ta);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) k3<<<g1, 128, smem1>>>(la); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms1, e0, e1);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) k4<<<g2, tc_threads, smem2>>>(ta); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms2, e0, e1);
    cudaMemcpy(a1.data(), m1, rows * 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(a2.data(), m2, rows * 16, cudaMemcpyDeviceToHost);
    double dm0 = 0;
    for (int64_t i = 0; i < rows * 4; ++i) dm0 = fmax(dm0, fabs(a1[i] - a2[i]));
    printf("tc mean-only output hash: %016llx\n", (unsigned long long)fnv(a2, rows * 3));
    printf("mean-only  cuda-core: %8.1f us   tensor-core: %8.1f us   max |dmean| %.3e   (%s)\n", ms1 / 5 * 1e3,
           ms2 / 5 * 1e3, dm0, cudaGetErrorString(cudaDeviceSynchronize()));
  }
  return 0;
}
