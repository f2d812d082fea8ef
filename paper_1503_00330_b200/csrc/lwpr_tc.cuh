// lwpr_tc.cuh — LWPR predict with the field GEMM on the 5th-gen tensor cores.
//
// For a metric shared by all fields of an axis (kLayShared) both per-field
// quantities the CUDA-core kernel spends 8 of its 14 FMA-pipe ops on are
// affine in the row features f(x) = [x~0, x~1, x~2, x~3, 1, q~, 0, 0]:
//   logit2_l(x) = DC_l.x~ + A0_l + q~      (log2-scaled, + 2^64 shift in A0)
//   y'_l(x)     = S'_l.x~ + Y0'_l          (local model minus g(x))
// so one GEMM D[128 rows, 2*Lc] = F[128, 8] . W[2*Lc, 8]^T per 128-row tile
// and field chunk (Lc <= 128 fields) puts both in TMEM.  The GEMM runs as
// 3xTF32 (hi.hi + hi.lo + lo.hi, fp32 accumulate) — tests/test_tc_emulation.py
// shows this keeps the LWPR mean within 1e-5 of the reference.  The CUDA cores
// then only do  e = 2^logit (MUFU), den += e, num += e y', m2 += e y'^2,
// lv += e var  on field pairs (FFMA2): the kernel becomes MUFU-bound.
//
// tcgen05 usage: 1 CTA = 128 threads = 4 warps, warp w owns TMEM lanes
// 32w..32w+31 = tile rows; thread 0 issues the 3 MMAs and commits to an
// mbarrier; operands are K-major, no swizzle (8x16B core matrices,
// LBO = 128 B between the two K halves, SBO = 256 B between 8-row groups).
// Persistent CTAs keep all axes' W in shared memory; 2 CTAs per SM (256 TMEM
// columns each) overlap one CTA's MMA with the other's exp phase.
#pragma once

#include <vector>

#include "fold.h"
#include "kernels.cuh"

namespace pi2 {

#ifndef PI2_TC_CHUNK
#define PI2_TC_CHUNK 64
#endif
#ifndef PI2_TC_CTAS
#define PI2_TC_CTAS 4
#endif
constexpr int kTcChunk = PI2_TC_CHUNK;        // max fields per MMA chunk (N = 2 * kTcChunk TMEM columns)
constexpr int kTcTmemCols = 2 * PI2_TC_CHUNK;  // power of two >= 32

constexpr int kTcMaxChunks = 16;    // fields per axis <= 16 * kTcChunk on this path

struct LwprTcArgs {
  const float *w;        // per axis, per chunk: W_hi then W_lo, each (2*Lc_pad rows x 8) in UMMA layout,
                         // then per axis the chunk-padded local variances
  int64_t w_floats;      // floats of the W matrices
  int64_t lv_floats;     // floats of the variance block (3 * nchunks * kTcChunk max)
  int64_t axis_off[3];   // float offset of each axis' first chunk in w
  int64_t lv_off[3];     // float offset of each axis' variances (after the W matrices)
  int nchunks[3];
  int chunk_pad[3][kTcMaxChunks];  // padded field count of each chunk (multiple of 16), <= kTcChunk
  AxisHeader axis[3];    // headers of the kLayShared records (exact path, g, mu, qd)
  const float *params;   // kLayShared records (exact path)
  int64_t rows;
  const float4 *x;
  float *mean_out, *sd_out;  // float4 rows (xyz = axes, w = 0)
  int sqrt_out;
};

// byte offset of element (row, k) in a K-major no-swizzle operand, K = 8 (fp32/tf32)
__host__ __device__ __forceinline__ uint32_t umma_kmajor_off(int row, int k) {
  return (uint32_t)(((row & 7) + (row >> 3) * 16 + (k >> 2) * 8) * 16 + (k & 3) * 4);
}

__device__ __forceinline__ uint64_t umma_smem_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);        // start address
  d |= (uint64_t)(128 >> 4) << 16;                // LBO: next K half (core matrix) 128 B
  d |= (uint64_t)(256 >> 4) << 32;                // SBO: next 8-row group 256 B
  d |= (uint64_t)1 << 46;                         // descriptor version (sm_100)
  return d;                                       // base offset 0, lbo mode 0, SWIZZLE_NONE
}

__device__ __forceinline__ uint32_t umma_idesc_tf32(int M, int N) {
  return (1u << 4)                                // D format F32
         | (2u << 7) | (2u << 10)                 // A, B format TF32
         | ((uint32_t)(N >> 3) << 17)             // N / 8
         | ((uint32_t)(M >> 4) << 24);            // M / 16
}

__device__ __forceinline__ float tf32_rna(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, int acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(mbar),
      "r"(phase));
}

#define PI2_TMEM_LD8(r, addr)                                                                      \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                \
               : "=r"((r)[0]), "=r"((r)[1]), "=r"((r)[2]), "=r"((r)[3]), "=r"((r)[4]), "=r"((r)[5]), \
                 "=r"((r)[6]), "=r"((r)[7])                                                            \
               : "r"(addr))

constexpr int kTcThreads = 128;  // 4 warps: warp w owns TMEM lanes 32w..32w+31 (tile rows)
constexpr int kTcCtasPerSm = PI2_TC_CTAS;  // co-resident CTAs: their MMA phases interleave

template <bool VAR>
__global__ void __launch_bounds__(kTcThreads, kTcCtasPerSm) lwpr_tc_kernel(LwprTcArgs a) {
  extern __shared__ __align__(128) uint8_t tsm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  // CTA i evaluates axis i % 3 for tiles i / 3, i / 3 + gridDim.x / 3, ...: only that
  // axis' weights (W chunks, then its chunk-padded variances) live in shared memory
  const int ax = blockIdx.x % 3;
  const int64_t wbeg = a.axis_off[ax], wend = ax < 2 ? a.axis_off[ax + 1] : a.w_floats;
  const int64_t nlv = (int64_t)a.nchunks[ax] * kTcChunk;
  float *sw = reinterpret_cast<float *>(tsm);
  float *slv_base = sw + (wend - wbeg);
  uint8_t *sa = tsm + (((wend - wbeg + nlv) * 4 + 127) / 128) * 128;  // A_hi | A_lo, 4 KB each
  const int tid = threadIdx.x, warp = tid >> 5;

  for (int64_t i = tid; i < (wend - wbeg) / 4; i += blockDim.x)
    reinterpret_cast<float4 *>(sw)[i] = __ldg(reinterpret_cast<const float4 *>(a.w + wbeg) + i);
  for (int64_t i = tid; i < nlv; i += blockDim.x) slv_base[i] = __ldg(a.w + a.lv_off[ax] + i);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)),
                 "n"(kTcTmemCols));
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
  const uint32_t tmem = tmem_base;
  const uint32_t tmem_lane = tmem + ((uint32_t)(warp * 32) << 16);
  const uint32_t sa_addr = (uint32_t)__cvta_generic_to_shared(sa);
  const uint32_t sw_addr = (uint32_t)__cvta_generic_to_shared(sw);
  uint32_t phase = 0;

  const int64_t ntiles = (a.rows + 127) / 128;
  const int64_t tstride = gridDim.x / 3;
  for (int64_t tile = blockIdx.x / 3; tile < ntiles; tile += tstride) {
    const int64_t row = tile * 128 + tid;
    const float4 x = __ldg(a.x + (row < a.rows ? row : a.rows - 1));
    {
      const AxisHeader h = a.axis[ax];
      const float4 xt = make_float4(__fsub_rn(x.x, h.mu[0]), __fsub_rn(x.y, h.mu[1]), __fsub_rn(x.z, h.mu[2]),
                                    __fsub_rn(x.w, h.mu[3]));
      const float q = shared_qrow(h, xt);
      {  // row features, hi and lo tf32 parts, into the A operands
        const float f[8] = {xt.x, xt.y, xt.z, xt.w, 1.0f, q, 0.0f, 0.0f};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float hi = tf32_rna(f[k]);
          *reinterpret_cast<float *>(sa + umma_kmajor_off(tid, k)) = hi;
          *reinterpret_cast<float *>(sa + 4096 + umma_kmajor_off(tid, k)) = tf32_rna(__fsub_rn(f[k], hi));
        }
      }
      float2 den = make_float2(0.f, 0.f), num = den, m2 = den, lv = den;
      int64_t woff = 0;  // within this axis' block in shared memory
      for (int c = 0; c < a.nchunks[ax]; ++c) {
        const int lc = a.chunk_pad[ax][c];  // fields of this chunk, multiple of 8, 2 lc <= 128 columns
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();  // A written, TMEM free
        if (tid == 0) {
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t idesc = umma_idesc_tf32(128, 2 * lc);
          const uint64_t a_hi = umma_smem_desc(sa_addr), a_lo = umma_smem_desc(sa_addr + 4096);
          const uint32_t wb = sw_addr + (uint32_t)(woff * 4);
          const uint64_t b_hi = umma_smem_desc(wb), b_lo = umma_smem_desc(wb + (uint32_t)(2 * lc * 8 * 4));
          mma_tf32(tmem, a_hi, b_hi, idesc, 0);
          mma_tf32(tmem, a_hi, b_lo, idesc, 1);
          mma_tf32(tmem, a_lo, b_hi, idesc, 1);
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              mbar_addr));
        }
        mbar_wait(mbar_addr, phase);
        phase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;");
        const float *slv = slv_base + (int64_t)c * kTcChunk;
        for (int j = 0; j < lc; j += 16) {
          const int nb = min(2, (lc - j) >> 3);
          uint32_t lg[16], yy[16];
          PI2_TMEM_LD8(lg, tmem_lane + j);
          PI2_TMEM_LD8(yy, tmem_lane + lc + j);
          if (nb == 2) {
            PI2_TMEM_LD8(lg + 8, tmem_lane + j + 8);
            PI2_TMEM_LD8(yy + 8, tmem_lane + lc + j + 8);
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            if (i >= 8 * nb) break;
            const float2 e = make_float2(ex2_ftz(__uint_as_float(lg[i])), ex2_ftz(__uint_as_float(lg[i + 1])));
            const float2 y = make_float2(__uint_as_float(yy[i]), __uint_as_float(yy[i + 1]));
            den = __fadd2_rn(den, e);
            if (VAR) {
              const float2 ey = __fmul2_rn(e, y);
              num = __fadd2_rn(num, ey);
              m2 = __ffma2_rn(ey, y, m2);
              lv = __ffma2_rn(e, *reinterpret_cast<const float2 *>(slv + j + i), lv);
            } else {
              num = __ffma2_rn(e, y, num);
            }
          }
        }
        woff += (int64_t)2 * (2 * lc * 8);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      if (row < a.rows) {
        const float dn = __fadd_rn(den.x, den.y), nm = __fadd_rn(num.x, num.y);
        const float gx = fmaf(h.gs[3], xt.w, fmaf(h.gs[2], xt.z, fmaf(h.gs[1], xt.y, fmaf(h.gs[0], xt.x, h.g0))));
        float mean, var = 0.0f;
        if (dn >= kSlowDen) {
          const float mp = __fdiv_rn(nm, dn);
          mean = __fadd_rn(gx, mp);
          if (VAR) {
            const float s2 = __fadd_rn(__fadd_rn(m2.x, m2.y), __fadd_rn(lv.x, lv.y));
            var = fmaxf(__fsub_rn(__fdiv_rn(s2, dn), __fmul_rn(mp, mp)), 0.0f);
          }
        } else {
          lwpr_row_exact<kLayShared>(a.params + h.offset, h.num_fields, xt, q, gx, &mean, &var);
        }
        a.mean_out[row * 4 + ax] = mean;
        if (VAR && a.sd_out) a.sd_out[row * 4 + ax] = a.sqrt_out ? __fsqrt_rn(var) : var;
        if (ax == 2) {
          a.mean_out[row * 4 + 3] = 0.0f;
          if (VAR && a.sd_out) a.sd_out[row * 4 + 3] = 0.0f;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTcTmemCols));
}

// ---- host: W operands of the tensor-core path ------------------------------
// Same fold as fold_axis(kLayShared) in float64, split into tf32 hi + lo
// (round to nearest, ties away, like cvt.rna.tf32) and laid out K-major.
inline float host_tf32_rna(float v) {
  uint32_t b;
  std::memcpy(&b, &v, 4);
  if ((b & 0x7f800000u) != 0x7f800000u) b = (b + 0x1000u) & ~0x1FFFu;
  float r;
  std::memcpy(&r, &b, 4);
  return r;
}

inline bool build_tc_weights(const AxisRaw *axes, std::vector<float> &blob, LwprTcArgs &ta) {
  if (choose_layout(axes, 3) != kLayShared) return false;
  std::vector<float> lvs;
  int64_t w_floats = 0;
  for (int ax = 0; ax < 3; ++ax) {
    const AxisRaw &a = axes[ax];
    if (a.L <= 0 || a.d != 4 || a.L > kTcChunk * kTcMaxChunks) return false;
    // the same numbers as fold_axis(kLayShared), float64
    double mu[4] = {0, 0, 0, 0};
    for (int l = 0; l < a.L; ++l)
      for (int i = 0; i < 4; ++i) mu[i] += a.centers[(size_t)l * 4 + i];
    for (double &v : mu) v /= a.L;
    double D[4][4];
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) D[i][j] = a.metrics[(size_t)i * 4 + j];
    double g0 = 0, gs[4] = {0, 0, 0, 0};
    std::vector<double> y0(a.L);
    for (int l = 0; l < a.L; ++l) {
      double yy = a.coefs[(size_t)l * 5];
      for (int i = 0; i < 4; ++i) {
        yy -= a.coefs[(size_t)l * 5 + 1 + i] * (a.centers[(size_t)l * 4 + i] - mu[i]);
        gs[i] += a.coefs[(size_t)l * 5 + 1 + i];
      }
      y0[l] = yy;
      g0 += yy;
    }
    g0 /= a.L;
    for (double &v : gs) v /= a.L;
    ta.axis_off[ax] = w_floats;
    ta.nchunks[ax] = (a.L + kTcChunk - 1) / kTcChunk;
    const int per = (a.L + ta.nchunks[ax] - 1) / ta.nchunks[ax];  // even split, e.g. 100 -> 50 + 50
    for (int c = 0; c < ta.nchunks[ax]; ++c) {
      const int l0 = c * per, n = std::min(per, a.L - l0);
      const int lc = (n + 7) / 8 * 8;
      ta.chunk_pad[ax][c] = lc;
      std::vector<float> hi(2 * lc * 8, 0.0f), lo(2 * lc * 8, 0.0f);
      auto put = [&](int r, int k, double v) {
        const float f = (float)v, fh = host_tf32_rna(f);
        hi[umma_kmajor_off(r, k) / 4] = fh;
        lo[umma_kmajor_off(r, k) / 4] = host_tf32_rna(f - fh);
      };
      for (int j = 0; j < lc; ++j) {
        const int l = l0 + j;
        if (j >= n) {  // padding field: weight 2^-1000 = 0, prediction 0
          put(j, 4, -1000.0);
          continue;
        }
        double c4[4], dc[4], a0 = 0;
        for (int i = 0; i < 4; ++i) c4[i] = a.centers[(size_t)l * 4 + i] - mu[i];
        for (int i = 0; i < 4; ++i) {
          dc[i] = 0;
          for (int k = 0; k < 4; ++k) dc[i] += D[i][k] * c4[k];
        }
        for (int i = 0; i < 4; ++i) a0 += dc[i] * c4[i];
        a0 = -0.5 * a0;
        for (int i = 0; i < 4; ++i) put(j, i, dc[i] * kLog2e);   // logit row: DC . x~
        put(j, 4, a0 * kLog2e + kExpShift);                      //   + A0 (shifted)
        put(j, 5, 1.0);                                           //   + q~
        for (int i = 0; i < 4; ++i) put(lc + j, i, a.coefs[(size_t)l * 5 + 1 + i] - gs[i]);  // y' row
        put(lc + j, 4, y0[l] - g0);
      }
      blob.insert(blob.end(), hi.begin(), hi.end());
      blob.insert(blob.end(), lo.begin(), lo.end());
      w_floats += (int64_t)hi.size() + (int64_t)lo.size();
      for (int j = 0; j < kTcChunk; ++j) lvs.push_back(j < n ? (float)a.lvar[l0 + j] : 0.0f);
      (void)per;
    }
  }
  ta.w_floats = w_floats;
  int64_t off = w_floats;
  for (int ax = 0; ax < 3; ++ax) {
    ta.lv_off[ax] = off;
    off += (int64_t)ta.nchunks[ax] * kTcChunk;
  }
  ta.lv_floats = (int64_t)lvs.size();
  while (ta.lv_floats % 4) {  // float4 copies
    lvs.push_back(0.0f);
    ++ta.lv_floats;
  }
  blob.insert(blob.end(), lvs.begin(), lvs.end());
  return true;
}

}  // namespace pi2
