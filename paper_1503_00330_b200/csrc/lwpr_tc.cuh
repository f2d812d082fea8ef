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
// then only do  e = 2^logit (MUFU), den += e, num += e y', m2 += e (y'^2 + var_l)
// on field pairs (FFMA2): the kernel becomes MUFU-bound.
//
// tcgen05 usage: 1 CTA = 128 threads = 4 warps, warp w owns TMEM lanes
// 32w..32w+31 = tile rows; thread 0 issues the 3 MMAs and commits to an
// mbarrier; operands are K-major, no swizzle (8x16B core matrices,
// LBO = 128 B between the two K halves, SBO = 256 B between 8-row groups).
// CTAs are axis-specialised (CTA i handles axis i % 3, tiles i / 3, i / 3 +
// gridDim / 3, ...) so only one axis' W sits in shared memory; 4 CTAs per SM
// (128 TMEM columns each, shared-memory request padded so no 5th CTA spins in
// tcgen05.alloc) overlap one CTA's MMA + TMEM latency with the others' exp
// phase.  Used for the variance path only: with 4 moments per field the
// CUDA-core kernel issues 14 FMA-pipe ops per field pair and the GEMM offload
// wins (C2 491 vs 510 us); the mean-only loop (10 ops) is already faster than
// this kernel's per-chunk synchronisation.
#pragma once

#include <type_traits>
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

constexpr int kTcMaxChunks = 32;    // fields per axis <= 32 * kTcChunk on this path
constexpr int kTcWSlotFloats = 2 * 2 * kTcChunk * 8;  // W of one chunk (hi + lo), streamed mode slot
constexpr int kTcBulkMaxTiles = 16;  // tiles per CTA up to which resident W arrives by bulk copy (WBULK)

struct LwprTcArgs {
  const float *w;        // per axis, per chunk: W_hi then W_lo, each (2*Lc_pad rows x 8) in UMMA layout,
                         // then per axis the chunk-padded local variances
  int64_t w_floats;      // floats of the W matrices
  int64_t lv_floats;     // floats of the variance block (3 * nchunks * kTcChunk max)
  int64_t axis_off[3];   // float offset of each axis' first chunk in w
  int64_t lv_off[3];     // float offset of each axis' variances (after the W matrices)
  int nchunks[3];
  int chunk_pad[3][kTcMaxChunks];  // padded field count of each chunk (multiple of 8), <= kTcChunk
  int chunk_woff[3][kTcMaxChunks]; // float offset of each chunk's W within its axis' block
  AxisHeader axis[3];    // headers of the kLayShared records (exact path, g, mu, qd)
  const float *params;   // kLayShared records (exact path)
  int64_t rows;
  const float4 *x;
  float *mean_out, *sd_out;  // planes: axis c of row r at [c * plane + r]
  int64_t plane;
  int sqrt_out;
  int sms;  // SM count: the MMA-issuing warp rotates over the co-resident CTAs (PI2_TC_ROTATE)
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

// tf32, round to nearest with ties away (cvt.rna.tf32.f32) for FINITE v, as two
// integer ops: the conversion instruction shares the MUFU/XU pipe with the 2^x
// flood of the co-resident warps and would queue behind it.  Non-finite rows
// never use the result (tc_finalize sends them to the exact path).
__device__ __forceinline__ float tf32_rna(float v) {
  return __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xFFFFE000u);
}

// 1/d and sqrt(v) on the FMA pipe (MUFU is saturated by the 2^x of the other warps):
// magic-constant seeds + Newton steps, relative error < 1e-7 for normal positive d
// and v (B200-independent host emulation); callers route anything else (0,
// denormals, inf, NaN) to the exact functions.
__device__ __forceinline__ float rcp_fma(float d) {
  float r = __uint_as_float(0x7EF311C3u - __float_as_uint(d));
#pragma unroll
  for (int i = 0; i < 3; ++i) r = __fmul_rn(r, __fmaf_rn(-d, r, 2.0f));
  return __fmaf_rn(r, __fmaf_rn(-d, r, 1.0f), r);
}
__device__ __forceinline__ float sqrt_fma(float v) {
  float y = __uint_as_float(0x5F3759DFu - (__float_as_uint(v) >> 1));  // ~ 1 / sqrt(v)
  const float h = __fmul_rn(0.5f, v);
#pragma unroll
  for (int i = 0; i < 3; ++i) y = __fmul_rn(y, __fmaf_rn(-h, __fmul_rn(y, y), 1.5f));
  const float s = __fmul_rn(v, y);  // sqrt(v), then one correction step
  return v > 0.0f ? __fmaf_rn(__fmaf_rn(-s, s, v), __fmul_rn(0.5f, y), s) : 0.0f;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, int acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// The same MMA issued by a converged warp: every lane executes the instruction and
// elect.sync picks one inside the asm, so the descriptors stay in uniform registers.
// Issued from a divergent `tid == 0` branch, ptxas wraps every UTCHMMA in an ELECT /
// BRA.U.ANY waterfall (profiles/micro/mma_tmem_a_b200.txt: 2 MMAs + commit issue in
// ~100 clocks converged vs ~260 from the divergent branch).
__device__ __forceinline__ void mma_tf32_elect(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, int acc) {
  asm volatile(
      "{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit_elect(uint32_t mbar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(mbar)
      : "memory");
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

#define PI2_TMEM_LD16(r, addr)                                                                     \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
               : "=r"((r)[0]), "=r"((r)[1]), "=r"((r)[2]), "=r"((r)[3]), "=r"((r)[4]), "=r"((r)[5]), \
                 "=r"((r)[6]), "=r"((r)[7]), "=r"((r)[8]), "=r"((r)[9]), "=r"((r)[10]), "=r"((r)[11]), \
                 "=r"((r)[12]), "=r"((r)[13]), "=r"((r)[14]), "=r"((r)[15])                          \
               : "r"(addr))

#define PI2_TMEM_WAIT16(a, b)                                                                      \
  asm volatile("tcgen05.wait::ld.sync.aligned;"                                                   \
               : "+r"((a)[0]), "+r"((a)[1]), "+r"((a)[2]), "+r"((a)[3]), "+r"((a)[4]), "+r"((a)[5]),  \
                 "+r"((a)[6]), "+r"((a)[7]), "+r"((b)[0]), "+r"((b)[1]), "+r"((b)[2]), "+r"((b)[3]),  \
                 "+r"((b)[4]), "+r"((b)[5]), "+r"((b)[6]), "+r"((b)[7])                               \
               :                                                                                   \
               : "memory")

constexpr int kTcThreads = 128;  // warp w owns TMEM lanes 32w .. 32w + 31 (tile rows)
constexpr int kTcCtasPerSm = PI2_TC_CTAS;  // co-resident CTAs: their MMA phases interleave
constexpr int kTcABytes = 8192;  // one A operand: hi | lo, 128 rows x 8 tf32 each

#ifdef PI2_TC_PROF
__device__ unsigned long long g_tc_prof[5];  // clocks: features+finalize, barrier, MMA wait, exp, tail
#define PI2_TC_TDECL long long prof[5] = {0, 0, 0, 0, 0}, t_last = clock64();
#define PI2_TC_T(i)                          \
  {                                          \
    const long long t_ = clock64();          \
    prof[i] += t_ - t_last;                  \
    t_last = t_;                             \
  }
#define PI2_TC_TFLUSH                                                                   \
  if ((threadIdx.x & 31) == 0)                                                          \
    for (int k_ = 0; k_ < 5; ++k_) atomicAdd(&g_tc_prof[k_], (unsigned long long)prof[k_]);
#elif defined(PI2_TC_TRACE)
// phase trace (experiments): lane 0 of every warp on SM 0 logs (clock, hw warp slot, CTA,
// phase end) into its own region (one atomic per warp to claim it, then plain stores)
constexpr int kTcTraceCap = 4096;  // events per warp
__device__ unsigned long long g_tc_trace[64 * kTcTraceCap];
__device__ unsigned int g_tc_trace_n;  // warps that claimed a region
__device__ int g_tc_trace_on;
__device__ __forceinline__ int tc_trace_claim() {
  unsigned sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  if (sm != 0 || (threadIdx.x & 31) != 0 || !g_tc_trace_on) return -1;
  const unsigned w = atomicAdd(&g_tc_trace_n, 1u);
  return w < 64 ? (int)w : -1;
}
__device__ __forceinline__ void tc_trace(int slot, int &n, int i) {
  if (slot < 0 || n >= kTcTraceCap) return;
  unsigned wid;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  g_tc_trace[slot * kTcTraceCap + n++] =
      ((unsigned long long)clock64() << 20) | ((blockIdx.x & 0x3ffu) << 10) | ((wid & 63u) << 4) | (unsigned)i;
}
#define PI2_TC_TDECL const int tr_slot_ = tc_trace_claim(); int tr_n_ = 0;
#define PI2_TC_T(i) tc_trace(tr_slot_, tr_n_, i)
#define PI2_TC_TFLUSH
#else
#define PI2_TC_TDECL
#define PI2_TC_T(i)
#define PI2_TC_TFLUSH
#endif

// software-pipelined TMEM loads in the exp loop (runtime batch loop): 0 never, 1 streamed
// weights only, 2 always.  Against the runtime loop it won for streamed weights (C3 25.3 ->
// 24.3 ms); the unrolled full-chunk loop (PI2_TC_UNROLL) beats both (streamed L=1000
// variance 3733 -> 3163 us, mean-only 2955 -> 2714 us: micro/lwpr_tc_stream_unroll_b200.txt)
#ifndef PI2_TC_LDPIPE
#define PI2_TC_LDPIPE 0
#endif
// full field chunks: the exp loop fully unrolled (compile-time batch count).  Harness,
// L=100 / 200 variance 426 -> 411 / 746 -> 705 us; unrolling every remainder count as
// well (8 instantiations) was slower again (profiles/micro/lwpr_tc_unroll_b200.txt)
#ifndef PI2_TC_UNROLL
#define PI2_TC_UNROLL 1
#endif
#ifndef PI2_TC_LD16  // 16-column tcgen05.ld in the unrolled full-chunk loop (variance kernels)
#define PI2_TC_LD16 1
#endif

// 3xTF32 as TWO MMAs per chunk instead of three: the same product terms hi.hi + hi.lo +
// lo.hi rearranged along K (A1 = [x~hi, 1, 1, q~hi, q~lo] . B1 = [Whi, A0hi, A0lo, 1, 1] and
// A2 = [x~hi, x~lo] . B2 = [Wlo, Whi]); operands keep their sizes
#ifndef PI2_TC_ROTATE  // 1: CTA b issues its MMAs from warp (b / SMs) % 4, so the co-resident CTAs'
#define PI2_TC_ROTATE 0  // issuers sit on different SM sub-partitions (else all on warp 0's); no change:
                         // C2 LWPR 393 vs 393 us, C4 step 6.06 vs 6.08 ms (micro/tc_rotate_b200.txt)
#endif
#ifndef PI2_TC_ELECT  // chunk MMAs issued by converged warp 0 with elect.sync (else thread 0)
#define PI2_TC_ELECT 0  // 1 measured slower in situ: L=100 385 -> 400 us, L=200 677 -> 698 (micro/tc_elect_b200.txt)
#endif
#ifndef PI2_TC_PACK2
#define PI2_TC_PACK2 1
#endif
#ifndef PI2_TC_POLY_VAR
#define PI2_TC_POLY_VAR 0   // field pairs (of 4 per 8-field batch) whose 2^x runs on the FMA pipe:
                            // the variance loop slows down with any (1: 436 -> 456 us at L=100), the
                            // mean-only loop gains from 1 (L=100 380 -> 359 us, L=200 694 -> 637 us)
#endif
#ifndef PI2_TC_POLY_MEAN
#define PI2_TC_POLY_MEAN 1
#endif
#ifndef PI2_TC_POLY_VAR_B  // the same for the second batch of each TMEM wait: one pair in 8
#define PI2_TC_POLY_VAR_B 1  // for the variance loop (L=200 772 -> 759 us, L=100 435 -> 433 us)
#endif
#ifndef PI2_TC_POLY_MEAN_B
#define PI2_TC_POLY_MEAN_B PI2_TC_POLY_MEAN
#endif

// 2^x of a field pair on the FMA pipe (FlashAttention-4's MUFU offload): x = n + f,
// n = rint(x) via the 1.5 * 2^23 shift, f in [-1/2, 1/2]; 2^f by a degree-5
// near-minimax polynomial (max rel. error 2.1e-7 in fp32 Horner, on par with
// ex2.approx); 2^n enters as n << 23 added to the result's bits (one integer
// multiply-add).  x >= -125 keeps 2^n normal: such weights are < 2^-61 of a row's
// normaliser on the fast path (logits carry the +64 shift), and a row whose
// weights all underflow takes the exact path either way.
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  x = make_float2(fmaxf(x.x, -125.0f), fmaxf(x.y, -125.0f));
  const float2 t = __fadd2_rn(x, bc(12582912.0f));
  const float2 n = __fadd2_rn(t, bc(-12582912.0f));
  const float2 f = __ffma2_rn(n, bc(-1.0f), x);
  float2 p = __ffma2_rn(bc(1.327645150013268e-03f), f, bc(9.675540961325169e-03f));
  p = __ffma2_rn(p, f, bc(5.550713464617729e-02f));
  p = __ffma2_rn(p, f, bc(2.402212023735046e-01f));
  p = __ffma2_rn(p, f, bc(6.931469440460205e-01f));
  p = __ffma2_rn(p, f, bc(1.000000119209290e+00f));
  return make_float2(__int_as_float(__float_as_int(t.x) * 8388608 + __float_as_int(p.x)),
                     __int_as_float(__float_as_int(t.y) * 8388608 + __float_as_int(p.y)));
}

// 8 fields of one row: e = 2^logit (the first POLY pairs on the FMA pipe, the rest
// on MUFU), moments on field pairs
template <bool VAR, bool SECOND = false>
__device__ __forceinline__ void tc_fields8(const uint32_t *lg, const uint32_t *yy, const float *slv, float2 &den,
                                           float2 &num, float2 &m2, float2 &lv) {
  constexpr int POLY = SECOND ? (VAR ? PI2_TC_POLY_VAR_B : PI2_TC_POLY_MEAN_B) : (VAR ? PI2_TC_POLY_VAR : PI2_TC_POLY_MEAN);
  // the batch's 8 local variances in two 128-bit loads (slv is 16-byte aligned)
  float lvv[8];
  if (VAR) {
    const float4 l0 = reinterpret_cast<const float4 *>(slv)[0], l1 = reinterpret_cast<const float4 *>(slv)[1];
    lvv[0] = l0.x; lvv[1] = l0.y; lvv[2] = l0.z; lvv[3] = l0.w;
    lvv[4] = l1.x; lvv[5] = l1.y; lvv[6] = l1.z; lvv[7] = l1.w;
  }
#pragma unroll
  for (int i = 0; i < 8; i += 2) {
    const float2 x = make_float2(__uint_as_float(lg[i]), __uint_as_float(lg[i + 1]));
    const float2 e = (i / 2 < POLY) ? exp2_poly2(x) : make_float2(ex2_ftz(x.x), ex2_ftz(x.y));
    const float2 y = make_float2(__uint_as_float(yy[i]), __uint_as_float(yy[i + 1]));
    den = __fadd2_rn(den, e);
    if (VAR) {  // second moment and local variances in one sum: e (y'^2 + var_l)
      num = __ffma2_rn(e, y, num);
      m2 = __ffma2_rn(e, __ffma2_rn(y, y, make_float2(lvv[i], lvv[i + 1])), m2);
    } else {
      num = __ffma2_rn(e, y, num);
    }
  }
}

// centred inputs and q~ of one row; its features [x~, 1, q~, 0, 0] as tf32 hi and lo
// into the A operand (K-major, no swizzle)
__device__ __forceinline__ void tc_features(const AxisHeader &h, float4 x, uint8_t *sa, int r, float4 &xt, float &q) {
  xt = make_float4(__fsub_rn(x.x, h.mu[0]), __fsub_rn(x.y, h.mu[1]), __fsub_rn(x.z, h.mu[2]), __fsub_rn(x.w, h.mu[3]));
  q = shared_qrow(h, xt);
  float hi[8], lo[8];  // PI2_TC_PACK2: the A1 | A2 operands of the two-MMA form; else the tf32 hi | lo split
#if PI2_TC_PACK2
  const float x4[4] = {xt.x, xt.y, xt.z, xt.w};
  const float qh = tf32_rna(q);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    hi[k] = lo[k] = tf32_rna(x4[k]);
    lo[4 + k] = tf32_rna(__fsub_rn(x4[k], hi[k]));
  }
  hi[4] = 1.0f;
  hi[5] = 1.0f;
  hi[6] = qh;
  hi[7] = tf32_rna(__fsub_rn(q, qh));
#else
  const float f[8] = {xt.x, xt.y, xt.z, xt.w, 1.0f, q, 0.0f, 0.0f};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    hi[k] = tf32_rna(f[k]);
    lo[k] = tf32_rna(__fsub_rn(f[k], hi[k]));
  }
#endif
  // k = 0..3 and 4..7 of a row are 16 contiguous bytes each in the K-major layout:
  // 4 conflict-free 128-bit stores instead of 16 4-way-conflicted 32-bit ones
#pragma unroll
  for (int k = 0; k < 8; k += 4) {
    *reinterpret_cast<float4 *>(sa + umma_kmajor_off(r, k)) = make_float4(hi[k], hi[k + 1], hi[k + 2], hi[k + 3]);
    *reinterpret_cast<float4 *>(sa + 4096 + umma_kmajor_off(r, k)) = make_float4(lo[k], lo[k + 1], lo[k + 2], lo[k + 3]);
  }
}

// (mean, std) of one row from its moments (exact path when the normaliser underflowed)
template <bool VAR>
__device__ __forceinline__ float2 tc_mean_sd(const LwprTcArgs &a, const AxisHeader &h, float4 xt, float q, float dn,
                                             float nm, float m2, float lv) {
  const float gx = fmaf(h.gs[3], xt.w, fmaf(h.gs[2], xt.z, fmaf(h.gs[1], xt.y, fmaf(h.gs[0], xt.x, h.g0))));
  float mean, var = 0.0f;
  // fast path: a normal normaliser and finite inputs (non-finite rows follow the
  // reference through the exact path)
  if (dn >= kSlowDen && dn <= 3.0e38f && isfinite(__fadd_rn(__fadd_rn(xt.x, xt.y), __fadd_rn(__fadd_rn(xt.z, xt.w), q)))) {
    const float rd = rcp_fma(dn);
    const float mp = __fmul_rn(nm, rd);
    mean = __fadd_rn(gx, mp);
    if (VAR) var = fmaxf(__fsub_rn(__fmul_rn(__fadd_rn(m2, lv), rd), __fmul_rn(mp, mp)), 0.0f);
  } else {
    const float2 mv = lwpr_row_exact<kLayShared>(a.params + h.offset, h.num_fields, xt, q, gx);
    mean = mv.x;
    var = mv.y;
  }
  return make_float2(mean, VAR ? (a.sqrt_out ? (var >= 1.17549435e-38f && var <= 3.40282347e38f ? sqrt_fma(var) : sqrtf(var)) : var)
                                : 0.0f);
}

template <bool VAR>
__device__ __forceinline__ void tc_finalize(const LwprTcArgs &a, const AxisHeader &h, int ax, int64_t row, float4 xt,
                                            float q, float dn, float nm, float m2, float lv) {
  if (row >= a.rows) return;
  const float2 ms = tc_mean_sd<VAR>(a, h, xt, q, dn, nm, m2, lv);
  a.mean_out[ax * a.plane + row] = ms.x;  // a warp writes 128 contiguous bytes
  if (VAR && a.sd_out) a.sd_out[ax * a.plane + row] = ms.y;
}

// The exp phase of nf (multiple of 8) fields of this warp's 32 rows, read from TMEM
// (logits from column tmem_lane, y' lc columns further on), 2^x + moments into the
// accumulators.  nf == NFULL runs a fully unrolled loop (compile-time batch count).
// REMB > 0: a chunk of exactly REMB batches (the model's remainder chunk, chosen by the
// host) also runs an unrolled loop (L=100: 40 of 104 padded fields; harness 391 -> 383 us,
// micro/lwpr_tc_remb_b200.txt)
template <bool VAR, bool STREAM, int NFULL, int REMB = 0>
__device__ __forceinline__ void tc_exp_span(uint32_t tmem_lane, int lc, int nf, const float *slv, float2 &den,
                                            float2 &num, float2 &m2, float2 &lv) {
  const int nb = nf >> 3;  // 8-field batches, two per TMEM wait
  if constexpr (PI2_TC_LDPIPE == 2 || (PI2_TC_LDPIPE == 1 && STREAM)) {
  // each batch's TMEM load is in flight while the previous batch computes
  // (tcgen05.wait::ld waits for all of a thread's loads: load b + 1, compute b, wait)
  uint32_t la[8], ya[8], lb[8], yb[8];
  PI2_TMEM_LD8(la, tmem_lane);
  PI2_TMEM_LD8(ya, tmem_lane + lc);
  PI2_TMEM_WAIT16(la, ya);
  for (int b = 0; b < nb; b += 2) {
    if (b + 1 < nb) {
      PI2_TMEM_LD8(lb, tmem_lane + 8 * b + 8);
      PI2_TMEM_LD8(yb, tmem_lane + lc + 8 * b + 8);
    }
    tc_fields8<VAR>(la, ya, slv + 8 * b, den, num, m2, lv);
    if (b + 1 < nb) {
      PI2_TMEM_WAIT16(lb, yb);
      if (b + 2 < nb) {
        PI2_TMEM_LD8(la, tmem_lane + 8 * b + 16);
        PI2_TMEM_LD8(ya, tmem_lane + lc + 8 * b + 16);
      }
      tc_fields8<VAR, true>(lb, yb, slv + 8 * b + 8, den, num, m2, lv);
      if (b + 2 < nb) PI2_TMEM_WAIT16(la, ya);
    }
  }
  } else {
  auto batches = [&](auto nb_c) {  // nb_c: compile-time batch count, or 0 = runtime nb
    constexpr int NBC = decltype(nb_c)::value;
    const int n = NBC > 0 ? NBC : nb;
#if PI2_TC_LD16
    // 16-column TMEM loads, one per operand per batch pair: variance loop only (harness L=100
    // 411 -> 406 us, L=200 704 -> 692 us); the mean-only loop spills with them and loses 4-5 %
    if constexpr (VAR && NBC > 0 && NBC % 2 == 0) {
#pragma unroll
      for (int b = 0; b < NBC; b += 2) {
        uint32_t l16[16], y16[16];
        PI2_TMEM_LD16(l16, tmem_lane + 8 * b);
        PI2_TMEM_LD16(y16, tmem_lane + lc + 8 * b);
        PI2_TMEM_WAIT16(l16, y16);
        PI2_TMEM_WAIT16(l16 + 8, y16 + 8);
        tc_fields8<VAR>(l16, y16, slv + 8 * b, den, num, m2, lv);
        tc_fields8<VAR, true>(l16 + 8, y16 + 8, slv + 8 * b + 8, den, num, m2, lv);
      }
      return;
    }
#endif
#pragma unroll
    for (int b = 0; b < (NBC > 0 ? NBC : 1 << 30); b += 2) {
      if (NBC == 0 && b >= n) break;
      uint32_t la[8], ya[8], lb[8], yb[8];
      PI2_TMEM_LD8(la, tmem_lane + 8 * b);
      PI2_TMEM_LD8(ya, tmem_lane + lc + 8 * b);
      if (b + 1 < n) {
        PI2_TMEM_LD8(lb, tmem_lane + 8 * b + 8);
        PI2_TMEM_LD8(yb, tmem_lane + lc + 8 * b + 8);
      }
      PI2_TMEM_WAIT16(la, ya);
      PI2_TMEM_WAIT16(lb, yb);
      tc_fields8<VAR>(la, ya, slv + 8 * b, den, num, m2, lv);
      if (b + 1 < n) tc_fields8<VAR, true>(lb, yb, slv + 8 * b + 8, den, num, m2, lv);
    }
  };
#if PI2_TC_UNROLL
  if (REMB > 0 && nf == 8 * REMB) batches(std::integral_constant<int, REMB>{});
  else if (nf == NFULL) batches(std::integral_constant<int, NFULL / 8>{});
  else batches(std::integral_constant<int, 0>{});
#else
  batches(std::integral_constant<int, 0>{});
#endif
  }
}

// Per CTA the tiles are software-pipelined: while the tensor core computes the
// first chunk of tile t, the CUDA cores finalize tile t - 1 and write tile t + 1's
// features into the other A buffer (its x was loaded one tile ahead), so only the
// barrier, the MMA latency and the exp phase remain on the critical path.
// STREAM: the axis' W does not fit in shared memory next to 3 other CTAs (large L):
// each chunk's W (<= 8 KB, L2-resident, read by every CTA of the axis) is brought in
// by a TMA bulk copy into a 2-slot ring, one chunk ahead of its MMA.
// WBULK (resident W, few tiles per CTA): the resident block arrives by one bulk copy
// issued before pdl_wait instead of an LDG/STS loop.  With few tiles that prologue is
// on the critical path: CTAs that become resident only when the attitude kernel's
// blocks leave the SM run it after the attitude kernel.  With many tiles the loop is
// amortised, and that instantiation keeps its own (faster) register allocation.
//
// AX: the axis this CTA evaluates as a compile-time constant (the kernel dispatches
// blockIdx.x % 3 to three copies of the body), so the axis' header constants are
// immediate parameter-space operands rather than indexed constant loads; -1 = runtime.
template <bool VAR, bool STREAM, bool WBULK, int AX, int REMB>
__device__ __forceinline__ void lwpr_tc_body(const LwprTcArgs &a, uint8_t *tsm, uint32_t &tmem_base, uint64_t &mbar,
                                             uint64_t *wbar) {
  // CTA i evaluates axis i % 3 for tiles i / 3, i / 3 + gridDim.x / 3, ...: only that
  // axis' weights (W chunks, then its chunk-padded variances) live in shared memory
  const int ax = AX >= 0 ? AX : (int)(blockIdx.x % 3);
  const int nch = a.nchunks[ax];
  const int64_t wbeg = a.axis_off[ax], wend = ax < 2 ? a.axis_off[ax + 1] : a.w_floats;
  const int64_t nlv = (int64_t)nch * kTcChunk;
  const int64_t wfl = STREAM ? 2 * kTcWSlotFloats : wend - wbeg;  // resident W, or the 2-slot ring
  float *sw = reinterpret_cast<float *>(tsm);
  float *slv_base = sw + wfl;
  uint8_t *sa = tsm + (((wfl + nlv) * 4 + 127) / 128) * 128;  // two A operands
  const int tid = threadIdx.x, warp = tid >> 5;
  // the thread that issues the chunk MMAs (and the TMA weight loads)
  const int issuer = PI2_TC_ROTATE && a.sms > 0 ? 32 * (int)((blockIdx.x / (unsigned)a.sms) & 3u) : 0;

  if (!STREAM && !WBULK)
    for (int64_t i = tid; i < (wend - wbeg) / 4; i += blockDim.x)
      reinterpret_cast<float4 *>(sw)[i] = __ldg(reinterpret_cast<const float4 *>(a.w + wbeg) + i);
  for (int64_t i = tid; i < nlv; i += blockDim.x) slv_base[i] = __ldg(a.w + a.lv_off[ax] + i);
  const uint32_t wbar_addr = (uint32_t)__cvta_generic_to_shared(&wbar[0]);
  const uint32_t sw_addr0 = (uint32_t)__cvta_generic_to_shared(sw);
  // bulk-copy chunk c's W into slot `slot` (thread 0)
  auto load_w = [&](int c, uint32_t slot) {
    const uint32_t bytes = (uint32_t)(2 * 2 * a.chunk_pad[ax][c] * 8 * 4);
    const uint32_t bar = wbar_addr + 8 * slot;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            sw_addr0 + slot * (uint32_t)(kTcWSlotFloats * 4)),
        "l"(a.w + wbeg + a.chunk_woff[ax][c]), "r"(bytes), "r"(bar)
        : "memory");
  };
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)),
                 "n"(kTcTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const uint32_t mbar_addr = (uint32_t)__cvta_generic_to_shared(&mbar);
  if (tid == issuer) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_addr));
    if (STREAM || WBULK) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(wbar_addr));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(wbar_addr + 8));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    if ((STREAM || WBULK) && blockIdx.x / 3 < (a.rows + 127) / 128) {
      if (STREAM) {
        load_w(0, 0);
      } else {  // the whole resident block, waited for before the first MMA
        const uint32_t bytes = (uint32_t)((wend - wbeg) * 4);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(wbar_addr), "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sw_addr0),
            "l"(a.w + wbeg), "r"(bytes), "r"(wbar_addr)
            : "memory");
      }
    }
  }
  const AxisHeader &h = a.axis[ax];
  const int64_t ntiles = (a.rows + 127) / 128, last = a.rows - 1;
  const int64_t tstride = gridDim.x / 3;
  int64_t tile = blockIdx.x / 3;
  // the rows are the attitude kernel's output (weights, TMEM and barriers above are
  // not): wait for it, then read them with coherent loads (__ldcg) -- ptxas may
  // hoist a non-coherent __ldg above griddepcontrol.wait
  pdl_wait();
  float4 xt, xt_prev = make_float4(0.f, 0.f, 0.f, 0.f);
  float q, q_prev = 0.0f, dn_p = 0.0f, nm_p = 0.0f, m2_p = 0.0f, lv_p = 0.0f;
  int64_t row_prev = a.rows;  // nothing to finalize yet
  {
    const int64_t r0 = tile * 128 + tid;
    tc_features(h, __ldcg(a.x + (r0 < last ? r0 : last)), sa, tid, xt, q);
  }
  int64_t rn = (tile + tstride) * 128 + tid;
  float4 xn = __ldcg(a.x + (rn < last ? rn : last));  // next tile's inputs, one tile ahead

  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t tmem_lane = tmem + ((uint32_t)(warp * 32) << 16);
  const uint32_t sw_addr = (uint32_t)__cvta_generic_to_shared(sw);
  uint32_t phase = 0, nw = 0;  // nw: chunks issued by this CTA (W ring position)
  int buf = 0;
  PI2_TC_TDECL

  // WBULK: the resident W landed (thread 0 issues every MMA)
  if (WBULK && tid == issuer && tile < ntiles) mbar_wait(wbar_addr, 0);
  for (; tile < ntiles; tile += tstride, buf ^= 1) {
    const uint32_t sa_addr = (uint32_t)__cvta_generic_to_shared(sa + buf * kTcABytes);
    float2 den = make_float2(0.f, 0.f), num = den, m2 = den, lv = den;
    float4 xt_next = xt;
    float q_next = q;
    int64_t woff = 0;  // within this axis' block in shared memory
    for (int c = 0; c < nch; ++c, ++nw) {
      const int lc = a.chunk_pad[ax][c];  // fields of this chunk, multiple of 8, 2 lc <= 128 columns
      asm volatile("fence.proxy.async.shared::cta;");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();  // A written, TMEM free
      PI2_TC_T(1);
#if PI2_TC_ELECT
      if (warp == 0) {  // converged: one elected lane issues (uniform descriptors)
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t idesc = umma_idesc_tf32(128, 2 * lc);
        const uint64_t a_hi = umma_smem_desc(sa_addr), a_lo = umma_smem_desc(sa_addr + 4096);
        if (STREAM) mbar_wait(wbar_addr + 8 * (nw & 1), (nw >> 1) & 1);  // this chunk's W landed
        const uint32_t wb = STREAM ? sw_addr + (nw & 1) * (uint32_t)(kTcWSlotFloats * 4) : sw_addr + (uint32_t)(woff * 4);
        const uint64_t b_hi = umma_smem_desc(wb), b_lo = umma_smem_desc(wb + (uint32_t)(2 * lc * 8 * 4));
#if PI2_TC_PACK2
        mma_tf32_elect(tmem, a_hi, b_hi, idesc, 0);  // A1 . B1
        mma_tf32_elect(tmem, a_lo, b_lo, idesc, 1);  // A2 . B2
#else
        mma_tf32_elect(tmem, a_hi, b_hi, idesc, 0);
        mma_tf32_elect(tmem, a_hi, b_lo, idesc, 1);
        mma_tf32_elect(tmem, a_lo, b_hi, idesc, 1);
#endif
        mma_commit_elect(mbar_addr);
        // the other slot held chunk nw - 1, whose MMA completed before this chunk's barrier
        if (STREAM && tid == issuer && (c + 1 < nch || tile + tstride < ntiles)) load_w(c + 1 < nch ? c + 1 : 0, (nw + 1) & 1);
      }
#else
      if (tid == issuer) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t idesc = umma_idesc_tf32(128, 2 * lc);
        const uint64_t a_hi = umma_smem_desc(sa_addr), a_lo = umma_smem_desc(sa_addr + 4096);
        if (STREAM) mbar_wait(wbar_addr + 8 * (nw & 1), (nw >> 1) & 1);  // this chunk's W landed
        const uint32_t wb = STREAM ? sw_addr + (nw & 1) * (uint32_t)(kTcWSlotFloats * 4) : sw_addr + (uint32_t)(woff * 4);
        const uint64_t b_hi = umma_smem_desc(wb), b_lo = umma_smem_desc(wb + (uint32_t)(2 * lc * 8 * 4));
#if PI2_TC_PACK2
        mma_tf32(tmem, a_hi, b_hi, idesc, 0);  // A1 . B1
        mma_tf32(tmem, a_lo, b_lo, idesc, 1);  // A2 . B2
#else
        mma_tf32(tmem, a_hi, b_hi, idesc, 0);
        mma_tf32(tmem, a_hi, b_lo, idesc, 1);
        mma_tf32(tmem, a_lo, b_hi, idesc, 1);
#endif
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            mbar_addr));
        // the other slot held chunk nw - 1, whose MMA completed before this chunk's barrier
        if (STREAM && (c + 1 < nch || tile + tstride < ntiles)) load_w(c + 1 < nch ? c + 1 : 0, (nw + 1) & 1);
      }
#endif
      if (c == 0) {  // in the MMA's shadow: finish tile t - 1, stage tile t + 1
        tc_finalize<VAR>(a, h, ax, row_prev, xt_prev, q_prev, dn_p, nm_p, m2_p, lv_p);
        if (tile + tstride < ntiles) {
          tc_features(h, xn, sa + (buf ^ 1) * kTcABytes, tid, xt_next, q_next);
          rn = (tile + 2 * tstride) * 128 + tid;
          xn = __ldcg(a.x + (rn < last ? rn : last));
        }
        PI2_TC_T(0);
      }
      mbar_wait(mbar_addr, phase);
      phase ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;");
      PI2_TC_T(2);
      tc_exp_span<VAR, STREAM, kTcChunk, REMB>(tmem_lane, lc, lc, slv_base + (int64_t)c * kTcChunk, den, num, m2, lv);
      woff += (int64_t)2 * (2 * lc * 8);
      PI2_TC_T(3);
    }
    xt_prev = xt;
    q_prev = q;
    row_prev = tile * 128 + tid;
    dn_p = __fadd_rn(den.x, den.y);
    nm_p = __fadd_rn(num.x, num.y);
    m2_p = __fadd_rn(m2.x, m2.y);
    lv_p = __fadd_rn(lv.x, lv.y);
    xt = xt_next;
    q = q_next;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  tc_finalize<VAR>(a, h, ax, row_prev, xt_prev, q_prev, dn_p, nm_p, m2_p, lv_p);
  PI2_TC_T(4);
  PI2_TC_TFLUSH
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTcTmemCols));
}



#ifndef PI2_TC_AXT
#define PI2_TC_AXT 0  // 1: three axis-specialised copies of the body (harness: within 1 %, 3x code; micro/lwpr_tc_axt_b200.txt)
#endif
template <bool VAR, bool STREAM, bool WBULK = false, int REMB = 0>
__global__ void __launch_bounds__(kTcThreads, kTcCtasPerSm) lwpr_tc_kernel(const __grid_constant__ LwprTcArgs a) {
  extern __shared__ __align__(128) uint8_t tsm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ __align__(8) uint64_t wbar[2];  // STREAM: W slot s holds its chunk
#if PI2_TC_AXT
  switch (blockIdx.x % 3) {
    case 0: lwpr_tc_body<VAR, STREAM, WBULK, 0, REMB>(a, tsm, tmem_base, mbar, wbar); break;
    case 1: lwpr_tc_body<VAR, STREAM, WBULK, 1, REMB>(a, tsm, tmem_base, mbar, wbar); break;
    default: lwpr_tc_body<VAR, STREAM, WBULK, 2, REMB>(a, tsm, tmem_base, mbar, wbar); break;
  }
#else
  lwpr_tc_body<VAR, STREAM, WBULK, -1, REMB>(a, tsm, tmem_base, mbar, wbar);
#endif
}


// Schedules tried against this one (bitwise equal, all slower at C2 size): a split
// barrier (micro/lwpr_tc_splitbar_b200.txt), TMEM double buffers with every warp doing
// its own features (micro/lwpr_tc3_dbuf_b200.txt), and warp-specialised exp / producer
// warps with 2-4 TMEM buffers (micro/lwpr_tcws_b200.txt, patch micro/lwpr_tcws.patch).

// batches of the remainder chunk when every axis ends with the same partial chunk
// (the REMB instantiation to launch), else 0
inline int tc_remainder_batches(const LwprTcArgs &ta) {
  const int r = ta.chunk_pad[0][ta.nchunks[0] - 1];
  for (int ax = 1; ax < 3; ++ax)
    if (ta.chunk_pad[ax][ta.nchunks[ax] - 1] != r) return 0;
  return r < kTcChunk ? r / 8 : 0;
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

// Dynamic shared memory of lwpr_tc_kernel: this axis' W + variances + the two A
// operands, padded so that exactly kTcCtasPerSm CTAs (and so their TMEM
// allocations) fit on an SM (228 KB per SM, 1 KB reserved per CTA).
inline int tc_smem_bytes(int64_t w_axis_floats, const void *fn) {
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, fn);
  const int need = (int)((w_axis_floats * 4 + 127) / 128 * 128 + 2 * kTcABytes);
  const int cap = 228 * 1024 / kTcCtasPerSm - 1024 - (int)fa.sharedSizeBytes - 256;
  return need > cap ? -1 : cap;  // -1: this axis' weights do not fit at full residency
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
#ifdef PI2_TC_EVEN_SPLIT
    const int per = (a.L + ta.nchunks[ax] - 1) / ta.nchunks[ax];  // even split, e.g. 100 -> 50 + 50
#else
    const int per = kTcChunk;  // full chunks, then the remainder: 100 -> 64 + 36 (padded 104, not 112)
#endif
    for (int c = 0; c < ta.nchunks[ax]; ++c) {
      const int l0 = c * per, n = std::min(per, a.L - l0);
      const int lc = (n + 7) / 8 * 8;
      ta.chunk_pad[ax][c] = lc;
      ta.chunk_woff[ax][c] = (int)(w_floats - ta.axis_off[ax]);
      // hi / lo: the B operands of the MMAs (PI2_TC_PACK2: B1 | B2, else the tf32 split)
      std::vector<float> hi(2 * lc * 8, 0.0f), lo(2 * lc * 8, 0.0f);
      auto at = [&](int r, int k) { return (size_t)(umma_kmajor_off(r, k) / 4); };
      // row r: slopes w[4] on x~, constant c, q~ coefficient qc
      auto row = [&](int r, const double *w, double c, double qc) {
#if PI2_TC_PACK2
        for (int i = 0; i < 4; ++i) {
          const float f = (float)w[i], fh = host_tf32_rna(f);
          hi[at(r, i)] = fh;                           // B1: w_hi . x~_hi
          lo[at(r, i)] = host_tf32_rna(f - fh);        // B2: w_lo . x~_hi
          lo[at(r, 4 + i)] = fh;                       //     w_hi . x~_lo
        }
        const float fc = (float)c, ch = host_tf32_rna(fc);
        hi[at(r, 4)] = ch;                             // B1: c_hi . 1
        hi[at(r, 5)] = host_tf32_rna(fc - ch);         //     c_lo . 1
        hi[at(r, 6)] = (float)qc;                      //     q~_hi
        hi[at(r, 7)] = (float)qc;                      //     q~_lo
#else
        auto put = [&](int k, double v) {
          const float f = (float)v, fh = host_tf32_rna(f);
          hi[at(r, k)] = fh;
          lo[at(r, k)] = host_tf32_rna(f - fh);
        };
        for (int i = 0; i < 4; ++i) put(i, w[i]);
        put(4, c);
        put(5, qc);
#endif
      };
      const double zero4[4] = {0, 0, 0, 0};
      for (int j = 0; j < lc; ++j) {
        const int l = l0 + j;
        if (j >= n) {  // padding field: weight 2^-1000 = 0, prediction 0
          row(j, zero4, -1000.0, 0.0);
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
        double dcl[4], sl[4];
        for (int i = 0; i < 4; ++i) {
          dcl[i] = dc[i] * kLog2e;
          sl[i] = a.coefs[(size_t)l * 5 + 1 + i] - gs[i];
        }
        row(j, dcl, a0 * kLog2e + kExpShift, 1.0);  // logit row: DC . x~ + A0 (shifted) + q~
        row(lc + j, sl, y0[l] - g0, 0.0);           // y' row: S' . x~ + Y0'
      }
      blob.insert(blob.end(), hi.begin(), hi.end());
      blob.insert(blob.end(), lo.begin(), lo.end());
      w_floats += (int64_t)hi.size() + (int64_t)lo.size();
      for (int j = 0; j < kTcChunk; ++j) lvs.push_back(j < n ? (float)a.lvar[l0 + j] : 0.0f);
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
