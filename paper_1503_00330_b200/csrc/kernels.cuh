// kernels.cuh — sm_100a kernels of one PI²-RH optimisation iteration.
//
//   attitude_kernel  K1-K3: perturb + clip, FP64 attitude recurrence, LWPR rows
//   lwpr_kernel      K4:    batched LWPR predict (FP32 CUDA cores + MUFU ex2)
//   rollout_kernel   K5-K10: sub-rollout integration, cost, M-mean, suffix sum
//   partials_kernel  K11a:  per-chunk (min, Z, V) softmax partials
//   combine_kernel   K11b:  fixed-order tree combine + plan update
//
// Rows are stored t-major on the device: row (k, t) is index t * K + k, so the
// 32 lanes of a warp (consecutive rollouts) touch one contiguous span at every
// step.  costs-to-go are kept t-major too and transposed to the reference's
// (K, N) layout (controller.py:212) only when handed back through the API.
#pragma once

#include "common.cuh"

namespace pi2 {

// Programmatic dependent launch: the step's kernels are launched with
// programmatic stream serialization, so a kernel may start while its predecessor
// drains.  pdl_wait() blocks until the predecessor grid has completed and its
// writes are visible (a no-op for a normal launch): every kernel calls it before
// touching anything an earlier kernel of the step writes; only constants
// (StepArgs, model weights) and TMEM allocation come before it.  Data written by
// the IMMEDIATE predecessor is read with coherent loads (__ldcg): a non-coherent
// __ldg (ld.global.nc) promises read-only data for the whole kernel, and ptxas
// does hoist it above griddepcontrol.wait (seen in SASS: a race).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// let the next kernel of the step launch (its CTAs then spin in pdl_wait)
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }


// ---------------------------------------------------------------------------
// device noise: Philox4x32-10 + Box-Muller, keyed by the reference's stream
// address (rng.py:33-44); counter = element-group index + key word 1.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Box-Muller on the MUFU unit: r = sqrt(-2 ln u1) via lg2/sqrt.approx,
// angle 2 pi u2 - pi in [-pi, pi) via sin/cos.approx (abs. error ~1e-6; the
// exploration noise is specified statistically, not bitwise).
__device__ __forceinline__ float2 box_muller(uint32_t a, uint32_t b) {
  const float u1 = fmaf((float)a, 2.3283064365386963e-10f, 1.1641532182693481e-10f);  // (0,1]
  const float th = fmaf((float)b, 1.4629180792671596e-09f, -3.14159265358979f);         // [-pi,pi)
  float lg, r, s, c;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(u1));
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(-1.3862943611198906f * lg));  // -2 ln 2 * lg2
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(th));
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(th));
  return make_float2(r * c, r * s);
}

__device__ __forceinline__ float4 normals4(uint64_t index, uint64_t k0, uint64_t k1) {
  const uint4 c = make_uint4((uint32_t)index, (uint32_t)(index >> 32), (uint32_t)k1,
                             (uint32_t)(k1 >> 32));
  const uint4 r = philox4x32_10(c, (uint32_t)k0, (uint32_t)(k0 >> 32));
  const float2 z0 = box_muller(r.x, r.y), z1 = box_muller(r.z, r.w);
  return make_float4(z0.x, z0.y, z1.x, z1.y);
}

// exploration noise eps[k, t, :] of the device stream (float32 normals x float64 std)
// (key: iter_key(sa->key_prefix[0], iteration), derived once per thread)
__device__ __forceinline__ void eps_from_z(const StepArgs *sa, float4 z, double e[4]) {
  e[0] = __dmul_rn((double)z.x, sa->std[0]);
  e[1] = __dmul_rn((double)z.y, sa->std[1]);
  e[2] = __dmul_rn((double)z.z, sa->std[2]);
  e[3] = __dmul_rn((double)z.w, sa->std[3]);
}
__device__ __forceinline__ float4 device_z(Key128 key, uint64_t kg, int N, int t) {
  return normals4(kg * (uint64_t)N + (uint64_t)t, key.k0, key.k1);
}
__device__ __forceinline__ void device_eps(const StepArgs *sa, Key128 key, uint64_t kg, int N, int t,
                                           double e[4]) {
  eps_from_z(sa, device_z(key, kg, N, t), e);
}

// Dynamics draws of the device stream: sub-rollout (k, m) consumes the normals of its
// Philox blocks in order, all four of each, 3 per step — step t takes normals 3t .. 3t+2
// of the sequence normals4(base + 0), normals4(base + 1), ... with base = (k M + m) * NB
// and NB = dyn_blocks(N) blocks per sub-rollout (4 steps per 3 blocks; tests/devnoise.py
// replicates it).
__host__ __device__ __forceinline__ int64_t dyn_blocks(int N) { return (3 * (int64_t)N + 3) / 4; }

// step t's three draws without state (two blocks when they straddle a block boundary)
__device__ __forceinline__ void dyn3(uint64_t base, int t, uint64_t k0, uint64_t k1, float d[3]) {
  const int64_t q = 3 * (int64_t)t;
  const int r = (int)(q & 3);
  const float4 z = normals4(base + (uint64_t)(q >> 2), k0, k1);
  const float v0[4] = {z.x, z.y, z.z, z.w};
  if (r <= 1) {
    d[0] = v0[r]; d[1] = v0[r + 1]; d[2] = v0[r + 2];
    return;
  }
  const float4 y = normals4(base + (uint64_t)(q >> 2) + 1, k0, k1);
  if (r == 2) {
    d[0] = z.z; d[1] = z.w; d[2] = y.x;
  } else {
    d[0] = z.w; d[1] = y.x; d[2] = y.y;
  }
}

// the same draws for t = 0, 1, 2, ... in order: one Philox block per step for three steps
// of four, the leftover normals carried (the round-1 stream used 3 of 4 normals per block)
struct DynDraws {
  float c0 = 0.f, c1 = 0.f, c2 = 0.f;
  __device__ __forceinline__ void next(uint64_t base, int t, uint64_t k0, uint64_t k1, float d[3]) {
    const int ph = t & 3;
    if (ph == 3) {
      d[0] = c0; d[1] = c1; d[2] = c2;
      return;
    }
    const float4 z = normals4(base + (uint64_t)(3 * (t >> 2) + ph), k0, k1);
    if (ph == 0) {
      d[0] = z.x; d[1] = z.y; d[2] = z.z;
      c0 = z.w;
    } else if (ph == 1) {
      d[0] = c0; d[1] = z.x; d[2] = z.y;
      c0 = z.z; c1 = z.w;
    } else {
      d[0] = c0; d[1] = c1; d[2] = z.x;
      c0 = z.y; c1 = z.z; c2 = z.w;
    }
  }
};

// np.clip(v, lo, hi, out=...) with array bounds (controller.py:259, :371): numpy's
// _NPY_MAX/_NPY_MIN, i.e. NaN propagates and max(-0, +0) = +0 ((a > b) ? a : b).
// Two compare-selects, against ~18 SASS instructions for the fmin/fmax pair.
__device__ __forceinline__ double clip_np(double v, double lo, double hi) {
  const double t = (v > lo || v != v) ? v : lo;
  return (t < hi || t != t) ? t : hi;
}
// The same for bounds that are not NaN (the host checks, DynParams): !(v <= lo) is
// (v > lo || v != v) when lo is not NaN -- one unordered compare and a select per bound
// instead of two compares, a predicate combine and two selects.
__device__ __forceinline__ double clip_np_nonan(double v, double lo, double hi) {
  const double t = !(v <= lo) ? v : lo;
  return !(t >= hi) ? t : hi;
}
template <bool NONAN>
__device__ __forceinline__ double clip_bounds(double v, double lo, double hi) {
  return NONAN ? clip_np_nonan(v, lo, hi) : clip_np(v, lo, hi);
}


// ---------------------------------------------------------------------------
// K1-K3: u = clip(plan + eps), attitude recurrence, LWPR input rows.
// controller.py:257-275.  One thread per rollout, FP64, no contraction.
// ---------------------------------------------------------------------------
// attitude_kernel: device noise of PI2_ATT_TB steps is generated ahead of their serial
// FP64 recurrence; PI2_ATT_UNROLL unrolls the outer loop (micro/att_tune_b200.txt: 4 / 1)
#ifndef PI2_ATT_TB
#define PI2_ATT_TB 4
#endif
#ifndef PI2_ATT_UNROLL
#define PI2_ATT_UNROLL 1
#endif
constexpr int kAttUnroll = PI2_ATT_UNROLL;

template <bool DEVICE_NOISE, bool NONAN = false>
__global__ void __launch_bounds__(kRolloutBlock)
    attitude_kernel(const StepArgs *__restrict__ sa, const double *__restrict__ plan,
                    const double *__restrict__ eps, int iteration, int64_t K, int64_t k_off, int N,
                    DynParams dp, float4 *__restrict__ xin, float4 *__restrict__ ang_last,
                    float4 *__restrict__ zout) {
  // zout (device noise): the exploration normals z(k, t) at zout[t * K + k] for the
  // partials kernel, which would otherwise regenerate them (e = z * std either way)
  extern __shared__ double smem_plan[];  // (N, 4) when N <= kMaxHorizon
  pdl_wait();     // the plan is the previous iteration's update
  pdl_trigger();  // one wave: the LWPR kernel's prologue may start on free SM resources
  // longer horizons read the plan rows from global memory (one broadcast load per row)
  const bool staged = N <= kMaxHorizon;
  if (staged)
    for (int i = threadIdx.x; i < 4 * N; i += blockDim.x) smem_plan[i] = plan[i];
  __syncthreads();
  const double *splan = staged ? smem_plan : plan;
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  double ang[3] = {sa->state[6], sa->state[7], sa->state[8]};
  double rate[3] = {sa->state[9], sa->state[10], sa->state[11]};
  const double *ek = DEVICE_NOISE ? nullptr : eps + k * (int64_t)N * 4;
  const Key128 ck = DEVICE_NOISE ? iter_key(sa->key_prefix[0], (uint64_t)iteration) : Key128{0, 0};
  float4 *xk = xin + k;  // row (k, t) at xk[t * K]
  constexpr int TB = PI2_ATT_TB;  // noise of TB steps is generated before their serial FP64 recurrence
  // host noise (the reference's streams in HBM): the next TB steps' rows are loaded while
  // this block's recurrence runs, so the DRAM latency is not exposed once per block
  double2 en[TB][2];
  auto load_block = [&](int t0) {
#pragma unroll
    for (int j = 0; j < TB; ++j) {
      const int t = t0 + j < N ? t0 + j : N - 1;
      en[j][0] = __ldg(reinterpret_cast<const double2 *>(ek + 4 * t));
      en[j][1] = __ldg(reinterpret_cast<const double2 *>(ek + 4 * t) + 1);
    }
  };
  if (!DEVICE_NOISE) load_block(0);
#pragma unroll(kAttUnroll)
  for (int t0 = 0; t0 < N; t0 += TB) {
    double e[TB][4];
#pragma unroll
    for (int j = 0; j < TB; ++j) {
      const int t = t0 + j < N ? t0 + j : N - 1;
      if (DEVICE_NOISE) {
        const float4 z = device_z(ck, (uint64_t)(k_off + k), N, t);
        if (zout && t0 + j < N) zout[(int64_t)t * K + k] = z;
        eps_from_z(sa, z, e[j]);
      } else {
        e[j][0] = en[j][0].x; e[j][1] = en[j][0].y; e[j][2] = en[j][1].x; e[j][3] = en[j][1].y;
      }
    }
    if (!DEVICE_NOISE && t0 + TB < N) load_block(t0 + TB);
#pragma unroll
    for (int j = 0; j < TB; ++j) {
      const int t = t0 + j;
      if (t >= N) break;
      double u[4];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        u[c] = clip_bounds<NONAN>(__dadd_rn(splan[4 * t + c], e[j][c]), dp.lo[c], dp.hi[c]);
      xk[(int64_t)t * K] = make_float4(__double2float_rn(ang[0]), __double2float_rn(ang[1]),
                          __double2float_rn(ang[2]), __double2float_rn(u[3]));
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        ang[c] = wrap_angle(__dadd_rn(ang[c], __dmul_rn(rate[c], dp.dt)));
        rate[c] = __dadd_rn(rate[c], __dmul_rn(dp.gain_dt, __dsub_rn(u[c], rate[c])));
      }
    }
  }
  ang_last[k] = make_float4(__double2float_rn(ang[0]), __double2float_rn(ang[1]),
                            __double2float_rn(ang[2]), 0.0f);
}

// ---------------------------------------------------------------------------
// K4: batched LWPR predict.  Weights 2^(logit2) with logit2 = Horner form of
// the folded quadratic (log2-scaled, +kExpShift); local models shifted by a
// global linear g(x) so the one-pass second moment does not cancel.
// Thread = kLwprRows rows; all threads of a block walk the same receptive
// field at the same time (shared-memory broadcast of the field record).
// ---------------------------------------------------------------------------
struct LwprArgs {
  const float *params;  // records of all axes (HBM)
  AxisHeader axis[3];
  int a_begin, a_end;
  int layout;           // kLay*
  int resident;         // all records of [a_begin, a_end) fit in shared memory
  int tile;             // fields per shared-memory tile when not resident
  int64_t rows;
  const float4 *x;      // (rows) inputs, padded to 4
  float *mean_out;      // [row * row_stride + (axis - a_begin) * axis_stride]
  float *sd_out;        // std (sqrt_out) or variance; may be null
  int row_stride;       // 1: planes (axis_stride = rows) or one axis; 4: float4 rows (w = 0)
  int64_t axis_stride;
  int sqrt_out;
};

__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Record layouts (floats per receptive field):
//   kLayDiag   16: A0, A1[4], A2[4], S[4], Y0, LV, -      per-field diagonal metric
//   kLayFull   24: A0, Q00 Q01 Q02 Q03 Q11 Q12 Q13 Q22 Q23 Q33, A2[4], S[4], Y0, LV, -
//   kLayShared 12: A0, DC[4], S[4], Y0, LV, -             metric shared by all fields
// A* / Q* / DC are log2(e)-scaled; with a shared metric D the quadratic
// -1/2 x'Dx is per row (qrow, added once per field), so a field costs
// 4 FMA + 1 ADD instead of 8 (reference LwprModel.update always copies
// d_init into new fields, lwpr.py:208-216, so trained models share D).
template <int LAY> struct Lay;
template <> struct Lay<kLayDiag> { static constexpr int RS = kRecDiag, S = 9, LV = 14; };
template <> struct Lay<kLayFull> { static constexpr int RS = kRecFull, S = 15, LV = 20; };
template <> struct Lay<kLayShared> { static constexpr int RS = kRecShared, S = 5, LV = 10; };

template <int LAY>
__device__ __forceinline__ float field_logit2(const float *f, const float4 &x, float qrow) {
  if (LAY == kLayDiag) {
    float lg = fmaf(fmaf(f[1], x.x, f[5]), x.x, f[0]);
    lg = fmaf(fmaf(f[2], x.y, f[6]), x.y, lg);
    lg = fmaf(fmaf(f[3], x.z, f[7]), x.z, lg);
    return fmaf(fmaf(f[4], x.w, f[8]), x.w, lg);
  } else if (LAY == kLayFull) {
    float h = fmaf(f[1], x.x, f[11]);
    h = fmaf(f[2], x.y, h);
    h = fmaf(f[3], x.z, h);
    h = fmaf(f[4], x.w, h);
    float lg = fmaf(h, x.x, f[0]);
    h = fmaf(f[5], x.y, f[12]);
    h = fmaf(f[6], x.z, h);
    h = fmaf(f[7], x.w, h);
    lg = fmaf(h, x.y, lg);
    h = fmaf(f[8], x.z, f[13]);
    h = fmaf(f[9], x.w, h);
    lg = fmaf(h, x.z, lg);
    h = fmaf(f[10], x.w, f[14]);
    return fmaf(h, x.w, lg);
  } else {
    const float lg = fmaf(f[4], x.w, fmaf(f[3], x.z, fmaf(f[2], x.y, fmaf(f[1], x.x, f[0]))));
    return __fadd_rn(lg, qrow);
  }
}

template <int LAY>
__device__ __forceinline__ float field_local(const float *f, const float4 &x) {
  constexpr int S = Lay<LAY>::S;
  float y = fmaf(f[S + 0], x.x, f[S + 4]);
  y = fmaf(f[S + 1], x.y, y);
  y = fmaf(f[S + 2], x.z, y);
  return fmaf(f[S + 3], x.w, y);
}

template <int LAY>
__device__ __forceinline__ float field_lvar(const float *f) {
  return f[Lay<LAY>::LV];
}

// per-row log2-scaled quadratic of a shared metric at centred x~
__device__ __forceinline__ float shared_qrow(const AxisHeader &h, const float4 &x) {
  float r = fmaf(h.qd[0], x.x, fmaf(h.qd[1], x.y, fmaf(h.qd[2], x.z, h.qd[3] * x.w)));
  float q = r * x.x;
  r = fmaf(h.qd[4], x.y, fmaf(h.qd[5], x.z, h.qd[6] * x.w));
  q = fmaf(r, x.y, q);
  r = fmaf(h.qd[7], x.z, h.qd[8] * x.w);
  q = fmaf(r, x.z, q);
  return fmaf(h.qd[9] * x.w, x.w, q);
}

// Rows whose centred quadratic q~ >= this (log2 units) take the field loop
// WITHOUT the per-field "+ q~" add: every accumulator is linear in the weight,
// so a per-row factor 2^-q~ cancels in mean and variance, and 2^(logit2 - q~)
// stays below 2^(64 + 60) (no overflow).  The decision is warp-uniform.
constexpr float kNearQ = -60.0f;

// Reference-exact evaluation of one row (rare: every weight is (nearly)
// denormal in float32).  Emulates numpy: e = expf(q) with float32 denormal
// rounding (here scaled by 2^64: multiples of 2^-85 below 2^-62), w = e/den
// (0/0 = NaN -> cost ceiling downstream), mean = sum w y, two-pass variance
// (lwpr.py:395-407).
template <int LAY>
__device__ __forceinline__ float exact_weight(const float *f, const float4 &x, float qrow) {
  float e = exp2f(field_logit2<LAY>(f, x, qrow));  // IEEE exp2f: never flushes
  // float32 denormal grid of exp(q) (step 2^-149), in 2^64-scaled units:
  // multiples of 2^-85 below 2^-62 (exact products by powers of two)
  if (e < 2.168404344971009e-19f) e = rintf(e * 3.8685626227668134e25f) * 2.5849394142282115e-26f;
  return e;
}

// (mean, variance) by value: output pointers to a non-inlined function would put the
// callers' mean/var in local memory on their fast path too
template <int LAY>
__device__ __noinline__ float2 lwpr_row_exact(const float *rec, int nf, float4 x, float qrow, float gx) {
  constexpr int RS = Lay<LAY>::RS;
  float den = 0.0f;
  for (int l = 0; l < nf; ++l) den = __fadd_rn(den, exact_weight<LAY>(rec + (int64_t)l * RS, x, qrow));
  float mean = 0.0f;
  for (int l = 0; l < nf; ++l) {
    const float *f = rec + (int64_t)l * RS;
    const float w = __fdiv_rn(exact_weight<LAY>(f, x, qrow), den);
    mean = __fadd_rn(mean, __fmul_rn(w, __fadd_rn(field_local<LAY>(f, x), gx)));
  }
  float var = 0.0f;
  for (int l = 0; l < nf; ++l) {
    const float *f = rec + (int64_t)l * RS;
    const float w = __fdiv_rn(exact_weight<LAY>(f, x, qrow), den);
    const float d = __fsub_rn(mean, __fadd_rn(field_local<LAY>(f, x), gx));
    var = __fadd_rn(var, __fmul_rn(w, __fadd_rn(__fmul_rn(d, d), field_lvar<LAY>(f))));
  }
  return make_float2(mean, var);
}

// Packed-pair forms: two rows per 64-bit register pair, field parameters
// broadcast (ptxas folds make_float2(p, p) into the FFMA2 .F32 operand).
// FFMA2 halves FMA-pipe issue slots, which lets the MUFU.EX2 of the weights
// dispatch without starving the FMA pipe (profiles/micro/mufu_mix.cu).
__device__ __forceinline__ float2 bc(float v) { return make_float2(v, v); }

template <int LAY, bool ADDQ>
__device__ __forceinline__ float2 field_logit2_x2(const float *f, const float2 *X, float2 Q) {
  if (LAY == kLayDiag) {
    float2 lg = __ffma2_rn(__ffma2_rn(bc(f[1]), X[0], bc(f[5])), X[0], bc(f[0]));
    lg = __ffma2_rn(__ffma2_rn(bc(f[2]), X[1], bc(f[6])), X[1], lg);
    lg = __ffma2_rn(__ffma2_rn(bc(f[3]), X[2], bc(f[7])), X[2], lg);
    return __ffma2_rn(__ffma2_rn(bc(f[4]), X[3], bc(f[8])), X[3], lg);
  } else if (LAY == kLayFull) {
    float2 h = __ffma2_rn(bc(f[1]), X[0], bc(f[11]));
    h = __ffma2_rn(bc(f[2]), X[1], h);
    h = __ffma2_rn(bc(f[3]), X[2], h);
    h = __ffma2_rn(bc(f[4]), X[3], h);
    float2 lg = __ffma2_rn(h, X[0], bc(f[0]));
    h = __ffma2_rn(bc(f[5]), X[1], bc(f[12]));
    h = __ffma2_rn(bc(f[6]), X[2], h);
    h = __ffma2_rn(bc(f[7]), X[3], h);
    lg = __ffma2_rn(h, X[1], lg);
    h = __ffma2_rn(bc(f[8]), X[2], bc(f[13]));
    h = __ffma2_rn(bc(f[9]), X[3], h);
    lg = __ffma2_rn(h, X[2], lg);
    h = __ffma2_rn(bc(f[10]), X[3], bc(f[14]));
    return __ffma2_rn(h, X[3], lg);
  } else {
    float2 lg = __ffma2_rn(bc(f[1]), X[0], bc(f[0]));
    lg = __ffma2_rn(bc(f[2]), X[1], lg);
    lg = __ffma2_rn(bc(f[3]), X[2], lg);
    lg = __ffma2_rn(bc(f[4]), X[3], lg);
    return ADDQ ? __fadd2_rn(lg, Q) : lg;
  }
}

template <int LAY>
__device__ __forceinline__ float2 field_local_x2(const float *f, const float2 *X) {
  constexpr int S = Lay<LAY>::S;
  float2 y = __ffma2_rn(bc(f[S + 0]), X[0], bc(f[S + 4]));
  y = __ffma2_rn(bc(f[S + 1]), X[1], y);
  y = __ffma2_rn(bc(f[S + 2]), X[2], y);
  return __ffma2_rn(bc(f[S + 3]), X[3], y);
}

// The field loop of one tile: P row pairs, accumulators updated in place.
template <int LAY, bool VAR, int P, bool ADDQ>
__device__ __forceinline__ void lwpr_fields(const float *sp, int nl, const float2 (*X)[4], const float2 *Q, float2 *den,
                                            float2 *num, float2 *m2, float2 *lv) {
  constexpr int RS = Lay<LAY>::RS;
#pragma unroll 2
  for (int l = 0; l < nl; ++l) {
    float f[RS];
#pragma unroll
    for (int i = 0; i < RS / 4; ++i) {
      const float4 v = reinterpret_cast<const float4 *>(sp + (int64_t)l * RS)[i];
      f[4 * i + 0] = v.x; f[4 * i + 1] = v.y; f[4 * i + 2] = v.z; f[4 * i + 3] = v.w;
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const float2 lg = field_logit2_x2<LAY, ADDQ>(f, X[p], Q[p]);
      const float2 e = make_float2(ex2_ftz(lg.x), ex2_ftz(lg.y));
      const float2 y = field_local_x2<LAY>(f, X[p]);
      den[p] = __fadd2_rn(den[p], e);
      if (VAR) {
        const float2 ey = __fmul2_rn(e, y);
        num[p] = __fadd2_rn(num[p], ey);
        m2[p] = __ffma2_rn(ey, y, m2[p]);
        lv[p] = __ffma2_rn(e, bc(field_lvar<LAY>(f)), lv[p]);
      } else {
        num[p] = __ffma2_rn(e, y, num[p]);
      }
    }
  }
}

template <int LAY, bool VAR, int R, int BLOCK = kLwprBlock, int MINB = 4>
__global__ void __launch_bounds__(BLOCK, MINB) lwpr_kernel(LwprArgs a) {
  static_assert(R % 2 == 0, "rows come in pairs");
  constexpr int RS = Lay<LAY>::RS;
  constexpr int P = R / 2;
  extern __shared__ float4 smem4[];
  float *srec = reinterpret_cast<float *>(smem4);
  pdl_wait();

  const int64_t row0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * R;
  float4 x[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t row = row0 + r < a.rows ? row0 + r : a.rows - 1;
    x[r] = __ldcg(a.x + row);  // the attitude kernel's output (see pdl_wait)
  }
  float2 X[P][4];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    X[p][0] = make_float2(x[2 * p].x, x[2 * p + 1].x);
    X[p][1] = make_float2(x[2 * p].y, x[2 * p + 1].y);
    X[p][2] = make_float2(x[2 * p].z, x[2 * p + 1].z);
    X[p][3] = make_float2(x[2 * p].w, x[2 * p + 1].w);
  }

  if (a.resident) {
    const int64_t base = a.axis[a.a_begin].offset;
    const int64_t n4 = (a.axis[a.a_end - 1].offset + (int64_t)a.axis[a.a_end - 1].num_fields * RS - base) / 4;
    const float4 *src = reinterpret_cast<const float4 *>(a.params + base);
    for (int64_t i = threadIdx.x; i < n4; i += blockDim.x) smem4[i] = __ldg(src + i);
    __syncthreads();
  }

  for (int ax = a.a_begin; ax < a.a_end; ++ax) {
    const AxisHeader h = a.axis[ax];
    float2 den[P], num[P], m2[P], lv[P], Q[P];
    float2 XT[P][4];  // centred inputs x~ = x - mu
    float4 xt[R];
    bool near_mine = true;
#pragma unroll
    for (int r = 0; r < R; ++r)
      xt[r] = make_float4(__fsub_rn(x[r].x, h.mu[0]), __fsub_rn(x[r].y, h.mu[1]), __fsub_rn(x[r].z, h.mu[2]),
                          __fsub_rn(x[r].w, h.mu[3]));
#pragma unroll
    for (int p = 0; p < P; ++p) {
      den[p] = num[p] = m2[p] = lv[p] = make_float2(0.0f, 0.0f);
      Q[p] = LAY == kLayShared ? make_float2(shared_qrow(h, xt[2 * p]), shared_qrow(h, xt[2 * p + 1]))
                               : make_float2(0.0f, 0.0f);
      near_mine = near_mine && Q[p].x >= kNearQ && Q[p].y >= kNearQ;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float *v0 = reinterpret_cast<const float *>(&xt[2 * p]), *v1 = reinterpret_cast<const float *>(&xt[2 * p + 1]);
        XT[p][i] = make_float2(v0[i], v1[i]);
      }
    }
    const bool near = __all_sync(0xffffffffu, near_mine);

    const int tile = a.resident ? h.num_fields : a.tile;
    for (int l0 = 0; l0 < h.num_fields; l0 += tile) {
      const int nl = min(tile, h.num_fields - l0);
      const float *sp;
      if (a.resident) {
        sp = srec + (h.offset - a.axis[a.a_begin].offset) + (int64_t)l0 * RS;
      } else {
        __syncthreads();
        const float4 *src = reinterpret_cast<const float4 *>(a.params + h.offset + (int64_t)l0 * RS);
        for (int i = threadIdx.x; i < nl * RS / 4; i += blockDim.x) smem4[i] = __ldg(src + i);
        __syncthreads();
        sp = srec;
      }
      if (LAY == kLayShared && near)
        lwpr_fields<LAY, VAR, P, false>(sp, nl, XT, Q, den, num, m2, lv);
      else
        lwpr_fields<LAY, VAR, P, LAY == kLayShared>(sp, nl, XT, Q, den, num, m2, lv);
    }

#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t row = row0 + r;
      if (row >= a.rows) continue;
      const int p = r / 2;
      const float dn = (r & 1) ? den[p].y : den[p].x;
      const float nm = (r & 1) ? num[p].y : num[p].x;
      const float sm2 = (r & 1) ? m2[p].y : m2[p].x;
      const float slv = (r & 1) ? lv[p].y : lv[p].x;
      const float qr = (r & 1) ? Q[p].y : Q[p].x;
      const float gx = fmaf(h.gs[3], xt[r].w, fmaf(h.gs[2], xt[r].z, fmaf(h.gs[1], xt[r].y, fmaf(h.gs[0], xt[r].x, h.g0))));
      // normaliser on the 2^(logit*log2e + 64) scale (the fast loop dropped 2^q~)
      const float dn_scaled = (LAY == kLayShared && near) ? dn * exp2f(qr) : dn;
      float mean, var = 0.0f;
      if (dn_scaled >= kSlowDen) {
        const float mp = __fdiv_rn(nm, dn);
        mean = __fadd_rn(gx, mp);
        if (VAR) var = fmaxf(__fsub_rn(__fdiv_rn(__fadd_rn(sm2, slv), dn), __fmul_rn(mp, mp)), 0.0f);
      } else {
        const float2 mv = lwpr_row_exact<LAY>(a.params + h.offset, h.num_fields, xt[r], qr, gx);
        mean = mv.x;
        var = mv.y;
      }
      const int64_t o = row * a.row_stride + (ax - a.a_begin) * a.axis_stride;
      a.mean_out[o] = mean;
      if (VAR && a.sd_out) a.sd_out[o] = a.sqrt_out ? __fsqrt_rn(var) : var;
      // float4 rows: the last pass also writes the pad lane, so every 32-byte
      // sector is fully written while it sits in L2 (no read-for-ownership)
      if (a.row_stride == 4 && ax == a.a_end - 1) {
        a.mean_out[row * 4 + 3] = 0.0f;
        if (VAR && a.sd_out) a.sd_out[row * 4 + 3] = 0.0f;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K5-K10: sub-rollout integration, crash, stage cost, pairwise M-mean,
// float64 suffix sum, non-finite -> ceiling.  controller.py:281-322,
// simworld.py:157-198.  One thread per rollout; FP32 without contraction so
// pos/vel match the reference's cumsum form bitwise given the same accels.
// ---------------------------------------------------------------------------
struct RollArgs {
  const StepArgs *sa;
  int iteration;
  int64_t K, k_off;
  int N, M;
  int model;        // PI2_MODEL_*
  int spread;       // model.probabilistic && M > 1
  int device_dyn;   // dynamics draws from the device stream (else dyn)
  int penalty;      // cost.variance_penalty > 0 with the hybrid model: std planes are read for it
  float two_point;  // TwoPointModel magnitude
  DynParams dp;
  const float4 *xin, *ang_last;
  const float *lw_mean, *lw_std;  // LWPR mean / std planes: axis c of row r at [c * lw_plane + r]
  int64_t lw_plane;
  const float *dyn;  // (K, M, N, 3)
  double *costs;     // (K, N)
  uint8_t *crash;    // (K)
  float *qs;         // horizons past kSmemHorizon: (N, K) stage-cost scratch in global memory (t-major)
                     // instead of the blocks' shared memory; nullptr otherwise
};

// opt-in uncertainty penalty (pi2_cost.variance_penalty, an extension; 0 = the
// reference): kappa * (sd_x^2 + sd_y^2 + sd_z^2), added to the sub-rollout-mean stage
// cost in float32
__device__ __forceinline__ float variance_term(float kappa, float3 sd) {
  return __fmul_rn(kappa, __fadd_rn(__fadd_rn(__fmul_rn(sd.x, sd.x), __fmul_rn(sd.y, sd.y)), __fmul_rn(sd.z, sd.z)));
}

// the LWPR kernel's output: coherent loads (see pdl_wait)
__device__ __forceinline__ float3 ld_planes(const float *p, int64_t plane, int64_t row) {
  return make_float3(__ldcg(p + row), __ldcg(p + plane + row), __ldcg(p + 2 * plane + row));
}
// the same with 32-bit element offsets (3 planes x K x N < 2^32, host-checked: RollArgs::rows32),
// so each address is one IMAD.WIDE.U32 instead of a 64-bit add chain
__device__ __forceinline__ float3 ld_planes32(const float *p, uint32_t plane, uint32_t row) {
  return make_float3(__ldcg(p + row), __ldcg(p + (plane + row)), __ldcg(p + (2u * plane + row)));
}

__device__ __forceinline__ float sign_of(float v) {  // np.sign (0 -> 0, NaN -> NaN)
  return v > 0.0f ? 1.0f : (v < 0.0f ? -1.0f : v);
}

// The cost plugin stays in shared memory (holding it in registers cost
// occupancy in the lane-per-sub-rollout kernel).
// crash_now: floor contact or arena exit (simworld.py:157-164)
__device__ __forceinline__ bool nav_crash_now(const pi2_cost &c, float px, float py, float pz) {
  return (pz <= c.z_floor) || (px < c.arena_lo[0]) || (px > c.arena_hi[0]) || (py < c.arena_lo[1]) ||
         (py > c.arena_hi[1]) || (pz > c.arena_hi[2]);
}

// obstacle term 100 exp(-10 d^2) as ex2.approx.ftz(d^2 * (-10 log2 e)): 2 instructions
// instead of __expf's 6 (its denormal fix-ups only matter below 2^-126, far under
// the >= 0.1 stage cost the term is added to); error <= 2e-7 of that cost.
__device__ __forceinline__ float obstacle_term(float px, float py, float ox, float oy) {
  const float dx = __fsub_rn(px, ox), dy = __fsub_rn(py, oy);
  const float t = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
  return __fmul_rn(ex2_ftz(__fmul_rn(t, -14.4269504088896341f)), 100.0f);
}

// stage cost q(x) in the reference's float32 operation order (simworld.py:166-198)
// extra: obstacles PI2_MAX_OBSTACLES.. (StepArgs::extra_obstacles), summed in the same order.
// XOBS = false (the FAST kernels, which the host runs only while the struct holds the whole
// list) drops that loop: it cost the group kernel 7 us at C2 even when never entered.
template <bool XOBS = true>
__device__ __forceinline__ float nav_stage_cost(const pi2_cost &c, const float *__restrict__ extra, float px, float py,
                                                float pz,
                                                float vx, float vy, float vz, float angterm,
                                                bool crashed) {
  float d = __fsub_rn(px, c.waypoint[0]);
  float out = __fmul_rn(d, d);
  d = __fsub_rn(py, c.waypoint[1]);
  out = __fadd_rn(out, __fmul_rn(d, d));
  d = __fsub_rn(pz, c.waypoint[2]);
  out = __fadd_rn(out, __fmul_rn(__fmul_rn(d, d), 10.0f));
  float t = __fmul_rn(vx, vx);
  t = __fadd_rn(t, __fmul_rn(vy, vy));
  t = __fadd_rn(t, __fmul_rn(vz, vz));
  out = __fadd_rn(out, __fmul_rn(t, 0.1f));
  out = __fadd_rn(out, angterm);
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (i < c.n_obstacles) out = __fadd_rn(out, obstacle_term(px, py, c.obstacles[2 * i], c.obstacles[2 * i + 1]));
  const int n_struct = c.n_obstacles < PI2_MAX_OBSTACLES ? c.n_obstacles : PI2_MAX_OBSTACLES;
  for (int i = 4; i < n_struct; ++i)
    out = __fadd_rn(out, obstacle_term(px, py, c.obstacles[2 * i], c.obstacles[2 * i + 1]));
  if (XOBS)
    for (int i = PI2_MAX_OBSTACLES; i < c.n_obstacles; ++i)
      out = __fadd_rn(out, obstacle_term(px, py, __ldg(extra + 2 * (i - PI2_MAX_OBSTACLES)),
                                         __ldg(extra + 2 * (i - PI2_MAX_OBSTACLES) + 1)));
  return __fadd_rn(out, crashed ? 10.0f : 0.0f);
}

#ifndef PI2_ROLL1_AHEAD
#define PI2_ROLL1_AHEAD 1  // rows in flight ahead of the step using them in rollout_kernel; 2 (64 regs) was
                           // slower: C4 rollout 395 -> 409 us (micro/roll_ahead_b200.txt)
#endif
#ifndef PI2_ROLL1_UNROLL
#define PI2_ROLL1_UNROLL 1  // t-loop unroll of rollout_kernel (2 / 4 within noise at C4: micro/roll_unroll_b200.txt)
#endif
constexpr int kRoll1Unroll = PI2_ROLL1_UNROLL;

// MM: compile-time sub-rollouts held in registers (1; more than one sub-rollout per
// rollout runs rollout_group_kernel, up to PI2_MAX_SUB_ROLLOUTS on 32 lanes).
// FAST: hybrid LWPR model + navigation cost, branches folded at compile time.
template <int MM, bool FAST, bool R32 = false>
__global__ void __launch_bounds__(kRolloutBlock) rollout_kernel(RollArgs a) {
  constexpr int MCAP = MM > 0 ? MM : 64;  // MM = 0 (runtime M) is not instantiated: S > 1 runs the group kernel
  extern __shared__ float sq[];  // (N, blockDim): this thread's stage costs, column tid
  __shared__ pi2_cost cost;
  if (threadIdx.x == 0) cost = a.sa->cost;
  __syncthreads();
  pdl_wait();
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= a.K) return;
  // this rollout's stage costs: shared memory, or the global scratch for long horizons
  float *qcol = a.qs ? a.qs + k : sq + threadIdx.x;
  const int64_t qstride = a.qs ? a.K : (int64_t)blockDim.x;
  const int M = MM > 0 ? MM : a.M;
  const int N = a.N;
  const int S = a.spread ? M : 1;
  const StepArgs *sa = a.sa;
  const float p0[3] = {__double2float_rn(sa->state[0]), __double2float_rn(sa->state[1]),
                       __double2float_rn(sa->state[2])};
  const float v0[3] = {__double2float_rn(sa->state[3]), __double2float_rn(sa->state[4]),
                       __double2float_rn(sa->state[5])};
  const Key128 dkey = iter_key(sa->key_prefix[1], (uint64_t)a.iteration);
  const uint64_t dk0 = dkey.k0, dk1 = dkey.k1;
  const uint64_t kg = (uint64_t)(a.k_off + k);
  const bool threshold_cost = !FAST && cost.kind == PI2_COST_THRESHOLD;
  const int model = FAST ? PI2_MODEL_HYBRID_LWPR : a.model;
  const pi2_cost &nav = cost;
  const float *xobs = a.sa->extra_obstacles;  // obstacles past the struct's PI2_MAX_OBSTACLES

  float cs[MCAP][3], ccs[MCAP][3];
  bool crashed[MCAP];
#pragma unroll
  for (int m = 0; m < MCAP; ++m) {
    crashed[m] = false;
#pragma unroll
    for (int c = 0; c < 3; ++c) cs[m][c] = ccs[m][c] = -0.0f;  // -0 + x == x: cumsum start
  }

  // the rows of step t + 1 are loaded while step t computes (hides HBM latency);
  // the analytic model's input row of step t + 1 is this step's post-step attitude row
  const bool hybrid = model == PI2_MODEL_HYBRID_LWPR;
  const bool with_std = hybrid && (a.spread || a.penalty);
  // ap_row(t): the post-step attitude row of step t (xin row t + 1; the last step's from ang_last)
  auto ap_row = [&](int t) { return (t + 1 < N) ? __ldcg(a.xin + (int64_t)(t + 1) * a.K + k) : __ldcg(a.ang_last + k); };
  float3 m4n = make_float3(0.f, 0.f, 0.f), s4n = m4n;
  if (hybrid) m4n = ld_planes(a.lw_mean, a.lw_plane, k);
  if (with_std) s4n = ld_planes(a.lw_std, a.lw_plane, k);
  float4 apn = ap_row(0);
#if PI2_ROLL1_AHEAD >= 2
  // a second row set in flight: one step of this warp's work does not cover the DRAM latency
  // (C4: 35 % of the stall samples sat on the first use of the one-ahead row)
  float3 m4nn = m4n, s4nn = s4n;
  float4 apnn = apn;
  if (1 < N) {
    if (hybrid) m4nn = ld_planes(a.lw_mean, a.lw_plane, a.K + k);
    if (with_std) s4nn = ld_planes(a.lw_std, a.lw_plane, a.K + k);
    apnn = ap_row(1);
  }
#endif
  float4 xr = (model == PI2_MODEL_ANALYTIC) ? __ldcg(a.xin + k) : make_float4(0.f, 0.f, 0.f, 0.f);
  uint32_t rn32 = (uint32_t)(a.K + k);  // R32: the next step's row index
#pragma unroll(kRoll1Unroll)
  for (int t = 0; t < N; ++t) {
    const int64_t row = (int64_t)t * a.K + k;
    const float3 m4 = m4n, s4 = s4n;
    const float4 ap = apn;
#if PI2_ROLL1_AHEAD >= 2
    m4n = m4nn;
    s4n = s4nn;
    apn = apnn;
    if (t + 2 < N) {
      if (hybrid) m4nn = ld_planes(a.lw_mean, a.lw_plane, row + 2 * a.K);
      if (with_std) s4nn = ld_planes(a.lw_std, a.lw_plane, row + 2 * a.K);
      apnn = ap_row(t + 2);
    }
#else
    if (t + 1 < N) {
      if (R32) {  // 32-bit element offsets (see ld_planes32); rn32 = (t + 1) K + k
        const uint32_t rn = rn32, pl = (uint32_t)a.lw_plane;
        rn32 += (uint32_t)a.K;
        if (hybrid) m4n = ld_planes32(a.lw_mean, pl, rn);
        if (with_std) s4n = ld_planes32(a.lw_std, pl, rn);
        apn = (t + 2 < N) ? __ldcg(a.xin + (rn + (uint32_t)a.K)) : __ldcg(a.ang_last + k);
      } else {
        if (hybrid) m4n = ld_planes(a.lw_mean, a.lw_plane, row + a.K);
        if (with_std) s4n = ld_planes(a.lw_std, a.lw_plane, row + a.K);
        apn = ap_row(t + 1);
      }
    }
#endif
    float mn[3], sd[3] = {0.0f, 0.0f, 0.0f};
    if (hybrid) {
      mn[0] = m4.x; mn[1] = m4.y; mn[2] = m4.z;
      if (a.spread) {
        sd[0] = s4.x; sd[1] = s4.y; sd[2] = s4.z;
      }
    } else if (model == PI2_MODEL_ANALYTIC) {  // dynamics.py:175-185
      float sr, cr, sp, cp, sy, cy;
      sincosf(xr.x, &sr, &cr);
      sincosf(xr.y, &sp, &cp);
      sincosf(xr.z, &sy, &cy);
      const float fm = __fmul_rn(xr.w, a.dp.inv_m32);
      const float crsp = __fmul_rn(cr, sp);
      mn[0] = __fmul_rn(fm, __fadd_rn(__fmul_rn(crsp, cy), __fmul_rn(sr, sy)));
      mn[1] = __fmul_rn(fm, __fsub_rn(__fmul_rn(crsp, sy), __fmul_rn(sr, cy)));
      mn[2] = __fsub_rn(__fmul_rn(fm, __fmul_rn(cr, cp)), a.dp.g32);
    } else {  // two-point test model (tests/synthetic.py:402-411)
      mn[0] = mn[1] = mn[2] = 0.0f;
      sd[2] = a.two_point;
    }
    const float pen = (hybrid && a.penalty) ? variance_term(cost.variance_penalty, s4) : 0.0f;
    float angterm = __fmul_rn(
        __fadd_rn(__fadd_rn(__fmul_rn(ap.x, ap.x), __fmul_rn(ap.y, ap.y)), __fmul_rn(ap.z, ap.z)), 0.2f);
    // consume the finite pad lane so ptxas keeps the in-flight prefetch registers (see
    // rollout_group_kernel)
    angterm = fmaf(ap.w, 0.0f, angterm);
    xr = ap;  // the analytic model's input row of step t + 1
    const float sdt = __fmul_rn(a.dp.dt32, (float)(t + 1));
    float q[MCAP];
#pragma unroll
    for (int m = 0; m < MCAP; ++m) {
      if (m >= S) break;
      float acc[3];
      if (a.spread) {
        float d[3];
        if (a.device_dyn) {
          dyn3((kg * (uint64_t)M + (uint64_t)m) * (uint64_t)dyn_blocks(N), t, dk0, dk1, d);
        } else {
          const float *dp = a.dyn + ((k * M + m) * (int64_t)N + t) * 3;
          d[0] = __ldg(dp); d[1] = __ldg(dp + 1); d[2] = __ldg(dp + 2);
        }
        if (model == PI2_MODEL_TWO_POINT) {
          d[0] = sign_of(d[0]); d[1] = sign_of(d[1]); d[2] = sign_of(d[2]);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c] = __fadd_rn(__fmul_rn(sd[c], d[c]), mn[c]);
      } else {
        acc[0] = mn[0]; acc[1] = mn[1]; acc[2] = mn[2];
      }
      float pos[3], vel[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        cs[m][c] = __fadd_rn(cs[m][c], acc[c]);
        ccs[m][c] = __fadd_rn(ccs[m][c], cs[m][c]);
        vel[c] = __fadd_rn(__fmul_rn(cs[m][c], a.dp.dt32), v0[c]);
        pos[c] = __fadd_rn(__fadd_rn(__fmul_rn(__fsub_rn(ccs[m][c], cs[m][c]), a.dp.dt2_32),
                                     __fmul_rn(sdt, v0[c])),
                           p0[c]);
      }
      if (threshold_cost) {
        q[m] = pos[2] > cost.threshold ? 1.0f : 0.0f;
      } else {
        crashed[m] = crashed[m] | nav_crash_now(nav, pos[0], pos[1], pos[2]);  // no short-circuit branch
        q[m] = nav_stage_cost<!FAST>(nav, xobs, pos[0], pos[1], pos[2], vel[0], vel[1], vel[2], angterm, crashed[m]);
      }
    }
    // sub-rollout mean: pairwise halving while even, plain mean when odd
    // (controller.py:314-319)
    int n = S;
    while (n > 1) {
      if ((n & 1) == 0) {
#pragma unroll
        for (int i = 0; i < MCAP / 2; ++i)
          if (i < n / 2) q[i] = __fmul_rn(0.5f, __fadd_rn(q[2 * i], q[2 * i + 1]));
        n >>= 1;
      } else {
        float s = q[0];
#pragma unroll
        for (int i = 1; i < MCAP; ++i)
          if (i < n) s = __fadd_rn(s, q[i]);
        q[0] = __fdiv_rn(s, (float)n);
        n = 1;
      }
    }
    qcol[(int64_t)t * qstride] = (hybrid && a.penalty) ? __fadd_rn(q[0], pen) : q[0];
  }

  bool crash = false;
#pragma unroll
  for (int m = 0; m < MCAP; ++m)
    if (m < S) crash = crash || crashed[m];
  // float64 suffix sum (controller.py:320-322) and ceiling (:243-246)
  const double dt = a.dp.dt, ceiling = sa->ceiling;
  double acc = 0.0;
  double *out = a.costs + k;  // t-major: S(k, t) at out[t * K]
  for (int t = N - 1; t >= 0; --t) {
    const double s = __dmul_rn((double)qcol[(int64_t)t * qstride], dt);
    acc = (t == N - 1) ? s : __dadd_rn(acc, s);
    double v = acc;
    if (!isfinite(v)) {
      v = ceiling;
      crash = true;
    }
    out[(int64_t)t * a.K] = v;
  }
  a.crash[k] = crash ? 1 : 0;
}

#ifndef PI2_ROLL_UNROLL
#define PI2_ROLL_UNROLL 4  // t-loop unroll of rollout_group_kernel (C2 0.633 -> 0.629 ms, micro/roll_unroll_b200.txt)
#endif
constexpr int kRollUnroll = PI2_ROLL_UNROLL;

// Sub-rollouts on lanes: a group of G lanes (G = S rounded up to a power of
// two, <= 32) per rollout, lane m integrating sub-rollout m; G = 64 .. 256
// (33 <= S <= 256) runs 32 lanes holding sub-rollouts m, m + 32, ... each.  The M-mean is
// the reference's pairwise tree (controller.py:314-319): for S == G an xor
// butterfly reproduces it exactly (adjacent pairs at every level, IEEE add
// is commutative; with two slots per lane the butterfly leaves the means of
// 0..31 and 32..63, the tree's last pair); otherwise lane 0 replays the
// reference loop from shared memory.  Lane 0 of the group owns the float64
// suffix sum.
// FAST: hybrid LWPR model, device dynamics noise, navigation cost (the
// real-time configuration) with every branch folded at compile time.
template <int G, bool FAST, bool R32 = false>
__global__ void __launch_bounds__(kRolloutBlock) rollout_group_kernel(RollArgs a) {
  constexpr int SPL = G > 32 ? G / 32 : 1;  // sub-rollouts per lane (G = 64 .. 256: 32 lanes)
  constexpr int GL = G / SPL;             // lanes per rollout
  constexpr int RPB = kRolloutBlock / GL;  // rollouts per block
  extern __shared__ float sq[];           // (N, RPB) stage costs
  __shared__ float qbuf[kRolloutBlock * SPL];
  __shared__ pi2_cost cost;
  if (threadIdx.x == 0) cost = a.sa->cost;
  __syncthreads();
  pdl_wait();
  const int lane_g = threadIdx.x % GL, grp = threadIdx.x / GL;
  const int64_t k = (int64_t)blockIdx.x * RPB + grp;
  const bool live = k < a.K;
  const int S = a.M;
  const int N = a.N;
  bool act[SPL];
#pragma unroll
  for (int j = 0; j < SPL; ++j) act[j] = live && lane_g + j * GL < S;
  const bool active = act[0];
  const StepArgs *sa = a.sa;
  const float p0[3] = {__double2float_rn(sa->state[0]), __double2float_rn(sa->state[1]),
                       __double2float_rn(sa->state[2])};
  const float v0[3] = {__double2float_rn(sa->state[3]), __double2float_rn(sa->state[4]),
                       __double2float_rn(sa->state[5])};
  const Key128 dkey = iter_key(sa->key_prefix[1], (uint64_t)a.iteration);
  const uint64_t dk0 = dkey.k0, dk1 = dkey.k1;
  const uint64_t kg = (uint64_t)(a.k_off + k);
  const bool threshold_cost = !FAST && cost.kind == PI2_COST_THRESHOLD;
  const pi2_cost &nav = cost;
  const float *xobs = a.sa->extra_obstacles;  // obstacles past the struct's PI2_MAX_OBSTACLES
  const int64_t kk = live ? k : 0;
  const bool device_dyn = FAST || a.device_dyn;
  const bool two_point = !FAST && a.model == PI2_MODEL_TWO_POINT;
  // first Philox block of each slot's sub-rollout m = lane_g + j * GL (DynDraws)
  const uint64_t nb = (uint64_t)dyn_blocks(N);
  const uint64_t dyn_base = (kg * (uint64_t)S + (uint64_t)lane_g) * nb;
  DynDraws draws[SPL];

  float cs[SPL][3], ccs[SPL][3];
  bool crashed[SPL];
#pragma unroll
  for (int j = 0; j < SPL; ++j) {
    crashed[j] = false;
#pragma unroll
    for (int c = 0; c < 3; ++c) cs[j][c] = ccs[j][c] = -0.0f;  // -0 + x == x: cumsum start
  }
  const bool hybrid = FAST || a.model == PI2_MODEL_HYBRID_LWPR;
  // rows of step t+1 are loaded while step t computes (hides HBM latency)
  float3 m4n = make_float3(0.f, 0.f, 0.f), s4n = m4n;
  float4 apn = make_float4(0.f, 0.f, 0.f, 0.f);
  if (active) {
    if (hybrid) {
      m4n = ld_planes(a.lw_mean, a.lw_plane, kk);
      s4n = ld_planes(a.lw_std, a.lw_plane, kk);
    }
    apn = (1 < N) ? __ldcg(a.xin + a.K + kk) : __ldcg(a.ang_last + kk);
  }
  const uint32_t plane32 = (uint32_t)a.lw_plane, k32 = (uint32_t)a.K;
  uint32_t row32 = (uint32_t)kk;  // rows32 path: t * K + k
#pragma unroll(kRollUnroll)
  for (int t = 0; t < N; ++t) {
    const int64_t row = (int64_t)t * a.K + kk;
    const float3 m4 = m4n, s4 = s4n;
    const float4 ap = apn;
    if (active && t + 1 < N) {
      if (R32) {
        const uint32_t rn = row32 + k32;
        if (hybrid) {
          m4n = ld_planes32(a.lw_mean, plane32, rn);
          s4n = ld_planes32(a.lw_std, plane32, rn);
        }
        apn = (t + 2 < N) ? __ldcg(a.xin + (rn + k32)) : __ldcg(a.ang_last + kk);
      } else {
        if (hybrid) {
          m4n = ld_planes(a.lw_mean, a.lw_plane, row + a.K);
          s4n = ld_planes(a.lw_std, a.lw_plane, row + a.K);
        }
        apn = (t + 2 < N) ? __ldcg(a.xin + row + 2 * a.K) : __ldcg(a.ang_last + kk);
      }
    }
    row32 += k32;
    float q[SPL];
#pragma unroll
    for (int j = 0; j < SPL; ++j) q[j] = 0.0f;
    const float pen = (hybrid && a.penalty) ? variance_term(cost.variance_penalty, s4) : 0.0f;
    if (active) {
      float mn[3], sd[3] = {0.0f, 0.0f, 0.0f};
      if (hybrid) {
        mn[0] = m4.x; mn[1] = m4.y; mn[2] = m4.z;
        sd[0] = s4.x; sd[1] = s4.y; sd[2] = s4.z;
      } else {  // two-point test model
        mn[0] = mn[1] = mn[2] = 0.0f;
        sd[2] = a.two_point;
      }
      float angterm = __fmul_rn(
          __fadd_rn(__fadd_rn(__fmul_rn(ap.x, ap.x), __fmul_rn(ap.y, ap.y)), __fmul_rn(ap.z, ap.z)), 0.2f);
      // consume the (finite) pad lane of the prefetched attitude row: an unused .w lets
      // ptxas reuse that register while the next step's 128-bit load is still in flight,
      // a write-after-write stall of a full DRAM latency per step (ncu, rollout kernel)
      angterm = fmaf(ap.w, 0.0f, angterm);
      const float sdt = __fmul_rn(a.dp.dt32, (float)(t + 1));
#pragma unroll
      for (int j = 0; j < SPL; ++j) {
        if (!act[j]) continue;
        const int m = lane_g + j * GL;
        float d[3];
        if (device_dyn) {
          draws[j].next(dyn_base + (uint64_t)(j * GL) * nb, t, dk0, dk1, d);
        } else {
          const float *dp = a.dyn + ((kk * S + m) * (int64_t)N + t) * 3;
          d[0] = __ldg(dp); d[1] = __ldg(dp + 1); d[2] = __ldg(dp + 2);
        }
        if (two_point) {
          d[0] = sign_of(d[0]); d[1] = sign_of(d[1]); d[2] = sign_of(d[2]);
        }
        float pos[3], vel[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const float acc = __fadd_rn(__fmul_rn(sd[c], d[c]), mn[c]);
          cs[j][c] = __fadd_rn(cs[j][c], acc);
          ccs[j][c] = __fadd_rn(ccs[j][c], cs[j][c]);
          vel[c] = __fadd_rn(__fmul_rn(cs[j][c], a.dp.dt32), v0[c]);
          pos[c] = __fadd_rn(__fadd_rn(__fmul_rn(__fsub_rn(ccs[j][c], cs[j][c]), a.dp.dt2_32),
                                       __fmul_rn(sdt, v0[c])),
                             p0[c]);
        }
        if (threshold_cost) {
          q[j] = pos[2] > cost.threshold ? 1.0f : 0.0f;
        } else {
          crashed[j] = crashed[j] | nav_crash_now(nav, pos[0], pos[1], pos[2]);  // no short-circuit branch
          q[j] = nav_stage_cost<!FAST>(nav, xobs, pos[0], pos[1], pos[2], vel[0], vel[1], vel[2], angterm, crashed[j]);
        }
      }
    }
    float qm;
    if (S == G) {
#pragma unroll
      for (int j = 0; j < SPL; ++j)
#pragma unroll
        for (int off = 1; off < GL; off <<= 1)
          q[j] = __fmul_rn(0.5f, __fadd_rn(q[j], __shfl_xor_sync(0xffffffffu, q[j], off)));
      // the tree's upper levels pair adjacent 32-blocks: slots (j, j + w)
#pragma unroll
      for (int w = 1; w < SPL; w <<= 1)
#pragma unroll
        for (int j = 0; j + w < SPL; j += 2 * w) q[j] = __fmul_rn(0.5f, __fadd_rn(q[j], q[j + w]));
      qm = q[0];
    } else if (G > 64) {  // replay the reference loop in place in shared memory (one lane)
#pragma unroll
      for (int j = 0; j < SPL; ++j) qbuf[j * kRolloutBlock + threadIdx.x] = q[j];
      __syncwarp();
      qm = 0.0f;
      if (lane_g == 0) {
        // element i of this rollout's sub-rollout costs: slot i / 32, lane i % 32
        auto at = [&](int i) -> float & { return qbuf[(i / GL) * kRolloutBlock + threadIdx.x + i % GL]; };
        int n = S;
        while (n > 1) {
          if ((n & 1) == 0) {
            for (int i = 0; i < n / 2; ++i) at(i) = __fmul_rn(0.5f, __fadd_rn(at(2 * i), at(2 * i + 1)));
            n >>= 1;
          } else {
            float sum = at(0);
            for (int i = 1; i < n; ++i) sum = __fadd_rn(sum, at(i));
            at(0) = __fdiv_rn(sum, (float)n);
            n = 1;
          }
        }
        qm = at(0);
      }
      __syncwarp();
    } else {
#pragma unroll
      for (int j = 0; j < SPL; ++j) qbuf[j * kRolloutBlock + threadIdx.x] = q[j];
      __syncwarp();
      qm = 0.0f;
      if (lane_g == 0) {
        float v[G];
#pragma unroll
        for (int i = 0; i < G; ++i) v[i] = qbuf[(i / GL) * kRolloutBlock + threadIdx.x + i % GL];
        int n = S;
        while (n > 1) {
          if ((n & 1) == 0) {
#pragma unroll
            for (int i = 0; i < G / 2; ++i)
              if (i < n / 2) v[i] = __fmul_rn(0.5f, __fadd_rn(v[2 * i], v[2 * i + 1]));
            n >>= 1;
          } else {
            float s = v[0];
#pragma unroll
            for (int i = 1; i < G; ++i)
              if (i < n) s = __fadd_rn(s, v[i]);
            v[0] = __fdiv_rn(s, (float)n);
            n = 1;
          }
        }
        qm = v[0];
      }
      __syncwarp();
    }
    if (hybrid && a.penalty) qm = __fadd_rn(qm, pen);
    if (lane_g == 0) {
      if (!a.qs) sq[t * RPB + grp] = qm;
      else if (live) a.qs[(int64_t)t * a.K + k] = qm;  // long horizon: global scratch
    }
  }
  // persistent crash of any sub-rollout (controller.py:310)
  bool any = false;
#pragma unroll
  for (int j = 0; j < SPL; ++j) any = any || crashed[j];
  const unsigned ballot = __ballot_sync(0xffffffffu, any);
  const unsigned gmask = (GL == 32) ? 0xffffffffu : (((1u << GL) - 1u) << ((threadIdx.x % 32) / GL * GL));
  // the float64 suffix sums run on the block's first RPB threads, one rollout each (the
  // lanes of the first warps rather than lane 0 of every group: 1/GL of the issue slots)
  __shared__ bool scrash[RPB];
  if (lane_g == 0) scrash[grp] = (ballot & gmask) != 0;
  __syncthreads();  // stage costs (shared memory or the global scratch) and crash flags
  const int r = (int)threadIdx.x;
  const int64_t kr = (int64_t)blockIdx.x * RPB + r;
  if (r >= RPB || kr >= a.K) return;
  bool crash = scrash[r];
  const double dt = a.dp.dt, ceiling = sa->ceiling;
  double acc = 0.0;
  double *out = a.costs + kr;  // t-major: S(k, t) at out[t * K]
  for (int t = N - 1; t >= 0; --t) {
    const double s = __dmul_rn((double)(a.qs ? a.qs[(int64_t)t * a.K + kr] : sq[t * RPB + r]), dt);
    acc = (t == N - 1) ? s : __dadd_rn(acc, s);
    double v = acc;
    if (!isfinite(v)) {
      v = ceiling;
      crash = true;
    }
    out[(int64_t)t * a.K] = v;
  }
  a.crash[kr] = crash ? 1 : 0;
}

// ---------------------------------------------------------------------------
// Small-K (latency) variants: one warp per rollout.  Work that is independent
// across timesteps (noise, clipping, stage costs) is spread over the lanes;
// only the true recurrences stay serial, each on its own lane: the FP64
// attitude/rate recurrence per channel (lanes 0-2), the FP32 cumsum per
// component (lanes 0-2) and the FP64 suffix sum (lane 0).  Same arithmetic,
// same order as the thread-per-rollout kernels -> identical results.
// ---------------------------------------------------------------------------
constexpr int kWideWarps = 4;  // rollouts per block

template <bool DEVICE_NOISE>
__global__ void __launch_bounds__(32 * kWideWarps)
    attitude_wide_kernel(const StepArgs *__restrict__ sa, const double *__restrict__ plan,
                         const double *__restrict__ eps, int iteration, int64_t K, int64_t k_off, int N,
                         DynParams dp, float4 *__restrict__ xin, float4 *__restrict__ ang_last,
                         float4 *__restrict__ zout) {
  extern __shared__ double wsm[];
  double *splan = wsm;                                   // (N, 4)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double *u = splan + 4 * N + (size_t)warp * 4 * N;      // (N, 4) clipped controls of this rollout
  float4 *stage = reinterpret_cast<float4 *>(splan + 4 * N + (size_t)kWideWarps * 4 * N) + (size_t)warp * (N + 1);
  pdl_wait();
  pdl_trigger();
  for (int i = threadIdx.x; i < 4 * N; i += blockDim.x) splan[i] = plan[i];
  __syncthreads();
  const int64_t k = (int64_t)blockIdx.x * kWideWarps + warp;
  if (k >= K) return;
  const Key128 ck = DEVICE_NOISE ? iter_key(sa->key_prefix[0], (uint64_t)iteration) : Key128{0, 0};
  for (int t = lane; t < N; t += 32) {
    double e[4];
    if (DEVICE_NOISE) {
      const float4 z = device_z(ck, (uint64_t)(k_off + k), N, t);
      if (zout) zout[(int64_t)t * K + k] = z;
      eps_from_z(sa, z, e);
    } else {
      const double2 a = __ldg(reinterpret_cast<const double2 *>(eps + (k * N + t) * 4));
      const double2 b = __ldg(reinterpret_cast<const double2 *>(eps + (k * N + t) * 4) + 1);
      e[0] = a.x; e[1] = a.y; e[2] = b.x; e[3] = b.y;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) u[4 * t + c] = clip_np(__dadd_rn(splan[4 * t + c], e[c]), dp.lo[c], dp.hi[c]);
    reinterpret_cast<float *>(&stage[t])[3] = __double2float_rn(u[4 * t + 3]);
  }
  __syncwarp();
  if (lane < 3) {
    const int c = lane;
    const double dt = dp.dt, gdt = dp.gain_dt;
    double ang = sa->state[6 + c], rate = sa->state[9 + c];
#pragma unroll 4
    for (int t = 0; t < N; ++t) {  // the serial chain: controls prefetched from shared memory by the unroll
      reinterpret_cast<float *>(&stage[t])[c] = __double2float_rn(ang);
      ang = wrap_angle(__dadd_rn(ang, __dmul_rn(rate, dt)));
      rate = __dadd_rn(rate, __dmul_rn(gdt, __dsub_rn(u[4 * t + c], rate)));
    }
    reinterpret_cast<float *>(&stage[N])[c] = __double2float_rn(ang);
  }
  __syncwarp();
  for (int t = lane; t < N; t += 32) xin[(int64_t)t * K + k] = stage[t];
  if (lane == 0) ang_last[k] = make_float4(stage[N].x, stage[N].y, stage[N].z, 0.0f);
}

template <bool FAST>
__global__ void __launch_bounds__(32 * kWideWarps) rollout_wide_kernel(RollArgs a) {
  extern __shared__ float fsm[];
  __shared__ pi2_cost cost;
  if (threadIdx.x == 0) cost = a.sa->cost;
  __syncthreads();
  pdl_wait();
  const int N = a.N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // per warp: acc (N,3) -> cs (N,3), ccs (N,3), angterm (N), q (N)
  float *acc = fsm + (size_t)warp * 9 * N, *cs = acc + 3 * N, *ccs = cs + 3 * N;
  float *angt = fsm + (size_t)kWideWarps * 9 * N + (size_t)warp * 2 * N, *q = angt + N;
  const int64_t k = (int64_t)blockIdx.x * kWideWarps + warp;
  if (k >= a.K) return;
  const StepArgs *sa = a.sa;
  const int model = FAST ? PI2_MODEL_HYBRID_LWPR : a.model;
  const bool threshold_cost = !FAST && cost.kind == PI2_COST_THRESHOLD;
  const pi2_cost &nav = cost;
  const float *xobs = a.sa->extra_obstacles;  // obstacles past the struct's PI2_MAX_OBSTACLES
  for (int t = lane; t < N; t += 32) {
    const int64_t row = (int64_t)t * a.K + k;
    float mn[3];
    if (model == PI2_MODEL_HYBRID_LWPR) {
      const float3 m4 = ld_planes(a.lw_mean, a.lw_plane, row);
      mn[0] = m4.x; mn[1] = m4.y; mn[2] = m4.z;
    } else if (model == PI2_MODEL_ANALYTIC) {
      const float4 xr = __ldcg(a.xin + row);
      float sr, cr, sp, cp, sy, cy;
      sincosf(xr.x, &sr, &cr);
      sincosf(xr.y, &sp, &cp);
      sincosf(xr.z, &sy, &cy);
      const float fm = __fmul_rn(xr.w, a.dp.inv_m32);
      const float crsp = __fmul_rn(cr, sp);
      mn[0] = __fmul_rn(fm, __fadd_rn(__fmul_rn(crsp, cy), __fmul_rn(sr, sy)));
      mn[1] = __fmul_rn(fm, __fsub_rn(__fmul_rn(crsp, sy), __fmul_rn(sr, cy)));
      mn[2] = __fsub_rn(__fmul_rn(fm, __fmul_rn(cr, cp)), a.dp.g32);
    } else {
      mn[0] = mn[1] = mn[2] = 0.0f;
    }
    acc[3 * t] = mn[0]; acc[3 * t + 1] = mn[1]; acc[3 * t + 2] = mn[2];
    const float4 ap = (t + 1 < N) ? __ldcg(a.xin + row + a.K) : __ldcg(a.ang_last + k);
    angt[t] = __fmul_rn(__fadd_rn(__fadd_rn(__fmul_rn(ap.x, ap.x), __fmul_rn(ap.y, ap.y)), __fmul_rn(ap.z, ap.z)),
                        0.2f);
  }
  __syncwarp();
  if (lane < 3) {  // np.cumsum twice, sequential (controller.py:294-295)
    float s = -0.0f, ss = -0.0f;
    for (int t = 0; t < N; ++t) {
      s = __fadd_rn(s, acc[3 * t + lane]);
      ss = __fadd_rn(ss, s);
      cs[3 * t + lane] = s;
      ccs[3 * t + lane] = ss;
    }
  }
  __syncwarp();
  const float p0[3] = {__double2float_rn(sa->state[0]), __double2float_rn(sa->state[1]),
                       __double2float_rn(sa->state[2])};
  const float v0[3] = {__double2float_rn(sa->state[3]), __double2float_rn(sa->state[4]),
                       __double2float_rn(sa->state[5])};
  bool carry = false;  // persistent crash indicator up to the previous 32 steps
  for (int t0 = 0; t0 < N; t0 += 32) {
    const int t = t0 + lane;
    float pos[3] = {0, 0, 0}, vel[3] = {0, 0, 0};
    bool now = false;
    if (t < N) {
      const float sdt = __fmul_rn(a.dp.dt32, (float)(t + 1));
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        vel[c] = __fadd_rn(__fmul_rn(cs[3 * t + c], a.dp.dt32), v0[c]);
        pos[c] = __fadd_rn(__fadd_rn(__fmul_rn(__fsub_rn(ccs[3 * t + c], cs[3 * t + c]), a.dp.dt2_32),
                                     __fmul_rn(sdt, v0[c])), p0[c]);
      }
      now = !threshold_cost && nav_crash_now(nav, pos[0], pos[1], pos[2]);
    }
    // logical_or.accumulate along t (controller.py:306): prefix OR via ballot
    const unsigned b = __ballot_sync(0xffffffffu, now);
    const bool crashed = carry || (b & (0xffffffffu >> (31 - lane))) != 0;
    carry = carry || b != 0;
    if (t < N) {
      q[t] = threshold_cost ? (pos[2] > cost.threshold ? 1.0f : 0.0f)
                            : nav_stage_cost<!FAST>(nav, xobs, pos[0], pos[1], pos[2], vel[0], vel[1], vel[2], angt[t], crashed);
      if (model == PI2_MODEL_HYBRID_LWPR && a.penalty)
        q[t] = __fadd_rn(q[t], variance_term(cost.variance_penalty, ld_planes(a.lw_std, a.lw_plane, (int64_t)t * a.K + k)));
    }
  }
  __syncwarp();
  if (lane != 0) return;
  bool crash = carry;
  const double dt = a.dp.dt, ceiling = sa->ceiling;
  double s = 0.0;
  double *out = a.costs + k;
  for (int t = N - 1; t >= 0; --t) {
    const double v = __dmul_rn((double)q[t], dt);
    s = (t == N - 1) ? v : __dadd_rn(s, v);
    double w = s;
    if (!isfinite(w)) {
      w = ceiling;
      crash = true;
    }
    out[(int64_t)t * a.K] = w;
  }
  a.crash[k] = crash ? 1 : 0;
}

// ---------------------------------------------------------------------------
// K11a: leaf partials of the per-timestep softmax (controller.py:367-370):
// per chunk of kChunk rollouts and per t: m = min S, Z = sum w, V = sum w eps,
// w = exp((S - m) * neg_inv).  Warp w handles t = w, w + 8, ...; lane order and
// the xor butterfly are fixed, lane 0's value is kept: deterministic.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

#ifndef PI2_PARTIALS_ZAHEAD
#define PI2_PARTIALS_ZAHEAD 3  // stored-normal loads issued this many elements ahead (0: in the loop);
                               // C4 partials 379 (0) / 285 (2) / 252 (3, 64 regs) us; 4 needs > 64 regs
                               // (3 blocks/SM): 330 us (micro/partials_zahead_b200.txt)
#endif
#ifndef PI2_PARTIALS_MINB
#define PI2_PARTIALS_MINB 0  // > 0: __launch_bounds__ minimum blocks per SM (register cap)
#endif
#if PI2_PARTIALS_MINB > 0
__global__ void __launch_bounds__(32 * kChunkWarps, PI2_PARTIALS_MINB)
#else
__global__ void __launch_bounds__(32 * kChunkWarps)
#endif
    partials_kernel(const double *__restrict__ costs, int64_t cs_k, int64_t cs_t,
                    const double *__restrict__ eps, const float4 *zin, const StepArgs *__restrict__ sa, int iteration,
                    int64_t K, int64_t k_off, int N, double neg_inv, double *__restrict__ out) {
  constexpr int J = kChunk / 32;
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = blockIdx.y * kChunkWarps + warp;  // one warp per (chunk, t)
  if (t >= N) return;
  const int64_t k0 = (int64_t)blockIdx.x * kChunk;
  double s[J];
  double m = INFINITY;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int64_t k = k0 + lane + 32 * j;
    s[j] = k < K ? __ldcg(costs + k * cs_k + t * cs_t) : INFINITY;  // S(k, t); coherent (see pdl_wait)
    m = fmin(m, s[j]);
  }
  m = warp_min(m);
  double z = 0.0, v[4] = {0.0, 0.0, 0.0, 0.0};
  const Key128 ck = (eps || zin) ? Key128{0, 0} : iter_key(sa->key_prefix[0], (uint64_t)iteration);
#if PI2_PARTIALS_ZAHEAD > 0
  if (zin && !eps) {  // stored normals: PI2_PARTIALS_ZAHEAD element loads in flight ahead of the f64 exp chain
    constexpr int ZA = PI2_PARTIALS_ZAHEAD;
    float4 zb[ZA];
#pragma unroll
    for (int j = 0; j < ZA; ++j) {
      const int64_t k = k0 + lane + 32 * j;
      zb[j] = k < K ? __ldcg(zin + (int64_t)t * K + k) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const float4 zc = zb[j % ZA];
      if (j + ZA < J) {
        const int64_t kn = k0 + lane + 32 * (j + ZA);
        zb[j % ZA] = kn < K ? __ldcg(zin + (int64_t)t * K + kn) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      const int64_t k = k0 + lane + 32 * j;
      if (k >= K) continue;
      const double w = exp(__dmul_rn(__dsub_rn(s[j], m), neg_inv));
      double e[4];
      eps_from_z(sa, zc, e);
      z = __dadd_rn(z, w);
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = __dadd_rn(v[c], __dmul_rn(w, e[c]));
    }
  } else
#endif
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int64_t k = k0 + lane + 32 * j;
    if (k >= K) continue;
    const double w = exp(__dmul_rn(__dsub_rn(s[j], m), neg_inv));
    double e[4];
    if (eps) {
      const double2 a = __ldg(reinterpret_cast<const double2 *>(eps + (k * N + t) * 4));
      const double2 b = __ldg(reinterpret_cast<const double2 *>(eps + (k * N + t) * 4) + 1);
      e[0] = a.x; e[1] = a.y; e[2] = b.x; e[3] = b.y;
    } else if (zin) {  // the attitude kernel's normals (coherent: written earlier in the chain)
      eps_from_z(sa, __ldcg(zin + (int64_t)t * K + k), e);
    } else {
      device_eps(sa, ck, (uint64_t)(k_off + k), N, t, e);
    }
    z = __dadd_rn(z, w);
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = __dadd_rn(v[c], __dmul_rn(w, e[c]));
  }
  z = warp_sum(z);
#pragma unroll
  for (int c = 0; c < 4; ++c) v[c] = warp_sum(v[c]);
  if (lane == 0) {
    double *o = out + ((int64_t)blockIdx.x * N + t) * PI2_PARTIAL_WIDTH;
    o[0] = m; o[1] = z; o[2] = v[0]; o[3] = v[1]; o[4] = v[2]; o[5] = v[3];
  }
}

// Few (chunk, t) pairs (small K): the same partials with each (chunk, t) spread over
// a block of kChunk / 32 warps, one element per lane, so the per-element f64 exp and
// noise regeneration run in parallel rather than as 8 sequential elements per lane.
// Bitwise equal to partials_kernel: the min is exact in any grouping, and warp 0
// adds the staged w and w*e in partials_kernel's j order before the same butterfly.
__global__ void __launch_bounds__(kChunk)
    partials_split_kernel(const double *__restrict__ costs, int64_t cs_k, int64_t cs_t,
                          const double *__restrict__ eps, const float4 *zin, const StepArgs *__restrict__ sa,
                          int iteration,
                          int64_t K, int64_t k_off, int N, double neg_inv, double *__restrict__ out) {
  constexpr int J = kChunk / 32;
  __shared__ double smin[J];
  __shared__ double sp[J][5][32];  // [j][w, w*e0..w*e3][lane]
  pdl_wait();
  const int lane = threadIdx.x & 31, j = threadIdx.x >> 5;
  const int t = blockIdx.y;
  const int64_t k0 = (int64_t)blockIdx.x * kChunk;
  const int64_t k = k0 + lane + 32 * j;
  const double s = k < K ? __ldcg(costs + k * cs_k + t * cs_t) : INFINITY;  // coherent (see pdl_wait)
  double m = warp_min(s);
  if (lane == 0) smin[j] = m;
  __syncthreads();
  m = smin[0];
#pragma unroll
  for (int i = 1; i < J; ++i) m = fmin(m, smin[i]);
  if (k < K) {
    const double w = exp(__dmul_rn(__dsub_rn(s, m), neg_inv));
    double e[4];
    if (eps) {
      const double2 a = __ldg(reinterpret_cast<const double2 *>(eps + (k * N + t) * 4));
      const double2 b = __ldg(reinterpret_cast<const double2 *>(eps + (k * N + t) * 4) + 1);
      e[0] = a.x; e[1] = a.y; e[2] = b.x; e[3] = b.y;
    } else if (zin) {
      eps_from_z(sa, __ldcg(zin + (int64_t)t * K + k), e);
    } else {
      device_eps(sa, iter_key(sa->key_prefix[0], (uint64_t)iteration), (uint64_t)(k_off + k), N, t, e);
    }
    sp[j][0][lane] = w;
#pragma unroll
    for (int c = 0; c < 4; ++c) sp[j][1 + c][lane] = __dmul_rn(w, e[c]);
  }
  __syncthreads();
  if (j != 0) return;
  double z = 0.0, v[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < J; ++i) {
    if (k0 + lane + 32 * i >= K) continue;
    z = __dadd_rn(z, sp[i][0][lane]);
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = __dadd_rn(v[c], sp[i][1 + c][lane]);
  }
  z = warp_sum(z);
#pragma unroll
  for (int c = 0; c < 4; ++c) v[c] = warp_sum(v[c]);
  if (lane == 0) {
    double *o = out + ((int64_t)blockIdx.x * N + t) * PI2_PARTIAL_WIDTH;
    o[0] = m; o[1] = z; o[2] = v[0]; o[3] = v[1]; o[4] = v[2]; o[5] = v[3];
  }
}

// t-major (N, K) -> reference (K, N), 32x32 tiles through shared memory
__global__ void transpose_costs_kernel(const double *__restrict__ src, double *__restrict__ dst, int64_t K,
                                       int N) {
  __shared__ double tile[32][33];
  const int64_t k0 = (int64_t)blockIdx.x * 32;
  const int t0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int t = t0 + i;
    const int64_t k = k0 + threadIdx.x;
    if (t < N && k < K) tile[i][threadIdx.x] = src[(int64_t)t * K + k];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t k = k0 + i;
    const int t = t0 + threadIdx.x;
    if (t < N && k < K) dst[k * N + t] = tile[threadIdx.x][i];
  }
}

// plan[t] += V/Z of a single partial, clipped (the world-size-1 finalize)
// plan_host (may be null): the updated plan is also stored there (pinned host memory,
// device-accessible under unified addressing) -- the last iteration of a host call
// so no device-to-host copy follows
// The step's inputs (StepArgs + plan) pulled from pinned host memory over
// unified addressing at the head of the I/O graph, instead of a copy-engine
// node.  No early trigger: every later kernel of the step starts after these
// writes are complete.  Volatile loads: the host rewrites the block between
// replays.
__global__ void io_pull_kernel(const uint4 *src_host, uint4 *__restrict__ dst, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldcv(src_host + i);
}

__global__ void apply_root_kernel(const double *__restrict__ root, int N, double *__restrict__ plan,
                                  DynParams dp, double *plan_host) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 4 * N) return;
  const int t = i / 4, c = i % 4;
  const double *r = root + t * PI2_PARTIAL_WIDTH;
  const double du = __ddiv_rn(__ldcg(r + 2 + c), __ldcg(r + 1));  // coherent (see pdl_wait)
  plan[i] = clip_np(__dadd_rn(plan[i], du), dp.lo[c], dp.hi[c]);
  if (plan_host) plan_host[i] = plan[i];
}

// ---------------------------------------------------------------------------
// K11b: per-timestep adjacent binary tree over `n` partials laid out
// (n, N, 6): segments of kSeg leaves reduced in shared memory, then the
// segment roots.  Identical tree for any split of the leaves into aligned
// power-of-two runs (one per GPU) => G-invariant update.  Optionally writes
// the root and/or applies plan[t] = clip(plan[t] + V/Z) (controller.py:369-371).
// ---------------------------------------------------------------------------
__device__ void smem_tree(double (*v)[PI2_PARTIAL_WIDTH], int n, double neg_inv) {
  for (int st = 1; st < n; st <<= 1) {
    // pair p = (v[2 st p], v[2 st p + st]); thread p, p + blockDim, ... (no division)
    for (int i = 2 * st * (int)threadIdx.x; i + st < n; i += 2 * st * (int)blockDim.x)
      partial_combine(v[i], v[i + st], neg_inv);
    __syncthreads();
  }
}

constexpr int kCombineThreads = 256;
__global__ void __launch_bounds__(kCombineThreads)
    combine_kernel(const double *__restrict__ leaves, int64_t n, int N, double neg_inv,
                   double *__restrict__ root_out, double *__restrict__ plan, DynParams dp, double *plan_host) {
  extern __shared__ double cmb[];
  double(*seg)[PI2_PARTIAL_WIDTH] = reinterpret_cast<double(*)[PI2_PARTIAL_WIDTH]>(cmb);
  double(*roots)[PI2_PARTIAL_WIDTH] = seg + kSeg;
  pdl_wait();
  const int t = blockIdx.x;
  const int64_t nseg = (n + kSeg - 1) / kSeg;
  // the next segment's leaves are loaded into registers while this one's tree runs
  // (blockDim = kCombineThreads: kSeg / kCombineThreads leaves per thread); a leaf's 6
  // doubles are 48 contiguous, 16-byte aligned bytes: three 128-bit loads
  constexpr int LPT = kSeg / kCombineThreads;
  double2 nx[LPT][PI2_PARTIAL_WIDTH / 2];
  auto load_seg = [&](int64_t s) {
    const int cnt = (int)(n - s * kSeg < kSeg ? n - s * kSeg : kSeg);
#pragma unroll
    for (int j = 0; j < LPT; ++j) {
      const int i = (int)threadIdx.x + j * kCombineThreads;
      if (i >= cnt) break;
      const double2 *src = reinterpret_cast<const double2 *>(leaves + ((s * kSeg + i) * N + t) * PI2_PARTIAL_WIDTH);
#pragma unroll
      for (int c = 0; c < PI2_PARTIAL_WIDTH / 2; ++c) nx[j][c] = __ldcg(src + c);  // coherent (see pdl_wait)
    }
  };
  load_seg(0);
  for (int64_t s = 0; s < nseg; ++s) {
    const int cnt = (int)(n - s * kSeg < kSeg ? n - s * kSeg : kSeg);
#pragma unroll
    for (int j = 0; j < LPT; ++j) {
      const int i = (int)threadIdx.x + j * kCombineThreads;
      if (i >= cnt) break;
#pragma unroll
      for (int c = 0; c < PI2_PARTIAL_WIDTH / 2; ++c) {
        seg[i][2 * c] = nx[j][c].x;
        seg[i][2 * c + 1] = nx[j][c].y;
      }
    }
    __syncthreads();
    if (s + 1 < nseg) load_seg(s + 1);
    smem_tree(seg, cnt, neg_inv);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int c = 0; c < PI2_PARTIAL_WIDTH; ++c) roots[s][c] = seg[0][c];
    }
    __syncthreads();
  }
  smem_tree(roots, (int)nseg, neg_inv);
  if (threadIdx.x == 0) {
    if (root_out) {
#pragma unroll
      for (int c = 0; c < PI2_PARTIAL_WIDTH; ++c) root_out[t * PI2_PARTIAL_WIDTH + c] = roots[0][c];
    }
    if (plan) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double du = __ddiv_rn(roots[0][2 + c], roots[0][1]);
        plan[4 * t + c] = clip_np(__dadd_rn(plan[4 * t + c], du), dp.lo[c], dp.hi[c]);
        if (plan_host) plan_host[4 * t + c] = plan[4 * t + c];
      }
    }
  }
}

// plan <- shifted plan (ControlPlan.shifted, controller.py:63-66), on device
__global__ void shift_plan_kernel(const double *__restrict__ src, double *__restrict__ dst, int N) {
  for (int i = threadIdx.x; i < 4 * N; i += blockDim.x) {
    const int t = i / 4, c = i % 4;
    dst[i] = src[4 * (t + 1 < N ? t + 1 : N - 1) + c];
  }
}

// device noise materialisation (tests / RolloutBatch.noise of device mode)
__global__ void noise_kernel(const StepArgs *__restrict__ sa, int which, uint64_t iteration, int64_t K,
                             int64_t k_off, int N, int M, double *__restrict__ eps_out,
                             float *__restrict__ dyn_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (which == PI2_STREAM_CONTROL) {
    if (i >= K * N) return;
    const int64_t k = i / N;
    const int t = (int)(i % N);
    double e[4];
    device_eps(sa, iter_key(sa->key_prefix[0], iteration), (uint64_t)(k_off + k), N, t, e);
#pragma unroll
    for (int c = 0; c < 4; ++c) eps_out[i * 4 + c] = e[c];
  } else {
    if (i >= K * M * N) return;  // i = (k * M + m) * N + t
    const int t = (int)(i % N);
    const uint64_t km = (uint64_t)(k_off * M + i / N);  // global (k, m)
    const Key128 dk = iter_key(sa->key_prefix[1], iteration);
    float d[3];
    dyn3(km * (uint64_t)dyn_blocks(N), t, dk.k0, dk.k1, d);
    dyn_out[i * 3 + 0] = d[0];
    dyn_out[i * 3 + 1] = d[1];
    dyn_out[i * 3 + 2] = d[2];
  }
}

}  // namespace pi2
