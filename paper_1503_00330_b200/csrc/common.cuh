// common.cuh — shared types and host/device helpers of the PI²-RH engine.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "pi2rh.h"

#define PI2_HD __host__ __device__ __forceinline__

namespace pi2 {

#ifndef PI2_ROLL_BLOCK  // threads per attitude / rollout block (micro/roll_block_b200.txt: 64 = 128 < 256)
#define PI2_ROLL_BLOCK 128
#endif
constexpr int kRolloutBlock = PI2_ROLL_BLOCK;  // threads (= rollouts) per attitude / rollout block
constexpr int kLwprBlock = 128;     // threads per LWPR block
constexpr int kLwprRows = 8;        // rows (k,t) per LWPR thread (register blocking)
constexpr int kChunk = 256;         // rollouts per leaf partial (fixed => G-invariant tree)
constexpr int kChunkWarps = 8;      // warps per partials block
constexpr int kPartialsSplitBlocks = 296;  // below this many partials_kernel blocks, partials_split_kernel
constexpr int kSeg = 1024;          // leaves per combine segment
constexpr int kMaxSmallM = 8;       // sub-rollouts held in registers
constexpr int kSmemHorizon = 400;     // up to this many steps the rollout kernels keep stage costs in shared
                                      // memory and the warp-per-rollout kernels are eligible
constexpr int kMaxHorizon = 4096;     // the attitude kernel stages the plan in shared memory up to this horizon
constexpr int64_t kWideMaxK = 8192;  // up to this K, attitude/rollout use a warp per rollout (latency);
                                     // measured crossover ~8192 (profiles/micro/wide_threshold_b200.txt)
constexpr double kPi = 3.141592653589793;        // np.pi
constexpr double kTwoPi = 6.283185307179586;     // 2.0 * math.pi
constexpr double kLog2e = 1.4426950408889634;
// LWPR weights are evaluated as 2^(logit*log2e + kExpShift): every weight the
// reference can represent (float32 denormals included) is a
// normal float here, so ex2.approx.ftz is exact-range.
constexpr double kExpShift = 64.0;
// below this (scaled) normaliser a row is re-evaluated with the reference's
// denormal rounding emulated: unscaled den < 2^-110.
constexpr float kSlowDen = 1.4210854715202004e-14f;  // 2^-46

// float records per receptive field in HBM/shared memory
constexpr int kRecDiag = 16;    // 4 x float4
constexpr int kRecFull = 24;    // 6 x float4
constexpr int kRecShared = 12;  // 3 x float4
constexpr int kLayDiag = 0, kLayFull = 1, kLayShared = 2;

// Host/device exact arithmetic (no contraction) for code whose rounding must
// match on both sides.
#ifdef __CUDA_ARCH__
#define PI2_DADD(a, b) __dadd_rn((a), (b))
#define PI2_DSUB(a, b) __dsub_rn((a), (b))
#define PI2_DMUL(a, b) __dmul_rn((a), (b))
#define PI2_DDIV(a, b) __ddiv_rn((a), (b))
#else
#define PI2_DADD(a, b) ((a) + (b))
#define PI2_DSUB(a, b) ((a) - (b))
#define PI2_DMUL(a, b) ((a) * (b))
#define PI2_DDIV(a, b) ((a) / (b))
#endif

// Per-call data read by the kernels from device memory (so that CUDA graph
// replays pick up new state / keys / cost without re-capture).
struct StepArgs {
  double state[12];
  // [control|dynamics]: the (seed, stream, cycle) links of the key chain; each
  // kernel derives its iteration's key itself (iter_key), so any iteration count
  // runs from one staged StepArgs
  uint64_t key_prefix[2];
  double std[4];
  double neg_inv_temp;  // -1 / temperature (controller.py:368)
  double ceiling;       // cost_ceiling (controller.py:243-246)
  pi2_cost cost;
  // obstacles PI2_MAX_OBSTACLES .. cost.n_obstacles - 1 as (x, y) pairs in HBM (the
  // reference takes any count, simworld.py:141-146); nullptr when the struct holds them all
  const float *extra_obstacles;
};

struct DynParams {
  double dt, gain_dt;  // gain_dt = rate_gain * dt (controller.py:266)
  double lo[4], hi[4];
  float dt32, dt2_32;   // float32(dt), float32(dt)^2 (controller.py:255, :297)
  float inv_m32, g32;   // AnalyticModel constants (dynamics.py:172-173)
};

struct AxisHeader {
  float g0, gs[4];  // global linear shift g(x) = g0 + gs.x folded out of the local models
  float qd[10];     // shared metric: log2e * (-1/2 x'Dx) coefficients (Q00 Q01 Q02 Q03 Q11 Q12 Q13 Q22 Q23 Q33)
  float mu[4];      // shared metric: inputs are centred, x~ = x - mu (mean field centre); 0 otherwise
  int num_fields;
  int64_t offset;   // float offset of the axis' first record
};

// ---- path-integral partials: (min S, Z, V[4]) per timestep ---------------
// Leaf: m = min_k S, Z = sum exp((S-m)*neg_inv), V = sum exp(..)*eps.
// a <- a (+) b, fixed arithmetic; Z == 0 marks the identity.
PI2_HD void partial_combine(double *a, const double *b, double neg_inv) {
  if (b[1] == 0.0) return;
  if (a[1] == 0.0) {
    for (int i = 0; i < PI2_PARTIAL_WIDTH; ++i) a[i] = b[i];
    return;
  }
  const double m = a[0] < b[0] ? a[0] : b[0];
  const double sa = exp(PI2_DMUL(PI2_DSUB(a[0], m), neg_inv));
  const double sb = exp(PI2_DMUL(PI2_DSUB(b[0], m), neg_inv));
  a[0] = m;
  for (int i = 1; i < PI2_PARTIAL_WIDTH; ++i)
    a[i] = PI2_DADD(PI2_DMUL(a[i], sa), PI2_DMUL(b[i], sb));
}

// wrap_angle: pi - mod(pi - a, 2 pi) with numpy float remainder semantics
// (dynamics.py:27-29; npy_divmod: fmod, then a negative remainder shifted by +2 pi).  For |x| < 2 pi fmod(x, 2 pi) is x itself, so the common
// path is branch-free (selects: no divergence between the lanes that run the three
// angles); on [2 pi, 4 pi) it is the exact x - 2 pi (Sterbenz); anything else takes
// the general, exact fmod.  Host and device compile the same IEEE operations
// (tests/test_wrap_host.py checks the host build against numpy bit for bit).
PI2_HD double wrap_angle(double a) {
  const double x = PI2_DSUB(kPi, a);
  double m;
  if (fabs(x) < kTwoPi) {
    // a zero remainder's sign (numpy makes it +0) cannot change pi - m
    m = x < 0.0 ? PI2_DADD(x, kTwoPi) : x;
  } else {
    m = (x >= kTwoPi && x < 2.0 * kTwoPi) ? PI2_DSUB(x, kTwoPi) : fmod(x, kTwoPi);  // 4 pi itself: fmod -> 0
    if (m != 0.0) {
      if (m < 0.0) m = PI2_DADD(m, kTwoPi);
    } else {
      m = 0.0;
    }
  }
  return PI2_DSUB(kPi, m);
}

// splitmix64 + the reference's stream-address chain (rng.py:24-44).
PI2_HD uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// 128-bit Philox key of one stream address
struct Key128 {
  uint64_t k0, k1;
};

// first links of the chain: (seed, stream, cycle)
inline uint64_t key_prefix(uint64_t seed, uint64_t stream, uint64_t cycle) {
  uint64_t h = splitmix64(seed);
  h = splitmix64(h ^ stream);
  return splitmix64(h ^ cycle);
}

// last links: the key of optimisation iteration `it` under a prefix
PI2_HD Key128 iter_key(uint64_t prefix, uint64_t it) {
  const uint64_t h = splitmix64(prefix ^ it);
  return Key128{splitmix64(h), splitmix64(h ^ 0xA5A5A5A5A5A5A5A5ull)};
}

inline void derive_key(uint64_t seed, uint64_t stream, uint64_t cycle, uint64_t iteration,
                       uint64_t out[2]) {
  const Key128 k = iter_key(key_prefix(seed, stream, cycle), iteration);
  out[0] = k.k0;
  out[1] = k.k1;
}

}  // namespace pi2
