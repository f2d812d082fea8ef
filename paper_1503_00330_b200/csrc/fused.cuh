// fused.cuh — a device-noise iteration's rollouts in ONE kernel:
//   attitude recurrence (FP64)  ->  LWPR predict of the 3 axes (tcgen05, lwpr_tc's per-row
//   arithmetic)  ->  sub-rollout integration + stage cost  ->  float64 suffix sum,
// per block of 128 rollouts, timestep by timestep (controller.py:257-322, simworld.py:157-198).
//
// The unfused chain (attitude_kernel -> lwpr_tc_kernel -> rollout kernels) hands the LWPR
// input rows (xin, 16 B per rollout-step) and the LWPR mean/std planes (24 B) through HBM;
// here they stay in registers and shared memory: thread i of a CTA owns rollout kb*128 + i
// at every step, which is also row i of the CTA's 128-row LWPR tile (TMEM lane i), so the
// finalized mean/std of its row is exactly what its rollout integrates next.  Only the
// exploration normals (for the path-integral update), the stage costs (for the suffix sum)
// and the costs-to-go leave the SM.
//
// Schedule: items (t, axis, chunk) in order; at every item one CTA barrier and one 3xTF32
// MMA chunk (as lwpr_tc_body), the chunk's W streamed by TMA one item ahead.  In the
// MMA's shadow at an axis' first chunk: finalize the previous axis, integrate the
// rollouts of the previous step (at axis 0), and stage the next axis' features
// (at axis 2: the attitude step t + 1 first).  Every value is computed with the same
// operations in the same order as the unfused kernels: costs, crash flags and normals
// are bitwise equal (tests/test_gpu_fused.py).
#pragma once

#include "lwpr_tc.cuh"

namespace pi2 {

struct FusedArgs {
  LwprTcArgs tc;        // W blob, chunk table, axis headers, exact-path records (x / mean_out / sd_out unused)
  const StepArgs *sa;
  const double *plan;   // (N, 4) device plan (the previous iteration's update)
  int iteration;
  int64_t K, k_off;
  int N, M;
  int spread, penalty;  // sub-rollouts integrated (M > 1, probabilistic model); variance penalty on
  DynParams dp;
  float4 *zout;         // (N, K) exploration normals, t-major (partials kernel)
  float *qbuf;          // (N, K) sub-rollout-mean stage costs, t-major (scratch, L2-resident)
  double *costs;        // (N, K) costs-to-go, t-major
  uint8_t *crash;       // (K)
};

constexpr int kFusedMaxChunks = 4;  // fields per axis <= kFusedMaxChunks * kTcChunk (variances resident)
constexpr int kFusedMaxM = 4;       // sub-rollouts held per thread

// shared-memory bytes of fused_step_kernel<., MM> for chunk counts nch[3]
inline int fused_smem_bytes(const int nch[3], int MM) {
  const int lv = (nch[0] + nch[1] + nch[2]) * kTcChunk;
  int b = ((2 * kTcWSlotFloats + lv) * 4 + 127) / 128 * 128;  // W ring + variances
  b += 2 * kTcABytes;                                         // A operands
  b += (8 + 6 + 6 * MM + 3) * 128 * 4;                        // xs (2 x float4), ms, rollout state
  return b;
}


template <bool VAR, int MM>
__global__ void __launch_bounds__(kTcThreads, kTcCtasPerSm) fused_step_kernel(const __grid_constant__ FusedArgs f) {
  extern __shared__ __align__(128) uint8_t tsm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ __align__(8) uint64_t wbar[2];
  __shared__ pi2_cost cost;
  __shared__ double splan[2][4];  // plan rows of the next attitude steps, staged an axis ahead (L2 latency)
  const LwprTcArgs &a = f.tc;
  const int tid = threadIdx.x, warp = tid >> 5;
  // chunk counts and variance offsets by axis without local arrays (runtime-indexed arrays
  // would live in local memory)
  const int nch0 = a.nchunks[0], nch1 = a.nchunks[1], nch2 = a.nchunks[2];
  auto nch_of = [&](int ax) { return ax == 0 ? nch0 : (ax == 1 ? nch1 : nch2); };
  auto lvb_of = [&](int ax) { return ax == 0 ? 0 : (ax == 1 ? nch0 * kTcChunk : (nch0 + nch1) * kTcChunk); };
  const int nlv = (nch0 + nch1 + nch2) * kTcChunk;
  // shared memory: W ring | variances | A x 2 | per-thread slots (slot s of thread i at [s * 128 + i])
  float *sw = reinterpret_cast<float *>(tsm);
  float *slv = sw + 2 * kTcWSlotFloats;
  uint8_t *sa = tsm + ((2 * kTcWSlotFloats + nlv) * 4 + 127) / 128 * 128;
  float4 *xs = reinterpret_cast<float4 *>(sa + 2 * kTcABytes);  // LWPR input row of step t at xs[(t & 1) * 128 + i]
  float *ms = reinterpret_cast<float *>(xs + 2 * 128);            // [axis][mean, std] of the step being integrated
  float *roll = ms + 6 * 128;  // cs[MM][3], ccs[MM][3], crashed bits, post-step attitude term of steps t & 1
  constexpr int kCrashSlot = 6 * MM, kAngSlot = 6 * MM + 1;

  for (int i = tid; i < nlv; i += blockDim.x) {
    const int ax = i < lvb_of(1) ? 0 : (i < lvb_of(2) ? 1 : 2);
    slv[i] = __ldg(a.w + a.lv_off[ax] + (i - lvb_of(ax)));
  }
  const uint32_t wbar_addr = (uint32_t)__cvta_generic_to_shared(&wbar[0]);
  const uint32_t mbar_addr = (uint32_t)__cvta_generic_to_shared(&mbar);
  const uint32_t sw_addr = (uint32_t)__cvta_generic_to_shared(sw);
  auto load_w = [&](int ax, int c, uint32_t slot) {  // thread 0: chunk (ax, c)'s W into ring slot `slot`
    const uint32_t bytes = (uint32_t)(2 * 2 * a.chunk_pad[ax][c] * 8 * 4);
    const uint32_t bar = wbar_addr + 8 * slot;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            sw_addr + slot * (uint32_t)(kTcWSlotFloats * 4)),
        "l"(a.w + a.axis_off[ax] + a.chunk_woff[ax][c]), "r"(bytes), "r"(bar)
        : "memory");
  };
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)),
                 "n"(kTcTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const int64_t K = f.K, nblocks = (K + kTcThreads - 1) / kTcThreads;
  const int N = f.N;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_addr));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(wbar_addr));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(wbar_addr + 8));
    asm volatile("fence.mbarrier_init.release.cluster;");
    if ((int64_t)blockIdx.x < nblocks) load_w(0, 0, 0);  // the first item's W
  }
  // the plan is the previous iteration's update, StepArgs may come from the I/O graph's
  // input-pull kernel, the normals / costs buffers are read by the previous iteration's
  // partials kernel: everything below waits for the predecessor grid
  pdl_wait();
  const StepArgs *sa_args = f.sa;
  if (tid == 0) cost = sa_args->cost;
  const float *xobs = nullptr;  // the host takes this kernel only while pi2_cost holds every obstacle
  const DynParams &dp = f.dp;
  const int S = f.spread ? f.M : 1;
  const Key128 ck = iter_key(sa_args->key_prefix[0], (uint64_t)f.iteration);
  const Key128 dkey = iter_key(sa_args->key_prefix[1], (uint64_t)f.iteration);
  const float p0[3] = {__double2float_rn(sa_args->state[0]), __double2float_rn(sa_args->state[1]),
                       __double2float_rn(sa_args->state[2])};
  const float v0[3] = {__double2float_rn(sa_args->state[3]), __double2float_rn(sa_args->state[4]),
                       __double2float_rn(sa_args->state[5])};
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t tmem_lane = tmem + ((uint32_t)(warp * 32) << 16);
  const uint32_t sa_addr0 = (uint32_t)__cvta_generic_to_shared(sa);
  PI2_TC_TDECL
  uint32_t phase = 0, nw = 0;  // MMA barrier phase; items issued (W ring position)
  int buf = 0;                 // A operand of the current axis: alternates per axis, continues across blocks

  for (int64_t kb = blockIdx.x; kb < nblocks; kb += gridDim.x) {
    const int64_t k = kb * kTcThreads + tid;
    const bool live = k < K;
    const uint64_t kg = (uint64_t)(f.k_off + (live ? k : K - 1));  // dead lanes shadow the last rollout, store nothing

    // the FP64 attitude state (ang, rate) stays in registers
    double ang[3] = {sa_args->state[6], sa_args->state[7], sa_args->state[8]};
    double rate[3] = {sa_args->state[9], sa_args->state[10], sa_args->state[11]};
    // attitude step t (attitude_kernel's arithmetic): LWPR input row of step t, exploration
    // normals out, state advanced to t + 1, the post-step attitude term of the stage cost
    auto attitude_step = [&](int t) {
      const float4 z = device_z(ck, kg, N, t);
      if (live && f.zout) f.zout[(int64_t)t * K + k] = z;
      double e[4];
      eps_from_z(sa_args, z, e);
      double u[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) u[c] = clip_np(__dadd_rn(splan[t & 1][c], e[c]), dp.lo[c], dp.hi[c]);
      const float4 x = make_float4(__double2float_rn(ang[0]), __double2float_rn(ang[1]), __double2float_rn(ang[2]),
                                   __double2float_rn(u[3]));
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        ang[c] = wrap_angle(__dadd_rn(ang[c], __dmul_rn(rate[c], dp.dt)));
        rate[c] = __dadd_rn(rate[c], __dmul_rn(dp.gain_dt, __dsub_rn(u[c], rate[c])));
      }
      const float ax = __double2float_rn(ang[0]), ay = __double2float_rn(ang[1]), az = __double2float_rn(ang[2]);
      roll[(kAngSlot + (t & 1)) * 128 + tid] =
          __fmul_rn(__fadd_rn(__fadd_rn(__fmul_rn(ax, ax), __fmul_rn(ay, ay)), __fmul_rn(az, az)), 0.2f);
      xs[(t & 1) * 128 + tid] = x;
      return x;
    };
    // axis ax's features of input row x into A operand `buf`
    auto features = [&](int ax, float4 x, int buf) {
      float4 xt;
      float q;
      tc_features(a.axis[ax], x, sa + buf * kTcABytes, tid, xt, q);
    };
    // (mean, std) of axis ax at step t from its moments: x~ and q recomputed from the
    // stored input row (the same operations as at staging, so the same bits)
    auto finalize = [&](int ax, int t, float dn, float nm, float m2, float lv) {
      const AxisHeader &h = a.axis[ax];
      const float4 x = xs[(t & 1) * 128 + tid];
      const float4 xt = make_float4(__fsub_rn(x.x, h.mu[0]), __fsub_rn(x.y, h.mu[1]), __fsub_rn(x.z, h.mu[2]),
                                    __fsub_rn(x.w, h.mu[3]));
      const float2 r = tc_mean_sd<VAR>(a, h, xt, shared_qrow(h, xt), dn, nm, m2, lv);
      ms[(2 * ax) * 128 + tid] = r.x;
      ms[(2 * ax + 1) * 128 + tid] = r.y;
    };
    // sub-rollouts of step t (rollout_kernel<MM, FAST>'s arithmetic); pad: the next input
    // row's thrust (0 after the last step), consumed as the unfused kernels do
    DynDraws draws[MM];  // dynamics draws carried between steps (kernels.cuh DynDraws)
    auto rollout_step = [&](int t, float pad) {
      float mn[3], sd[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        mn[c] = ms[(2 * c) * 128 + tid];
        sd[c] = ms[(2 * c + 1) * 128 + tid];
      }
      const float pen = f.penalty ? variance_term(cost.variance_penalty, make_float3(sd[0], sd[1], sd[2])) : 0.0f;
      const float angterm = fmaf(pad, 0.0f, roll[(kAngSlot + (t & 1)) * 128 + tid]);
      const float sdt = __fmul_rn(dp.dt32, (float)(t + 1));
      uint32_t crashed = __float_as_uint(roll[kCrashSlot * 128 + tid]);
      float q[MM];
#pragma unroll
      for (int m = 0; m < MM; ++m) {
        if (m >= S) break;
        float acc[3];
        if (f.spread) {
          float z[3];
          draws[m].next((kg * (uint64_t)f.M + (uint64_t)m) * (uint64_t)dyn_blocks(N), t, dkey.k0, dkey.k1, z);
          acc[0] = __fadd_rn(__fmul_rn(sd[0], z[0]), mn[0]);
          acc[1] = __fadd_rn(__fmul_rn(sd[1], z[1]), mn[1]);
          acc[2] = __fadd_rn(__fmul_rn(sd[2], z[2]), mn[2]);
        } else {
          acc[0] = mn[0]; acc[1] = mn[1]; acc[2] = mn[2];
        }
        float pos[3], vel[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          float *cs = roll + (m * 6 + c) * 128 + tid, *ccs = roll + (m * 6 + 3 + c) * 128 + tid;
          const float csn = __fadd_rn(*cs, acc[c]);
          const float ccsn = __fadd_rn(*ccs, csn);
          *cs = csn;
          *ccs = ccsn;
          vel[c] = __fadd_rn(__fmul_rn(csn, dp.dt32), v0[c]);
          pos[c] = __fadd_rn(__fadd_rn(__fmul_rn(__fsub_rn(ccsn, csn), dp.dt2_32), __fmul_rn(sdt, v0[c])), p0[c]);
        }
        bool cm = ((crashed >> m) & 1u) != 0;
        cm = cm | nav_crash_now(cost, pos[0], pos[1], pos[2]);
        crashed |= (cm ? 1u : 0u) << m;
        q[m] = nav_stage_cost<false>(cost, xobs, pos[0], pos[1], pos[2], vel[0], vel[1], vel[2], angterm, cm);
      }
      int n = S;  // pairwise halving while even, plain mean when odd (controller.py:314-319)
      while (n > 1) {
        if ((n & 1) == 0) {
#pragma unroll
          for (int i = 0; i < MM / 2; ++i)
            if (i < n / 2) q[i] = __fmul_rn(0.5f, __fadd_rn(q[2 * i], q[2 * i + 1]));
          n >>= 1;
        } else {
          float s = q[0];
#pragma unroll
          for (int i = 1; i < MM; ++i)
            if (i < n) s = __fadd_rn(s, q[i]);
          q[0] = __fdiv_rn(s, (float)n);
          n = 1;
        }
      }
      roll[kCrashSlot * 128 + tid] = __uint_as_float(crashed);
      if (live) f.qbuf[(int64_t)t * K + k] = f.penalty ? __fadd_rn(q[0], pen) : q[0];
    };

    // ---- this block: initial state, step 0's row and axis 0's features ----
    if (tid < 4) splan[0][tid] = __ldcg(f.plan + tid);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 6 * MM; ++i) roll[i * 128 + tid] = -0.0f;  // -0 + x == x: cumsum start
    roll[kCrashSlot * 128 + tid] = __uint_as_float(0u);
    {
      const float4 x0 = attitude_step(0);
      features(0, x0, buf);
    }
    float2 den = make_float2(0.f, 0.f), num = den, m2 = den, lv = den;
    float dn_p = 0.f, nm_p = 0.f, m2_p = 0.f, lv_p = 0.f;  // moments of the axis awaiting finalize
    int t = 0, ax = 0, c = 0;
    for (;;) {
      const int lc = a.chunk_pad[ax][c];
      asm volatile("fence.proxy.async.shared::cta;");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();  // A written, TMEM free
      PI2_TC_T(1);
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t idesc = umma_idesc_tf32(128, 2 * lc);
        const uint32_t sa_addr = sa_addr0 + (uint32_t)buf * kTcABytes;
        const uint64_t a_hi = umma_smem_desc(sa_addr), a_lo = umma_smem_desc(sa_addr + 4096);
        // the next item's W into the other slot first (it held this item's predecessor,
        // whose MMA completed before every warp read it): next chunk, next axis, next step
        // or the next block's first item
        int nax = ax, nc = c + 1;
        if (nc == nch_of(ax)) {
          nc = 0;
          nax = ax == 2 ? 0 : ax + 1;
        }
        const bool more = !(t == N - 1 && ax == 2 && c + 1 == nch2) || kb + gridDim.x < nblocks;
        if (more) load_w(nax, nc, (nw + 1) & 1);
        mbar_wait(wbar_addr + 8 * (nw & 1), (nw >> 1) & 1);  // this chunk's W landed
        const uint32_t wb = sw_addr + (nw & 1) * (uint32_t)(kTcWSlotFloats * 4);
        const uint64_t b_hi = umma_smem_desc(wb), b_lo = umma_smem_desc(wb + (uint32_t)(2 * lc * 8 * 4));
#if PI2_TC_PACK2
        mma_tf32(tmem, a_hi, b_hi, idesc, 0);  // A1 . B1
        mma_tf32(tmem, a_lo, b_lo, idesc, 1);  // A2 . B2
#else
        mma_tf32(tmem, a_hi, b_hi, idesc, 0);
        mma_tf32(tmem, a_hi, b_lo, idesc, 1);
        mma_tf32(tmem, a_lo, b_hi, idesc, 1);
#endif
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar_addr));
      }
      PI2_TC_T(8);
      if (c == 0) {  // in the MMA's shadow
        if (ax > 0 || t > 0) {  // finalize the previous axis
          const int pax = ax == 0 ? 2 : ax - 1, pt = ax == 0 ? t - 1 : t;
          finalize(pax, pt, dn_p, nm_p, m2_p, lv_p);
          PI2_TC_T(5);
          if (ax == 0) {
            rollout_step(t - 1, xs[(t & 1) * 128 + tid].w);  // step t - 1 integrated
            PI2_TC_T(6);
          }
        }
        if (ax == 1 && tid < 4 && t + 1 < N)  // step t + 1's plan row, read at axis 2 (after this item's barrier)
          splan[(t + 1) & 1][tid] = __ldcg(f.plan + 4 * (t + 1) + tid);
        if (ax < 2) {
          features(ax + 1, xs[(t & 1) * 128 + tid], buf ^ 1);
        } else if (t + 1 < N) {
          const float4 xn = attitude_step(t + 1);
          PI2_TC_T(7);
          features(0, xn, buf ^ 1);
        }
        PI2_TC_T(0);
      }
      mbar_wait(mbar_addr, phase);
      phase ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;");
      PI2_TC_T(2);
      tc_exp_span<VAR, true, kTcChunk>(tmem_lane, lc, lc, slv + lvb_of(ax) + c * kTcChunk, den, num, m2, lv);
      PI2_TC_T(3);
      ++nw;
      if (++c < nch_of(ax)) continue;
      // axis done: its moments wait for finalize in the next item's shadow
      dn_p = __fadd_rn(den.x, den.y);
      nm_p = __fadd_rn(num.x, num.y);
      m2_p = __fadd_rn(m2.x, m2.y);
      lv_p = __fadd_rn(lv.x, lv.y);
      den = make_float2(0.f, 0.f);
      num = den;
      m2 = den;
      lv = den;
      c = 0;
      buf ^= 1;
      if (++ax < 3) continue;
      ax = 0;
      if (++t == N) break;
    }
    // the last step: axis 2's finalize and the integration, then the suffix sums
    finalize(2, N - 1, dn_p, nm_p, m2_p, lv_p);
    rollout_step(N - 1, 0.0f);  // ang_last's pad lane
    __syncwarp();
    const uint32_t crashed = __float_as_uint(roll[kCrashSlot * 128 + tid]);
    bool crash = false;
#pragma unroll
    for (int m = 0; m < MM; ++m)
      if (m < S) crash = crash || ((crashed >> m) & 1u);
    if (live) {  // float64 suffix sum (controller.py:320-322) and ceiling (:243-246)
      const double dt = dp.dt, ceiling = sa_args->ceiling;
      double acc = 0.0;
      for (int tt = N - 1; tt >= 0; --tt) {
        const double s = __dmul_rn((double)f.qbuf[(int64_t)tt * K + k], dt);
        acc = (tt == N - 1) ? s : __dadd_rn(acc, s);
        double v = acc;
        if (!isfinite(v)) {
          v = ceiling;
          crash = true;
        }
        f.costs[(int64_t)tt * K + k] = v;
      }
      f.crash[k] = crash ? 1 : 0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTcTmemCols));
}

}  // namespace pi2
