// lwpr_tc2.cuh — tensor-core LWPR, chunk-pipelined without CTA barriers (experimental).
//
// The same numerics as lwpr_tc_kernel (3xTF32 field GEMM into TMEM, 2^x and moments
// on the CUDA cores, identical finalize), scheduled differently: the CTA's TMEM holds
// TWO chunk buffers, every (tile, chunk) item j uses buffer j & 1, and the MMA of
// item j + 2 is issued by the LAST warp to finish reading item j (a shared-memory
// counter per buffer), so no warp ever waits at a CTA barrier and the MMA of the next
// chunk runs while the current one is in its exp phase.  Tile features are written two
// tiles ahead into a double-buffered A operand.  Resident weights only.
#pragma once

#include "lwpr_tc.cuh"

namespace pi2 {

constexpr int kTc2Cols = 4 * kTcChunk;  // two buffers of (logits | y') for kTcChunk fields

// issue the 3 MMAs of item (tile buffer abuf, chunk c) into TMEM buffer b and commit to bar
__device__ __forceinline__ void tc2_issue(const LwprTcArgs &a, int ax, int c, uint32_t sa_addr, uint32_t sw_addr,
                                          uint32_t tmem, int b, uint32_t bar) {
  const int lc = a.chunk_pad[ax][c];
  const uint32_t idesc = umma_idesc_tf32(128, 2 * lc);
  const uint64_t a_hi = umma_smem_desc(sa_addr), a_lo = umma_smem_desc(sa_addr + 4096);
  const uint32_t wb = sw_addr + (uint32_t)(a.chunk_woff[ax][c] * 4);
  const uint64_t b_hi = umma_smem_desc(wb), b_lo = umma_smem_desc(wb + (uint32_t)(2 * lc * 8 * 4));
  const uint32_t d = tmem + (uint32_t)(b * 2 * kTcChunk);
  mma_tf32(d, a_hi, b_hi, idesc, 0);
  mma_tf32(d, a_hi, b_lo, idesc, 1);
  mma_tf32(d, a_lo, b_hi, idesc, 1);
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar));
}

template <bool VAR>
__global__ void __launch_bounds__(kTcThreads, kTcCtasPerSm) lwpr_tc2_kernel(const __grid_constant__ LwprTcArgs a) {
  static_assert(kTc2Cols <= 128 && (kTc2Cols & (kTc2Cols - 1)) == 0, "two chunk buffers must fit 128 columns");
  extern __shared__ __align__(128) uint8_t tsm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t full[2];
  __shared__ uint32_t done[2];
  const int ax = blockIdx.x % 3;
  const int nch = a.nchunks[ax];
  const int64_t wbeg = a.axis_off[ax], wend = ax < 2 ? a.axis_off[ax + 1] : a.w_floats;
  const int64_t nlv = (int64_t)nch * kTcChunk;
  const int64_t wfl = wend - wbeg;
  float *sw = reinterpret_cast<float *>(tsm);
  float *slv_base = sw + wfl;
  uint8_t *sa = tsm + (((wfl + nlv) * 4 + 127) / 128) * 128;  // two A operands
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (int64_t i = tid; i < wfl / 4; i += blockDim.x)
    reinterpret_cast<float4 *>(sw)[i] = __ldg(reinterpret_cast<const float4 *>(a.w + wbeg) + i);
  for (int64_t i = tid; i < nlv; i += blockDim.x) slv_base[i] = __ldg(a.w + a.lv_off[ax] + i);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)),
                 "n"(kTc2Cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const uint32_t full_addr = (uint32_t)__cvta_generic_to_shared(&full[0]);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full_addr));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full_addr + 8));
    asm volatile("fence.mbarrier_init.release.cluster;");
    done[0] = done[1] = 0;
  }
  const AxisHeader &h = a.axis[ax];
  const int64_t ntiles = (a.rows + 127) / 128, last = a.rows - 1;
  const int64_t tstride = gridDim.x / 3, tile0 = blockIdx.x / 3;
  const int64_t nt = tile0 < ntiles ? (ntiles - tile0 + tstride - 1) / tstride : 0;  // tiles of this CTA
  const int64_t nitems = nt * nch;
  pdl_wait();
  // features of this CTA's tiles 0 and 1 (A buffers 0 and 1); x of tile 2 in flight
  // centred inputs of the two tiles in flight (finalize needs them): tile i, tile i + 1
  float4 xt_c = make_float4(0.f, 0.f, 0.f, 0.f), xt_n = xt_c;
  float q_c = 0.0f, q_n = 0.0f;
  auto row_of = [&](int64_t i) { return (tile0 + i * tstride) * 128 + tid; };
  auto load_x = [&](int64_t i) {
    const int64_t r = row_of(i);
    return __ldcg(a.x + (r < last ? r : last));
  };
  if (nt > 0) tc_features(h, load_x(0), sa, tid, xt_c, q_c);
  if (nt > 1) tc_features(h, load_x(1), sa + kTcABytes, tid, xt_n, q_n);
  float4 xn = nt > 2 ? load_x(2) : make_float4(0.f, 0.f, 0.f, 0.f);
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t tmem_lane = tmem + ((uint32_t)(warp * 32) << 16);
  const uint32_t sw_addr = (uint32_t)__cvta_generic_to_shared(sw);
  const uint32_t sa_addr0 = (uint32_t)__cvta_generic_to_shared(sa);
  // item j = (tile i, chunk c), j = i * nch + c; the first two are issued up front
  if (tid == 0)
    for (int64_t j = 0; j < 2 && j < nitems; ++j)
      tc2_issue(a, ax, (int)(j % nch), sa_addr0 + (uint32_t)((j / nch) & 1) * kTcABytes, sw_addr, tmem, (int)(j & 1),
                full_addr + 8 * (uint32_t)(j & 1));

  int64_t j = 0;
  for (int64_t i = 0; i < nt; ++i) {
    float2 den = make_float2(0.f, 0.f), num = den, m2 = den, lv = den;
    for (int c = 0; c < nch; ++c, ++j) {
      const int b = (int)(j & 1);
      const int lc = a.chunk_pad[ax][c];
      mbar_wait(full_addr + 8 * b, (uint32_t)((j >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tl = tmem_lane + (uint32_t)(b * 2 * kTcChunk);
      const float *slv = slv_base + (int64_t)c * kTcChunk;
      const int nb = lc >> 3;
      auto batches = [&](auto nb_c) {  // nb_c: compile-time batch count, or 0 = runtime nb
        constexpr int NBC = decltype(nb_c)::value;
        const int n = NBC > 0 ? NBC : nb;
        if constexpr (VAR && NBC > 0 && NBC % 2 == 0) {
#pragma unroll
          for (int bb = 0; bb < NBC; bb += 2) {
            uint32_t l16[16], y16[16];
            PI2_TMEM_LD16(l16, tl + 8 * bb);
            PI2_TMEM_LD16(y16, tl + lc + 8 * bb);
            PI2_TMEM_WAIT16(l16, y16);
            PI2_TMEM_WAIT16(l16 + 8, y16 + 8);
            tc_fields8<VAR>(l16, y16, slv + 8 * bb, den, num, m2, lv);
            tc_fields8<VAR, true>(l16 + 8, y16 + 8, slv + 8 * bb + 8, den, num, m2, lv);
          }
          return;
        }
#pragma unroll
        for (int bb = 0; bb < (NBC > 0 ? NBC : 1 << 30); bb += 2) {
          if (NBC == 0 && bb >= n) break;
          uint32_t la[8], ya[8], lb[8], yb[8];
          PI2_TMEM_LD8(la, tl + 8 * bb);
          PI2_TMEM_LD8(ya, tl + lc + 8 * bb);
          if (bb + 1 < n) {
            PI2_TMEM_LD8(lb, tl + 8 * bb + 8);
            PI2_TMEM_LD8(yb, tl + lc + 8 * bb + 8);
          }
          PI2_TMEM_WAIT16(la, ya);
          PI2_TMEM_WAIT16(lb, yb);
          tc_fields8<VAR>(la, ya, slv + 8 * bb, den, num, m2, lv);
          if (bb + 1 < n) tc_fields8<VAR, true>(lb, yb, slv + 8 * bb + 8, den, num, m2, lv);
        }
      };
      if (lc == kTcChunk) batches(std::integral_constant<int, kTcChunk / 8>{});
      else batches(std::integral_constant<int, 0>{});
      asm volatile("tcgen05.fence::before_thread_sync;");
      // the tile's last chunk: its A buffer is free again (every MMA of the tile has been
      // consumed), so the features of tile i + 2 go there now -- before this warp reports
      // the chunk done, which orders them before the MMA that reads them
      const bool tile_end = c == nch - 1;
      if (tile_end && i + 2 < nt) {
        float4 xt2;
        float q2;
        tc_features(h, xn, sa + (i & 1) * kTcABytes, tid, xt2, q2);
        asm volatile("fence.proxy.async.shared::cta;");
        // finalize needs tile i's centred inputs: keep them until then
        const float4 xti = xt_c;
        const float qi = q_c;
        xt_c = xt_n;
        q_c = q_n;
        xt_n = xt2;
        q_n = q2;
        if (i + 3 < nt) xn = load_x(i + 3);
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          const uint32_t old = atomicAdd(&done[b], 1u);
          if (old == 3) {  // the last warp out of item j: buffer b is free, issue item j + 2
            done[b] = 0;
            __threadfence_block();
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (j + 2 < nitems)
              tc2_issue(a, ax, (int)((j + 2) % nch), sa_addr0 + (uint32_t)(((j + 2) / nch) & 1) * kTcABytes, sw_addr,
                        tmem, b, full_addr + 8 * (uint32_t)b);
          }
        }
        __syncwarp();
        tc_finalize<VAR>(a, h, ax, row_of(i), xti, qi, __fadd_rn(den.x, den.y), __fadd_rn(num.x, num.y),
                         __fadd_rn(m2.x, m2.y), __fadd_rn(lv.x, lv.y));
        continue;
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        const uint32_t old = atomicAdd(&done[b], 1u);
        if (old == 3) {
          done[b] = 0;
          __threadfence_block();
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (j + 2 < nitems)
            tc2_issue(a, ax, (int)((j + 2) % nch), sa_addr0 + (uint32_t)(((j + 2) / nch) & 1) * kTcABytes, sw_addr, tmem,
                      b, full_addr + 8 * (uint32_t)b);
        }
      }
      __syncwarp();
      if (tile_end) {
        tc_finalize<VAR>(a, h, ax, row_of(i), xt_c, q_c, __fadd_rn(den.x, den.y), __fadd_rn(num.x, num.y),
                         __fadd_rn(m2.x, m2.y), __fadd_rn(lv.x, lv.y));
        xt_c = xt_n;
        q_c = q_n;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTc2Cols));
}

}  // namespace pi2
