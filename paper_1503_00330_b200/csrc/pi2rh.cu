// pi2rh.cu — C ABI of the B200 PI²-RH engine (declared in include/pi2rh.h).
//
// One context = one RolloutEngine (controller.py:161-247) bound to one GPU:
// it owns the HBM workspaces of its K x N batch, the staged model / cost
// plugins, pinned staging memory and a cached CUDA graph of a whole control
// step.  Host compute here is limited to parameter folding (FrozenLwpr's
// constructor, lwpr.py:339-358) and stream-key hashing (rng.py:33-44).

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fold.h"
#include "kernels.cuh"
#include "lwpr_tc.cuh"
#include "fused.cuh"

namespace {
// NVTX range (header-only NVTX3: a no-op unless a tool such as ncu --nvtx or nsys is
// attached): every C-ABI entry point and every stage launch is a named range, so a
// profiler can filter by them (ncu --nvtx --nvtx-include "lwpr/").
#ifndef PI2_NVTX
#define PI2_NVTX 1
#endif
struct Range {
  explicit Range(const char *name) {
    if (PI2_NVTX) nvtxRangePushA(name);
  }
  ~Range() {
    if (PI2_NVTX) nvtxRangePop();
  }
  Range(const Range &) = delete;
  Range &operator=(const Range &) = delete;
};
}  // namespace

using namespace pi2;

struct pi2_ctx {
  int device = 0;
  pi2_dims dims{};
  int64_t K = 0;
  int N = 0, M = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t staged = nullptr;  // last H2D from the pinned staging block
  std::string err;

  // plugins
  bool have_dyn = false;
  pi2_dynamics dyn{};
  DynParams dp{};
  bool have_cost = false;
  pi2_cost cost{};
  int model = PI2_MODEL_NONE;
  double model_param = 0.0;
  AxisRaw axes[3];
  bool params_dirty = true;
  int layout = kLayDiag;
  AxisHeader hdr[3]{};
  float *d_params = nullptr;
  size_t params_cap = 0;
  // tensor-core LWPR operands (shared-metric models, lwpr_tc.cuh)
  bool tc_ok = false;
  bool tc_enabled = true;  // PI2_LWPR_TC=0 forces the CUDA-core kernel
  int tc_mode = 1;         // see tc_wanted
  bool tc_stream = false;  // W streamed per chunk (large L)
  bool pdl = true;         // programmatic dependent launch along the step's kernels (PI2_PDL=0: off)
  bool uva = false;        // pinned host memory is device-accessible (unified addressing)
  bool io_pull = true;     // I/O graph: inputs pulled by io_pull_kernel (PI2_IO_PULL=0: copy node)
  int partials_split = 1;  // partials_split_kernel: 0 never, 1 when few (chunk, t) warps, 2 always
  int fused = 0;
  int smem_horizon = kSmemHorizon;  // longer horizons: rollout stage costs in global scratch, no warp-per-rollout
                                    // kernels (PI2_SMEM_HORIZON lowers it, for tests)           // device-noise iterations through fused_step_kernel when eligible (PI2_FUSED=1; slower, see DESIGN)
  int64_t wide_max_k = kWideMaxK;  // attitude/rollout use a warp per rollout up to this K (PI2_WIDE_MAX_K)
  int64_t tc_bulk_max_tiles = kTcBulkMaxTiles;  // WBULK LWPR up to this many tiles per CTA (PI2_TC_BULK_MAX_TILES)
  LwprTcArgs tc{};
  float *d_tc = nullptr;
  size_t tc_cap = 0;
  int tc_smem = 0;

  // device workspaces (sized by dims); StepArgs and the plan share one block (d_io)
  // so that one copy stages both
  uint8_t *d_io = nullptr;
  StepArgs *d_args = nullptr;
  double *d_plan = nullptr, *d_plan2 = nullptr;
  float4 *d_xin = nullptr, *d_ang_last = nullptr, *d_lw = nullptr;  // d_lw: LWPR mean planes, std planes
  double *d_costs = nullptr;
  uint8_t *d_crash = nullptr;
  double *d_partials = nullptr, *d_root = nullptr;
  float4 *d_z = nullptr;  // device-noise exploration normals z(k, t) at [t * K + k] (attitude -> partials)
  bool store_z = true;    // PI2_STORE_Z=0: the partials kernel regenerates z instead (experiments)
  bool bounds_nonan = false;  // no control bound is NaN: the attitude kernel's cheaper clip (pi2_set_dynamics)
  int64_t n_chunks = 0;
  // lazily grown scratch
  double *d_noise = nullptr;
  size_t noise_cap = 0;
  float *d_dynbuf = nullptr;
  size_t dyn_cap = 0;
  float *d_xobs = nullptr;  // navigation-cost obstacles past PI2_MAX_OBSTACLES (StepArgs::extra_obstacles)
  size_t xobs_cap = 0;
  std::vector<float> h_xobs;  // their host copy (re-staged only on change)
  float *d_qs = nullptr;  // long-horizon stage-cost scratch (RollArgs::qs)
  size_t qs_cap = 0;
  void *d_scratch = nullptr;
  size_t scratch_cap = 0;

  // pinned staging, same layout as d_io
  uint8_t *h_io = nullptr;
  StepArgs *h_args = nullptr;
  double *h_plan = nullptr;  // N x 4

  // graph cache: `graph` = the iterations (pi2_iterate_device); `graph_io` = H2D of
  // StepArgs + plan, the iterations, D2H of the plan (pi2_optimize)
  cudaGraphExec_t graph = nullptr, graph_io = nullptr;
  int graph_iters = -1, graph_io_iters = -1;
  double graph_neg_inv = 0.0, graph_io_neg_inv = 0.0;

  int smem_optin = 0;
};

namespace {

thread_local std::string g_noctx_err;

int fail(pi2_ctx *ctx, int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf; else g_noctx_err = buf;
  return code;
}

#define CU(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? PI2_ERR_OOM : PI2_ERR_CUDA,          \
                  "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__);       \
  } while (0)

#define TRY(expr)            \
  do {                       \
    int rc_ = (expr);        \
    if (rc_ != PI2_OK) return rc_; \
  } while (0)

cudaStream_t pick(pi2_ctx *ctx, void *s) { return s ? (cudaStream_t)s : ctx->stream; }

int ensure(pi2_ctx *ctx, void **p, size_t *cap, size_t bytes) {
  if (*cap >= bytes && *p) return PI2_OK;
  if (*p) CU(cudaFree(*p));
  *p = nullptr;
  *cap = 0;
  CU(cudaMalloc(p, std::max<size_t>(bytes, 256)));
  *cap = bytes;
  return PI2_OK;
}

int bind(pi2_ctx *ctx) {
  CU(cudaSetDevice(ctx->device));
  return PI2_OK;
}

void invalidate_graph(pi2_ctx *ctx) {
  if (ctx->graph) cudaGraphExecDestroy(ctx->graph);
  if (ctx->graph_io) cudaGraphExecDestroy(ctx->graph_io);
  ctx->graph = ctx->graph_io = nullptr;
  ctx->graph_iters = ctx->graph_io_iters = -1;
}

// StepArgs is padded to this in the d_io / h_io blocks (the plan follows)
constexpr size_t kIoArgsBytes = (sizeof(StepArgs) + 255) / 256 * 256;

int ensure_params(pi2_ctx *ctx) {
  if (!ctx->params_dirty) return PI2_OK;
  const int layout = choose_layout(ctx->axes, 3);
  std::vector<float> rec;
  for (int ax = 0; ax < 3; ++ax) {
    if (ctx->axes[ax].L > 0) fold_axis(ctx->axes[ax], layout, rec, ctx->hdr[ax]);
    else ctx->hdr[ax] = AxisHeader{};
  }
  if (!rec.empty()) {
    TRY(ensure(ctx, (void **)&ctx->d_params, &ctx->params_cap, rec.size() * sizeof(float)));
    CU(cudaMemcpy(ctx->d_params, rec.data(), rec.size() * sizeof(float), cudaMemcpyHostToDevice));
  }
  ctx->layout = layout;
  // tensor-core operands when every axis shares its metric and has 4 inputs
  ctx->tc_ok = false;
  if (ctx->tc_enabled && ctx->axes[0].L > 0 && ctx->axes[1].L > 0 && ctx->axes[2].L > 0) {
    std::vector<float> blob;
    LwprTcArgs ta{};
    if (build_tc_weights(ctx->axes, blob, ta)) {
      TRY(ensure(ctx, (void **)&ctx->d_tc, &ctx->tc_cap, blob.size() * sizeof(float)));
      CU(cudaMemcpy(ctx->d_tc, blob.data(), blob.size() * sizeof(float), cudaMemcpyHostToDevice));
      ta.w = ctx->d_tc;
      int64_t wmax = 0, lvmax = 0;
      for (int i = 0; i < 3; ++i) {
        const int64_t we = i < 2 ? ta.axis_off[i + 1] : ta.w_floats;
        wmax = std::max<int64_t>(wmax, we - ta.axis_off[i] + (int64_t)ta.nchunks[i] * kTcChunk);
        lvmax = std::max<int64_t>(lvmax, (int64_t)ta.nchunks[i] * kTcChunk);
      }
      // W resident in shared memory when it fits next to 3 other CTAs, else streamed
      ctx->tc_stream = false;
      ctx->tc_smem = tc_smem_bytes(wmax, (const void *)lwpr_tc_kernel<true, false>);
      if (ctx->tc_smem < 0 || getenv("PI2_LWPR_TC_STREAM")) {
        ctx->tc_stream = true;
        ctx->tc_smem = tc_smem_bytes(2 * kTcWSlotFloats + lvmax, (const void *)lwpr_tc_kernel<true, true>);
      }
      ctx->tc = ta;
      ctx->tc_ok = ctx->tc_smem > 0 && ctx->tc_smem <= ctx->smem_optin;
    }
  }
  ctx->params_dirty = false;
  return PI2_OK;
}

// ---- kernel attribute setup -------------------------------------------------
template <typename F>
int set_smem(pi2_ctx *ctx, F *fn, int bytes) {
  CU(cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  return PI2_OK;
}

// a kernel of the step's chain, launched with programmatic stream serialization
// (PDL, see pdl_wait in kernels.cuh) unless PI2_PDL=0 or `pdl` is false.  Only
// for kernels whose stream predecessor is a kernel of the chain: griddepcontrol.wait
// waits for the previous GRID, not for a copy or an event wait before it.
template <typename... KArgs, typename... Args>
int launch_pdl_if(bool pdl, pi2_ctx *ctx, void (*fn)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                  Args &&...args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = (pdl && ctx->pdl) ? 1 : 0;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  CU(cudaLaunchKernelEx(&cfg, fn, std::forward<Args>(args)...));
  return PI2_OK;
}
template <typename... KArgs, typename... Args>
int launch_pdl(pi2_ctx *ctx, void (*fn)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
               Args &&...args) {
  return launch_pdl_if(true, ctx, fn, grid, block, smem, st, std::forward<Args>(args)...);
}

int lwpr_smem_limit(pi2_ctx *ctx) { return std::min(ctx->smem_optin, 64 * 1024); }

template <int LAY, bool VAR, int R>
int launch_lwpr_t(pi2_ctx *ctx, LwprArgs a, int smem, cudaStream_t st, bool pdl) {
  auto *fn = lwpr_kernel<LAY, VAR, R>;
  TRY(set_smem(ctx, fn, smem));
  const int64_t per_block = (int64_t)kLwprBlock * R;
  const int64_t grid = (a.rows + per_block - 1) / per_block;
  TRY(launch_pdl_if(pdl, ctx, fn, dim3((unsigned)grid), dim3(kLwprBlock), smem, st, a));
  CU(cudaGetLastError());
  return PI2_OK;
}

// PI2_LWPR_TC: unset / 1 = tensor cores for every eligible launch, 2 = variance path
// only, 0 = never
bool tc_wanted(const pi2_ctx *ctx, bool var) { return ctx->tc_mode == 1 || (ctx->tc_mode == 2 && var); }

template <bool VAR>
int launch_lwpr_tc(pi2_ctx *ctx, int64_t rows, const float4 *x, float *mean_out, float *sd_out, cudaStream_t st,
                   bool pdl) {
  LwprTcArgs a = ctx->tc;
  for (int i = 0; i < 3; ++i) a.axis[i] = ctx->hdr[i];
  a.params = ctx->d_params;
  a.rows = rows;
  a.x = x;
  a.mean_out = mean_out;
  a.sd_out = sd_out;
  a.plane = rows;
  a.sqrt_out = 1;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  a.sms = sms;
  const int64_t tiles = (rows + 127) / 128;
  const int64_t per_axis = std::min<int64_t>((int64_t)kTcCtasPerSm * sms / 3, tiles);
  const int64_t grid = per_axis * 3;  // CTA i -> axis i % 3
  // few tiles per CTA: resident weights by one bulk copy (see WBULK)
  const bool bulk = (tiles + per_axis - 1) / per_axis <= ctx->tc_bulk_max_tiles;
  // resident weights, many tiles: the instantiation whose remainder chunk loop is unrolled too
  using Fn = void (*)(LwprTcArgs);
  static constexpr Fn kResident[8] = {lwpr_tc_kernel<VAR, false, false, 0>, lwpr_tc_kernel<VAR, false, false, 1>,
                                      lwpr_tc_kernel<VAR, false, false, 2>, lwpr_tc_kernel<VAR, false, false, 3>,
                                      lwpr_tc_kernel<VAR, false, false, 4>, lwpr_tc_kernel<VAR, false, false, 5>,
                                      lwpr_tc_kernel<VAR, false, false, 6>, lwpr_tc_kernel<VAR, false, false, 7>};
  auto *fn = ctx->tc_stream ? lwpr_tc_kernel<VAR, true>
                            : (bulk ? lwpr_tc_kernel<VAR, false, true> : kResident[tc_remainder_batches(ctx->tc)]);
  TRY(set_smem(ctx, fn, ctx->tc_smem));
  TRY(launch_pdl_if(pdl, ctx, fn, dim3((unsigned)grid), dim3(kTcThreads), ctx->tc_smem, st, a));
  CU(cudaGetLastError());
  return PI2_OK;
}

// outputs: element (row, axis) at out[row * row_stride + (axis - a_begin) * axis_stride]
// pdl: the stream predecessor is the attitude kernel (rollout chain)
int launch_lwpr(pi2_ctx *ctx, int a_begin, int a_end, int64_t rows, const float4 *x, float *mean_out,
                float *sd_out, int row_stride, int64_t axis_stride, int sqrt_out, cudaStream_t st, bool pdl = false) {
  Range range_("lwpr");
  TRY(ensure_params(ctx));
  // all three axes into planes (the rollout path): tensor cores when eligible
  // (shared metric, each axis' weights fit at full residency; PI2_LWPR_TC=0 disables)
  if (ctx->tc_ok && tc_wanted(ctx, sd_out != nullptr) && a_begin == 0 && a_end == 3 && row_stride == 1 &&
      axis_stride == rows && sqrt_out)
    return sd_out ? launch_lwpr_tc<true>(ctx, rows, x, mean_out, sd_out, st, pdl)
                  : launch_lwpr_tc<false>(ctx, rows, x, mean_out, nullptr, st, pdl);
  LwprArgs a{};
  a.params = ctx->d_params;
  for (int i = 0; i < 3; ++i) a.axis[i] = ctx->hdr[i];
  a.a_begin = a_begin;
  a.a_end = a_end;
  a.layout = ctx->layout;
  const int RS = record_floats(ctx->layout);
  int64_t fields = 0, maxL = 0;
  for (int ax = a_begin; ax < a_end; ++ax) {
    fields += ctx->hdr[ax].num_fields;
    maxL = std::max<int64_t>(maxL, ctx->hdr[ax].num_fields);
  }
  const int limit = lwpr_smem_limit(ctx);
  const int64_t need = fields * RS * (int64_t)sizeof(float);
  int smem;
  if (need <= limit) {
    a.resident = 1;
    a.tile = 0;
    smem = (int)need;
  } else {
    a.resident = 0;
    a.tile = (int)std::min<int64_t>(maxL, limit / (RS * (int64_t)sizeof(float)));
    smem = a.tile * RS * (int)sizeof(float);
  }
  a.rows = rows;
  a.x = x;
  a.mean_out = mean_out;
  a.sd_out = sd_out;
  a.row_stride = row_stride;
  a.axis_stride = axis_stride;
  a.sqrt_out = sqrt_out;
  const bool var = sd_out != nullptr;
  const bool small = rows < (int64_t)2 * 148 * kLwprBlock * kLwprRows;
#define PI2_LWPR_CASE(LAY)                                                                          \
  if (ctx->layout == LAY) {                                                                         \
    if (var) return small ? launch_lwpr_t<LAY, true, 2>(ctx, a, smem, st, pdl)                           \
                          : launch_lwpr_t<LAY, true, kLwprRows>(ctx, a, smem, st, pdl);                  \
    return small ? launch_lwpr_t<LAY, false, 2>(ctx, a, smem, st, pdl)                                   \
                 : launch_lwpr_t<LAY, false, kLwprRows>(ctx, a, smem, st, pdl);                          \
  }
  PI2_LWPR_CASE(kLayShared)
  PI2_LWPR_CASE(kLayDiag)
  PI2_LWPR_CASE(kLayFull)
#undef PI2_LWPR_CASE
  return fail(ctx, PI2_ERR_STATE, "unknown LWPR layout %d", ctx->layout);
}

bool spread(const pi2_ctx *ctx) {
  const bool prob = ctx->model == PI2_MODEL_HYBRID_LWPR || ctx->model == PI2_MODEL_TWO_POINT;
  return prob && ctx->M > 1;
}

// the opt-in uncertainty penalty (hybrid model, navigation cost): needs the LWPR std planes
bool penalty(const pi2_ctx *ctx) {
  return ctx->model == PI2_MODEL_HYBRID_LWPR && ctx->cost.kind == PI2_COST_NAVIGATION && ctx->cost.variance_penalty > 0;
}

template <int MM, bool FAST>
int launch_rollout_t(pi2_ctx *ctx, const RollArgs &a, cudaStream_t st) {
  const bool r32 = FAST && 3 * a.lw_plane < (int64_t(1) << 32) && a.K * a.N * 4 < (int64_t(1) << 32);
  auto *fn = r32 ? rollout_kernel<MM, FAST, FAST> : rollout_kernel<MM, FAST, false>;
  const int smem = a.qs ? 0 : a.N * kRolloutBlock * (int)sizeof(float);
  TRY(set_smem(ctx, fn, smem));
  const int64_t grid = (a.K + kRolloutBlock - 1) / kRolloutBlock;
  TRY(launch_pdl(ctx, fn, dim3((unsigned)grid), dim3(kRolloutBlock), smem, st, a));
  CU(cudaGetLastError());
  return PI2_OK;
}

template <int G, bool FAST>
int launch_group_t(pi2_ctx *ctx, const RollArgs &a, cudaStream_t st) {
  // 32-bit row offsets when every plane element index fits (3 planes x K x N < 2^32)
  const bool r32 = FAST && 3 * a.lw_plane < (int64_t(1) << 32) && a.K * a.N * 4 < (int64_t(1) << 32);
  auto *fn = r32 ? rollout_group_kernel<G, FAST, FAST> : rollout_group_kernel<G, FAST, false>;
  constexpr int RPB = kRolloutBlock / (G > 32 ? 32 : G);
  const int smem = a.qs ? 0 : a.N * RPB * (int)sizeof(float);
  TRY(set_smem(ctx, fn, smem));
  const int64_t grid = (a.K + RPB - 1) / RPB;
  TRY(launch_pdl(ctx, fn, dim3((unsigned)grid), dim3(kRolloutBlock), smem, st, a));
  CU(cudaGetLastError());
  return PI2_OK;
}

template <int G>
int launch_group_g(pi2_ctx *ctx, const RollArgs &a, bool fast, cudaStream_t st) {
  return fast ? launch_group_t<G, true>(ctx, a, st) : launch_group_t<G, false>(ctx, a, st);
}

// the whole obstacle list sits in pi2_cost (no StepArgs::extra_obstacles): the FAST
// rollout kernels and the fused kernel, which have no loop over the HBM tail, may run
inline bool struct_obstacles(const pi2_ctx *ctx) { return ctx->cost.n_obstacles <= PI2_MAX_OBSTACLES; }

int launch_rollout(pi2_ctx *ctx, const RollArgs &a, cudaStream_t st) {
  const int S = a.spread ? a.M : 1;
  const bool nav = ctx->cost.kind == PI2_COST_NAVIGATION && struct_obstacles(ctx);  // FAST-eligible
  const bool hybrid = a.model == PI2_MODEL_HYBRID_LWPR;
  // sub-rollouts on lanes (any model but the analytic one, which is never spread);
  // 33..256 on 32 lanes with S / 32 rounded up to a power of two each (S <= PI2_MAX_SUB_ROLLOUTS)
  if (S > 1) {
    const bool fast = hybrid && nav && a.device_dyn;
    if (S <= 2) return launch_group_g<2>(ctx, a, fast, st);
    if (S <= 4) return launch_group_g<4>(ctx, a, fast, st);
    if (S <= 8) return launch_group_g<8>(ctx, a, fast, st);
    if (S <= 16) return launch_group_g<16>(ctx, a, fast, st);
    if (S <= 32) return launch_group_g<32>(ctx, a, fast, st);
    if (S <= 64) return launch_group_g<64>(ctx, a, fast, st);
    if (S <= 128) return launch_group_g<128>(ctx, a, fast, st);
    return launch_group_g<256>(ctx, a, fast, st);
  }
  if (S == 1 && a.K <= ctx->wide_max_k && a.N <= ctx->smem_horizon) {  // latency regime: a warp per rollout
    const unsigned grid = (unsigned)((a.K + kWideWarps - 1) / kWideWarps);
    const int smem = kWideWarps * 11 * a.N * (int)sizeof(float);
    if (hybrid && nav) {
      TRY(set_smem(ctx, rollout_wide_kernel<true>, smem));
      TRY(launch_pdl(ctx, rollout_wide_kernel<true>, dim3(grid), dim3(32 * kWideWarps), smem, st, a));
    } else {
      TRY(set_smem(ctx, rollout_wide_kernel<false>, smem));
      TRY(launch_pdl(ctx, rollout_wide_kernel<false>, dim3(grid), dim3(32 * kWideWarps), smem, st, a));
    }
    CU(cudaGetLastError());
    return PI2_OK;
  }
  return (hybrid && nav) ? launch_rollout_t<1, true>(ctx, a, st) : launch_rollout_t<1, false>(ctx, a, st);
}

int check_ready(pi2_ctx *ctx) {
  if (!ctx) return fail(nullptr, PI2_ERR_INVALID, "null context");
  if (!ctx->have_dyn) return fail(ctx, PI2_ERR_STATE, "dynamics not set (pi2_set_dynamics)");
  if (!ctx->have_cost) return fail(ctx, PI2_ERR_STATE, "cost plugin not set (pi2_set_cost)");
  if (ctx->model == PI2_MODEL_NONE) return fail(ctx, PI2_ERR_STATE, "model plugin not selected");
  if (ctx->cost.kind == PI2_COST_NAVIGATION && ctx->cost.variance_penalty > 0 && ctx->model != PI2_MODEL_HYBRID_LWPR)
    return fail(ctx, PI2_ERR_UNSUPPORTED, "variance_penalty needs a probabilistic (hybrid LWPR) model");
  return PI2_OK;
}

// Fill the pinned StepArgs and queue its H2D copy (waits for the previous one).
// host side of stage_args: state, cost, keys into the pinned StepArgs (caller has
// waited for ctx->staged)
void fill_args(pi2_ctx *ctx, const double *state, const pi2_optimize_args *opt, double ceiling) {
  StepArgs &h = *ctx->h_args;
  if (state) std::memcpy(h.state, state, sizeof h.state);
  h.cost = ctx->cost;
  h.extra_obstacles = ctx->cost.n_obstacles > PI2_MAX_OBSTACLES ? ctx->d_xobs : nullptr;
  h.ceiling = ceiling;
  if (opt) {
    h.neg_inv_temp = -1.0 / opt->temperature;
    h.ceiling = opt->cost_ceiling;
    for (int c = 0; c < 4; ++c) h.std[c] = opt->exploration_std[c];
    h.key_prefix[0] = key_prefix(opt->seed, PI2_STREAM_CONTROL, opt->cycle);
    h.key_prefix[1] = key_prefix(opt->seed, PI2_STREAM_DYNAMICS, opt->cycle);
  }
}

int stage_args(pi2_ctx *ctx, const double *state, const pi2_optimize_args *opt, double ceiling,
               cudaStream_t st) {
  CU(cudaEventSynchronize(ctx->staged));
  fill_args(ctx, state, opt, ceiling);
  CU(cudaMemcpyAsync(ctx->d_args, ctx->h_args, sizeof(StepArgs), cudaMemcpyHostToDevice, st));
  CU(cudaEventRecord(ctx->staged, st));
  return PI2_OK;
}

int stage_plan(pi2_ctx *ctx, const double *plan, cudaStream_t st) {
  CU(cudaEventSynchronize(ctx->staged));
  std::memcpy(ctx->h_plan, plan, sizeof(double) * 4 * ctx->N);
  CU(cudaMemcpyAsync(ctx->d_plan, ctx->h_plan, sizeof(double) * 4 * ctx->N, cudaMemcpyHostToDevice, st));
  CU(cudaEventRecord(ctx->staged, st));
  return PI2_OK;
}

// The fused kernel (fused.cuh) runs a device-noise iteration's rollouts when the model
// is the hybrid LWPR on the tensor cores (shared metric, <= kFusedMaxChunks chunks per
// axis), the cost is the navigation cost, K is past the latency regime and the
// sub-rollouts fit (S <= kFusedMaxM); its shared memory must leave room for
// kTcCtasPerSm CTAs.  Returns the sub-rollout template (1, 2, 4) or 0.
int fused_mm(pi2_ctx *ctx) {
  if (!ctx->fused || ctx->model != PI2_MODEL_HYBRID_LWPR || ctx->cost.kind != PI2_COST_NAVIGATION ||
      !struct_obstacles(ctx))
    return 0;
  if (ensure_params(ctx) != PI2_OK || !ctx->tc_ok || ctx->K <= ctx->wide_max_k) return 0;
  const bool var = spread(ctx) || penalty(ctx);
  if (!tc_wanted(ctx, var)) return 0;
  for (int i = 0; i < 3; ++i)
    if (ctx->tc.nchunks[i] > kFusedMaxChunks) return 0;
  const int S = spread(ctx) ? ctx->M : 1;
  const int mm = S <= 1 ? 1 : (S <= 2 ? 2 : (S <= 4 ? 4 : 0));
  if (!mm) return 0;
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, (const void *)fused_step_kernel<true, 4>);  // static shared memory: same for all
  const int cap = 228 * 1024 / kTcCtasPerSm - 1024 - (int)fa.sharedSizeBytes - 256;
  return fused_smem_bytes(ctx->tc.nchunks, mm) <= cap ? mm : 0;
}

template <bool VAR, int MM>
int launch_fused_t(pi2_ctx *ctx, const FusedArgs &f, cudaStream_t st, bool pdl) {
  auto *fn = fused_step_kernel<VAR, MM>;
  const int smem = fused_smem_bytes(f.tc.nchunks, MM);
  TRY(set_smem(ctx, fn, smem));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  const int64_t blocks = (f.K + kTcThreads - 1) / kTcThreads;
  const int64_t grid = std::min<int64_t>((int64_t)kTcCtasPerSm * sms, blocks);
  TRY(launch_pdl_if(pdl, ctx, fn, dim3((unsigned)grid), dim3(kTcThreads), smem, st, f));
  CU(cudaGetLastError());
  return PI2_OK;
}

int launch_fused(pi2_ctx *ctx, int mm, int iteration, double *costs, uint8_t *crash, cudaStream_t st, bool pdl) {
  FusedArgs f{};
  f.tc = ctx->tc;
  f.tc.params = ctx->d_params;
  for (int i = 0; i < 3; ++i) f.tc.axis[i] = ctx->hdr[i];
  f.tc.rows = ctx->K * ctx->N;
  f.tc.sqrt_out = 1;
  f.sa = ctx->d_args;
  f.plan = ctx->d_plan;
  f.iteration = iteration;
  f.K = ctx->K;
  f.k_off = ctx->dims.rollout_offset;
  f.N = ctx->N;
  f.M = ctx->M;
  f.spread = spread(ctx) ? 1 : 0;
  f.penalty = penalty(ctx) ? 1 : 0;
  f.dp = ctx->dp;
  f.zout = ctx->d_z;
  f.qbuf = reinterpret_cast<float *>(ctx->d_lw);  // the LWPR planes are not used on this path
  f.costs = costs;
  f.crash = crash;
  const bool var = f.spread || f.penalty;
  if (var) {
    if (mm == 1) return launch_fused_t<true, 1>(ctx, f, st, pdl);
    if (mm == 2) return launch_fused_t<true, 2>(ctx, f, st, pdl);
    return launch_fused_t<true, 4>(ctx, f, st, pdl);
  }
  return launch_fused_t<false, 1>(ctx, f, st, pdl);
}

// rollouts of one iteration: attitude -> LWPR -> rollout/cost
// att_pdl: the attitude kernel may be a programmatic dependent launch (its stream
// predecessor is a kernel whose outputs it reads only after pdl_wait)
int launch_rollouts(pi2_ctx *ctx, int iteration, const double *noise_dev, const float *dyn_dev,
                    double *costs, uint8_t *crash, cudaStream_t st, cudaEvent_t *ev = nullptr,
                    bool att_pdl = false) {
  Range range_("rollouts");
  const int64_t K = ctx->K;
  const int N = ctx->N;
  if (!noise_dev && !dyn_dev) {  // device noise: the fused kernel when eligible
    const int mm = fused_mm(ctx);
    if (mm) {
      if (ev) {  // profiling: the attitude and LWPR stages are empty, the whole kernel is "rollout"
        CU(cudaEventRecord(ev[1], st));
        CU(cudaEventRecord(ev[2], st));
      }
      return launch_fused(ctx, mm, iteration, costs, crash, st, att_pdl);
    }
  }
  const unsigned grid = (unsigned)((K + kRolloutBlock - 1) / kRolloutBlock);
  const int psmem = N <= kMaxHorizon ? 4 * N * (int)sizeof(double) : 0;  // plan rows staged up to kMaxHorizon
  if (K <= ctx->wide_max_k && N <= ctx->smem_horizon) {  // latency regime: a warp per rollout
    const unsigned wgrid = (unsigned)((K + kWideWarps - 1) / kWideWarps);
    const int wsmem = psmem + kWideWarps * 4 * N * (int)sizeof(double) + kWideWarps * (N + 1) * (int)sizeof(float4);
    if (noise_dev) {
      TRY(set_smem(ctx, attitude_wide_kernel<false>, wsmem));
      TRY(launch_pdl_if(att_pdl, ctx, attitude_wide_kernel<false>, dim3(wgrid), dim3(32 * kWideWarps), wsmem, st, ctx->d_args,
                     ctx->d_plan, noise_dev, iteration, K, ctx->dims.rollout_offset, N, ctx->dp, ctx->d_xin,
                     ctx->d_ang_last, nullptr));
    } else {
      TRY(set_smem(ctx, attitude_wide_kernel<true>, wsmem));
      TRY(launch_pdl_if(att_pdl, ctx, attitude_wide_kernel<true>, dim3(wgrid), dim3(32 * kWideWarps), wsmem, st, ctx->d_args,
                     ctx->d_plan, nullptr, iteration, K, ctx->dims.rollout_offset, N, ctx->dp, ctx->d_xin,
                     ctx->d_ang_last, ctx->store_z ? ctx->d_z : nullptr));
    }
  } else if (noise_dev) {
    auto *fn = ctx->bounds_nonan ? attitude_kernel<false, true> : attitude_kernel<false, false>;
    TRY(set_smem(ctx, fn, psmem));
    TRY(launch_pdl_if(att_pdl, ctx, fn, dim3(grid), dim3(kRolloutBlock), psmem, st, ctx->d_args, ctx->d_plan,
                   noise_dev, iteration, K, ctx->dims.rollout_offset, N, ctx->dp, ctx->d_xin, ctx->d_ang_last,
                   nullptr));
  } else {
    auto *fn = ctx->bounds_nonan ? attitude_kernel<true, true> : attitude_kernel<true, false>;
    TRY(set_smem(ctx, fn, psmem));
    TRY(launch_pdl_if(att_pdl, ctx, fn, dim3(grid), dim3(kRolloutBlock), psmem, st, ctx->d_args, ctx->d_plan,
                   nullptr, iteration, K, ctx->dims.rollout_offset, N, ctx->dp, ctx->d_xin, ctx->d_ang_last, ctx->store_z ? ctx->d_z : nullptr));
  }
  CU(cudaGetLastError());
  if (ev) CU(cudaEventRecord(ev[1], st));
  const bool sp = spread(ctx), pen = penalty(ctx);
  // LWPR outputs as planes: mean x|y|z then std x|y|z, K*N floats each
  float *lw_mean = reinterpret_cast<float *>(ctx->d_lw), *lw_std = lw_mean + 3 * K * N;
  if (ctx->model == PI2_MODEL_HYBRID_LWPR)
    TRY(launch_lwpr(ctx, 0, 3, K * N, ctx->d_xin, lw_mean, (sp || pen) ? lw_std : nullptr, 1, K * N, 1, st, true));
  if (ev) CU(cudaEventRecord(ev[2], st));
  RollArgs a{};
  a.sa = ctx->d_args;
  a.iteration = iteration;
  a.K = K;
  a.k_off = ctx->dims.rollout_offset;
  a.N = N;
  a.M = ctx->M;
  a.model = ctx->model;
  a.spread = sp;
  a.device_dyn = (sp && dyn_dev == nullptr) ? 1 : 0;
  a.penalty = pen ? 1 : 0;
  a.two_point = (float)ctx->model_param;
  a.dp = ctx->dp;
  a.xin = ctx->d_xin;
  a.ang_last = ctx->d_ang_last;
  a.lw_mean = lw_mean;
  a.lw_std = lw_std;
  a.lw_plane = K * N;
  a.dyn = dyn_dev;
  a.costs = costs;
  a.crash = crash;
  if (N > ctx->smem_horizon) a.qs = ctx->d_qs;  // long horizon: stage costs through the (N, K) global scratch
  return launch_rollout(ctx, a, st);
}

dim3 partials_grid(int64_t chunks, int N) {
  return dim3((unsigned)chunks, (unsigned)((N + kChunkWarps - 1) / kChunkWarps));
}

// leaf partials of `chunks` chunks x N timesteps; the block-per-(chunk, t) kernel when
// a warp per (chunk, t) would leave most of the GPU idle (same bits either way)
// zin: the device-noise normals the attitude kernel stored (ctx->d_z); nullptr with host
// noise (eps)
int launch_partials(pi2_ctx *ctx, const double *costs, int64_t cs_k, int64_t cs_t, const double *eps,
                    const float4 *zin, int it, int64_t K, int64_t k_off, int N, double neg_inv, double *out,
                    cudaStream_t st, bool pdl) {
  Range range_("partials");
  const int64_t chunks = (K + kChunk - 1) / kChunk;
  const dim3 g = partials_grid(chunks, N);
  const bool split = ctx->partials_split == 2 || (ctx->partials_split == 1 && (int64_t)g.x * g.y < kPartialsSplitBlocks);
  if (split)
    TRY(launch_pdl_if(pdl, ctx, partials_split_kernel, dim3((unsigned)chunks, (unsigned)N), dim3(kChunk), 0, st, costs,
                      cs_k, cs_t, eps, zin, ctx->d_args, it, K, k_off, N, neg_inv, out));
  else
    TRY(launch_pdl_if(pdl, ctx, partials_kernel, g, dim3(32 * kChunkWarps), 0, st, costs, cs_k, cs_t, eps, zin,
                      ctx->d_args, it, K, k_off, N, neg_inv, out));
  CU(cudaGetLastError());
  return PI2_OK;
}

// after_kernel: the stream predecessor is the partials kernel (PDL allowed);
// plan_host: also store the updated plan there (see apply_root_kernel)
int launch_combine(pi2_ctx *ctx, const double *leaves, int64_t n, int N, double neg_inv, double *root,
                   double *plan, cudaStream_t st, bool after_kernel = false, double *plan_host = nullptr) {
  Range range_("combine");
  if (n == 1 && !root && plan) {  // a single partial: just apply it
    TRY(launch_pdl_if(after_kernel, ctx, apply_root_kernel, dim3((4 * N + 127) / 128), dim3(128), 0, st, leaves, N, plan, ctx->dp, plan_host));
    CU(cudaGetLastError());
    return PI2_OK;
  }
  if ((n + kSeg - 1) / kSeg > kSeg) return fail(ctx, PI2_ERR_INVALID, "too many partials (%lld)", (long long)n);
  const int smem = 2 * kSeg * PI2_PARTIAL_WIDTH * (int)sizeof(double);
  TRY(set_smem(ctx, combine_kernel, smem));
  TRY(launch_pdl_if(after_kernel, ctx, combine_kernel, dim3(N), dim3(kCombineThreads), smem, st, leaves, n, N, neg_inv, root, plan,
                    ctx->dp, plan_host));
  CU(cudaGetLastError());
  return PI2_OK;
}

// one full device-noise iteration on the device plan (optionally local-only)
int launch_iteration(pi2_ctx *ctx, int it, double neg_inv, double *root, bool update_plan,
                     cudaStream_t st, double *plan_host = nullptr, bool att_pdl = false) {
  TRY(launch_rollouts(ctx, it, nullptr, nullptr, ctx->d_costs, ctx->d_crash, st, nullptr, att_pdl));
  TRY(launch_partials(ctx, ctx->d_costs, 1, ctx->K, nullptr, ctx->store_z ? ctx->d_z : nullptr, it, ctx->K, ctx->dims.rollout_offset, ctx->N, neg_inv,
                      ctx->d_partials, st, true));
  return launch_combine(ctx, ctx->d_partials, ctx->n_chunks, ctx->N, neg_inv, root,
                        update_plan ? ctx->d_plan : nullptr, st, true, plan_host);
}

int validate_opt(pi2_ctx *ctx, const pi2_optimize_args *args) {
  if (!args) return fail(ctx, PI2_ERR_INVALID, "null optimize args");
  if (!(args->temperature > 0)) return fail(ctx, PI2_ERR_INVALID, "temperature must be positive");
  for (double s : args->exploration_std)
    if (!(s > 0)) return fail(ctx, PI2_ERR_INVALID, "exploration_std must be positive");
  if (args->iterations < 0) return fail(ctx, PI2_ERR_INVALID, "iterations must be >= 0");
  return PI2_OK;
}

}  // namespace

// =============================================================================
extern "C" {

int pi2_version(void) { return PI2_ABI_VERSION; }

const char *pi2_strerror(int s) {
  switch (s) {
    case PI2_OK: return "ok";
    case PI2_ERR_INVALID: return "invalid argument";
    case PI2_ERR_STATE: return "invalid state";
    case PI2_ERR_UNSUPPORTED: return "unsupported plugin";
    case PI2_ERR_CUDA: return "CUDA error";
    case PI2_ERR_OOM: return "out of device memory";
    default: return "unknown status";
  }
}

int pi2_device_count(int32_t *count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  if (count) *count = n;
  return PI2_OK;
}

const char *pi2_last_error(const pi2_ctx *ctx) {
  return ctx ? ctx->err.c_str() : g_noctx_err.c_str();
}

int pi2_get_dims(const pi2_ctx *ctx, pi2_dims *out) {
  if (!ctx || !out) return PI2_ERR_INVALID;
  *out = ctx->dims;
  return PI2_OK;
}

int pi2_create(int32_t device, const pi2_dims *dims, pi2_ctx **out) {
  pi2_ctx *ctx = nullptr;
  if (!out || !dims) return fail(nullptr, PI2_ERR_INVALID, "null argument");
  *out = nullptr;
  if (dims->num_rollouts < 1 || dims->sub_rollouts < 1 || dims->horizon_steps < 1)
    return fail(nullptr, PI2_ERR_INVALID, "num_rollouts, sub_rollouts, horizon_steps must be >= 1");
  if (dims->sub_rollouts > PI2_MAX_SUB_ROLLOUTS)
    return fail(nullptr, PI2_ERR_INVALID, "sub_rollouts must be <= %d", PI2_MAX_SUB_ROLLOUTS);
  // the partials grid has ceil(N / kChunkWarps) rows (grid.y <= 65535)
  constexpr int kHorizonLimit = kChunkWarps * 65535;
  if (dims->horizon_steps > kHorizonLimit)
    return fail(nullptr, PI2_ERR_INVALID, "horizon_steps must be <= %d", kHorizonLimit);
  if (dims->rollout_offset < 0) return fail(nullptr, PI2_ERR_INVALID, "rollout_offset must be >= 0");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(nullptr, PI2_ERR_CUDA, "no CUDA device available");
  }
  if (device < 0 || device >= n) return fail(nullptr, PI2_ERR_INVALID, "device %d out of range", device);
  ctx = new pi2_ctx();
  ctx->device = device;
  ctx->dims = *dims;
  if (ctx->dims.num_rollouts_total <= 0) ctx->dims.num_rollouts_total = dims->num_rollouts;
  ctx->K = dims->num_rollouts;
  ctx->N = dims->horizon_steps;
  ctx->M = dims->sub_rollouts;
  int rc = PI2_OK;
  auto cleanup = [&](int code) {
    pi2_destroy(ctx);
    return code;
  };
  if ((rc = bind(ctx)) != PI2_OK) { g_noctx_err = ctx->err; return cleanup(rc); }
  cudaDeviceGetAttribute(&ctx->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (const char *e = getenv("PI2_PDL")) ctx->pdl = std::atoi(e) != 0;
  if (const char *e = getenv("PI2_IO_PULL")) ctx->io_pull = std::atoi(e) != 0;
  if (const char *e = getenv("PI2_PARTIALS_SPLIT")) ctx->partials_split = std::atoi(e);
  if (const char *e = getenv("PI2_WIDE_MAX_K")) ctx->wide_max_k = std::atoll(e);
  if (const char *e = getenv("PI2_TC_BULK_MAX_TILES")) ctx->tc_bulk_max_tiles = std::atoll(e);
  if (const char *e = getenv("PI2_FUSED")) ctx->fused = std::atoi(e);
  if (const char *e = getenv("PI2_STORE_Z")) ctx->store_z = std::atoi(e) != 0;
  if (const char *e = getenv("PI2_SMEM_HORIZON")) ctx->smem_horizon = std::min(std::atoi(e), kSmemHorizon);
  {
    int uva = 0;
    cudaDeviceGetAttribute(&uva, cudaDevAttrUnifiedAddressing, device);
    ctx->uva = uva != 0;
  }
  if (const char *e = getenv("PI2_LWPR_TC")) {
    ctx->tc_mode = std::atoi(e);
    ctx->tc_enabled = ctx->tc_mode != 0;
  }
  const int64_t K = ctx->K, N = ctx->N;
  ctx->n_chunks = (K + kChunk - 1) / kChunk;
#define ALLOC(p, bytes)                                                               \
  if (cudaMalloc((void **)&(p), (bytes)) != cudaSuccess) {                           \
    cudaGetLastError();                                                               \
    g_noctx_err = "device allocation failed: " #p;                                    \
    return cleanup(PI2_ERR_OOM);                                                      \
  }
  ALLOC(ctx->d_io, kIoArgsBytes + sizeof(double) * 4 * N);
  ctx->d_args = reinterpret_cast<StepArgs *>(ctx->d_io);
  ctx->d_plan = reinterpret_cast<double *>(ctx->d_io + kIoArgsBytes);
  ALLOC(ctx->d_plan2, sizeof(double) * 4 * N);
  ALLOC(ctx->d_xin, sizeof(float4) * K * N);
  ALLOC(ctx->d_ang_last, sizeof(float4) * K);
  ALLOC(ctx->d_lw, sizeof(float4) * K * N * 2);
  if (N > ctx->smem_horizon) {  // long horizons: the rollout kernels' stage costs go through global memory
    ALLOC(ctx->d_qs, sizeof(float) * K * N);
    ctx->qs_cap = sizeof(float) * K * N;
  }
  ALLOC(ctx->d_costs, sizeof(double) * K * N);
  ALLOC(ctx->d_crash, K);
  ALLOC(ctx->d_partials, sizeof(double) * PI2_PARTIAL_WIDTH * ctx->n_chunks * N);
  ALLOC(ctx->d_root, sizeof(double) * PI2_PARTIAL_WIDTH * N);
  ALLOC(ctx->d_z, sizeof(float4) * K * N);
#undef ALLOC
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->staged, cudaEventDisableTiming) != cudaSuccess ||
      cudaMallocHost((void **)&ctx->h_io, kIoArgsBytes + sizeof(double) * 4 * N) != cudaSuccess) {
    cudaGetLastError();
    g_noctx_err = "stream/event/pinned allocation failed";
    return cleanup(PI2_ERR_CUDA);
  }
  ctx->h_args = reinterpret_cast<StepArgs *>(ctx->h_io);
  ctx->h_plan = reinterpret_cast<double *>(ctx->h_io + kIoArgsBytes);
  std::memset(ctx->h_args, 0, sizeof(StepArgs));
  ctx->h_args->neg_inv_temp = -1.0;
  ctx->h_args->ceiling = 1e8;
  cudaEventRecord(ctx->staged, ctx->stream);
  *out = ctx;
  return PI2_OK;
}

void pi2_destroy(pi2_ctx *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  invalidate_graph(ctx);
  void *bufs[] = {ctx->d_params, ctx->d_tc, ctx->d_io,     ctx->d_plan2,    ctx->d_xin,
                  ctx->d_ang_last, ctx->d_lw,   ctx->d_costs, ctx->d_crash,    ctx->d_partials,
                  ctx->d_root,   ctx->d_noise,  ctx->d_dynbuf, ctx->d_scratch, ctx->d_z, ctx->d_qs,
                  ctx->d_xobs};
  for (void *p : bufs)
    if (p) cudaFree(p);
  if (ctx->h_io) cudaFreeHost(ctx->h_io);
  if (ctx->staged) cudaEventDestroy(ctx->staged);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  cudaGetLastError();
  delete ctx;
}

int pi2_set_dynamics(pi2_ctx *ctx, const pi2_dynamics *d) {
  if (!ctx || !d) return fail(ctx, PI2_ERR_INVALID, "null argument");
  if (!(d->mass > 0) || !(d->dt > 0) || !(d->rate_gain > 0))
    return fail(ctx, PI2_ERR_INVALID, "mass, dt and rate_gain must be positive");
  // DynParams are kernel arguments baked into the cached graph: re-capture only on change
  if (ctx->have_dyn && std::memcmp(&ctx->dyn, d, sizeof(pi2_dynamics)) == 0) return PI2_OK;
  ctx->dyn = *d;
  DynParams &p = ctx->dp;
  p.dt = d->dt;
  p.gain_dt = d->rate_gain * d->dt;
  ctx->bounds_nonan = true;
  for (int c = 0; c < 4; ++c) {
    p.lo[c] = d->lo[c];
    p.hi[c] = d->hi[c];
    if (std::isnan(d->lo[c]) || std::isnan(d->hi[c])) ctx->bounds_nonan = false;
  }
  p.dt32 = (float)d->dt;
  p.dt2_32 = p.dt32 * p.dt32;
  p.inv_m32 = (float)(1.0 / d->mass);
  p.g32 = (float)d->gravity;
  ctx->have_dyn = true;
  invalidate_graph(ctx);
  return PI2_OK;
}

int pi2_set_lwpr_axis(pi2_ctx *ctx, int32_t axis, int32_t L, int32_t d, const double *centers,
                      const double *metrics, const double *coefs, const double *lvar) {
  if (!ctx) return fail(nullptr, PI2_ERR_INVALID, "null context");
  if (axis < 0 || axis > 2) return fail(ctx, PI2_ERR_INVALID, "axis must be 0, 1 or 2");
  if (L < 1) return fail(ctx, PI2_ERR_INVALID, "no receptive fields");
  if (d < 1 || d > 4) return fail(ctx, PI2_ERR_UNSUPPORTED, "input_dim must be 1..4");
  if (!centers || !metrics || !coefs || !lvar) return fail(ctx, PI2_ERR_INVALID, "null field array");
  AxisRaw &a = ctx->axes[axis];
  a.L = L;
  a.d = d;
  a.centers.assign(centers, centers + (size_t)L * d);
  a.metrics.assign(metrics, metrics + (size_t)L * d * d);
  a.coefs.assign(coefs, coefs + (size_t)L * (d + 1));
  a.lvar.assign(lvar, lvar + L);
  for (double v : a.centers) if (!std::isfinite(v)) return fail(ctx, PI2_ERR_INVALID, "non-finite center");
  for (double v : a.metrics) if (!std::isfinite(v)) return fail(ctx, PI2_ERR_INVALID, "non-finite metric");
  for (double v : a.coefs) if (!std::isfinite(v)) return fail(ctx, PI2_ERR_INVALID, "non-finite coefficient");
  ctx->params_dirty = true;
  invalidate_graph(ctx);
  return PI2_OK;
}

int pi2_select_model(pi2_ctx *ctx, int32_t kind, double param) {
  if (!ctx) return fail(nullptr, PI2_ERR_INVALID, "null context");
  switch (kind) {
    case PI2_MODEL_HYBRID_LWPR: {
      const char *names = "xyz";
      for (int ax = 0; ax < 3; ++ax) {
        if (ctx->axes[ax].L == 0)
          return fail(ctx, PI2_ERR_INVALID, "acceleration model for %c axis is untrained", names[ax]);
        if (ctx->axes[ax].d != 4) return fail(ctx, PI2_ERR_INVALID, "acceleration models take 4 inputs");
      }
      break;
    }
    case PI2_MODEL_ANALYTIC:
    case PI2_MODEL_TWO_POINT:
      break;
    default:
      return fail(ctx, PI2_ERR_UNSUPPORTED, "unknown model kind %d", kind);
  }
  if (ctx->model != kind || ctx->model_param != param) invalidate_graph(ctx);
  ctx->model = kind;
  ctx->model_param = param;
  return PI2_OK;
}

int pi2_set_cost(pi2_ctx *ctx, const pi2_cost *c) {
  if (!ctx || !c) return fail(ctx, PI2_ERR_INVALID, "null argument");
  if (c->kind != PI2_COST_NAVIGATION && c->kind != PI2_COST_THRESHOLD)
    return fail(ctx, PI2_ERR_UNSUPPORTED, "unknown cost kind %d", c->kind);
  if (c->n_obstacles < 0 || c->n_obstacles > PI2_MAX_OBSTACLES)
    return fail(ctx, PI2_ERR_UNSUPPORTED, "at most %d obstacles in pi2_cost (longer lists: pi2_set_cost_obstacles)",
                PI2_MAX_OBSTACLES);
  if (!(c->variance_penalty >= 0.0f) || !std::isfinite(c->variance_penalty))
    return fail(ctx, PI2_ERR_INVALID, "variance_penalty must be finite and >= 0");
  // kernel variants depend on the kind and on whether the penalty is on
  if (ctx->have_cost && (ctx->cost.kind != c->kind || (ctx->cost.variance_penalty > 0) != (c->variance_penalty > 0) ||
                         !struct_obstacles(ctx)))
    invalidate_graph(ctx);
  ctx->cost = *c;
  ctx->have_cost = true;
  return PI2_OK;
}

int pi2_set_cost_obstacles(pi2_ctx *ctx, int32_t n, const float *xy) {
  if (!ctx) return fail(nullptr, PI2_ERR_INVALID, "null context");
  if (!ctx->have_cost || ctx->cost.kind != PI2_COST_NAVIGATION)
    return fail(ctx, PI2_ERR_STATE, "set a navigation cost (pi2_set_cost) first");
  if (n < 0 || (n > 0 && !xy)) return fail(ctx, PI2_ERR_INVALID, "bad obstacle list");
  const int head = n < PI2_MAX_OBSTACLES ? n : PI2_MAX_OBSTACLES;
  // kernel selection depends on whether the list fits the struct (struct_obstacles)
  if ((ctx->cost.n_obstacles > PI2_MAX_OBSTACLES) != (n > PI2_MAX_OBSTACLES)) invalidate_graph(ctx);
  std::memset(ctx->cost.obstacles, 0, sizeof ctx->cost.obstacles);
  std::memcpy(ctx->cost.obstacles, xy, sizeof(float) * 2 * head);
  ctx->cost.n_obstacles = n;
  std::vector<float> tail(xy + 2 * head, xy + 2 * (size_t)n);
  if (tail == ctx->h_xobs) return PI2_OK;
  // rare (the list changed): no kernel of this device may still read the old list
  CU(cudaSetDevice(ctx->device));
  CU(cudaDeviceSynchronize());
  if (tail.size() > ctx->xobs_cap) {
    if (ctx->d_xobs) CU(cudaFree(ctx->d_xobs));
    ctx->d_xobs = nullptr;
    ctx->xobs_cap = 0;
    if (cudaMalloc(&ctx->d_xobs, tail.size() * sizeof(float)) != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, PI2_ERR_OOM, "obstacle list allocation failed");
    }
    ctx->xobs_cap = tail.size();
  }
  if (!tail.empty()) CU(cudaMemcpy(ctx->d_xobs, tail.data(), tail.size() * sizeof(float), cudaMemcpyHostToDevice));
  ctx->h_xobs = std::move(tail);
  return PI2_OK;
}

int pi2_evaluate_device(pi2_ctx *ctx, const double *state, const double *plan, const double *noise_dev,
                        const float *dyn_dev, double ceiling, double *costs_dev, uint8_t *crash_dev,
                        void *stream) {
  Range range_("pi2_evaluate_device");
  TRY(check_ready(ctx));
  TRY(bind(ctx));
  if (!state || !plan || !noise_dev || !costs_dev || !crash_dev)
    return fail(ctx, PI2_ERR_INVALID, "null argument");
  if (spread(ctx) && !dyn_dev)
    return fail(ctx, PI2_ERR_INVALID, "probabilistic model with sub_rollouts > 1 needs dyn_noise");
  cudaStream_t st = pick(ctx, stream);
  TRY(stage_args(ctx, state, nullptr, ceiling, st));
  TRY(stage_plan(ctx, plan, st));
  TRY(launch_rollouts(ctx, 0, noise_dev, dyn_dev, ctx->d_costs, crash_dev, st));
  const dim3 tg((unsigned)((ctx->K + 31) / 32), (unsigned)((ctx->N + 31) / 32));
  transpose_costs_kernel<<<tg, dim3(32, 8), 0, st>>>(ctx->d_costs, costs_dev, ctx->K, ctx->N);
  CU(cudaGetLastError());
  return PI2_OK;
}

int pi2_evaluate_device_noise(pi2_ctx *ctx, const double *state, const double *plan, const pi2_optimize_args *args,
                              int32_t iteration, double *costs_dev, uint8_t *crash_dev, void *stream) {
  Range range_("pi2_evaluate_device_noise");
  TRY(check_ready(ctx));
  TRY(bind(ctx));
  TRY(validate_opt(ctx, args));
  if (!state || !plan || !costs_dev || !crash_dev || iteration < 0) return fail(ctx, PI2_ERR_INVALID, "bad argument");
  cudaStream_t st = pick(ctx, stream);
  TRY(ensure_params(ctx));
  TRY(stage_args(ctx, state, args, args->cost_ceiling, st));
  TRY(stage_plan(ctx, plan, st));
  TRY(launch_rollouts(ctx, iteration, nullptr, nullptr, ctx->d_costs, crash_dev, st));
  const dim3 tg((unsigned)((ctx->K + 31) / 32), (unsigned)((ctx->N + 31) / 32));
  transpose_costs_kernel<<<tg, dim3(32, 8), 0, st>>>(ctx->d_costs, costs_dev, ctx->K, ctx->N);
  CU(cudaGetLastError());
  return PI2_OK;
}

int pi2_evaluate(pi2_ctx *ctx, const double *state, const double *plan, const double *noise,
                 const float *dyn, double ceiling, double *costs_out, uint8_t *crash_out) {
  Range range_("pi2_evaluate");
  TRY(check_ready(ctx));
  TRY(bind(ctx));
  if (!state || !plan || !noise || !costs_out || !crash_out) return fail(ctx, PI2_ERR_INVALID, "null argument");
  const bool sp = spread(ctx);
  if (sp && !dyn)
    return fail(ctx, PI2_ERR_INVALID, "probabilistic model with sub_rollouts > 1 needs dyn_noise");
  const int64_t K = ctx->K, N = ctx->N, M = ctx->M;
  cudaStream_t st = ctx->stream;
  TRY(ensure(ctx, (void **)&ctx->d_noise, &ctx->noise_cap, sizeof(double) * K * N * 4));
  CU(cudaMemcpyAsync(ctx->d_noise, noise, sizeof(double) * K * N * 4, cudaMemcpyHostToDevice, st));
  const float *dyn_dev = nullptr;
  if (sp) {
    TRY(ensure(ctx, (void **)&ctx->d_dynbuf, &ctx->dyn_cap, sizeof(float) * K * M * N * 3));
    CU(cudaMemcpyAsync(ctx->d_dynbuf, dyn, sizeof(float) * K * M * N * 3, cudaMemcpyHostToDevice, st));
    dyn_dev = ctx->d_dynbuf;
  }
  TRY(ensure(ctx, &ctx->d_scratch, &ctx->scratch_cap, sizeof(double) * K * N));
  double *out = (double *)ctx->d_scratch;
  TRY(pi2_evaluate_device(ctx, state, plan, ctx->d_noise, dyn_dev, ceiling, out, ctx->d_crash, st));
  CU(cudaMemcpyAsync(costs_out, out, sizeof(double) * K * N, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(crash_out, ctx->d_crash, K, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return PI2_OK;
}

int pi2_update_device(pi2_ctx *ctx, int64_t K, int32_t N, const double *plan, const double *costs_dev,
                      const double *noise_dev, double temperature, double *plan_out, void *stream) {
  Range range_("pi2_update_device");
  if (!ctx) return fail(nullptr, PI2_ERR_INVALID, "null context");
  TRY(bind(ctx));
  if (!ctx->have_dyn) return fail(ctx, PI2_ERR_STATE, "dynamics not set (pi2_set_dynamics)");
  if (K < 1 || N < 1 || !plan || !costs_dev || !noise_dev || !plan_out)
    return fail(ctx, PI2_ERR_INVALID, "batch does not match plan dimensions");
  if (!(temperature > 0)) return fail(ctx, PI2_ERR_INVALID, "temperature must be positive");
  cudaStream_t st = pick(ctx, stream);
  const int64_t chunks = (K + kChunk - 1) / kChunk;
  const size_t pbytes = sizeof(double) * PI2_PARTIAL_WIDTH * chunks * N;
  const size_t plbytes = sizeof(double) * 4 * N;
  TRY(ensure(ctx, &ctx->d_scratch, &ctx->scratch_cap, pbytes + plbytes));
  double *partials = (double *)ctx->d_scratch;
  double *dplan = partials + PI2_PARTIAL_WIDTH * chunks * N;
  CU(cudaMemcpyAsync(dplan, plan, plbytes, cudaMemcpyHostToDevice, st));
  const double neg_inv = -1.0 / temperature;
  TRY(launch_partials(ctx, costs_dev, N, 1, noise_dev, nullptr, 0, K, 0, N, neg_inv, partials, st, false));
  TRY(launch_combine(ctx, partials, chunks, N, neg_inv, nullptr, dplan, st));
  CU(cudaMemcpyAsync(plan_out, dplan, plbytes, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return PI2_OK;
}

int pi2_update(pi2_ctx *ctx, int64_t K, int32_t N, const double *plan, const double *costs,
               const double *noise, double temperature, double *plan_out) {
  Range range_("pi2_update");
  if (!ctx) return fail(nullptr, PI2_ERR_INVALID, "null context");
  TRY(bind(ctx));
  if (K < 1 || N < 1 || !costs || !noise) return fail(ctx, PI2_ERR_INVALID, "batch does not match plan dimensions");
  cudaStream_t st = ctx->stream;
  TRY(ensure(ctx, (void **)&ctx->d_noise, &ctx->noise_cap, sizeof(double) * K * N * 5));
  double *dnoise = ctx->d_noise, *dcosts = ctx->d_noise + K * N * 4;
  CU(cudaMemcpyAsync(dnoise, noise, sizeof(double) * K * N * 4, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(dcosts, costs, sizeof(double) * K * N, cudaMemcpyHostToDevice, st));
  return pi2_update_device(ctx, K, N, plan, dcosts, dnoise, temperature, plan_out, st);
}

// All iterations of a step on the device plan: eager, or one cached CUDA graph
// (kernel arguments are fixed pointers; per-call state, keys and cost come
// from the staged StepArgs, so replays need no re-capture).
// io: also copy StepArgs + plan in from the pinned block first and the plan back out last
static int enqueue_iterations(pi2_ctx *ctx, int iterations, double neg_inv, bool io, cudaStream_t st) {
  const size_t plan_bytes = sizeof(double) * 4 * ctx->N;
  const bool pull = io && ctx->uva && ctx->io_pull;
  if (pull) {
    io_pull_kernel<<<1, 256, 0, st>>>(reinterpret_cast<const uint4 *>(ctx->h_io), reinterpret_cast<uint4 *>(ctx->d_io),
                                      (int)((kIoArgsBytes + plan_bytes) / sizeof(uint4)));
    CU(cudaGetLastError());
  } else if (io) {
    CU(cudaMemcpyAsync(ctx->d_io, ctx->h_io, kIoArgsBytes + plan_bytes, cudaMemcpyHostToDevice, st));
  }
  // the last iteration's update also lands in the pinned host plan (no D2H copy node)
  const bool direct = io && ctx->uva;
  for (int it = 0; it < iterations; ++it)
    TRY(launch_iteration(ctx, it, neg_inv, nullptr, true, st, direct && it == iterations - 1 ? ctx->h_plan : nullptr,
                         pull && it == 0));
  if (io && !direct) CU(cudaMemcpyAsync(ctx->h_plan, ctx->d_plan, plan_bytes, cudaMemcpyDeviceToHost, st));
  return PI2_OK;
}

static int run_iterations(pi2_ctx *ctx, const pi2_optimize_args *args, cudaStream_t st, bool io = false) {
  const double neg_inv = -1.0 / args->temperature;
  if (!args->use_graph) return enqueue_iterations(ctx, args->iterations, neg_inv, io, st);
  cudaGraphExec_t &exec = io ? ctx->graph_io : ctx->graph;
  int &iters = io ? ctx->graph_io_iters : ctx->graph_iters;
  double &ninv = io ? ctx->graph_io_neg_inv : ctx->graph_neg_inv;
  if (!(exec && iters == args->iterations && ninv == neg_inv)) {
    if (exec) cudaGraphExecDestroy(exec);
    exec = nullptr;
    iters = -1;
    // capture on the private stream (never a caller's), ordered after `st` by the launch below
    cudaGraph_t g = nullptr;
    CU(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    const int rc = enqueue_iterations(ctx, args->iterations, neg_inv, io, ctx->stream);
    const cudaError_t ec = cudaStreamEndCapture(ctx->stream, &g);
    if (rc != PI2_OK) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (ec != cudaSuccess) return fail(ctx, PI2_ERR_CUDA, "graph capture: %s", cudaGetErrorString(ec));
    const cudaError_t ei = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) return fail(ctx, PI2_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(ei));
    iters = args->iterations;
    ninv = neg_inv;
  }
  CU(cudaGraphLaunch(exec, st));
  return PI2_OK;
}

int pi2_iterate_device(pi2_ctx *ctx, const pi2_optimize_args *args, void *stream) {
  Range range_("pi2_iterate_device");
  TRY(check_ready(ctx));
  TRY(bind(ctx));
  TRY(validate_opt(ctx, args));
  if (args->iterations == 0) return PI2_OK;
  cudaStream_t st = pick(ctx, stream);
  TRY(ensure_params(ctx));
  TRY(stage_args(ctx, nullptr, args, args->cost_ceiling, st));
  return run_iterations(ctx, args, st);
}

int pi2_optimize(pi2_ctx *ctx, const double *state, double *plan_inout, const pi2_optimize_args *args) {
  Range range_("pi2_optimize");
  TRY(check_ready(ctx));
  TRY(bind(ctx));
  TRY(validate_opt(ctx, args));
  if (!state || !plan_inout) return fail(ctx, PI2_ERR_INVALID, "null argument");
  if (args->iterations == 0) return PI2_OK;  // plan unchanged (test_controller.py:261-265)
  cudaStream_t st = ctx->stream;
  TRY(ensure_params(ctx));
  // one graph launch: H2D of StepArgs + plan, the iterations, D2H of the plan
  CU(cudaEventSynchronize(ctx->staged));
  fill_args(ctx, state, args, args->cost_ceiling);
  std::memcpy(ctx->h_plan, plan_inout, sizeof(double) * 4 * ctx->N);
  TRY(run_iterations(ctx, args, st, true));
  CU(cudaStreamSynchronize(st));
  std::memcpy(plan_inout, ctx->h_plan, sizeof(double) * 4 * ctx->N);
  return PI2_OK;
}

int pi2_receding_horizon_step(pi2_ctx *ctx, const double *state, double *plan_inout,
                              const pi2_optimize_args *args, double *control_out) {
  Range range_("pi2_receding_horizon_step");
  TRY(pi2_optimize(ctx, state, plan_inout, args));
  const int N = ctx->N;
  if (control_out) std::memcpy(control_out, plan_inout, 4 * sizeof(double));
  std::memmove(plan_inout, plan_inout + 4, sizeof(double) * 4 * (N - 1));
  if (N > 1) std::memcpy(plan_inout + 4 * (N - 1), plan_inout + 4 * (N - 2), 4 * sizeof(double));
  return PI2_OK;
}

int pi2_load_plan(pi2_ctx *ctx, const double *state, const double *plan, void *stream) {
  if (!ctx || !plan) return fail(ctx, PI2_ERR_INVALID, "null argument");
  TRY(bind(ctx));
  cudaStream_t st = pick(ctx, stream);
  CU(cudaEventSynchronize(ctx->staged));
  if (state) std::memcpy(ctx->h_args->state, state, sizeof(double) * 12);
  return stage_plan(ctx, plan, st);
}

int pi2_read_plan(pi2_ctx *ctx, double *plan_out, void *stream) {
  if (!ctx || !plan_out) return fail(ctx, PI2_ERR_INVALID, "null argument");
  TRY(bind(ctx));
  cudaStream_t st = pick(ctx, stream);
  CU(cudaMemcpyAsync(plan_out, ctx->d_plan, sizeof(double) * 4 * ctx->N, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return PI2_OK;
}

int pi2_iterate_local(pi2_ctx *ctx, const pi2_optimize_args *args, int32_t iteration, double *root_dev,
                      void *stream) {
  Range range_("pi2_iterate_local");
  TRY(check_ready(ctx));
  TRY(bind(ctx));
  TRY(validate_opt(ctx, args));
  if (iteration < 0 || iteration >= std::max(1, args->iterations) || !root_dev)
    return fail(ctx, PI2_ERR_INVALID, "bad iteration index or null partial buffer");
  cudaStream_t st = pick(ctx, stream);
  TRY(ensure_params(ctx));
  TRY(stage_args(ctx, nullptr, args, args->cost_ceiling, st));
  return launch_iteration(ctx, iteration, -1.0 / args->temperature, root_dev, false, st);
}

// ---- a rank's control step as one caller-captured CUDA graph (N > 1) ----------
// The collective sits between the kernels, so the caller (torch.distributed) owns
// the graph; these calls only enqueue work on `stream` (no host synchronisation,
// no allocation), so they can be captured together with the NCCL all-gather.
int pi2_stage_step(pi2_ctx *ctx, const double *state, const double *plan, const pi2_optimize_args *args) {
  TRY(check_ready(ctx));
  TRY(bind(ctx));
  TRY(validate_opt(ctx, args));
  if (!state || !plan) return fail(ctx, PI2_ERR_INVALID, "null argument");
  TRY(ensure_params(ctx));  // model staging happens here, never inside a capture
  CU(cudaEventSynchronize(ctx->staged));
  fill_args(ctx, state, args, args->cost_ceiling);
  std::memcpy(ctx->h_plan, plan, sizeof(double) * 4 * ctx->N);
  return PI2_OK;
}

int pi2_enqueue_pull(pi2_ctx *ctx, void *stream) {
  if (!ctx) return fail(nullptr, PI2_ERR_INVALID, "null context");
  TRY(bind(ctx));
  cudaStream_t st = pick(ctx, stream);
  const size_t bytes = kIoArgsBytes + sizeof(double) * 4 * ctx->N;
  if (ctx->uva && ctx->io_pull) {
    io_pull_kernel<<<1, 256, 0, st>>>(reinterpret_cast<const uint4 *>(ctx->h_io), reinterpret_cast<uint4 *>(ctx->d_io),
                                      (int)(bytes / sizeof(uint4)));
    CU(cudaGetLastError());
  } else {
    CU(cudaMemcpyAsync(ctx->d_io, ctx->h_io, bytes, cudaMemcpyHostToDevice, st));
  }
  return PI2_OK;
}

int pi2_iterate_local_staged(pi2_ctx *ctx, int32_t iteration, double temperature, double *root_dev, void *stream) {
  Range range_("pi2_iterate_local_staged");
  TRY(check_ready(ctx));
  TRY(bind(ctx));
  if (iteration < 0 || !root_dev) return fail(ctx, PI2_ERR_INVALID, "bad iteration index or null partial buffer");
  if (!(temperature > 0)) return fail(ctx, PI2_ERR_INVALID, "temperature must be positive");
  if (ctx->params_dirty) return fail(ctx, PI2_ERR_STATE, "model changed since pi2_stage_step");
  return launch_iteration(ctx, iteration, -1.0 / temperature, root_dev, false, pick(ctx, stream));
}

int pi2_enqueue_push(pi2_ctx *ctx, void *stream) {
  if (!ctx) return fail(nullptr, PI2_ERR_INVALID, "null context");
  TRY(bind(ctx));
  CU(cudaMemcpyAsync(ctx->h_plan, ctx->d_plan, sizeof(double) * 4 * ctx->N, cudaMemcpyDeviceToHost,
                     pick(ctx, stream)));
  return PI2_OK;
}

int pi2_fetch_plan(pi2_ctx *ctx, double *plan_out, void *stream) {
  if (!ctx || !plan_out) return fail(ctx, PI2_ERR_INVALID, "null argument");
  TRY(bind(ctx));
  CU(cudaStreamSynchronize(pick(ctx, stream)));
  std::memcpy(plan_out, ctx->h_plan, sizeof(double) * 4 * ctx->N);
  return PI2_OK;
}

int pi2_lwpr_kernel(pi2_ctx *ctx, int32_t variance, int32_t *kernel_out, double *mufu_share) {
  TRY(check_ready(ctx));
  if (!kernel_out) return fail(ctx, PI2_ERR_INVALID, "null argument");
  TRY(bind(ctx));
  TRY(ensure_params(ctx));
  const bool var = variance != 0;
  const bool tc = ctx->tc_ok && tc_wanted(ctx, var);
  *kernel_out = tc ? PI2_LWPR_TENSOR_CORES : PI2_LWPR_CUDA_CORES;
  if (mufu_share)  // field pairs on the FMA pipe, of 4 + 4 per two batches
    *mufu_share = tc ? 1.0 - (var ? PI2_TC_POLY_VAR + PI2_TC_POLY_VAR_B : PI2_TC_POLY_MEAN + PI2_TC_POLY_MEAN_B) / 8.0
                     : 1.0;
  return PI2_OK;
}

int pi2_fused_step(pi2_ctx *ctx, int32_t *sub_rollouts_out) {
  TRY(check_ready(ctx));
  if (!sub_rollouts_out) return fail(ctx, PI2_ERR_INVALID, "null argument");
  TRY(bind(ctx));
  TRY(ensure_params(ctx));
  *sub_rollouts_out = fused_mm(ctx);
  return PI2_OK;
}

int pi2_profile_iteration(pi2_ctx *ctx, const pi2_optimize_args *args, int32_t reps, double *stage_ms) {
  Range range_("pi2_profile_iteration");
  TRY(check_ready(ctx));
  TRY(bind(ctx));
  TRY(validate_opt(ctx, args));
  if (reps < 1 || !stage_ms) return fail(ctx, PI2_ERR_INVALID, "reps must be >= 1");
  cudaStream_t st = ctx->stream;
  TRY(ensure_params(ctx));
  TRY(stage_args(ctx, nullptr, args, args->cost_ceiling, st));
  cudaEvent_t ev[6];
  for (auto &e : ev) CU(cudaEventCreate(&e));
  const double neg_inv = -1.0 / args->temperature;
  double acc[5] = {0, 0, 0, 0, 0};
  int rc = PI2_OK;
  for (int r = 0; r < reps && rc == PI2_OK; ++r) {
    cudaEventRecord(ev[0], st);
    rc = launch_rollouts(ctx, 0, nullptr, nullptr, ctx->d_costs, ctx->d_crash, st, ev);
    if (rc != PI2_OK) break;
    cudaEventRecord(ev[3], st);
    rc = launch_partials(ctx, ctx->d_costs, 1, ctx->K, nullptr, ctx->store_z ? ctx->d_z : nullptr, 0, ctx->K, ctx->dims.rollout_offset, ctx->N, neg_inv,
                         ctx->d_partials, st, false);
    if (rc != PI2_OK) break;
    cudaEventRecord(ev[4], st);
    rc = launch_combine(ctx, ctx->d_partials, ctx->n_chunks, ctx->N, neg_inv, ctx->d_root, nullptr, st);
    cudaEventRecord(ev[5], st);
    if (cudaEventSynchronize(ev[5]) != cudaSuccess) rc = fail(ctx, PI2_ERR_CUDA, "profile: %s", cudaGetErrorString(cudaGetLastError()));
    for (int i = 0; i < 5 && rc == PI2_OK; ++i) {
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      acc[i] += ms;
    }
  }
  for (auto &e : ev) cudaEventDestroy(e);
  TRY(rc);
  for (int i = 0; i < 5; ++i) stage_ms[i] = acc[i] / reps;
  return PI2_OK;
}

int pi2_profile_evaluate(pi2_ctx *ctx, const double *state, const double *plan, const double *noise_dev,
                         const float *dyn_dev, int32_t reps, double *stage_ms) {
  TRY(check_ready(ctx));
  TRY(bind(ctx));
  if (!state || !plan || !noise_dev || reps < 1 || !stage_ms) return fail(ctx, PI2_ERR_INVALID, "bad argument");
  if (spread(ctx) && !dyn_dev)
    return fail(ctx, PI2_ERR_INVALID, "probabilistic model with sub_rollouts > 1 needs dyn_noise");
  cudaStream_t st = ctx->stream;
  TRY(ensure_params(ctx));
  TRY(stage_args(ctx, state, nullptr, 1e8, st));
  TRY(stage_plan(ctx, plan, st));
  cudaEvent_t ev[4];
  for (auto &e : ev) CU(cudaEventCreate(&e));
  double acc[3] = {0, 0, 0};
  int rc = PI2_OK;
  for (int r = 0; r < reps && rc == PI2_OK; ++r) {
    cudaEventRecord(ev[0], st);
    rc = launch_rollouts(ctx, 0, noise_dev, dyn_dev, ctx->d_costs, ctx->d_crash, st, ev);
    if (rc != PI2_OK) break;
    cudaEventRecord(ev[3], st);
    if (cudaEventSynchronize(ev[3]) != cudaSuccess) rc = fail(ctx, PI2_ERR_CUDA, "profile: %s", cudaGetErrorString(cudaGetLastError()));
    for (int i = 0; i < 3 && rc == PI2_OK; ++i) {
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      acc[i] += ms;
    }
  }
  for (auto &e : ev) cudaEventDestroy(e);
  TRY(rc);
  for (int i = 0; i < 3; ++i) stage_ms[i] = acc[i] / reps;
  return PI2_OK;
}

int pi2_iterate_finalize(pi2_ctx *ctx, const double *gathered, int32_t world, double temperature,
                         void *stream) {
  Range range_("pi2_iterate_finalize");
  if (!ctx || !gathered || world < 1) return fail(ctx, PI2_ERR_INVALID, "bad gathered partials");
  TRY(bind(ctx));
  if (!(temperature > 0)) return fail(ctx, PI2_ERR_INVALID, "temperature must be positive");
  return launch_combine(ctx, gathered, world, ctx->N, -1.0 / temperature, nullptr, ctx->d_plan,
                        pick(ctx, stream));
}

int64_t pi2_partial_chunk(void) { return kChunk; }

int pi2_chunk_partials_host(const double *costs, const double *noise, int64_t K, int32_t N,
                            double temperature, double *out) {
  if (!costs || !noise || !out || K < 1 || N < 1 || !(temperature > 0)) return PI2_ERR_INVALID;
  const double neg_inv = -1.0 / temperature;
  const int64_t chunks = (K + kChunk - 1) / kChunk;
  for (int64_t c = 0; c < chunks; ++c)
    for (int t = 0; t < N; ++t) {
      double m = INFINITY;
      const int64_t k0 = c * kChunk, k1 = std::min<int64_t>(K, k0 + kChunk);
      for (int64_t k = k0; k < k1; ++k) m = std::min(m, costs[k * N + t]);
      double z = 0, v[4] = {0, 0, 0, 0};
      for (int64_t k = k0; k < k1; ++k) {
        const double w = std::exp((costs[k * N + t] - m) * neg_inv);
        z += w;
        for (int q = 0; q < 4; ++q) v[q] += w * noise[(k * N + t) * 4 + q];
      }
      double *o = out + (c * N + t) * PI2_PARTIAL_WIDTH;
      o[0] = m; o[1] = z;
      for (int q = 0; q < 4; ++q) o[2 + q] = v[q];
    }
  return PI2_OK;
}

int pi2_combine_partials_host(const double *partials, int64_t count, int32_t N, double temperature,
                              double *out) {
  if (!partials || !out || count < 1 || N < 1 || !(temperature > 0)) return PI2_ERR_INVALID;
  const double neg_inv = -1.0 / temperature;
  std::vector<double> v((size_t)count * PI2_PARTIAL_WIDTH);
  for (int t = 0; t < N; ++t) {
    for (int64_t i = 0; i < count; ++i)
      for (int c = 0; c < PI2_PARTIAL_WIDTH; ++c)
        v[(size_t)i * PI2_PARTIAL_WIDTH + c] = partials[(i * N + t) * PI2_PARTIAL_WIDTH + c];
    // the device tree: segments of kSeg leaves, then the segment roots
    const int64_t nseg = (count + kSeg - 1) / kSeg;
    std::vector<double> roots((size_t)nseg * PI2_PARTIAL_WIDTH);
    auto tree = [&](double *base, int64_t n) {
      for (int64_t st = 1; st < n; st <<= 1)
        for (int64_t i = 0; i + st < n; i += 2 * st)
          partial_combine(base + i * PI2_PARTIAL_WIDTH, base + (i + st) * PI2_PARTIAL_WIDTH, neg_inv);
    };
    for (int64_t s = 0; s < nseg; ++s) {
      const int64_t cnt = std::min<int64_t>(kSeg, count - s * kSeg);
      tree(v.data() + s * kSeg * PI2_PARTIAL_WIDTH, cnt);
      std::memcpy(&roots[(size_t)s * PI2_PARTIAL_WIDTH], v.data() + s * kSeg * PI2_PARTIAL_WIDTH,
                  sizeof(double) * PI2_PARTIAL_WIDTH);
    }
    tree(roots.data(), nseg);
    std::memcpy(out + (size_t)t * PI2_PARTIAL_WIDTH, roots.data(), sizeof(double) * PI2_PARTIAL_WIDTH);
  }
  return PI2_OK;
}

int pi2_device_noise(pi2_ctx *ctx, int32_t which, uint64_t seed, uint64_t cycle, uint64_t iteration,
                     const double *std_, void *out_host) {
  Range range_("pi2_device_noise");
  if (!ctx || !out_host) return fail(ctx, PI2_ERR_INVALID, "null argument");
  if (which != PI2_STREAM_CONTROL && which != PI2_STREAM_DYNAMICS)
    return fail(ctx, PI2_ERR_INVALID, "unknown noise stream %d", which);
  TRY(bind(ctx));
  cudaStream_t st = ctx->stream;
  pi2_optimize_args a{};
  a.temperature = 1.0;
  a.cost_ceiling = 1e8;
  for (int c = 0; c < 4; ++c) a.exploration_std[c] = std_ ? std_[c] : 1.0;
  a.seed = seed;
  a.cycle = cycle;
  a.iterations = 1;
  CU(cudaEventSynchronize(ctx->staged));
  StepArgs &h = *ctx->h_args;
  for (int c = 0; c < 4; ++c) h.std[c] = a.exploration_std[c];
  h.key_prefix[0] = key_prefix(seed, PI2_STREAM_CONTROL, cycle);
  h.key_prefix[1] = key_prefix(seed, PI2_STREAM_DYNAMICS, cycle);
  CU(cudaMemcpyAsync(ctx->d_args, ctx->h_args, sizeof(StepArgs), cudaMemcpyHostToDevice, st));
  CU(cudaEventRecord(ctx->staged, st));
  const int64_t K = ctx->K, N = ctx->N, M = ctx->M;
  const int64_t n = which == PI2_STREAM_CONTROL ? K * N : K * M * N;
  const size_t bytes = which == PI2_STREAM_CONTROL ? sizeof(double) * n * 4 : sizeof(float) * n * 3;
  TRY(ensure(ctx, &ctx->d_scratch, &ctx->scratch_cap, bytes));
  noise_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      ctx->d_args, which, iteration, K, ctx->dims.rollout_offset, (int)N, (int)M, (double *)ctx->d_scratch,
      (float *)ctx->d_scratch);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(out_host, ctx->d_scratch, bytes, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return PI2_OK;
}

int pi2_lwpr_predict(pi2_ctx *ctx, int32_t axis, int64_t rows, const float *X, float *mean_out,
                     float *var_out) {
  Range range_("pi2_lwpr_predict");
  if (!ctx) return fail(nullptr, PI2_ERR_INVALID, "null context");
  if (axis < 0 || axis > 2 || ctx->axes[axis].L == 0) return fail(ctx, PI2_ERR_INVALID, "no receptive fields");
  if (rows < 1 || !X || !mean_out) return fail(ctx, PI2_ERR_INVALID, "X must have shape (B, input_dim)");
  TRY(bind(ctx));
  const int d = ctx->axes[axis].d;
  cudaStream_t st = ctx->stream;
  std::vector<float4> xp((size_t)rows);
  for (int64_t r = 0; r < rows; ++r) {
    float v[4] = {0, 0, 0, 0};
    for (int i = 0; i < d; ++i) v[i] = X[r * d + i];
    xp[r] = make_float4(v[0], v[1], v[2], v[3]);
  }
  const size_t xb = sizeof(float4) * rows, ob = sizeof(float) * rows;
  TRY(ensure(ctx, &ctx->d_scratch, &ctx->scratch_cap, xb + 2 * ob));
  float4 *dx = (float4 *)ctx->d_scratch;
  float *dm = (float *)(dx + rows), *dv = dm + rows;
  CU(cudaMemcpyAsync(dx, xp.data(), xb, cudaMemcpyHostToDevice, st));
  TRY(launch_lwpr(ctx, axis, axis + 1, rows, dx, dm, var_out ? dv : nullptr, 1, 0, 0, st));
  CU(cudaMemcpyAsync(mean_out, dm, ob, cudaMemcpyDeviceToHost, st));
  if (var_out) CU(cudaMemcpyAsync(var_out, dv, ob, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return PI2_OK;
}

}  // extern "C"

#ifdef PI2_TC_TRACE
// experiments only (trace builds, not in include/pi2rh.h): arm the phase tracer / read it
extern "C" int pi2_debug_trace_arm(int on) {
  const unsigned zero = 0;
  void *buf = nullptr;
  cudaGetSymbolAddress(&buf, pi2::g_tc_trace);
  cudaMemset(buf, 0, sizeof(unsigned long long) * 64 * pi2::kTcTraceCap);
  cudaMemcpyToSymbol(pi2::g_tc_trace_n, &zero, 4);
  cudaMemcpyToSymbol(pi2::g_tc_trace_on, &on, 4);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : -1;
}
extern "C" int pi2_debug_trace_read(unsigned long long *out) {  // 64 * kTcTraceCap entries
  return cudaMemcpyFromSymbol(out, pi2::g_tc_trace, sizeof(unsigned long long) * 64 * pi2::kTcTraceCap) == cudaSuccess ? 0 : -1;
}
#endif
