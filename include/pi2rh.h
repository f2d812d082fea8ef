/*
 * pi2rh.h — C ABI of the B200-native PI²-RH control step.
 *
 * The reference (pimpc, pure Python/numpy) has no native boundary: its
 * drop-in seams are duck-typed Python protocols.  Each
 * entry point below replaces one of them; the comment on each cites the
 * reference interface (file:line, relative to /root/reference/pkg/src/pimpc)
 * whose behaviour it reproduces.  The ctypes binding the Python host layer
 * uses (paper_1503_00330_b200/_abi.py) is shown in INTEGRATION.md.
 *
 * Conventions
 *   - Every call returns an int status (PI2_OK == 0) and never throws;
 *     pi2_last_error() gives the message of the last failure on a context.
 *   - The context owns all device buffers it allocates.  Caller pointers are
 *     borrowed for the duration of the call.  "_device" variants take device
 *     pointers (e.g. torch tensor data_ptr()) and a cudaStream_t passed as
 *     void* (NULL = the context's own stream); the others take HOST buffers
 *     and include the host<->device copies.
 *   - Arrays are C-contiguous, float64 unless stated, shapes as in the
 *     reference: noise (K, N, 4), dyn_noise (K, M, N, 3) float32,
 *     costs (K, N), crash flags (K,) uint8, plan (N, 4), state (12,) =
 *     [position, velocity, angles, rates] (dynamics.py:79-110).
 *   - One context per host thread; a context is bound to one CUDA device.
 */
#ifndef PI2RH_H
#define PI2RH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PI2_ABI_VERSION 1
#define PI2_MAX_OBSTACLES 16
#define PI2_MAX_SUB_ROLLOUTS 256
#define PI2_PARTIAL_WIDTH 6 /* (min S, Z, V[4]) per timestep, float64 */

/* status codes */
#define PI2_OK 0
#define PI2_ERR_INVALID 1     /* bad argument (reference: ValueError)          */
#define PI2_ERR_STATE 2       /* call order / missing model or cost             */
#define PI2_ERR_UNSUPPORTED 3 /* plugin the device path cannot run (TypeError)  */
#define PI2_ERR_CUDA 4        /* CUDA runtime failure                           */
#define PI2_ERR_OOM 5         /* device allocation failed                       */

/* model plugins (RolloutEngine model protocol, controller.py:169-173) */
#define PI2_MODEL_NONE 0
#define PI2_MODEL_HYBRID_LWPR 1 /* HybridModel, dynamics.py:214-277             */
#define PI2_MODEL_ANALYTIC 2    /* AnalyticModel, dynamics.py:152-187           */
#define PI2_MODEL_TWO_POINT 3   /* tests/synthetic.py:17-40 (noise_transform=sign) */

/* cost plugins (simworld.py:157-198, tests/synthetic.py:43-53) */
#define PI2_COST_NAVIGATION 0 /* RolloutCost */
#define PI2_COST_THRESHOLD 1  /* ThresholdCost */

/* noise streams (rng.py:19-21) */
#define PI2_STREAM_CONTROL 1
#define PI2_STREAM_DYNAMICS 2

typedef struct pi2_ctx pi2_ctx;

/* Shapes fixed for the life of a context (RolloutEngine.__init__,
 * controller.py:176-185).  A multi-GPU shard evaluates rollouts
 * [rollout_offset, rollout_offset + num_rollouts) of num_rollouts_total. */
typedef struct pi2_dims {
  int64_t num_rollouts;       /* K of this context                      */
  int64_t rollout_offset;     /* global index of its first rollout      */
  int64_t num_rollouts_total; /* global K (0 = num_rollouts)            */
  int32_t horizon_steps;      /* N (<= 524280)                          */
  int32_t sub_rollouts;       /* M (1..PI2_MAX_SUB_ROLLOUTS)            */
} pi2_dims;

/* QuadParams (dynamics.py:32-62) plus the ControlPlan clip bounds
 * (control_bounds, dynamics.py:53-57; ControlPlan.__post_init__ :39-45). */
typedef struct pi2_dynamics {
  double mass, gravity, rate_gain, dt;
  double lo[4], hi[4];
} pi2_dynamics;

/* RolloutCost bound to one waypoint (simworld.py:141-146), float32 like the
 * reference; or ThresholdCost (tests/synthetic.py:43-53). */
typedef struct pi2_cost {
  int32_t kind;        /* PI2_COST_*                        */
  int32_t n_obstacles; /* <= PI2_MAX_OBSTACLES              */
  float waypoint[3];
  float z_floor;
  float arena_lo[3];
  float arena_hi[3];
  float obstacles[2 * PI2_MAX_OBSTACLES]; /* (x, y) pairs */
  float threshold; /* PI2_COST_THRESHOLD: stage cost = (z > threshold) */
  /* Opt-in uncertainty penalty kappa >= 0 (an EXTENSION: the reference's cost
   * has no variance term, simworld.py:166-198; parity unpinned,
   * default 0 = the reference).  With kappa > 0 and the hybrid LWPR model the
   * sub-rollout-mean stage cost of rollout k at step t gains
   * kappa * (sd_x^2 + sd_y^2 + sd_z^2), float32, from the LWPR predictive
   * standard deviations of that rollout-step (dynamics.py:274-275). */
  float variance_penalty;
} pi2_cost;

/* PiConfig fields consumed by optimize (controller.py:72-100, 374-395). */
typedef struct pi2_optimize_args {
  double temperature;
  double cost_ceiling;
  double exploration_std[4];
  uint64_t seed;
  uint64_t cycle;
  int32_t iterations; /* >= 0; keys are derived per iteration on the device */
  int32_t use_graph;  /* capture/replay the whole step as one CUDA graph */
} pi2_optimize_args;

/* ---- library ---------------------------------------------------------- */
int pi2_version(void);
const char *pi2_strerror(int status);
int pi2_device_count(int32_t *count);

/* ---- context (RolloutEngine.__init__ / _workspace, controller.py:142-195) */
int pi2_create(int32_t device, const pi2_dims *dims, pi2_ctx **out);
void pi2_destroy(pi2_ctx *ctx);
const char *pi2_last_error(const pi2_ctx *ctx);
int pi2_get_dims(const pi2_ctx *ctx, pi2_dims *out);

/* ---- plugins ------------------------------------------------------------ */
/* QuadParams + plan bounds; dynamics.py:32-62. */
int pi2_set_dynamics(pi2_ctx *ctx, const pi2_dynamics *dyn);
/* One axis of a HybridModel: the raw receptive-field stacks of
 * LwprModel._stacks() (lwpr.py:141-150) — centers (L,d), metrics (L,d,d),
 * coefs (L,d+1), local_variance (L) — folded on the host exactly as
 * FrozenLwpr.__init__ does (lwpr.py:339-358), then staged to HBM.
 * input_dim d in 1..4 (HybridModel needs 4, dynamics.py:226-228). */
int pi2_set_lwpr_axis(pi2_ctx *ctx, int32_t axis, int32_t num_fields, int32_t input_dim,
                      const double *centers, const double *metrics, const double *coefs,
                      const double *local_variance);
/* Select the model plugin.  HYBRID_LWPR needs all 3 axes set (else the
 * reference's "untrained" ValueError, dynamics.py:232-235); TWO_POINT takes
 * the magnitude in `param`. */
int pi2_select_model(pi2_ctx *ctx, int32_t kind, double param);
/* RolloutCost / ThresholdCost; simworld.py:141-146. */
int pi2_set_cost(pi2_ctx *ctx, const pi2_cost *cost);
/* The navigation cost's full obstacle list, any length (RolloutCost.obstacles,
 * simworld.py:141-146, has no limit; pi2_cost holds PI2_MAX_OBSTACLES): (n, 2)
 * float32 (x, y), summed in list order like simworld.py:188-190.  Call after
 * pi2_set_cost (which resets the list to the struct's).  When the part past
 * the struct changes, the call synchronises the device before restaging it. */
int pi2_set_cost_obstacles(pi2_ctx *ctx, int32_t n, const float *obstacles_xy);

/* ---- hot path ----------------------------------------------------------- */
/* RolloutEngine.evaluate (controller.py:197-247): perturb + clip, FP64
 * attitude, LWPR (or analytic) accelerations, FP32 integration, cost,
 * sub-rollout mean, FP64 suffix sum, non-finite -> cost_ceiling + crash.
 * HOST buffers.  dyn_noise is required iff the model is probabilistic and
 * M > 1 (controller.py:210-211). */
int pi2_evaluate(pi2_ctx *ctx, const double *state, const double *plan, const double *noise,
                 const float *dyn_noise, double cost_ceiling, double *costs_out,
                 uint8_t *crash_out);
/* Same with DEVICE noise / outputs (state and plan stay host arrays). */
int pi2_evaluate_device(pi2_ctx *ctx, const double *state, const double *plan,
                        const double *noise_dev, const float *dyn_noise_dev, double cost_ceiling,
                        double *costs_dev, uint8_t *crash_dev, void *stream);

/* RolloutEngine.evaluate on the DEVICE noise streams of (seed, cycle,
 * iteration) that pi2_optimize draws (the same kernels as one optimisation
 * iteration, without the update): costs (K,N) and crash flags (K,) to DEVICE
 * buffers.  The noise itself is pi2_device_noise's output. */
int pi2_evaluate_device_noise(pi2_ctx *ctx, const double *state, const double *plan,
                              const pi2_optimize_args *args, int32_t iteration, double *costs_dev,
                              uint8_t *crash_dev, void *stream);
/* path_integral_update (controller.py:356-371) for an arbitrary batch:
 * per-timestep min-shifted softmax of -costs/temperature, weighted noise sum,
 * clip to the plan bounds.  HOST buffers; K may differ from the context's. */
int pi2_update(pi2_ctx *ctx, int64_t num_rollouts, int32_t horizon_steps, const double *plan,
               const double *costs, const double *noise, double temperature, double *plan_out);
int pi2_update_device(pi2_ctx *ctx, int64_t num_rollouts, int32_t horizon_steps,
                      const double *plan, const double *costs_dev, const double *noise_dev,
                      double temperature, double *plan_out, void *stream);

/* optimize (controller.py:374-395) with device-generated exploration and
 * dynamics noise (Philox4x32-10 + Box-Muller keyed by the reference's
 * splitmix64 stream address, rng.py:33-44).  plan_inout (N,4) HOST. */
int pi2_optimize(pi2_ctx *ctx, const double *state, double *plan_inout,
                 const pi2_optimize_args *args);
/* The optimise loop on the device-resident plan (set by pi2_load_plan, read
 * back by pi2_read_plan): no host transfers or synchronisation, replayed as
 * one CUDA graph when args->use_graph. */
int pi2_iterate_device(pi2_ctx *ctx, const pi2_optimize_args *args, void *stream);
/* receding_horizon_step (controller.py:398-413): optimize, return the first
 * control (4,) and replace plan_inout by the shifted plan (:63-66). */
int pi2_receding_horizon_step(pi2_ctx *ctx, const double *state, double *plan_inout,
                              const pi2_optimize_args *args, double *control_out);

/* ---- multi-GPU split of one optimisation iteration ----------------------
 * Rank r owns rollouts [rollout_offset, +num_rollouts).  Per iteration:
 *   pi2_iterate_local      -> rank partial (N x PI2_PARTIAL_WIDTH f64, device)
 *   all-gather of partials (NCCL via torch.distributed, done by the caller)
 *   pi2_iterate_finalize   -> fixed-order combine + plan update (device)
 * The plan lives on the device between pi2_load_plan and pi2_read_plan. */
int pi2_load_plan(pi2_ctx *ctx, const double *state, const double *plan, void *stream);
int pi2_read_plan(pi2_ctx *ctx, double *plan_out, void *stream);
int pi2_iterate_local(pi2_ctx *ctx, const pi2_optimize_args *args, int32_t iteration,
                      double *rank_partial_dev, void *stream);
int pi2_iterate_finalize(pi2_ctx *ctx, const double *gathered_partials_dev, int32_t world_size,
                         double temperature, void *stream);
/* A rank's whole control step as one CUDA graph that the CALLER captures (the
 * NCCL all-gather sits between the kernels), replacing the per-call staging and
 * host synchronisation of pi2_iterate_local / pi2_load_plan / pi2_read_plan
 * (controller.py:374-395 split at the update's reduction, controller.py:367-371):
 *   pi2_stage_step            host only: state, keys, cost, plan -> pinned block
 *                             (after the previous step's pi2_fetch_plan)
 *   --- captured once, replayed every step on `stream` ---
 *   pi2_enqueue_pull          pinned block -> device (args + plan)
 *   per iteration:
 *     pi2_iterate_local_staged   -> rank partial (device)
 *     all-gather of the partials (caller, e.g. torch.distributed NCCL)
 *     pi2_iterate_finalize       -> combine + plan update (device)
 *   pi2_enqueue_push          device plan -> pinned block
 *   ---
 *   pi2_fetch_plan            synchronise `stream`, copy the plan out (host)
 * The enqueue calls never synchronise or allocate, so they are capturable. */
int pi2_stage_step(pi2_ctx *ctx, const double *state, const double *plan, const pi2_optimize_args *args);
int pi2_enqueue_pull(pi2_ctx *ctx, void *stream);
int pi2_iterate_local_staged(pi2_ctx *ctx, int32_t iteration, double temperature, double *rank_partial_dev,
                             void *stream);
int pi2_enqueue_push(pi2_ctx *ctx, void *stream);
int pi2_fetch_plan(pi2_ctx *ctx, double *plan_out, void *stream);
/* The same fixed-order partial combine on the host (no GPU needed):
 * partials (count, N, PI2_PARTIAL_WIDTH) -> out (N, PI2_PARTIAL_WIDTH). */
int pi2_combine_partials_host(const double *partials, int64_t count, int32_t horizon_steps,
                              double temperature, double *out);
/* Chunk partials of one batch on the host: costs (K,N), noise (K,N,4) ->
 * (ceil(K/chunk), N, PI2_PARTIAL_WIDTH); the leaf rule of the device path. */
int pi2_chunk_partials_host(const double *costs, const double *noise, int64_t num_rollouts,
                            int32_t horizon_steps, double temperature, double *out);
int64_t pi2_partial_chunk(void); /* rollouts per leaf partial */

/* Stage timing of one device-noise iteration on the plan loaded with
 * pi2_load_plan: CUDA events on the context stream around each kernel,
 * averaged over `reps` (plan not updated).  stage_ms[5] = attitude, LWPR,
 * rollout/cost, partials, combine (ms). */
int pi2_profile_iteration(pi2_ctx *ctx, const pi2_optimize_args *args, int32_t reps, double *stage_ms);
/* Stage timing of the host-noise evaluate path (pi2_evaluate_device on DEVICE
 * copies of the reference's noise streams, controller.py:112-139, 197-247):
 * stage_ms[3] = attitude (reads the (K,N,4) f64 exploration noise), LWPR,
 * rollout/cost (reads the (K,M,N,3) f32 dynamics noise when M > 1), averaged
 * over `reps`.  Benchmark introspection: the noise-stream HBM bandwidth. */
int pi2_profile_evaluate(pi2_ctx *ctx, const double *state, const double *plan, const double *noise_dev,
                         const float *dyn_dev, int32_t reps, double *stage_ms);
/* Which LWPR kernel the rollout path of this context runs for the staged
 * model (variance != 0: the sub-rollout path with standard deviations):
 * *kernel_out = PI2_LWPR_CUDA_CORES or PI2_LWPR_TENSOR_CORES; *mufu_share
 * (may be NULL) = fraction of its 2^x evaluated on the MUFU unit (the rest
 * on the FMA pipe).  Benchmark introspection. */
#define PI2_LWPR_CUDA_CORES 0
#define PI2_LWPR_TENSOR_CORES 1
int pi2_lwpr_kernel(pi2_ctx *ctx, int32_t variance, int32_t *kernel_out, double *mufu_share);
/* Whether this context's device-noise iterations run the fused step kernel
 * (attitude + LWPR + rollout/cost in one kernel, csrc/fused.cuh; opt-in with
 * the environment variable PI2_FUSED=1 at pi2_create, and only for eligible
 * models, costs and sizes): *sub_rollouts_out = its per-thread sub-rollout
 * template (1, 2 or 4), 0 when the unfused kernels run.  Introspection. */
int pi2_fused_step(pi2_ctx *ctx, int32_t *sub_rollouts_out);

/* ---- noise / LWPR building blocks ------------------------------------- */
/* Device noise for stream (seed, stream_id, cycle, iteration): control
 * noise (K,N,4) f64 scaled by std (stream_id == PI2_STREAM_CONTROL) or
 * standard normals (K,M,N,3) f32 (PI2_STREAM_DYNAMICS), written to HOST. */
int pi2_device_noise(pi2_ctx *ctx, int32_t stream_id, uint64_t seed, uint64_t cycle,
                     uint64_t iteration, const double *std, void *out_host);
/* FrozenLwpr.predict_into (lwpr.py:369-407) for one staged axis:
 * X (rows, input_dim) f32 HOST -> mean (rows,), variance (rows,) or NULL. */
int pi2_lwpr_predict(pi2_ctx *ctx, int32_t axis, int64_t rows, const float *X, float *mean_out,
                     float *var_out);

#ifdef __cplusplus
}
#endif
#endif /* PI2RH_H */
