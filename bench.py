#!/usr/bin/env python
"""PI²-RH control-step benchmark (BASELINE.json metric: rollout-steps/s = K x T LWPR predicts).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A step is one receding-horizon control step with iterations_per_step=1 on the
named workload (default C2: K=65536 rollouts, T=50, L=100 receptive fields per
axis, M=4 sub-rollouts — "uncertainty penalty on"), synthetic
hybrid-LWPR model (paper_1503_00330_b200.synthetic), device-generated noise.

* value: K*T*steps / device time of `steps` back-to-back iterations whose state,
  plan and model are already resident in HBM (CUDA events on the launch stream,
  barrier + synchronize on both sides, max over ranks).
* e2e: the same metric through the public API `receding_horizon_step(...)`
  with host state/plan in and host control/plan out (H2D + D2H inside).
* roofline: the LWPR kernel (dominant) — algorithmic FP32 FLOPs per launch over
  its CUDA-event duration vs the FP32 CUDA-core peak.
* cpu_baseline / --impl reference: the reference algorithm (numpy oracle port,
  oracle/) on the host cores, on a bounded sample of the same workload.

Under torchrun (N > 1) rollouts are sharded across ranks and the per-timestep
softmax partials are all-gathered over NCCL.  Default --scaling weak: every GPU
keeps the named workload's K rollouts (K_total = K x N, the same control step
with N times the samples at the same latency); --scaling strong splits the
named K over the N GPUs (BASELINE C4's framing: K=2^20 on 8 GPUs).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "rollout-steps/sec (K×T LWPR predicts)"
UNIT = "rollout-steps/s"
KERNELS_PER_ITER = 5  # attitude, lwpr, rollout, partials, combine


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="C2")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                   help="N > 1: weak = K rollouts per GPU, strong = K rollouts in total")
    p.add_argument("--cpu-sample", type=int, default=4096, help="rollouts in the CPU baseline sample")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--closed-loop-steps", type=int, default=200,
                   help="control steps of the closed-loop trial (latency p50/p99); 0 disables")
    return p.parse_args()


def workload(name: str):
    from paper_1503_00330_b200.synthetic import CONFIGS

    c = dict(CONFIGS[name])
    desc = {
        "C1": "single PI²-RH control step, K=1024, T=50, L=100, M=1",
        "C2": "quadrotor obstacle-navigation step, K=65536, T=50, L=100, uncertainty on (M=4 sub-rollouts)",
        "C3": "large LWPR L=1000, K=262144, T=100, M=1",
        "C4": "K=2^20, T=50, L=100, M=1 control step",
        "C5": "K=2^22, T=50, L=200, M=1",
    }[name]
    return c, desc


# ---------------------------------------------------------------- CPU reference
def cpu_reference(cfgd, sample_k: int, min_seconds: float, max_steps: int | None = None):
    """Reference algorithm (oracle port) on the host cores: one optimisation iteration
    (sample_noise [+ dyn] + evaluate + update) per step on a bounded sample."""
    from threadpoolctl import threadpool_limits

    from oracle import rollout as RO
    from paper_1503_00330_b200 import synthetic

    T, L, M = cfgd["T"], cfgd["L"], cfgd["M"]
    k = min(sample_k, cfgd["K"])
    workers = RO.default_workers()
    chunk = min(1024, -(-k // workers))
    model = RO.Model(synthetic.hybrid_stacks(L, seed=0))
    cost = RO.Cost(synthetic.DEFAULT_WAYPOINTS[1], synthetic.DEFAULT_OBSTACLES)
    state = np.zeros(12)
    state[0:3] = synthetic.DEFAULT_WAYPOINTS[0]
    plan = np.tile([0.0, 0.0, 0.0, model.dyn.hover_thrust], (T, 1))
    times = []
    with threadpool_limits(1, "blas"):
        RO.optimize(model, state, plan, cost, K=k, M=M, iterations=1, chunk=chunk, workers=workers)  # warm-up
        t_all = time.perf_counter()
        cyc = 0
        while True:
            t0 = time.perf_counter()
            RO.optimize(model, state, plan, cost, K=k, M=M, iterations=1, chunk=chunk, workers=workers,
                        cycle=cyc)
            times.append(time.perf_counter() - t0)
            cyc += 1
            if max_steps is not None and cyc >= max_steps:
                break
            if max_steps is None and (time.perf_counter() - t_all >= min_seconds and cyc >= 2):
                break
    step = statistics.median(times)
    return {
        "value": k * T / step,
        "unit": UNIT,
        "cores": workers,
        "kind": "port",
        "sample": f"K={k} of {cfgd['K']} rollouts, T={T}, L={L}, M={M}; numpy oracle (oracle/rollout.py), "
                  f"{workers} worker threads, BLAS 1 thread; median of {len(times)} steps "
                  f"(noise + evaluate + update)",
        "ms_per_step": step * 1e3,
        "step_times_s": times,
    }


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock, max clock and throttle reasons sampled DURING the timed region.

    NVML (nvidia_ml_py) is polled every ~2 ms from a thread, so even a
    millisecond-scale timed region gets samples; only samples between mark_start()
    and mark_end() (the caller's timed window) are summarised.  Falls back to
    `nvidia-smi -lms 100` when NVML is unavailable."""

    REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples: list[tuple] = []  # (t, sm_mhz, max_mhz, reasons)
        self.t0 = self.t1 = None
        self._stop = threading.Event()
        self.proc = self.thread = None
        self.source = None

    def mark_start(self):
        self.t0 = time.monotonic()

    def mark_end(self):
        self.t1 = time.monotonic()

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            bits = (pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self._stop.is_set():
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((time.monotonic(), float(sm), float(mx),
                                         tuple(n for n, b in zip(self.REASONS, bits) if r & b)))
                    time.sleep(0.002)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            self.source = "nvml"
            return self
        except Exception:  # noqa: BLE001 - no NVML: nvidia-smi
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read_smi, daemon=True)
            self.thread.start()
            self.source = "nvidia-smi"
        except OSError:
            self.proc = None
        return self

    def _read_smi(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            try:
                sm, mx = float(parts[0]), float(parts[1])
            except (ValueError, IndexError):
                continue
            reasons = tuple(n for n, v in zip(self.REASONS, parts[4:8]) if v.lower().startswith("active"))
            self.samples.append((time.monotonic(), sm, mx, reasons))

    def __exit__(self, *exc):
        self._stop.set()
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=1)

    def summary(self):
        inside = [s for s in self.samples if self.t0 is not None and self.t1 is not None and self.t0 <= s[0] <= self.t1]
        use = inside or self.samples
        if not use:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": self.source}
        reasons = sorted({r for s in use for r in s[3]})
        return {"sm_mhz": statistics.median(s[1] for s in use), "sm_max_mhz": max(s[2] for s in use),
                "reasons": reasons, "samples": len(use), "in_timed_region": bool(inside), "source": self.source}


# ---------------------------------------------------------------- ours
def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def lwpr_traffic(config: str, tc: bool):
    """dram bytes per LWPR launch from a committed `ncu --set full` capture, if any."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "lwpr_traffic.json")))
        return d.get(config + ("_tc" if tc else ""))
    except (OSError, ValueError):
        return None


def run_ours(args, rank: int, world: int, local: int):
    import torch

    import paper_1503_00330_b200 as P
    from paper_1503_00330_b200 import _abi, synthetic
    from paper_1503_00330_b200.controller import dynamics_struct, optimize_args
    from paper_1503_00330_b200.simworld import cost_struct

    dist = None
    # one rank per GPU; PI2_DIST_BACKEND=gloo lets several ranks share a GPU to
    # exercise the multi-rank path where only one GPU exists (timings meaningless)
    backend = os.environ.get("PI2_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    cfgd, desc = workload(args.config)
    if args.scaling == "weak":
        cfgd["K"] *= world
    K, T, L, M = cfgd["K"], cfgd["T"], cfgd["L"], cfgd["M"]
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(synthetic.hybrid_stacks(L, seed=0), params)
    task = P.Task.default()
    cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=T, iterations_per_step=1, rng_seed=0)
    state = P.QuadState.hover(task.spawn)
    plan0 = P.ControlPlan.hover(params, T)
    cost = P.RolloutCost(task, 1)
    stream = torch.cuda.Stream(device=local)  # dedicated stream: kernels, events and NCCL share it
    torch.cuda.set_stream(stream)
    sptr = _abi.torch_stream(local)

    if world > 1:
        from paper_1503_00330_b200.distributed import ShardedEngine, gather_partials

        eng = ShardedEngine(model, cfg, device=local)
        ctx = eng.ctx
        k_local = eng.stop - eng.start
    else:
        eng = P.RolloutEngine(model, cfg, device=local, noise="device", use_graph=True)
        ctx = eng.context(K, T)
        k_local = K
    ctx.call("pi2_set_dynamics", dynamics_struct(params, plan0.lo, plan0.hi))
    ctx.call("pi2_set_cost", cost_struct(cost))
    ctx.call("pi2_load_plan", _abi.ptr(state.as_array()), _abi.ptr(np.ascontiguousarray(plan0.controls)), sptr)
    partial = torch.empty((T, _abi.PARTIAL_WIDTH), dtype=torch.float64, device=f"cuda:{local}")

    def device_step(cycle):
        if world == 1:  # the whole iteration as one CUDA graph on the device-resident plan
            ctx.call("pi2_iterate_device", optimize_args(cfg, cycle, use_graph=True), sptr)
            return
        a = optimize_args(cfg, cycle, use_graph=False)
        ctx.call("pi2_iterate_local", a, 0, _abi.ptr(partial), sptr)
        g = gather_partials(partial)
        ctx.call("pi2_iterate_finalize", _abi.ptr(g), world, float(cfg.temperature), sptr)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident throughput (value)
    for w in range(args.warmup):
        device_step(10_000 + w)
    barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        clocks.mark_start()
        start.record(stream)
        for s in range(args.steps):
            device_step(s)
        end.record(stream)
        while not end.query():  # a sleeping wait keeps the GIL free for the clock sampler
            time.sleep(0.0005)
        barrier()
        clocks.mark_end()
    dev_ms = max_over_ranks(start.elapsed_time(end))
    ms_per_step = dev_ms / args.steps
    value = K * T * args.steps / (dev_ms / 1e3)

    # ---- stage profile (dominant kernel = LWPR), CUDA events on the context stream
    stage_ms = (_abi.C.c_double * 5)()
    ctx.call("pi2_profile_iteration", optimize_args(cfg, 0, use_graph=False), 10, stage_ms)
    stages = dict(zip(["attitude", "lwpr", "rollout_cost", "partials", "combine"], list(stage_ms)))

    # ---- end to end through the public API (host state/plan in, control/plan out)
    plan = plan0
    lat = []
    if world > 1:
        for w in range(args.warmup):
            eng.optimize(state, plan, cost, 10_000 + w)
        barrier()
        for s in range(args.steps):
            t0 = time.perf_counter()
            opt = eng.optimize(state, plan, cost, s)
            ctrl, plan = opt.control_at(0), opt.shifted()
            lat.append(time.perf_counter() - t0)
    else:
        for w in range(args.warmup):
            P.receding_horizon_step(state, plan0, cfg, model, cost, 10_000 + w, eng)
        barrier()
        for s in range(args.steps):
            t0 = time.perf_counter()
            ctrl, plan = P.receding_horizon_step(state, plan, cfg, model, cost, s, eng)
            lat.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(sum(lat))
    lat_ms = sorted(x * 1e3 for x in lat)
    p50 = max_over_ranks(statistics.median(lat_ms))
    p99 = max_over_ranks(lat_ms[min(len(lat_ms) - 1, math.ceil(0.99 * len(lat_ms)) - 1)])

    if rank != 0:
        return None

    peaks = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    n_sm = torch.cuda.get_device_properties(local).multi_processor_count
    peak_tflops = n_sm * 128 * 2 * sm_max * 1e6 / 1e12
    rows = k_local * T
    flops_per_field = 32 if M > 1 else 27  # 27 (+5 variance) per (row, axis, field)
    lwpr_flops = rows * 3 * L * flops_per_field
    achieved = lwpr_flops / (stages["lwpr"] / 1e3) / 1e12
    # which LWPR kernel ran: the tcgen05 one for the variance path unless disabled
    # which LWPR kernel ran, and the share of its 2^x on MUFU (the rest on the FMA pipe)
    kern, share = _abi.C.c_int32(), _abi.C.c_double()
    ctx.call("pi2_lwpr_kernel", int(M > 1), _abi.C.byref(kern), _abi.C.byref(share))
    tc = kern.value == 1
    exps = rows * 3 * L  # one 2^x per (row, axis, field)
    mufu_peak = float(peaks.get("mufu_ex2_per_s", 4.60e12))
    lw_s = stages["lwpr"] / 1e3
    clk = clocks.summary()
    peak_obs = n_sm * 128 * 2 * clk["sm_mhz"] * 1e6 / 1e12 if clk.get("sm_mhz") else None
    h2d = 12 * 8 + T * 4 * 8 + 8 * (12 + 4 * 16 + 4 + 2) + 4 * 48  # state + plan + StepArgs
    d2h = T * 4 * 8
    fp32 = {
        "achieved": achieved, "peak": peak_tflops, "unit": "TFLOP/s", "frac": achieved / peak_tflops,
        "peak_source": f"{n_sm} SMs x 128 FP32 lanes x 2 x sm_max_mhz {sm_max:.0f} (MEASURED_PEAKS.json)",
        "frac_at_observed_clock": (achieved / peak_obs) if peak_obs else None,
        "flops_per_launch": lwpr_flops, "flops_per_field": flops_per_field,
    }
    mufu = {"ex2_per_launch": exps, "mufu_share": share.value,
            "achieved": exps * share.value / lw_s / 1e12, "peak": mufu_peak / 1e12, "unit": "Tex2/s",
            "frac": exps * share.value / lw_s / mufu_peak,
            "peak_source": "profiles/micro/mufu_mix_b200.txt (MUFU-only ex2 stream, 148 SMs)"}
    if tc:  # binding unit: MUFU (the linear parts are on the tensor cores)
        roofline = {"bound": "mufu", "kernel": "lwpr_tc_kernel (tcgen05 3xTF32 field GEMM + exp/moments)",
                    **{k: mufu[k] for k in ("achieved", "peak", "unit", "frac", "peak_source")},
                    "ex2_per_launch": exps, "mufu_share": share.value,
                    "traffic": lwpr_traffic(args.config, tc) if world == 1 else None,
                    "fp32_equivalent": {**fp32, "note": "the same algorithmic FLOPs against the FP32 CUDA-core "
                                        "peak; above 1 when the tensor cores carry the linear parts"}}
    else:
        roofline = {"bound": "fp32", "kernel": "lwpr_kernel (CUDA cores, FFMA2)", **fp32,
                    "traffic": lwpr_traffic(args.config, tc) if world == 1 else None, "mufu": mufu}
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "f32 (LWPR: linear parts as 3xTF32 tcgen05 products with f32 accumulation, exp/moments f32; "
                 "integration, cost) + f64 (attitude, cost-to-go, update)",
        "data": "synthetic (seeded hybrid-LWPR model linearising the rigid-body quadrotor; device Philox noise)",
        "config": {
            "workload": f"{args.config}: {desc}" + (f" (x{world} GPUs, weak scaling: K per GPU)"
                                                    if world > 1 and args.scaling == "weak" else ""),
            "K": K, "K_per_gpu": k_local, "T": T, "L": L, "M": M, "iterations_per_step": 1,
            "parallelism": f"rollouts sharded over {world} GPU(s)",
            "l2": "working set > L2 (xin + LWPR planes + exploration normals + costs ≈ %.0f MB per GPU)"
                  % ((k_local * T * (16 + 24 + 16 + 8)) / 1e6),
        },
        "e2e": {
            "value": K * T * args.steps / e2e_s,
            "unit": UNIT,
            "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h,
            "api": "paper_1503_00330_b200.receding_horizon_step(noise='device' engine)" if world == 1
                   else "distributed.ShardedEngine.optimize",
        },
        "latency_ms": {"p50": p50, "p99": p99, "what": "e2e control step (host state/plan -> control)"},
        "roofline": roofline,
        "stages_ms": stages,
        "clocks": clk,
        "gpu_launches": args.steps * (KERNELS_PER_ITER + (1 if world > 1 else 0)),
    }
    if world == 1 and args.closed_loop_steps > 0:
        gt = P.PerturbedModel(params, drag_coeff=0.08, thrust_scale=0.97)
        trial = P.run_trial(task, P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=T, iterations_per_step=1),
                            model, gt, seed=0, step_cap=args.closed_loop_steps, noise="device", device=local)
        raw = np.asarray(trial.step_latency_s) * 1e3
        tl = np.sort(raw[1:]) if len(raw) > 1 else np.sort(raw)  # steady state: after the setup step
        line["closed_loop"] = {
            "what": "simworld.run_trial with device noise: latency of each receding_horizon_step (host state in, "
                    "control out); plant = PerturbedModel(drag 0.08, thrust x0.97)",
            "steps": int(trial.steps), "outcome": trial.outcome,
            "p50_ms": float(np.median(tl)), "p99_ms": float(tl[min(len(tl) - 1, math.ceil(0.99 * len(tl)) - 1)]),
            "max_ms": float(tl[-1]), "budget_ms": 20.0,
            "first_step_ms": float(raw[0]) if len(raw) else None,
            "first_step": "context creation, weight staging and CUDA graph capture; p50/p99/max cover the later steps",
        }
    if world == 1 and not args.no_cpu_baseline:
        cb = cpu_reference(cfgd, args.cpu_sample, args.cpu_seconds)
        cb.pop("step_times_s", None)
        cb["cpu_model"] = cpu_model()
        line["cpu_baseline"] = cb
    return line


def run_reference(args, world: int = 1):
    cfgd, desc = workload(args.config)
    if args.scaling == "weak":
        cfgd["K"] *= world  # the same config as our arm; the CPU sample below is bounded anyway
    cb = cpu_reference(cfgd, args.cpu_sample, 0.0, max_steps=args.warmup + args.steps)
    times = cb.pop("step_times_s")[args.warmup:] or [cb["ms_per_step"] / 1e3]
    step = sum(times) / len(times)
    k = min(args.cpu_sample, cfgd["K"])
    value = k * cfgd["T"] / step
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": 0,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": step * 1e3,
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "f32 + f64 (numpy)",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {desc}", **cfgd, "iterations_per_step": 1},
        "cpu_baseline": {**cb, "value": value, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, world)), flush=True)
        return 0
    line = run_ours(args, rank, world, local)
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
