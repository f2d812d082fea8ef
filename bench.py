#!/usr/bin/env python
"""PI²-RH control-step benchmark (BASELINE.json metric: rollout-steps/s = K x T LWPR predicts,
and control-step latency p50 at 1/2/4/8 B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A step is one receding-horizon control step with iterations_per_step=1 on the
named workload (default C2 = BASELINE configs[1]: K=65536 rollouts, T=50, L=100
receptive fields per axis, M=4 sub-rollouts — "uncertainty penalty on", SURVEY.md
§0.6), synthetic hybrid-LWPR model (paper_1503_00330_b200.synthetic),
device-generated noise.

* value: K*T*steps / device time of `steps` back-to-back graph-replayed steps whose
  state, plan and model are resident in HBM (CUDA events on the launch stream,
  barrier + synchronize on both sides, max over ranks).
* e2e: the same metric through the public API — `receding_horizon_step(...)` at
  N=1, `distributed.ShardedEngine.optimize` at N>1 — host state/plan in, host
  control/plan out (H2D + D2H inside the timed region).
* roofline: the LWPR kernel (dominant): algorithmic 2^x per second over its
  CUDA-event duration against the measured MUFU ex2 peak.
* north_star: BASELINE C4 (K=2^20, T=50, L=100, M=1) on the same GPUs (strong
  scaling): device ms/step, e2e p50/p99 against the 20 ms budget, the closed-loop
  trial of the reference's own run_trial with this engine dropped in (N=1), and
  at N>1 the speed-up over the same step on one GPU measured in the same run.
* noise_stream: the host-noise path's exploration / dynamics noise streams
  (controller.py:112-139) read by the attitude / rollout kernels, in GB/s.
* cpu_baseline / --impl reference: the reference's own CPU implementation
  (`pimpc` installed in baseline/_ref; the numpy oracle port if it is absent) on
  the host cores.  --impl reference runs the FULL configured K.

N > 1: one process per GPU.  When WORLD_SIZE is unset, `--gpus N` re-launches
itself under torch.distributed.run.  Rollouts are sharded across ranks (default
--scaling strong: the named K split over the N GPUs; weak: K per GPU) and the
per-timestep softmax partials are all-gathered over NCCL inside each rank's
captured CUDA graph.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
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
BUDGET_MS = 20.0      # the receding-horizon real-time budget (north star)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="C2")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                   help="N > 1: strong = the named K split over the GPUs, weak = K rollouts per GPU")
    p.add_argument("--cpu-sample", type=int, default=4096, help="rollouts in the cpu_baseline sample")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--ref-budget-s", type=float, default=150.0,
                   help="--impl reference: wall-clock budget of the timed steps (full K each)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-north-star", action="store_true")
    p.add_argument("--no-other-configs", action="store_true",
                   help="N=1: skip the short measurements of the other BASELINE configs (C1, C3, C5 + K sweep)")
    p.add_argument("--closed-loop-steps", type=int, default=500,
                   help="north star: control steps of the closed-loop trial (BASELINE C4: 500); 0 disables")
    return p.parse_args()


def workload(name: str, world: int, scaling: str):
    from paper_1503_00330_b200.synthetic import CONFIGS

    c = dict(CONFIGS[name])
    desc = {
        "C1": "single PI²-RH control step, K=1024, T=50, L=100, M=1",
        "C2": "quadrotor obstacle-navigation step, K=65536, T=50, L=100, uncertainty on (M=4 sub-rollouts)",
        "C3": "large LWPR L=1000, K=262144, T=100, M=1",
        "C4": "K=2^20, T=50, L=100, M=1 control step",
        "C5": "K=2^22, T=50, L=200, M=1",
    }[name]
    if scaling == "weak":
        c["K"] *= world
        if world > 1:
            desc += f" (x{world} GPUs, weak scaling: K per GPU)"
    return c, f"{name}: {desc}"


def config_dict(cfgd, desc):
    """The `config` object of both arms' lines (identical for the same workload)."""
    k = cfgd["K"]
    return {"workload": desc, "K": k, "T": cfgd["T"], "L": cfgd["L"], "M": cfgd["M"], "iterations_per_step": 1,
            "l2": "working set > L2: rows + LWPR planes + normals + costs = %.0f MB" % (k * cfgd["T"] * 64 / 1e6)}


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn(args) -> int:
    """--gpus N without a launcher: one process per GPU under torch.distributed.run."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


# ---------------------------------------------------------------- CPU reference
class ThreadLocalCost:
    """One reference RolloutCost per worker thread.  The reference's RolloutCost keeps
    per-shape scratch buffers that its worker threads share (simworld.py:149-155, a race
    when workers > 1); this harness-side proxy gives each thread its own."""

    def __init__(self, ref, task, waypoint):
        self.ref, self.task, self.waypoint, self._tl = ref, task, waypoint, threading.local()

    def _cost(self):
        c = getattr(self._tl, "c", None)
        if c is None:
            c = self._tl.c = self.ref.simworld.RolloutCost(self.task, self.waypoint)
        return c

    def crash_now(self, pos, out):
        self._cost().crash_now(pos, out)

    def stage_costs(self, pos, vel, ang, crashed, out):
        self._cost().stage_costs(pos, vel, ang, crashed, out)


def cpu_reference(cfgd, k, min_seconds=0.0, max_steps=None, budget_s=None):
    """The reference's CPU implementation of one optimisation iteration (sample_noise
    [+ dyn] + evaluate + update, controller.py:374-395) on K=k rollouts of the workload,
    all host cores (thread pool over chunks, BLAS 1 thread).  pimpc itself when it is
    installed (baseline/_ref), else the numpy oracle port (oracle/rollout.py)."""
    from threadpoolctl import threadpool_limits

    from oracle import rollout as RO
    from paper_1503_00330_b200 import synthetic

    T, L, M = cfgd["T"], cfgd["L"], cfgd["M"]
    workers = RO.default_workers()
    chunk = min(1024, -(-k // workers))
    stacks = synthetic.hybrid_stacks(L, seed=0)
    ref = synthetic.import_reference()
    if ref is not None:
        C = ref.controller
        task = ref.simworld.Task.default()
        model = synthetic.reference_hybrid(ref, stacks)
        cfg = C.PiConfig(num_rollouts=k, sub_rollouts=M, horizon_steps=T, iterations_per_step=1, rng_seed=0,
                         workers=workers, chunk_size=chunk)
        cost = ThreadLocalCost(ref, task, 1) if workers > 1 else ref.simworld.RolloutCost(task, 1)
        state = ref.dynamics.QuadState.hover(task.spawn)
        plan = C.ControlPlan.hover(ref.dynamics.QuadParams(), T)
        eng = C.RolloutEngine(model, cfg)

        def one(cyc):
            C.optimize(state, plan, cfg, model, cost, cyc, eng)
        kind, what = "reference", "pimpc.controller.optimize (the reference package, baseline/_ref)"
    else:
        model = RO.Model(stacks)
        cost = RO.Cost(synthetic.DEFAULT_WAYPOINTS[1], synthetic.DEFAULT_OBSTACLES)
        state = np.zeros(12)
        state[0:3] = synthetic.DEFAULT_WAYPOINTS[0]
        plan = np.tile([0.0, 0.0, 0.0, model.dyn.hover_thrust], (T, 1))

        def one(cyc):
            RO.optimize(model, state, plan, cost, K=k, M=M, iterations=1, chunk=chunk, workers=workers, cycle=cyc)
        kind, what = "port", "numpy oracle port of the reference (oracle/rollout.py; pimpc not installed)"
    times = []
    with threadpool_limits(1, "blas"):
        one(10_000)  # warm-up (workspaces, thread pool)
        t_all = time.perf_counter()
        cyc = 0
        while True:
            t0 = time.perf_counter()
            one(cyc)
            times.append(time.perf_counter() - t0)
            cyc += 1
            el = time.perf_counter() - t_all
            if max_steps is not None and cyc >= max_steps:
                break
            if budget_s is not None and el + times[-1] > budget_s:
                break
            if max_steps is None and budget_s is None and el >= min_seconds and cyc >= 2:
                break
    step = statistics.median(times)
    return {
        "value": k * T / step,
        "unit": UNIT,
        "cores": workers,
        "kind": kind,
        "sample": f"K={k} of {cfgd['K']} rollouts, T={T}, L={L}, M={M}; {what}, {workers} worker threads, "
                  f"BLAS 1 thread; median of {len(times)} steps (noise + evaluate + update)",
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


def pct(xs, q):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, max(0, math.ceil(q * len(xs)) - 1))]


class Rig:
    """One workload on this rank: the engine (one context at N=1, this rank's shard at
    N>1), the device-resident step, and the public-API step with host buffers."""

    def __init__(self, cfgd, world, local, stream, dist):
        import paper_1503_00330_b200 as P
        from paper_1503_00330_b200 import _abi, synthetic
        from paper_1503_00330_b200.controller import dynamics_struct
        from paper_1503_00330_b200.simworld import apply_cost

        self.P, self._abi = P, _abi
        self.cfgd, self.world, self.local, self.stream, self.dist = cfgd, world, local, stream, dist
        K, T, L, M = cfgd["K"], cfgd["T"], cfgd["L"], cfgd["M"]
        self.params = P.QuadParams()
        self.model = P.HybridModel.from_stacks(synthetic.hybrid_stacks(L, seed=0), self.params)
        self.task = P.Task.default()
        self.cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=T, iterations_per_step=1, rng_seed=0)
        self.state = P.QuadState.hover(self.task.spawn)
        self.plan0 = P.ControlPlan.hover(self.params, T)
        self.cost = P.RolloutCost(self.task, 1)
        self.sptr = _abi.torch_stream(local)
        if world > 1:
            from paper_1503_00330_b200.distributed import ShardedEngine

            self.eng = ShardedEngine(self.model, self.cfg, device=local)
            self.ctx = self.eng.ctx
            self.k_local = self.eng.stop - self.eng.start
            self.eng.optimize(self.state, self.plan0, self.cost, 0)  # binds, stages, captures the graph
        else:
            self.eng = P.RolloutEngine(self.model, self.cfg, device=local, noise="device", use_graph=True)
            self.ctx = self.eng.context(K, T)
            self.k_local = K
            self.ctx.call("pi2_set_dynamics", dynamics_struct(self.params, self.plan0.lo, self.plan0.hi))
            apply_cost(self.ctx, self.cost)
            self.ctx.call("pi2_load_plan", _abi.ptr(self.state.as_array()),
                          _abi.ptr(np.ascontiguousarray(self.plan0.controls)), self.sptr)

    def device_step(self, cycle):
        """One step on device-resident inputs (no host transfer, no synchronisation)."""
        from paper_1503_00330_b200.controller import optimize_args

        if self.world == 1:  # the whole iteration as one CUDA graph on the device-resident plan
            self.ctx.call("pi2_iterate_device", optimize_args(self.cfg, cycle, use_graph=True), self.sptr)
        else:  # this rank's captured step: pull, local kernels, NCCL all-gather, combine, push
            self.eng.step_device()

    def api_step(self, plan, cycle):
        """receding_horizon_step through the public API with host state/plan."""
        if self.world == 1:
            return self.P.receding_horizon_step(self.state, plan, self.cfg, self.model, self.cost, cycle, self.eng)
        opt = self.eng.optimize(self.state, plan, self.cost, cycle)
        return opt.control_at(0), opt.shifted()

    def barrier(self):
        import torch

        torch.cuda.synchronize()
        if self.dist is not None:
            self.dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(self, x: float) -> float:
        import torch

        if self.dist is None:
            return x
        dev = f"cuda:{self.local}" if self.dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def time_device(self, steps, warmup, clocks=None):
        """ms per step: `steps` back-to-back device steps, CUDA events on the launch stream,
        barrier + synchronize on both sides, max over ranks."""
        import torch

        for w in range(warmup):
            self.device_step(10_000 + w)
        self.barrier()
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if clocks is not None:
            clocks.mark_start()
        start.record(self.stream)
        for s in range(steps):
            self.device_step(s)
        end.record(self.stream)
        while not end.query():  # a sleeping wait keeps the GIL free for the clock sampler
            time.sleep(0.0005)
        self.barrier()
        if clocks is not None:
            clocks.mark_end()
        return self.max_over_ranks(start.elapsed_time(end)) / steps

    def time_device_iterations(self, iterations, steps, warmup):
        """ms per control step with `iterations` optimisation iterations per step (N=1: the
        reference's default is 2); one CUDA graph per step, CUDA events."""
        import torch

        from paper_1503_00330_b200.controller import optimize_args

        cfg = self.P.PiConfig(num_rollouts=self.cfg.num_rollouts, sub_rollouts=self.cfg.sub_rollouts,
                              horizon_steps=self.cfg.horizon_steps, iterations_per_step=iterations, rng_seed=0)
        for w in range(warmup):
            self.ctx.call("pi2_iterate_device", optimize_args(cfg, 20_000 + w, use_graph=True), self.sptr)
        self.barrier()
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(self.stream)
        for s in range(steps):
            self.ctx.call("pi2_iterate_device", optimize_args(cfg, s, use_graph=True), self.sptr)
        end.record(self.stream)
        end.synchronize()
        self.barrier()
        return start.elapsed_time(end) / steps

    def time_api(self, steps, warmup):
        """(total seconds, per-step latencies in ms) of the public-API step, max over ranks."""
        for w in range(warmup):
            self.api_step(self.plan0, 10_000 + w)
        self.barrier()
        plan, lat = self.plan0, []
        for s in range(steps):
            t0 = time.perf_counter()
            _, plan = self.api_step(plan, s)
            lat.append(time.perf_counter() - t0)
        total = self.max_over_ranks(sum(lat))
        lat_ms = [x * 1e3 for x in lat]
        return total, {"p50": self.max_over_ranks(statistics.median(lat_ms)),
                       "p99": self.max_over_ranks(pct(lat_ms, 0.99)), "max": self.max_over_ranks(max(lat_ms))}


def noise_stream(rig, local):
    """Host-noise path (controller.py:112-139: the reference's (K,N,4) f64 exploration and
    (K,M,N,3) f32 dynamics noise, resident in HBM): bandwidth of the kernels that stream
    them, from CUDA events around each kernel (pi2_profile_evaluate)."""
    import torch

    _abi = rig._abi
    K, T, M = rig.cfgd["K"], rig.cfgd["T"], rig.cfgd["M"]
    dev = f"cuda:{local}"
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    eps = torch.randn((K, T, 4), dtype=torch.float64, device=dev, generator=g) * torch.tensor(
        rig.cfg.exploration_std, dtype=torch.float64, device=dev)
    dyn = torch.randn((K, M, T, 3), dtype=torch.float32, device=dev, generator=g) if M > 1 else None
    ms = (_abi.C.c_double * 3)()
    torch.cuda.synchronize()  # the noise tensors were written on torch's stream
    rig.ctx.call("pi2_profile_evaluate", _abi.ptr(rig.state.as_array()), _abi.ptr(np.ascontiguousarray(rig.plan0.controls)),
                 _abi.ptr(eps), _abi.ptr(dyn), 10, ms)
    att, lw, roll = list(ms)
    eps_b = K * T * 4 * 8
    dyn_b = K * M * T * 3 * 4 if M > 1 else 0
    peak = float(measured_peaks().get("hbm_gbs", 6547.2))
    out = {"attitude_ms": att, "lwpr_ms": lw, "rollout_ms": roll,
           "eps_bytes": eps_b, "eps_gbs": eps_b / (att * 1e-3) / 1e9,
           # the attitude kernel also writes the (K*N) float4 LWPR rows and reads the plan
           "attitude_kernel_gbs": (eps_b + K * T * 16) / (att * 1e-3) / 1e9,
           "peak_gbs": peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"}
    out["eps_frac"] = out["eps_gbs"] / peak
    out["attitude_kernel_frac"] = out["attitude_kernel_gbs"] / peak
    if dyn_b:
        out.update({"dyn_bytes": dyn_b, "dyn_gbs": dyn_b / (roll * 1e-3) / 1e9,
                    "combined_gbs": (eps_b + dyn_b) / ((att + roll) * 1e-3) / 1e9})
        out["combined_frac"] = out["combined_gbs"] / peak
    out["what"] = ("algorithmic noise bytes / CUDA-event time of the kernel that streams them (attitude: "
                   "exploration noise; rollout/cost: dynamics noise); the rollout kernel is issue-bound, "
                   "so its rate is not a bandwidth ceiling")
    del eps, dyn
    return out


def closed_loop(cfgd, local, steps):
    """BASELINE C4's closed loop: the reference's own run_trial (simworld.py:270-380:
    plant, waypoints, crash verdicts, K=1 plan-cost probe) with this engine dropped in
    (device noise, one CUDA graph per control step); latency of every
    receding_horizon_step call, host state in, control out."""
    from paper_1503_00330_b200 import dropin, synthetic

    ref = synthetic.import_reference()
    if ref is None:
        return {"skipped": "reference package pimpc not installed (baseline/_ref)"}
    p = ref.dynamics.QuadParams()
    model = synthetic.reference_hybrid(ref, synthetic.hybrid_stacks(cfgd["L"], seed=0), p)
    gt = ref.dynamics.PerturbedModel(p, drag_coeff=0.08, thrust_scale=0.97)
    cfg = ref.controller.PiConfig(num_rollouts=cfgd["K"], sub_rollouts=cfgd["M"], horizon_steps=cfgd["T"],
                                  iterations_per_step=1)
    lat = []
    with dropin.patched(ref.controller, noise="device", device=local, step_times=lat):
        t0 = time.perf_counter()
        trial = ref.simworld.run_trial(ref.simworld.Task.default(), cfg, model, gt, seed=0, step_cap=steps)
        wall = time.perf_counter() - t0
    raw = np.asarray(lat) * 1e3
    tl = sorted(raw[1:]) if len(raw) > 1 else sorted(raw)  # steady state: after the setup step
    return {
        "what": "pimpc.simworld.run_trial (the reference's closed loop) with paper_1503_00330_b200.RolloutEngine "
                "dropped in (dropin.patched, device noise); plant = pimpc PerturbedModel(drag 0.08, thrust x0.97)",
        "steps": int(trial.steps), "outcome": trial.outcome,
        "p50_ms": float(np.median(tl)), "p99_ms": float(pct(tl, 0.99)), "max_ms": float(tl[-1]),
        "budget_ms": BUDGET_MS, "within_budget": bool(tl[-1] < BUDGET_MS),
        "first_step_ms": float(raw[0]) if len(raw) else None,
        "first_step": "context creation, weight staging and CUDA graph capture; p50/p99/max cover the later steps",
        "trial_wall_s": wall,
    }


def north_star(args, world, local, stream, dist, rank):
    """BASELINE C4 (K=2^20, T=50, L=100, M=1): one step split over the N GPUs."""
    import torch

    cfgd, desc = workload("C4", world, "strong")
    rig = Rig(cfgd, world, local, stream, dist)
    steps = max(5, min(args.steps, 20))
    ms = rig.time_device(steps, max(3, min(args.warmup, 5)))
    _, lat = rig.time_api(steps, 3)
    out = {"workload": desc, "K": cfgd["K"], "K_per_gpu": rig.k_local, "n_gpus": world, "scaling": "strong",
           "device_ms_per_step": ms, "value": cfgd["K"] * cfgd["T"] / (ms * 1e-3), "unit": UNIT,
           "e2e_ms": lat, "budget_ms": BUDGET_MS, "within_budget": bool(lat["p99"] < BUDGET_MS),
           "api": "receding_horizon_step" if world == 1 else "distributed.ShardedEngine.optimize (graph-captured)"}
    del rig
    torch.cuda.empty_cache()
    if world > 1:  # the same step on one GPU, same run: the strong-scaling speed-up
        one_ms = None
        if rank == 0:
            solo = Rig(cfgd, 1, local, stream, None)
            one_ms = solo.time_device(steps, 3)
            del solo
            torch.cuda.empty_cache()
        dist.barrier()
        if rank == 0:
            out["one_gpu_ms_per_step"] = one_ms
            out["speedup_vs_1gpu"] = one_ms / ms
            out["strong_scaling_efficiency"] = one_ms / ms / world
    elif args.closed_loop_steps > 0:
        out["closed_loop"] = closed_loop(cfgd, local, args.closed_loop_steps)
    return out


def lwpr_frac(rig, cfgd):
    """Stage ms of one iteration (CUDA events, pi2_profile_iteration) and the LWPR kernel's
    algorithmic 2^x rate against the MUFU peak, as in the headline roofline."""
    from paper_1503_00330_b200.controller import optimize_args

    _abi = rig._abi
    stage_ms = (_abi.C.c_double * 5)()
    rig.ctx.call("pi2_profile_iteration", optimize_args(rig.cfg, 0, use_graph=False), 5, stage_ms)
    stages = dict(zip(["attitude", "lwpr", "rollout_cost", "partials", "combine"], list(stage_ms)))
    exps = cfgd["K"] * cfgd["T"] * 3 * cfgd["L"]
    mufu_peak = float(measured_peaks().get("mufu_ex2_per_s", 4.60e12))
    return stages, exps / (stages["lwpr"] / 1e3) / mufu_peak


def other_configs(args, local, stream):
    """N=1: the other BASELINE configs measured briefly in the same run (device ms per step
    over back-to-back graph replays, e2e p50/p99 through receding_horizon_step, the LWPR
    kernel's MUFU fraction), and C5's rollout-count sweep K = 2^10 .. 2^22."""
    import torch

    out = {}
    for name, steps in (("C1", 50), ("C3", 10), ("C5", 10)):
        cfgd, desc = workload(name, 1, "strong")
        rig = Rig(cfgd, 1, local, stream, None)
        ms = rig.time_device(steps, 3)
        _, lat = rig.time_api(min(steps, 10), 2)
        stages, frac = lwpr_frac(rig, cfgd)
        out[name] = {"workload": desc, "device_ms_per_step": ms, "value": cfgd["K"] * cfgd["T"] / (ms * 1e-3),
                     "unit": UNIT, "e2e_ms": lat, "stages_ms": stages, "lwpr_mufu_frac": frac, "steps": steps}
        del rig
        torch.cuda.empty_cache()
    sweep = []
    for lk in range(10, 23, 2):
        cfgd, _ = workload("C5", 1, "strong")
        cfgd["K"] = 1 << lk
        rig = Rig(cfgd, 1, local, stream, None)
        ms = rig.time_device(10 if lk >= 18 else 50, 3)
        sweep.append({"K": cfgd["K"], "device_ms_per_step": ms, "value": cfgd["K"] * cfgd["T"] / (ms * 1e-3)})
        del rig
        torch.cuda.empty_cache()
    out["C5_k_sweep"] = {"T": 50, "L": 200, "M": 1, "unit": UNIT, "points": sweep}
    return out


def run_ours(args, rank: int, world: int, local: int):
    import torch

    dist = None
    # one rank per GPU; PI2_DIST_BACKEND=gloo lets several ranks share a GPU to
    # exercise the multi-rank path where only one GPU exists (timings meaningless)
    backend = os.environ.get("PI2_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfgd, desc = workload(args.config, world, args.scaling)
    K, T, L, M = cfgd["K"], cfgd["T"], cfgd["L"], cfgd["M"]
    stream = torch.cuda.Stream(device=local)  # dedicated stream: kernels, events and NCCL share it
    torch.cuda.set_stream(stream)
    rig = Rig(cfgd, world, local, stream, dist)
    _abi = rig._abi

    # ---- device-resident throughput (value)
    with ClockSampler(local) as clocks:
        ms_per_step = rig.time_device(args.steps, args.warmup, clocks)
    value = K * T / (ms_per_step * 1e-3)

    # ---- stage profile (dominant kernel = LWPR), CUDA events on the context stream
    from paper_1503_00330_b200.controller import optimize_args

    stage_ms = (_abi.C.c_double * 5)()
    rig.ctx.call("pi2_profile_iteration", optimize_args(rig.cfg, 0, use_graph=False), 10, stage_ms)
    stages = dict(zip(["attitude", "lwpr", "rollout_cost", "partials", "combine"], list(stage_ms)))
    # which LWPR kernel ran, and the share of its 2^x on MUFU (the rest on the FMA pipe)
    kern, share = _abi.C.c_int32(), _abi.C.c_double()
    rig.ctx.call("pi2_lwpr_kernel", int(M > 1), _abi.C.byref(kern), _abi.C.byref(share))

    # ---- the reference's default of 2 iterations per control step (N=1)
    it2 = None
    if world == 1:
        it2_ms = rig.time_device_iterations(2, max(5, args.steps // 4), args.warmup)
        it2 = {"iterations_per_step": 2, "ms_per_step": it2_ms, "value": 2 * K * T / (it2_ms * 1e-3), "unit": UNIT,
               "what": "the same workload with the reference's default iterations_per_step=2 (PiConfig, "
                       "controller.py:79): device ms per control step, rollout-steps of both iterations per second"}

    # ---- end to end through the public API (host state/plan in, control/plan out)
    e2e_s, lat = rig.time_api(args.steps, args.warmup)

    # ---- noise-stream bandwidth of the host-noise path (N=1)
    ns = noise_stream(rig, local) if world == 1 else None

    k_local = rig.k_local
    del rig
    torch.cuda.empty_cache()
    ns_obj = None
    if not args.no_north_star:
        ns_obj = north_star(args, world, local, stream, dist, rank)
    oc = (other_configs(args, local, stream)
          if world == 1 and args.config == "C2" and not args.no_other_configs else None)

    if rank != 0:
        return None

    peaks = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    n_sm = torch.cuda.get_device_properties(local).multi_processor_count
    peak_tflops = n_sm * 128 * 2 * sm_max * 1e6 / 1e12
    rows = k_local * T
    flops_per_field = 32 if M > 1 else 27  # 27 (+5 variance) per (row, axis, field)
    lwpr_flops = rows * 3 * L * flops_per_field
    lw_s = stages["lwpr"] / 1e3
    achieved = lwpr_flops / lw_s / 1e12
    tc = kern.value == 1
    exps = rows * 3 * L  # one 2^x per (row, axis, field): the algorithmic count
    mufu_peak = float(peaks.get("mufu_ex2_per_s", 4.60e12))
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
    ex_rate = exps / lw_s
    if tc:  # binding unit: the exponentials (the linear parts are on the tensor cores)
        roofline = {"bound": "mufu", "kernel": "lwpr_tc_kernel (tcgen05 3xTF32 field GEMM + exp/moments)",
                    "achieved": ex_rate / 1e12, "peak": mufu_peak / 1e12, "unit": "Tex2/s",
                    "frac": ex_rate / mufu_peak,
                    "peak_source": "profiles/micro/mufu_mix_b200.txt (MUFU-only ex2 stream, 148 SMs)",
                    "what": "algorithmic 2^x per launch (rows x 3 axes x L fields) / CUDA-event duration; a share "
                            "runs as a polynomial on the FMA pipe (mufu_share on MUFU)",
                    "ex2_per_launch": exps, "mufu_share": share.value,
                    "mufu_busy_frac": ex_rate * share.value / mufu_peak,
                    "traffic": lwpr_traffic(args.config, tc) if world == 1 else None,
                    "fp32_equivalent": {**fp32, "note": "the same algorithmic FLOPs against the FP32 CUDA-core "
                                        "peak; above 1 when the tensor cores carry the linear parts"}}
    else:
        roofline = {"bound": "fp32", "kernel": "lwpr_kernel (CUDA cores, FFMA2)", **fp32,
                    "traffic": lwpr_traffic(args.config, tc) if world == 1 else None,
                    "mufu": {"achieved": ex_rate / 1e12, "peak": mufu_peak / 1e12, "unit": "Tex2/s"}}
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
        "config": config_dict(cfgd, desc),
        "sharding": {"K_per_gpu": k_local, "parallelism": f"rollouts sharded over {world} GPU(s)"
                     + ("" if world == 1 else "; NCCL all-gather of per-timestep softmax partials inside each "
                        "rank's captured CUDA graph")},
        "e2e": {
            "value": K * T * args.steps / e2e_s,
            "unit": UNIT,
            "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h,
            "api": "paper_1503_00330_b200.receding_horizon_step(noise='device' engine)" if world == 1
                   else "distributed.ShardedEngine.optimize",
        },
        "latency_ms": {**lat, "what": "e2e control step (host state/plan -> control)"},
        "roofline": roofline,
        "stages_ms": stages,
        "clocks": clk,
        "gpu_launches": args.steps * (KERNELS_PER_ITER + (2 if world > 1 else 0)),
    }
    if ns is not None:
        line["noise_stream"] = ns
    if ns_obj is not None:
        line["north_star"] = ns_obj
    if it2 is not None:
        line["iterations_per_step_2"] = it2
    if oc is not None:
        line["other_configs"] = oc
    if world == 1 and not args.no_cpu_baseline:
        cb = cpu_reference(cfgd, min(args.cpu_sample, K), min_seconds=args.cpu_seconds)
        cb.pop("step_times_s", None)
        cb["cpu_model"] = cpu_model()
        line["cpu_baseline"] = cb
    return line


def run_reference(args, world: int = 1):
    """The reference arm: the reference's own CPU path on the FULL configured workload
    (same config object as our arm), on the host cores; the number of timed steps is
    bounded by --ref-budget-s (each step is a whole iteration at full K)."""
    cfgd, desc = workload(args.config, world, args.scaling)
    cb = cpu_reference(cfgd, cfgd["K"], max_steps=args.warmup + args.steps, budget_s=args.ref_budget_s)
    times = cb.pop("step_times_s")
    timed = times[args.warmup:] if len(times) > args.warmup else times[-max(1, len(times) // 2):]
    step = sum(timed) / len(timed)
    value = cfgd["K"] * cfgd["T"] / step
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": 0,
        "steps": len(timed),
        "warmup": len(times) - len(timed) + 1,
        "steps_requested": args.steps,
        "ms_per_step": step * 1e3,
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "f32 + f64 (numpy)",
        "data": "synthetic",
        "config": config_dict(cfgd, desc),
        "cpu_baseline": {**cb, "value": value, "cpu_model": cpu_model(),
                         "sample": cb["sample"] + f"; {len(timed)} timed steps within a {args.ref_budget_s:.0f} s "
                                                  "budget"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn(args)
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
