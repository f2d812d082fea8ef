"""Receding-horizon PI² optimisation on B200 (API of reference ``controller.py``).

Same names, signatures, errors and semantics as the reference module
(``ControlPlan`` :29-69, ``PiConfig`` :72-100, ``RolloutBatch`` :103-109,
``sample_noise`` :112-125, ``sample_dynamics_noise`` :128-139,
``RolloutEngine`` :161-247, ``evaluate_rollouts`` :325-353,
``path_integral_update`` :356-371, ``optimize`` :374-395,
``receding_horizon_step`` :398-413), with every rollout, cost and update
computed by the CUDA engine behind ``include/pi2rh.h``.

Noise: ``RolloutEngine(..., noise="reference")`` (default) consumes the
reference's host noise streams (numpy Philox + ziggurat, bit-identical
arrays), so results match the reference on identical inputs.
``noise="device"`` generates the same-addressed streams on the GPU
(Philox4x32-10 + Box–Muller) inside the kernels and runs the whole
``iterations_per_step`` loop as one CUDA graph — the real-time mode.
"""

from __future__ import annotations

import os
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _abi, rng
from .dynamics import AnalyticModel, Control, QuadParams, QuadState
from .lwpr import stage_axis
from .simworld import apply_cost

NOISE_MODES = ("reference", "device")


@dataclass
class ControlPlan:
    """N control rows (3 desired rates + thrust), clipped on construction (controller.py:29-69)."""

    controls: np.ndarray
    dt: float
    origin_time: float
    lo: np.ndarray
    hi: np.ndarray

    def __post_init__(self):
        self.controls = np.asarray(self.controls, float)
        if self.controls.ndim != 2 or self.controls.shape[1] != 4:
            raise ValueError("controls must be (N, 4)")
        if len(self.controls) < 1:
            raise ValueError("plan must have at least one control")
        self.controls = np.clip(self.controls, self.lo[None, :], self.hi[None, :])

    @classmethod
    def hover(cls, params: QuadParams, horizon_steps: int, origin_time=0.0) -> "ControlPlan":
        lo, hi = params.control_bounds()
        controls = np.tile([0.0, 0.0, 0.0, params.hover_thrust], (horizon_steps, 1))
        return cls(controls, params.dt, origin_time, lo, hi)

    def __len__(self) -> int:
        return len(self.controls)

    def controls_array(self) -> np.ndarray:
        return self.controls

    def control_at(self, i: int) -> Control:
        row = self.controls[i]
        return Control(row[:3].copy(), float(row[3]))

    def shifted(self) -> "ControlPlan":
        controls = np.vstack([self.controls[1:], self.controls[-1:]])
        return ControlPlan(controls, self.dt, self.origin_time + self.dt, self.lo, self.hi)

    def replaced(self, controls) -> "ControlPlan":
        return ControlPlan(np.asarray(controls, float), self.dt, self.origin_time, self.lo, self.hi)

    @classmethod
    def _clipped(cls, controls, dt, origin_time, lo, hi) -> "ControlPlan":
        """A plan from (N, 4) float64 controls already inside [lo, hi] (the device update
        clips), skipping the constructor's re-clip."""
        p = cls.__new__(cls)
        p.controls, p.dt, p.origin_time, p.lo, p.hi = controls, dt, origin_time, lo, hi
        return p


@dataclass
class PiConfig:
    """Path-integral optimiser settings (controller.py:72-100)."""

    num_rollouts: int = 1000
    sub_rollouts: int = 1
    horizon_steps: int = 50
    iterations_per_step: int = 2
    temperature: float = 1.0
    exploration_std: np.ndarray = field(default_factory=lambda: np.array([2.0, 2.0, 0.8, 0.05]))
    rng_seed: int = 0
    workers: int = 1
    chunk_size: int = 1000
    cost_ceiling: float = 1e8

    def __post_init__(self):
        self.exploration_std = np.asarray(self.exploration_std, float).reshape(4)
        if self.num_rollouts < 1 or self.sub_rollouts < 1 or self.horizon_steps < 1:
            raise ValueError("num_rollouts, sub_rollouts, horizon_steps must be >= 1")
        if self.temperature <= 0:
            raise ValueError("temperature must be positive")
        if np.any(self.exploration_std <= 0):
            raise ValueError("exploration_std must be positive")
        if self.iterations_per_step < 0:
            raise ValueError("iterations_per_step must be >= 0")
        if self.workers < 1 or self.chunk_size < 1:
            raise ValueError("workers and chunk_size must be >= 1")


@dataclass
class RolloutBatch:
    """Evaluated rollouts for one optimisation iteration (controller.py:103-109)."""

    noise: np.ndarray        # (K, N, 4)
    costs_to_go: np.ndarray  # (K, N)
    crash_flags: np.ndarray  # (K,)


def sample_noise(config: PiConfig, cycle_index: int, iteration: int = 0) -> np.ndarray:
    """Host exploration noise (K, N, 4) of the reference stream (controller.py:112-125)."""
    block = rng.normal_block(config.rng_seed, (rng.STREAM_CONTROL, cycle_index, iteration),
                             (config.num_rollouts, config.horizon_steps, 4))
    block *= config.exploration_std[None, None, :]
    return block


def sample_dynamics_noise(config: PiConfig, cycle_index: int, iteration: int = 0) -> np.ndarray:
    """Host standard normals (K, M, N, 3) float32 of the reference stream (controller.py:128-139)."""
    return rng.normal_block(config.rng_seed, (rng.STREAM_DYNAMICS, cycle_index, iteration),
                            (config.num_rollouts, config.sub_rollouts, config.horizon_steps, 3),
                            dtype=np.float32)


def _default_device() -> int:
    return int(os.environ.get("LOCAL_RANK", "0")) if os.environ.get("PI2_DEVICE") is None \
        else int(os.environ["PI2_DEVICE"])


def model_kind(model) -> tuple[int, float]:
    """Device plugin of a model object (RolloutEngine model protocol, controller.py:169-173).

    HybridModel-like (``models`` = 3 LWPR models) -> LWPR; AnalyticModel ->
    rigid body; TwoPointModel-like (``magnitude`` + sign noise transform) ->
    two-point test model.  Anything else has no device implementation.
    """
    if getattr(model, "drag_coeff", None) is not None:
        raise TypeError("velocity-dependent ground-truth model cannot serve rollouts")
    if hasattr(model, "models"):
        return _abi.MODEL_HYBRID_LWPR, 0.0
    nt = getattr(model, "noise_transform", None)
    if hasattr(model, "magnitude") and nt is np.sign:
        return _abi.MODEL_TWO_POINT, float(np.float32(model.magnitude))
    if nt is not None:
        raise TypeError("noise_transform has no device implementation (only np.sign)")
    if isinstance(model, AnalyticModel) or type(model).__name__ == "AnalyticModel":
        return _abi.MODEL_ANALYTIC, 0.0
    raise TypeError(f"model {type(model).__name__} has no device implementation")


def dynamics_struct(params, lo, hi) -> "_abi.Dynamics":
    d = _abi.Dynamics()
    d.mass, d.gravity = float(params.mass), float(params.gravity)
    d.rate_gain, d.dt = float(params.rate_gain), float(params.dt)
    d.lo[:] = [float(v) for v in lo]
    d.hi[:] = [float(v) for v in hi]
    return d


class RolloutEngine:
    """GPU rollout engine with the reference engine protocol (controller.py:161-247).

    ``evaluate`` returns the reference's ``RolloutBatch``; ``chunk_size`` and
    ``workers`` are accepted and ignored (results never depend on them, as in
    the reference).  Extra keyword arguments: ``device`` (CUDA ordinal),
    ``noise`` ("reference" | "device", see module docstring), ``use_graph``.
    """

    def __init__(self, model, config: PiConfig, *, device: int | None = None,
                 noise: str = "reference", use_graph: bool = True):
        if noise not in NOISE_MODES:
            raise ValueError(f"noise must be one of {NOISE_MODES}")
        self.model = model
        self.config = config
        self.params: QuadParams = model.params
        self.chunk = min(config.chunk_size, config.num_rollouts)
        self.use_spread = bool(getattr(model, "probabilistic", False)) and config.sub_rollouts > 1
        self.noise_transform = getattr(model, "noise_transform", None)
        self.kind, self.kind_param = model_kind(model)
        self.device = _default_device() if device is None else int(device)
        self.noise = noise
        self.use_graph = bool(use_graph)
        self._ctxs: dict[tuple[int, int], _abi.Context] = {}
        self._bound: dict[int, tuple] = {}  # per context: key of the dynamics + cost last bound
        self._io: dict[int, tuple] = {}     # receding_device host buffers per horizon
        self._args = _abi.OptimizeArgs()

    def context(self, num_rollouts: int, horizon: int) -> "_abi.Context":
        key = (int(num_rollouts), int(horizon))
        ctx = self._ctxs.get(key)
        if ctx is None:
            ctx = _abi.Context(self.device, num_rollouts, horizon, self.config.sub_rollouts)
            if self.kind == _abi.MODEL_HYBRID_LWPR:
                if len(self.model.models) != 3:
                    raise ValueError("need one model per acceleration axis")
                for axis, m in zip("xyz", self.model.models):
                    if m.num_fields == 0:
                        raise ValueError(f"acceleration model for {axis} axis is untrained")
                for a in range(3):
                    stage_axis(ctx, a, self.model.models[a])
            ctx.call("pi2_select_model", self.kind, self.kind_param)
            self._ctxs[key] = ctx
        return ctx

    def _bind(self, ctx, plan, cost_model) -> None:
        """Stage the dynamics constants and the cost plugin; skipped when both are unchanged
        since the last call on this context (compared by value, so mutating the plugin
        between steps, e.g. switching waypoints, is picked up)."""
        p = self.params
        key = (p.mass, p.gravity, p.rate_gain, p.dt, np.asarray(plan.lo, float).tobytes(),
               np.asarray(plan.hi, float).tobytes(), _cost_key(cost_model))
        if self._bound.get(id(ctx)) == key and key[-1] is not None:
            return
        self._bound.pop(id(ctx), None)
        ctx.call("pi2_set_dynamics", dynamics_struct(self.params, plan.lo, plan.hi))
        apply_cost(ctx, cost_model)
        self._bound[id(ctx)] = key

    def evaluate(self, state: QuadState, plan: ControlPlan, noise, cost_model,
                 dyn_noise=None) -> RolloutBatch:
        """Propagate every perturbed plan and accumulate cost-to-go (controller.py:197-247)."""
        k_total, n_steps = noise.shape[0], noise.shape[1]
        if n_steps != len(plan):
            raise ValueError("noise horizon does not match plan length")
        if self.use_spread and dyn_noise is None:
            raise ValueError("probabilistic model with sub_rollouts > 1 needs dyn_noise")
        eps = np.ascontiguousarray(noise, dtype=np.float64)
        dyn = None
        if self.use_spread:
            dyn = np.ascontiguousarray(dyn_noise, dtype=np.float32)
            if dyn.shape != (k_total, self.config.sub_rollouts, n_steps, 3):
                raise ValueError("dyn_noise must be (K, M, N, 3)")
        ctx = self.context(k_total, n_steps)
        self._bind(ctx, plan, cost_model)
        costs = np.empty((k_total, n_steps))
        crash = np.empty(k_total, np.uint8)
        ctx.call("pi2_evaluate", _abi.ptr(np.ascontiguousarray(state.as_array())),
                 _abi.ptr(np.ascontiguousarray(plan.controls)), _abi.ptr(eps), _abi.ptr(dyn),
                 float(self.config.cost_ceiling), _abi.ptr(costs), _abi.ptr(crash))
        return RolloutBatch(noise=noise, costs_to_go=costs, crash_flags=crash.astype(bool))

    def optimize_device(self, state: QuadState, plan: ControlPlan, cost_model,
                        cycle_index: int = 0) -> ControlPlan:
        """All ``iterations_per_step`` iterations on the GPU with device noise (one CUDA graph)."""
        cfg = self.config
        ctx = self.context(cfg.num_rollouts, len(plan))
        self._bind(ctx, plan, cost_model)
        controls = np.ascontiguousarray(plan.controls, dtype=np.float64).copy()
        ctx.call("pi2_optimize", _abi.ptr(np.ascontiguousarray(state.as_array())), _abi.ptr(controls),
                 optimize_args(cfg, cycle_index, self.use_graph))
        return plan.replaced(controls)

    def receding_device(self, state: QuadState, plan: ControlPlan, cost_model, cycle_index: int = 0):
        """``receding_horizon_step`` on the GPU with device noise: optimise, then take the
        first control and shift the plan inside the C ABI (pi2_receding_horizon_step).
        Host buffers, their pointers and the argument struct persist across calls
        (the per-call host overhead is what a real-time loop pays)."""
        cfg = self.config
        n = len(plan)
        ctx = self.context(cfg.num_rollouts, n)
        self._bind(ctx, plan, cost_model)
        io = self._io.get(n)
        if io is None:
            st, pl, first = np.empty(12), np.empty((n, 4)), np.empty(4)
            io = self._io[n] = (st, pl, first, _abi.ptr(st), _abi.ptr(pl), _abi.ptr(first))
        st, pl, first, p_st, p_pl, p_first = io
        st[0:3], st[3:6], st[6:9], st[9:12] = state.position, state.velocity, state.angles, state.rates
        pl[...] = plan.controls
        ctx.call("pi2_receding_horizon_step", p_st, p_pl, self._opt_args(cycle_index), p_first)
        return (Control(first[:3].copy(), float(first[3])),
                ControlPlan._clipped(pl.copy(), plan.dt, plan.origin_time + plan.dt, plan.lo, plan.hi))

    def _opt_args(self, cycle_index: int) -> "_abi.OptimizeArgs":
        """The engine's OptimizeArgs, refreshed from the config (which may be mutated)."""
        cfg, a = self.config, self._args
        a.temperature = float(cfg.temperature)
        a.cost_ceiling = float(cfg.cost_ceiling)
        std = cfg.exploration_std
        if a.exploration_std[0] != std[0] or a.exploration_std[1] != std[1] or \
                a.exploration_std[2] != std[2] or a.exploration_std[3] != std[3]:
            a.exploration_std[:] = [float(v) for v in std]
        a.seed = int(cfg.rng_seed) & ((1 << 64) - 1)
        a.cycle = int(cycle_index) & ((1 << 64) - 1)
        a.iterations = int(cfg.iterations_per_step)
        a.use_graph = int(self.use_graph)
        return a


def _cost_key(cost_model):
    """Value key of a cost plugin's device descriptor (see simworld.cost_struct); None when
    the plugin has no device form (cost_struct then raises)."""
    try:
        wp, obs, zf = cost_model.waypoint, cost_model.obstacles, cost_model.z_floor
        lo, hi = cost_model.lo, cost_model.hi
    except AttributeError:
        if hasattr(cost_model, "threshold") and not hasattr(cost_model, "waypoint"):
            return ("threshold", float(np.float32(cost_model.threshold)))
        return None
    f32 = np.float32
    return ("nav", np.asarray(wp, f32).tobytes(), np.asarray(obs, f32).tobytes(), float(f32(zf)),
            np.asarray(lo, f32).tobytes(), np.asarray(hi, f32).tobytes(),
            float(f32(getattr(cost_model, "variance_penalty", 0.0))))


def optimize_args(cfg: PiConfig, cycle_index: int, use_graph: bool = True) -> "_abi.OptimizeArgs":
    a = _abi.OptimizeArgs()
    a.temperature = float(cfg.temperature)
    a.cost_ceiling = float(cfg.cost_ceiling)
    a.exploration_std[:] = [float(v) for v in cfg.exploration_std]
    a.seed = int(cfg.rng_seed) & ((1 << 64) - 1)
    a.cycle = int(cycle_index) & ((1 << 64) - 1)
    a.iterations = int(cfg.iterations_per_step)
    a.use_graph = int(bool(use_graph))
    return a


def evaluate_rollouts(state, plan, noise, model, cost_model, sub_rollouts: int = 1, dyn_noise=None,
                      workers: int = 1, chunk_size: int = 250, cost_ceiling: float = 1e8,
                      device: int | None = None) -> RolloutBatch:
    """One-shot rollout evaluation (controller.py:325-353)."""
    cfg = PiConfig(num_rollouts=noise.shape[0], sub_rollouts=sub_rollouts, horizon_steps=noise.shape[1],
                   iterations_per_step=1, workers=workers, chunk_size=chunk_size, cost_ceiling=cost_ceiling)
    return RolloutEngine(model, cfg, device=device).evaluate(state, plan, noise, cost_model, dyn_noise)


# path_integral_update is a pure function in the reference; here it runs on a context
# (stream + scratch), and contexts are one per host thread (include/pi2rh.h), so each
# thread keeps its own per device.
_UPDATE_TLS = threading.local()


def _update_context(dev: int) -> _abi.Context:
    ctxs = getattr(_UPDATE_TLS, "ctxs", None)
    if ctxs is None:
        ctxs = _UPDATE_TLS.ctxs = {}
    ctx = ctxs.get(dev)
    if ctx is None:
        ctx = ctxs[dev] = _abi.Context(dev, 1, 1, 1)
    return ctx


def path_integral_update(plan: ControlPlan, batch: RolloutBatch, temperature: float,
                         device: int | None = None) -> ControlPlan:
    """Per-timestep min-shifted softmax update of the plan (controller.py:356-371), on the GPU."""
    costs = np.ascontiguousarray(batch.costs_to_go, dtype=np.float64)
    noise = np.ascontiguousarray(batch.noise, dtype=np.float64)
    if costs.ndim != 2 or noise.ndim != 3 or costs.shape != noise.shape[:2] or len(plan) != costs.shape[1]:
        raise ValueError("batch does not match plan dimensions")
    if not temperature > 0:
        raise ValueError("temperature must be positive")
    dev = _default_device() if device is None else int(device)
    ctx = _update_context(dev)
    ctx.call("pi2_set_dynamics", dynamics_struct(QuadParams(), plan.lo, plan.hi))
    out = np.empty((len(plan), 4))
    ctx.call("pi2_update", int(costs.shape[0]), int(costs.shape[1]),
             _abi.ptr(np.ascontiguousarray(plan.controls)), _abi.ptr(costs), _abi.ptr(noise),
             float(temperature), _abi.ptr(out))
    return plan.replaced(out)


def optimize(state: QuadState, plan: ControlPlan, config: PiConfig, model, cost_model,
             cycle_index: int = 0, engine: RolloutEngine | None = None) -> ControlPlan:
    """Run iterations_per_step rounds of sample / evaluate / update (controller.py:374-395)."""
    if engine is None:
        engine = RolloutEngine(model, config)
    if config.iterations_per_step == 0:
        return plan
    if engine.noise == "device":
        return engine.optimize_device(state, plan, cost_model, cycle_index)
    for iteration in range(config.iterations_per_step):
        noise = sample_noise(config, cycle_index, iteration)
        dyn = sample_dynamics_noise(config, cycle_index, iteration) if engine.use_spread else None
        batch = engine.evaluate(state, plan, noise, cost_model, dyn)
        plan = path_integral_update(plan, batch, config.temperature, device=engine.device)
    return plan


def receding_horizon_step(state: QuadState, plan: ControlPlan, config: PiConfig, model, cost_model,
                          cycle_index: int = 0, engine: RolloutEngine | None = None):
    """Optimise; return the first control and the shifted plan (controller.py:398-413)."""
    if engine is not None and engine.noise == "device" and engine.config is config:
        return engine.receding_device(state, plan, cost_model, cycle_index)
    optimized = optimize(state, plan, config, model, cost_model, cycle_index, engine)
    return optimized.control_at(0), optimized.shifted()
