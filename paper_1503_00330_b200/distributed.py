"""Rollout sharding across GPUs (one process per GPU, torch.distributed).

The reference parallelises rollouts over a thread pool in fixed chunks so
results never depend on the worker count (controller.py:10-13, 214-242).
Here rank r of G owns a contiguous, chunk-aligned slice of the K rollouts;
every iteration it produces one (min S, Z, V[4]) partial per timestep for
its slice (``pi2_iterate_local``), the G partials are all-gathered (NCCL
over NVLink, ~6·N·8 bytes per rank) and every rank applies the same
fixed-order tree combine and plan update (``pi2_iterate_finalize``).  With
power-of-two chunk counts per rank the tree is exactly the single-GPU tree,
so the update is bitwise identical for 1/2/4/8 GPUs.
"""

from __future__ import annotations

import numpy as np

from . import _abi
from .controller import ControlPlan, PiConfig, _cost_key, dynamics_struct, model_kind, optimize_args
from .lwpr import stage_axis
from .simworld import apply_cost


def shard_range(num_rollouts: int, rank: int, world: int, chunk: int | None = None) -> tuple[int, int]:
    """[start, stop) of rank's rollouts: contiguous, chunk-aligned, sizes differ by <= one chunk."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    chunk = int(chunk or _abi.lib().pi2_partial_chunk())
    n_chunks = -(-num_rollouts // chunk)
    base, extra = divmod(n_chunks, world)
    c0 = rank * base + min(rank, extra)
    c1 = c0 + base + (1 if rank < extra else 0)
    return min(c0 * chunk, num_rollouts), min(c1 * chunk, num_rollouts)


def gather_partials(partial, group=None):
    """All-gather a (N, 6) partial from every rank into (G, N, 6), rank order.

    NCCL gathers the device tensor in place on the current stream; a gloo
    group (CPU tests, several ranks sharing one GPU) stages through the host.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world,) + tuple(partial.shape), dtype=partial.dtype, device=partial.device)
        torch.cuda.nvtx.range_push("gather_partials")  # NVTX, like the C ABI's entry points
        dist.all_gather_into_tensor(out, partial.contiguous(), group=group)
        torch.cuda.nvtx.range_pop()
        return out
    host = partial.detach().to("cpu")  # synchronises with the kernels that wrote it
    parts = [torch.empty_like(host) for _ in range(world)]
    dist.all_gather(parts, host, group=group)
    return torch.stack(parts).to(partial.device)


def combine_gathered_host(gathered: np.ndarray, temperature: float) -> np.ndarray:
    """Fixed-order combine of (G, N, 6) partials on the host (same tree as the device)."""
    g = np.ascontiguousarray(gathered, dtype=np.float64)
    out = np.empty(g.shape[1:])
    _abi.check(_abi.lib().pi2_combine_partials_host(_abi.ptr(g), g.shape[0], g.shape[1],
                                                    float(temperature), _abi.ptr(out)))
    return out


def apply_partial(plan: np.ndarray, root: np.ndarray, lo, hi) -> np.ndarray:
    """plan + V/Z clipped to the bounds (controller.py:369-371) — host form of the finalize."""
    return np.clip(plan + root[:, 2:6] / root[:, 1:2], lo[None, :], hi[None, :])


class ShardedEngine:
    """This rank's share of a PI²-RH optimisation with device noise.

    ``optimize(state, plan, cost_model, cycle_index)`` has the semantics of
    ``controller.optimize`` with a ``noise="device"`` engine; all ranks return
    the same plan.

    With NCCL (``use_graph`` default) the rank's whole control step — input pull,
    per iteration local kernels -> ``all_gather_into_tensor`` -> combine + plan
    update, plan push — is captured once into one CUDA graph (torch.cuda.graph,
    NCCL collectives are capturable) and replayed every step: one graph launch
    and one stream synchronisation per control step, no per-iteration host
    round trip.  The gloo backend (CPU tests, several ranks sharing one GPU)
    runs the same calls eagerly with the exchange staged through the host.
    """

    def __init__(self, model, config: PiConfig, group=None, device: int | None = None,
                 use_graph: bool | None = None):
        import torch
        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.config = config
        self.model = model
        self.params = model.params
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.start, self.stop = shard_range(config.num_rollouts, self.rank, self.world)
        if self.stop <= self.start:
            raise ValueError("more ranks than rollout chunks")
        kind, param = model_kind(model)
        self.ctx = _abi.Context(self.device, self.stop - self.start, config.horizon_steps,
                                config.sub_rollouts, rollout_offset=self.start,
                                num_rollouts_total=config.num_rollouts)
        if kind == _abi.MODEL_HYBRID_LWPR:
            for a in range(3):
                stage_axis(self.ctx, a, model.models[a])
        self.ctx.call("pi2_select_model", kind, param)
        dev = torch.device("cuda", self.device)
        n = config.horizon_steps
        self.partial = torch.empty((n, _abi.PARTIAL_WIDTH), dtype=torch.float64, device=dev)
        self.gathered = torch.empty((self.world, n, _abi.PARTIAL_WIDTH), dtype=torch.float64, device=dev)
        self.nccl = dist.get_backend(group) == "nccl"
        self.use_graph = self.nccl if use_graph is None else bool(use_graph and self.nccl)
        self._graph = None
        self._graph_key = None
        self._bound = None
        self._plan_buf = np.empty((n, 4))
        self._state_buf = np.empty(12)
        self.graph_captures = 0

    def _bind(self, plan, cost_model) -> None:
        key = (np.asarray(plan.lo, float).tobytes(), np.asarray(plan.hi, float).tobytes(), _cost_key(cost_model))
        if key == self._bound and key[-1] is not None:
            return
        self.ctx.call("pi2_set_dynamics", dynamics_struct(self.params, plan.lo, plan.hi))
        apply_cost(self.ctx, cost_model)
        self._bound = key

    def _enqueue_step(self, iterations: int, temperature: float, stream) -> None:
        """The step's device work on ``stream``: pull, iterations with the exchange, push."""
        import torch.distributed as dist

        self.ctx.call("pi2_enqueue_pull", stream)
        for it in range(iterations):
            self.ctx.call("pi2_iterate_local_staged", it, temperature, _abi.ptr(self.partial), stream)
            dist.all_gather_into_tensor(self.gathered, self.partial, group=self.group)
            self.ctx.call("pi2_iterate_finalize", _abi.ptr(self.gathered), self.world, temperature, stream)
        self.ctx.call("pi2_enqueue_push", stream)

    def _capture(self, iterations: int, temperature: float):
        import torch
        import torch.distributed as dist

        # the communicator must exist before capture: one eager collective
        dist.all_gather_into_tensor(self.gathered, self.partial, group=self.group)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(self.device)
        with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
            self._enqueue_step(iterations, temperature, _abi.torch_stream(self.device))
        self.graph_captures += 1
        return g

    def step_device(self) -> None:
        """The staged step's device work on torch's current stream (the captured graph's
        replay with NCCL; eager otherwise); the plan lands in the pinned block."""
        cfg = self.config
        stream = _abi.torch_stream(self.device)
        temperature = float(cfg.temperature)
        if self.use_graph:
            key = (int(cfg.iterations_per_step), temperature)
            if self._graph is None or self._graph_key != key:
                self._graph, self._graph_key = self._capture(*key), key
            self._graph.replay()
        elif self.nccl:
            self._enqueue_step(int(cfg.iterations_per_step), temperature, stream)
        else:  # gloo: the exchange goes through the host
            self.ctx.call("pi2_enqueue_pull", stream)
            for it in range(cfg.iterations_per_step):
                self.ctx.call("pi2_iterate_local_staged", it, temperature, _abi.ptr(self.partial), stream)
                gathered = gather_partials(self.partial, self.group)
                self.ctx.call("pi2_iterate_finalize", _abi.ptr(gathered), self.world, temperature, stream)
            self.ctx.call("pi2_enqueue_push", stream)

    def optimize(self, state, plan: ControlPlan, cost_model, cycle_index: int = 0) -> ControlPlan:
        cfg = self.config
        if cfg.iterations_per_step == 0:
            return plan
        self._bind(plan, cost_model)
        args = optimize_args(cfg, cycle_index, use_graph=self.use_graph)
        st = self._state_buf
        st[0:3], st[3:6], st[6:9], st[9:12] = state.position, state.velocity, state.angles, state.rates
        self._plan_buf[...] = plan.controls
        self.ctx.call("pi2_stage_step", _abi.ptr(st), _abi.ptr(self._plan_buf), args)
        self.step_device()
        out = np.empty_like(self._plan_buf)
        self.ctx.call("pi2_fetch_plan", _abi.ptr(out), _abi.torch_stream(self.device))
        return plan.replaced(out)
