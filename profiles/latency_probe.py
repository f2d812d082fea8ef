"""Host-overhead probe: where the end-to-end control-step latency goes.

    python profiles/latency_probe.py [--config C2] [--steps 200] [--cprofile]

Prints p50 latency of (1) the public API `receding_horizon_step`, (2) the bare
C-ABI `pi2_optimize` call with host state/plan (ctypes), (3) one synchronous
`pi2_iterate_device` graph launch on the device-resident plan, and (4) the
per-step device time of back-to-back graph launches (bench.py's `value`).
"""

import argparse
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_00330_b200 as P  # noqa: E402
from paper_1503_00330_b200 import _abi, synthetic  # noqa: E402
from paper_1503_00330_b200.controller import optimize_args  # noqa: E402


def p50(f, n):
    lat = []
    for i in range(n):
        t0 = time.perf_counter()
        f(i)
        lat.append(time.perf_counter() - t0)
    return float(np.median(lat) * 1e3)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--cprofile", action="store_true")
    a = ap.parse_args()
    c = synthetic.CONFIGS[a.config]
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(synthetic.hybrid_stacks(c["L"], seed=0), params)
    task = P.Task.default()
    cfg = P.PiConfig(num_rollouts=c["K"], sub_rollouts=c["M"], horizon_steps=c["T"], iterations_per_step=1)
    eng = P.RolloutEngine(model, cfg, device=0, noise="device")
    state = P.QuadState.hover(task.spawn)
    plan0 = P.ControlPlan.hover(params, c["T"])
    cost = P.RolloutCost(task, 1)
    for i in range(10):
        P.receding_horizon_step(state, plan0, cfg, model, cost, i, eng)
    torch.cuda.synchronize()

    api = p50(lambda i: P.receding_horizon_step(state, plan0, cfg, model, cost, i, eng), a.steps)
    box = [plan0]

    def evolving(i):  # bench.py's e2e loop: each step starts from the previous shifted plan
        box[0] = P.receding_horizon_step(state, box[0], cfg, model, cost, i, eng)[1]

    api_evolving = p50(evolving, a.steps)

    ctx = eng.context(c["K"], c["T"])
    st = np.ascontiguousarray(state.as_array())
    pl = np.ascontiguousarray(plan0.controls).copy()
    args = optimize_args(cfg, 0, True)

    def bare(i):
        pl[:] = plan0.controls
        ctx.call("pi2_optimize", _abi.ptr(st), _abi.ptr(pl), args)

    bare_ms = p50(bare, a.steps)

    s = torch.cuda.Stream(0)
    sptr = _abi.C.c_void_p(s.cuda_stream)
    ctx.call("pi2_load_plan", _abi.ptr(st), _abi.ptr(pl), sptr)

    def one_graph(i):
        ctx.call("pi2_iterate_device", args, sptr)
        s.synchronize()

    graph_sync = p50(one_graph, a.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for i in range(a.steps):
        ctx.call("pi2_iterate_device", args, sptr)
    e1.record(s)
    s.synchronize()
    b2b = e0.elapsed_time(e1) / a.steps
    print(f"{a.config}: api p50 {api:.4f} ms (evolving plan {api_evolving:.4f}) | bare pi2_optimize {bare_ms:.4f} | one graph + sync "
          f"{graph_sync:.4f} | back-to-back device {b2b:.4f} ms/step")
    if a.cprofile:
        pr = cProfile.Profile()
        pr.enable()
        for i in range(a.steps):
            P.receding_horizon_step(state, plan0, cfg, model, cost, i, eng)
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(14)


if __name__ == "__main__":
    main()
