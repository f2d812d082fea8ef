"""BASELINE C5 as specified: K = 2^10 ... 2^22 rollouts, T=50, L=200, M=1, one B200.

Per K: device time per control-step iteration (back-to-back replays of the
iteration graph on the device-resident plan, CUDA events), the throughput in
rollout-steps/s, and the end-to-end p50 latency of `receding_horizon_step`
(host state and plan in, control and shifted plan out).

    python profiles/k_sweep.py [--T 50] [--L 200] [--M 1] [--min-log2 10] [--max-log2 22]
"""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_00330_b200 as P  # noqa: E402
from paper_1503_00330_b200 import _abi, synthetic  # noqa: E402
from paper_1503_00330_b200.controller import optimize_args  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=50)
    ap.add_argument("--L", type=int, default=200)
    ap.add_argument("--M", type=int, default=1)
    ap.add_argument("--min-log2", type=int, default=10)
    ap.add_argument("--max-log2", type=int, default=22)
    a = ap.parse_args()
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(synthetic.hybrid_stacks(a.L, seed=0), params)
    task = P.Task.default()
    state = P.QuadState.hover(task.spawn)
    plan0 = P.ControlPlan.hover(params, a.T)
    cost = P.RolloutCost(task, 1)
    print(f"T={a.T} L={a.L} M={a.M}; device: back-to-back graph replays; e2e: receding_horizon_step p50")
    print(f"{'K':>9} {'ms/step':>9} {'G rollout-steps/s':>18} {'e2e p50 ms':>11}")
    for lk in range(a.min_log2, a.max_log2 + 1, 2):
        K = 1 << lk
        cfg = P.PiConfig(num_rollouts=K, sub_rollouts=a.M, horizon_steps=a.T, iterations_per_step=1)
        eng = P.RolloutEngine(model, cfg, device=0, noise="device")
        steps = max(10, min(2000, (1 << 24) // (K * a.T // 64 + 1)))
        # end to end (also binds dynamics/cost and warms the graph)
        for i in range(5):
            P.receding_horizon_step(state, plan0, cfg, model, cost, i, eng)
        lat = []
        for i in range(min(steps, 200)):
            t0 = time.perf_counter()
            P.receding_horizon_step(state, plan0, cfg, model, cost, i, eng)
            lat.append(time.perf_counter() - t0)
        e2e = float(np.median(lat) * 1e3)
        # device: the iteration graph back to back
        ctx = eng.context(K, a.T)
        s = torch.cuda.Stream(0)
        sptr = _abi.C.c_void_p(s.cuda_stream)
        ctx.call("pi2_load_plan", _abi.ptr(state.as_array()), _abi.ptr(np.ascontiguousarray(plan0.controls)), sptr)
        args = optimize_args(cfg, 0, True)
        for i in range(3):
            ctx.call("pi2_iterate_device", args, sptr)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(steps):
            ctx.call("pi2_iterate_device", args, sptr)
        e1.record(s)
        s.synchronize()
        ms = e0.elapsed_time(e1) / steps
        print(f"{K:>9} {ms:9.4f} {K * a.T / (ms / 1e3) / 1e9:18.3f} {e2e:11.4f}", flush=True)
        del eng, ctx
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
