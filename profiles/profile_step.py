"""Minimal driver for ncu captures: a few device-noise control-step iterations of a config.

    python profiles/profile_step.py [--config C2] [--iters 3]

Launch order per iteration: attitude_kernel, lwpr_kernel, rollout_kernel,
partials_kernel, combine_kernel (local root), combine_kernel (finalize).
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1503_00330_b200 as P  # noqa: E402
from paper_1503_00330_b200 import _abi, synthetic  # noqa: E402
from paper_1503_00330_b200.controller import dynamics_struct, optimize_args  # noqa: E402
from paper_1503_00330_b200.simworld import cost_struct  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    c = synthetic.CONFIGS[a.config]
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(synthetic.hybrid_stacks(c["L"], seed=0), params)
    cfg = P.PiConfig(num_rollouts=c["K"], sub_rollouts=c["M"], horizon_steps=c["T"], iterations_per_step=1)
    task = P.Task.default()
    eng = P.RolloutEngine(model, cfg, device=0, noise="device", use_graph=False)
    ctx = eng.context(c["K"], c["T"])
    plan = P.ControlPlan.hover(params, c["T"])
    ctx.call("pi2_set_dynamics", dynamics_struct(params, plan.lo, plan.hi))
    ctx.call("pi2_set_cost", cost_struct(P.RolloutCost(task, 1)))
    ctx.call("pi2_load_plan", _abi.ptr(P.QuadState.hover(task.spawn).as_array()),
             _abi.ptr(np.ascontiguousarray(plan.controls)), None)
    import ctypes

    for it in range(a.iters):
        ctx.call("pi2_profile_iteration", optimize_args(cfg, it, use_graph=False), 1,
                 (ctypes.c_double * 5)())
    out = np.empty((c["T"], 4))
    ctx.call("pi2_read_plan", _abi.ptr(out), None)
    assert np.all(np.isfinite(out))
    print("ok", a.config, a.iters)


if __name__ == "__main__":
    main()
