"""A/B of a rollout-kernel knob on one config: device ms of the rollout stage and bitwise costs.

    python profiles/micro/roll_variant.py --env PI2_SOME_KNOB --config C2

Two device-noise engines (knob 0 / 1, read at context creation) evaluate the same state/plan;
costs-to-go and crash flags are compared bit for bit; the per-stage CUDA-event times of
pi2_profile_iteration (attitude, lwpr, rollout, partials, combine) are averaged over reps.
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_1503_00330_b200 as P  # noqa: E402
from paper_1503_00330_b200 import _abi, synthetic  # noqa: E402
from paper_1503_00330_b200.controller import dynamics_struct, optimize_args  # noqa: E402
from paper_1503_00330_b200.simworld import cost_struct  # noqa: E402


def run(env, val, c, reps):
    os.environ[env] = str(val)
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
    st = np.zeros(5)
    for it in range(reps + 2):
        ms = (ctypes.c_double * 5)()
        ctx.call("pi2_profile_iteration", optimize_args(cfg, 0, use_graph=False), 1, ms)
        if it >= 2:
            st += np.array(ms[:])
    # one device-noise evaluate (the iteration's kernels) for the bitwise check
    import torch
    costs = torch.empty((c["K"], c["T"]), dtype=torch.float64, device="cuda")
    crash = torch.empty((c["K"],), dtype=torch.uint8, device="cuda")
    ctx.call("pi2_evaluate_device_noise", _abi.ptr(P.QuadState.hover(task.spawn).as_array()),
             _abi.ptr(np.ascontiguousarray(plan.controls)), optimize_args(cfg, 0, use_graph=False), 0,
             _abi.ptr(costs), _abi.ptr(crash), _abi.torch_stream(0))
    torch.cuda.synchronize()
    return st / reps, costs.cpu().numpy(), crash.cpu().numpy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--env", default="PI2_ROLL_QUAD")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    c = synthetic.CONFIGS[a.config]
    r0 = run(a.env, 0, c, a.reps)
    r1 = run(a.env, 1, c, a.reps)
    names = ["attitude", "lwpr", "rollout", "partials", "combine"]
    for v, r in ((0, r0), (1, r1)):
        print(f"{a.env}={v} {a.config}: " + " ".join(f"{n} {t * 1e3:.1f}us" for n, t in zip(names, r[0])))
    print("costs bitwise equal:", np.array_equal(r0[1].view(np.uint64), r1[1].view(np.uint64)),
          "crash equal:", np.array_equal(r0[2], r1[2]))


if __name__ == "__main__":
    main()
