"""attitude stage time vs K: attitude_quad_kernel (quad of lanes per rollout) against
attitude_kernel (thread per rollout), from pi2_profile_iteration's CUDA events.

    python profiles/attitude_sweep.py
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1503_00330_b200 as P  # noqa: E402
from paper_1503_00330_b200 import _abi, synthetic  # noqa: E402
from paper_1503_00330_b200.controller import dynamics_struct, optimize_args  # noqa: E402
from paper_1503_00330_b200.simworld import cost_struct  # noqa: E402


def stage_ms(K, M, quad):
    os.environ["PI2_ATT_QUAD_MAXK"] = str(1 << 30 if quad else 0)
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(synthetic.hybrid_stacks(100, seed=0), params)
    cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=50, iterations_per_step=1)
    task = P.Task.default()
    eng = P.RolloutEngine(model, cfg, device=0, noise="device", use_graph=False)
    ctx = eng.context(K, 50)
    plan = P.ControlPlan.hover(params, 50)
    ctx.call("pi2_set_dynamics", dynamics_struct(params, plan.lo, plan.hi))
    ctx.call("pi2_set_cost", cost_struct(P.RolloutCost(task, 1)))
    ctx.call("pi2_load_plan", _abi.ptr(P.QuadState.hover(task.spawn).as_array()),
             _abi.ptr(np.ascontiguousarray(plan.controls)), None)
    out = (ctypes.c_double * 5)()
    ctx.call("pi2_profile_iteration", optimize_args(cfg, 0, use_graph=False), 3, out)
    ctx.call("pi2_profile_iteration", optimize_args(cfg, 0, use_graph=False), 20, out)
    return list(out)


for K in (32768, 65536, 131072, 262144, 524288, 1048576):
    q, t = stage_ms(K, 1, True), stage_ms(K, 1, False)
    print(f"K {K:8d}: attitude quad {q[0] * 1e3:7.1f} us   thread {t[0] * 1e3:7.1f} us   (step stages quad {sum(q):.4f} ms, thread {sum(t):.4f} ms)")
