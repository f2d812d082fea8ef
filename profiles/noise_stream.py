"""Driver for the noise-stream ncu evidence: the host-noise evaluate path of a config
(the reference's exploration noise (K,N,4) f64 and, for M > 1, dynamics noise
(K,M,N,3) f32, resident in HBM, controller.py:112-139) -- the attitude kernel streams
the first, the rollout/cost kernel the second.

    python profiles/noise_stream.py [--config C2] [--reps 3]
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
        -k regex:"attitude|rollout" python profiles/noise_stream.py --reps 1

Prints the CUDA-event stage times (pi2_profile_evaluate) and the noise GB/s.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_00330_b200 as P  # noqa: E402
from paper_1503_00330_b200 import _abi, synthetic  # noqa: E402
from paper_1503_00330_b200.controller import dynamics_struct  # noqa: E402
from paper_1503_00330_b200.simworld import cost_struct  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    c = synthetic.CONFIGS[a.config]
    K, T, L, M = c["K"], c["T"], c["L"], c["M"]
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(synthetic.hybrid_stacks(L, seed=0), params)
    cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=T, iterations_per_step=1)
    task = P.Task.default()
    eng = P.RolloutEngine(model, cfg, device=0)
    ctx = eng.context(K, T)
    plan = P.ControlPlan.hover(params, T)
    ctx.call("pi2_set_dynamics", dynamics_struct(params, plan.lo, plan.hi))
    ctx.call("pi2_set_cost", cost_struct(P.RolloutCost(task, 1)))
    g = torch.Generator(device="cuda:0")
    g.manual_seed(0)
    eps = torch.randn((K, T, 4), dtype=torch.float64, device="cuda:0", generator=g) * torch.tensor(
        cfg.exploration_std, dtype=torch.float64, device="cuda:0")
    dyn = torch.randn((K, M, T, 3), dtype=torch.float32, device="cuda:0", generator=g) if M > 1 else None
    torch.cuda.synchronize()
    ms = (_abi.C.c_double * 3)()
    ctx.call("pi2_profile_evaluate", _abi.ptr(P.QuadState.hover(task.spawn).as_array()),
             _abi.ptr(np.ascontiguousarray(plan.controls)), _abi.ptr(eps), _abi.ptr(dyn), a.reps, ms)
    att, lw, roll = list(ms)
    out = {"config": a.config, "attitude_ms": att, "lwpr_ms": lw, "rollout_ms": roll,
           "eps_gbs": K * T * 32 / (att * 1e-3) / 1e9}
    if dyn is not None:
        out["dyn_gbs"] = K * M * T * 12 / (roll * 1e-3) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
