"""Warp-per-rollout ('wide') vs thread-per-rollout attitude/rollout kernels around the
K threshold (PI2_WIDE_MAX_K): device ms per control-step iteration, graph replays.

    python profiles/micro/wide_threshold.py [--L 100] [--M 1]
"""
import argparse
import os
import subprocess
import sys

CODE = r'''
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1503_00330_b200 as P
from paper_1503_00330_b200 import _abi, synthetic
from paper_1503_00330_b200.controller import optimize_args
K, L, M = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
params = P.QuadParams(); task = P.Task.default()
model = P.HybridModel.from_stacks(synthetic.hybrid_stacks(L, seed=0), params)
cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=50, iterations_per_step=1)
eng = P.RolloutEngine(model, cfg, device=0, noise="device")
state = P.QuadState.hover(task.spawn); plan = P.ControlPlan.hover(params, 50)
P.receding_horizon_step(state, plan, cfg, model, P.RolloutCost(task, 1), 0, eng)
ctx = eng.context(K, 50)
s = torch.cuda.Stream(0); sp = _abi.C.c_void_p(s.cuda_stream)
ctx.call("pi2_load_plan", _abi.ptr(state.as_array()), _abi.ptr(np.ascontiguousarray(plan.controls)), sp)
a = optimize_args(cfg, 0, True)
for i in range(5): ctx.call("pi2_iterate_device", a, sp)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 300
e0.record(s)
for i in range(n): ctx.call("pi2_iterate_device", a, sp)
e1.record(s); s.synchronize()
print(f"{e0.elapsed_time(e1) / n:.4f}")
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=100)
    ap.add_argument("--M", type=int, default=1)
    a = ap.parse_args()
    print(f"L={a.L} M={a.M} T=50: device ms per iteration, wide (warp per rollout) vs thread per rollout")
    for K in [int(k) for k in os.environ.get("KS", "1024,2048,4096,8192,12288,16384").split(",")]:
        res = {}
        for mode, thr in (("wide", str(1 << 30)), ("thread", "0")):
            env = dict(os.environ, PI2_WIDE_MAX_K=thr)
            out = subprocess.run([sys.executable, "-c", CODE, str(K), str(a.L), str(a.M)], env=env,
                                 capture_output=True, text=True, check=True)
            res[mode] = float(out.stdout.strip().splitlines()[-1])
        print(f"K={K:6d}  wide {res['wide']:.4f}  thread {res['thread']:.4f}", flush=True)


if __name__ == "__main__":
    main()
