"""Device ms per control-step iteration (graph replays) over K for values of one
runtime switch, to place a size threshold.

    python profiles/micro/threshold_sweep.py --var PI2_PARTIALS_SPLIT --values 0,2 \
        --ks 4096,8192,16384,32768 [--L 100] [--M 1] [--T 50]
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
K, L, M, T = (int(v) for v in sys.argv[1:5])
params = P.QuadParams(); task = P.Task.default()
model = P.HybridModel.from_stacks(synthetic.hybrid_stacks(L, seed=0), params)
cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=T, iterations_per_step=1)
eng = P.RolloutEngine(model, cfg, device=0, noise="device")
state = P.QuadState.hover(task.spawn); plan = P.ControlPlan.hover(params, T)
P.receding_horizon_step(state, plan, cfg, model, P.RolloutCost(task, 1), 0, eng)
ctx = eng.context(K, T)
s = torch.cuda.Stream(0); sp = _abi.C.c_void_p(s.cuda_stream)
ctx.call("pi2_load_plan", _abi.ptr(state.as_array()), _abi.ptr(np.ascontiguousarray(plan.controls)), sp)
a = optimize_args(cfg, 0, True)
for i in range(5): ctx.call("pi2_iterate_device", a, sp)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = max(20, min(500, (1 << 22) // K))
e0.record(s)
for i in range(n): ctx.call("pi2_iterate_device", a, sp)
e1.record(s); s.synchronize()
print(f"{e0.elapsed_time(e1) / n:.4f}")
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--var", required=True)
    ap.add_argument("--values", required=True)
    ap.add_argument("--ks", required=True)
    ap.add_argument("--L", type=int, default=100)
    ap.add_argument("--M", type=int, default=1)
    ap.add_argument("--T", type=int, default=50)
    a = ap.parse_args()
    vals = a.values.split(",")
    print(f"{a.var} in {vals}; L={a.L} M={a.M} T={a.T}: device ms per iteration")
    for K in (int(k) for k in a.ks.split(",")):
        row = []
        for v in vals:
            env = dict(os.environ, **{a.var: v})
            out = subprocess.run([sys.executable, "-c", CODE, str(K), str(a.L), str(a.M), str(a.T)], env=env,
                                 capture_output=True, text=True, check=True)
            row.append(f"{a.var}={v}: {float(out.stdout.strip().splitlines()[-1]):.4f}")
        print(f"K={K:7d}  " + "  ".join(row), flush=True)


if __name__ == "__main__":
    main()
