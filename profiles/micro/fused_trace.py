"""Phase trace of fused_step_kernel (library built with -DPI2_TC_TRACE): per SM sub-partition the time
share with n warps in the exp phase, and per warp the clocks per step spent in each phase.

    PI2_NVCC_EXTRA=-DPI2_TC_TRACE python -c "from paper_1503_00330_b200 import _build; _build.build(force=True)"
    python profiles/micro/fused_trace.py --config C2
"""
import argparse
import ctypes
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_1503_00330_b200 as P  # noqa: E402
from paper_1503_00330_b200 import _abi, synthetic  # noqa: E402
from paper_1503_00330_b200.controller import dynamics_struct, optimize_args  # noqa: E402
from paper_1503_00330_b200.simworld import cost_struct  # noqa: E402

NAMES = {1: "barrier", 8: "issue", 5: "finalize", 6: "rollout", 7: "attitude", 0: "features", 2: "mma-wait", 3: "exp",
         4: "tail"}
CAP = 4096


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
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
    lib = _abi.lib()
    ms = (ctypes.c_double * 5)()
    ctx.call("pi2_profile_iteration", optimize_args(cfg, 0, use_graph=False), 1, ms)
    lib.pi2_debug_trace_arm(1)
    ctx.call("pi2_profile_iteration", optimize_args(cfg, 0, use_graph=False), 1, ms)
    lib.pi2_debug_trace_arm(0) if False else None
    buf = np.zeros(64 * CAP, np.uint64)
    lib.pi2_debug_trace_read(buf.ctypes.data_as(ctypes.c_void_p))
    lib.pi2_debug_trace_arm(0)
    print(a.config, "stage ms:", [round(x, 4) for x in ms[:]])
    ev = buf[buf != 0]
    clk = (ev >> np.uint64(20)).astype(np.int64)
    wid = ((ev >> np.uint64(4)) & np.uint64(63)).astype(np.int64)
    cta = ((ev >> np.uint64(10)) & np.uint64(0x3FF)).astype(np.int64)
    ph = (ev & np.uint64(15)).astype(np.int64)
    order = np.argsort(clk, kind="stable")
    clk, wid, cta, ph = clk[order], wid[order], cta[order], ph[order]
    last = {}
    ivs = []  # (start, end, warp, phase)
    for t, w, b, p in zip(clk, wid, cta, ph):
        key = (w, b)
        if key in last:
            ivs.append((last[key], t, w, p))
        last[key] = t
    t0 = min(i[0] for i in ivs)
    t1 = max(i[1] for i in ivs)
    T = t1 - t0
    for sp in range(4):
        d = []
        tot = defaultdict(float)
        for s, e, w, p in ivs:
            if w % 4 != sp:
                continue
            tot[p] += e - s
            if p == 3:
                d += [(s, 1), (e, -1)]
        d.sort()
        hist = [0.0] * 6
        k, prev = 0, t0
        for x, dd in d:
            hist[min(k, 5)] += x - prev
            prev, k = x, k + dd
        hist[0] += t1 - prev
        nwarps = len({(w, b) for s, e, w, p in ivs if w % 4 == sp and True} or [1])
        print(f"SMSP {sp} ({T} clk): n warps in exp " + " ".join(f"{i}:{h / T:.2f}" for i, h in enumerate(hist[:5])) +
              " | per-warp share: " + " ".join(f"{NAMES.get(p, p)} {v / T / max(nwarps / 1, 1):.3f}"
                                              for p, v in sorted(tot.items(), key=lambda x: -x[1])))


if __name__ == "__main__":
    main()
