import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1503_00330_b200 as P
from paper_1503_00330_b200 import synthetic
from tests._cases import load, stacks_from
z = load("trial")
p = P.QuadParams()
model = P.HybridModel.from_stacks(stacks_from(z, "hybrid_"), p)
K, M, N = int(z["hybrid_K"]), int(z["hybrid_M"]), int(z["hybrid_N"])
res = {}
for pdl in ("1", "0"):
    os.environ["PI2_PDL"] = pdl
    cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=N, iterations_per_step=1)
    eng = P.RolloutEngine(model, cfg, device=0)
    task = P.Task.default()
    outs = []
    for cyc in range(4):
        noise = P.sample_noise(cfg, cyc, 0)
        dyn = P.sample_dynamics_noise(cfg, cyc, 0) if M > 1 else None
        b = eng.evaluate(P.QuadState.hover(task.spawn), P.ControlPlan.hover(p, N), noise, P.RolloutCost(task, 1), dyn)
        outs.append(b.costs_to_go.copy())
    # K=1 probe engine and predict
    probe = P.RolloutEngine(model, P.PiConfig(num_rollouts=1, sub_rollouts=1, horizon_steps=N, iterations_per_step=1), device=0)
    pb = probe.evaluate(P.QuadState.hover(task.spawn), P.ControlPlan.hover(p, N), np.zeros((1, N, 4)), P.RolloutCost(task, 1))
    outs.append(pb.costs_to_go.copy())
    res[pdl] = outs
for i, (a, b) in enumerate(zip(res["1"], res["0"])):
    d = np.abs(a - b); print(i, a.shape, "max diff", d.max(), "rows differing", int((d.max(axis=1) > 0).sum()))
