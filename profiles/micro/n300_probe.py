import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1503_00330_b200 as P
from paper_1503_00330_b200 import synthetic
from oracle import rollout as RO
from tests._cases import TASK_OBSTACLES, TASK_WAYPOINTS
K, N, L, M = 17000, 300, 16, 1
stacks = synthetic.hybrid_stacks(L, seed=K + N)
params = P.QuadParams(); model = P.HybridModel.from_stacks(stacks, params)
cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=N, iterations_per_step=1, rng_seed=K)
task = P.Task.default(); state = P.QuadState.hover(task.spawn + np.array([0.05, -0.1, 0.07])); plan = P.ControlPlan.hover(params, N)
noise = P.sample_noise(cfg, 1, 0)
b = P.RolloutEngine(model, cfg, device=0).evaluate(state, plan, noise, P.RolloutCost(task, 2), None)
om = RO.Model(stacks); lo, hi = om.dyn.bounds()
rc, rf = RO.evaluate(om, state.as_array(), plan.controls, lo, hi, noise, RO.Cost(TASK_WAYPOINTS[2], TASK_OBSTACLES), None, M)
rel = np.abs(b.costs_to_go - rc) / np.maximum(np.abs(rc), 1e-300)
i = np.unravel_index(rel.argmax(), rel.shape)
print(os.environ.get("PI2_LWPR_TC", "1"), "max rel", rel.max(), "at", i, "cost", rc[i], "t<=100 max", rel[:, :100].max(), "crash frac", rf.mean(), "rel>1e-5 count", int((rel > 1e-5).sum()))
