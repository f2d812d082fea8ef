"""Host-overhead probe: C1 receding_horizon_step latency through the public API + cProfile."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, cProfile, pstats
import paper_1503_00330_b200 as P
from paper_1503_00330_b200 import synthetic
params = P.QuadParams()
model = P.HybridModel.from_stacks(synthetic.hybrid_stacks(100, seed=0), params)
task = P.Task.default()
cfg = P.PiConfig(num_rollouts=1024, sub_rollouts=1, horizon_steps=50, iterations_per_step=1)
eng = P.RolloutEngine(model, cfg, noise="device")
state = P.QuadState.hover(task.spawn); plan = P.ControlPlan.hover(params, 50); cost = P.RolloutCost(task, 1)
for i in range(20): P.receding_horizon_step(state, plan, cfg, model, cost, i, eng)
lat = []
for i in range(200):
    t0 = time.perf_counter(); ctrl, plan = P.receding_horizon_step(state, plan, cfg, model, cost, i, eng); lat.append(time.perf_counter() - t0)
lat = np.array(lat) * 1e3
print("C1 e2e ms p50 %.4f p99 %.4f" % (np.median(lat), np.percentile(lat, 99)))
pr = cProfile.Profile(); pr.enable()
for i in range(200): P.receding_horizon_step(state, plan, cfg, model, cost, i, eng)
pr.disable(); pstats.Stats(pr).sort_stats('cumulative').print_stats(18)
