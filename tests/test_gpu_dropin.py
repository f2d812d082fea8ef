"""The GPU engine dropped into the REAL reference package (``pimpc``).

The reference is imported from ``baseline/_ref`` (installed from /root/reference
with pip --target; it travels to the GPU box with the repo) or from the source
tree; without it these tests skip with the reason.  Nothing here restates the
reference: its own ``optimize``, ``receding_horizon_step`` and ``run_trial``
(controller.py:374-413, simworld.py:270-380) run with this package's
``RolloutEngine`` injected through the seams they expose (``engine=`` and the
function-local import in run_trial, simworld.py:288-307), on the reference's own
model, cost, state and plan objects.
"""

import numpy as np
import pytest

import paper_1503_00330_b200 as B
from paper_1503_00330_b200 import dropin, synthetic
from tests._cases import load, stacks_from

pytestmark = pytest.mark.gpu

REF = synthetic.import_reference()
needs_ref = pytest.mark.skipif(REF is None, reason="reference package pimpc not importable "
                               "(baseline/_ref missing: pip install --target baseline/_ref /root/reference)")

COST_RTOL = 1e-5
DU_TOL = 1e-4


def du_err(new, want, plan):
    du, wdu = new - plan, want - plan
    return np.max(np.abs(du - wdu), axis=0) / np.maximum(np.max(np.abs(wdu), axis=0), 1e-300)


def ref_state(vec):
    v = np.asarray(vec, float)
    return REF.dynamics.QuadState(v[0:3], v[3:6], v[6:9], v[9:12])


@needs_ref
def test_reference_optimize_with_gpu_engine_matches_golden():
    """pimpc.controller.optimize / receding_horizon_step with engine=B.RolloutEngine
    (the reference's host noise and numpy update, our rollouts) against the golden
    outputs of the reference's own engine."""
    z = load("optimize")
    model = synthetic.reference_hybrid(REF, stacks_from(z))
    C = REF.controller
    cfg = C.PiConfig(num_rollouts=int(z["K"]), sub_rollouts=int(z["M"]), horizon_steps=int(z["N"]),
                     iterations_per_step=int(z["iterations"]), rng_seed=int(z["seed"]), chunk_size=16)
    task = REF.simworld.Task.default()
    state = ref_state(z["state"])
    plan = C.ControlPlan.hover(REF.dynamics.QuadParams(), int(z["N"]))
    cost = REF.simworld.RolloutCost(task, int(z["waypoint_index"]))
    eng = B.RolloutEngine(model, cfg, device=0)
    opt = C.optimize(state, plan, cfg, model, cost, cycle_index=int(z["cycle"]), engine=eng)
    assert isinstance(opt, C.ControlPlan)  # the reference's own loop produced it
    assert np.all(du_err(opt.controls, z["optimized"], z["plan"]) < DU_TOL)
    ctrl, carried = C.receding_horizon_step(state, plan, cfg, model, cost, cycle_index=int(z["cycle"]), engine=eng)
    np.testing.assert_allclose(ctrl.as_array(), z["control"], rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(carried.controls, z["carried"], rtol=1e-4, atol=1e-6)


@needs_ref
@pytest.mark.parametrize("K,L,M", [(4096, 100, 4), (3000, 100, 1)])
def test_reference_engine_and_gpu_engine_same_run(K, L, M):
    """The reference's RolloutEngine and ours on identical inputs in the same run (the
    reference's host noise streams): costs within 1e-5 relative, crash flags exact,
    and the reference's path_integral_update of either batch within the Δu gate."""
    C = REF.controller
    stacks = synthetic.hybrid_stacks(L, seed=K + M)
    model = synthetic.reference_hybrid(REF, stacks)
    cfg = C.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=50, iterations_per_step=1, rng_seed=11)
    task = REF.simworld.Task.default()
    state = ref_state(np.r_[task.spawn + [0.04, -0.03, 0.02], np.zeros(9)])
    plan = C.ControlPlan.hover(REF.dynamics.QuadParams(), 50)
    cost = REF.simworld.RolloutCost(task, 1)
    noise = C.sample_noise(cfg, 2, 0)
    dyn = C.sample_dynamics_noise(cfg, 2, 0) if M > 1 else None
    want = C.RolloutEngine(model, cfg).evaluate(state, plan, noise, cost, dyn)
    got = B.RolloutEngine(model, cfg, device=0).evaluate(state, plan, noise, cost, dyn)
    np.testing.assert_array_equal(got.crash_flags, want.crash_flags)
    rel = np.abs(got.costs_to_go - want.costs_to_go) / np.abs(want.costs_to_go)
    assert rel.max() < COST_RTOL
    new = C.path_integral_update(plan, got, cfg.temperature)
    ref_new = C.path_integral_update(plan, want, cfg.temperature)
    assert np.all(du_err(new.controls, ref_new.controls, plan.controls) < DU_TOL)
    # our device update of the reference's batch: the same gate
    dev_new = B.path_integral_update(plan, want, cfg.temperature)
    assert np.all(du_err(dev_new.controls, ref_new.controls, plan.controls) < DU_TOL)


def trial_case(z, name):
    p = REF.dynamics.QuadParams()
    if name == "analytic":
        model = REF.dynamics.AnalyticModel(p)
    else:
        model = synthetic.reference_hybrid(REF, stacks_from(z, "hybrid_"), p)
    cfg = REF.controller.PiConfig(num_rollouts=int(z[f"{name}_K"]), sub_rollouts=int(z[f"{name}_M"]),
                                  horizon_steps=int(z[f"{name}_N"]),
                                  iterations_per_step=int(z[f"{name}_iters"]),
                                  temperature=float(z[f"{name}_temperature"]))
    gt = REF.dynamics.PerturbedModel(p, drag_coeff=0.08, thrust_scale=0.97)
    return model, cfg, gt, int(z[f"{name}_seed"]), int(z[f"{name}_cap"])


@needs_ref
@pytest.mark.parametrize("replace_step", [False, True])
@pytest.mark.parametrize("name", ["analytic", "hybrid"])
def test_reference_run_trial_on_gpu_engine_matches_golden(name, replace_step):
    """The reference's run_trial with pimpc.controller.RolloutEngine patched (and, with
    replace_step, receding_horizon_step: the update on the GPU too), reference noise:
    the flight log matches the golden trial of the unpatched reference up to the
    float32 drift of the rollout costs, amplified a little by the closed loop."""
    z = load("trial")
    model, cfg, gt, seed, cap = trial_case(z, name)
    with dropin.patched(REF.controller, noise="reference", device=0, replace_step=replace_step):
        r = REF.simworld.run_trial(REF.simworld.Task.default(), cfg, model, gt, seed=seed, step_cap=cap)
    want = z[f"{name}_rows"]
    assert r.outcome == str(z[f"{name}_outcome"]) and r.steps == int(z[f"{name}_steps"])
    got = r.log_rows
    assert got.shape == want.shape
    np.testing.assert_allclose(got[:, 1:13], want[:, 1:13], rtol=1e-4, atol=1e-5)    # states
    np.testing.assert_allclose(got[:, 13:17], want[:, 13:17], rtol=1e-3, atol=1e-4)  # controls
    np.testing.assert_allclose(got[:, 21], want[:, 21], rtol=1e-4)                    # q cost
    np.testing.assert_allclose(got[:, 22], want[:, 22], rtol=1e-3)                    # plan horizon cost
    assert r.total_cost == pytest.approx(float(z[f"{name}_total_cost"]), rel=1e-4)
    if name == "hybrid":
        np.testing.assert_allclose(got[:, 23:26], want[:, 23:26], rtol=1e-3, atol=1e-5)  # LWPR variance log


@needs_ref
def test_reference_run_trial_real_time_mode():
    """Real-time mode inside the reference's closed loop: device noise, every control step
    one CUDA graph; the trial flies (finite log, no crash) and each step's host-in /
    control-out latency is well inside the 20 ms budget."""
    z = load("trial")
    model, cfg, gt, seed, cap = trial_case(z, "hybrid")
    times = []
    with dropin.patched(REF.controller, noise="device", device=0, step_times=times):
        r = REF.simworld.run_trial(REF.simworld.Task.default(), cfg, model, gt, seed=seed, step_cap=cap)
    assert r.outcome == "timeout" and r.steps == cap
    assert np.all(np.isfinite(r.log_rows))
    assert len(times) == cap and np.median(times) < 0.01
