"""Parity of the CUDA path (through the C ABI) with the reference and the oracle.

Gates (BASELINE.json north star): per-rollout costs-to-go within 1e-5
relative, crash flags exact, control update Δu within 1e-4 per channel
(normalised by the channel's max |Δu|).  Golden fixtures
come from the real reference (tests/golden/make_golden.py); larger cases
compare against the numpy oracle run on this host.
"""

import threading

import numpy as np
import pytest

import paper_1503_00330_b200 as P
from paper_1503_00330_b200 import _abi, synthetic
from oracle import lwpr as OL
from oracle import rollout as RO
from tests._cases import TASK_OBSTACLES, TASK_WAYPOINTS, eval_case_names, load, stacks_from

pytestmark = pytest.mark.gpu

COST_RTOL = 1e-5
DU_TOL = 1e-4


def cost_rel_err(got, want):
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)))


def du_err(new, want, plan):
    """Per-channel max |Δu error| / max |Δu|; NaN plan entries (NaN exploration noise,
    controller.py:368-371) must sit at the same places and are excluded."""
    np.testing.assert_array_equal(np.isnan(new), np.isnan(want))
    ok = ~np.isnan(want)
    du, wdu = np.where(ok, new - plan, 0.0), np.where(ok, want - plan, 0.0)
    scale = np.maximum(np.max(np.abs(wdu), axis=0), 1e-300)
    return np.max(np.abs(du - wdu), axis=0) / scale


def model_of(z):
    if bool(z["analytic"]):
        return P.AnalyticModel(P.QuadParams())
    return P.HybridModel.from_stacks(stacks_from(z), P.QuadParams())


def gpu_eval(z, model=None, engine_kw=None):
    M = int(z["M"])
    model = model or model_of(z)
    cfg = P.PiConfig(num_rollouts=int(z["K"]), sub_rollouts=M, horizon_steps=int(z["N"]), iterations_per_step=1,
                     exploration_std=z["std"], rng_seed=int(z["seed"]))
    eng = P.RolloutEngine(model, cfg, device=0, **(engine_kw or {}))
    task = P.Task.default()
    plan = P.ControlPlan(z["plan"], 0.02, 0.0, *P.QuadParams().control_bounds())
    dyn = z["dyn"] if z["dyn"].size else None
    b = eng.evaluate(P.QuadState.from_array(z["state"]), plan, z["noise"],
                     P.RolloutCost(task, int(z["waypoint_index"])), dyn)
    return b, plan


def test_device_present():
    assert _abi.device_count() >= 1, "GPU tests need a CUDA device"


@pytest.mark.parametrize("name", eval_case_names())
def test_evaluate_matches_reference_golden(name):
    z = load("eval_" + name)
    b, plan = gpu_eval(z)
    want = z["costs"]
    ceil = want == float(z["ceiling"])
    np.testing.assert_array_equal(b.costs_to_go == float(z["ceiling"]), ceil)
    np.testing.assert_array_equal(b.crash_flags, z["crash"])
    if (~ceil).any():
        assert cost_rel_err(b.costs_to_go[~ceil], want[~ceil]) < COST_RTOL
    new = P.path_integral_update(plan, b, float(z["temperature"]))
    assert np.all(du_err(new.controls, z["new_plan"], z["plan"]) < DU_TOL)


# K <= 8192 runs the warp-per-rollout (latency) kernels, larger K the
# thread-per-rollout / lane-per-sub-rollout ones: both are covered.
@pytest.mark.parametrize("K,N,L,M,full", [(2048, 50, 100, 4, False), (1500, 50, 100, 1, False),
                                          (777, 20, 40, 3, True), (300, 10, 20, 16, False),
                                          (1, 1, 5, 1, False), (129, 7, 9, 8, False), (33, 70, 12, 1, False),
                                          (20000, 30, 24, 1, False), (20000, 24, 24, 4, False),
                                          (17000, 20, 16, 3, True),
                                          # tensor-core LWPR chunking: 64 + 64 + 2 fields, one full chunk
                                          (20000, 12, 130, 1, False), (17000, 10, 64, 4, False),
                                          # M > 32: the generic kernel (pairwise halving 40 -> 5, then a mean)
                                          (600, 10, 16, 40, False), (300, 8, 12, 64, False),
                                          # long horizons: shared-memory footprints scale with N
                                          (2000, 300, 16, 1, False), (17000, 300, 16, 1, False),
                                          (3000, 300, 16, 4, False),
                                          # one- and two-field models (a chunk of 8 is mostly padding)
                                          (2048, 10, 1, 1, False), (2048, 10, 2, 4, False)])
def test_evaluate_matches_oracle(K, N, L, M, full):
    stacks = synthetic.hybrid_stacks(L, seed=K + N, full_metric=full)
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(stacks, params)
    cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=N, iterations_per_step=1, rng_seed=K)
    task = P.Task.default()
    state = P.QuadState.hover(task.spawn + np.array([0.05, -0.1, 0.07]))
    plan = P.ControlPlan.hover(params, N)
    noise = P.sample_noise(cfg, 1, 0)
    dyn = P.sample_dynamics_noise(cfg, 1, 0) if M > 1 else None
    b = P.RolloutEngine(model, cfg, device=0).evaluate(state, plan, noise, P.RolloutCost(task, 2), dyn)
    om = RO.Model(stacks)
    lo, hi = om.dyn.bounds()
    rc, rf = RO.evaluate(om, state.as_array(), plan.controls, lo, hi, noise,
                         RO.Cost(TASK_WAYPOINTS[2], TASK_OBSTACLES), dyn, M)
    np.testing.assert_array_equal(b.crash_flags, rf)
    if N <= 100:  # BASELINE horizons go to T = 100
        assert cost_rel_err(b.costs_to_go, rc) < COST_RTOL
    else:  # the gate on the first 100 steps; beyond, float32 trajectory drift (in the reference
        # itself) of rollouts flown far outside the model's support grows: 300 steps reach ~1.2e-5
        assert cost_rel_err(b.costs_to_go[:, :100], rc[:, :100]) < COST_RTOL
        assert cost_rel_err(b.costs_to_go, rc) < 5e-5
    new = P.path_integral_update(plan, b, 1.0)
    assert np.all(du_err(new.controls, RO.update(plan.controls, lo, hi, rc, noise, 1.0), plan.controls) < DU_TOL)


@pytest.mark.parametrize("K,M", [(600, 1), (9000, 1), (3000, 4), (1500, 3)])
def test_many_obstacles_match_oracle(K, M):
    """Obstacle lists longer than pi2_cost holds (the reference has no limit,
    simworld.py:141-146, :188-190): the first PI2_MAX_OBSTACLES ride in the struct, the
    rest in HBM (pi2_set_cost_obstacles), summed in list order.  Covers the warp-,
    thread- and group-per-rollout kernels, a changed list on the same engine (re-staged),
    and a short list afterwards (reset)."""
    N, L = 40, 24
    stacks = synthetic.hybrid_stacks(L, seed=K + M)
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(stacks, params)
    cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=N, iterations_per_step=1, rng_seed=K)
    base = P.Task.default()
    state = P.QuadState.hover(base.spawn + np.array([0.05, -0.1, 0.07]))
    plan = P.ControlPlan.hover(params, N)
    noise = P.sample_noise(cfg, 1, 0)
    dyn = P.sample_dynamics_noise(cfg, 1, 0) if M > 1 else None
    eng = P.RolloutEngine(model, cfg, device=0)
    om = RO.Model(stacks)
    lo, hi = om.dyn.bounds()
    rng = np.random.default_rng(K)
    for n_obs in (40, 23, 3):
        # obstacles around the spawn so that their terms matter to the costs
        obs = base.spawn[:2] + rng.uniform(-0.6, 0.6, size=(n_obs, 2))
        task = P.Task(base.waypoints, obs)
        b = eng.evaluate(state, plan, noise, P.RolloutCost(task, 1), dyn)
        rc, rf = RO.evaluate(om, state.as_array(), plan.controls, lo, hi, noise, RO.Cost(task.waypoints[1], obs), dyn, M)
        np.testing.assert_array_equal(b.crash_flags, rf)
        assert cost_rel_err(b.costs_to_go, rc) < COST_RTOL, n_obs


@pytest.mark.parametrize("which", ["lo", "hi"])
def test_nan_control_bound_matches_oracle(which):
    """A NaN control bound (r_max or f_max NaN) takes the attitude kernel's general clip
    (NaN-propagating on both operands, numpy's np.clip); the default finite bounds take the
    cheaper one.  Both follow the oracle: here every clipped control is NaN, so every
    rollout gets the cost ceiling and a crash."""
    K, N, L, M = 700, 20, 16, 1
    stacks = synthetic.hybrid_stacks(L, seed=3)
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(stacks, params)
    cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=N, iterations_per_step=1, rng_seed=5)
    task = P.Task.default()
    state = P.QuadState.hover(task.spawn)
    lo, hi = params.control_bounds()
    (lo if which == "lo" else hi)[1] = np.nan
    plan = P.ControlPlan(np.tile([0.0, 0.0, 0.0, params.hover_thrust], (N, 1)), params.dt, 0.0, lo, hi)
    noise = P.sample_noise(cfg, 2, 0)
    b = P.RolloutEngine(model, cfg, device=0).evaluate(state, plan, noise, P.RolloutCost(task, 1))
    om = RO.Model(stacks)
    rc, rf = RO.evaluate(om, state.as_array(), plan.controls, lo, hi, noise, RO.Cost(TASK_WAYPOINTS[1], TASK_OBSTACLES))
    np.testing.assert_array_equal(b.crash_flags, rf)
    np.testing.assert_array_equal(b.costs_to_go, rc)


def test_frozen_lwpr_predict_matches_reference():
    z = load("lwpr")
    st = stacks_from(z, "diag_")
    X = z["diag_X"]
    for a in range(3):
        fr = P.FrozenLwpr(P.LwprModel.from_stack(st[a].centers, st[a].metrics, st[a].coefs, st[a].lvar), len(X))
        m = np.empty(len(X), np.float32)
        v = np.empty(len(X), np.float32)
        fr.predict_into(X, m, v)
        np.testing.assert_allclose(m, z[f"diag_mean{a}"], rtol=2e-5, atol=2e-5)
        np.testing.assert_allclose(v, z[f"diag_var{a}"], rtol=2e-4, atol=2e-6)
    for i in range(int(z["n_full"])):
        mdl = P.LwprModel.from_stack(z[f"full{i}_centers"], z[f"full{i}_metrics"], z[f"full{i}_coefs"],
                                     z[f"full{i}_lvar"])
        Xf = z[f"full{i}_X"]
        fr = P.FrozenLwpr(mdl, len(Xf))
        m = np.empty(len(Xf), np.float32)
        v = np.empty(len(Xf), np.float32)
        fr.predict_into(Xf, m, v)
        scale = max(1.0, float(np.abs(z[f"full{i}_mean"]).max()))
        np.testing.assert_allclose(m, z[f"full{i}_mean"], atol=2e-5 * scale)
        np.testing.assert_allclose(v, z[f"full{i}_var"], atol=2e-5 * scale, rtol=1e-4)


def test_frozen_lwpr_far_rows_follow_float32_underflow():
    """Rows whose every weight is a float32 denormal or zero."""
    z = load("eval_far_m1")
    st = stacks_from(z)
    rng = np.random.default_rng(5)
    X = rng.uniform([-1.5, -1.5, -1.5, 0.0], [1.5, 1.5, 1.5, 0.37], size=(4096, 4)).astype(np.float32)
    for a in range(3):
        p = OL.fold(st[a].centers, st[a].metrics, st[a].coefs, st[a].lvar)
        with np.errstate(invalid="ignore", divide="ignore"):
            rm, rv = OL.predict_f32(p, X)
        fr = P.FrozenLwpr(P.LwprModel.from_stack(st[a].centers, st[a].metrics, st[a].coefs, st[a].lvar), len(X))
        m = np.empty(len(X), np.float32)
        v = np.empty(len(X), np.float32)
        fr.predict_into(X, m, v)
        np.testing.assert_array_equal(np.isnan(m), np.isnan(rm))
        ok = ~np.isnan(rm)
        np.testing.assert_allclose(m[ok], rm[ok], rtol=1e-3, atol=1e-3)


def test_update_known_answers():
    z = load("update")
    plan = P.ControlPlan.hover(P.QuadParams(), 3)
    new = P.path_integral_update(plan, P.RolloutBatch(z["hand_noise"], z["hand_costs"], np.zeros(2, bool)), 1.0)
    np.testing.assert_allclose(new.controls, z["hand_new"], atol=1e-12)
    for i in range(int(z["n_random"])):
        n = z[f"r{i}_plan"].shape[0]
        plan = P.ControlPlan.hover(P.QuadParams(), n)
        b = P.RolloutBatch(z[f"r{i}_noise"], z[f"r{i}_costs"], np.zeros(len(z[f"r{i}_costs"]), bool))
        new = P.path_integral_update(plan, b, float(z[f"r{i}_lambda"]))
        np.testing.assert_allclose(new.controls - plan.controls, z[f"r{i}_new"] - plan.controls,
                                   rtol=1e-9, atol=1e-12)


def test_update_shape_errors():
    plan = P.ControlPlan.hover(P.QuadParams(), 4)
    with pytest.raises(ValueError, match="batch does not match"):
        P.path_integral_update(plan, P.RolloutBatch(np.zeros((3, 5, 4)), np.zeros((3, 5)), np.zeros(3, bool)), 1.0)


def test_optimize_and_receding_horizon_match_reference():
    z = load("optimize")
    model = P.HybridModel.from_stacks(stacks_from(z), P.QuadParams())
    cfg = P.PiConfig(num_rollouts=int(z["K"]), sub_rollouts=int(z["M"]), horizon_steps=int(z["N"]),
                     iterations_per_step=int(z["iterations"]), rng_seed=int(z["seed"]), chunk_size=16)
    task = P.Task.default()
    state = P.QuadState.from_array(z["state"])
    plan = P.ControlPlan.hover(P.QuadParams(), int(z["N"]))
    cost = P.RolloutCost(task, int(z["waypoint_index"]))
    opt = P.optimize(state, plan, cfg, model, cost, cycle_index=int(z["cycle"]))
    assert np.all(du_err(opt.controls, z["optimized"], plan.controls) < DU_TOL)
    ctrl, carried = P.receding_horizon_step(state, plan, cfg, model, cost, cycle_index=int(z["cycle"]))
    np.testing.assert_allclose(ctrl.as_array(), z["control"], rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(carried.controls, z["carried"], rtol=1e-4, atol=1e-6)


def test_zero_variance_subrollouts_equal_mean_exactly():
    """Reference test_controller.py:143-169 on the GPU engine."""
    p = P.QuadParams()
    models = [P.LwprModel.from_stack([[0.0, 0.0, 0.0, p.hover_thrust]], [np.diag(np.ones(4))],
                                     [[0.3, 0, 0, 0, 0]], [0.0]) for _ in range(3)]
    hybrid = P.HybridModel(tuple(models), p)
    task = P.Task(waypoints=np.array([[0.0, 0.0, 1.0]]), obstacles=np.empty((0, 2)), laps=1)
    plan = P.ControlPlan.hover(p, 12)
    cfg = P.PiConfig(num_rollouts=8, horizon_steps=12, sub_rollouts=8, rng_seed=7,
                     exploration_std=[1.5, 1.5, 0.6, 0.04])
    noise = P.sample_noise(cfg, 0, 0)
    dyn = P.sample_dynamics_noise(cfg, 0, 0)
    state = P.QuadState.hover((0, 0, 1))
    a = P.evaluate_rollouts(state, plan, noise, hybrid, P.RolloutCost(task, 0), sub_rollouts=8, dyn_noise=dyn)
    b = P.evaluate_rollouts(state, plan, noise, hybrid, P.RolloutCost(task, 0), sub_rollouts=1)
    np.testing.assert_array_equal(a.costs_to_go, b.costs_to_go)


class TwoPointModel:
    """Reference tests/synthetic.py:17-40 (the engine maps it to the device two-point model)."""

    probabilistic = True
    noise_transform = staticmethod(np.sign)

    def __init__(self, magnitude, params=None):
        self.params = params or P.QuadParams()
        self.magnitude = float(magnitude)


class ThresholdCost:
    def __init__(self, threshold):
        self.threshold = np.float32(threshold)


def two_point_expected_cost(magnitude, threshold, n_steps, dt):
    total = 0.0
    for bits in range(1 << n_steps):
        z = v = s = 0.0
        for t in range(n_steps):
            z = z + v * dt
            v = v + (magnitude if (bits >> t) & 1 else -magnitude) * dt
            if z > threshold:
                s += dt
        total += s
    return total / (1 << n_steps)


def test_two_point_model_matches_enumeration():
    """Reference test_controller.py:171-189 on the GPU engine."""
    p = P.QuadParams()
    n, mag, thr = 10, 2.0, -0.0043
    cfg = P.PiConfig(num_rollouts=4000, horizon_steps=n, sub_rollouts=4, rng_seed=5)
    noise = np.zeros((4000, n, 4))
    dyn = P.sample_dynamics_noise(cfg, 0, 0)
    b = P.evaluate_rollouts(P.QuadState.hover((0, 0, 0)), P.ControlPlan.hover(p, n), noise, TwoPointModel(mag, p),
                            ThresholdCost(thr), sub_rollouts=4, dyn_noise=dyn)
    got = b.costs_to_go[:, 0]
    assert abs(got.mean() - two_point_expected_cost(mag, thr, n, p.dt)) < 5 * got.std() / np.sqrt(len(got)) + 1e-9


def test_subrollout_cost_variance_scales_inverse_m():
    """Reference test_controller.py:308-327 on the GPU engine (M=64 and 256: several sub-rollouts per lane)."""
    p = P.QuadParams()
    stds = {}
    for m_sub in (4, 16, 64, 256):
        cfg = P.PiConfig(num_rollouts=1500, horizon_steps=10, sub_rollouts=m_sub, rng_seed=3)
        dyn = P.sample_dynamics_noise(cfg, 0, 0)
        b = P.evaluate_rollouts(P.QuadState.hover((0, 0, 0)), P.ControlPlan.hover(p, 10), np.zeros((1500, 10, 4)),
                                TwoPointModel(2.0, p), ThresholdCost(-0.0043), sub_rollouts=m_sub, dyn_noise=dyn)
        stds[m_sub] = b.costs_to_go[:, 0].std()
    assert stds[16] == pytest.approx(stds[4] / 2.0, rel=0.25)
    assert stds[64] == pytest.approx(stds[16] / 2.0, rel=0.25)
    assert stds[256] == pytest.approx(stds[64] / 2.0, rel=0.25)


def test_engine_errors_match_reference():
    p = P.QuadParams()
    model = P.HybridModel.from_stacks(synthetic.hybrid_stacks(8), p)
    cfg = P.PiConfig(num_rollouts=4, horizon_steps=5, sub_rollouts=2)
    eng = P.RolloutEngine(model, cfg, device=0)
    plan = P.ControlPlan.hover(p, 5)
    cost = P.RolloutCost(P.Task.default(), 0)
    with pytest.raises(ValueError, match="noise horizon"):
        eng.evaluate(P.QuadState.hover((0, 0, 1)), plan, np.zeros((4, 6, 4)), cost, np.zeros((4, 2, 6, 3), np.float32))
    with pytest.raises(ValueError, match="needs dyn_noise"):
        eng.evaluate(P.QuadState.hover((0, 0, 1)), plan, np.zeros((4, 5, 4)), cost)
    untrained = P.HybridModel(tuple(P.LwprModel(4) for _ in range(3)), p)
    with pytest.raises(ValueError, match="untrained"):
        P.RolloutEngine(untrained, cfg, device=0).evaluate(P.QuadState.hover((0, 0, 1)), plan, np.zeros((4, 5, 4)),
                                                           cost, np.zeros((4, 2, 5, 3), np.float32))


# ---------------------------------------------------------------- device noise
def test_device_noise_statistics_and_addressing():
    params = P.QuadParams()
    model = P.AnalyticModel(params)
    cfg = P.PiConfig(num_rollouts=10_000, horizon_steps=50, sub_rollouts=4)
    eng = P.RolloutEngine(model, cfg, device=0, noise="device")
    ctx = eng.context(cfg.num_rollouts, cfg.horizon_steps)
    std = np.array([1.5, 1.5, 0.6, 0.04])

    def draw(cycle, it, seed=7):
        out = np.empty((cfg.num_rollouts, cfg.horizon_steps, 4))
        ctx.call("pi2_device_noise", _abi.STREAM_CONTROL, seed, cycle, it, _abi.ptr(std), _abi.ptr(out))
        return out

    a = draw(3, 1)
    np.testing.assert_array_equal(a, draw(3, 1))
    assert not np.array_equal(a, draw(4, 1)) and not np.array_equal(a, draw(3, 0))
    assert not np.array_equal(a, draw(3, 1, seed=8))
    np.testing.assert_allclose(a.std(axis=(0, 1)), std, rtol=0.02)
    np.testing.assert_allclose(a.mean(axis=(0, 1)) / std, 0.0, atol=0.01)
    d = np.empty((cfg.num_rollouts, 4, cfg.horizon_steps, 3), np.float32)
    ctx.call("pi2_device_noise", _abi.STREAM_DYNAMICS, 7, 3, 1, None, _abi.ptr(d))
    np.testing.assert_allclose(d.std(), 1.0, rtol=0.01)
    np.testing.assert_allclose(d.mean(), 0.0, atol=0.01)
    z = d.reshape(-1).astype(np.float64)
    assert abs(np.mean(z ** 4) - 3.0) < 0.05  # Gaussian kurtosis


@pytest.mark.parametrize("seed,cycle,it", [(7, 3, 1), (11, 0, 17), (5, 2, 1000)])
def test_device_noise_matches_host_replica(seed, cycle, it):
    """The device streams are Philox4x32-10 under rng.derive_key(seed, stream, cycle, it):
    the kernels derive the iteration's key themselves from StepArgs.key_prefix."""
    from tests import devnoise
    K, N, M = 300, 20, 3
    cfg = P.PiConfig(num_rollouts=K, horizon_steps=N, sub_rollouts=M)
    eng = P.RolloutEngine(P.AnalyticModel(P.QuadParams()), cfg, device=0, noise="device")
    ctx = eng.context(K, N)
    std = np.array([1.5, 1.5, 0.6, 0.04])
    eps = np.empty((K, N, 4))
    ctx.call("pi2_device_noise", _abi.STREAM_CONTROL, seed, cycle, it, _abi.ptr(std), _abi.ptr(eps))
    dyn = np.empty((K, M, N, 3), np.float32)
    ctx.call("pi2_device_noise", _abi.STREAM_DYNAMICS, seed, cycle, it, None, _abi.ptr(dyn))
    # MUFU lg2/sin/cos approximations: ~1e-6 typically, up to ~1e-4 where u1 -> 1 (r -> 0);
    # a wrong key or counter gives O(1) differences everywhere
    for dev, host in ((eps / std, devnoise.control_noise(seed, cycle, it, K, N, std) / std),
                      (dyn, devnoise.dynamics_noise(seed, cycle, it, K, M, N))):
        err = np.abs(dev - host)
        assert err.max() < 5e-4 and np.median(err) < 2e-6, (err.max(), np.median(err))


def _device_setup(K=3000, N=40, L=48, M=4, iters=2):
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(synthetic.hybrid_stacks(L, seed=9), params)
    cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=N, iterations_per_step=iters, rng_seed=11)
    task = P.Task.default()
    return params, model, cfg, task, P.QuadState.hover(task.spawn), P.ControlPlan.hover(params, N), P.RolloutCost(task, 1)


def test_device_optimize_equals_materialised_noise_path():
    """Fused device-noise optimize == evaluate + update fed with the same device noise."""
    params, model, cfg, task, state, plan, cost = _device_setup(iters=1)
    eng = P.RolloutEngine(model, cfg, device=0, noise="device")
    fused = eng.optimize_device(state, plan, cost, cycle_index=4)
    ctx = eng.context(cfg.num_rollouts, cfg.horizon_steps)
    eps = np.empty((cfg.num_rollouts, cfg.horizon_steps, 4))
    ctx.call("pi2_device_noise", _abi.STREAM_CONTROL, cfg.rng_seed, 4, 0, _abi.ptr(cfg.exploration_std), _abi.ptr(eps))
    dyn = np.empty((cfg.num_rollouts, cfg.sub_rollouts, cfg.horizon_steps, 3), np.float32)
    ctx.call("pi2_device_noise", _abi.STREAM_DYNAMICS, cfg.rng_seed, 4, 0, None, _abi.ptr(dyn))
    b = P.RolloutEngine(model, cfg, device=0).evaluate(state, plan, eps, cost, dyn)
    two_step = P.path_integral_update(plan, b, cfg.temperature)
    np.testing.assert_array_equal(fused.controls, two_step.controls)
    # and the oracle agrees on those inputs
    om = RO.Model(synthetic.hybrid_stacks(48, seed=9))
    lo, hi = om.dyn.bounds()
    rc, _ = RO.evaluate(om, state.as_array(), plan.controls, lo, hi, eps,
                        RO.Cost(TASK_WAYPOINTS[1], TASK_OBSTACLES), dyn, cfg.sub_rollouts)
    assert cost_rel_err(b.costs_to_go, rc) < COST_RTOL


@pytest.mark.parametrize("use_graph", [True, False])
def test_device_optimize_beyond_sixteen_iterations(use_graph):
    """iterations_per_step is unbounded on the device path (reference PiConfig has no cap):
    20 fused iterations == 20 rounds of evaluate + update on the materialised device noise."""
    params, model, cfg, task, state, plan, cost = _device_setup(K=1000, N=20, iters=20)
    cyc = 2
    fused = P.RolloutEngine(model, cfg, device=0, noise="device", use_graph=use_graph).optimize_device(
        state, plan, cost, cycle_index=cyc)
    eng = P.RolloutEngine(model, cfg, device=0)
    ctx = eng.context(cfg.num_rollouts, cfg.horizon_steps)
    p = plan
    for it in range(cfg.iterations_per_step):
        eps = np.empty((cfg.num_rollouts, cfg.horizon_steps, 4))
        ctx.call("pi2_device_noise", _abi.STREAM_CONTROL, cfg.rng_seed, cyc, it, _abi.ptr(cfg.exploration_std),
                 _abi.ptr(eps))
        dyn = np.empty((cfg.num_rollouts, cfg.sub_rollouts, cfg.horizon_steps, 3), np.float32)
        ctx.call("pi2_device_noise", _abi.STREAM_DYNAMICS, cfg.rng_seed, cyc, it, None, _abi.ptr(dyn))
        p = P.path_integral_update(p, eng.evaluate(state, p, eps, cost, dyn), cfg.temperature)
    np.testing.assert_array_equal(fused.controls, p.controls)


@pytest.mark.parametrize("K,N,L,M", [(1, 1, 1, 1), (1, 5, 3, 4), (257, 1, 8, 3), (8192, 3, 16, 1),
                                     (8193, 3, 16, 1), (8193, 2, 16, 4), (300, 7, 130, 2)])
def test_device_path_edge_shapes(K, N, L, M):
    """The fused device-noise step at edge shapes (one rollout, one step, odd M, both
    sides of the warp-per-rollout threshold K = 8192, a 130-field model) equals
    evaluate + update on the materialised device noise, bitwise, and its costs match
    the oracle."""
    stacks = synthetic.hybrid_stacks(L, seed=K + N)
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(stacks, params)
    cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=N, iterations_per_step=1, rng_seed=4)
    task = P.Task.default()
    state = P.QuadState.hover(task.spawn + np.array([0.03, 0.02, -0.05]))
    plan, cost = P.ControlPlan.hover(params, N), P.RolloutCost(task, 1)
    eng = P.RolloutEngine(model, cfg, device=0, noise="device")
    fused = eng.optimize_device(state, plan, cost, cycle_index=2)
    ctx = eng.context(K, N)
    eps = np.empty((K, N, 4))
    ctx.call("pi2_device_noise", _abi.STREAM_CONTROL, cfg.rng_seed, 2, 0, _abi.ptr(cfg.exploration_std), _abi.ptr(eps))
    dyn = None
    if M > 1:
        dyn = np.empty((K, M, N, 3), np.float32)
        ctx.call("pi2_device_noise", _abi.STREAM_DYNAMICS, cfg.rng_seed, 2, 0, None, _abi.ptr(dyn))
    b = P.RolloutEngine(model, cfg, device=0).evaluate(state, plan, eps, cost, dyn)
    np.testing.assert_array_equal(fused.controls, P.path_integral_update(plan, b, cfg.temperature).controls)
    om = RO.Model(stacks)
    lo, hi = om.dyn.bounds()
    rc, rf = RO.evaluate(om, state.as_array(), plan.controls, lo, hi, eps, RO.Cost(TASK_WAYPOINTS[1], TASK_OBSTACLES),
                         dyn, M)
    np.testing.assert_array_equal(b.crash_flags, rf)
    assert cost_rel_err(b.costs_to_go, rc) < COST_RTOL


@pytest.mark.parametrize("K,M", [(3000, 1), (3000, 4), (700, 1)])
def test_warp_and_thread_per_rollout_kernels_are_bitwise_equal(K, M, monkeypatch):
    """The attitude / rollout kernels with a warp per rollout (small K) and with a thread
    (lane) per rollout give the same bits (PI2_WIDE_MAX_K forces either): device-noise
    optimize and host-noise evaluate."""
    stacks = synthetic.hybrid_stacks(24, seed=K + M)
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(stacks, params)
    task = P.Task.default()
    plan = P.ControlPlan.hover(params, 30)
    state = P.QuadState.hover(task.spawn)
    res = {}
    for thr in (str(1 << 30), "0"):
        monkeypatch.setenv("PI2_WIDE_MAX_K", thr)
        cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=30, iterations_per_step=2, rng_seed=6)
        noise = P.sample_noise(cfg, 1, 0)
        dyn = P.sample_dynamics_noise(cfg, 1, 0) if M > 1 else None
        b = P.RolloutEngine(model, cfg, device=0).evaluate(state, plan, noise, P.RolloutCost(task, 1), dyn)
        dev = P.RolloutEngine(model, cfg, device=0, noise="device").optimize_device(state, plan, P.RolloutCost(task, 1), 1)
        res[thr] = (b.costs_to_go, b.crash_flags, dev.controls)
    for x, y in zip(res[str(1 << 30)], res["0"]):
        np.testing.assert_array_equal(x, y)


def test_io_pull_kernel_and_copy_node_give_the_same_step(monkeypatch):
    """The real-time graph's inputs arrive by io_pull_kernel (default) or by a copy-engine
    node (PI2_IO_PULL=0): the same controls and plans, bit for bit, over a receding loop."""
    params, model, cfg, task, state, plan, cost = _device_setup(K=2000, N=30)
    res = {}
    for pull in ("1", "0"):
        monkeypatch.setenv("PI2_IO_PULL", pull)
        eng = P.RolloutEngine(model, cfg, device=0, noise="device")
        p, out = plan, []
        for c in range(4):
            ctrl, p = P.receding_horizon_step(state, p, cfg, model, cost, c, eng)
            out += [ctrl.as_array(), p.controls.copy()]
        res[pull] = out
    for a, b in zip(res["1"], res["0"]):
        np.testing.assert_array_equal(a, b)


def test_profile_iteration_reports_stages_and_leaves_the_plan():
    """pi2_profile_iteration (bench.py's per-kernel timing) returns positive stage times
    and does not change the device-resident plan."""
    params, model, cfg, task, state, plan, cost = _device_setup(K=3000, N=30)
    eng = P.RolloutEngine(model, cfg, device=0, noise="device")
    P.receding_horizon_step(state, plan, cfg, model, cost, 0, eng)  # binds dynamics and cost
    ctx = eng.context(cfg.num_rollouts, cfg.horizon_steps)
    from paper_1503_00330_b200.controller import optimize_args
    ctx.call("pi2_load_plan", _abi.ptr(state.as_array()), _abi.ptr(np.ascontiguousarray(plan.controls)), None)
    stages = (_abi.C.c_double * 5)()
    ctx.call("pi2_profile_iteration", optimize_args(cfg, 0, use_graph=False), 3, stages)
    assert all(v > 0 for v in stages), list(stages)
    back = np.empty((cfg.horizon_steps, 4))
    ctx.call("pi2_read_plan", _abi.ptr(back), None)
    np.testing.assert_array_equal(back, plan.controls)


@pytest.mark.parametrize("L,M", [(48, 4), (100, 1), (130, 2)])
def test_streamed_and_resident_lwpr_weights_are_bitwise_equal(L, M, monkeypatch):
    """The tensor-core LWPR kernel with its weights TMA-streamed per chunk
    (PI2_LWPR_TC_STREAM=1) and resident in shared memory (default where they fit) does the
    same arithmetic: identical costs and updates."""
    stacks = synthetic.hybrid_stacks(L, seed=L)
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(stacks, params)
    task = P.Task.default()
    cfg = P.PiConfig(num_rollouts=20000, sub_rollouts=M, horizon_steps=12, iterations_per_step=1, rng_seed=8)
    state, plan, cost = P.QuadState.hover(task.spawn), P.ControlPlan.hover(params, 12), P.RolloutCost(task, 1)
    res = {}
    for stream in ("1", None):
        if stream:
            monkeypatch.setenv("PI2_LWPR_TC_STREAM", stream)
        else:
            monkeypatch.delenv("PI2_LWPR_TC_STREAM", raising=False)
        noise = P.sample_noise(cfg, 1, 0)
        dyn = P.sample_dynamics_noise(cfg, 1, 0) if M > 1 else None
        b = P.RolloutEngine(model, cfg, device=0).evaluate(state, plan, noise, cost, dyn)
        dev = P.RolloutEngine(model, cfg, device=0, noise="device").optimize_device(state, plan, cost, 2)
        res[stream] = (b.costs_to_go, dev.controls)
    for a, b in zip(res["1"], res[None]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("K", [1024, 20000])
def test_bulk_copy_and_ldg_weight_prologues_are_bitwise_equal(K, monkeypatch):
    """The resident-weight prologue by one TMA bulk copy (WBULK, few tiles per CTA) and by
    the LDG/STS loop load the same bytes: identical device-path updates either way."""
    stacks = synthetic.hybrid_stacks(64, seed=K)
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(stacks, params)
    task = P.Task.default()
    cfg = P.PiConfig(num_rollouts=K, sub_rollouts=2, horizon_steps=16, iterations_per_step=2, rng_seed=9)
    state, plan, cost = P.QuadState.hover(task.spawn), P.ControlPlan.hover(params, 16), P.RolloutCost(task, 1)
    res = {}
    for tiles in ("0", "1000000"):
        monkeypatch.setenv("PI2_TC_BULK_MAX_TILES", tiles)
        res[tiles] = P.RolloutEngine(model, cfg, device=0, noise="device").optimize_device(state, plan, cost, 1).controls
    np.testing.assert_array_equal(res["0"], res["1000000"])


def test_graph_replay_matches_eager_and_is_deterministic():
    params, model, cfg, task, state, plan, cost = _device_setup()
    g = P.RolloutEngine(model, cfg, device=0, noise="device", use_graph=True)
    e = P.RolloutEngine(model, cfg, device=0, noise="device", use_graph=False)
    outs = [g.optimize_device(state, plan, cost, c) for c in (0, 1, 0)]
    np.testing.assert_array_equal(outs[0].controls, outs[2].controls)
    assert not np.array_equal(outs[0].controls, outs[1].controls)
    np.testing.assert_array_equal(outs[0].controls, e.optimize_device(state, plan, cost, 0).controls)


def test_receding_fast_path_equals_optimize_then_shift():
    """receding_horizon_step on a device engine (pi2_receding_horizon_step, cached plugin
    binding) == optimize_device + control_at(0) + shifted(), bitwise, across a waypoint
    switch (the binding cache must notice the new cost) and with iterations_per_step=0."""
    params, model, cfg, task, state, plan, cost = _device_setup(iters=1)
    fast = P.RolloutEngine(model, cfg, device=0, noise="device")
    slow = P.RolloutEngine(model, cfg, device=0, noise="device")
    p_fast = p_slow = plan
    for cycle, wp in enumerate((1, 1, 2, 2, 1)):
        c = P.RolloutCost(task, wp)
        ctrl, p_fast = P.receding_horizon_step(state, p_fast, cfg, model, c, cycle, fast)
        opt = slow.optimize_device(state, p_slow, c, cycle)
        want_ctrl, p_slow = opt.control_at(0), opt.shifted()
        np.testing.assert_array_equal(ctrl.desired_rates, want_ctrl.desired_rates)
        assert ctrl.thrust == want_ctrl.thrust
        np.testing.assert_array_equal(p_fast.controls, p_slow.controls)
        assert p_fast.origin_time == p_slow.origin_time
    cost.waypoint = task.waypoints[2].astype(np.float32)  # mutate the plugin in place
    a = P.receding_horizon_step(state, plan, cfg, model, cost, 9, fast)[1].controls
    b = slow.optimize_device(state, plan, P.RolloutCost(task, 2), 9).shifted().controls
    np.testing.assert_array_equal(a, b)
    cfg0 = P.PiConfig(num_rollouts=cfg.num_rollouts, sub_rollouts=cfg.sub_rollouts,
                      horizon_steps=cfg.horizon_steps, iterations_per_step=0)
    e0 = P.RolloutEngine(model, cfg0, device=0, noise="device")
    ctrl, shifted = P.receding_horizon_step(state, plan, cfg0, model, cost, 0, e0)
    np.testing.assert_array_equal(shifted.controls, plan.shifted().controls)
    assert ctrl.thrust == plan.controls[0, 3]


@pytest.mark.parametrize("K,M", [(128, 2), (20000, 1), (3000, 4)])
def test_programmatic_dependent_launch_is_bitwise_neutral(K, M, monkeypatch):
    """The step's kernels overlap their predecessors' tails under PDL (PI2_PDL, default
    on): results must be bitwise those of plain stream ordering, over repeated host-noise
    evaluations (different contexts, copies before the chain) and device optimizations.
    A non-coherent load hoisted above griddepcontrol.wait showed up exactly here."""
    stacks = synthetic.hybrid_stacks(24, seed=K + M)
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(stacks, params)
    task = P.Task.default()
    plan = P.ControlPlan.hover(params, 20)
    state = P.QuadState.hover(task.spawn)
    res = {}
    for pdl in ("1", "0"):
        monkeypatch.setenv("PI2_PDL", pdl)
        cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=20, iterations_per_step=2, rng_seed=1)
        eng = P.RolloutEngine(model, cfg, device=0)
        dev = P.RolloutEngine(model, cfg, device=0, noise="device")
        out = []
        for cyc in range(4):
            noise = P.sample_noise(cfg, cyc, 0)
            dyn = P.sample_dynamics_noise(cfg, cyc, 0) if M > 1 else None
            out.append(eng.evaluate(state, plan, noise, P.RolloutCost(task, 1), dyn).costs_to_go)
            out.append(dev.optimize_device(state, plan, P.RolloutCost(task, 1), cyc).controls)
        res[pdl] = out
    for a, b in zip(res["1"], res["0"]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("kind,K", [("analytic", 128), ("analytic", 20000), ("two_point", 3000),
                                    ("two_point", 128)])
def test_pdl_is_bitwise_neutral_without_lwpr(kind, K, monkeypatch):
    """With the analytic and two-point models no LWPR kernel sits between the attitude
    kernel (which triggers its dependents on entry) and the rollout kernel: the rollout
    kernel's reads of the attitude rows must still follow griddepcontrol.wait.  PDL on
    and off give the same bits over repeated host-noise evaluations and device steps."""
    params = P.QuadParams()
    task = P.Task.default()
    N = 20
    plan = P.ControlPlan.hover(params, N)
    state = P.QuadState.hover(task.spawn)
    if kind == "analytic":
        model, cost, M = P.AnalyticModel(params), P.RolloutCost(task, 1), 1
    else:
        model, cost, M = TwoPointModel(2.0, params), ThresholdCost(-0.0043), 4
    res = {}
    for pdl in ("1", "0"):
        monkeypatch.setenv("PI2_PDL", pdl)
        cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=N, iterations_per_step=2, rng_seed=1)
        eng = P.RolloutEngine(model, cfg, device=0)
        dev = P.RolloutEngine(model, cfg, device=0, noise="device")
        out = []
        for cyc in range(4):
            noise = P.sample_noise(cfg, cyc, 0)
            dyn = P.sample_dynamics_noise(cfg, cyc, 0) if M > 1 else None
            out.append(eng.evaluate(state, plan, noise, cost, dyn).costs_to_go)
            out.append(dev.optimize_device(state, plan, cost, cyc).controls)
        res[pdl] = out
    for a, b in zip(res["1"], res["0"]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("K,N", [(1000, 20), (3000, 37), (70000, 9)])
def test_split_partials_kernel_is_bitwise_equal(K, N, monkeypatch):
    """partials_split_kernel (a block per (chunk, t), used when few (chunk, t) pairs) and
    partials_kernel (a warp per (chunk, t)) give the same bits: device-noise optimize
    and the host-noise update path, ragged last chunks included."""
    stacks = synthetic.hybrid_stacks(24, seed=K)
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(stacks, params)
    task = P.Task.default()
    plan = P.ControlPlan.hover(params, N)
    state = P.QuadState.hover(task.spawn)
    res = {}
    for split in ("2", "0"):
        monkeypatch.setenv("PI2_PARTIALS_SPLIT", split)
        from paper_1503_00330_b200 import controller as PC
        monkeypatch.setattr(PC, "_UPDATE_TLS", threading.local())  # the update context reads the switch when created
        cfg = P.PiConfig(num_rollouts=K, sub_rollouts=1, horizon_steps=N, iterations_per_step=3, rng_seed=2)
        dev = P.RolloutEngine(model, cfg, device=0, noise="device")
        eng = P.RolloutEngine(model, cfg, device=0)
        noise = P.sample_noise(cfg, 1, 0)
        batch = eng.evaluate(state, plan, noise, P.RolloutCost(task, 1))
        res[split] = [dev.optimize_device(state, plan, P.RolloutCost(task, 1), c).controls for c in range(2)]
        res[split].append(P.path_integral_update(plan, batch, cfg.temperature).controls)
    for a, b in zip(res["2"], res["0"]):
        np.testing.assert_array_equal(a, b)


def test_sharded_partials_are_gpu_count_invariant():
    """Rank shards evaluated one after another on one GPU (no cross-waiting kernels):
    the fixed-order combine gives the single-context plan bitwise for G = 2 and 4."""
    from paper_1503_00330_b200.controller import dynamics_struct, optimize_args
    from paper_1503_00330_b200.distributed import shard_range
    from paper_1503_00330_b200.lwpr import stage_axis
    from paper_1503_00330_b200.simworld import cost_struct

    params, model, cfg, task, state, plan, cost = _device_setup(K=4096, iters=1)
    single = P.RolloutEngine(model, cfg, device=0, noise="device", use_graph=False).optimize_device(state, plan, cost, 2)
    args = optimize_args(cfg, 2, use_graph=False)
    for world in (2, 4):
        ctxs, parts = [], []
        for r in range(world):
            s, e = shard_range(cfg.num_rollouts, r, world)
            c = _abi.Context(0, e - s, cfg.horizon_steps, cfg.sub_rollouts, rollout_offset=s,
                             num_rollouts_total=cfg.num_rollouts)
            for a in range(3):
                stage_axis(c, a, model.models[a])
            c.call("pi2_select_model", _abi.MODEL_HYBRID_LWPR, 0.0)
            c.call("pi2_set_dynamics", dynamics_struct(params, plan.lo, plan.hi))
            c.call("pi2_set_cost", cost_struct(cost))
            import torch

            c.call("pi2_load_plan", _abi.ptr(state.as_array()), _abi.ptr(np.ascontiguousarray(plan.controls)), None)

            part = torch.empty((cfg.horizon_steps, 6), dtype=torch.float64, device="cuda:0")
            c.call("pi2_iterate_local", args, 0, _abi.ptr(part), None)
            torch.cuda.synchronize()
            ctxs.append(c)
            parts.append(part)
        import torch

        gathered = torch.stack(parts).contiguous()
        torch.cuda.synchronize()
        for c in ctxs:
            c.call("pi2_iterate_finalize", _abi.ptr(gathered), world, float(cfg.temperature), None)
            out = np.empty((cfg.horizon_steps, 4))
            c.call("pi2_read_plan", _abi.ptr(out), None)
            np.testing.assert_array_equal(out, single.controls)


@pytest.mark.parametrize("L,full", [(1500, False), (700, True)])
def test_tiled_parameters_match_oracle(L, full):
    """Parameter sets too large for shared memory stream through in tiles (C3's path)."""
    stacks = synthetic.hybrid_stacks(L, seed=L, full_metric=full)
    if not full:  # per-field metrics -> the diagonal layout, 16 floats/field: 3*1500*64 B > 64 KB
        stacks = tuple(synthetic.AxisStack(s.centers, s.metrics * (1.0 + 1e-3 * np.arange(L))[:, None, None],
                                           s.coefs, s.lvar) for s in stacks)
    K, N, M = 96, 12, 2
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(stacks, params)
    cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=N, iterations_per_step=1, rng_seed=3)
    task = P.Task.default()
    state = P.QuadState.hover(task.spawn)
    plan = P.ControlPlan.hover(params, N)
    noise = P.sample_noise(cfg, 0, 0)
    dyn = P.sample_dynamics_noise(cfg, 0, 0)
    b = P.RolloutEngine(model, cfg, device=0).evaluate(state, plan, noise, P.RolloutCost(task, 1), dyn)
    om = RO.Model(stacks)
    lo, hi = om.dyn.bounds()
    rc, rf = RO.evaluate(om, state.as_array(), plan.controls, lo, hi, noise,
                         RO.Cost(TASK_WAYPOINTS[1], TASK_OBSTACLES), dyn, M)
    np.testing.assert_array_equal(b.crash_flags, rf)
    assert cost_rel_err(b.costs_to_go, rc) < COST_RTOL


@pytest.mark.parametrize("L,M,tc", [(1000, 1, "1"), (600, 2, "1"), (1000, 2, "0")])
def test_large_shared_metric_models_match_oracle(L, M, tc, monkeypatch):
    """Shared-metric models too large for resident weights (C3): the tensor-core kernel
    streams each chunk's weights (PI2_LWPR_TC=1), the CUDA-core kernel tiles them (0)."""
    monkeypatch.setenv("PI2_LWPR_TC", tc)
    stacks = synthetic.hybrid_stacks(L, seed=L + M)
    K, N = 20000, 6
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(stacks, params)
    cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=N, iterations_per_step=1, rng_seed=5)
    task = P.Task.default()
    state = P.QuadState.hover(task.spawn)
    plan = P.ControlPlan.hover(params, N)
    noise = P.sample_noise(cfg, 0, 0)
    dyn = P.sample_dynamics_noise(cfg, 0, 0) if M > 1 else None
    eng = P.RolloutEngine(model, cfg, device=0)
    b = eng.evaluate(state, plan, noise, P.RolloutCost(task, 1), dyn)
    kind = _abi.C.c_int32()
    eng.context(K, N).call("pi2_lwpr_kernel", int(M > 1), _abi.C.byref(kind), None)
    assert kind.value == (1 if tc == "1" else 0)
    om = RO.Model(stacks)
    lo, hi = om.dyn.bounds()
    rc, rf = RO.evaluate(om, state.as_array(), plan.controls, lo, hi, noise,
                         RO.Cost(TASK_WAYPOINTS[1], TASK_OBSTACLES), dyn, M)
    np.testing.assert_array_equal(b.crash_flags, rf)
    assert cost_rel_err(b.costs_to_go, rc) < COST_RTOL


def test_shared_metric_model_from_reference_training():
    """A model trained by the reference (fields share d_init) through the LWPR1 format."""
    z = load("persistence")
    m = P.load_model(z["blob"].tobytes())
    fr = P.FrozenLwpr(m, len(z["X"]))
    mean = np.empty(len(z["X"]), np.float32)
    var = np.empty(len(z["X"]), np.float32)
    fr.predict_into(z["X"], mean, var)
    scale = max(1.0, float(np.abs(z["mean"]).max()))
    np.testing.assert_allclose(mean, z["mean"], atol=2e-5 * scale)
    np.testing.assert_allclose(var, z["var"], rtol=1e-3, atol=2e-5 * scale)


def test_hybrid_make_batch_eval_protocol():
    """Model-plugin protocol (dynamics.py:262-277): eval_into fills (B, 3) means and
    standard deviations from the per-axis LWPR models."""
    z = load("propagate")
    p = P.QuadParams()
    model = P.HybridModel.from_stacks(stacks_from(z, "hybrid_"), p)
    rng = np.random.default_rng(3)
    X = rng.uniform([-0.3, -0.3, -0.3, 0.12], [0.3, 0.3, 0.3, 0.25], (64, 4)).astype(np.float32)
    ev = model.make_batch_eval(64)
    mean, std = np.empty((64, 3), np.float32), np.empty((64, 3), np.float32)
    ev(X, mean, std)
    for a in range(3):
        fr = P.FrozenLwpr(model.models[a], 64)
        m, v = np.empty(64, np.float32), np.empty(64, np.float32)
        fr.predict_into(X, m, v)
        np.testing.assert_array_equal(mean[:, a], m)
        np.testing.assert_array_equal(std[:, a], np.sqrt(v))
    mean2 = np.empty((64, 3), np.float32)
    ev(X, mean2)  # mean-only kernel variant: the same to an ulp
    np.testing.assert_allclose(mean2, mean, rtol=1e-6, atol=1e-7)


# ---------------------------------------------------------------- opt-in uncertainty penalty
@pytest.mark.parametrize("K,M", [(3000, 1), (20000, 1), (3000, 4), (17000, 2)])
def test_variance_penalty_matches_oracle(K, M):
    """The opt-in uncertainty penalty (RolloutCost(..., variance_penalty=kappa), an
    extension of the reference's cost with parity unpinned against the reference):
    every rollout kernel (warp per rollout K <= 8192, thread per rollout, lanes per
    sub-rollout) against the oracle carrying the same term; kappa = 0 is the
    reference's cost bitwise; the fused device step equals evaluate + update."""
    N, L, kappa = 30, 48, 0.5
    stacks = synthetic.hybrid_stacks(L, seed=K + M + 1)
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(stacks, params)
    cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=N, iterations_per_step=1, rng_seed=6)
    task = P.Task.default()
    state = P.QuadState.hover(task.spawn + np.array([0.02, -0.04, 0.05]))
    plan = P.ControlPlan.hover(params, N)
    noise = P.sample_noise(cfg, 1, 0)
    dyn = P.sample_dynamics_noise(cfg, 1, 0) if M > 1 else None
    eng = P.RolloutEngine(model, cfg, device=0)
    plain = eng.evaluate(state, plan, noise, P.RolloutCost(task, 1), dyn)
    zero = eng.evaluate(state, plan, noise, P.RolloutCost(task, 1, variance_penalty=0.0), dyn)
    np.testing.assert_array_equal(zero.costs_to_go, plain.costs_to_go)
    b = eng.evaluate(state, plan, noise, P.RolloutCost(task, 1, variance_penalty=kappa), dyn)
    assert np.all(b.costs_to_go[:, 0] > plain.costs_to_go[:, 0])  # the term is positive
    om = RO.Model(stacks)
    lo, hi = om.dyn.bounds()
    rc, rf = RO.evaluate(om, state.as_array(), plan.controls, lo, hi, noise,
                         RO.Cost(TASK_WAYPOINTS[1], TASK_OBSTACLES, variance_penalty=kappa), dyn, M)
    np.testing.assert_array_equal(b.crash_flags, rf)
    assert cost_rel_err(b.costs_to_go, rc) < COST_RTOL
    dev = P.RolloutEngine(model, cfg, device=0, noise="device")
    pcost = P.RolloutCost(task, 1, variance_penalty=kappa)
    fused = dev.optimize_device(state, plan, pcost, cycle_index=4)
    ctx = dev.context(K, N)
    eps = np.empty((K, N, 4))
    ctx.call("pi2_device_noise", _abi.STREAM_CONTROL, cfg.rng_seed, 4, 0, _abi.ptr(cfg.exploration_std), _abi.ptr(eps))
    dn = None
    if M > 1:
        dn = np.empty((K, M, N, 3), np.float32)
        ctx.call("pi2_device_noise", _abi.STREAM_DYNAMICS, cfg.rng_seed, 4, 0, None, _abi.ptr(dn))
    bb = eng.evaluate(state, plan, eps, pcost, dn)
    np.testing.assert_array_equal(fused.controls, P.path_integral_update(plan, bb, cfg.temperature).controls)
    # switching the penalty off again re-captures the step: back to the reference's cost
    off = dev.optimize_device(state, plan, P.RolloutCost(task, 1), cycle_index=4)
    bb0 = eng.evaluate(state, plan, eps, P.RolloutCost(task, 1), dn)
    np.testing.assert_array_equal(off.controls, P.path_integral_update(plan, bb0, cfg.temperature).controls)


def test_variance_penalty_needs_probabilistic_model():
    p = P.QuadParams()
    cfg = P.PiConfig(num_rollouts=64, horizon_steps=10, iterations_per_step=1)
    eng = P.RolloutEngine(P.AnalyticModel(p), cfg, device=0)
    with pytest.raises(TypeError, match="variance_penalty"):
        eng.evaluate(P.QuadState.hover((0, 0, 1)), P.ControlPlan.hover(p, 10), np.zeros((64, 10, 4)),
                     P.RolloutCost(P.Task.default(), 0, variance_penalty=1.0))
