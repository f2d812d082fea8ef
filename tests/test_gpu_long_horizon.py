"""Horizons past 400 steps (the reference has no cap; this engine takes up to 524 280).

Above PI2_SMEM_HORIZON (400) the rollout kernels keep each rollout's stage costs in
a global (N, K) scratch instead of their blocks' shared memory, and the
warp-per-rollout latency kernels are not used.  The global path is bitwise equal
to the shared-memory path (forced here by lowering PI2_SMEM_HORIZON), and long
horizons match the oracle.
"""

import os

import numpy as np
import pytest

import paper_1503_00330_b200 as P
from paper_1503_00330_b200 import synthetic
from oracle import rollout as RO
from tests._cases import TASK_OBSTACLES, TASK_WAYPOINTS

pytestmark = pytest.mark.gpu


def evaluate(K, N, L, M, smem_horizon=None, noise_seed=1):
    old = os.environ.get("PI2_SMEM_HORIZON")
    if smem_horizon is not None:
        os.environ["PI2_SMEM_HORIZON"] = str(smem_horizon)
    try:
        stacks = synthetic.hybrid_stacks(L, seed=K + N)
        params = P.QuadParams()
        model = P.HybridModel.from_stacks(stacks, params)
        cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=N, iterations_per_step=1, rng_seed=K)
        task = P.Task.default()
        state = P.QuadState.hover(task.spawn + np.array([0.05, -0.1, 0.07]))
        plan = P.ControlPlan.hover(params, N)
        noise = P.sample_noise(cfg, noise_seed, 0)
        dyn = P.sample_dynamics_noise(cfg, noise_seed, 0) if M > 1 else None
        b = P.RolloutEngine(model, cfg, device=0).evaluate(state, plan, noise, P.RolloutCost(task, 2), dyn)
        return b, (stacks, state, plan, noise, dyn)
    finally:
        if old is None:
            os.environ.pop("PI2_SMEM_HORIZON", None)
        else:
            os.environ["PI2_SMEM_HORIZON"] = old


@pytest.mark.parametrize("K,N,M", [(3000, 120, 1),    # warp-per-rollout kernels vs thread per rollout + scratch
                                   (20000, 90, 1),    # thread per rollout: shared memory vs scratch
                                   (3000, 60, 4),     # lane per sub-rollout: shared memory vs scratch
                                   (777, 33, 3)])     # odd M (lane 0 replays the mean), ragged K
def test_global_stage_cost_scratch_is_bitwise_equal(K, N, M):
    ref, _ = evaluate(K, N, 48, M)
    got, _ = evaluate(K, N, 48, M, smem_horizon=N // 2)
    np.testing.assert_array_equal(got.costs_to_go.view(np.uint64), ref.costs_to_go.view(np.uint64))
    np.testing.assert_array_equal(got.crash_flags, ref.crash_flags)


@pytest.mark.parametrize("K,N,M", [(1200, 600, 1), (600, 450, 4),
                                   (96, 5000, 1), (64, 4500, 3)])  # past 4096: plan rows read from global memory
def test_long_horizon_matches_oracle(K, N, M):
    b, (stacks, state, plan, noise, dyn) = evaluate(K, N, 60, M)
    om = RO.Model(stacks)
    lo, hi = om.dyn.bounds()
    rc, rf = RO.evaluate(om, state.as_array(), plan.controls, lo, hi, noise,
                         RO.Cost(TASK_WAYPOINTS[2], TASK_OBSTACLES), dyn, M)
    np.testing.assert_array_equal(b.crash_flags, rf)
    rel = np.abs(b.costs_to_go - rc) / np.abs(rc)
    # the BASELINE gate on the first 100 steps; further out, float32 trajectory drift of
    # rollouts flown far outside the model's support grows (in the reference itself)
    assert rel[:, :100].max() < 1e-5
    print(f"\nN={N} M={M}: max cost rel err {rel[:, :100].max():.2e} (t < 100), {rel.max():.2e} (all)")
    assert rel.max() < 1e-4


def test_long_horizon_device_step():
    """The real-time path (device noise, one CUDA graph) at N = 1000: the update equals our
    own evaluate + update of the materialised device noise, bitwise."""
    from tests.test_gpu_baseline_configs import CYCLE, device_costs, device_noise, setup

    K, N, L, M = 10000, 1000, 60, 2
    stacks, model, cfg, state, plan, cost = setup(K, N, L, M)
    eng = P.RolloutEngine(model, cfg, device=0, noise="device")
    new = eng.optimize_device(state, plan, cost, cycle_index=CYCLE)
    ctx = eng.context(K, N)
    costs, crash = device_costs(ctx, cfg, state, plan, K, N)
    eps, _ = device_noise(ctx, cfg, K, N, M)
    ours = P.path_integral_update(plan, P.RolloutBatch(eps, costs.cpu().numpy(), crash.cpu().numpy().astype(bool)),
                                  cfg.temperature)
    np.testing.assert_array_equal(new.controls, ours.controls)
    assert np.all(np.isfinite(new.controls))


def test_horizon_limit():
    """Past 4096 steps is fine (test_long_horizon_matches_oracle); the bound is 8 x 65535."""
    from paper_1503_00330_b200 import _abi

    with pytest.raises(ValueError, match="horizon_steps"):
        _abi.Context(0, 16, 8 * 65535 + 1, 1)
