"""The fused step kernel (csrc/fused.cuh, opt-in with PI2_FUSED=1) against the unfused chain.

fused_step_kernel runs a device-noise iteration's attitude recurrence, the three
axes' tensor-core LWPR and the sub-rollout integration/cost in one kernel, with the
LWPR inputs and outputs kept on chip.  It computes every value with the same
operations in the same order as attitude_kernel -> lwpr_tc_kernel -> the rollout
kernels, so per-rollout costs-to-go, crash flags and the updated plan (which also
reads the stored exploration normals) must be BITWISE equal to the unfused path
(itself pinned to the oracle by tests/test_gpu_parity.py and
tests/test_gpu_baseline_configs.py).  One case is also checked against the oracle
directly.  Cases cover every sub-rollout template (M = 1, 2, 3 -> 4, 4), 1 to 4
field chunks per axis, K not a multiple of the 128-rollout block, and the opt-in
variance penalty.
"""

import os

import numpy as np
import pytest

import paper_1503_00330_b200 as P
from paper_1503_00330_b200 import _abi
from tests.test_gpu_baseline_configs import (CYCLE, check_costs, device_costs, device_noise, oracle_eval,
                                             setup)

pytestmark = pytest.mark.gpu


def run(K, N, L, M, fused, penalty=0.0):
    old = os.environ.get("PI2_FUSED")
    os.environ["PI2_FUSED"] = "1" if fused else "0"
    try:
        stacks, model, cfg, state, plan, cost = setup(K, N, L, M)
        if penalty:
            cost = P.RolloutCost(P.Task.default(), 1, variance_penalty=penalty)
        eng = P.RolloutEngine(model, cfg, device=0, noise="device")
        new = eng.optimize_device(state, plan, cost, cycle_index=CYCLE)
        ctx = eng.context(K, N)
        mm = _abi.C.c_int32(-1)
        ctx.call("pi2_fused_step", _abi.C.byref(mm))
        costs, crash = device_costs(ctx, cfg, state, plan, K, N)
        return mm.value, new.controls, costs.cpu().numpy(), crash.cpu().numpy(), (stacks, cfg, state, plan, ctx)
    finally:
        if old is None:
            os.environ.pop("PI2_FUSED", None)
        else:
            os.environ["PI2_FUSED"] = old


# horizons >= 40 so that some rollouts crash (crash flags, the +10 crash cost)
@pytest.mark.parametrize("K,N,L,M,mm", [(20000, 50, 100, 4, 4),   # C2-like: 2 chunks/axis (64 + 40)
                                         (9000, 45, 60, 1, 1),     # one chunk per axis, mean-only
                                         (12345, 50, 200, 2, 2),   # 4 chunks (64 + 64 + 64 + 8)
                                         (16384, 40, 150, 3, 4),   # odd M: pairwise tree then plain mean
                                         (10000, 47, 256, 1, 1)])  # 4 full chunks
def test_fused_equals_unfused_bitwise(K, N, L, M, mm):
    got_mm, plan_f, costs_f, crash_f, _ = run(K, N, L, M, True)
    ref_mm, plan_u, costs_u, crash_u, _ = run(K, N, L, M, False)
    assert got_mm == mm and ref_mm == 0
    np.testing.assert_array_equal(costs_f.view(np.uint64), costs_u.view(np.uint64))
    np.testing.assert_array_equal(crash_f, crash_u)
    np.testing.assert_array_equal(plan_f.view(np.uint64), plan_u.view(np.uint64))
    print(f"\nfused == unfused bitwise: K={K} N={N} L={L} M={M}, crashes {int(crash_f.sum())}")


def test_fused_variance_penalty_bitwise():
    """The opt-in uncertainty penalty reads the LWPR std planes even at M = 1: the fused
    kernel then runs its variance instantiation."""
    got_mm, plan_f, costs_f, crash_f, _ = run(12000, 20, 100, 1, True, penalty=0.3)
    _, plan_u, costs_u, crash_u, _ = run(12000, 20, 100, 1, False, penalty=0.3)
    assert got_mm == 1
    np.testing.assert_array_equal(costs_f.view(np.uint64), costs_u.view(np.uint64))
    np.testing.assert_array_equal(crash_f, crash_u)
    np.testing.assert_array_equal(plan_f.view(np.uint64), plan_u.view(np.uint64))


def test_fused_matches_oracle():
    """Direct oracle check of the fused path (the BASELINE gates: costs 1e-5 relative,
    crash flags exact) on every rollout of a C2-shaped batch."""
    K, N, L, M = 16384, 50, 100, 4
    mm, _, costs, crash, (stacks, cfg, state, plan, ctx) = run(K, N, L, M, True)
    assert mm == 4
    eps, dyn = device_noise(ctx, cfg, K, N, M)
    rc, rf, _, _ = oracle_eval(stacks, state, plan, eps, dyn, M, chunk=1024)
    worst = check_costs(costs, crash.astype(bool), rc, rf)
    print(f"\nfused K={K}: max cost rel err {worst:.3e}")


def test_fused_not_taken_when_ineligible():
    """Small K (the warp-per-rollout latency regime) and M > 4 keep the unfused kernels."""
    assert run(4096, 20, 100, 1, True)[0] == 0
    assert run(12000, 20, 100, 8, True)[0] == 0
