"""Parity at every BASELINE.json config, at its full size, through the real-time path.

For each config the engine runs the device-noise control step the benchmark
measures (one CUDA graph: attitude -> tensor-core LWPR -> rollout/cost ->
partials -> combine).  The same iteration's device noise is materialised
(pi2_device_noise) and handed to the oracle (oracle/rollout.py, the numpy
restatement of controller.py:197-247 / :356-371, pinned to the reference's
golden vectors by tests/test_oracle.py), which evaluates the rollouts on the
host cores.  Gates (north star):

* per-rollout costs-to-go within 1e-5 relative, crash flags exact — for EVERY
  rollout at C1, C2, C3 (L=1000, T=100), C4 and C5 (K=2^16); for a
  65,536-rollout sample (8 blocks, the last one ending at the last rollout) at
  C5's K=2^22;
* the control update Δu within 1e-4 per channel against the ORACLE's update of
  the ORACLE's costs (not of ours) at full K;
* the fused step equals our own evaluate + update of the same batch bitwise.
"""

import numpy as np
import pytest

import paper_1503_00330_b200 as P
from paper_1503_00330_b200 import _abi, synthetic
from paper_1503_00330_b200.controller import optimize_args
from oracle import rollout as RO
from tests._cases import TASK_OBSTACLES, TASK_WAYPOINTS

pytestmark = pytest.mark.gpu

COST_RTOL = 1e-5
DU_TOL = 1e-4
CYCLE = 3


def du_err(new, want, plan):
    du, wdu = new - plan, want - plan
    return np.max(np.abs(du - wdu), axis=0) / np.maximum(np.max(np.abs(wdu), axis=0), 1e-300)


def setup(K, N, L, M):
    stacks = synthetic.hybrid_stacks(L, seed=0)
    params = P.QuadParams()
    model = P.HybridModel.from_stacks(stacks, params)
    cfg = P.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=N, iterations_per_step=1, rng_seed=0)
    task = P.Task.default()
    return stacks, model, cfg, P.QuadState.hover(task.spawn), P.ControlPlan.hover(params, N), P.RolloutCost(task, 1)


def device_costs(ctx, cfg, state, plan, K, N):
    """(costs (K,N) f64, crash (K,) bool) of the device-noise iteration, on the GPU."""
    import torch

    costs = torch.empty((K, N), dtype=torch.float64, device="cuda:0")
    crash = torch.empty(K, dtype=torch.uint8, device="cuda:0")
    ctx.call("pi2_evaluate_device_noise", _abi.ptr(state.as_array()), _abi.ptr(np.ascontiguousarray(plan.controls)),
             optimize_args(cfg, CYCLE, use_graph=False), 0, _abi.ptr(costs), _abi.ptr(crash), _abi.torch_stream(0))
    torch.cuda.synchronize()
    return costs, crash


def device_noise(ctx, cfg, K, N, M):
    eps = np.empty((K, N, 4))
    ctx.call("pi2_device_noise", _abi.STREAM_CONTROL, cfg.rng_seed, CYCLE, 0, _abi.ptr(cfg.exploration_std),
             _abi.ptr(eps))
    dyn = None
    if M > 1:
        dyn = np.empty((K, M, N, 3), np.float32)
        ctx.call("pi2_device_noise", _abi.STREAM_DYNAMICS, cfg.rng_seed, CYCLE, 0, None, _abi.ptr(dyn))
    return eps, dyn


def oracle_eval(stacks, state, plan, eps, dyn, M, chunk):
    from threadpoolctl import threadpool_limits

    om = RO.Model(stacks)
    lo, hi = om.dyn.bounds()
    with threadpool_limits(1, "blas"):
        rc, rf = RO.evaluate(om, state.as_array(), plan.controls, lo, hi, eps,
                             RO.Cost(TASK_WAYPOINTS[1], TASK_OBSTACLES), dyn, M, chunk=chunk,
                             workers=RO.default_workers())
    return rc, rf, lo, hi


def check_costs(got_c, got_f, want_c, want_f):
    np.testing.assert_array_equal(got_f, want_f)
    rel = np.abs(got_c - want_c) / np.abs(want_c)
    assert rel.max() < COST_RTOL, (rel.max(), np.unravel_index(rel.argmax(), rel.shape))
    return float(rel.max())


@pytest.mark.parametrize("name,K,N,L,M", [("C1", 1024, 50, 100, 1),
                                          ("C2", 65536, 50, 100, 4),
                                          ("C3", 262144, 100, 1000, 1),
                                          ("C4", 1 << 20, 50, 100, 1),
                                          ("C5", 1 << 16, 50, 200, 1)])
def test_baseline_config_full_k(name, K, N, L, M):
    stacks, model, cfg, state, plan, cost = setup(K, N, L, M)
    eng = P.RolloutEngine(model, cfg, device=0, noise="device")
    fused = eng.optimize_device(state, plan, cost, cycle_index=CYCLE)
    ctx = eng.context(K, N)
    costs_d, crash_d = device_costs(ctx, cfg, state, plan, K, N)
    costs, crash = costs_d.cpu().numpy(), crash_d.cpu().numpy().astype(bool)
    del costs_d, crash_d
    eps, dyn = device_noise(ctx, cfg, K, N, M)
    # the fused step is our evaluate + update of this batch, bitwise
    ours = P.path_integral_update(plan, P.RolloutBatch(eps, costs, crash), cfg.temperature)
    np.testing.assert_array_equal(fused.controls, ours.controls)
    assert 0 < crash.sum() < K  # the workload has both outcomes
    rc, rf, lo, hi = oracle_eval(stacks, state, plan, eps, dyn, M, chunk=256 if L > 500 else 1024)
    worst = check_costs(costs, crash, rc, rf)
    want = RO.update(plan.controls, lo, hi, rc, eps, cfg.temperature)  # the oracle's costs, not ours
    du = du_err(fused.controls, want, plan.controls)
    print(f"\n{name} K={K}: max cost rel err {worst:.3e}, crashes {int(crash.sum())}, du err {du}")
    assert np.all(du < DU_TOL)


def sampled_check(K, N, L, M, sample, blocks=4, chunk=1024):
    """Costs and crash flags of `sample` rollouts (`blocks` contiguous blocks spread over
    K, the last ending at K - 1) from the full-size context against the oracle; the
    blocks' noise comes from shard contexts (device noise is addressed by the global
    rollout index, so a shard draws exactly the full context's numbers)."""
    stacks, model, cfg, state, plan, cost = setup(K, N, L, M)
    eng = P.RolloutEngine(model, cfg, device=0, noise="device")
    fused = eng.optimize_device(state, plan, cost, cycle_index=CYCLE)
    assert np.all(np.isfinite(fused.controls))
    ctx = eng.context(K, N)
    costs_d, crash_d = device_costs(ctx, cfg, state, plan, K, N)
    n = sample // blocks
    starts = [int(s) // 256 * 256 for s in np.linspace(0, K - n, blocks)]
    starts[-1] = K - n
    worst = 0.0
    for s in starts:
        got_c = costs_d[s:s + n].cpu().numpy()
        got_f = crash_d[s:s + n].cpu().numpy().astype(bool)
        shard = _abi.Context(0, n, N, M, rollout_offset=s, num_rollouts_total=K)
        eps, dyn = device_noise(shard, cfg, n, N, M)
        del shard
        rc, rf, _, _ = oracle_eval(stacks, state, plan, eps, dyn, M, chunk)
        worst = max(worst, check_costs(got_c, got_f, rc, rf))
    print(f"\nK={K} L={L}: {len(starts)} blocks of {n}: max cost rel err {worst:.3e}")
    return worst


def test_c5_largest_k_sampled():
    """C5 at its largest K (2^22, L=200): 65,536 rollouts in 8 blocks spread over the
    batch, including the last ones (float4 row indices beyond 2^31 / 16 bytes)."""
    sampled_check(1 << 22, 50, 200, 1, 65536, blocks=8)


@pytest.mark.parametrize("M", [100, 128, 200, 256])
def test_many_sub_rollouts_match_oracle(M):
    """M up to PI2_MAX_SUB_ROLLOUTS = 256 (32 lanes x up to 8 sub-rollouts per rollout; the
    reference has no limit): the device-noise iteration's costs and crash flags against
    the oracle on the same (materialised) noise, power-of-two M (butterfly + slot tree)
    and not (the reference loop replayed in shared memory); ragged K."""
    K, N, L = 700, 16, 24
    stacks, model, cfg, state, plan, cost = setup(K, N, L, M)
    eng = P.RolloutEngine(model, cfg, device=0, noise="device")
    eng.optimize_device(state, plan, cost, cycle_index=CYCLE)  # binds and stages the context
    ctx = eng.context(K, N)
    costs_d, crash_d = device_costs(ctx, cfg, state, plan, K, N)
    eps, dyn = device_noise(ctx, cfg, K, N, M)
    rc, rf, _, _ = oracle_eval(stacks, state, plan, eps, dyn, M, chunk=128)
    check_costs(costs_d.cpu().numpy(), crash_d.cpu().numpy().astype(bool), rc, rf)
    # host-noise evaluate through the engine API (the reference's own sampled streams)
    hb = P.RolloutEngine(model, cfg, device=0).evaluate(state, plan, P.sample_noise(cfg, 1, 0), cost,
                                                       P.sample_dynamics_noise(cfg, 1, 0))
    rc2, rf2, _, _ = oracle_eval(stacks, state, plan, P.sample_noise(cfg, 1, 0), P.sample_dynamics_noise(cfg, 1, 0), M,
                                 chunk=128)
    check_costs(hb.costs_to_go, hb.crash_flags, rc2, rf2)
