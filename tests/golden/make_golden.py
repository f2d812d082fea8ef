"""Generate the golden fixtures from the REAL reference implementation.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py

It imports ``pimpc`` from ``/root/reference/pkg/src`` (read-only, never
copied), builds seeded inputs with ``paper_1503_00330_b200.synthetic``,
calls the reference's own public API (``FrozenLwpr.predict_into``,
``LwprModel.predict_batch``, ``RolloutEngine.evaluate``,
``path_integral_update``, ``optimize``, ``receding_horizon_step``,
``rng.derive_key``/``normal_block``, ``wrap_angle``) and writes the inputs
and outputs to ``tests/golden/*.npz``.  The fixtures pin both the oracle
(tests/test_oracle.py) and the CUDA path (tests/test_gpu_*.py).
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg"
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

from pimpc import controller as C  # noqa: E402
from pimpc import dynamics as D  # noqa: E402
from pimpc import lwpr as LW  # noqa: E402
from pimpc import rng as R  # noqa: E402
from pimpc import simworld as S  # noqa: E402

from paper_1503_00330_b200 import synthetic  # noqa: E402


def ref_model(stack) -> LW.LwprModel:
    m = LW.LwprModel(input_dim=stack.centers.shape[1])
    for i in range(stack.num_fields):
        m.fields.append(
            LW.ReceptiveField(
                center=stack.centers[i].copy(),
                metric=stack.metrics[i].copy(),
                coef=stack.coefs[i].copy(),
                local_variance=float(stack.lvar[i]),
                inv_gram=np.eye(stack.centers.shape[1] + 1),
            )
        )
    m._stacked = None
    return m


def ref_hybrid(stacks) -> D.HybridModel:
    return D.HybridModel(tuple(ref_model(s) for s in stacks), D.QuadParams())


def stack_arrays(prefix, stacks):
    out = {}
    for a, s in enumerate(stacks):
        out[f"{prefix}centers{a}"] = s.centers
        out[f"{prefix}metrics{a}"] = s.metrics
        out[f"{prefix}coefs{a}"] = s.coefs
        out[f"{prefix}lvar{a}"] = s.lvar
    return out


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def far_stacks(num_fields=4):
    """A model whose kernels are so narrow that many rollout rows have every
    weight denormal (exp in (-103.97, -87.3)) or zero (0/0 = NaN → cost
    ceiling + crash flag): the FP32 underflow semantics of SURVEY.md §0.9."""
    base = synthetic.hybrid_stacks(num_fields, seed=11)
    out = []
    for s in base:
        m = s.metrics.copy()
        m[:, 3, 3] = 6.0e3
        m[:, 0, 0] = m[:, 1, 1] = m[:, 2, 2] = 3.0e2
        out.append(synthetic.AxisStack(s.centers, m, s.coefs, s.lvar))
    return tuple(out)


def make_lwpr():
    rng = np.random.default_rng(123)
    arrays = {}
    # (1) synthetic diagonal-metric axis models, FP32 fast path + FP64 path
    stacks = synthetic.hybrid_stacks(24, seed=5)
    X = rng.uniform([-0.6, -0.6, -0.6, 0.0], [0.6, 0.6, 0.6, 0.37], size=(257, 4)).astype(np.float32)
    arrays["diag_X"] = X
    arrays.update(stack_arrays("diag_", stacks))
    for a, s in enumerate(stacks):
        m = ref_model(s)
        fr = LW.FrozenLwpr(m, batch_rows=X.shape[0])
        assert fr._diagonal_only
        mean = np.empty(X.shape[0], np.float32)
        var = np.empty(X.shape[0], np.float32)
        fr.predict_into(X, mean, var)
        arrays[f"diag_mean{a}"], arrays[f"diag_var{a}"] = mean, var
        m64, v64 = m.predict_batch(X.astype(np.float64))
        arrays[f"diag_mean64_{a}"], arrays[f"diag_var64_{a}"] = m64, v64
    # (2) full SPD metrics of random dimension (reference tests/oracles.py:47-67)
    from oracles import random_small_model

    r2 = np.random.default_rng(21)
    for i in range(8):
        m = random_small_model(r2)
        c, mt, cf, lv = m._stacks()
        Xf = r2.normal(size=(64, m.input_dim)).astype(np.float32)
        fr = LW.FrozenLwpr(m, batch_rows=64)
        mean = np.empty(64, np.float32)
        var = np.empty(64, np.float32)
        fr.predict_into(Xf, mean, var)
        arrays.update({f"full{i}_centers": c, f"full{i}_metrics": mt, f"full{i}_coefs": cf,
                       f"full{i}_lvar": lv, f"full{i}_X": Xf, f"full{i}_mean": mean,
                       f"full{i}_var": var, f"full{i}_diag": np.array(fr._diagonal_only)})
    # (3) scalar hand cases of tests/test_lwpr.py:54-67 via the scalar oracle
    arrays["n_full"] = np.array(8)
    save("lwpr", **arrays)


def evaluate_case(name, stacks, K, N, M, seed, cycle, waypoint, state_pos=None,
                  plan_thrust=None, chunk=7, std=(2.0, 2.0, 0.8, 0.05), plant=None):
    p = D.QuadParams()
    model = D.AnalyticModel(p) if stacks is None else ref_hybrid(stacks)
    task = S.Task.default()
    cfg = C.PiConfig(num_rollouts=K, sub_rollouts=M, horizon_steps=N, iterations_per_step=1,
                     exploration_std=np.array(std), rng_seed=seed, chunk_size=chunk)
    state = D.QuadState.hover(task.spawn if state_pos is None else np.asarray(state_pos, float))
    plan = C.ControlPlan.hover(p, N)
    if plan_thrust is not None:
        plan = plan.replaced(np.tile([0.0, 0.0, 0.0, plan_thrust], (N, 1)))
    noise = C.sample_noise(cfg, cycle, 0)
    for (k, t, c), v in (plant or {}).items():  # non-finite exploration samples
        noise[k, t, c] = v
    engine = C.RolloutEngine(model, cfg)
    dyn = C.sample_dynamics_noise(cfg, cycle, 0) if engine.use_spread else None
    with np.errstate(invalid="ignore", over="ignore"):
        batch = engine.evaluate(state, plan, noise, S.RolloutCost(task, waypoint), dyn)
        new_plan = C.path_integral_update(plan, batch, cfg.temperature)
    arrays = dict(
        K=np.array(K), N=np.array(N), M=np.array(M), seed=np.array(seed), cycle=np.array(cycle),
        waypoint_index=np.array(waypoint), analytic=np.array(stacks is None),
        state=state.as_array(), plan=plan.controls, noise=noise,
        dyn=dyn if dyn is not None else np.zeros((0,), np.float32),
        std=np.array(std), costs=batch.costs_to_go, crash=batch.crash_flags,
        new_plan=new_plan.controls, temperature=np.array(cfg.temperature),
        ceiling=np.array(cfg.cost_ceiling),
    )
    if stacks is not None:
        arrays.update(stack_arrays("", stacks))
    save("eval_" + name, **arrays)
    return batch


def make_eval():
    evaluate_case("hybrid_m1", synthetic.hybrid_stacks(16, seed=1), K=64, N=20, M=1,
                  seed=0, cycle=0, waypoint=1)
    evaluate_case("hybrid_m4", synthetic.hybrid_stacks(16, seed=2), K=48, N=15, M=4,
                  seed=3, cycle=2, waypoint=0)
    evaluate_case("hybrid_m3", synthetic.hybrid_stacks(12, seed=3), K=40, N=12, M=3,
                  seed=4, cycle=1, waypoint=2)
    evaluate_case("hybrid_m6", synthetic.hybrid_stacks(12, seed=4), K=24, N=10, M=6,
                  seed=5, cycle=0, waypoint=1)
    evaluate_case("full_m2", synthetic.hybrid_stacks(10, seed=6, full_metric=True), K=32, N=10,
                  M=2, seed=6, cycle=3, waypoint=0)
    evaluate_case("analytic", None, K=64, N=25, M=1, seed=7, cycle=1, waypoint=0,
                  state_pos=np.array([-1.0, -0.7, 1.1]), std=(1.5, 1.5, 0.6, 0.04))
    b = evaluate_case("far_m1", far_stacks(), K=64, N=30, M=1, seed=8, cycle=0, waypoint=1,
                      std=(4.0, 4.0, 1.5, 0.08))
    print("far_m1: ceiling rows", int((b.costs_to_go == 1e8).any(axis=1).sum()))
    b = evaluate_case("far_m4", far_stacks(), K=32, N=24, M=4, seed=9, cycle=0, waypoint=1,
                      std=(4.0, 4.0, 1.5, 0.08))
    print("far_m4: ceiling rows", int((b.costs_to_go == 1e8).any(axis=1).sum()))
    b = evaluate_case("crash_m1", synthetic.hybrid_stacks(16, seed=10), K=64, N=30, M=1,
                      seed=10, cycle=0, waypoint=0, state_pos=np.array([-1.1, -0.9, 0.3]),
                      plan_thrust=0.175)
    print("crash_m1: crashed", int(b.crash_flags.sum()))
    make_nonfinite()


NONFINITE = {(1, 3, 0): np.nan, (2, 0, 3): np.inf, (3, 5, 1): -np.inf, (5, 9, 2): np.nan,
             (6, 11, 3): np.nan, (7, 2, 0): np.inf}


def make_nonfinite():
    """NaN / +-inf exploration samples: the clip keeps NaN and saturates +-inf
    (controller.py:259), NaN rollouts take the cost ceiling and the crash flag
    (:243-246), and the update's sum over the raw noise turns NaN / inf into a
    NaN or saturated plan entry (:368-371)."""
    for name, m, stacks in (("nonfinite_m1", 1, synthetic.hybrid_stacks(16, seed=11)),
                            ("nonfinite_m4", 4, synthetic.hybrid_stacks(12, seed=12))):
        b = evaluate_case(name, stacks, K=40, N=14, M=m, seed=13, cycle=0, waypoint=1, plant=NONFINITE)
        print(name, "ceiling rollouts", int((b.costs_to_go == 1e8).all(axis=1).sum()),
              "crashed", int(b.crash_flags.sum()))


def make_update():
    arrays = {}
    # hand softmax (test_controller.py:213-223)
    noise = np.zeros((2, 3, 4))
    noise[0] += 0.02
    noise[1] -= 0.02
    costs = np.vstack([np.ones(3), 2.0 * np.ones(3)])
    plan = C.ControlPlan.hover(D.QuadParams(), 3)
    arrays["hand_noise"], arrays["hand_costs"], arrays["hand_plan"] = noise, costs, plan.controls
    arrays["hand_new"] = C.path_integral_update(
        plan, C.RolloutBatch(noise, costs, np.zeros(2, bool)), 1.0).controls
    # random batches at several temperatures, incl. huge cost spreads
    r = np.random.default_rng(77)
    for i, (k, n, lam, scale) in enumerate([(30, 8, 2.0, 100.0), (257, 13, 0.05, 10.0),
                                            (1000, 5, 1.0, 1e4), (3, 50, 1e3, 1.0)]):
        costs = r.uniform(0, scale, size=(k, n))
        noise = r.normal(size=(k, n, 4)) * np.array([2.0, 2.0, 0.8, 0.05])
        plan = C.ControlPlan.hover(D.QuadParams(), n)
        new = C.path_integral_update(plan, C.RolloutBatch(noise, costs, np.zeros(k, bool)), lam)
        arrays.update({f"r{i}_costs": costs, f"r{i}_noise": noise, f"r{i}_plan": plan.controls,
                       f"r{i}_lambda": np.array(lam), f"r{i}_new": new.controls})
    arrays["n_random"] = np.array(4)
    save("update", **arrays)


def make_optimize():
    stacks = synthetic.hybrid_stacks(16, seed=12)
    p = D.QuadParams()
    model = ref_hybrid(stacks)
    task = S.Task.default()
    cfg = C.PiConfig(num_rollouts=64, sub_rollouts=4, horizon_steps=20, iterations_per_step=2,
                     rng_seed=3, chunk_size=16)
    state = D.QuadState.hover(task.spawn + np.array([0.05, -0.02, 0.03]))
    plan = C.ControlPlan.hover(p, 20)
    cost = S.RolloutCost(task, 1)
    opt = C.optimize(state, plan, cfg, model, cost, cycle_index=5)
    ctrl, carried = C.receding_horizon_step(state, plan, cfg, model, cost, cycle_index=5)
    save("optimize", **stack_arrays("", stacks), state=state.as_array(), plan=plan.controls,
         K=np.array(64), M=np.array(4), N=np.array(20), iterations=np.array(2), seed=np.array(3),
         cycle=np.array(5), waypoint_index=np.array(1), optimized=opt.controls,
         control=ctrl.as_array(), carried=carried.controls)


def make_rng():
    coords = [(0,), (1, 0, 0), (1, 3, 1), (2, 7, 0), (3, 2**40, 5), (1, 2**64 - 1, 2)]
    seeds = [0, 1, 8, 2**63 + 5]
    keys = np.array([[R.derive_key(s, *c) for c in coords] for s in seeds], dtype=np.uint64)
    sm = np.array([R.splitmix64(v) for v in [0, 1, 2**64 - 1, 0x123456789ABCDEF]], np.uint64)
    blk = R.normal_block(8, (1, 3, 1), (3, 4, 4))
    blk32 = R.normal_block(8, (2, 3, 1), (2, 3, 4, 3), dtype=np.float32)
    angles = np.array([0.0, np.pi, -np.pi, 3 * np.pi, -3 * np.pi, 1e-300, -1e-300, 7.5, -7.5,
                       np.nextafter(np.pi, 4), np.nextafter(-np.pi, -4), 100.0, -100.0,
                       2 * np.pi, -2 * np.pi, 1e6, 1.0e-17])
    save("rng", coords_len=np.array([len(c) for c in coords]), keys=keys, splitmix=sm,
         seeds=np.array(seeds, dtype=np.uint64), normal_block=blk, normal_block32=blk32,
         angles=angles, wrapped=D.wrap_angle(angles))


def make_persistence():
    """An LWPR1 payload written by the reference's save_model (lwpr.py:261-285) from a
    model trained with the reference's RLS update (so its fields share d_init)."""
    m = LW.LwprModel(input_dim=4, d_init=[30.0, 30.0, 30.0, 1500.0], ridge=1e-4)
    r = np.random.default_rng(31)
    for _ in range(400):
        x = r.uniform([-0.35, -0.35, -0.35, 0.1], [0.35, 0.35, 0.35, 0.28])
        m.update(x, float(np.sin(x[0]) * x[3] / 0.019 + 0.01 * r.normal()))
    blob = LW.save_model(m)
    X = r.uniform([-0.4, -0.4, -0.4, 0.05], [0.4, 0.4, 0.4, 0.33], size=(200, 4)).astype(np.float32)
    fr = LW.FrozenLwpr(m, batch_rows=200)
    mean = np.empty(200, np.float32)
    var = np.empty(200, np.float32)
    fr.predict_into(X, mean, var)
    c, mt, cf, lv = m._stacks()
    save("persistence", blob=np.frombuffer(blob, np.uint8), X=X, mean=mean, var=var, centers=c, metrics=mt,
         coefs=cf, lvar=lv, num_fields=np.array(m.num_fields))
    print("persistence: fields", m.num_fields)


def make_propagate():
    """dynamics.propagate (dynamics.py:305-342) for the analytic, perturbed and hybrid
    models, mean and sample modes, plus a diverging plan."""
    p = D.QuadParams()
    rng = np.random.default_rng(17)
    plan = C.ControlPlan.hover(p, 30).replaced(
        np.column_stack([rng.normal(0, 1.5, (30, 3)), p.hover_thrust + rng.normal(0, 0.01, 30)]))
    state = D.QuadState(np.array([0.2, -0.1, 1.0]), np.array([0.1, 0.0, -0.05]), np.array([0.05, -0.02, 0.3]),
                        np.zeros(3))
    noise = rng.standard_normal((30, 3))
    stacks = synthetic.hybrid_stacks(16, seed=17)
    hyb = ref_hybrid(stacks)
    arrays = dict(plan=plan.controls, state=state.as_array(), noise=noise, **stack_arrays("hybrid_", stacks))
    for name, model, mode in (("analytic", D.AnalyticModel(p), "mean"),
                              ("perturbed", D.PerturbedModel(p, drag_coeff=0.08, thrust_scale=0.97), "mean"),
                              ("hybrid_mean", hyb, "mean"), ("hybrid_sample", hyb, "sample")):
        tr = D.propagate(model, state, plan, 30, mode=mode, noise_seq=noise if mode == "sample" else None)
        arrays[name + "_states"] = tr.states
        arrays[name + "_diverged"] = np.array(tr.diverged)
    wild = plan.replaced(np.tile([0.0, 0.0, 0.0, p.f_max], (30, 1)))  # full thrust: leaves the sanity box
    tr = D.propagate(D.AnalyticModel(p), state, wild, 30, sanity_box=np.array([1.0, 1.0, 1.5]))
    arrays["wild_states"], arrays["wild_diverged"] = tr.states, np.array(tr.diverged)
    save("propagate", **arrays)


def make_trial():
    """Closed loop: reference run_trial (simworld.py:270-380), plan with the control
    model, advance a drag/thrust-biased PerturbedModel."""
    p = D.QuadParams()
    task = S.Task.default()
    gt = D.PerturbedModel(p, drag_coeff=0.08, thrust_scale=0.97)
    cases = {
        "analytic": (D.AnalyticModel(p), C.PiConfig(num_rollouts=256, horizon_steps=30, iterations_per_step=1,
                                                     temperature=0.5), 4, 60),
        "hybrid": (ref_hybrid(synthetic.hybrid_stacks(24, seed=13)),
                   C.PiConfig(num_rollouts=128, sub_rollouts=2, horizon_steps=20, iterations_per_step=2), 2, 40),
    }
    arrays = {}
    for name, (model, cfg, seed, cap) in cases.items():
        r = S.run_trial(task, cfg, model, gt, seed=seed, step_cap=cap)
        arrays.update({f"{name}_rows": r.log_rows, f"{name}_outcome": np.array(r.outcome),
                       f"{name}_steps": np.array(r.steps), f"{name}_total_cost": np.array(r.total_cost),
                       f"{name}_avg_cost": np.array(r.avg_cost_per_sec_horizon),
                       f"{name}_K": np.array(cfg.num_rollouts), f"{name}_M": np.array(cfg.sub_rollouts),
                       f"{name}_N": np.array(cfg.horizon_steps), f"{name}_iters": np.array(cfg.iterations_per_step),
                       f"{name}_temperature": np.array(cfg.temperature), f"{name}_seed": np.array(seed),
                       f"{name}_cap": np.array(cap)})
        print(name, r.outcome, r.steps, r.total_cost)
    arrays.update(stack_arrays("hybrid_", synthetic.hybrid_stacks(24, seed=13)))
    save("trial", **arrays)


if __name__ == "__main__":
    if sys.argv[1:] == ["nonfinite"]:
        make_nonfinite()
        sys.exit(0)
    if sys.argv[1:] == ["propagate"]:
        make_propagate()
        sys.exit(0)
    make_rng()
    make_lwpr()
    make_eval()
    make_update()
    make_optimize()
    make_trial()
    make_persistence()
    make_propagate()
