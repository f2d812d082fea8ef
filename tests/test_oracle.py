"""The CPU oracle against the golden fixtures produced by the real reference.

On the machine that generated the fixtures (same numpy/OpenBLAS build) the
oracle is bitwise equal; elsewhere numpy's SIMD exp/sgemm dispatch may
move the last float32 ulp, so the assertions allow a few ulps.
"""

import numpy as np
import pytest

from oracle import lwpr as OL
from oracle import rng as OR
from oracle import rollout as RO
from tests._cases import TASK_OBSTACLES, TASK_WAYPOINTS, eval_case_names, load, stacks_from


def test_rng_keys_and_blocks():
    z = load("rng")
    coords = [(0,), (1, 0, 0), (1, 3, 1), (2, 7, 0), (3, 2**40, 5), (1, 2**64 - 1, 2)]
    for i, s in enumerate(z["seeds"]):
        for j, c in enumerate(coords):
            assert OR.philox_key(int(s), *c) == tuple(int(v) for v in z["keys"][i, j])
    for v, want in zip([0, 1, 2**64 - 1, 0x123456789ABCDEF], z["splitmix"]):
        assert OR.mix64(v) == int(want)
    np.testing.assert_array_equal(OR.normals(8, (1, 3, 1), (3, 4, 4)), z["normal_block"])
    np.testing.assert_array_equal(OR.normals(8, (2, 3, 1), (2, 3, 4, 3), np.float32), z["normal_block32"])


def test_wrap_angle():
    z = load("rng")
    np.testing.assert_array_equal(RO.wrap(z["angles"]), z["wrapped"])


def test_lwpr_fast_path_diag():
    z = load("lwpr")
    st = stacks_from(z, "diag_")
    for a in range(3):
        p = OL.fold(st[a].centers, st[a].metrics, st[a].coefs, st[a].lvar)
        assert p["diagonal"]
        m, v = OL.predict_f32(p, z["diag_X"])
        np.testing.assert_allclose(m, z[f"diag_mean{a}"], rtol=2e-6, atol=2e-6)
        np.testing.assert_allclose(v, z[f"diag_var{a}"], rtol=2e-6, atol=2e-7)
        m64, v64 = OL.predict_f64(st[a].centers, st[a].metrics, st[a].coefs, st[a].lvar,
                                  z["diag_X"].astype(np.float64))
        np.testing.assert_allclose(m64, z[f"diag_mean64_{a}"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(v64, z[f"diag_var64_{a}"], rtol=1e-12, atol=1e-12)


def test_lwpr_fast_path_full_metric():
    z = load("lwpr")
    for i in range(int(z["n_full"])):
        p = OL.fold(z[f"full{i}_centers"], z[f"full{i}_metrics"], z[f"full{i}_coefs"], z[f"full{i}_lvar"])
        assert p["diagonal"] == bool(z[f"full{i}_diag"])
        m, v = OL.predict_f32(p, z[f"full{i}_X"])
        np.testing.assert_allclose(m, z[f"full{i}_mean"], rtol=2e-6, atol=2e-6)
        np.testing.assert_allclose(v, z[f"full{i}_var"], rtol=2e-6, atol=2e-6)


def test_scalar_loop_oracle_agrees_with_f64_path():
    z = load("lwpr")
    st = stacks_from(z, "diag_")
    X = z["diag_X"].astype(np.float64)[:20]
    m64, v64 = OL.predict_f64(st[0].centers, st[0].metrics, st[0].coefs, st[0].lvar, X)
    for b in range(len(X)):
        m, v = OL.blend_loop(st[0].centers, st[0].metrics, st[0].coefs, st[0].lvar, X[b])
        assert m == pytest.approx(m64[b], rel=1e-10, abs=1e-12)
        assert v == pytest.approx(v64[b], rel=1e-10, abs=1e-12)


def oracle_eval(z, workers=1, chunk=7):
    stacks = stacks_from(z)
    model = RO.Model(stacks)
    cost = RO.Cost(TASK_WAYPOINTS[int(z["waypoint_index"])], TASK_OBSTACLES)
    lo, hi = model.dyn.bounds()
    M = int(z["M"])
    dyn = z["dyn"] if z["dyn"].size else None
    return RO.evaluate(model, z["state"], z["plan"], lo, hi, z["noise"], cost, dyn, M, chunk, workers,
                       float(z["ceiling"]))


@pytest.mark.parametrize("name", eval_case_names())
def test_evaluate_matches_reference(name):
    z = load("eval_" + name)
    costs, crash = oracle_eval(z)
    np.testing.assert_array_equal(crash, z["crash"])
    np.testing.assert_allclose(costs, z["costs"], rtol=1e-6, atol=0)
    assert np.array_equal(costs == z["ceiling"], z["costs"] == z["ceiling"])
    lo, hi = RO.Dyn().bounds()
    new = RO.update(z["plan"], lo, hi, costs, z["noise"], float(z["temperature"]))
    np.testing.assert_allclose(new, z["new_plan"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("name", ["hybrid_m4", "far_m1"])
def test_evaluate_worker_and_chunk_invariance(name):
    """Private scratch per worker: any worker count / chunk gives the serial result."""
    z = load("eval_" + name)
    base, bcrash = oracle_eval(z, workers=1, chunk=7)
    for workers, chunk in [(4, 5), (3, 16), (2, 1000)]:
        c, f = oracle_eval(z, workers=workers, chunk=chunk)
        np.testing.assert_array_equal(c, base)
        np.testing.assert_array_equal(f, bcrash)


def test_update_known_answers():
    z = load("update")
    lo, hi = RO.Dyn().bounds()
    new = RO.update(z["hand_plan"], lo, hi, z["hand_costs"], z["hand_noise"], 1.0)
    np.testing.assert_array_equal(new, z["hand_new"])
    w1 = 1.0 / (1.0 + np.exp(-1.0))
    np.testing.assert_allclose(new[:, :3] - z["hand_plan"][:, :3], w1 * 0.02 - (1 - w1) * 0.02, atol=1e-12)
    for i in range(int(z["n_random"])):
        new = RO.update(z[f"r{i}_plan"], lo, hi, z[f"r{i}_costs"], z[f"r{i}_noise"], float(z[f"r{i}_lambda"]))
        np.testing.assert_allclose(new, z[f"r{i}_new"], rtol=1e-12, atol=1e-14)


def test_optimize_and_receding_horizon():
    z = load("optimize")
    model = RO.Model(stacks_from(z))
    cost = RO.Cost(TASK_WAYPOINTS[int(z["waypoint_index"])], TASK_OBSTACLES)
    kw = dict(K=int(z["K"]), M=int(z["M"]), iterations=int(z["iterations"]), seed=int(z["seed"]),
              cycle=int(z["cycle"]), chunk=16)
    opt = RO.optimize(model, z["state"], z["plan"], cost, **kw)
    np.testing.assert_allclose(opt, z["optimized"], rtol=1e-9, atol=1e-12)
    ctrl, carried = RO.receding_horizon_step(model, z["state"], z["plan"], cost, **kw)
    np.testing.assert_allclose(ctrl, z["control"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(carried, z["carried"], rtol=1e-9, atol=1e-12)
