"""Host-side API (no GPU): reference-compatible types, LWPR1 persistence,
plugin classification and errors."""

import numpy as np
import pytest

import paper_1503_00330_b200 as P
from paper_1503_00330_b200 import _abi
from paper_1503_00330_b200.controller import model_kind
from paper_1503_00330_b200.lwpr import LwprFormatError, stacks_of
from paper_1503_00330_b200.simworld import cost_struct
from tests._cases import load


def test_load_reference_lwpr1_payload():
    z = load("persistence")
    m = P.load_model(z["blob"].tobytes())
    assert m.num_fields == int(z["num_fields"]) and m.input_dim == 4
    c, mt, cf, lv = stacks_of(m)
    np.testing.assert_array_equal(c, z["centers"])
    np.testing.assert_array_equal(mt, z["metrics"])
    np.testing.assert_array_equal(cf, z["coefs"])
    np.testing.assert_array_equal(lv, z["lvar"])
    # round trip through our writer is lossless
    m2 = P.load_model(P.save_model(m))
    for a, b in zip(stacks_of(m2), stacks_of(m)):
        np.testing.assert_array_equal(a, b)


def test_lwpr1_errors():
    with pytest.raises(LwprFormatError, match="bad magic"):
        P.load_model(b"nope")
    with pytest.raises(LwprFormatError, match="invalid payload"):
        P.load_model(b"LWPR1\n{not json")
    with pytest.raises(LwprFormatError, match="incomplete payload"):
        P.load_model(b'LWPR1\n{"input_dim": 4}')


def test_config_and_plan_validation():
    with pytest.raises(ValueError, match=">= 1"):
        P.PiConfig(num_rollouts=0)
    with pytest.raises(ValueError, match="temperature"):
        P.PiConfig(temperature=0.0)
    with pytest.raises(ValueError, match="exploration_std"):
        P.PiConfig(exploration_std=[1, 1, 0, 1])
    p = P.QuadParams()
    plan = P.ControlPlan.hover(p, 5)
    assert plan.controls.shape == (5, 4)
    sh = plan.shifted()
    np.testing.assert_array_equal(sh.controls[-1], sh.controls[-2])
    assert sh.origin_time == pytest.approx(p.dt)
    clipped = plan.replaced(np.full((5, 4), 100.0))
    np.testing.assert_array_equal(clipped.controls[:, 3], p.f_max)


def test_plugin_classification():
    p = P.QuadParams()
    assert model_kind(P.AnalyticModel(p))[0] == _abi.MODEL_ANALYTIC
    assert model_kind(P.HybridModel.from_stacks(
        __import__("paper_1503_00330_b200.synthetic", fromlist=["x"]).hybrid_stacks(4), p))[0] == _abi.MODEL_HYBRID_LWPR
    class Perturbed:  # the reference's ground-truth PerturbedModel (dynamics.py:190-211)
        params, probabilistic, drag_coeff = p, False, 0.1
    with pytest.raises(TypeError, match="velocity-dependent"):
        model_kind(Perturbed())

    class Weird:
        params = p
    with pytest.raises(TypeError, match="no device implementation"):
        model_kind(Weird())
    c = cost_struct(P.RolloutCost(P.Task.default(), 2))
    assert c.kind == _abi.COST_NAVIGATION and c.n_obstacles == 3
    assert list(c.waypoint) == [0.0, pytest.approx(1.1), 1.0]
    with pytest.raises(TypeError):
        cost_struct(object())
    # longer obstacle lists than the struct holds: the struct carries the first
    # MAX_OBSTACLES and apply_cost stages the whole list (pi2_set_cost_obstacles)
    rng = np.random.default_rng(0)
    task = P.Task(P.Task.default().waypoints, rng.uniform(-1.5, 1.5, size=(40, 2)))
    c = cost_struct(P.RolloutCost(task, 0))
    assert c.n_obstacles == _abi.MAX_OBSTACLES
    assert list(c.obstacles)[:2] == [pytest.approx(float(np.float32(v))) for v in task.obstacles[0]]


def test_lwpr_model_reference_constructor():
    """LwprModel takes the reference's keyword constructor (lwpr.py:100-124): same
    defaults, validation and d_init normalisation, and round-trips through LWPR1."""
    m = P.LwprModel(input_dim=4, d_init=[30.0, 30.0, 30.0, 1500.0], ridge=1e-4)
    np.testing.assert_array_equal(m.d_init, np.diag([30.0, 30.0, 30.0, 1500.0]))
    assert (m.w_gen, m.forgetting, m.ridge, m.participation) == (0.1, 1.0, 1e-4, 1e-3)
    np.testing.assert_array_equal(P.LwprModel(2, d_init=3.0).d_init, 3.0 * np.eye(2))
    np.testing.assert_array_equal(P.LwprModel(2, d_init=[[1.0, 2.0], [0.0, 1.0]]).d_init, [[1.0, 1.0], [1.0, 1.0]])
    for kw, msg in [(dict(input_dim=0), "input_dim"), (dict(input_dim=2, w_gen=1.0), "w_gen"),
                    (dict(input_dim=2, forgetting=0.0), "forgetting"), (dict(input_dim=2, ridge=-1.0), "ridge"),
                    (dict(input_dim=2, d_init=[1.0, 2.0, 3.0]), "length 2"),
                    (dict(input_dim=2, d_init=np.ones((2, 3))), "d_init must be")]:
        with pytest.raises(ValueError, match=msg):
            P.LwprModel(**kw)
    m.fields.append(P.ReceptiveField(np.zeros(4), np.diag([30.0, 30.0, 30.0, 1500.0]), np.arange(5.0), 0.02,
                                     inv_gram=np.eye(5)))
    m2 = P.load_model(P.save_model(m))
    assert (m2.w_gen, m2.ridge) == (0.1, 1e-4)
    np.testing.assert_array_equal(m2.d_init, m.d_init)
    for a, b in zip(stacks_of(m2), stacks_of(m)):
        np.testing.assert_array_equal(a, b)


def test_dropin_patch_restores_reference_module():
    """dropin.patched swaps the engine and step of a controller module for the block only."""
    import types

    from paper_1503_00330_b200 import dropin

    mod = types.SimpleNamespace(RolloutEngine="ref-engine", receding_horizon_step="ref-step")
    times = []
    with dropin.patched(mod, noise="device", device=0, step_times=times):
        assert mod.RolloutEngine.func is P.RolloutEngine
        assert mod.RolloutEngine.keywords == {"noise": "device", "device": 0, "use_graph": True}
        assert mod.receding_horizon_step is not P.receding_horizon_step  # timed wrapper
    assert (mod.RolloutEngine, mod.receding_horizon_step) == ("ref-engine", "ref-step")
    with dropin.patched(mod, noise="reference", replace_step=False):
        assert mod.receding_horizon_step == "ref-step"
    assert P.Task.default().total_switches == 3 * 4
