"""Host-side API (no GPU): reference-compatible types, LWPR1 persistence,
plugin classification and errors."""

import numpy as np
import pytest

import paper_1503_00330_b200 as P
from paper_1503_00330_b200 import _abi
from paper_1503_00330_b200.controller import model_kind
from paper_1503_00330_b200.lwpr import LwprFormatError, stacks_of
from paper_1503_00330_b200.simworld import cost_struct, closest_pass_metric
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
    with pytest.raises(TypeError, match="velocity-dependent"):
        model_kind(P.PerturbedModel(p, drag_coeff=0.1))

    class Weird:
        params = p
    with pytest.raises(TypeError, match="no device implementation"):
        model_kind(Weird())
    c = cost_struct(P.RolloutCost(P.Task.default(), 2))
    assert c.kind == _abi.COST_NAVIGATION and c.n_obstacles == 3
    assert list(c.waypoint) == [0.0, pytest.approx(1.1), 1.0]
    with pytest.raises(TypeError):
        cost_struct(object())


def test_closest_pass_metric_matches_definition():
    xs = np.linspace(-1.5, 1.5, 200)
    pos = np.stack([xs, np.full_like(xs, -0.9), np.ones_like(xs)], 1)
    passes, avg = closest_pass_metric(pos, np.array([[0.0, -0.9]]))
    assert len(passes) == 1 and passes[0] == pytest.approx(np.abs(xs).min())
    assert avg == passes[0]


def test_plant_step_matches_reference_euler():
    p = P.QuadParams()
    st = P.QuadState(np.array([0.1, 0.2, 1.0]), np.array([0.3, -0.1, 0.0]), np.array([0.05, -0.02, 0.1]),
                     np.array([0.5, 0.0, -0.2]))
    c = p.control([1.0, -2.0, 0.5], 0.2)
    nxt = P.AnalyticModel(p).step(st, c)
    np.testing.assert_array_equal(nxt.position, st.position + st.velocity * p.dt)
    np.testing.assert_allclose(nxt.rates, st.rates + p.rate_gain * (c.desired_rates - st.rates) * p.dt)


def _propagate_inputs(z):
    p = P.QuadParams()
    plan = P.ControlPlan(z["plan"], p.dt, 0.0, *p.control_bounds())
    return p, plan, P.QuadState.from_array(z["state"])


@pytest.mark.parametrize("name", ["analytic", "perturbed"])
def test_propagate_matches_reference(name):
    """dynamics.propagate (dynamics.py:305-342) with the host models: bitwise."""
    z = load("propagate")
    p, plan, state = _propagate_inputs(z)
    model = P.AnalyticModel(p) if name == "analytic" else P.PerturbedModel(p, drag_coeff=0.08, thrust_scale=0.97)
    tr = P.propagate(model, state, plan, 30)
    np.testing.assert_array_equal(tr.states, z[name + "_states"])
    assert tr.diverged == bool(z[name + "_diverged"])
    np.testing.assert_array_equal(tr.positions, tr.states[:, :3])
    np.testing.assert_array_equal(tr.final_state().as_array(), tr.states[-1])
    # the same through step_analytic for the analytic model
    if name == "analytic":
        s = state
        for i in range(30):
            s = P.step_analytic(s, p.control(plan.controls[i, :3], plan.controls[i, 3]), p)
        np.testing.assert_array_equal(s.as_array(), tr.states[-1])


def test_propagate_divergence_and_errors():
    z = load("propagate")
    p, plan, state = _propagate_inputs(z)
    wild = np.tile([0.0, 0.0, 0.0, p.f_max], (30, 1))
    tr = P.propagate(P.AnalyticModel(p), state, wild, 30, sanity_box=np.array([1.0, 1.0, 1.5]))
    np.testing.assert_array_equal(tr.states, z["wild_states"])
    assert tr.diverged and bool(z["wild_diverged"])
    with pytest.raises(ValueError, match="exceeds plan length"):
        P.propagate(P.AnalyticModel(p), state, plan, 31)
    with pytest.raises(ValueError, match="requires noise"):
        P.propagate(P.AnalyticModel(p), state, plan, 30, mode="sample")
    with pytest.raises(TypeError, match="velocity-dependent"):
        P.PerturbedModel(p, drag_coeff=0.1).make_batch_eval(8)
    assert P.Task.default().total_switches == 3 * 4
