"""Closed-loop trials on the GPU engine vs the reference's run_trial (golden).

The reference noise streams are used, so the trajectories coincide up to
the float32 drift of the rollout costs, amplified a little by the softmax
feedback over the trial; the tolerances below are checked per column.
"""

import numpy as np
import pytest

import paper_1503_00330_b200 as P
from tests._cases import load, stacks_from

pytestmark = pytest.mark.gpu


def trial_inputs(z, name):
    p = P.QuadParams()
    if name == "analytic":
        model = P.AnalyticModel(p)
    else:
        model = P.HybridModel.from_stacks(stacks_from(z, "hybrid_"), p)
    cfg = P.PiConfig(num_rollouts=int(z[f"{name}_K"]), sub_rollouts=int(z[f"{name}_M"]),
                     horizon_steps=int(z[f"{name}_N"]), iterations_per_step=int(z[f"{name}_iters"]),
                     temperature=float(z[f"{name}_temperature"]))
    return model, cfg, int(z[f"{name}_seed"]), int(z[f"{name}_cap"])


@pytest.mark.parametrize("name", ["analytic", "hybrid"])
def test_trial_matches_reference(name):
    z = load("trial")
    model, cfg, seed, cap = trial_inputs(z, name)
    gt = P.PerturbedModel(P.QuadParams(), drag_coeff=0.08, thrust_scale=0.97)
    r = P.run_trial(P.Task.default(), cfg, model, gt, seed=seed, step_cap=cap)
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
    assert len(r.step_latency_s) == r.steps


def test_device_noise_trial_flies():
    """Real-time mode: device noise, whole control step as one CUDA graph."""
    z = load("trial")
    model, cfg, seed, cap = trial_inputs(z, "hybrid")
    gt = P.PerturbedModel(P.QuadParams(), drag_coeff=0.08, thrust_scale=0.97)
    r = P.run_trial(P.Task.default(), cfg, model, gt, seed=seed, step_cap=cap, noise="device")
    assert r.outcome == "timeout" and r.steps == cap
    assert np.all(np.isfinite(r.log_rows))
    assert np.median(r.step_latency_s) < 0.01
