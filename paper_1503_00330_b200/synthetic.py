"""Synthetic workloads for the PI²-RH control step.

The reference ships no trained models and no golden data, so every
benchmark and parity case is built from this seeded generator.  It
produces the three per-axis receptive-field stacks of a hybrid LWPR
acceleration model (``HybridModel``, reference ``dynamics.py:214-277``)
whose local models are the linearisations of the rigid-body acceleration
(``dynamics.py:113-130``) at their centres, plus the default navigation
task of ``simworld.py:71-79``.

Field layout per axis (what ``LwprModel._stacks`` returns,
``lwpr.py:141-150``): centres (L, 4), metrics (L, 4, 4), coefs (L, 5) as
[offset, slope_roll, slope_pitch, slope_yaw, slope_thrust] on inputs
centred at the field centre, local variances (L,).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

MASS = 0.019
GRAVITY = 9.81

# training-grid ranges of the reference's hybrid tests (test_dynamics.py:44-46)
CENTER_LO = np.array([-0.35, -0.35, -0.35, 0.10])
CENTER_HI = np.array([0.35, 0.35, 0.35, 0.28])
METRIC_DIAG = np.array([30.0, 30.0, 30.0, 1500.0])  # test_dynamics.py:39


@dataclass
class AxisStack:
    """Receptive-field stack of one acceleration-axis model."""

    centers: np.ndarray   # (L, 4) float64
    metrics: np.ndarray   # (L, 4, 4) float64
    coefs: np.ndarray     # (L, 5) float64
    lvar: np.ndarray      # (L,) float64

    @property
    def num_fields(self) -> int:
        return int(self.centers.shape[0])


def _thrust_dir_and_jacobian(ang):
    """Body z-axis in the world frame and its derivative w.r.t. (roll, pitch, yaw)."""
    r, p, y = ang
    sr, cr = math.sin(r), math.cos(r)
    sp, cp = math.sin(p), math.cos(p)
    sy, cy = math.sin(y), math.cos(y)
    d = np.array([cr * sp * cy + sr * sy, cr * sp * sy - sr * cy, cr * cp])
    jac = np.array(
        [
            [-sr * sp * cy + cr * sy, cr * cp * cy, -cr * sp * sy + sr * cy],
            [-sr * sp * sy - cr * cy, cr * cp * sy, cr * sp * cy + sr * sy],
            [-sr * cp, -cr * sp, 0.0],
        ]
    )
    return d, jac


def linearised_accel(center, mass=MASS, gravity=GRAVITY):
    """(value (3,), gradient (3, 4)) of the rigid-body acceleration at center."""
    d, jac = _thrust_dir_and_jacobian(center[:3])
    f = center[3]
    a = (f / mass) * d
    a[2] -= gravity
    grad = np.empty((3, 4))
    grad[:, :3] = (f / mass) * jac
    grad[:, 3] = d / mass
    return a, grad


def hybrid_stacks(
    num_fields: int,
    seed: int = 0,
    offset_noise: float = 0.05,
    full_metric: bool = False,
    mass: float = MASS,
    gravity: float = GRAVITY,
) -> tuple[AxisStack, AxisStack, AxisStack]:
    """Three per-axis stacks of ``num_fields`` receptive fields each.

    Drawn axis by axis from ``np.random.default_rng(seed)``:
    centres uniform on the training box, metric diag(30,30,30,1500)
    (``full_metric`` adds a small symmetric off-diagonal part that keeps
    the metric SPD), coefficients = local linearisation of the analytic
    acceleration plus N(0, offset_noise²) on the offset, local variance
    uniform on [0.01, 0.1].
    """
    rng = np.random.default_rng(seed)
    out = []
    for axis in range(3):
        centers = rng.uniform(CENTER_LO, CENTER_HI, size=(num_fields, 4))
        metrics = np.tile(np.diag(METRIC_DIAG), (num_fields, 1, 1))
        if full_metric:
            # off-diagonal coupling at 20 % of the geometric mean of the
            # diagonal entries: strictly diagonally dominant => SPD
            sq = np.sqrt(METRIC_DIAG)
            cross = 0.2 / 3.0 * np.outer(sq, sq)
            np.fill_diagonal(cross, 0.0)
            signs = rng.choice([-1.0, 1.0], size=(num_fields, 4, 4))
            signs = np.triu(signs, 1)
            signs = signs + np.transpose(signs, (0, 2, 1))
            metrics = metrics + signs * cross[None]
        coefs = np.empty((num_fields, 5))
        noise = rng.normal(0.0, offset_noise, size=num_fields)
        for i in range(num_fields):
            a, grad = linearised_accel(centers[i], mass, gravity)
            coefs[i, 0] = a[axis] + noise[i]
            coefs[i, 1:] = grad[axis]
        lvar = rng.uniform(0.01, 0.1, size=num_fields)
        out.append(AxisStack(centers, metrics, coefs, lvar))
    return tuple(out)


# default navigation task (simworld.py:71-79, defaults simworld.py:41-49)
DEFAULT_WAYPOINTS = np.array([[-1.1, -0.9, 1.0], [1.1, -0.9, 1.0], [0.0, 1.1, 1.0]])
DEFAULT_OBSTACLES = np.array([[0.0, -0.9], [0.55, 0.1], [-0.55, 0.1]])
DEFAULT_ARENA_MIN = np.array([-2.0, -2.0, 0.0])
DEFAULT_ARENA_MAX = np.array([2.0, 2.0, 2.5])
DEFAULT_Z_FLOOR = 0.05

# BASELINE.json configs (SURVEY.md §8 notation); "uncertainty penalty on"
# is M=4 sub-rollouts.
CONFIGS = {
    "C1": dict(K=1024, T=50, L=100, M=1),
    "C2": dict(K=65536, T=50, L=100, M=4),
    "C3": dict(K=262144, T=100, L=1000, M=1),
    "C4": dict(K=1 << 20, T=50, L=100, M=1),
    "C5": dict(K=1 << 22, T=50, L=200, M=1),
}


# ---------------------------------------------------------------- the reference's objects
def import_reference():
    """The reference package ``pimpc`` (for the drop-in tests, the closed-loop bench and
    the reference arm): already importable, else the copy installed under
    ``baseline/_ref`` (pip --target from /root/reference; it travels to the GPU box),
    else the source tree.  Returns a namespace with ``controller``, ``dynamics``,
    ``lwpr``, ``simworld``, or None when the reference is not present."""
    import importlib
    import os
    import sys
    import types

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for path in (None, os.path.join(root, "baseline", "_ref"), "/root/reference/pkg/src"):
        if path is not None:
            if not os.path.isdir(os.path.join(path, "pimpc")):
                continue
            if path not in sys.path:
                sys.path.append(path)
        try:
            mods = {n: importlib.import_module(f"pimpc.{n}") for n in ("controller", "dynamics", "lwpr", "simworld")}
        except ImportError:
            continue
        return types.SimpleNamespace(**mods)
    return None


def reference_hybrid(ref, stacks, params=None):
    """A reference ``HybridModel`` (dynamics.py:214-235) holding exactly these receptive
    fields (built field by field, as the reference's own tests build models,
    tests/oracles.py:47-67)."""
    models = []
    for s in stacks:
        m = ref.lwpr.LwprModel(input_dim=s.centers.shape[1])
        for i in range(s.num_fields):
            m.fields.append(ref.lwpr.ReceptiveField(
                center=s.centers[i].copy(), metric=s.metrics[i].copy(), coef=s.coefs[i].copy(),
                local_variance=float(s.lvar[i]), inv_gram=np.eye(s.centers.shape[1] + 1)))
        m._stacked = None
        models.append(m)
    return ref.dynamics.HybridModel(tuple(models), params or ref.dynamics.QuadParams())
