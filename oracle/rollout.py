"""Rollout engine, cost plugin and update restated from the reference (test infrastructure only).

Follows reference ``controller.py:142-413`` and ``simworld.py:133-198``
operation by operation (float64 attitude loop, float32 LWPR inputs and
integration, float32 stage cost, pairwise sub-rollout mean, float64
suffix sum, non-finite → ceiling, float64 per-timestep softmax update).
Worker threads get private workspaces *and* private cost scratch (the
reference shares the latter — SURVEY.md §0.3), so any worker count gives
the workers=1 result bitwise.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from . import rng
from .lwpr import analytic_eval, fold, hybrid_eval

TWO_PI = 2.0 * math.pi


def wrap(a):
    """Angle wrap into (-pi, pi] — dynamics.py:27-29."""
    return np.pi - np.mod(np.pi - np.asarray(a), TWO_PI)


@dataclass
class Dyn:
    """QuadParams subset used by rollouts — dynamics.py:32-62."""

    mass: float = 0.019
    gravity: float = 9.81
    rate_gain: float = 25.0
    r_max: float = 10.0
    dt: float = 0.02
    f_max: float | None = None

    def __post_init__(self):
        if self.f_max is None:
            self.f_max = 2.0 * self.mass * self.gravity

    def bounds(self):
        """control_bounds — dynamics.py:53-57."""
        return (np.array([-self.r_max, -self.r_max, -self.r_max, 0.0]),
                np.array([self.r_max, self.r_max, self.r_max, self.f_max]))

    @property
    def hover_thrust(self):
        return self.mass * self.gravity


@dataclass
class Cost:
    """RolloutCost bound to one waypoint — simworld.py:141-146 (float32 copies)."""

    waypoint: np.ndarray
    obstacles: np.ndarray
    z_floor: float = 0.05
    lo: np.ndarray = field(default_factory=lambda: np.array([-2.0, -2.0, 0.0]))
    hi: np.ndarray = field(default_factory=lambda: np.array([2.0, 2.0, 2.5]))
    # opt-in uncertainty penalty (the engine's extension, pi2_cost.variance_penalty;
    # NOT in the reference: 0 reproduces simworld.py:166-198)
    variance_penalty: float = 0.0

    def __post_init__(self):
        self.waypoint = np.asarray(self.waypoint, float).astype(np.float32)
        self.obstacles = np.asarray(self.obstacles, float).reshape(-1, 2).astype(np.float32)
        self.z_floor = np.float32(self.z_floor)
        self.lo = np.asarray(self.lo, float).astype(np.float32)
        self.hi = np.asarray(self.hi, float).astype(np.float32)

    def crash_now(self, pos, out):
        """simworld.py:157-164."""
        np.less_equal(pos[..., 2], self.z_floor, out=out)
        out |= pos[..., 0] < self.lo[0]
        out |= pos[..., 0] > self.hi[0]
        out |= pos[..., 1] < self.lo[1]
        out |= pos[..., 1] > self.hi[1]
        out |= pos[..., 2] > self.hi[2]

    def stage_costs(self, pos, vel, ang, crashed, out):
        """simworld.py:166-198 with per-call scratch."""
        t = np.empty(out.shape, np.float32)
        t2 = np.empty(out.shape, np.float32)
        np.subtract(pos[..., 0], self.waypoint[0], out=out)
        out *= out
        np.subtract(pos[..., 1], self.waypoint[1], out=t)
        t *= t
        out += t
        np.subtract(pos[..., 2], self.waypoint[2], out=t)
        t *= t
        t *= np.float32(10.0)
        out += t
        np.multiply(vel[..., 0], vel[..., 0], out=t)
        t += vel[..., 1] * vel[..., 1]
        t += vel[..., 2] * vel[..., 2]
        t *= np.float32(0.1)
        out += t
        out += (ang * ang).sum(axis=-1) * np.float32(0.2)
        for ox, oy in self.obstacles:
            np.subtract(pos[..., 0], ox, out=t)
            t *= t
            np.subtract(pos[..., 1], oy, out=t2)
            t2 *= t2
            t += t2
            t *= np.float32(-10.0)
            np.exp(t, out=t)
            t *= np.float32(100.0)
            out += t
        out += np.float32(10.0) * crashed


class Model:
    """Model plugin: hybrid LWPR (3 folded axes) or analytic rigid body."""

    def __init__(self, stacks=None, dyn: Dyn | None = None):
        self.dyn = dyn or Dyn()
        self.folded = None if stacks is None else [
            fold(s.centers, s.metrics, s.coefs, s.lvar) for s in stacks
        ]
        self.probabilistic = stacks is not None

    def eval(self, X, want_std):
        if self.folded is None:
            return analytic_eval(X, self.dyn.mass, self.dyn.gravity, want_std)
        return hybrid_eval(self.folded, X, want_std)


def run_chunk(model: Model, state, plan, lo, hi, eps, dyn_c, cost: Cost, use_spread):
    """One chunk of rollouts — controller.py:249-322.  Returns (costs (ch,N), crash (ch,))."""
    p = model.dyn
    ch, n = eps.shape[0], eps.shape[1]
    dt32 = np.float32(p.dt)
    u = np.add(plan[None, :, :], eps)                                    # :258
    np.clip(u, lo[None, None, :], hi[None, None, :], out=u)              # :259
    angs = np.empty((ch, n + 1, 3))
    ang = np.tile(state[6:9], (ch, 1))                                   # :264
    rate = np.tile(state[9:12], (ch, 1))                                 # :265
    gain_dt = p.rate_gain * p.dt                                         # :266
    for t in range(n):                                                   # :267-270
        angs[:, t, :] = ang
        ang = wrap(ang + rate * p.dt)
        rate = rate + gain_dt * (u[:, t, :3] - rate)
    angs[:, n, :] = ang                                                  # :271
    xin = np.empty((ch * n, 4), np.float32)                              # :272-275
    xin.reshape(ch, n, 4)[:, :, :3] = angs[:, :n]
    xin.reshape(ch, n, 4)[:, :, 3] = u[:, :, 3]
    pen = cost.variance_penalty > 0 and model.probabilistic              # extension (see Cost)
    mean, std = model.eval(xin, use_spread or pen)                       # :277-279
    m_sub = dyn_c.shape[1] if use_spread else 1
    shape = (ch, m_sub, n, 3)
    acc = np.empty(shape, np.float32)
    mean4 = mean.reshape(ch, 1, n, 3)
    if use_spread:                                                       # :288-293
        np.multiply(std.reshape(ch, 1, n, 3), dyn_c, out=acc)
        acc += mean4
    else:
        acc[:] = mean4
    vel = np.cumsum(acc, axis=2)                                         # :294
    pos = np.cumsum(vel, axis=2)                                         # :295
    pos -= vel                                                           # :296
    pos *= dt32 * dt32                                                   # :297
    vel *= dt32                                                          # :298
    v0 = state[3:6].astype(np.float32)
    vel += v0[None, None, None, :]                                       # :299
    steps32 = np.arange(1, n + 1, dtype=np.float32)[None, None, :, None]
    pos += (dt32 * steps32) * v0[None, None, None, :]                    # :300-301
    pos += state[0:3].astype(np.float32)[None, None, None, :]           # :302
    crashed = np.empty(shape[:3], bool)
    cost.crash_now(pos, crashed)                                         # :305
    np.logical_or.accumulate(crashed, axis=2, out=crashed)               # :306
    ang32 = angs[:, 1:].astype(np.float32)[:, None, :, :]                # :307
    q = np.empty(shape[:3], np.float32)
    cost.stage_costs(pos, vel, ang32, crashed, q)                        # :309
    crash = crashed[:, :, -1].any(axis=1)                                # :310
    qm = q
    while qm.shape[1] > 1:                                               # :314-319
        if qm.shape[1] % 2 == 0:
            qm = 0.5 * (qm[:, 0::2] + qm[:, 1::2])
        else:
            qm = qm.mean(axis=1, keepdims=True)
    qm = qm[:, 0, :]
    if pen:  # kappa * (sd_x^2 + sd_y^2 + sd_z^2) on the sub-rollout-mean stage cost, float32
        s3 = std.reshape(ch, n, 3)
        tr = (s3[..., 0] * s3[..., 0] + s3[..., 1] * s3[..., 1]) + s3[..., 2] * s3[..., 2]
        qm = qm + np.float32(cost.variance_penalty) * tr
    stage = qm.astype(np.float64)                                        # :320
    stage *= p.dt                                                        # :321
    return np.cumsum(stage[:, ::-1], axis=1)[:, ::-1], crash             # :322


def evaluate(model: Model, state, plan, lo, hi, eps, cost: Cost, dyn=None,
             sub_rollouts: int = 1, chunk: int = 1000, workers: int = 1,
             ceiling: float = 1e8):
    """RolloutEngine.evaluate — controller.py:197-247.  Returns (costs (K,N) f64, crash (K,) bool)."""
    state = np.asarray(state, float)
    plan = np.asarray(plan, float)
    k_total, n = eps.shape[0], eps.shape[1]
    if n != plan.shape[0]:
        raise ValueError("noise horizon does not match plan length")
    use_spread = model.probabilistic and sub_rollouts > 1
    if use_spread and dyn is None:
        raise ValueError("probabilistic model with sub_rollouts > 1 needs dyn_noise")
    chunk = min(chunk, k_total)
    costs = np.empty((k_total, n))
    crash = np.empty(k_total, bool)
    spans = [(s, min(s + chunk, k_total)) for s in range(0, k_total, chunk)]

    def one(span):
        s, e = span
        c, f = run_chunk(model, state, plan, lo, hi, eps[s:e],
                         dyn[s:e] if use_spread else None, cost, use_spread)
        costs[s:e] = c
        crash[s:e] = f

    if workers <= 1 or len(spans) == 1:
        for sp in spans:
            one(sp)
    else:
        with ThreadPoolExecutor(max_workers=min(workers, len(spans))) as pool:
            list(pool.map(one, spans))
    bad = ~np.isfinite(costs)                                            # :243-246
    if bad.any():
        costs[bad] = ceiling
        crash |= bad.any(axis=1)
    return costs, crash


def update(plan, lo, hi, costs, eps, temperature):
    """path_integral_update — controller.py:356-371 (returns clipped (N,4))."""
    costs = np.asarray(costs, float)
    eps = np.asarray(eps, float)
    if costs.shape != eps.shape[:2] or plan.shape[0] != costs.shape[1]:
        raise ValueError("batch does not match plan dimensions")
    shifted = costs - costs.min(axis=0)[None, :]
    w = np.exp(shifted * (-1.0 / temperature))
    w /= w.sum(axis=0)[None, :]
    delta = np.einsum("kn,knc->nc", w, eps)
    return np.clip(plan + delta, lo[None, :], hi[None, :])               # ControlPlan :39-45


def optimize(model: Model, state, plan, cost: Cost, K, M=1, iterations=1,
             temperature=1.0, std=(2.0, 2.0, 0.8, 0.05), seed=0, cycle=0,
             chunk=1000, workers=1, ceiling=1e8, return_batches=False):
    """optimize — controller.py:374-395 (host numpy noise, reference stream layout)."""
    lo, hi = model.dyn.bounds()
    plan = np.clip(np.asarray(plan, float), lo[None, :], hi[None, :])
    n = plan.shape[0]
    use_spread = model.probabilistic and M > 1
    batches = []
    for it in range(iterations):
        eps = rng.control_noise(seed, cycle, it, K, n, std)
        dyn = rng.dynamics_noise(seed, cycle, it, K, M, n) if use_spread else None
        c, f = evaluate(model, state, plan, lo, hi, eps, cost, dyn, M, chunk, workers, ceiling)
        if return_batches:
            batches.append((eps, dyn, c, f, plan.copy()))
        plan = update(plan, lo, hi, c, eps, temperature)
    return (plan, batches) if return_batches else plan


def receding_horizon_step(model, state, plan, cost, **kw):
    """controller.py:398-413 → (first control (4,), shifted plan (N,4))."""
    opt = optimize(model, state, plan, cost, **kw)
    return opt[0].copy(), np.vstack([opt[1:], opt[-1:]])


def default_workers() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
