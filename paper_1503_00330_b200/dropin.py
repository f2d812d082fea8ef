"""Drop the GPU engine into the reference package (``pimpc``) in place.

The reference's seams for this path are duck-typed:

* ``optimize`` / ``receding_horizon_step`` take ``engine=`` (controller.py:374-413),
  so ``pimpc.controller.optimize(..., engine=RolloutEngine(model, cfg))`` runs the
  reference's own loop (its host noise streams and its numpy update) with every
  rollout evaluated by the CUDA engine;
* ``run_trial`` builds its engines through a function-local
  ``from .controller import ... RolloutEngine, receding_horizon_step``
  (simworld.py:288, 299-307), so replacing those two attributes of the
  ``pimpc.controller`` module routes the reference's own closed loop — its
  plant, waypoint logic, crash verdicts, K=1 plan-cost probe and metrics —
  through this package.

``patched`` does the replacement for the duration of a ``with`` block.  With
``noise="device"`` each control step is one CUDA graph with device-generated
noise (the real-time mode); with ``noise="reference"`` the engine consumes the
reference's host noise and the results match the reference's to the parity
gates.  The reference objects (``HybridModel`` / ``AnalyticModel``,
``RolloutCost``, ``QuadState``, ``ControlPlan``) are accepted as they are.
"""

from __future__ import annotations

import contextlib
import functools
import time


@contextlib.contextmanager
def patched(controller_module, *, noise: str = "device", device: int | None = None, use_graph: bool = True,
            replace_step: bool = True, step_times: list | None = None):
    """Replace ``controller_module.RolloutEngine`` (and, with ``replace_step``, its
    ``receding_horizon_step``) by this package's for the block.

    ``replace_step=False`` keeps the reference's ``receding_horizon_step`` /
    ``optimize`` (host noise, host update) and swaps only the engine.
    ``step_times``: a list that receives the wall-clock seconds of every
    ``receding_horizon_step`` call (host state in, control out).
    """
    from . import controller as C

    saved = {n: getattr(controller_module, n) for n in ("RolloutEngine", "receding_horizon_step")}
    controller_module.RolloutEngine = functools.partial(C.RolloutEngine, noise=noise, device=device,
                                                        use_graph=use_graph)
    step = C.receding_horizon_step if replace_step else saved["receding_horizon_step"]
    if step_times is not None:
        inner = step

        def step(*args, **kwargs):  # noqa: F811 - the timed wrapper
            t0 = time.perf_counter()
            out = inner(*args, **kwargs)
            step_times.append(time.perf_counter() - t0)
            return out

    controller_module.receding_horizon_step = step
    try:
        yield controller_module
    finally:
        for n, v in saved.items():
            setattr(controller_module, n, v)
