"""B200-native PI²-RH control step (arXiv 1503.00330) behind the reference ``pimpc`` API.

The hot path — noise, FP64 attitude recurrence, batched LWPR predict,
sub-rollout integration + cost, suffix sums and the per-timestep softmax
update — runs in hand-written sm_100a CUDA kernels (``csrc/``) reached
through the C ABI ``include/pi2rh.h``.  There is no CPU fallback.
"""

from .controller import (  # noqa: F401
    ControlPlan,
    PiConfig,
    RolloutBatch,
    RolloutEngine,
    evaluate_rollouts,
    optimize,
    path_integral_update,
    receding_horizon_step,
    sample_dynamics_noise,
    sample_noise,
)
from .dynamics import AnalyticModel, Control, HybridModel, QuadParams, QuadState, wrap_angle  # noqa: F401
from .lwpr import FrozenLwpr, LwprFormatError, LwprModel, ReceptiveField, load_model, save_model  # noqa: F401
from .simworld import RolloutCost, Task  # noqa: F401

__all__ = [
    "ControlPlan", "PiConfig", "RolloutBatch", "RolloutEngine", "evaluate_rollouts", "optimize",
    "path_integral_update", "receding_horizon_step", "sample_dynamics_noise", "sample_noise",
    "AnalyticModel", "Control", "HybridModel", "QuadParams", "QuadState", "wrap_angle",
    "FrozenLwpr", "LwprFormatError", "LwprModel", "ReceptiveField", "load_model", "save_model",
    "RolloutCost", "Task",
]
