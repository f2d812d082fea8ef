"""ctypes binding of the C ABI in ``include/pi2rh.h`` (``_lib/libpi2rh.so``).

There is no CPU fallback: if the shared library is missing or no CUDA
device is visible, the calls raise.  Build with
``python -c "import __graft_entry__ as g; g.build()"`` (or
``python -m paper_1503_00330_b200._build``).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libpi2rh.so")

PI2_OK, PI2_ERR_INVALID, PI2_ERR_STATE, PI2_ERR_UNSUPPORTED, PI2_ERR_CUDA, PI2_ERR_OOM = range(6)
MODEL_HYBRID_LWPR, MODEL_ANALYTIC, MODEL_TWO_POINT = 1, 2, 3
COST_NAVIGATION, COST_THRESHOLD = 0, 1
STREAM_CONTROL, STREAM_DYNAMICS = 1, 2
MAX_OBSTACLES = 16
MAX_SUB_ROLLOUTS = 256
PARTIAL_WIDTH = 6


class Dims(C.Structure):
    _fields_ = [("num_rollouts", C.c_int64), ("rollout_offset", C.c_int64),
                ("num_rollouts_total", C.c_int64), ("horizon_steps", C.c_int32),
                ("sub_rollouts", C.c_int32)]


class Dynamics(C.Structure):
    _fields_ = [("mass", C.c_double), ("gravity", C.c_double), ("rate_gain", C.c_double),
                ("dt", C.c_double), ("lo", C.c_double * 4), ("hi", C.c_double * 4)]


class Cost(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_obstacles", C.c_int32), ("waypoint", C.c_float * 3),
                ("z_floor", C.c_float), ("arena_lo", C.c_float * 3), ("arena_hi", C.c_float * 3),
                ("obstacles", C.c_float * (2 * MAX_OBSTACLES)), ("threshold", C.c_float),
                ("variance_penalty", C.c_float)]


class OptimizeArgs(C.Structure):
    _fields_ = [("temperature", C.c_double), ("cost_ceiling", C.c_double),
                ("exploration_std", C.c_double * 4), ("seed", C.c_uint64), ("cycle", C.c_uint64),
                ("iterations", C.c_int32), ("use_graph", C.c_int32)]


_P = C.c_void_p
_SIGNATURES = {
    "pi2_version": (C.c_int, []),
    "pi2_strerror": (C.c_char_p, [C.c_int]),
    "pi2_device_count": (C.c_int, [C.POINTER(C.c_int32)]),
    "pi2_create": (C.c_int, [C.c_int32, C.POINTER(Dims), C.POINTER(_P)]),
    "pi2_destroy": (None, [_P]),
    "pi2_last_error": (C.c_char_p, [_P]),
    "pi2_get_dims": (C.c_int, [_P, C.POINTER(Dims)]),
    "pi2_set_dynamics": (C.c_int, [_P, C.POINTER(Dynamics)]),
    "pi2_set_lwpr_axis": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _P, _P, _P, _P]),
    "pi2_select_model": (C.c_int, [_P, C.c_int32, C.c_double]),
    "pi2_set_cost": (C.c_int, [_P, C.POINTER(Cost)]),
    "pi2_set_cost_obstacles": (C.c_int, [_P, C.c_int32, _P]),
    "pi2_evaluate": (C.c_int, [_P, _P, _P, _P, _P, C.c_double, _P, _P]),
    "pi2_evaluate_device": (C.c_int, [_P, _P, _P, _P, _P, C.c_double, _P, _P, _P]),
    "pi2_evaluate_device_noise": (C.c_int, [_P, _P, _P, C.POINTER(OptimizeArgs), C.c_int32, _P, _P, _P]),
    "pi2_update": (C.c_int, [_P, C.c_int64, C.c_int32, _P, _P, _P, C.c_double, _P]),
    "pi2_update_device": (C.c_int, [_P, C.c_int64, C.c_int32, _P, _P, _P, C.c_double, _P, _P]),
    "pi2_optimize": (C.c_int, [_P, _P, _P, C.POINTER(OptimizeArgs)]),
    "pi2_iterate_device": (C.c_int, [_P, C.POINTER(OptimizeArgs), _P]),
    "pi2_receding_horizon_step": (C.c_int, [_P, _P, _P, C.POINTER(OptimizeArgs), _P]),
    "pi2_load_plan": (C.c_int, [_P, _P, _P, _P]),
    "pi2_read_plan": (C.c_int, [_P, _P, _P]),
    "pi2_iterate_local": (C.c_int, [_P, C.POINTER(OptimizeArgs), C.c_int32, _P, _P]),
    "pi2_iterate_finalize": (C.c_int, [_P, _P, C.c_int32, C.c_double, _P]),
    "pi2_stage_step": (C.c_int, [_P, _P, _P, C.POINTER(OptimizeArgs)]),
    "pi2_enqueue_pull": (C.c_int, [_P, _P]),
    "pi2_iterate_local_staged": (C.c_int, [_P, C.c_int32, C.c_double, _P, _P]),
    "pi2_enqueue_push": (C.c_int, [_P, _P]),
    "pi2_fetch_plan": (C.c_int, [_P, _P, _P]),
    "pi2_combine_partials_host": (C.c_int, [_P, C.c_int64, C.c_int32, C.c_double, _P]),
    "pi2_chunk_partials_host": (C.c_int, [_P, _P, C.c_int64, C.c_int32, C.c_double, _P]),
    "pi2_partial_chunk": (C.c_int64, []),
    "pi2_profile_iteration": (C.c_int, [_P, C.POINTER(OptimizeArgs), C.c_int32, _P]),
    "pi2_profile_evaluate": (C.c_int, [_P, _P, _P, _P, _P, C.c_int32, _P]),
    "pi2_lwpr_kernel": (C.c_int, [_P, C.c_int32, _P, _P]),
    "pi2_fused_step": (C.c_int, [_P, _P]),
    "pi2_device_noise": (C.c_int, [_P, C.c_int32, C.c_uint64, C.c_uint64, C.c_uint64, _P, _P]),
    "pi2_lwpr_predict": (C.c_int, [_P, C.c_int32, C.c_int64, _P, _P, _P]),
}

_lib = None


def lib():
    """Load ``libpi2rh.so`` once (raises ImportError when it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"CUDA extension {LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(the PI²-RH path has no CPU fallback)")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


class Pi2Error(RuntimeError):
    """A failed ABI call; ``status`` is the PI2_* code."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


def check(status: int, ctx=None) -> None:
    if status == PI2_OK:
        return
    msg = lib().pi2_last_error(ctx).decode(errors="replace") or lib().pi2_strerror(status).decode()
    if status == PI2_ERR_INVALID:
        raise ValueError(msg)
    if status == PI2_ERR_UNSUPPORTED:
        raise TypeError(msg)
    if status == PI2_ERR_STATE:
        raise ValueError(msg)
    raise Pi2Error(status, msg)


def ptr(a) -> C.c_void_p | None:
    """Data pointer of a C-contiguous numpy array / torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays passed to the C ABI must be C-contiguous")
        return C.c_void_p(a.ctypes.data)
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    if isinstance(a, int):
        return C.c_void_p(a)
    raise TypeError(f"cannot pass {type(a).__name__} to the C ABI")


CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: the legacy default stream


def torch_stream(device=None) -> C.c_void_p:
    """ABI stream handle of torch's current stream on ``device``.

    torch reports its default stream as handle 0, which the ABI would read as
    "the context's own stream"; map it to cudaStreamLegacy so kernels, torch
    events and torch collectives really share one stream.
    """
    import torch

    h = torch.cuda.current_stream(device).cuda_stream
    return C.c_void_p(h if h else CUDA_STREAM_LEGACY)


def device_count() -> int:
    n = C.c_int32(0)
    lib().pi2_device_count(C.byref(n))
    return int(n.value)


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


class Context:
    """Owning handle of one ``pi2_ctx`` (one RolloutEngine workspace on one GPU)."""

    def __init__(self, device: int, num_rollouts: int, horizon: int, sub_rollouts: int,
                 rollout_offset: int = 0, num_rollouts_total: int = 0):
        L = lib()
        self.dims = Dims(int(num_rollouts), int(rollout_offset), int(num_rollouts_total or num_rollouts),
                         int(horizon), int(sub_rollouts))
        h = C.c_void_p()
        check(L.pi2_create(int(device), C.byref(self.dims), C.byref(h)), None)
        self.handle = h
        self.device = int(device)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _lib is not None:
            _lib.pi2_destroy(h)
            self.handle = None

    def call(self, name: str, *args):
        check(getattr(lib(), name)(self.handle, *args), self.handle)
