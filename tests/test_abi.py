"""CPU-side checks of the C ABI: the library loads, exports every symbol of
include/pi2rh.h, and fails loudly (no CPU fallback) without a GPU."""

import os
import re

import numpy as np
import pytest

from paper_1503_00330_b200 import _abi

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "pi2rh.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pi2_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(_abi.exported_symbols())


def test_library_exports_every_declared_symbol():
    lib = _abi.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.pi2_version() == 1
    assert lib.pi2_partial_chunk() == 256


def test_struct_layouts_match_header():
    import ctypes as C

    assert C.sizeof(_abi.Dims) == 32
    assert C.sizeof(_abi.Dynamics) == 96
    assert C.sizeof(_abi.Cost) == 4 * (2 + 3 + 1 + 3 + 3 + 32 + 1 + 1)
    assert C.sizeof(_abi.OptimizeArgs) == 8 * 8 + 8


def test_no_gpu_fails_loudly():
    if _abi.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(Exception, match="CUDA"):
        _abi.Context(0, 16, 4, 1)


def test_invalid_dims_rejected_before_device_lookup():
    with pytest.raises(ValueError, match=">= 1"):
        _abi.Context(0, 0, 4, 1)
    with pytest.raises(ValueError, match="sub_rollouts"):
        _abi.Context(0, 8, 4, 257)


def test_host_partials_reproduce_update():
    """Leaf + tree combine on the host give the reference's path_integral_update."""
    from tests._cases import load

    z = load("update")
    lo = np.array([-10.0, -10.0, -10.0, 0.0])
    hi = np.array([10.0, 10.0, 10.0, 2 * 0.019 * 9.81])
    lib = _abi.lib()
    for i in range(int(z["n_random"])):
        costs, noise, lam = z[f"r{i}_costs"], z[f"r{i}_noise"], float(z[f"r{i}_lambda"])
        K, N = costs.shape
        nch = -(-K // lib.pi2_partial_chunk())
        parts = np.empty((nch, N, 6))
        _abi.check(lib.pi2_chunk_partials_host(_abi.ptr(costs), _abi.ptr(np.ascontiguousarray(noise)), K, N,
                                               lam, _abi.ptr(parts)))
        root = np.empty((N, 6))
        _abi.check(lib.pi2_combine_partials_host(_abi.ptr(parts), nch, N, lam, _abi.ptr(root)))
        new = np.clip(z[f"r{i}_plan"] + root[:, 2:] / root[:, 1:2], lo, hi)
        want = z[f"r{i}_new"]
        du, wdu = new - z[f"r{i}_plan"], want - z[f"r{i}_plan"]
        np.testing.assert_allclose(du, wdu, rtol=1e-10, atol=1e-13)
