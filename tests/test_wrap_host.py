"""The engine's wrap_angle (csrc/common.cuh, the same source the kernels compile) built
for the host with g++, against the oracle's numpy wrap (dynamics.py:27-29) bit for bit:
edge cases (signed zeros, +-pi, +-2pi, 4pi boundaries, tiny remainders, NaN/inf) and
random angles."""

import os
import shutil
import subprocess

import numpy as np
import pytest

from oracle import rollout as RO

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def wrap_bin(tmp_path_factory):
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ not available")
    out = str(tmp_path_factory.mktemp("wrap") / "wrap_check")
    cuda_inc = next((p for p in ("/usr/local/cuda/include",) if os.path.isdir(p)), None)
    if cuda_inc is None:
        pytest.skip("CUDA headers not available")
    cmd = [gxx, "-O2", "-std=c++17", "-ffp-contract=off", "-I", cuda_inc, "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(ROOT, "paper_1503_00330_b200", "csrc"), os.path.join(ROOT, "tests", "wrap_check.cpp"),
           "-o", out]
    subprocess.run(cmd, check=True, capture_output=True)
    return out


def run(wrap_bin, tmp_path, x):
    src, dst = tmp_path / "in.bin", tmp_path / "out.bin"
    np.asarray(x, np.float64).tofile(src)
    subprocess.run([wrap_bin, str(src), str(dst)], check=True)
    return np.fromfile(dst, np.float64)


def test_wrap_angle_host_build_matches_numpy(wrap_bin, tmp_path):
    pi, tau = np.pi, 2.0 * np.pi
    edge = [0.0, -0.0, pi, -pi, tau, -tau, 2 * tau, -2 * tau, 3 * tau, pi + tau, pi - tau, pi + 2 * tau,
            np.nextafter(pi, 0), np.nextafter(pi, 4), np.nextafter(-pi, 0), np.nextafter(-pi, -4),
            np.nextafter(pi + tau, 0), np.nextafter(pi + tau, 10), np.nextafter(pi - tau, 0),
            np.nextafter(pi - tau, -10), pi - 2 * tau, -3 * pi, np.nextafter(pi - 2 * tau, 0),
            np.nextafter(pi - 2 * tau, -20), 1e-300, -1e-300, 5e-324, -5e-324, 1e-17, -1e-17,
            1e6, -1e6, 1e300, -1e300, np.inf, -np.inf, np.nan]
    rng = np.random.default_rng(0)
    x = np.concatenate([edge, rng.uniform(-4, 4, 20000), rng.uniform(-40, 40, 20000),
                        pi + rng.uniform(-1e-12, 1e-12, 2000), rng.normal(0, 1e3, 2000)])
    got, want = run(wrap_bin, tmp_path, x), RO.wrap(x)
    same = (got.view(np.uint64) == want.view(np.uint64)) | (np.isnan(got) & np.isnan(want))
    bad = np.flatnonzero(~same)
    assert bad.size == 0, [(x[i], got[i], want[i]) for i in bad[:5]]
