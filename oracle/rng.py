"""Noise addressing restated from reference ``rng.py`` (test infrastructure only).

A stream is a numpy ``Philox`` (4x64-10) generator keyed by a splitmix64
hash chain over (seed, *coords); normals are numpy's ziggurat
``standard_normal`` in C order.  numpy is the third-party dependency that
owns the arithmetic (reference pin: ``numpy>=1.24``, ``pyproject.toml:11``).
"""

from __future__ import annotations

import numpy as np

M64 = 0xFFFFFFFFFFFFFFFF
STREAM_CONTROL, STREAM_DYNAMICS, STREAM_GENERIC = 1, 2, 3  # rng.py:19-21


def mix64(v: int) -> int:
    """splitmix64 finaliser — rng.py:24-30."""
    v = (v + 0x9E3779B97F4A7C15) & M64
    v = ((v ^ (v >> 30)) * 0xBF58476D1CE4E5B9) & M64
    v = ((v ^ (v >> 27)) * 0x94D049BB133111EB) & M64
    return v ^ (v >> 31)


def philox_key(seed: int, *coords: int) -> tuple[int, int]:
    """128-bit key from the address chain — rng.py:33-44."""
    acc = mix64(int(seed) & M64)
    for c in coords:
        acc = mix64(acc ^ (int(c) & M64))
    return mix64(acc), mix64(acc ^ 0xA5A5A5A5A5A5A5A5)


def normals(seed: int, coords, shape, dtype=np.float64) -> np.ndarray:
    """Standard-normal block for a stream address — rng.py:47-64."""
    key = np.array(philox_key(seed, *coords), dtype=np.uint64)
    gen = np.random.Generator(np.random.Philox(key=key))
    return gen.standard_normal(shape, dtype=dtype)


def control_noise(seed, cycle, iteration, K, N, std):
    """``sample_noise`` — controller.py:112-125."""
    eps = normals(seed, (STREAM_CONTROL, cycle, iteration), (K, N, 4))
    eps *= np.asarray(std, float)[None, None, :]
    return eps


def dynamics_noise(seed, cycle, iteration, K, M, N):
    """``sample_dynamics_noise`` — controller.py:128-139."""
    return normals(seed, (STREAM_DYNAMICS, cycle, iteration), (K, M, N, 3), np.float32)
