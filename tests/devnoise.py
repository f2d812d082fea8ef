"""Host replica of the CUDA engine's device noise (test infrastructure only).

The device streams (kernels.cuh: philox4x32_10, box_muller, device_eps,
noise_kernel) are Philox4x32-10 keyed by the reference's stream address
(rng.py:33-44 -> paper_1503_00330_b200.rng.derive_key) with counter
(element-group index, key word 1), then Box-Muller.  The kernels evaluate
Box-Muller with MUFU approximations, so this replica agrees to ~1e-5
absolute, while the Philox bits and the addressing must agree exactly
(a wrong key or counter gives unrelated normals).
"""

import numpy as np

from paper_1503_00330_b200 import rng

_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
_LO = np.uint64(0xFFFFFFFF)


def philox_rounds(c, k0_lo, k0_hi):
    """Philox4x32-10 of counter words c = [c0, c1, c2, c3] (uint32 arrays) under key (k0_lo, k0_hi)."""
    c = [np.asarray(w, np.uint32) for w in c]
    a, b = np.uint32(k0_lo), np.uint32(k0_hi)
    with np.errstate(over="ignore"):  # the key schedule wraps mod 2^32
        return _rounds(c, a, b)


def _rounds(c, a, b):
    for _ in range(10):
        p0 = c[0].astype(np.uint64) * _M0
        p1 = c[2].astype(np.uint64) * _M1
        hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), (p0 & _LO).astype(np.uint32)
        hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), (p1 & _LO).astype(np.uint32)
        c = [hi1 ^ c[1] ^ a, lo1, hi0 ^ c[3] ^ b, lo0]
        a, b = a + _W0, b + _W1
    return np.stack(c, axis=-1)


def philox4x32_10(index: np.ndarray, key: tuple[int, int]) -> np.ndarray:
    """(n, 4) uint32 blocks for counters (index lo, index hi, k1 lo, k1 hi), key (k0 lo, k0 hi)."""
    k0, k1 = key
    idx = np.asarray(index, dtype=np.uint64)
    c = [(idx & _LO).astype(np.uint32), (idx >> np.uint64(32)).astype(np.uint32),
         np.full(idx.shape, k1 & 0xFFFFFFFF, np.uint32), np.full(idx.shape, k1 >> 32, np.uint32)]
    return philox_rounds(c, k0 & 0xFFFFFFFF, k0 >> 32)


def _box_muller(u, v):
    u1 = (u.astype(np.float32).astype(np.float64) * 2.0 ** -32 + 2.0 ** -33).astype(np.float32).astype(np.float64)
    th = (v.astype(np.float32).astype(np.float64) * np.float64(np.float32(1.4629180792671596e-09))
          + np.float64(np.float32(-3.14159265358979))).astype(np.float32).astype(np.float64)
    r = np.sqrt(-2.0 * np.log(u1))
    return r * np.cos(th), r * np.sin(th)


def normals4(index: np.ndarray, key: tuple[int, int]) -> np.ndarray:
    """(n, 4) normals of kernels.cuh normals4 (float64, ~1e-5 of the device's float32)."""
    r = philox4x32_10(index, key)
    z0 = _box_muller(r[:, 0], r[:, 1])
    z1 = _box_muller(r[:, 2], r[:, 3])
    return np.stack([z0[0], z0[1], z1[0], z1[1]], axis=-1)


def control_noise(seed, cycle, iteration, K, N, std, k_off=0):
    """eps (K, N, 4) of the control stream (device_eps)."""
    key = rng.derive_key(seed, rng.STREAM_CONTROL, cycle, iteration)
    k = np.arange(k_off, k_off + K, dtype=np.uint64)
    idx = (k[:, None] * np.uint64(N) + np.arange(N, dtype=np.uint64)[None, :]).reshape(-1)
    return (normals4(idx, key) * np.asarray(std, np.float64)).reshape(K, N, 4)


def dynamics_noise(seed, cycle, iteration, K, M, N, k_off=0):
    """z (K, M, N, 3) of the dynamics stream (rollout kernels / noise_kernel): sub-rollout
    (k, m) reads its Philox blocks (k M + m) * NB + j, j < NB = ceil(3N / 4), as one
    sequence of normals, all four of each block, and step t takes normals 3t .. 3t + 2
    (csrc/kernels.cuh DynDraws / dyn3)."""
    key = rng.derive_key(seed, rng.STREAM_DYNAMICS, cycle, iteration)
    nb = (3 * N + 3) // 4
    km = np.arange(k_off * M, (k_off + K) * M, dtype=np.uint64)
    idx = (km[:, None] * np.uint64(nb) + np.arange(nb, dtype=np.uint64)[None, :]).reshape(-1)
    seq = normals4(idx, key).reshape(K * M, 4 * nb)[:, :3 * N]
    return seq.reshape(K, M, N, 3)
