"""The host replica of the device noise (tests/devnoise.py) against Philox4x32-10's
published known-answer vectors (Random123 kat_vectors), and its Box-Muller
statistics.  The GPU side (pi2_device_noise == replica) is in test_gpu_parity.py."""

import numpy as np
import pytest

from tests import devnoise


@pytest.mark.parametrize("ctr,key,expect", [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
])
def test_philox4x32_10_known_answers(ctr, key, expect):
    out = devnoise.philox_rounds([np.array([w], np.uint32) for w in ctr], *key)[0]
    assert tuple(int(x) for x in out) == expect


def test_replica_streams_are_standard_normal_and_addressed():
    std = np.array([1.5, 1.5, 0.6, 0.04])
    e = devnoise.control_noise(7, 3, 1, 2000, 50, std)
    np.testing.assert_allclose(e.std(axis=(0, 1)) / std, 1.0, atol=0.02)
    np.testing.assert_allclose(e.mean(axis=(0, 1)) / std, 0.0, atol=0.02)
    assert not np.array_equal(e, devnoise.control_noise(7, 3, 17, 2000, 50, std))
    # a shard's rows are the same rows of the whole population
    np.testing.assert_array_equal(devnoise.control_noise(7, 3, 1, 500, 50, std, k_off=1500), e[1500:])
    z = devnoise.dynamics_noise(7, 3, 1, 300, 4, 50)
    np.testing.assert_allclose(z.std(), 1.0, atol=0.02)


def test_dynamics_stream_uses_all_four_normals_of_each_block():
    """Dynamics draws: sub-rollout (k, m) reads its Philox blocks as one sequence, all
    four normals of each (csrc/kernels.cuh DynDraws), 3 per step; shards read the same
    numbers as the whole population."""
    from paper_1503_00330_b200 import rng

    K, M, N = 3, 2, 8  # N = 8: 6 blocks of 4 = 24 normals, all of them used
    z = devnoise.dynamics_noise(5, 2, 0, K, M, N)
    key = rng.derive_key(5, rng.STREAM_DYNAMICS, 2, 0)
    nb = (3 * N + 3) // 4
    assert nb * 4 == 3 * N
    for k in range(K):
        for m in range(M):
            base = (k * M + m) * nb
            seq = devnoise.normals4(np.arange(base, base + nb, dtype=np.uint64), key).reshape(-1)
            np.testing.assert_array_equal(z[k, m].reshape(-1), seq)
    np.testing.assert_array_equal(devnoise.dynamics_noise(5, 2, 0, 1, M, N, k_off=2), z[2:])
    # an odd horizon: the last block's trailing normals are the only ones left unused
    z5 = devnoise.dynamics_noise(5, 2, 0, 1, 1, 5)
    seq = devnoise.normals4(np.arange(0, 4, dtype=np.uint64), key).reshape(-1)
    np.testing.assert_array_equal(z5[0, 0].reshape(-1), seq[:15])
