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
