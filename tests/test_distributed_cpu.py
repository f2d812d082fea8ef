"""Multi-rank host logic on CPU (gloo, world_size 2 and 4).

Each rank takes its chunk-aligned shard (``distributed.shard_range``) of a
reference batch, reduces it to per-timestep (min S, Z, V) partials with the
library's host leaf/tree functions (the same arithmetic as the device
kernels), all-gathers the rank partials over gloo in rank order and combines
them with the fixed tree.  The update must equal the single-process one
bitwise (G-invariance) and the reference's path_integral_update to 1e-12.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1503_00330_b200 import _abi
from paper_1503_00330_b200.distributed import apply_partial, combine_gathered_host, shard_range

LO = np.array([-10.0, -10.0, -10.0, 0.0])
HI = np.array([10.0, 10.0, 10.0, 2 * 0.019 * 9.81])


def batch(K=4096, N=13, seed=5):
    r = np.random.default_rng(seed)
    costs = r.uniform(0.0, 25.0, size=(K, N))
    noise = r.normal(size=(K, N, 4)) * np.array([2.0, 2.0, 0.8, 0.05])
    plan = np.tile([0.0, 0.0, 0.0, 0.019 * 9.81], (N, 1))
    return costs, noise, plan


def rank_root(costs, noise, lam):
    lib = _abi.lib()
    K, N = costs.shape
    chunks = -(-K // lib.pi2_partial_chunk())
    leaves = np.empty((chunks, N, 6))
    _abi.check(lib.pi2_chunk_partials_host(_abi.ptr(np.ascontiguousarray(costs)), _abi.ptr(np.ascontiguousarray(noise)),
                                           K, N, lam, _abi.ptr(leaves)))
    return combine_gathered_host(leaves, lam)


def single_process_update(lam=0.7):
    costs, noise, plan = batch()
    return apply_partial(plan, rank_root(costs, noise, lam), LO, HI)


def worker(rank, world, port, lam, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    costs, noise, plan = batch()
    s, e = shard_range(costs.shape[0], rank, world)
    root = torch.from_numpy(rank_root(costs[s:e], noise[s:e], lam))
    gathered = [torch.empty_like(root) for _ in range(world)]
    dist.all_gather(gathered, root)
    new = apply_partial(plan, combine_gathered_host(torch.stack(gathered).numpy(), lam), LO, HI)
    np.save(f"{out_path}.{rank}.npy", new)
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_ranges_cover_and_align():
    for K in (1, 255, 256, 4096, 65536, 100_000):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(K, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == K
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            for a, _ in spans:
                assert a % 256 == 0 or a == K


def test_single_process_matches_reference_update():
    from oracle.rollout import update

    costs, noise, plan = batch()
    want = update(plan, LO, HI, costs, noise, 0.7)
    np.testing.assert_allclose(single_process_update() - plan, want - plan, rtol=1e-11, atol=1e-14)


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_ranks_reproduce_single_process_bitwise(world, tmp_path):
    out = str(tmp_path / "plan")
    mp.start_processes(worker, args=(world, free_port(), 0.7, out), nprocs=world, join=True, start_method="spawn")
    ref = single_process_update()
    for r in range(world):
        np.testing.assert_array_equal(np.load(f"{out}.{r}.npy"), ref)
