"""ShardedEngine end to end on the GPU: 2 and 4 ranks (processes) share GPU 0,
each with its own context on its rollout shard; the per-timestep partials are
exchanged over gloo through the host (the NCCL path differs only in the
transport).  No kernel waits on another rank's kernel.  Every rank must return
the single-process plan bitwise (G-invariant combine tree)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def setup():
    import paper_1503_00330_b200 as P
    from paper_1503_00330_b200 import synthetic

    params = P.QuadParams()
    model = P.HybridModel.from_stacks(synthetic.hybrid_stacks(32, seed=21), params)
    cfg = P.PiConfig(num_rollouts=4096, sub_rollouts=4, horizon_steps=25, iterations_per_step=2, rng_seed=9)
    task = P.Task.default()
    return P, model, cfg, P.QuadState.hover(task.spawn), P.ControlPlan.hover(params, 25), P.RolloutCost(task, 2)


def worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from paper_1503_00330_b200.distributed import ShardedEngine

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P, model, cfg, state, plan, cost = setup()
    eng = ShardedEngine(model, cfg, device=0)
    res = eng.optimize(state, plan, cost, cycle_index=7)
    np.save(f"{out}.{rank}.npy", res.controls)
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_engine_matches_single_gpu(world, tmp_path):
    P, model, cfg, state, plan, cost = setup()
    ref = P.RolloutEngine(model, cfg, device=0, noise="device", use_graph=False).optimize_device(state, plan, cost, 7)
    out = str(tmp_path / "plan")
    mp.start_processes(worker, args=(world, free_port(), out), nprocs=world, join=True, start_method="spawn")
    for r in range(world):
        np.testing.assert_array_equal(np.load(f"{out}.{r}.npy"), ref.controls)


def nccl_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from paper_1503_00330_b200.distributed import ShardedEngine

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    P, model, cfg, state, plan, cost = setup()
    stream = torch.cuda.Stream(0)
    torch.cuda.set_stream(stream)
    eng = ShardedEngine(model, cfg, device=0)
    assert eng.use_graph
    plans = []
    for cyc in (7, 8, 7):  # capture on the first call, replays after; cycle changes only staged keys
        plans.append(eng.optimize(state, plan, cost, cycle_index=cyc).controls)
    # a new cost plugin (waypoint switch) is staged data too: no re-capture
    plans.append(eng.optimize(state, plan, P.RolloutCost(P.Task.default(), 0), cycle_index=7).controls)
    assert eng.graph_captures == 1
    np.save(f"{out}.{rank}.npy", np.stack(plans))
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_graph_captured_step_matches_single_gpu(tmp_path):
    """The N>1 production path — the rank's whole step (pull, local kernels, NCCL
    all-gather, combine, push) captured once into one CUDA graph and replayed — on the
    one GPU this box has (world size 1: NCCL cannot put two ranks on one device):
    every replay equals the single-context device step bitwise, across cycles and a
    waypoint switch, without re-capture."""
    P, model, cfg, state, plan, cost = setup()
    eng = P.RolloutEngine(model, cfg, device=0, noise="device", use_graph=False)
    want = [eng.optimize_device(state, plan, cost, c).controls for c in (7, 8, 7)]
    want.append(eng.optimize_device(state, plan, P.RolloutCost(P.Task.default(), 0), 7).controls)
    out = str(tmp_path / "plan")
    mp.start_processes(nccl_worker, args=(1, free_port(), out), nprocs=1, join=True, start_method="spawn")
    np.testing.assert_array_equal(np.load(f"{out}.0.npy"), np.stack(want))
