"""Is the oracle port a fair stand-in for the reference's CPU speed?

Times one optimisation iteration (sample_noise + sample_dynamics_noise +
evaluate + path_integral_update) of the reference `pimpc.controller.optimize`
and of the oracle port `oracle.rollout.optimize` on the same host, the same
synthetic model (synthetic.hybrid_stacks) and the same sample (default
K=4096, T=50, L=100, M=4), with the same worker count, BLAS at 1 thread.

Runs only where /root/reference exists (this build container; the GPU box has
no reference tree).  The reference's RolloutCost keeps per-shape scratch and is
not thread-safe, so it is wrapped in a thread-local proxy.

    python profiles/cpu_port_vs_reference.py [--K 4096] [--M 4] [--L 100] [--reps 5]
"""

import argparse
import os
import statistics
import sys
import threading
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from oracle import rollout as RO  # noqa: E402
from paper_1503_00330_b200 import synthetic  # noqa: E402
from tests.golden.make_golden import ref_hybrid  # noqa: E402
from pimpc import controller as C  # noqa: E402
from pimpc import dynamics as D  # noqa: E402
from pimpc import simworld as S  # noqa: E402


class ThreadLocalCost:
    """One reference RolloutCost per worker thread (its scratch buffers are per object)."""

    def __init__(self, task, waypoint):
        self.task, self.waypoint, self._tl = task, waypoint, threading.local()

    def _cost(self):
        c = getattr(self._tl, "c", None)
        if c is None:
            c = self._tl.c = S.RolloutCost(self.task, self.waypoint)
        return c

    def crash_now(self, pos, out):
        self._cost().crash_now(pos, out)

    def stage_costs(self, pos, vel, ang, crashed, out):
        self._cost().stage_costs(pos, vel, ang, crashed, out)


def timed(f, reps):
    f(0)
    ts = []
    for i in range(reps):
        t0 = time.perf_counter()
        f(i + 1)
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--T", type=int, default=50)
    ap.add_argument("--L", type=int, default=100)
    ap.add_argument("--M", type=int, default=4)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    from threadpoolctl import threadpool_limits

    stacks = synthetic.hybrid_stacks(a.L, seed=0)
    workers_all = RO.default_workers()
    task = S.Task.default()
    ref_model = ref_hybrid(stacks)
    state = D.QuadState.hover(task.spawn)
    plan = C.ControlPlan.hover(D.QuadParams(), a.T)
    om = RO.Model(stacks)
    ocost = RO.Cost(synthetic.DEFAULT_WAYPOINTS[1], synthetic.DEFAULT_OBSTACLES)
    ostate = state.as_array()
    print(f"host: {os.cpu_count()} cpus, {workers_all} usable; K={a.K} T={a.T} L={a.L} M={a.M}")
    with threadpool_limits(1, "blas"):
        for workers in sorted({1, workers_all}):
            chunk = min(1024, -(-a.K // workers))
            cfg = C.PiConfig(num_rollouts=a.K, sub_rollouts=a.M, horizon_steps=a.T, iterations_per_step=1,
                             workers=workers, chunk_size=chunk)
            cost = ThreadLocalCost(task, 1) if workers > 1 else S.RolloutCost(task, 1)
            eng = C.RolloutEngine(ref_model, cfg)
            t_ref = timed(lambda c: C.optimize(state, plan, cfg, ref_model, cost, c, eng), a.reps)
            t_port = timed(lambda c: RO.optimize(om, ostate, plan.controls, ocost, K=a.K, M=a.M, iterations=1,
                                                 chunk=chunk, workers=workers, cycle=c), a.reps)
            print(f"workers {workers:2d}: reference {a.K * a.T / t_ref / 1e6:7.3f} M rollout-steps/s "
                  f"({t_ref * 1e3:8.1f} ms)   oracle port {a.K * a.T / t_port / 1e6:7.3f} M rollout-steps/s "
                  f"({t_port * 1e3:8.1f} ms)   port/reference speed {t_ref / t_port:.2f}")


if __name__ == "__main__":
    main()
