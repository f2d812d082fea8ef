"""Shared helpers: rebuild golden-case inputs for the oracle and the CUDA path."""

from __future__ import annotations

import glob
import os

import numpy as np

from paper_1503_00330_b200.synthetic import AxisStack

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TASK_WAYPOINTS = np.array([[-1.1, -0.9, 1.0], [1.1, -0.9, 1.0], [0.0, 1.1, 1.0]])
TASK_OBSTACLES = np.array([[0.0, -0.9], [0.55, 0.1], [-0.55, 0.1]])


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def eval_case_names():
    return sorted(os.path.basename(p)[5:-4] for p in glob.glob(os.path.join(GOLDEN, "eval_*.npz")))


def stacks_from(z, prefix=""):
    if f"{prefix}centers0" not in z:
        return None
    return tuple(
        AxisStack(z[f"{prefix}centers{a}"], z[f"{prefix}metrics{a}"], z[f"{prefix}coefs{a}"],
                  z[f"{prefix}lvar{a}"])
        for a in range(3)
    )
