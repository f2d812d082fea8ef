"""bench.py's JSON-line contract (the driver parses it): one short run of our arm at N=1,
the multi-rank path at N=2 (gloo ranks sharing the one GPU: exercises the self-spawn,
sharding and gather; its timings mean nothing), and the reference arm's line."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def run_bench(*args, env=None, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout, env={**os.environ, **(env or {})})
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_n1():
    d = run_bench("--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--closed-loop-steps", "0",
                  "--no-other-configs", "--no-north-star")
    assert BASE_KEYS <= d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["config"]["K"] == 65536 and d["config"]["workload"].startswith("C2")
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] == "mufu" and 0 < r["frac"] < 1 and r["peak"] > 0
    assert d["gpu_launches"] >= 5 * d["steps"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()


def test_bench_line_n2_multi_rank_path():
    d = run_bench("--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--closed-loop-steps", "0",
                  "--no-north-star", env={"PI2_DIST_BACKEND": "gloo"})
    assert BASE_KEYS <= d.keys()
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["sharding"]["K_per_gpu"] == 32768
    assert "other_configs" not in d  # N=1 only


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-budget-s", "20", timeout=1200)
    assert d["impl"] == "reference"
    if "unavailable" in d:
        pytest.skip(d["unavailable"])
    assert BASE_KEYS <= d.keys() and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["cores"] >= 1
