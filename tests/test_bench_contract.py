"""bench.py's JSON line carries every key of the driver's contract (task statement).
The reference arm (the CPU oracle, --impl reference) runs here; our arm's line is checked on the GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config"}


def _run(*args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run("--impl", "reference", "--workload", "c1", "--steps", "2", "--warmup", "3")
    assert BASE <= set(d) and d["impl"] == "reference"
    assert d["steps"] == 2 and d["warmup"] == 3 and d["ms_per_step"] < 60e3   # a step = one bounded sample
    assert d["value"] > 0 and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("c1")


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [[], ["--workload", "c1"], ["--path", "structured", "--workload", "c3"],
                                   ["--path", "mc", "--workload", "c1"],
                                   ["--path", "spectral_dense", "--workload", "c3"]])
def test_our_line(extra):
    d = _run("--steps", "2", "--warmup", "3", *extra)
    assert BASE <= set(d) and d["impl"] == "ours" and d["n_gpus"] == 1 and d["warmup"] >= 3
    assert d["value"] > 0 and d["scaling"] == "weak" and d["data"].startswith("synthetic")
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert r["bound"] in ("hbm", "tensor", "alu") and r["peak"] > 0
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
    assert d["gpu_launches"] > 0
    if d["e2e"] is not None:
        assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    if "spectral_dense" not in extra:        # (no oracle spectrum is timed for the stored-matrix lambda_2)
        cb = d["cpu_baseline"]
        assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0
    if not extra:                        # the default line: c5, HBM-bound GEMV near the roofline
        assert d["config"]["workload"].startswith("c5") and r["frac"] > 0.7 and d["roofline_build"]["frac"] > 0.7
        # the GEMV's own device time (splidar_plan_gemv_time): one timed launch per GEMV pass, shorter than
        # the solve phase per pass, so the kernel's rate is at least the solve phase's
        its = max(d["iterations"][0])
        assert r["kernel_launches"] == 2 * (its - 1) and r["kernel_ms_per_launch"] > 0
        assert r["frac"] >= r["frac_solve_phase"]


def test_gpus_flag_must_match_world():
    """--gpus N under a launcher with a different WORLD_SIZE is an error (exit 2), never a silent
    single-rank run; without WORLD_SIZE, --gpus N > 1 re-launches itself through torch.distributed.run."""
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert out.returncode == 2 and "WORLD_SIZE=1" in out.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("workload,dtype", [("c5", "f64"), ("c4", "f32")])
def test_row_shard_line(workload, dtype):
    """--shard rows on one GPU: a row shard of 1, strong scaling, same solves."""
    d = _run("--shard", "rows", "--workload", workload, "--dtype", dtype, "--steps", "2", "--warmup", "3",
             "--no-cpu-baseline")
    assert BASE <= set(d) and d["scaling"] == "strong" and d["n_gpus"] == 1 and d["value"] > 0
    assert d["config"]["rows_per_rank"] == d["config"]["n_bins"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(d["roofline"])
    assert d["roofline"]["frac"] > 0.5
