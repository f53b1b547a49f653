"""bench.py contract checks: the reference arm (no GPU), the config block, and one small GPU-arm line (-m gpu)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--cpu-sample-batch", "1", "--config", "kat-t"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "elements/s"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_reference_arm_non_zero_rank_is_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--cpu-sample-batch", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_config_block_weak_and_strong():
    sys.path.insert(0, ROOT)
    import bench
    weak = bench.config_block(bench.parse_args(["--gpus", "4"]), bench.CONFIGS["kat-b"], world=4)
    assert weak["batch_per_gpu"] == 256 and weak["global_batch"] == 1024 and weak["parallelism"] == "dp4"
    strong = bench.config_block(bench.parse_args(["--gpus", "4", "--scaling", "strong"]),
                                bench.CONFIGS["kat-b"], world=4)
    assert strong["batch_per_gpu"] == 64 and strong["global_batch"] == 256
    assert "B=64" in strong["workload"]


@pytest.mark.gpu
def test_b200_arm_json_line_small_config():
    """The GPU arm's JSON line carries every key the driver reads (KAT-T, a few steps)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "kat-t", "--steps", "3",
                          "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches"):
        assert key in d, key
    assert d["value"] > 0 and d["steps"] == 3 and d["gpu_launches"] == 3 * 3
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in d["roofline"], key
    for key in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert key in d["e2e"], key
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["reference_api"]["value"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
