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
    # the reference itself when installed into baseline/_ref (build()), else the oracle port
    kind = "reference" if os.path.isfile(os.path.join(ROOT, "baseline", "_ref", "grkan", "backward.py")) else "port"
    assert d["cpu_baseline"]["kind"] == kind and d["cpu_baseline"]["cores"] >= 1
    assert "cpu_model" in d["cpu_baseline"]
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


def test_world_size_and_gpus_must_agree():
    env = dict(os.environ, RANK="0", WORLD_SIZE="2", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--config", "kat-t"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 2 and "WORLD_SIZE=2" in out.stderr and out.stdout.strip() == ""


def test_gpus_without_launcher_spawns_ranks(monkeypatch):
    """--gpus N with no WORLD_SIZE re-executes under torch.distributed.run with N ranks."""
    sys.path.insert(0, ROOT)
    import bench
    seen = {}

    class Done:
        returncode = 0

    def fake_run(cmd, env=None):
        seen["cmd"], seen["env"] = cmd, env
        return Done()

    import subprocess as sp
    monkeypatch.setattr(sp, "run", fake_run)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    assert bench.main(["--gpus", "8", "--steps", "20", "--warmup", "5"]) == 0
    cmd = seen["cmd"]
    i = cmd.index("--nproc-per-node")
    assert cmd[i + 1] == "8" and "torch.distributed.run" in cmd and "127.0.0.1" in cmd
    assert cmd[-6:] == ["--gpus", "8", "--steps", "20", "--warmup", "5"]


def test_run_bench_flag_surface_reference_arm():
    """run_bench's workload flags (pkg/src/grkan/cli.py:341-361) reach the config block and the CPU arm."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "kat-t",
                          "--steps", "1", "--warmup", "0", "--batch", "2", "--seqlen", "5", "--dim", "64",
                          "--groups", "4", "--num-coeffs", "4", "--den-coeffs", "2", "--seed", "3",
                          "--no-single-thread-baseline"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    d = json.loads(out.stdout.strip().splitlines()[-1])
    c = d["config"]
    assert (c["batch_per_gpu"], c["seq_len"], c["dim"], c["groups"], c["degrees"], c["seed"]) == \
        (2, 5, 64, 4, [3, 2], 3)
    assert "E=640" in d["cpu_baseline"]["sample"]
    bad = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--dim", "10",
                          "--groups", "4"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert bad.returncode != 0 and "layout mismatch" in bad.stderr


@pytest.mark.gpu
def test_gpus_2_without_launcher_runs_two_ranks():
    """bench.py --gpus 2 with no torchrun wrapper: two ranks (sharing the test box's GPU over
    gloo), n_gpus 2, and da||db bitwise identical on both ranks after the exchange."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "kat-t",
                          "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1",
                          "--dist-backend", "gloo"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT,
                         env=dict({k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")},
                                  GRKAN_BENCH_TRACE_AFTER="600", GRKAN_PG_TIMEOUT_S="300"))
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "dp2" and d["dist"]["world_size"] == 2
    assert d["kernels"]["collective_check"]["bitwise_identical"] is True


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
