"""Access model: the reference's closed forms, restated, against
the values the reference itself produced (tests/golden/access_golden.json, from
tests/golden/make_access_golden.py), and the B200 kernels' byte model.

Host arithmetic only (grkan_plan is a host function of the library): no GPU.
"""
import json
import os

import pytest

from paper_2505_13813_b200 import access

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "access_golden.json")))["cases"]


@pytest.mark.parametrize("c", GOLD, ids=lambda c: "%dx%dx%d-g%d-bs%d" % (c["batch"], c["seq"], c["feature"],
                                                                         c["groups"], c["block_size"]))
def test_reference_closed_forms(c):
    mc = c["m1"] + c["n"]
    assert access.predict_accesses_naive(c["batch"], c["seq"], c["feature"], mc) == c["naive"]
    if c["blocked"] is None:
        with pytest.raises(access.TailNotCoveredError):
            access.predict_accesses_blocked(c["batch"], c["seq"], c["feature"], c["block_size"],
                                            c["feature"] // c["groups"], mc)
    else:
        assert access.predict_accesses_blocked(c["batch"], c["seq"], c["feature"], c["block_size"],
                                               c["feature"] // c["groups"], mc) == c["blocked"]
    for naive in (False, True):
        got = access.predicted_total_for_plan(c["batch"], c["seq"], c["feature"], c["block_size"], c["groups"],
                                              mc, naive=naive)
        assert got == c["plan_naive" if naive else "plan_blocked"]
        inst = c.get("instrumented_" + ("naive" if naive else "blocked"))
        if inst:  # the reference's own instrumentation agrees with its model
            assert inst["total"] == got == inst["predicted_total"]


def test_argument_checks_match_the_reference():
    with pytest.raises(ValueError):
        access.predict_accesses_naive(0, 1, 1, 10)
    with pytest.raises(ValueError):
        access.predict_accesses_naive(1, 1, 1, -1)
    with pytest.raises(ValueError):
        access.predict_accesses_blocked(1, 4, 8, 0, 4, 10)
    with pytest.raises(ValueError):
        access.device_traffic(10, 8, 2, "fp16")
    with pytest.raises(ValueError):
        access.device_traffic(10, 8, 2, "fp32", "naive")


@pytest.mark.parametrize("dtype,es", [("fp32", 4), ("bf16", 2), ("fp64", 8)])
@pytest.mark.parametrize("rows,d", [(8 * 197, 192), (128 * 197, 1536), (256 * 197, 3072), (9, 8)])
def test_device_model(dtype, es, rows, d):
    g = 8 if d >= 64 else 2
    e = rows * d
    f = access.device_traffic(rows, d, g, dtype, "fwd")
    assert f.total_bytes == 2 * es * e == f.reference_bytes
    bw = access.device_traffic(rows, d, g, dtype, "bwd")
    assert bw.tensor_bytes == 3 * es * e and bw.atomics == 0
    # the reference's blocked model, in bytes, is the same tensor term plus
    # its per-block coefficient traffic
    assert bw.reference_bytes == es * access.predicted_total_for_plan(1, rows, d, 256, g, 10)
    assert bw.reference_bytes - bw.tensor_bytes == es * 3 * 10 * (-(-rows // 256)) * g
    if rows >= 128 * 197:  # coefficient-partial traffic is noise at the model shapes
        assert bw.partial_bytes < 1e-3 * bw.tensor_bytes
    at = access.device_traffic(rows, d, g, dtype, "bwd_atomic")
    assert at.atomics == 10 * e and at.tensor_bytes == 3 * es * e
    assert at.reference_accesses == access.predict_accesses_naive(1, rows, d, 10)


def test_measured_traffic_recorded_in_profiles():
    """profiles/r1/access_model_vs_ncu.json (tools/access_ncu.py, ncu on a B200):
    K1/K2+K3 DRAM bytes within the model (L2 keeps some dirty lines), K4's
    RED count equal to the model's m_c * E atomics, none in K1-K3."""
    path = os.path.join(os.path.dirname(HERE), "profiles", "r1", "access_model_vs_ncu.json")
    d = json.load(open(path))
    for shape, v in d["shapes"].items():
        for op in ("fwd", "bwd", "bwd_atomic"):
            r = v[op]
            m = access.device_traffic(v["rows"], v["d"], v["groups"], "fp32", op)
            assert r["model_bytes"] == m.total_bytes
            assert 0.8 < r["dram_over_model"] < 1.05, (shape, op)
            assert r["red_thread_ops"] == m.atomics, (shape, op)


def test_summary_reproduces_from_the_committed_ncu_csvs():
    """tools/access_ncu.py summarize, re-run here on the committed raw ncu CSVs,
    gives the committed profiles/r1/access_model_vs_ncu.json numbers."""
    import subprocess
    import sys
    root = os.path.dirname(HERE)
    csvs = [os.path.join(root, "profiles", "r1", "access", "access_%s.csv" % s) for s in ("kat-s", "kat-b")]
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "access_ncu.py"), "summarize", *csvs],
                         capture_output=True, text=True, timeout=120, cwd=root)
    assert out.returncode == 0, out.stderr
    got = json.loads(out.stdout)["shapes"]
    want = json.load(open(os.path.join(root, "profiles", "r1", "access_model_vs_ncu.json")))["shapes"]
    for shape in want:
        for op in ("fwd", "bwd", "bwd_atomic"):
            for key in ("dram_bytes", "model_bytes", "red_thread_ops", "reference_bytes"):
                assert got[shape][op][key] == want[shape][op][key], (shape, op, key)
