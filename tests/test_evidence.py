"""The accuracy claims DESIGN.md makes from committed GPU evidence, checked against
that evidence (profiles/r1/*.jsonl, produced on a B200 by tools/stress_sweep.py
and tools/term_error_probe.py).  No GPU needed."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lines(name):
    with open(os.path.join(ROOT, "profiles", "r1", name)) as f:
        return [json.loads(ln) for ln in f if ln.strip()]


def test_stress_sweep_claims():
    rows = _lines("stress_sweep_p20.jsonl")
    assert {r["elements"] // 10 ** 5 for r in rows} >= {1, 10, 100}  # 1e5 .. 1e9 swept
    for r in rows:
        assert r["passes"] >= 3
        ex = r["b200_exact"]
        # EXACT's reduction vs the fp64 sum of the reference's own terms
        assert max(ex["acc_maxrel_da"], ex["acc_maxrel_db"]) <= 2e-6, r["elements"]
        if "reference_blocked" in r:  # same instance (pass 0): device below the reference
            rb = r["reference_blocked"]
            assert ex["p0_acc_mae_da"] < rb["acc_mae_da"] and ex["p0_acc_mae_db"] < rb["acc_mae_db"]
            fa = r["b200_fast"]
            assert fa["p0_mae_da"] < rb["mae_da"] and fa["p0_mae_db"] < rb["mae_db"]


def test_large_fp64_errors_are_sign_flips():
    for r in _lines("term_error_probe.jsonl"):
        if r["db_maxrel"] > 1e-6:
            assert r["sign_flips"] >= 1
            assert abs(r["err_from_sign_flips"] - r["err"]) <= 4e-3 * abs(r["err"]), r
