"""Pin the CPU oracle (NumPy + C restatements) to the reference's own outputs.

The fixtures were recorded by importing the reference (tests/golden/make_golden.py);
here both restatements must reproduce them bit for bit.  CPU-only.
"""

import numpy as np
import pytest

from oracle import c_oracle
from oracle import grkan_oracle as orc
from grkan_testutil import sha

CASES_NO_ERR = None


def _cases(golden):
    return [c for c in golden.cases]


def test_manifest_nonempty(golden):
    assert len(golden.cases) >= 20
    assert len(golden.scalars) >= 40


@pytest.mark.parametrize("impl", ["numpy", "c"])
def test_forward_bitwise(golden, impl):
    for case, meta in golden.cases.items():
        x, u, num, den = golden.inputs(case)
        y = orc.forward(x, num, den) if impl == "numpy" else c_oracle.forward(x, num, den)
        assert y.dtype == x.dtype
        assert sha(y) == meta["sha_y"], case


@pytest.mark.parametrize("impl", ["numpy", "c"])
def test_backward_blocked_bitwise(golden, impl):
    for case, meta in golden.cases.items():
        x, u, num, den = golden.inputs(case)
        blk = meta["block_size"]
        if impl == "numpy":
            with np.errstate(over="ignore", invalid="ignore"):
                if meta["error"]:
                    with pytest.raises(FloatingPointError):
                        orc.backward_blocked(x, u, num, den, blk, workers=3)
                    continue
                dx, da, db = orc.backward_blocked(x, u, num, den, blk, workers=3)
        else:
            r = c_oracle.backward(x, u, num, den, blk)
            if meta["error"]:
                assert r["overflow"], case
                continue
            assert not r["overflow"], case
            dx, da, db = r["dx"], r["blocked_da"], r["blocked_db"]
        assert sha(dx) == meta["sha_dx"], case
        assert da.tobytes() == golden.get(case, "blocked_da").tobytes(), case
        assert db.tobytes() == golden.get(case, "blocked_db").tobytes(), case


@pytest.mark.parametrize("impl", ["numpy", "c"])
def test_backward_naive_and_ref64_bitwise(golden, impl):
    for case, meta in golden.cases.items():
        x, u, num, den = golden.inputs(case)
        if impl == "numpy":
            with np.errstate(over="ignore", invalid="ignore"):
                if meta.get("error_naive"):
                    with pytest.raises(FloatingPointError):
                        orc.backward_naive(x, u, num, den)
                else:
                    dx, da, db = orc.backward_naive(x, u, num, den)
                    assert sha(dx) == meta["sha_dx_naive"], case
                    assert da.tobytes() == golden.get(case, "naive_da").tobytes(), case
                    assert db.tobytes() == golden.get(case, "naive_db").tobytes(), case
                ra, rb = orc.ref64_coeff_grads(x, u, num, den)
        else:
            r = c_oracle.backward(x, u, num, den, meta["block_size"])
            if not meta.get("error_naive"):
                assert r["naive_da"].tobytes() == golden.get(case, "naive_da").tobytes(), case
                assert r["naive_db"].tobytes() == golden.get(case, "naive_db").tobytes(), case
            ra, rb = r["ref64_da"], r["ref64_db"]
        np.testing.assert_array_equal(ra, golden.get(case, "ref64_da"), err_msg=case)
        np.testing.assert_array_equal(rb, golden.get(case, "ref64_db"), err_msg=case)


def test_true64_matches_triple_loop_oracle(golden):
    """The fp64 oracles agree with the reference's triple-loop oracle_backward (verification.py:49)."""
    checked = 0
    for case in golden.cases:
        oa = golden.get(case, "oracle_da")
        if oa is None:
            continue
        x, u, num, den = golden.inputs(case)
        num_run = num.astype(x.dtype).astype(np.float64)
        den_run = den.astype(x.dtype).astype(np.float64)
        dx64, da64, db64 = orc.true64_grads(x, u, num_run, den_run)
        r = c_oracle.backward(x, u, num_run, den_run, 7, want=("true64",))
        if x.dtype == np.float64:  # inputs identical to the triple loop's
            assert orc.matrix_rel(da64, oa) <= 1e-12, case
            assert orc.matrix_rel(db64, golden.get(case, "oracle_db")) <= 1e-12, case
            assert orc.matrix_rel(dx64, golden.get(case, "oracle_dx")) <= 1e-12, case
        assert orc.matrix_rel(r["true64_da"], da64) <= 1e-13, case
        assert orc.matrix_rel(r["true64_db"], db64) <= 1e-13, case
        checked += 1
    assert checked >= 8


def test_katt_inputs_regenerate(golden):
    case = "katt_seed0_f32_8x197x192_g8"
    x, u, _, _ = golden.inputs(case)
    assert sha(x) == golden.cases[case]["sha_x"]
    assert sha(u) == golden.cases[case]["sha_u"]


def test_scalar_kats(golden):
    """eval_rational / elementwise_grads known answers (pkg/tests/test_rational.py:25-98)."""
    for s in golden.scalars:
        a = np.array(s["a"], dtype=np.float64)
        b = np.array(s["b"], dtype=np.float64)
        x = np.array([s["x"]])
        u = np.array([s["u"]])
        assert orc.rational(x, a, b)[0] == s["y"], s["tag"]
        dx, ta, tb = orc.element_terms(x, u, a, b)
        assert dx[0] == s["d_x"], s["tag"]
        assert [t[0] for t in ta] == s["d_a"], s["tag"]
        assert [t[0] for t in tb] == s["d_b"], s["tag"]


def test_hand_values():
    # SPEC.md:53-62 / pkg/tests/test_rational.py:26-81
    one = np.array([1.0])
    assert orc.rational(np.array([2.0]), [1.0, 0, 0, 0, 0, 0], [0.0] * 4)[0] == 1.0
    assert orc.rational(np.array([3.0]), [0.0, 1, 0, 0, 0, 0], [0.0] * 4)[0] == 3.0
    assert orc.rational(one, [1.0, 1.0], [1.0])[0] == 1.0
    assert orc.rational(np.array([2.0]), [1.0, 2.0], [])[0] == 5.0
    dx, ta, tb = orc.element_terms(one, one, np.array([1.0, 1.0]), np.array([1.0]))
    assert [t[0] for t in ta] == [0.5, 0.5] and [t[0] for t in tb] == [-0.5] and dx[0] == 0.0


def test_oracle_combine_partials_known_answers():
    """The oracle's combine fold on the reference's own known answers
    (pkg/tests/test_backward.py:176-209): round-robin routing and fp32 absorption."""
    parts = [(0, np.array([1.0]), np.array([10.0])), (1, np.array([2.0]), np.array([20.0])),
             (2, np.array([4.0]), np.array([40.0])), (3, np.array([8.0]), np.array([80.0]))]
    d_a, d_b = orc.combine_partials(parts, 2)
    assert np.array_equal(d_a, [[5.0], [10.0]]) and np.array_equal(d_b, [[50.0], [100.0]])
    tiny = np.float32(2.0 ** -24)
    fresh = [(i, np.array([tiny], dtype=np.float32), np.zeros(0, np.float32)) for i in range(64)]
    assert orc.combine_partials(fresh, 1)[0][0, 0] == np.float32(2.0 ** -18)
    unit = [(0, np.array([1.0], dtype=np.float32), np.zeros(0, np.float32))]
    unit += [(i + 1, np.array([tiny], dtype=np.float32), np.zeros(0, np.float32)) for i in range(64)]
    assert orc.combine_partials(unit, 1)[0][0, 0] == np.float32(1.0)
