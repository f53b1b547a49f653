"""combine_partials through the shim (K3 on the GPU), ported from the reference's
TestCombinePartials (pkg/tests/test_backward.py:167-233).

Same coverage errors and group routing as the reference; the fold is K3's
fixed-order fp64 sum, so the absorption case shows the GPU KEEPING the 64
tiny partials that the reference's fp32 fold loses (the paper's reduced-
rounding claim on the reference's own example).
"""
import numpy as np
import pytest

from paper_2505_13813_b200 import grkan

pytestmark = pytest.mark.gpu


def test_two_partials_one_group():
    d_a, d_b = grkan.combine_partials([(0, np.array([1.0]), np.array([])), (1, np.array([2.0]), np.array([]))],
                                      num_groups=1)
    assert np.array_equal(d_a, [[3.0]])
    assert d_b.shape == (1, 0)


def test_empty_denominator_zero_columns():
    d_a, d_b = grkan.combine_partials([(0, np.array([1.0, 2.0]), np.zeros(0))], num_groups=1)
    assert np.array_equal(d_a, [[1.0, 2.0]])
    assert d_b.shape == (1, 0)


def test_group_assignment_round_robin():
    parts = [(0, np.array([1.0]), np.array([10.0])), (1, np.array([2.0]), np.array([20.0])),
             (2, np.array([4.0]), np.array([40.0])), (3, np.array([8.0]), np.array([80.0]))]
    d_a, d_b = grkan.combine_partials(parts, num_groups=2)
    assert np.array_equal(d_a, [[5.0], [10.0]])
    assert np.array_equal(d_b, [[50.0], [100.0]])


def test_ragged_last_row_block():
    # 3 partials over 2 groups: the second row block has only group 0
    parts = [(0, np.array([1.0]), np.array([1.0])), (1, np.array([2.0]), np.array([2.0])),
             (2, np.array([4.0]), np.array([4.0]))]
    d_a, d_b = grkan.combine_partials(parts, num_groups=2)
    assert np.array_equal(d_a, [[5.0], [2.0]]) and np.array_equal(d_b, [[5.0], [2.0]])


def test_absorption_kept_by_the_fp64_fold():
    tiny = np.float32(2.0 ** -24)
    parts = [(i, np.array([tiny], dtype=np.float32), np.zeros(0, np.float32)) for i in range(64)]
    d_a, _ = grkan.combine_partials(parts, num_groups=1)
    assert d_a.dtype == np.float32 and d_a[0, 0] == np.float32(2.0 ** -18)
    with_unit = [(0, np.array([1.0], dtype=np.float32), np.zeros(0, np.float32))]
    with_unit += [(i + 1, np.array([tiny], dtype=np.float32), np.zeros(0, np.float32)) for i in range(64)]
    kept, _ = grkan.combine_partials(with_unit, num_groups=1)
    # the reference's fp32 fold returns exactly 1.0 here (every tiny add absorbed)
    assert kept[0, 0] == np.float32(1.0 + 2.0 ** -18)


@pytest.mark.parametrize("parts", [
    [(0, np.array([1.0]), np.zeros(0)), (0, np.array([1.0]), np.zeros(0))],   # duplicate id
    [(0, np.array([1.0]), np.zeros(0)), (2, np.array([1.0]), np.zeros(0))],   # missing id
    [],                                                                       # no partials
    [(0, np.array([1.0]), np.zeros(0)), (1, np.array([1.0, 2.0]), np.zeros(0))],  # ragged widths
])
def test_coverage_violations(parts):
    with pytest.raises(grkan.PartialCoverageError):
        grkan.combine_partials(parts, num_groups=1)


def test_unknown_mode():
    with pytest.raises(ValueError):
        grkan.combine_partials([(0, np.array([1.0]), np.zeros(0))], num_groups=1, mode="nope")


@pytest.mark.parametrize("mode", [grkan.COMBINE_ORDERED, grkan.COMBINE_UNORDERED])
def test_input_order_does_not_change_bits(mode):
    rng = np.random.default_rng(7)
    parts = [(i, rng.standard_normal(3).astype(np.float32), rng.standard_normal(2).astype(np.float32))
             for i in range(8)]
    ref = grkan.combine_partials(parts, num_groups=2, mode=mode)
    shuffled = list(parts)
    rng.shuffle(shuffled)
    out = grkan.combine_partials(shuffled, num_groups=2, mode=mode)
    assert out[0].tobytes() == ref[0].tobytes() and out[1].tobytes() == ref[1].tobytes()
    # against an fp64 sum of the same partials, rounded once
    want_a = np.zeros((2, 3))
    for i, pa, _ in parts:
        want_a[i % 2] += pa.astype(np.float64)
    assert np.array_equal(out[0], want_a.astype(np.float32))
