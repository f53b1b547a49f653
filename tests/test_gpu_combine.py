"""combine_partials through the shim (grkan_combine_partials on the GPU), ported from
the reference's TestCombinePartials (pkg/tests/test_backward.py:167-233).

Same coverage errors, group routing and fold as the reference: ``d_a[g] += pa`` in
the partials' dtype in fold order, so results are bitwise the reference's --
including the absorption case, where the fp32 fold loses the 64 tiny partials.
(K3, the backward's own reduction, folds in fp64 and keeps them; see
test_gpu_rounding.py for that claim.)
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


def test_absorption_versus_fresh_accumulator():
    """pkg/tests/test_backward.py:193-209, bit for bit."""
    tiny = np.float32(2.0 ** -24)
    parts = [(i, np.array([tiny], dtype=np.float32), np.zeros(0, np.float32)) for i in range(64)]
    d_a, _ = grkan.combine_partials(parts, num_groups=1)
    assert d_a.dtype == np.float32 and d_a[0, 0] == np.float32(2.0 ** -18)
    with_unit = [(0, np.array([1.0], dtype=np.float32), np.zeros(0, np.float32))]
    with_unit += [(i + 1, np.array([tiny], dtype=np.float32), np.zeros(0, np.float32)) for i in range(64)]
    absorbed, _ = grkan.combine_partials(with_unit, num_groups=1)
    assert absorbed[0, 0] == np.float32(1.0)  # every tiny add was lost, as in the reference


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


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("mode", [grkan.COMBINE_ORDERED, grkan.COMBINE_UNORDERED])
def test_bitwise_the_reference_fold(mode, dtype):
    """Random partials in shuffled submission order: bitwise the reference's fold
    (ascending ids for deterministic_ordered, the given order for unordered_scatter)."""
    from oracle import grkan_oracle as orc
    rng = np.random.default_rng(7)
    parts = [(i, (rng.standard_normal(3) * 10.0 ** rng.integers(-6, 6)).astype(dtype),
              rng.standard_normal(2).astype(dtype)) for i in range(40)]
    rng.shuffle(parts)
    got = grkan.combine_partials(parts, num_groups=4, mode=mode)
    want = orc.combine_partials(parts, 4, ordered=(mode == grkan.COMBINE_ORDERED))
    assert got[0].dtype == dtype
    assert got[0].tobytes() == want[0].tobytes() and got[1].tobytes() == want[1].tobytes()
    if mode == grkan.COMBINE_ORDERED:  # submission order does not matter
        again = grkan.combine_partials(list(reversed(parts)), num_groups=4, mode=mode)
        assert again[0].tobytes() == got[0].tobytes()
