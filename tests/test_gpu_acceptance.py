"""The reference's acceptance criteria that concern the hot path, run through the GPU shim
(pkg/tests/test_acceptance.py).

  2  strategy equivalence: random small instances (verification.py:447-469) vs the
     fp64 oracle <= 1e-12 in double precision; dx bitwise across strategies in f32 and f64
  8  determinism: 5 runs x {f32, f64} bitwise identical (test_acceptance.py:232-252)
  4  rounding: covered by tests/test_gpu_rounding.py (desk preset, 20 passes)
"""

import numpy as np
import pytest

from oracle import grkan_oracle as orc

pytestmark = pytest.mark.gpu


def G():
    from paper_2505_13813_b200 import grkan
    return grkan


def random_small_instance(rng):
    """verification.py:447-459 (without the layer)."""
    g = G()
    batch = int(rng.integers(1, 5))
    seq = int(rng.integers(1, 5))
    n_g = int(rng.choice([1, 2, 4]))
    d_g = int(rng.integers(1, 16 // n_g + 1))
    layout = g.GroupLayout(n_g * d_g, n_g)
    params = g.GroupRationalParams(rng.standard_normal((n_g, 6)), rng.standard_normal((n_g, 4)))
    x = g.ActivationTensor(rng.standard_normal((batch, seq, n_g * d_g)))
    up = g.ActivationTensor(rng.standard_normal((batch, seq, n_g * d_g)))
    return x, up, params, layout


def test_criterion_2_strategy_equivalence():
    g = G()
    rng = np.random.default_rng(12)
    worst = 0.0
    for _ in range(20):
        x, up, params, layout = random_small_instance(rng)
        block = int(rng.choice([1, 2, 3, 4, 8]))
        plan = g.ExecutionPlan.blocked(x.batch, x.seq, layout, block)
        dx64, da64, db64 = orc.true64_grads(x.data, up.data, params.numerator, params.denominator)
        naive = g.backward_naive(x, up, params)
        blocked = g.backward_blocked(x, up, params, plan)
        rel = max(orc.matrix_rel(naive.d_a, da64), orc.matrix_rel(naive.d_b, db64),
                  orc.matrix_rel(blocked.d_a, da64), orc.matrix_rel(blocked.d_b, db64),
                  orc.matrix_rel(naive.d_x.data, dx64))
        worst = max(worst, rel)
        assert rel <= 1e-12
        assert naive.d_x.data.tobytes() == blocked.d_x.data.tobytes()
        x32 = g.ActivationTensor(x.data.astype(np.float32))
        up32 = g.ActivationTensor(up.data.astype(np.float32))
        assert (g.backward_naive(x32, up32, params).d_x.data.tobytes()
                == g.backward_blocked(x32, up32, params, plan).d_x.data.tobytes())
    print("ACCEPTANCE 2 strategy equivalence PASS (max rel err vs fp64 %.2e)" % worst)


@pytest.mark.parametrize("exact", [True, False])
def test_criterion_8_determinism(exact):
    g = G()
    rng = np.random.default_rng(808)
    layout = g.GroupLayout(64, 8)
    params = g.GroupRationalParams(rng.standard_normal((8, 6)), rng.standard_normal((8, 4)))
    for dtype in (np.float32, np.float64):
        x = g.ActivationTensor(rng.standard_normal((8, 16, 64)).astype(dtype))
        up = g.ActivationTensor(rng.standard_normal((8, 16, 64)).astype(dtype))
        plan = g.ExecutionPlan.blocked(8, 16, layout, 16)
        sigs = set()
        for workers in (1, 4, 16):
            for _ in range(5):
                b = g.backward_blocked(x, up, params, plan, workers=workers, exact=exact)
                sigs.add((b.d_a.tobytes(), b.d_b.tobytes(), b.d_x.data.tobytes()))
        assert len(sigs) == 1
