"""The fused forward + backward step (grkan_fwd_bwd / ops.rational_forward_backward):
forward_tensor and backward_blocked of the same x in one pass must give what the two
passes give -- EXACT y and dx bitwise the reference's (rational.py:218-278), da/db the
same fold as rational_backward's -- in every kernel family (the fused staged kernel, and
the two-pass fallback for other plans)."""

import numpy as np
import pytest
import torch

from oracle import c_oracle
from oracle import grkan_oracle as orc

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


def ops():
    from paper_2505_13813_b200 import ops as o
    return o


@pytest.mark.parametrize("shape,groups", [((8, 197, 192), 8), ((4, 197, 768), 8), ((2, 33, 64), 1)])
def test_exact_bitwise_against_the_reference_restatement(shape, groups):
    x, u, num, den = orc.bench_inputs(*shape, groups, seed=70)
    a = torch.from_numpy(num.astype(np.float32)).to(DEV)
    b = torch.from_numpy(den.astype(np.float32)).to(DEV)
    y, dx, da, db = ops().rational_forward_backward(torch.from_numpy(x).to(DEV), torch.from_numpy(u).to(DEV),
                                                    a, b, exact=True, check_overflow=True)
    assert np.array_equal(y.cpu().numpy().view(np.uint32), orc.forward(x, num, den).view(np.uint32))
    r = c_oracle.backward(x, u, num, den, 256)
    assert np.array_equal(dx.cpu().numpy().view(np.uint32), r["dx"].view(np.uint32))
    _, da64, db64 = orc.true64_grads(x, u, num.astype(np.float32).astype(np.float64),
                                     den.astype(np.float32).astype(np.float64))
    assert orc.matrix_rel(da.cpu().numpy(), da64) <= 1e-5 and orc.matrix_rel(db.cpu().numpy(), db64) <= 1e-5


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float64])
@pytest.mark.parametrize("exact", [False, True])
def test_same_results_as_the_two_passes(dtype, exact):
    """dx / da / db bitwise those of rational_backward (the same K2 accumulation, the same
    K3 fold) -- except bf16 FAST, where rational_backward takes the x-factor table body
    (terms rounded differently; the fused step has no table variant): within the FAST
    tolerances there; y bitwise rational_forward's in EXACT mode, within 1e-5 (bf16:
    one ulp of the output) in FAST mode (pq vs K1's P * rcp(Q) of a differently
    evaluated A)."""
    g = torch.Generator(device="cpu").manual_seed(71)
    x = torch.randn(16, 197, 384, generator=g).to(dtype).to(DEV)
    u = torch.randn(16, 197, 384, generator=g).to(dtype).to(DEV)
    cd = torch.float64 if dtype == torch.float64 else torch.float32
    a = torch.randn(8, 6, generator=g).to(cd).to(DEV)
    b = torch.randn(8, 4, generator=g).to(cd).to(DEV)
    y, dx, da, db = ops().rational_forward_backward(x, u, a, b, exact=exact)
    y2 = ops().rational_forward(x, a, b, exact=exact)
    dx2, da2, db2 = ops().rational_backward(x, u, a, b, exact=exact)
    if dtype == torch.bfloat16 and not exact:
        assert orc.matrix_rel(dx.double().cpu().numpy(), dx2.double().cpu().numpy()) <= 1e-2
        assert orc.matrix_rel(da.double().cpu().numpy(), da2.double().cpu().numpy()) <= 1e-5
        assert orc.matrix_rel(db.double().cpu().numpy(), db2.double().cpu().numpy()) <= 1e-5
    else:
        assert torch.equal(dx, dx2) and torch.equal(da, da2) and torch.equal(db, db2)
    if exact:
        assert torch.equal(y, y2)
    else:
        tol = 1e-2 if dtype == torch.bfloat16 else 1e-5
        assert orc.matrix_rel(y.double().cpu().numpy(), y2.double().cpu().numpy()) <= tol


@pytest.mark.parametrize("m1,n,dim,groups", [(4, 2, 384, 8), (6, 4, 12, 4), (8, 5, 64, 2)])
def test_fallback_plans_match_the_two_passes(m1, n, dim, groups):
    """Plans without the fused kernel (other degrees, d_g not a vector multiple) run the
    two passes back to back inside grkan_fwd_bwd."""
    g = torch.Generator(device="cpu").manual_seed(72)
    x = torch.randn(5, 37, dim, generator=g).to(DEV)
    u = torch.randn(5, 37, dim, generator=g).to(DEV)
    a = torch.randn(groups, m1, generator=g).to(DEV)
    b = torch.randn(groups, n, generator=g).to(DEV)
    y, dx, da, db = ops().rational_forward_backward(x, u, a, b, exact=True)
    assert torch.equal(y, ops().rational_forward(x, a, b, exact=True))
    dx2, da2, db2 = ops().rational_backward(x, u, a, b, exact=True)
    assert torch.equal(dx, dx2) and torch.equal(da, da2) and torch.equal(db, db2)


def test_checked_mode_and_overflow():
    from paper_2505_13813_b200 import errors
    x = torch.randn(4, 64, 384, device=DEV)
    u = torch.randn(4, 64, 384, device=DEV)
    a, b = torch.randn(8, 6, device=DEV), torch.randn(8, 4, device=DEV)
    x[3, 63, 383] = float("nan")
    with pytest.raises(errors.NonFiniteInputError):
        ops().rational_forward_backward(x, u, a, b, check_finite=True)
    big = torch.full((1, 128, 8), 1e30, device=DEV)
    with pytest.raises(errors.AccumulationOverflowError):
        ops().rational_forward_backward(big, torch.ones_like(big), torch.ones(1, 6, device=DEV),
                                        torch.zeros(1, 4, device=DEV), exact=True, check_overflow=True)
