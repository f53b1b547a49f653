"""The per-shape kernel variants against the oracle at sizes that select them.

make_plan picks, from the layout alone, the wide geometry (one CTA of 16
consumer warps per SM: bf16 I/O, fp32 rows >= 1536 B), the bf16 table body,
tensor-map stage copies and the staged kernels' compile-time degrees (5,4) and
(3,2).  Each combination here is checked the way the parity tests check the
default path: EXACT y/dx bitwise the reference (bf16: bf16_rn of the
reference on the rounded inputs), FAST within 1e-5 (bf16 1e-2), da/db within
1e-5 of the fp64 oracle; and checked mode raising on a non-finite input.
"""

import os

import numpy as np
import pytest
import torch

from oracle import c_oracle
from oracle import grkan_oracle as orc

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


def ops():
    from paper_2505_13813_b200 import ops as _ops
    return _ops


CASES = [
    # (B, L, D, groups, m, n), dtype: wide fp32 (1536-byte rows), wide bf16 + table,
    # wide bf16 (3,2) (no table: paper degrees only), default fp32 (768-byte rows) (3,2)
    ((24, 197, 3072, 8, 5, 4), torch.float32),
    ((24, 197, 3072, 8, 5, 4), torch.bfloat16),
    ((24, 197, 3072, 8, 3, 2), torch.bfloat16),
    ((24, 197, 1536, 8, 3, 2), torch.float32),
    ((12, 197, 3072, 64, 5, 4), torch.bfloat16),
]


@pytest.mark.parametrize("shape,dtype", CASES)
@pytest.mark.parametrize("wide", ["default", "0"])
def test_variants_against_the_oracle(shape, dtype, wide):
    B, L, D, ng, m, n = shape
    rng = np.random.default_rng(B + D + m)
    x = rng.standard_normal((B, L, D)).astype(np.float32)
    u = rng.standard_normal((B, L, D)).astype(np.float32)
    num = rng.standard_normal((ng, m + 1))
    den = rng.standard_normal((ng, n))
    xt = torch.from_numpy(x).to(dtype)
    ut = torch.from_numpy(u).to(dtype)
    xr, ur = xt.float().numpy(), ut.float().numpy()
    a = torch.from_numpy(num.astype(np.float32)).to(DEV)
    b = torch.from_numpy(den.astype(np.float32)).to(DEV)
    old = os.environ.get("GRKAN_WIDE")
    if wide != "default":
        os.environ["GRKAN_WIDE"] = wide
    try:
        xd, ud = xt.to(DEV), ut.to(DEV)
        r = c_oracle.backward(xr, ur, num, den, 256)
        y_ref = c_oracle.forward(xr, num, den)
        dx, da, db = ops().rational_backward(xd, ud, a, b, exact=True, check_overflow=True)
        y = ops().rational_forward(xd, a, b, exact=True)
        if dtype == torch.float32:
            assert np.array_equal(dx.cpu().numpy().view(np.uint32), r["dx"].view(np.uint32))
            assert np.array_equal(y.cpu().numpy().view(np.uint32), y_ref.view(np.uint32))
        else:
            assert torch.equal(dx.cpu(), torch.from_numpy(r["dx"]).bfloat16())
            assert torch.equal(y.cpu(), torch.from_numpy(y_ref).bfloat16())
        dxf, daf, dbf = ops().rational_backward(xd, ud, a, b, check_overflow=True)
        tol = 1e-5 if dtype == torch.float32 else 1e-2
        assert orc.matrix_rel(dxf.float().cpu().numpy(), r["dx"]) <= tol
        for ga, gb in ((da, db), (daf, dbf)):
            assert orc.matrix_rel(ga.cpu().numpy(), r["true64_da"]) <= 1e-5
            assert orc.matrix_rel(gb.cpu().numpy(), r["true64_db"]) <= 1e-5
        # checked mode flags a non-finite input on every variant
        from paper_2505_13813_b200.errors import NonFiniteInputError
        xbad = xd.clone()
        xbad[B // 2, L // 2, D // 3] = float("nan")
        with pytest.raises(NonFiniteInputError):
            ops().rational_backward(xbad, ud, a, b, check_finite=True)
    finally:
        if wide != "default":
            if old is None:
                del os.environ["GRKAN_WIDE"]
            else:
                os.environ["GRKAN_WIDE"] = old
