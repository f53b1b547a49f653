"""Staged kernels with tensor-map stage copies (geo.tma_rows > 0: short row segments,
and the bf16 backward at any row length, boxes of up to 256-column chunks).

How a stage reaches shared memory must not change a single bit: every output
of the forward, backward, fused step and deterministic partials path is
compared bitwise between GRKAN_TMA2D=1 (2-D TMA boxes) and GRKAN_TMA2D=0 (one
bulk copy per row segment), on group widths from 16 to 256 columns and ragged
row counts whose last stage runs past the end of the tensor (zero-filled box
rows that the consumers must ignore).  Values against the oracle are covered
by the parity tests, which now run on this path at their short-row shapes.
"""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


def ops():
    from paper_2505_13813_b200 import ops as _ops
    return _ops


def _with_env(name, value, fn):
    old = os.environ.get(name)
    os.environ[name] = value
    try:
        out = fn()
        torch.cuda.synchronize()
        return out
    finally:
        if old is None:
            del os.environ[name]
        else:
            os.environ[name] = old


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("rows,d,groups", [(3001, 768, 16), (777, 3072, 64), (1000, 192, 8), (513, 1536, 8),
                                           (4099, 256, 1), (37, 128, 8), (1003, 3072, 8), (300, 1536, 1)])
def test_tensor_map_copies_are_bitwise_the_row_copies(dtype, rows, d, groups):
    g = torch.Generator(device="cpu").manual_seed(rows + d)
    x = torch.randn(rows, d, generator=g).to(dtype).to(DEV)
    u = torch.randn(rows, d, generator=g).to(dtype).to(DEV)
    a = torch.randn(groups, 6, generator=g).to(DEV)
    b = torch.randn(groups, 4, generator=g).to(DEV)
    O = ops()

    def run():
        y = O.rational_forward(x, a, b)
        dx, da, db = O.rational_backward(x, u, a, b)
        dxd, dad, dbd = O.rational_backward(x, u, a, b, deterministic=True)
        return y, dx, da, db, dxd, dad, dbd

    on = _with_env("GRKAN_TMA2D", "1", run)
    off = _with_env("GRKAN_TMA2D", "0", run)
    for k, (p, q) in enumerate(zip(on, off)):
        assert torch.equal(p, q), k
    yf = _with_env("GRKAN_TMA2D", "1", lambda: O.rational_forward_backward(x, u, a, b))
    yg = _with_env("GRKAN_TMA2D", "0", lambda: O.rational_forward_backward(x, u, a, b))
    for p, q in zip(yf, yg):
        assert torch.equal(p, q)
