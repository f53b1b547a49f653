"""Deterministic mode: da/db bitwise independent of how rows are sharded.

SURVEY.md section 8e: with partials keyed by global row block and folded in
global block order, 1/2/3/4/8-way block-aligned shardings (emulated here in one
process: shard views -> grkan_bwd_partials -> rank-order concatenation, i.e.
what parallel.gather_blocks' all-gather produces -> grkan_reduce_partials) give
the same bits as grkan_bwd(..., GRKAN_FLAG_DETERMINISTIC) on the whole tensor.
The multi-GPU analogue of the reference's worker-count invariance
(pkg/tests/test_acceptance.py:232-252, test_backward.py:128-138).
"""

import numpy as np
import pytest
import torch

from oracle import grkan_oracle as orc

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


def _inputs(B, L, D, ng, m, n, dtype, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((B, L, D)).astype(np.float32)
    u = rng.standard_normal((B, L, D)).astype(np.float32)
    a = rng.standard_normal((ng, m + 1)).astype(np.float32)
    b = rng.standard_normal((ng, n)).astype(np.float32)
    xt = torch.from_numpy(x).to(DEV).to(dtype)
    ut = torch.from_numpy(u).to(DEV).to(dtype)
    return xt, ut, torch.from_numpy(a).to(DEV), torch.from_numpy(b).to(DEV)


CASES = [
    # name, (B, L, D, groups, m, n), dtype
    ("kat-t-fp32", (8, 197, 192, 8, 5, 4), torch.float32),
    ("kat-t-bf16", (8, 197, 192, 8, 5, 4), torch.bfloat16),
    ("kat-s-fp32", (16, 197, 1536, 8, 5, 4), torch.float32),
    ("tail-bf16", (3, 67, 384, 4, 5, 4), torch.bfloat16),
    ("generic-degree", (4, 100, 256, 4, 3, 2), torch.float32),
    # bf16 FAST at a size where the whole tensor takes the x-factor table by the
    # row-run heuristic but the 8-way shards would not: the table choice must
    # not depend on the shard
    ("kat-b-bf16-table", (64, 197, 3072, 8, 5, 4), torch.bfloat16),
]


@pytest.mark.parametrize("name,shape,dtype", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("exact", [False, True])
def test_world_size_invariance(name, shape, dtype, exact):
    from paper_2505_13813_b200 import ops, parallel
    B, L, D, ng, m, n = shape
    x, u, a, b = _inputs(B, L, D, ng, m, n, dtype, seed=11)
    rows = B * L
    x2, u2 = x.reshape(rows, D), u.reshape(rows, D)
    rb = ops.det_block_rows(D, ng, dtype)
    dx_ref, da_ref, db_ref = ops.rational_backward(x, u, a, b, exact=exact, deterministic=True)
    dx_plain, _, _ = ops.rational_backward(x, u, a, b, exact=exact)
    assert torch.equal(dx_ref, dx_plain)  # deterministic mode leaves dx alone
    for world in (1, 2, 3, 4, 8):
        counts = parallel.block_counts(rows, world, rb)
        parts, dxs = [], []
        for r in range(world):
            lo, hi = parallel.block_shard(rows, world, r, rb)
            if hi == lo:
                parts.append(torch.empty((0, ng, m + 1 + n), dtype=a.dtype, device=DEV))
                continue
            dxr, pr = ops.backward_partials(x2[lo:hi], u2[lo:hi], a, b, exact=exact)
            assert pr.shape[0] == counts[r]
            parts.append(pr)
            dxs.append(dxr)
        full = torch.cat(parts, 0).contiguous()
        da, db = ops.reduce_partials(full, m + 1, n, check_overflow=True)
        assert torch.equal(da, da_ref) and torch.equal(db, db_ref), (name, world)
        assert torch.equal(torch.cat(dxs, 0), dx_ref.reshape(rows, D))
    # and the deterministic gradients are as accurate as the default path
    xn = x.float().cpu().numpy().astype(np.float64)
    un = u.float().cpu().numpy().astype(np.float64)
    _, da64, db64 = orc.true64_grads(xn, un, a.double().cpu().numpy(), b.double().cpu().numpy())
    assert orc.matrix_rel(da_ref.double().cpu().numpy(), da64) <= 1e-5
    assert orc.matrix_rel(db_ref.double().cpu().numpy(), db64) <= 1e-5


def test_partials_api_errors():
    from paper_2505_13813_b200 import ops
    from paper_2505_13813_b200.errors import LayoutMismatchError
    x, u, a, b = _inputs(2, 10, 64, 4, 5, 4, torch.float32, seed=1)
    with pytest.raises(ValueError):
        ops.backward_partials(x, u, a, b, part_out=torch.empty((2, 4, 10), device=DEV))
    with pytest.raises(LayoutMismatchError):
        ops.reduce_partials(torch.zeros((3, 4, 9), device=DEV), 6, 4)
    da, db = ops.reduce_partials(torch.zeros((0, 4, 10), device=DEV), 6, 4)
    assert float(da.abs().sum()) == 0.0 and float(db.abs().sum()) == 0.0
