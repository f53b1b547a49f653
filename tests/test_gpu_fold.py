"""K3 folded into the staged K2 (grkan_staged.cuh fold_if_last; opt-in, GRKAN_FOLD=1 --
measured slower than the PDL-launched K3): da/db bitwise those of k_bwd_reduce (the reference's combine in a
fixed order, backward.py:142-184), dx unchanged, with reused, garbage-filled and
graph-replayed workspaces (the arrival counters live in the workspace header)."""

import os

import pytest
import torch

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


def _inputs(rows, d, ng, m1, n, dtype, seed):
    g = torch.Generator(device=DEV).manual_seed(seed)
    x = torch.randn(rows, d, device=DEV, generator=g).to(dtype)
    dy = torch.randn(rows, d, device=DEV, generator=g).to(dtype)
    a = torch.randn(ng, m1, device=DEV, generator=g) * 0.3
    b = torch.randn(ng, n, device=DEV, generator=g) * 0.3
    return x, dy, a, b


def _bwd(x, dy, a, b, fold, ws=None, exact=False):
    from paper_2505_13813_b200 import ops
    old = os.environ.get("GRKAN_FOLD")
    os.environ["GRKAN_FOLD"] = "1" if fold else "0"
    try:
        out = ops.rational_backward(x, dy, a, b, exact=exact, check_overflow=True, workspace=ws)
        torch.cuda.synchronize()
        return out
    finally:
        if old is None:
            del os.environ["GRKAN_FOLD"]
        else:
            os.environ["GRKAN_FOLD"] = old


CASES = [  # rows, d, groups, (m1, n), dtype -- default / wide geometry, table, (3,2), 30 groups, 31 (K3)
    (4 * 197, 768, 8, (6, 4), torch.float32),
    (16 * 197, 3072, 8, (6, 4), torch.float32),
    (16 * 197, 3072, 8, (6, 4), torch.bfloat16),
    (8 * 197, 1536, 8, (4, 2), torch.float32),
    (2 * 197, 1920, 30, (6, 4), torch.bfloat16),
    (2 * 197, 1984, 31, (6, 4), torch.float32),
    (1, 768, 8, (6, 4), torch.float32),
]


@pytest.mark.parametrize("rows,d,ng,deg,dtype", CASES)
@pytest.mark.parametrize("exact", [False, True])
def test_fold_matches_k3_bitwise(rows, d, ng, deg, dtype, exact):
    x, dy, a, b = _inputs(rows, d, ng, deg[0], deg[1], dtype, seed=rows + d + ng)
    dx0, da0, db0 = _bwd(x, dy, a, b, fold=False, exact=exact)
    dx1, da1, db1 = _bwd(x, dy, a, b, fold=True, exact=exact)
    assert torch.equal(dx0, dx1)
    assert torch.equal(da0, da1) and torch.equal(db0, db1)


def test_fold_with_reused_and_garbage_workspace():
    from paper_2505_13813_b200 import ops
    rows, d, ng = 32 * 197, 1536, 8
    x, dy, a, b = _inputs(rows, d, ng, 6, 4, torch.float32, seed=11)
    ref = _bwd(x, dy, a, b, fold=False)
    nbytes = ops.workspace_bytes(rows, d, ng, 6, 4, torch.float32)
    ws = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=DEV)  # never-zeroed header
    os.environ["GRKAN_FOLD"] = "1"
    try:
        for _ in range(4):  # back to back, no host sync in between
            out = ops.rational_backward(x, dy, a, b, workspace=ws)
        torch.cuda.synchronize()
    finally:
        del os.environ["GRKAN_FOLD"]
    for r, o in zip(ref, out):
        assert torch.equal(r, o)
    ws.fill_(0xff)
    out = _bwd(x, dy, a, b, fold=True, ws=ws)
    for r, o in zip(ref, out):
        assert torch.equal(r, o)


def test_fold_graph_replays():
    from paper_2505_13813_b200 import ops
    rows, d, ng = 16 * 197, 768, 8
    x, dy, a, b = _inputs(rows, d, ng, 6, 4, torch.float32, seed=5)
    ref = _bwd(x, dy, a, b, fold=False)
    ws = torch.empty(ops.workspace_bytes(rows, d, ng, 6, 4, torch.float32), dtype=torch.uint8, device=DEV)
    os.environ["GRKAN_FOLD"] = "1"  # read when the call is planned, i.e. at capture
    try:
        _capture_and_replay(ops, x, dy, a, b, ws, ref)
    finally:
        del os.environ["GRKAN_FOLD"]


def _capture_and_replay(ops, x, dy, a, b, ws, ref):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ops.rational_backward(x, dy, a, b, workspace=ws)
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        out = ops.rational_backward(x, dy, a, b, workspace=ws)
    for _ in range(3):  # the same sequence number every replay: the last CTA resets the counters
        for t in out:
            t.zero_()
        graph.replay()
        torch.cuda.synchronize()
        for r, o in zip(ref, out):
            assert torch.equal(r, o)


def test_fold_overflow_flag():
    from paper_2505_13813_b200.errors import AccumulationOverflowError
    x, dy, a, b = _inputs(8 * 197, 768, 8, 6, 4, torch.float32, seed=3)
    dy = dy * 3e37  # fp32 coefficient partials overflow to inf
    with pytest.raises(AccumulationOverflowError):
        _bwd(x, dy, a, b, fold=True)
