"""The native host-array pipeline (grkan_host_*, include/grkan_b200.h): the reference's
forward_tensor / backward_blocked calling convention (host arrays in and out,
pkg/src/grkan/rational.py:325-345, backward.py:275-372) with host copies, PCIe and
kernels overlapped.  Small staging chunks force many chunks, ragged tails and slot
reuse at oracle-sized inputs."""

import ctypes
import threading

import numpy as np
import pytest
import torch

from oracle import c_oracle
from oracle import grkan_oracle as orc

pytestmark = pytest.mark.gpu


def N():
    from paper_2505_13813_b200 import _native
    return _native


class Ctx:
    def __init__(self, chunk_bytes=0, threads=0):
        self.h = ctypes.c_void_p()
        rc = N().lib().grkan_host_create(0, chunk_bytes, threads, ctypes.byref(self.h))
        assert rc == 0, N().lib().grkan_host_last_error()

    def close(self):
        N().lib().grkan_host_destroy(self.h)

    def fwd(self, x, num, den, flags):
        y = np.empty_like(x)
        rows, d = x.shape[0] * x.shape[1], x.shape[2]
        dt = N().DT_F64 if x.dtype == np.float64 else N().DT_F32
        a = np.ascontiguousarray(num, dtype=x.dtype)
        b = np.ascontiguousarray(den, dtype=x.dtype)
        rc = N().lib().grkan_host_fwd(self.h, x.ctypes.data, y.ctypes.data, a.ctypes.data, b.ctypes.data, rows,
                                      d, a.shape[0], a.shape[1], b.shape[1], dt, flags)
        return rc, y

    def bwd(self, x, u, num, den, flags):
        dx = np.empty_like(x)
        rows, d = x.shape[0] * x.shape[1], x.shape[2]
        dt = N().DT_F64 if x.dtype == np.float64 else N().DT_F32
        a = np.ascontiguousarray(num, dtype=x.dtype)
        b = np.ascontiguousarray(den, dtype=x.dtype)
        da = np.empty(a.shape, dtype=x.dtype)
        db = np.empty(b.shape, dtype=x.dtype)
        rc = N().lib().grkan_host_bwd(self.h, x.ctypes.data, u.ctypes.data, a.ctypes.data, b.ctypes.data,
                                      dx.ctypes.data, da.ctypes.data, db.ctypes.data, rows, d, a.shape[0],
                                      a.shape[1], b.shape[1], dt, flags)
        return rc, dx, da, db


def device_det(x, u, num, den):
    """grkan_bwd(..., DETERMINISTIC) on the whole tensor, on the device."""
    from paper_2505_13813_b200 import ops
    cd = torch.float64 if x.dtype == np.float64 else torch.float32
    a = torch.from_numpy(num).to(cd).cuda()
    b = torch.from_numpy(den).to(cd).cuda()
    dx, da, db = ops.rational_backward(torch.from_numpy(x).cuda(), torch.from_numpy(u).cuda(), a, b, exact=True,
                                       deterministic=True)
    return dx.cpu().numpy(), da.cpu().numpy(), db.cpu().numpy()


@pytest.mark.parametrize("shape,groups", [((8, 197, 192), 8), ((3, 101, 384), 8), ((2, 77, 64), 1)])
@pytest.mark.parametrize("chunk", [64 << 10, 200 << 10])
def test_forward_exact_bitwise_many_chunks(shape, groups, chunk):
    x, _, num, den = orc.bench_inputs(*shape, groups, seed=11)
    ctx = Ctx(chunk_bytes=chunk, threads=4)
    try:
        rc, y = ctx.fwd(x, num, den, N().FLAG_EXACT)
        assert rc == 0
        assert np.array_equal(y.view(np.uint32), orc.forward(x, num, den).view(np.uint32))
        rc, yf = ctx.fwd(x, num, den, N().FLAG_FAST)
        assert rc == 0 and orc.matrix_rel(yf, orc.forward(x, num, den)) <= 1e-5
    finally:
        ctx.close()


@pytest.mark.parametrize("chunk", [96 << 10, 1 << 20])
def test_backward_exact_bitwise_and_chunk_invariant(chunk):
    """dx bitwise vs the reference restatement; da/db bitwise equal to the deterministic
    device fold on the whole tensor (so independent of the chunk size), and within
    1e-5 of the fp64 oracle."""
    x, u, num, den = orc.bench_inputs(8, 197, 192, 8, seed=12)
    ctx = Ctx(chunk_bytes=chunk, threads=3)
    try:
        rc, dx, da, db = ctx.bwd(x, u, num, den, N().FLAG_EXACT)
    finally:
        ctx.close()
    assert rc == 0
    r = c_oracle.backward(x, u, num, den, 256)
    assert np.array_equal(dx.view(np.uint32), r["dx"].view(np.uint32))
    _, da_d, db_d = device_det(x, u, num, den)
    assert da.tobytes() == da_d.tobytes() and db.tobytes() == db_d.tobytes()
    _, da64, db64 = orc.true64_grads(x, u, num.astype(np.float32).astype(np.float64),
                                     den.astype(np.float32).astype(np.float64))
    assert orc.matrix_rel(da, da64) <= 1e-5 and orc.matrix_rel(db, db64) <= 1e-5


def test_fp64_tensors():
    x, u, num, den = orc.bench_inputs(4, 150, 64, 4, seed=13, dtype=np.float64)
    ctx = Ctx(chunk_bytes=32 << 10, threads=2)
    try:
        rc, y = ctx.fwd(x, num, den, N().FLAG_EXACT)
        assert rc == 0 and np.array_equal(y, orc.forward(x, num, den))
        rc, dx, da, db = ctx.bwd(x, u, num, den, N().FLAG_EXACT)
        assert rc == 0
    finally:
        ctx.close()
    rdx, rda, rdb = orc.backward_blocked(x, u, num, den)
    assert np.array_equal(dx, rdx)
    assert orc.matrix_rel(da, rda) <= 1e-12 and orc.matrix_rel(db, rdb) <= 1e-12


def test_errors_map_to_the_reference_classes():
    x, u, num, den = orc.bench_inputs(4, 250, 64, 8, seed=14)
    ctx = Ctx(chunk_bytes=16 << 10, threads=2)  # grown to one 384-row block: 3 chunks
    try:
        bad = x.copy()
        bad[3, 249, 63] = np.nan  # in the last chunk
        rc, _ = ctx.fwd(bad, num, den, N().FLAG_CHECK_FINITE)
        assert rc == N().ERR_NONFINITE_INPUT
        rc, *_ = ctx.bwd(x, bad, num, den, N().FLAG_CHECK_FINITE)
        assert rc == N().ERR_NONFINITE_INPUT
        rc, _ = ctx.fwd(bad, num, den, N().FLAG_FAST)  # unchecked: runs
        assert rc == 0
        # x = 1e30, n = 0: the fp32 power terms overflow (pkg/tests/test_backward.py:59-65)
        big = np.full((1, 3, 8), 1e30, dtype=np.float32)
        rc, *_ = ctx.bwd(big, np.ones_like(big), np.ones((1, 6)), np.zeros((1, 0)), N().FLAG_EXACT)
        assert rc == N().ERR_ACCUM_OVERFLOW
        rc, _ = ctx.fwd(x[:, :, :60].copy(), num, den, 0)  # 60 % 8 != 0
        assert rc == N().ERR_LAYOUT
        # the context is still usable after errors
        rc, y = ctx.fwd(x, num, den, N().FLAG_EXACT)
        assert rc == 0 and np.array_equal(y, orc.forward(x, num, den))
    finally:
        ctx.close()


def test_empty_rows():
    ctx = Ctx(chunk_bytes=16 << 10, threads=2)
    try:
        x = np.zeros((0, 5, 16), dtype=np.float32)
        rc, y = ctx.fwd(x, np.ones((2, 6)), np.ones((2, 4)), 0)
        assert rc == 0 and y.shape == x.shape
        rc, dx, da, db = ctx.bwd(x, x, np.ones((2, 6)), np.ones((2, 4)), 0)
        assert rc == 0 and not da.any() and not db.any()
    finally:
        ctx.close()


def test_back_to_back_calls_with_different_inputs():
    """No slot is overwritten before the previous call's kernels and copies are done."""
    ctx = Ctx(chunk_bytes=64 << 10, threads=4)
    try:
        ins = [orc.bench_inputs(4, 197, 192, 8, seed=30 + i) for i in range(3)]
        outs = [ctx.bwd(x, u, num, den, N().FLAG_EXACT) for x, u, num, den in ins]
        for (x, u, num, den), (rc, dx, _, _) in zip(ins, outs):
            assert rc == 0
            assert np.array_equal(dx.view(np.uint32), c_oracle.backward(x, u, num, den, 256)["dx"].view(np.uint32))
    finally:
        ctx.close()


def test_shim_threads_each_get_their_own_pipeline():
    """The reference's functions are safe from concurrent callers."""
    from paper_2505_13813_b200 import grkan as G
    rng = np.random.default_rng(40)
    params = G.GroupRationalParams(rng.standard_normal((8, 6)), rng.standard_normal((8, 4)))
    layout = G.GroupLayout(192, 8)
    xs = [G.ActivationTensor(rng.standard_normal((8, 197, 192)).astype(np.float32)) for _ in range(4)]
    want = [orc.forward(x.data, params.numerator, params.denominator) for x in xs]
    got = [None] * 4

    def work(i):
        got[i] = G.forward_tensor(xs[i], params, layout).data

    ts = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for g, w in zip(got, want):
        assert np.array_equal(g.view(np.uint32), w.view(np.uint32))


def test_page_locked_buffers_are_transferred_in_place():
    """Pinned x / dy / y / dx (torch pinned tensors behind NumPy arrays) skip the staging
    copies; results are bitwise the pageable path's, in every in/out combination."""
    x, u, num, den = orc.bench_inputs(4, 197, 192, 8, seed=50)
    ctx = Ctx(chunk_bytes=128 << 10, threads=4)
    try:
        rc, y_ref = ctx.fwd(x, num, den, N().FLAG_EXACT)
        rc2, dx_ref, da_ref, db_ref = ctx.bwd(x, u, num, den, N().FLAG_EXACT)
        assert rc == 0 and rc2 == 0
        px = torch.from_numpy(x).pin_memory().numpy()
        pu = torch.from_numpy(u).pin_memory().numpy()
        for xin, uin in ((px, pu), (px, u), (x, pu)):
            for pinned_out in (False, True):
                out = torch.empty(x.shape, pin_memory=True).numpy() if pinned_out else np.empty_like(x)
                a = np.ascontiguousarray(num, dtype=np.float32)
                b = np.ascontiguousarray(den, dtype=np.float32)
                rows, d = x.shape[0] * x.shape[1], x.shape[2]
                assert N().lib().grkan_host_fwd(ctx.h, xin.ctypes.data, out.ctypes.data, a.ctypes.data,
                                                b.ctypes.data, rows, d, 8, 6, 4, N().DT_F32, N().FLAG_EXACT) == 0
                assert out.tobytes() == y_ref.tobytes()
                da = np.empty((8, 6), np.float32)
                db = np.empty((8, 4), np.float32)
                assert N().lib().grkan_host_bwd(ctx.h, xin.ctypes.data, uin.ctypes.data, a.ctypes.data,
                                                b.ctypes.data, out.ctypes.data, da.ctypes.data, db.ctypes.data,
                                                rows, d, 8, 6, 4, N().DT_F32, N().FLAG_EXACT) == 0
                assert out.tobytes() == dx_ref.tobytes()
                assert da.tobytes() == da_ref.tobytes() and db.tobytes() == db_ref.tobytes()
    finally:
        ctx.close()


def test_shim_outputs_are_independent_arrays():
    """Large shim outputs come from the pinned caching allocator: results held at the same
    time never alias, and a dropped output's memory is safely reused."""
    from paper_2505_13813_b200 import grkan as G
    rng = np.random.default_rng(60)
    params = G.GroupRationalParams(rng.standard_normal((8, 6)), rng.standard_normal((8, 4)))
    layout = G.GroupLayout(384, 8)
    xs = [G.ActivationTensor(rng.standard_normal((4, 197, 384)).astype(np.float32)) for _ in range(3)]
    ys = [G.forward_tensor(x, params, layout).data for x in xs]
    assert len({y.ctypes.data for y in ys}) == 3
    for x, y in zip(xs, ys):
        assert y.flags.c_contiguous and y.flags.writeable and y.dtype == np.float32
        assert np.array_equal(y.view(np.uint32), orc.forward(x.data, params.numerator, params.denominator).view(np.uint32))
    del ys
    again = G.forward_tensor(xs[0], params, layout).data
    assert np.array_equal(again.view(np.uint32),
                          orc.forward(xs[0].data, params.numerator, params.denominator).view(np.uint32))
