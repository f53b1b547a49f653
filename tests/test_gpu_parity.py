"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle and the golden fixtures.

Tolerances:
  * EXACT policy: y and dx bitwise equal to the reference (golden hashes);
    da/db within 1e-6 (fp32) / 1e-12 (fp64) max-scaled of the fp64 fold of
    the *same* run-precision terms (the terms are bitwise the reference's).
  * FAST policy: y, dx max-scaled <= 1e-5 vs the reference fp32 run;
    da/db max-scaled <= 1e-5 vs the true-fp64 oracle.
  * bf16 I/O: EXACT gives bitwise bf16_rn(reference fp32 on the bf16-rounded
    inputs); FAST within 1e-2 max-scaled.
"""

import numpy as np
import pytest
import torch

from grkan_testutil import sha
from oracle import c_oracle
from oracle import grkan_oracle as orc

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


def ops():
    from paper_2505_13813_b200 import ops as _ops
    return _ops


def to_dev(arr):
    return torch.from_numpy(np.ascontiguousarray(arr)).to(DEV)


def coeffs(num, den, dtype):
    cd = np.float64 if dtype == np.float64 else np.float32
    return to_dev(np.asarray(num).astype(cd)), to_dev(np.asarray(den).astype(cd).reshape(num.shape[0], -1))


def run_cases(golden):
    for case, meta in golden.cases.items():
        yield case, meta, golden.inputs(case)


def test_native_library_is_the_in_tree_build():
    from paper_2505_13813_b200 import _native
    import os
    lib = _native.lib()
    assert "sm_100a" in _native.version()
    assert os.path.samefile(lib._name, _native.LIB_PATH)
    with open("/proc/self/maps") as fh:
        assert _native.LIB_PATH in fh.read()


@pytest.mark.parametrize("exact", [True, False])
def test_forward_golden(golden, exact):
    for case, meta, (x, u, num, den) in run_cases(golden):
        a, b = coeffs(num, den, x.dtype)
        y = ops().rational_forward(to_dev(x), a, b, exact=exact).cpu().numpy()
        if exact:
            assert sha(y) == meta["sha_y"], case
        else:
            ref = golden.get(case, "y")
            if ref is None:
                ref = orc.forward(x, num, den)
            assert orc.matrix_rel(y, ref) <= 1e-5, case


@pytest.mark.parametrize("exact", [True, False])
def test_backward_golden(golden, exact):
    for case, meta, (x, u, num, den) in run_cases(golden):
        a, b = coeffs(num, den, x.dtype)
        if meta["error"]:
            from paper_2505_13813_b200.errors import AccumulationOverflowError
            with pytest.raises(AccumulationOverflowError):
                ops().rational_backward(to_dev(x), to_dev(u), a, b, exact=exact, check_overflow=True)
            continue
        dx, da, db = ops().rational_backward(to_dev(x), to_dev(u), a, b, exact=exact,
                                             check_overflow=True)
        dx, da, db = dx.cpu().numpy(), da.cpu().numpy(), db.cpu().numpy()
        assert da.shape == (meta["groups"], meta["m1"]) and db.shape == (meta["groups"], meta["n"])
        if exact:
            assert sha(dx) == meta["sha_dx"], case
            tol = 1e-12 if x.dtype == np.float64 else 1e-6
            assert orc.matrix_rel(da, golden.get(case, "ref64_da")) <= tol, case
            assert orc.matrix_rel(db, golden.get(case, "ref64_db")) <= tol, case
        else:
            ref_dx = golden.get(case, "dx")
            if ref_dx is None:
                ref_dx = orc.backward_blocked(x, u, num, den, 256)[0]
            assert orc.matrix_rel(dx, ref_dx) <= 1e-5, case
            num_run = num.astype(x.dtype).astype(np.float64)
            den_run = den.astype(x.dtype).astype(np.float64)
            _, da64, db64 = orc.true64_grads(x, u, num_run, den_run)
            # fp64 tensors: the fast policy still rounds in fp64
            tol = 1e-12 if x.dtype == np.float64 else 1e-5
            assert orc.matrix_rel(da, da64) <= tol, case
            assert orc.matrix_rel(db, db64) <= tol, case


def test_triple_loop_oracle_small_cases(golden):
    """verify_oracle analogue: device results vs the reference's triple-loop fp64 oracle."""
    checked = 0
    for case, meta, (x, u, num, den) in run_cases(golden):
        oa = golden.get(case, "oracle_da")
        if oa is None or x.dtype != np.float64:
            continue
        a, b = coeffs(num, den, x.dtype)
        dx, da, db = ops().rational_backward(to_dev(x), to_dev(u), a, b, exact=True)
        assert orc.matrix_rel(da.cpu().numpy(), oa) <= 1e-12, case
        assert orc.matrix_rel(db.cpu().numpy(), golden.get(case, "oracle_db")) <= 1e-12, case
        assert orc.matrix_rel(dx.cpu().numpy(), golden.get(case, "oracle_dx")) <= 1e-12, case
        checked += 1
    assert checked >= 3


def test_checked_mode_nonfinite():
    from paper_2505_13813_b200.errors import NonFiniteInputError
    x = torch.randn(4, 8, 16, device=DEV)
    x[1, 2, 3] = float("nan")
    a = torch.randn(2, 6, device=DEV)
    b = torch.randn(2, 4, device=DEV)
    with pytest.raises(NonFiniteInputError):
        ops().rational_forward(x, a, b, check_finite=True)
    with pytest.raises(NonFiniteInputError):
        ops().rational_backward(torch.randn_like(x), x, a, b, check_finite=True)
    # unchecked: NaN propagates, no error
    y = ops().rational_forward(x, a, b)
    assert torch.isnan(y[1, 2, 3])


def test_layout_errors():
    from paper_2505_13813_b200.errors import LayoutMismatchError, UnsupportedError
    x = torch.randn(2, 3, 10, device=DEV)
    with pytest.raises(LayoutMismatchError):
        ops().rational_forward(x, torch.randn(4, 6, device=DEV), torch.randn(4, 4, device=DEV))
    with pytest.raises(UnsupportedError):
        ops().rational_forward(x, torch.randn(2, 13, device=DEV), torch.randn(2, 4, device=DEV))
    with pytest.raises(UnsupportedError):
        ops().rational_forward(x.cpu(), torch.randn(2, 6), torch.randn(2, 4))


@pytest.mark.parametrize("shape,groups", [((8, 197, 192), 8), ((3, 7, 48), 4), ((5, 7, 12), 4),
                                          ((2, 9, 3072), 1), ((2, 5, 64), 64)])
def test_bf16(shape, groups):
    rng = np.random.default_rng(5)
    x32 = rng.standard_normal(shape).astype(np.float32)
    u32 = rng.standard_normal(shape).astype(np.float32)
    xb = torch.from_numpy(x32).to(DEV).bfloat16()
    ub = torch.from_numpy(u32).to(DEV).bfloat16()
    xr = xb.float().cpu().numpy()
    ur = ub.float().cpu().numpy()
    num = rng.standard_normal((groups, 6))
    den = rng.standard_normal((groups, 4))
    a, b = coeffs(num, den, np.float32)
    y_ref = orc.forward(xr, num, den)
    dx_ref = c_oracle.backward(xr, ur, num, den, 256)["dx"]
    # exact: bitwise bf16_rn(reference fp32)
    y = ops().rational_forward(xb, a, b, exact=True)
    dx, da, db = ops().rational_backward(xb, ub, a, b, exact=True)
    assert torch.equal(y, torch.from_numpy(y_ref).to(DEV).bfloat16())
    assert torch.equal(dx, torch.from_numpy(dx_ref).to(DEV).bfloat16())
    # fast: 1e-2
    yf = ops().rational_forward(xb, a, b)
    dxf, daf, dbf = ops().rational_backward(xb, ub, a, b)
    assert orc.matrix_rel(yf.float().cpu().numpy(), y_ref) <= 1e-2
    assert orc.matrix_rel(dxf.float().cpu().numpy(), dx_ref) <= 1e-2
    assert daf.dtype == torch.float32 and dbf.dtype == torch.float32
    _, da64, db64 = orc.true64_grads(xr, ur, num.astype(np.float32).astype(np.float64),
                                     den.astype(np.float32).astype(np.float64))
    assert orc.matrix_rel(daf.cpu().numpy(), da64) <= 1e-5
    assert orc.matrix_rel(dbf.cpu().numpy(), db64) <= 1e-5


def test_unaligned_and_strided_inputs_take_the_scalar_path():
    rng = np.random.default_rng(9)
    base = torch.from_numpy(rng.standard_normal(4 * 6 * 32 + 1).astype(np.float32)).to(DEV)
    x = base[1:].view(4, 6, 32)  # 4-byte offset: not 16-byte aligned
    u = torch.from_numpy(rng.standard_normal((4, 6, 32)).astype(np.float32)).to(DEV)
    num = rng.standard_normal((4, 6))
    den = rng.standard_normal((4, 4))
    a, b = coeffs(num, den, np.float32)
    xh = x.cpu().numpy()
    y = ops().rational_forward(x, a, b, exact=True).cpu().numpy()
    assert np.array_equal(y, orc.forward(xh, num, den))
    dx = ops().rational_backward(x, u, a, b, exact=True)[0].cpu().numpy()
    assert np.array_equal(dx, c_oracle.backward(xh, u.cpu().numpy(), num, den)["dx"])


def test_empty_rows():
    a = torch.randn(2, 6, device=DEV)
    b = torch.randn(2, 4, device=DEV)
    x = torch.empty(0, 7, 8, device=DEV)
    assert ops().rational_forward(x, a, b).shape == x.shape
    dx, da, db = ops().rational_backward(x, x, a, b)
    assert dx.shape == x.shape and torch.all(da == 0) and torch.all(db == 0)


def test_determinism_repeated_runs():
    rng = np.random.default_rng(808)
    x = to_dev(rng.standard_normal((64, 197, 768)).astype(np.float32))
    u = to_dev(rng.standard_normal((64, 197, 768)).astype(np.float32))
    a, b = coeffs(rng.standard_normal((8, 6)), rng.standard_normal((8, 4)), np.float32)
    outs = [ops().rational_backward(x, u, a, b) for _ in range(5)]
    for dx, da, db in outs[1:]:
        assert torch.equal(dx, outs[0][0]) and torch.equal(da, outs[0][1]) and torch.equal(db, outs[0][2])


def test_atomic_comparator_dx_matches_and_grads_close(golden):
    case = "katt_seed0_f32_8x197x192_g8"
    x, u, num, den = golden.inputs(case)
    a, b = coeffs(num, den, x.dtype)
    dx_b, da_b, db_b = ops().rational_backward(to_dev(x), to_dev(u), a, b, exact=True)
    dx_a, da_a, db_a = ops().rational_backward_atomic(to_dev(x), to_dev(u), a, b, exact=True)
    assert torch.equal(dx_a, dx_b)
    assert sha(dx_a.cpu().numpy()) == golden.cases[case]["sha_dx"]
    ref_a = golden.get(case, "ref64_da")
    assert orc.matrix_rel(da_a.cpu().numpy(), ref_a) <= 1e-4


def _kat(batch, seq, dim, groups=8, seed=0):
    return orc.bench_inputs(batch, seq, dim, groups, seed=seed)


@pytest.mark.parametrize("name,shape", [("KAT-S", (128, 197, 1536)), ("KAT-B", (256, 197, 3072))])
def test_full_size_parity(name, shape):
    """Configs 1 and 2 at full size: exact y/dx bitwise vs the C oracle, da/db vs fp64,
    and the device error beside the reference's own blocked / naive error."""
    x, u, num, den = _kat(*shape, 8, seed=0)
    a, b = coeffs(num, den, np.float32)
    xd, ud = to_dev(x), to_dev(u)
    r = c_oracle.backward(x, u, num, den, 256)
    y = ops().rational_forward(xd, a, b, exact=True)
    y_ref = c_oracle.forward(x, num, den)
    assert sha(y.cpu().numpy()) == sha(y_ref), name
    yf = ops().rational_forward(xd, a, b)
    assert orc.matrix_rel(yf.cpu().numpy(), y_ref) <= 1e-5, name  # FAST y at full size
    del yf, y_ref
    dx, da, db = ops().rational_backward(xd, ud, a, b, exact=True, check_overflow=True)
    assert sha(dx.cpu().numpy()) == sha(r["dx"]), name
    del y, dx
    dxf, daf, dbf = ops().rational_backward(xd, ud, a, b, check_overflow=True)
    assert orc.matrix_rel(dxf.cpu().numpy(), r["dx"]) <= 1e-5
    del dxf
    for got_a, got_b in ((da, db), (daf, dbf)):
        ga, gb = got_a.cpu().numpy(), got_b.cpu().numpy()
        ea = orc.matrix_rel(ga, r["true64_da"])
        eb = orc.matrix_rel(gb, r["true64_db"])
        assert ea <= 1e-5 and eb <= 1e-5, (name, ea, eb)
        # at least as accurate as the reference's blocked strategy (MAE, paper metric)
        assert orc.mae(ga, r["true64_da"]) <= orc.mae(r["blocked_da"], r["true64_da"]), name
        assert orc.mae(gb, r["true64_db"]) <= orc.mae(r["blocked_db"], r["true64_db"]), name


@pytest.mark.parametrize("name,shape", [("KAT-S", (128, 197, 1536)), ("KAT-B", (256, 197, 3072))])
def test_full_size_bf16_parity(name, shape):
    """Config 2 (KAT-S fp32/bf16) and config 3 (KAT-B) with bf16 I/O at full size.
    The reference has no bf16 (pkg/src/grkan/rational.py:143-144): its fp32 path
    runs on the bf16-rounded inputs.  EXACT y/dx are bitwise bf16_rn(reference
    fp32); FAST within 1e-2 max-scaled (north_star); da/db (fp32) within 1e-5 of
    the fp64 oracle on the same rounded inputs, with MAE no worse than the
    reference's own blocked strategy (pkg/src/grkan/verification.py:497-510)."""
    x, u, num, den = _kat(*shape, 8, seed=2)
    xb = torch.from_numpy(x).bfloat16()
    ub = torch.from_numpy(u).bfloat16()
    del x, u
    xr, ur = xb.float().numpy(), ub.float().numpy()
    a, b = coeffs(num, den, np.float32)
    xd, ud = xb.to(DEV), ub.to(DEV)
    y_ref = c_oracle.forward(xr, num, den)
    y_ref_b = torch.from_numpy(y_ref).bfloat16()  # round-to-nearest-even
    assert torch.equal(ops().rational_forward(xd, a, b, exact=True).cpu(), y_ref_b), name
    yf = ops().rational_forward(xd, a, b)
    assert orc.matrix_rel(yf.float().cpu().numpy(), y_ref) <= 1e-2, name
    del yf, y_ref, y_ref_b
    r = c_oracle.backward(xr, ur, num, den, 256)
    dx, da, db = ops().rational_backward(xd, ud, a, b, exact=True, check_overflow=True)
    assert torch.equal(dx.cpu(), torch.from_numpy(r["dx"]).bfloat16()), name
    del dx
    dxf, daf, dbf = ops().rational_backward(xd, ud, a, b, check_overflow=True)
    assert orc.matrix_rel(dxf.float().cpu().numpy(), r["dx"]) <= 1e-2, name
    del dxf
    for got_a, got_b in ((da, db), (daf, dbf)):
        assert got_a.dtype == torch.float32 and got_b.dtype == torch.float32
        ga, gb = got_a.cpu().numpy(), got_b.cpu().numpy()
        ea = orc.matrix_rel(ga, r["true64_da"])
        eb = orc.matrix_rel(gb, r["true64_db"])
        assert ea <= 1e-5 and eb <= 1e-5, (name, ea, eb)
        assert orc.mae(ga, r["true64_da"]) <= orc.mae(r["blocked_da"], r["true64_da"]), name
        assert orc.mae(gb, r["true64_db"]) <= orc.mae(r["blocked_db"], r["true64_db"]), name


def test_full_size_properties_kat_b():
    """Size-independent properties at KAT-B: exact linearity in dy (x2 is exact), determinism."""
    x, u, num, den = _kat(256, 197, 3072, 8, seed=1)
    a, b = coeffs(num, den, np.float32)
    xd, ud = to_dev(x), to_dev(u)
    del x, u
    dx1, da1, db1 = ops().rational_backward(xd, ud, a, b, exact=True)
    dx2, da2, db2 = ops().rational_backward(xd, ud * 2, a, b, exact=True)
    assert torch.equal(dx2, dx1 * 2)
    assert torch.equal(da2, da1 * 2) and torch.equal(db2, db1 * 2)
    dx3, da3, db3 = ops().rational_backward(xd, ud, a, b, exact=True)
    assert torch.equal(dx3, dx1) and torch.equal(da3, da1) and torch.equal(db3, db1)


def _terms64(x, u, a, b, ng, chunk_rows=4096):
    """fp64 sums of the EXACT per-element terms (bitwise the reference's), chunked."""
    from paper_2505_13813_b200 import _native as N
    rows, d = x.shape
    acc = torch.zeros(10, ng, dtype=torch.float64, device=x.device)
    dxc = torch.empty(chunk_rows, d, dtype=x.dtype, device=x.device)
    t = torch.empty(10 * chunk_rows * d, dtype=torch.float32, device=x.device)
    dt = N.DT_BF16 if x.dtype == torch.bfloat16 else N.DT_F32
    for r0 in range(0, rows, chunk_rows):
        r = min(chunk_rows, rows - r0)
        rc = N.lib().grkan_bwd_terms(x[r0].data_ptr(), u[r0].data_ptr(), a.data_ptr(), b.data_ptr(),
                                     dxc.data_ptr(), t.data_ptr(), r, d, ng, 6, 4, dt, N.FLAG_EXACT,
                                     torch.cuda.current_stream().cuda_stream)
        assert rc == 0, N.last_error()
        acc += t[:10 * r * d].view(10, r, ng, d // ng).double().sum(dim=(1, 3))
    return acc[:6].T, acc[6:].T


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_more_than_2_31_elements(dtype):
    """Maximum sizes: E > 2^31 elements (64-bit indexing in every kernel).  Rows
    past the 2^31 boundary must equal, bit for bit, the same rows computed as a
    small tensor of their own (EXACT is elementwise); da/db within 1e-5
    max-scaled of the fp64 sum of the reference's own terms."""
    d, ng = 3072, 8
    rows = (1 << 31) // d + 64
    g = torch.Generator(device=DEV).manual_seed(31)
    x = torch.randn(rows, d, device=DEV, generator=g).to(dtype)
    u = torch.randn(rows, d, device=DEV, generator=g).to(dtype)
    a = torch.randn(ng, 6, device=DEV, generator=g)
    b = torch.randn(ng, 4, device=DEV, generator=g)
    assert x.numel() > (1 << 31)
    y = ops().rational_forward(x, a, b, exact=True)
    tail = slice(rows - 80, rows)  # straddles element 2^31
    assert torch.equal(y[tail], ops().rational_forward(x[tail].clone(), a, b, exact=True))
    del y
    dx, da, db = ops().rational_backward(x, u, a, b, exact=True, check_overflow=True)
    dx_t, _, _ = ops().rational_backward(x[tail].clone(), u[tail].clone(), a, b, exact=True)
    assert torch.equal(dx[tail], dx_t)
    del dx
    ta, tb = _terms64(x, u, a, b, ng)
    for got_a, got_b in [(da, db),
                         ops().rational_backward(x, u, a, b, check_overflow=True)[1:],
                         ops().rational_backward(x, u, a, b, deterministic=True, check_overflow=True)[1:]]:
        ea = float((got_a.double() - ta).abs().max() / ta.abs().max())
        eb = float((got_b.double() - tb).abs().max() / tb.abs().max())
        assert ea <= 1e-5 and eb <= 1e-5, (dtype, ea, eb)
