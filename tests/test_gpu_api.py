"""GPU tests of the public APIs: the reference-API shim (ported from the reference's own
tests, pkg/tests/test_rational.py / test_backward.py), the autograd Function and
nn.Module (against a plain PyTorch fp32/fp64 restatement), CUDA-graph capture and
torch.compile."""

import numpy as np
import pytest
import torch

from grkan_testutil import sha
from oracle import grkan_oracle as orc

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


def G():
    from paper_2505_13813_b200 import grkan
    return grkan


def random_instance(rng, batch=2, seq=3, feature=8, groups=2, degrees=(5, 4), dtype=np.float64):
    """pkg/tests/conftest.py:random_instance."""
    g = G()
    m, n = degrees
    layout = g.GroupLayout(feature, groups)
    params = g.GroupRationalParams(rng.standard_normal((groups, m + 1)), rng.standard_normal((groups, n)))
    x = g.ActivationTensor(rng.standard_normal((batch, seq, feature)).astype(dtype))
    up = g.ActivationTensor(rng.standard_normal((batch, seq, feature)).astype(dtype))
    return x, up, params, layout


def rel_err(a, b, floor=1e-12):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)
    return float(np.max(np.abs(a - b) / scale)) if a.size else 0.0


# ---- pkg/tests/test_rational.py, through the shim ------------------------------

def test_scalar_known_answers(golden):
    g = G()
    for s in golden.scalars:
        assert g.eval_rational(s["x"], s["a"], s["b"]) == s["y"], s["tag"]
        eg = g.elementwise_grads(s["x"], s["u"], s["a"], s["b"])
        assert eg.d_x == s["d_x"], s["tag"]
        assert list(eg.d_a) == s["d_a"], s["tag"]
        assert list(eg.d_b) == s["d_b"], s["tag"]


def test_hand_values():
    g = G()
    assert g.eval_rational(2.0, [1.0, 0, 0, 0, 0, 0], [0.0] * 4) == 1.0
    assert g.eval_rational(3.0, [0.0, 1, 0, 0, 0, 0], [0.0] * 4) == 3.0
    assert g.eval_rational(1.0, [1.0, 1.0], [1.0]) == 1.0
    assert g.eval_rational(2.0, [1.0, 2.0], []) == 5.0
    e = g.elementwise_grads(1.0, 1.0, [1.0, 1.0], [1.0])
    assert list(e.d_a) == [0.5, 0.5] and list(e.d_b) == [-0.5] and e.d_x == 0.0
    rng = np.random.default_rng(3)
    a, b = rng.standard_normal(6), rng.standard_normal(4)
    e0 = g.elementwise_grads(0.0, 1.0, a, b)
    assert e0.d_a[0] == 1.0 and np.all(e0.d_a[1:] == 0) and np.all(e0.d_b == 0) and e0.d_x == a[1]
    ez = g.elementwise_grads(2.0, 0.0, a, b)
    assert ez.d_x == 0.0 and np.all(ez.d_a == 0) and np.all(ez.d_b == 0)
    with pytest.raises(g.NonFiniteInputError):
        g.eval_rational(float("nan"), [1.0], [])


def test_safety_large_magnitudes():
    g = G()
    rng = np.random.default_rng(4)
    for _ in range(50):
        a = rng.uniform(-1e3, 1e3, 6)
        b = rng.uniform(-1e3, 1e3, 4)
        x = float(rng.uniform(-1e3, 1e3))
        assert np.isfinite(g.eval_rational(x, a, b))
        e = g.elementwise_grads(x, 1.0, a, b)
        assert np.isfinite(e.d_x) and np.all(np.isfinite(e.d_a)) and np.all(np.isfinite(e.d_b))


def test_forward_routing_and_isolation():
    g = G()
    x = g.ActivationTensor(np.array([[[1.0, 2.0, 3.0, 4.0]]]))
    y = g.forward_tensor(x, g.GroupRationalParams.identity(2), g.GroupLayout(4, 2))
    assert np.array_equal(y.data.ravel(), [1.0, 2.0, 3.0, 4.0])
    num = np.zeros((2, 6)); num[0, 1] = 1.0; num[1, 0] = 5.0
    y = g.forward_tensor(x, g.GroupRationalParams(num, np.zeros((2, 4))), g.GroupLayout(4, 2))
    assert np.array_equal(y.data.ravel(), [1.0, 2.0, 5.0, 5.0])
    rng = np.random.default_rng(1234)
    layout = g.GroupLayout(8, 4)
    num = rng.standard_normal((4, 6)); den = rng.standard_normal((4, 4))
    x = g.ActivationTensor(rng.standard_normal((2, 3, 8)))
    base = g.forward_tensor(x, g.GroupRationalParams(num, den), layout)
    for grp in range(4):
        num2 = num.copy(); num2[grp] += 1.0
        changed = g.forward_tensor(x, g.GroupRationalParams(num2, den), layout)
        diff = np.any(changed.data != base.data, axis=(0, 1))
        expect = np.zeros(8, dtype=bool); expect[grp * 2:(grp + 1) * 2] = True
        assert np.array_equal(diff, expect)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_scalar_loop_oracle_zero_ulp(dtype):
    """pkg/tests/test_rational.py:165-195 against the GPU forward."""
    g = G()
    rng = np.random.default_rng(1234)
    layout = g.GroupLayout(8, 2)
    a = rng.standard_normal((2, 6)); b = rng.standard_normal((2, 4))
    x = g.ActivationTensor(rng.standard_normal((2, 3, 8)).astype(dtype))
    y = g.forward_tensor(x, g.GroupRationalParams(a, b), layout)
    assert y.data.dtype == dtype

    def scalar_eval(v, ar, br):
        ar = ar.astype(dtype); br = br.astype(dtype)
        acc = ar[-1]
        for c in ar[-2::-1]:
            acc = dtype(acc * v + c)
        den = br[-1]
        for c in br[-2::-1]:
            den = dtype(den * v + c)
        q = dtype(dtype(1.0) + abs(dtype(den * v)))
        return dtype(acc / q)

    rows = x.rows(); yr = y.data.reshape(rows.shape)
    for r in range(rows.shape[0]):
        for f in range(8):
            assert yr[r, f] == scalar_eval(rows[r, f], a[f // 4], b[f // 4])


def test_checked_mode_and_layout_errors():
    g = G()
    params = g.GroupRationalParams.identity(1)
    bad = g.ActivationTensor(np.array([[[np.nan, 1.0]]]))
    with pytest.raises(g.NonFiniteInputError):
        g.forward_tensor(bad, params, g.GroupLayout(2, 1))
    y = g.forward_tensor(g.ActivationTensor(np.array([[[np.nan, 1.0]]])), params, g.GroupLayout(2, 1),
                         validate=False)
    assert np.isnan(y.data[0, 0, 0])
    with pytest.raises(g.NonFiniteInputError):
        g.ActivationTensor.from_array(np.array([[[1.0, np.inf]]]))


# ---- pkg/tests/test_backward.py, through the shim ------------------------------

def test_single_element():
    g = G()
    params = g.GroupRationalParams.identity(1)
    x = g.ActivationTensor(np.array([[[3.0]]]))
    up = g.ActivationTensor(np.array([[[1.0]]]))
    for fn in (g.backward_blocked, g.backward_naive):
        bundle = fn(x, up, params)
        assert np.array_equal(bundle.d_a, [[1.0, 3.0, 9.0, 27.0, 81.0, 243.0]])
        assert np.array_equal(bundle.d_b, np.zeros((1, 4)))
        assert np.array_equal(bundle.d_x.data, [[[1.0]]])


def test_zero_upstream_and_overflow():
    g = G()
    rng = np.random.default_rng(1234)
    x, up, params, layout = random_instance(rng)
    zero = g.ActivationTensor(np.zeros_like(up.data))
    bundle = g.backward_blocked(x, zero, params)
    assert np.all(bundle.d_a == 0) and np.all(bundle.d_b == 0) and np.all(bundle.d_x.data == 0)
    params = g.GroupRationalParams.identity(1, degrees=(5, 0))
    xo = g.ActivationTensor(np.full((4, 4, 1), 1.0e30, dtype=np.float32))
    uo = g.ActivationTensor(np.ones((4, 4, 1), dtype=np.float32))
    with pytest.raises(g.AccumulationOverflowError):
        g.backward_blocked(xo, uo, params)
    with pytest.raises(g.AccumulationOverflowError):
        g.backward_naive(xo, uo, params)


def test_geometry_errors():
    g = G()
    rng = np.random.default_rng(1234)
    x, up, params, layout = random_instance(rng)
    with pytest.raises(g.GridGeometryError):
        g.backward_blocked(x, g.ActivationTensor(up.data[:, :1]), params)
    bad = g.ExecutionPlan("blocked_reduction", 2, layout, 1, 2)
    with pytest.raises(g.GridGeometryError):
        g.backward_blocked(x, up, params, bad)
    badn = g.ExecutionPlan("naive_atomic", 4, layout, 1, 1)
    with pytest.raises(g.GridGeometryError):
        g.backward_naive(x, up, params, badn)


def test_tail_blocks_and_oracle(golden):
    from oracle import grkan_oracle as orc
    g = G()
    rng = np.random.default_rng(1234)
    x, up, params, layout = random_instance(rng, batch=3, seq=3, feature=8, groups=2)
    plan = g.ExecutionPlan.blocked(3, 3, layout, block_size=4)
    assert plan.grid_rows == 3
    blocked = g.backward_blocked(x, up, params, plan)
    _, da, db = orc.true64_grads(x.data, up.data, params.numerator, params.denominator)
    assert rel_err(blocked.d_a, da) <= 1e-12
    assert rel_err(blocked.d_b, db) <= 1e-12


def test_dx_bitwise_across_strategies_and_reference(golden):
    g = G()
    for case in ("f32_3x5x8_g4", "f64_2x3x8_g2", "tail_f32_7x13x64_g8", "deg32_f32_4x2x8_g2"):
        meta = golden.cases[case]
        xv, uv, num, den = golden.inputs(case)
        x, up = g.ActivationTensor(xv), g.ActivationTensor(uv)
        params = g.GroupRationalParams(num, den)
        plan = g.ExecutionPlan.blocked(xv.shape[0], xv.shape[1], g.GroupLayout(xv.shape[2], meta["groups"]),
                                       meta["block_size"])
        blocked = g.backward_blocked(x, up, params, plan)
        naive = g.backward_naive(x, up, params)
        assert blocked.d_x.data.tobytes() == naive.d_x.data.tobytes()
        assert sha(blocked.d_x.data) == meta["sha_dx"], case
        assert blocked.d_a.dtype == xv.dtype and blocked.precision == ("single" if xv.dtype == np.float32 else "double")
        assert blocked.strategy == "blocked_reduction" and naive.strategy == "naive_atomic"


def test_worker_count_and_repeat_do_not_change_bits():
    g = G()
    rng = np.random.default_rng(1234)
    x, up, params, layout = random_instance(rng, batch=4, seq=16, feature=32, groups=4, dtype=np.float32)
    plan = g.ExecutionPlan.blocked(4, 16, layout, block_size=8)
    ref = g.backward_blocked(x, up, params, plan, workers=1)
    for workers in (2, 4, 8, 1, 1):
        other = g.backward_blocked(x, up, params, plan, workers=workers)
        assert other.d_a.tobytes() == ref.d_a.tobytes()
        assert other.d_b.tobytes() == ref.d_b.tobytes()
        assert other.d_x.data.tobytes() == ref.d_x.data.tobytes()
    unordered = g.backward_blocked(x, up, params, plan, combine_mode=g.COMBINE_UNORDERED)
    assert unordered.combine_mode == g.COMBINE_UNORDERED
    assert rel_err(unordered.d_a, ref.d_a, floor=1e-6) <= 1e-5


def test_run_backward_dispatch():
    g = G()
    rng = np.random.default_rng(5)
    x, up, params, layout = random_instance(rng, dtype=np.float32)
    b1 = g.run_backward(x, up, params, g.ExecutionPlan.blocked(2, 3, layout, 2))
    b2 = g.run_backward(x, up, params, g.ExecutionPlan.naive(2, 3, layout))
    assert b1.strategy == "blocked_reduction" and b2.strategy == "naive_atomic"
    assert b1.d_x.data.tobytes() == b2.d_x.data.tobytes()


# ---- autograd / nn.Module vs a plain PyTorch restatement ----------------------

def torch_reference(x, a, b):
    """Plain PyTorch restatement of y = P(x)/(1+|A(x)|) per group (autograd gives the grads)."""
    d = x.shape[-1]
    ng = a.shape[0]
    xs = x.reshape(-1, ng, d // ng)
    p = torch.zeros_like(xs)
    for k in range(a.shape[1] - 1, -1, -1):
        p = p * xs + a[:, k].view(1, ng, 1)
    s = torch.zeros_like(xs)
    for k in range(b.shape[1] - 1, -1, -1):
        s = s * xs + b[:, k].view(1, ng, 1)
    s = s * xs
    return (p / (1 + s.abs())).reshape(x.shape)


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-5), (torch.float64, 1e-12),
                                       (torch.bfloat16, 1e-2)])
def test_autograd_matches_torch_reference(dtype, tol):
    from paper_2505_13813_b200.module import GroupRationalFn
    torch.manual_seed(0)
    cd = torch.float64 if dtype == torch.float64 else torch.float32
    x = torch.randn(4, 33, 96, device=DEV, dtype=torch.float32).to(dtype).requires_grad_()
    a = torch.randn(8, 6, device=DEV, dtype=cd, requires_grad=True)
    b = torch.randn(8, 4, device=DEV, dtype=cd, requires_grad=True)
    dy = torch.randn(4, 33, 96, device=DEV, dtype=torch.float32).to(dtype)
    y = GroupRationalFn.apply(x, a, b)
    y.backward(dy)
    x64 = x.detach().double().requires_grad_()
    a64 = a.detach().double().requires_grad_()
    b64 = b.detach().double().requires_grad_()
    y64 = torch_reference(x64, a64, b64)
    y64.backward(dy.double())

    def mrel(u, v):
        u, v = u.double(), v.double()
        return ((u - v).abs().max() / max(u.abs().max(), v.abs().max(), 1e-30)).item()

    assert y.dtype == dtype and x.grad.dtype == dtype and a.grad.dtype == cd
    assert mrel(y, y64) <= tol
    assert mrel(x.grad, x64.grad) <= tol
    gtol = 1e-12 if dtype == torch.float64 else 1e-5
    assert mrel(a.grad, a64.grad) <= gtol
    assert mrel(b.grad, b64.grad) <= gtol


def test_gradcheck_fp64():
    from paper_2505_13813_b200.module import GroupRationalFn
    torch.manual_seed(1)
    x = torch.randn(2, 3, 8, device=DEV, dtype=torch.float64, requires_grad=True)
    a = torch.randn(2, 6, device=DEV, dtype=torch.float64, requires_grad=True)
    b = torch.randn(2, 4, device=DEV, dtype=torch.float64, requires_grad=True)
    assert torch.autograd.gradcheck(lambda x, a, b: GroupRationalFn.apply(x, a, b, True), (x, a, b),
                                    eps=1e-6, atol=1e-7, rtol=1e-6)


def test_module_presets_and_training_step():
    from paper_2505_13813_b200 import presets
    from paper_2505_13813_b200.module import GroupRational
    torch.manual_seed(2)
    ident = GroupRational(8, init="identity").to(DEV)
    x = torch.randn(2, 197, 768, device=DEV)
    assert torch.equal(ident(x), x)
    sw = GroupRational(8, init="swish").to(DEV)
    y = sw(x)
    ref = torch.nn.functional.silu(x)
    inside = x.abs() <= 3
    assert (y - ref)[inside].abs().max().item() < 1e-3  # the preset's fit domain is [-3, 3]
    opt = torch.optim.SGD(sw.parameters(), lr=1e-3)
    loss = sw(x).square().mean()
    loss.backward()
    assert sw.a.grad is not None and sw.a.grad.shape == (8, 6) and torch.isfinite(sw.a.grad).all()
    opt.step()
    xb = x.bfloat16()
    yb = sw(xb)
    assert yb.dtype == torch.bfloat16
    assert presets.PRESETS["swish"]["fit_error"] < 1e-5


def test_cuda_graph_capture():
    from paper_2505_13813_b200 import ops
    torch.manual_seed(3)
    x = torch.randn(64, 197, 768, device=DEV)
    dy = torch.randn_like(x)
    a = torch.randn(8, 6, device=DEV)
    b = torch.randn(8, 4, device=DEV)
    ws = torch.empty(ops.workspace_bytes(64 * 197, 768, 8, 6, 4, torch.float32), dtype=torch.uint8, device=DEV)
    y_ref = ops.rational_forward(x, a, b)
    dx_ref, da_ref, db_ref = ops.rational_backward(x, dy, a, b)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ops.rational_forward(x, a, b)
        ops.rational_backward(x, dy, a, b, workspace=ws)
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        y = ops.rational_forward(x, a, b)
        dx, da, db = ops.rational_backward(x, dy, a, b, workspace=ws)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref) and torch.equal(dx, dx_ref)
    assert torch.equal(da, da_ref) and torch.equal(db, db_ref)


def test_torch_compile_traces_the_custom_ops():
    from paper_2505_13813_b200.module import GroupRational
    torch.manual_seed(4)
    m = GroupRational(8, init="gelu").to(DEV)
    x = torch.randn(2, 50, 256, device=DEV, requires_grad=True)
    eager = m(x)
    compiled = torch.compile(m, fullgraph=True)
    out = compiled(x)
    assert torch.equal(out, eager)
    out.sum().backward()
    assert x.grad is not None


def test_host_pipeline_matches_one_shot():
    """streaming.HostPipeline: chunked pinned-host fwd+bwd == one-shot device results."""
    from paper_2505_13813_b200 import ops
    from paper_2505_13813_b200.streaming import HostPipeline
    torch.manual_seed(6)
    x = torch.randn(7, 197, 768)
    dy = torch.randn_like(x)
    a = torch.randn(8, 6, device=DEV)
    b = torch.randn(8, 4, device=DEV)
    xh, dyh = x.pin_memory(), dy.pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    dxh = torch.empty_like(xh).pin_memory()
    pipe = HostPipeline(DEV, 768, 8, chunk_rows=300)  # 1379 rows -> 5 chunks, ragged tail
    for exact in (False, True):
        da, db = pipe.fwd_bwd(xh, dyh, a, b, yh, dxh, exact=exact)
        torch.cuda.synchronize()
        y_ref = ops.rational_forward(x.to(DEV), a, b, exact=exact)
        dx_ref, da_ref, db_ref = ops.rational_backward(x.to(DEV), dy.to(DEV), a, b, exact=exact)
        assert torch.equal(yh, y_ref.cpu()) and torch.equal(dxh, dx_ref.cpu())
        rel = lambda u, v: ((u - v).abs().max() / v.abs().max()).item()  # noqa: E731
        assert rel(da, da_ref) <= 1e-6 and rel(db, db_ref) <= 1e-6
        da2, db2 = pipe.fwd_bwd(xh, dyh, a, b, yh, dxh, exact=exact)
        assert torch.equal(da, da2) and torch.equal(db, db2)  # deterministic


def test_host_pipeline_back_to_back_calls_do_not_race():
    """Two fwd_bwd calls with different inputs and no synchronisation in between:
    the second call's first chunks reuse the device slots the first call's last
    chunks read, so it must wait for them (write-after-read across calls)."""
    from paper_2505_13813_b200 import ops
    from paper_2505_13813_b200.streaming import HostPipeline
    torch.manual_seed(16)
    xs = [torch.randn(1379, 768) for _ in range(3)]
    dys = [torch.randn(1379, 768) for _ in range(3)]
    a = torch.randn(8, 6, device=DEV)
    b = torch.randn(8, 4, device=DEV)
    pipe = HostPipeline(DEV, 768, 8, chunk_rows=300)
    pin = lambda t: t.pin_memory()  # noqa: E731
    xh, dyh = [pin(t) for t in xs], [pin(t) for t in dys]
    yh = [torch.empty_like(t).pin_memory() for t in xs]
    dxh = [torch.empty_like(t).pin_memory() for t in xs]
    grads = [pipe.fwd_bwd(xh[k], dyh[k], a, b, yh[k], dxh[k]) for k in range(3)]  # no sync between
    torch.cuda.synchronize()
    for k in range(3):
        y_ref = ops.rational_forward(xs[k].to(DEV), a, b)
        dx_ref, da_ref, db_ref = ops.rational_backward(xs[k].to(DEV), dys[k].to(DEV), a, b)
        assert torch.equal(yh[k], y_ref.cpu()) and torch.equal(dxh[k], dx_ref.cpu()), k
        rel = lambda u, v: ((u - v).abs().max() / v.abs().max()).item()  # noqa: E731
        assert rel(grads[k][0], da_ref) <= 1e-6 and rel(grads[k][1], db_ref) <= 1e-6, k


def test_kat_training_smoke():
    """KAT-T (GR-KAN MLPs on the B200 unit) fits a fixed tiny batch (cf. pkg/tests/test_acceptance.py:174-229)."""
    from paper_2505_13813_b200 import kat
    torch.manual_seed(7)
    model = kat.KAT(img=32, patch=8, dim=96, depth=2, heads=3, classes=10).to(DEV)
    imgs = torch.randn(16, 3, 32, 32, device=DEV)
    labels = torch.randint(0, 10, (16,), device=DEV)
    opt = torch.optim.AdamW(model.parameters(), lr=3e-3)
    losses = []
    for _ in range(60):
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = torch.nn.functional.cross_entropy(model(imgs), labels)
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)
        losses.append(loss.item())
    assert losses[-1] < 0.1 * losses[0]
    act = model.blocks[0].mlp.act2
    assert not torch.equal(act.a.detach().cpu(), kat.GroupRational(8, init="swish").a.detach())  # trained


def test_grkb_dump_of_gpu_dx_is_byte_identical(golden, tmp_path):
    """the device dx, dumped as GRKB, equals the reference CLI's dump byte for byte."""
    import os
    from paper_2505_13813_b200 import grkb
    g = G()
    case = "f32_2x4x16_g2"
    x, u, num, den = golden.inputs(case)
    b = g.backward_blocked(g.ActivationTensor(x), g.ActivationTensor(u), g.GroupRationalParams(num, den))
    out = tmp_path / "dx.grkb"
    g.write_tensor_dump(str(out), b.d_x)
    ref = os.path.join(os.path.dirname(__file__), "golden", "dx_f32_2x4x16.grkb")
    assert out.read_bytes() == open(ref, "rb").read()
    assert np.array_equal(grkb.load(str(out)), b.d_x.data)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("degrees", [(5, 4), (3, 2), (5, 0)])
def test_gradient_terms_bitwise_vs_reference_restatement(dtype, degrees):
    """shim.gradient_terms (grkan_bwd_terms, EXACT) == the reference's per-element terms, bit for bit."""
    from paper_2505_13813_b200 import grkan as shim
    m, n = degrees
    rng = np.random.default_rng(9 + m + n)
    x = rng.standard_normal((3, 7, 11)).astype(dtype)
    u = rng.standard_normal((3, 7, 11)).astype(dtype)
    x.reshape(-1)[:3] = [0.0, -0.0, 2.0]
    u.reshape(-1)[3] = -0.0
    num = rng.standard_normal(m + 1)
    den = rng.standard_normal(n)
    dx, ta, tb = shim.gradient_terms(x, u, num, den)
    rdx, rta, rtb = orc.element_terms(x, u, num, den)
    assert dx.tobytes() == rdx.tobytes()
    assert len(ta) == m + 1 and len(tb) == n
    for got, ref in zip(ta + tb, rta + rtb):
        assert got.dtype == ref.dtype and got.tobytes() == ref.tobytes()
    y = shim.rational_values(x, num, den)
    assert y.tobytes() == orc.rational(x, num, den).tobytes()


def test_large_outputs_through_the_staged_download():
    """Outputs above two 32 MB staging chunks take the pinned double-buffered download;
    bytes must equal the device result (fp32 and fp64, ragged last chunk)."""
    import torch
    from paper_2505_13813_b200 import grkan as G
    from paper_2505_13813_b200 import ops
    for dtype, shape in ((np.float32, (5, 1031, 4096)), (np.float64, (3, 1000, 4096))):
        rng = np.random.default_rng(3)
        x = G.ActivationTensor(rng.standard_normal(shape).astype(dtype))
        params = G.GroupRationalParams(rng.standard_normal((8, 6)), rng.standard_normal((8, 4)))
        layout = G.GroupLayout(shape[2], 8)
        y = G.forward_tensor(x, params, layout)
        xd = torch.from_numpy(x.data).cuda()
        cd = torch.float64 if dtype == np.float64 else torch.float32
        a = torch.from_numpy(params.numerator).to(cd).cuda()
        b = torch.from_numpy(params.denominator).to(cd).cuda()
        want = ops.rational_forward(xd, a, b, exact=True).cpu().numpy()
        assert y.data.dtype == dtype and y.data.tobytes() == want.tobytes()


def test_large_inputs_through_the_staged_upload():
    """Inputs larger than the native pipeline's staging slots stream through them:
    backward equals the direct device computation bit for bit -- dx elementwise, da/db
    as the deterministic family's fold (the pipeline's, independent of chunking);
    back-to-back calls reuse the slots."""
    import torch
    from paper_2505_13813_b200 import grkan as G
    from paper_2505_13813_b200 import ops
    rng = np.random.default_rng(5)
    shape = (5, 1031, 4096)
    x = G.ActivationTensor(rng.standard_normal(shape).astype(np.float32))
    u = G.ActivationTensor(rng.standard_normal(shape).astype(np.float32))
    params = G.GroupRationalParams(rng.standard_normal((8, 6)), rng.standard_normal((8, 4)))
    plan = G.ExecutionPlan.blocked(shape[0], shape[1], G.GroupLayout(shape[2], 8))
    bundles = [G.backward_blocked(x, u, params, plan) for _ in range(2)]
    a = torch.from_numpy(params.numerator).float().cuda()
    b = torch.from_numpy(params.denominator).float().cuda()
    dx, da, db = ops.rational_backward(torch.from_numpy(x.data).cuda(), torch.from_numpy(u.data).cuda(), a, b,
                                       exact=True, deterministic=True)
    for bd in bundles:
        assert bd.d_x.data.tobytes() == dx.cpu().numpy().tobytes()
        assert bd.d_a.tobytes() == da.cpu().numpy().tobytes() and bd.d_b.tobytes() == db.cpu().numpy().tobytes()


def test_concurrent_callers_with_large_arrays():
    """The reference's functions are safe from concurrent callers: two
    threads pushing large arrays through the shim's staging chunks get their own results."""
    import threading
    from paper_2505_13813_b200 import grkan as G
    shape = (5, 1031, 4096)
    params = G.GroupRationalParams(np.random.default_rng(9).standard_normal((8, 6)),
                                   np.random.default_rng(10).standard_normal((8, 4)))
    layout = G.GroupLayout(shape[2], 8)
    inputs = [G.ActivationTensor(np.random.default_rng(20 + i).standard_normal(shape).astype(np.float32))
              for i in range(2)]
    want = [G.forward_tensor(x, params, layout).data for x in inputs]
    got = [[None, None], [None, None]]

    def work(i):
        for r in range(2):
            got[i][r] = G.forward_tensor(inputs[i], params, layout).data

    ts = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for i in range(2):
        for r in range(2):
            assert got[i][r].tobytes() == want[i].tobytes()


def test_double_backward_raises():
    """The backward is first-order only (as the reference's): asking for a second
    derivative through it fails loudly instead of returning silent zeros."""
    import torch
    from paper_2505_13813_b200 import GroupRationalFn
    x = torch.randn(4, 16, device="cuda", requires_grad=True)
    a = torch.randn(2, 6, device="cuda", requires_grad=True)
    b = torch.randn(2, 4, device="cuda", requires_grad=True)
    y = GroupRationalFn.apply(x, a, b)
    (gx,) = torch.autograd.grad(y.sum(), x, create_graph=True)
    with pytest.raises(RuntimeError):
        gx.sum().backward()
