"""Host-side logic that needs no GPU: the reference-API shim's types and checks,
presets, error mapping, and that the product path refuses to run without CUDA."""

import os

import numpy as np
import pytest
import torch

from paper_2505_13813_b200 import errors, grkan, presets


def test_presets_match_reference_files(golden):
    for name, rec in golden.presets.items():
        assert list(presets.PRESETS[name]["numerator"]) == rec["numerator"]
        assert list(presets.PRESETS[name]["denominator"]) == rec["denominator"]
        assert presets.PRESETS[name]["fit_error"] == rec["fit_error"]


def test_preset_rows():
    num, den = presets.preset_row("identity", (3, 2))
    assert num == (0.0, 1.0, 0.0, 0.0) and den == (0.0, 0.0)
    with pytest.raises(ValueError):
        presets.preset_row("swish", (3, 2))
    with pytest.raises(ValueError):
        presets.preset_row("nonesuch")
    with pytest.raises(ValueError):
        presets.preset_row("identity", (0, 0))


def test_layout_invariants():
    # pkg/tests/test_rational.py:201-205
    layout = grkan.GroupLayout(12, 3)
    assert layout.group_width == 4
    assert list(layout.group_slices()) == [(0, 0, 4), (1, 4, 8), (2, 8, 12)]
    with pytest.raises(errors.LayoutMismatchError):
        grkan.GroupLayout(7, 2)
    with pytest.raises(errors.LayoutMismatchError):
        grkan.GroupLayout(0, 1)


def test_params_and_tensor_types():
    rng = np.random.default_rng(1)
    p = grkan.GroupRationalParams(rng.standard_normal((3, 6)), rng.standard_normal((3, 4)))
    assert p.degrees == (5, 4) and p.num_coeffs == 6 and p.den_coeffs == 4 and p.total_coeffs == 10
    with pytest.raises(errors.NonFiniteInputError):
        grkan.GroupRationalParams([[np.inf, 1.0]], [[0.0]])
    ident = grkan.GroupRationalParams.identity(2)
    assert ident.numerator.tolist() == [[0, 1, 0, 0, 0, 0]] * 2
    row = grkan.GroupRationalParams.from_row([1.0, 2.0], [3.0], 4)
    assert row.numerator.shape == (4, 2) and row.denominator.shape == (4, 1)
    t = grkan.ActivationTensor(rng.standard_normal((2, 3, 4)).astype(np.float32))
    assert (t.batch, t.seq, t.feature, t.num_elements, t.precision) == (2, 3, 4, 24, "single")
    assert grkan.ActivationTensor(np.zeros((1, 1, 2), dtype=np.int32)).data.dtype == np.float64
    with pytest.raises(ValueError):
        grkan.ActivationTensor(np.zeros((2, 2)))
    assert t.rows().shape == (6, 4)


def test_execution_plan_geometry():
    layout = grkan.GroupLayout(8, 2)
    x = grkan.ActivationTensor(np.zeros((3, 3, 8)))
    plan = grkan.ExecutionPlan.blocked(3, 3, layout, 4)
    assert plan.grid_rows == 3 and plan.grid_cols == 2
    plan.validate_for(x)
    bad = grkan.ExecutionPlan("blocked_reduction", 2, layout, 1, 2)
    with pytest.raises(errors.GridGeometryError):
        bad.validate_for(x)
    with pytest.raises(errors.GridGeometryError):
        grkan.ExecutionPlan("blocked_reduction", 0, layout, 1, 1)
    with pytest.raises(ValueError):
        grkan.ExecutionPlan("other", 1, layout, 1, 1)
    naive = grkan.ExecutionPlan.naive(3, 3, layout, 4)
    assert naive.grid_rows == 18 and naive.grid_cols == 1


def test_shim_errors_before_any_device_work():
    rng = np.random.default_rng(2)
    params = grkan.GroupRationalParams.identity(2)
    x = grkan.ActivationTensor(rng.standard_normal((1, 1, 6)))
    with pytest.raises(errors.LayoutMismatchError):
        grkan.forward_tensor(x, params, grkan.GroupLayout(4, 2))
    x = grkan.ActivationTensor(rng.standard_normal((2, 3, 8)))
    up = grkan.ActivationTensor(rng.standard_normal((2, 1, 8)))
    with pytest.raises(errors.GridGeometryError):
        grkan.backward_blocked(x, up, params)
    with pytest.raises(ValueError):
        grkan.backward_blocked(x, x, params, combine_mode="nonesuch")


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    from paper_2505_13813_b200 import ops
    x = torch.randn(2, 3, 8)
    a = torch.randn(2, 6)
    b = torch.randn(2, 4)
    with pytest.raises(errors.UnsupportedError):
        ops.rational_forward(x, a, b)
    with pytest.raises(errors.UnsupportedError):
        ops.rational_backward(x, x, a, b)
    params = grkan.GroupRationalParams.identity(2)
    with pytest.raises(errors.UnsupportedError):
        grkan.forward_tensor(grkan.ActivationTensor(np.zeros((1, 1, 8))), params, grkan.GroupLayout(8, 2))


def test_status_mapping():
    from paper_2505_13813_b200 import _native as N
    for code, cls in [(N.ERR_LAYOUT, errors.LayoutMismatchError), (N.ERR_GRID, errors.GridGeometryError),
                      (N.ERR_NONFINITE_INPUT, errors.NonFiniteInputError),
                      (N.ERR_ACCUM_OVERFLOW, errors.AccumulationOverflowError),
                      (N.ERR_UNSUPPORTED, errors.UnsupportedError), (N.ERR_CUDA, errors.CudaError)]:
        with pytest.raises(cls):
            errors.raise_for_status(code, "x")
    errors.raise_for_status(N.OK)
    assert issubclass(errors.AccumulationOverflowError, errors.GrkanError)


def test_module_construction_cpu():
    from paper_2505_13813_b200.module import GroupRational
    m = GroupRational(8, init="swish")
    assert m.a.shape == (8, 6) and m.b.shape == (8, 4) and m.a.dtype == torch.float32
    assert torch.equal(m.a[3], torch.tensor(presets.PRESETS["swish"]["numerator"], dtype=torch.float32))
    m2 = GroupRational(4, init="identity", degrees=(3, 2))
    assert m2.a.shape == (4, 4) and m2.b.shape == (4, 2)
    assert "num_groups=4" in repr(m2)


def test_kat_model_shapes_and_init_cpu():
    from paper_2505_13813_b200 import kat
    m = kat.kat_t()
    assert abs(sum(p.numel() for p in m.parameters()) - 5.7e6) < 0.1e6  # PAPER.md Table: 5.7 M
    mlp = m.blocks[0].mlp
    assert mlp.act1.init == "identity" and mlp.act2.init == "swish"
    # variance-preserving: std(W) = 1 / sqrt(alpha * d_in) (pkg/src/grkan/layer.py:293-315)
    alpha = kat.rational_alpha(mlp.act2)
    std = mlp.fc2.weight.std().item()
    assert abs(std - (alpha * mlp.fc2.in_features) ** -0.5) < 0.02 * std
    assert abs(kat.rational_alpha(mlp.act1) - 1.0) < 0.02


def test_grkb_reads_and_writes_reference_dumps(golden, tmp_path):
    """GRKB interop (cli.py:104-129): dumps written by the reference load, and ours are byte-identical."""
    import os
    from paper_2505_13813_b200 import grkb
    for fname, meta in golden.manifest["grkb"].items():
        path = os.path.join(os.path.dirname(__file__), "golden", fname)
        arr = grkb.load(path)
        want = golden.get(meta["case"], meta["key"])
        assert arr.dtype == want.dtype and np.array_equal(arr, want)
        out = tmp_path / fname
        grkb.save(str(out), want)
        assert out.read_bytes() == open(path, "rb").read()
        t = grkan.read_tensor_dump(path)
        assert t.data.shape == want.shape
        grkan.write_tensor_dump(str(out), t)
        assert out.read_bytes() == open(path, "rb").read()
    with pytest.raises(ValueError):
        grkb.loads(b"XXXX" + bytes(29))
    with pytest.raises(ValueError):
        grkb.dumps(np.zeros((2, 2), np.float32))
    with pytest.raises(ValueError):
        grkb.dumps(np.zeros((1, 1, 2), np.int32))


def test_missing_library_fails_loudly():
    """No CUDA extension -> NativeLibraryError at the first call; nothing falls back to a CPU path."""
    import subprocess
    import sys
    code = ("import torch\n"
            "from paper_2505_13813_b200 import _native as N, ops\n"
            "try:\n"
            "    N.lib()\n"
            "except N.NativeLibraryError as e:\n"
            "    print('raised', e)\n")
    env = dict(os.environ, GRKAN_LIB="/nonexistent/libgrkan_b200.so")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=300)
    assert out.returncode == 0, out.stderr
    assert "raised" in out.stdout and "not built" in out.stdout


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_fused_and_parallel_paths_have_no_cpu_fallback():
    from paper_2505_13813_b200 import ops
    x = torch.randn(4, 256).to(torch.bfloat16)
    with pytest.raises(errors.UnsupportedError):
        ops.linear_backward_fused(torch.randn(4, 64).to(torch.bfloat16), torch.randn(64, 256).to(torch.bfloat16),
                                  x, torch.randn(2, 6), torch.randn(2, 4))
