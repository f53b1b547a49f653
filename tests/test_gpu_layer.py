"""The layer around the hot path against the reference's own layer fixtures
(layer_forward / layer_backward, pkg/src/grkan/layer.py:318-379; recorded by
tests/golden/make_layer_golden.py):

* the reference-API layer shim (paper_2505_13813_b200.layer) -- same calls, host arrays;
* the PyTorch path a KAT block uses: GroupRational -> nn.Linear with autograd;
* the fused tcgen05 layer (GroupRationalLinearFn, bf16) on its supported shape.

The W products run on cuBLAS (a different summation order from NumPy's BLAS), so the
gates are max-scaled tolerances: 1e-5 for fp32 (north_star's fp32 bound), 1e-12 for
fp64, 1e-2 for bf16 I/O.  F(x) itself is bitwise (EXACT) -- checked through the
identity-initialised case, where y = x W^T + bias exactly as the reference computes it.
"""

import json
import os

import numpy as np
import pytest
import torch

from oracle import grkan_oracle as orc

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def cases():
    with open(os.path.join(HERE, "golden", "layer_golden.json")) as fh:
        man = json.load(fh)
    z = np.load(os.path.join(HERE, "golden", "layer_golden.npz"))
    return [(name, meta, {k.split("/", 1)[1]: z[k] for k in z.files if k.startswith(name + "/")})
            for name, meta in sorted(man["cases"].items())]


CASES = cases()
IDS = [c[0] for c in CASES]


def tol(dtype):
    return 1e-12 if np.dtype(dtype) == np.float64 else 1e-5


@pytest.mark.parametrize("name,meta,arr", CASES, ids=IDS)
def test_layer_shim_matches_reference_fixtures(name, meta, arr):
    from paper_2505_13813_b200 import grkan as G
    from paper_2505_13813_b200 import layer as L
    groups = meta["groups"]
    layer = L.GrKanLayer(params=G.GroupRationalParams(arr["num"], arr["den"]),
                         layout=G.GroupLayout(arr["x"].shape[2], groups), weight=arr["weight"], bias=arr["bias"])
    x = G.ActivationTensor(arr["x"])
    uy = G.ActivationTensor(arr["uy"])
    t = tol(arr["x"].dtype)
    y = L.layer_forward(layer, x).data
    assert y.dtype == arr["y"].dtype and orc.matrix_rel(y, arr["y"]) <= t, name
    bundle, d_w, d_b = L.layer_backward(layer, x, uy, strategy=meta["strategy"], block_size=meta["block_size"])
    assert orc.matrix_rel(bundle.d_x.data, arr["d_x"]) <= t, name
    assert orc.matrix_rel(bundle.d_a, arr["d_a"]) <= t and orc.matrix_rel(bundle.d_b, arr["d_b"]) <= t, name
    assert d_w.dtype == np.float64 and orc.matrix_rel(d_w, arr["d_weight"]) <= t, name
    assert orc.matrix_rel(d_b, arr["d_bias"]) <= t, name
    assert bundle.strategy == meta["strategy"]


def test_identity_layer_rational_stage_is_exact():
    """Identity coefficients: F(x) = x bit for bit, so y - bias is x W^T (the reference's
    activated rows are x itself)."""
    name, meta, arr = next(c for c in CASES if "identity" in c[0])
    from paper_2505_13813_b200 import grkan as G
    y = G.forward_tensor(G.ActivationTensor(arr["x"]), G.GroupRationalParams(arr["num"], arr["den"]),
                         G.GroupLayout(arr["x"].shape[2], meta["groups"])).data
    assert y.tobytes() == arr["x"].tobytes()


def test_layer_errors_as_the_reference():
    from paper_2505_13813_b200 import grkan as G
    from paper_2505_13813_b200 import layer as L
    layer = L.make_layer(16, 8, 4, target="swish", weight=np.ones((8, 16)))
    x = G.ActivationTensor(np.zeros((2, 3, 16), dtype=np.float32))
    with pytest.raises(G.LayoutMismatchError):
        L.layer_backward(layer, x, G.ActivationTensor(np.zeros((2, 3, 7), dtype=np.float32)))
    with pytest.raises(G.LayoutMismatchError):
        L.layer_backward(layer, x, G.ActivationTensor(np.zeros((2, 4, 8), dtype=np.float32)))
    with pytest.raises(G.LayoutMismatchError):
        L.GrKanLayer(params=layer.params, layout=layer.layout, weight=np.ones((8, 12)))
    with pytest.raises(G.UnsupportedError):
        L.make_layer(16, 8, 4, target="tanh")


@pytest.mark.parametrize("name,meta,arr", [c for c in CASES if c[1]["dtype"] == "float32"
                                           and c[1]["strategy"] == "blocked_reduction"],
                         ids=[c[0] for c in CASES if c[1]["dtype"] == "float32"
                              and c[1]["strategy"] == "blocked_reduction"])
def test_torch_group_rational_then_linear(name, meta, arr):
    """The KAT-block path: GroupRational -> nn.Linear, autograd, fp32 on the GPU."""
    from paper_2505_13813_b200.module import GroupRational
    dev = torch.device("cuda", 0)
    d_in, d_out = arr["weight"].shape[1], arr["weight"].shape[0]
    act = GroupRational(num_groups=meta["groups"], exact=True, device=dev)
    with torch.no_grad():
        act.a.copy_(torch.from_numpy(arr["num"]).float())
        act.b.copy_(torch.from_numpy(arr["den"]).float())
    fc = torch.nn.Linear(d_in, d_out).to(dev)
    with torch.no_grad():
        fc.weight.copy_(torch.from_numpy(arr["weight"]).float())
        fc.bias.copy_(torch.from_numpy(arr["bias"]).float())
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        x = torch.from_numpy(arr["x"]).to(dev).requires_grad_(True)
        y = fc(act(x))
        y.backward(torch.from_numpy(arr["uy"]).to(dev))
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    t = 1e-5
    assert orc.matrix_rel(y.detach().cpu().numpy(), arr["y"]) <= t
    assert orc.matrix_rel(x.grad.cpu().numpy(), arr["d_x"]) <= t
    assert orc.matrix_rel(act.a.grad.cpu().numpy(), arr["d_a"]) <= t
    assert orc.matrix_rel(act.b.grad.cpu().numpy(), arr["d_b"]) <= t
    assert orc.matrix_rel(fc.weight.grad.double().cpu().numpy(), arr["d_weight"]) <= t
    assert orc.matrix_rel(fc.bias.grad.double().cpu().numpy(), arr["d_bias"]) <= t


def test_fused_tcgen05_layer_bf16():
    """GroupRationalLinearFn (rational forward + cuBLAS; fused tcgen05 backward) with bf16
    activations against the reference's fp32 layer on the same case: within the bf16
    I/O tolerance (1e-2 max-scaled), the inputs themselves being rounded to bf16."""
    from paper_2505_13813_b200.module import GroupRationalLinearFn
    name, meta, arr = next(c for c in CASES if c[0] == "f32_swish_2x16x256_o64_g8")
    dev = torch.device("cuda", 0)
    x = torch.from_numpy(arr["x"]).to(dev, torch.bfloat16).requires_grad_(True)
    a = torch.from_numpy(arr["num"]).float().to(dev).requires_grad_(True)
    b = torch.from_numpy(arr["den"]).float().to(dev).requires_grad_(True)
    w = torch.from_numpy(arr["weight"]).float().to(dev).requires_grad_(True)
    bias = torch.from_numpy(arr["bias"]).float().to(dev).requires_grad_(True)
    y = GroupRationalLinearFn.apply(x, a, b, w, bias)
    y.backward(torch.from_numpy(arr["uy"]).to(dev, torch.bfloat16))
    t = 1e-2
    assert orc.matrix_rel(y.float().detach().cpu().numpy(), arr["y"]) <= t
    assert orc.matrix_rel(x.grad.float().cpu().numpy(), arr["d_x"]) <= t
    assert orc.matrix_rel(a.grad.cpu().numpy(), arr["d_a"]) <= t
    assert orc.matrix_rel(b.grad.cpu().numpy(), arr["d_b"]) <= t
    assert orc.matrix_rel(w.grad.double().cpu().numpy(), arr["d_weight"]) <= t
    assert orc.matrix_rel(bias.grad.double().cpu().numpy(), arr["d_bias"]) <= t
