"""Fused GR-KAN layer backward (tcgen05 GEMM + rational-backward epilogue), SURVEY.md 8f #3.

Reference: the unfused chain the reference's layer_backward performs
(pkg/src/grkan/layer.py:318-379): dF = dY . W, then backward_blocked(X, dF).
Here dF comes from an fp32 torch matmul of the same bf16 operands (TF32 off)
and the rational backward from this package's own parity-tested kernel, and,
at small sizes, from the fp64 oracle.  Tolerances: dx (bf16 output)
max-scaled <= 1e-2 (north_star's bf16 bar); da/db max-scaled <= 1e-4 vs the
fp32 chain (dF summation order differs) and <= 1e-5 vs fp64.
"""

import pytest
import torch

from oracle import grkan_oracle as orc

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None

SHAPES = [
    # M, F (features of X), K (out features of W), groups
    (256, 256, 128, 2),       # dg 128 -> BN 128, 128B-swizzle B atoms
    (200, 256, 64, 4),        # M tail (TMA zero fill, masked rows); dg 64
    (384, 768, 192, 8),       # dg 96 -> BN 96, 64B-swizzle B atoms
    (1024, 3072, 768, 8),     # KAT-B second rational -> fc2 (dg 384 -> BN 192)
    (512, 768, 3072, 8),      # KAT-B first rational -> fc1 (K = 3072)
]


def _inputs(M, F, K, ng, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = torch.randn(M, F, generator=g).to(torch.bfloat16)
    dy = torch.randn(M, K, generator=g).to(torch.bfloat16)
    w = (torch.randn(K, F, generator=g) / K ** 0.5).to(torch.bfloat16)
    a = torch.randn(ng, 6, generator=g)
    b = torch.randn(ng, 4, generator=g)
    return [t.to(DEV) for t in (x, dy, w, a, b)]


@pytest.mark.parametrize("M,F,K,ng", SHAPES)
def test_fused_matches_unfused_chain(M, F, K, ng):
    from paper_2505_13813_b200 import ops
    torch.backends.cuda.matmul.allow_tf32 = False
    x, dy, w, a, b = _inputs(M, F, K, ng, seed=M + F + K)
    dx, da, db = ops.linear_backward_fused(dy, w, x, a, b, check_overflow=True)
    dF = dy.float() @ w.float()
    dx_ref, da_ref, db_ref = ops.rational_backward(x.float(), dF, a, b)
    assert orc.matrix_rel(dx.float().cpu().numpy(), dx_ref.cpu().numpy()) <= 1e-2
    assert orc.matrix_rel(da.cpu().numpy(), da_ref.cpu().numpy()) <= 1e-4
    assert orc.matrix_rel(db.cpu().numpy(), db_ref.cpu().numpy()) <= 1e-4
    if M * F <= 300_000:  # fp64 oracle at small sizes
        dF64 = dy.double().cpu().numpy() @ w.double().cpu().numpy()
        xs = x.double().cpu().numpy()[None]
        dx64, da64, db64 = orc.true64_grads(xs, dF64[None], a.double().cpu().numpy(), b.double().cpu().numpy())
        assert orc.matrix_rel(da.double().cpu().numpy(), da64) <= 1e-5
        assert orc.matrix_rel(db.double().cpu().numpy(), db64) <= 1e-5
        assert orc.matrix_rel(dx.double().cpu().numpy(), dx64[0]) <= 1e-2


def test_fused_is_deterministic_and_rejects_bad_shapes():
    from paper_2505_13813_b200 import ops
    from paper_2505_13813_b200.errors import GrkanError
    x, dy, w, a, b = _inputs(256, 256, 128, 2, seed=3)
    r1 = ops.linear_backward_fused(dy, w, x, a, b)
    r2 = ops.linear_backward_fused(dy, w, x, a, b)
    for t1, t2 in zip(r1, r2):
        assert torch.equal(t1, t2)
    with pytest.raises(GrkanError):  # K not a multiple of 64
        ops.linear_backward_fused(dy[:, :100].contiguous(), w[:100].contiguous(), x, a, b)
    with pytest.raises(GrkanError):  # group width 40 (not a multiple of 32)
        x2, dy2, w2, a2, b2 = _inputs(128, 80, 64, 2, seed=4)
        ops.linear_backward_fused(dy2, w2, x2, a2, b2)


def test_fused_grkan_layer_matches_unfused_in_a_kat_block():
    """GroupRationalLinearFn (fused backward) vs the module-by-module GR-KAN MLP, bf16 autocast."""
    from paper_2505_13813_b200 import kat
    torch.manual_seed(5)
    ref = kat.GRKAN(256, 1024, 8).to(DEV)
    fus = kat.GRKAN(256, 1024, 8, fused=True).to(DEV)
    fus.load_state_dict(ref.state_dict())
    with torch.no_grad():  # non-trivial coefficients for both rationals
        for m in (ref, fus):
            m.act1.b.copy_(torch.linspace(-0.3, 0.3, 32, device=DEV).reshape(8, 4))
    x = torch.randn(4, 50, 256, device=DEV).to(torch.bfloat16)  # both paths see the same bf16 input
    outs = []
    for m in (ref, fus):
        xi = x.clone().requires_grad_(True)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            y = m(xi)
        y.float().square().mean().backward()
        outs.append((y.float(), xi.grad.float(), [p.grad.float() for p in m.parameters()]))
    (y0, g0, p0), (y1, g1, p1) = outs
    assert orc.matrix_rel(y1.detach().cpu().numpy(), y0.detach().cpu().numpy()) <= 2e-2
    assert orc.matrix_rel(g1.cpu().numpy(), g0.cpu().numpy()) <= 3e-2
    for a, b in zip(p1, p0):
        assert orc.matrix_rel(a.cpu().numpy(), b.cpu().numpy()) <= 3e-2


def test_kat_training_with_fused_mlp():
    from paper_2505_13813_b200 import kat
    torch.manual_seed(7)
    model = kat.KAT(img=32, patch=8, dim=256, depth=2, heads=4, classes=10, fused_mlp=True).to(DEV)
    imgs = torch.randn(16, 3, 32, 32, device=DEV)
    labels = torch.randint(0, 10, (16,), device=DEV)
    opt = torch.optim.AdamW(model.parameters(), lr=1e-3)
    losses = []
    for _ in range(40):
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = torch.nn.functional.cross_entropy(model(imgs), labels)
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)
        losses.append(loss.item())
    assert losses[-1] < 0.2 * losses[0]


@pytest.mark.parametrize("M", [512, 300, 130])
def test_cta_pair_path_matches(monkeypatch, M):
    """GRKAN_FUSED_PAIR=1: the long-K shape on CTA pairs (cluster of 2, tcgen05.mma.cta_group::2,
    each CTA loading half of the W tile) gives the single-CTA kernel's results."""
    from paper_2505_13813_b200 import ops
    x, dy, w, a, b = _inputs(M, 768, 3072, 8, seed=21)  # ragged last pair tile at M = 300, 130
    monkeypatch.delenv("GRKAN_FUSED_PAIR", raising=False)
    dx1, da1, db1 = ops.linear_backward_fused(dy, w, x, a, b)
    monkeypatch.setenv("GRKAN_FUSED_PAIR", "1")
    dx2, da2, db2 = ops.linear_backward_fused(dy, w, x, a, b, check_overflow=True)
    # same dF up to fp32 summation order inside the tensor core -> bf16 dx within one ulp-ish
    assert orc.matrix_rel(dx2.float().cpu().numpy(), dx1.float().cpu().numpy()) <= 1e-2
    assert orc.matrix_rel(da2.cpu().numpy(), da1.cpu().numpy()) <= 1e-4
    assert orc.matrix_rel(db2.cpu().numpy(), db1.cpu().numpy()) <= 1e-4
