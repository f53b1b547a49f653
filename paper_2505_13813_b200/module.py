"""The PyTorch-facing API: ``GroupRationalFn`` (autograd) and ``GroupRational`` (nn.Module).

The FlashKAT/KAT boundary named by north_star: forward(x, a, b) -> y and a
backward returning (dx, da, db).  Both directions run the sm_100a kernels
through the torch.library ops of ``ops.py``.
"""

from __future__ import annotations

import torch
from torch import nn
from torch.autograd.function import once_differentiable

from . import ops  # noqa: F401  (registers torch.ops.grkan_b200.*)
from .presets import preset_row


class GroupRationalFn(torch.autograd.Function):
    """y = P(x) / (1 + |A(x)|) with per-group coefficients a [G, m+1], b [G, n].

    forward(x, a, b[, exact]) -> y (same shape and dtype as x)
    backward(dy) -> (dx, da, db): dx like x; da, db in the coefficient dtype,
    reduced over every row with no atomics and bitwise-reproducible order.
    """

    @staticmethod
    def forward(ctx, x, a, b, exact: bool = False):
        ctx.exact = bool(exact)
        ctx.save_for_backward(x, a, b)
        return torch.ops.grkan_b200.rational_fwd(x, a, b, ctx.exact)

    @staticmethod
    @once_differentiable  # the reference has no second derivative either; double backward raises
    def backward(ctx, dy):
        x, a, b = ctx.saved_tensors
        dx, da, db = torch.ops.grkan_b200.rational_bwd(x, dy.contiguous(), a, b, ctx.exact)
        return dx, da, db, None


def group_rational(x, a, b, exact: bool = False):
    return GroupRationalFn.apply(x, a, b, exact)


class GroupRational(nn.Module):
    """Group-rational activation over the last dim of x (KAT's GR-KAN unit).

    Coefficients are shared by the ``num_groups`` contiguous channel groups
    and initialised by broadcasting one preset row to every group, as
    make_layer does (pkg/src/grkan/layer.py:265-279).
    """

    def __init__(self, num_groups: int = 8, init: str = "identity", degrees=(5, 4),
                 exact: bool = False, device=None, dtype=torch.float32):
        super().__init__()
        num, den = preset_row(init, tuple(degrees))
        self.num_groups = int(num_groups)
        self.init = init
        self.degrees = tuple(degrees)
        self.exact = bool(exact)
        a = torch.tensor(num, dtype=torch.float64).repeat(self.num_groups, 1)
        b = torch.tensor(den, dtype=torch.float64).reshape(1, -1).repeat(self.num_groups, 1)
        self.a = nn.Parameter(a.to(device=device, dtype=dtype))
        self.b = nn.Parameter(b.to(device=device, dtype=dtype))

    def forward(self, x):
        a, b = self.a, self.b
        want = ops.coeff_dtype(x.dtype)
        if a.dtype != want:
            a, b = a.to(want), b.to(want)
        return GroupRationalFn.apply(x, a, b, self.exact)

    def extra_repr(self) -> str:
        return "num_groups=%d, init=%s, degrees=%s, exact=%s" % (
            self.num_groups, self.init, self.degrees, self.exact)


class GroupRationalLinearFn(torch.autograd.Function):
    """y = R(x) W^T + bias -- a GR-KAN layer -- with the fused tcgen05 backward.

    Forward runs the rational kernel and cuBLAS; backward computes
    (dx, da, db) in ONE kernel (ops.linear_backward_fused: dy.W on the tensor
    cores, the rational backward in its epilogue, dF never stored) and
    dW = dy^T R(x), dbias = sum(dy) with cuBLAS.  bf16 activations (autocast)
    with fp32 coefficients, degrees (5, 4); see ops.linear_backward_fused for
    the supported shapes.  Reference: layer_forward / layer_backward
    (pkg/src/grkan/layer.py:318-379).
    """

    @staticmethod
    def forward(ctx, x, a, b, weight, bias):
        w = weight.to(x.dtype)
        f = torch.ops.grkan_b200.rational_fwd(x, a, b, False)
        y = torch.nn.functional.linear(f, w, None if bias is None else bias.to(x.dtype))
        ctx.save_for_backward(x, a, b, w, f)
        ctx.has_bias = bias is not None
        ctx.weight_dtype = weight.dtype
        return y

    @staticmethod
    @once_differentiable
    def backward(ctx, dy):
        x, a, b, w, f = ctx.saved_tensors
        dy = dy.contiguous()
        dx, da, db = ops.linear_backward_fused(dy, w, x, a, b)
        dy2 = dy.reshape(-1, dy.shape[-1])
        dw = (dy2.t() @ f.reshape(-1, f.shape[-1])).to(ctx.weight_dtype)
        dbias = dy2.sum(0).to(ctx.weight_dtype) if ctx.has_bias else None
        return dx, da, db, dw, dbias


def fused_layer_supported(x: torch.Tensor, act: "GroupRational", fc: nn.Linear) -> bool:
    """The fused backward's contract: bf16 CUDA activations, degrees (5, 4), fp32 coefficients,
    K % 64 == 0, group width a multiple of 32, at most 64 groups."""
    n, k = fc.in_features, fc.out_features
    return (x.is_cuda and x.dtype == torch.bfloat16 and act.degrees == (5, 4) and act.a.dtype == torch.float32
            and k % 64 == 0 and n % act.num_groups == 0 and (n // act.num_groups) % 32 == 0
            and act.num_groups <= 64)
