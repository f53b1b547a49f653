"""The GR-KAN layer around the hot path, with the reference's API, on the B200.

Same names, argument meaning and errors as ``grkan.layer`` (pkg/src/grkan/layer.py):
``GrKanLayer``, ``make_layer``, ``layer_forward`` (y = W F(x) + bias) and
``layer_backward`` (rational-stage GradBundle, d_weight, d_bias).  Host NumPy arrays
in and out; F and its backward run on the sm_100a kernels, the two W products on
cuBLAS in the input precision (TF32 off, so fp32 stays fp32).  d_weight is one GEMM
over all rows rather than the reference's per-row-block fold; it matches to within
fp32 reassociation (tests/test_gpu_layer.py against the reference's fixtures).
"""

from __future__ import annotations

import contextlib
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .errors import LayoutMismatchError, UnsupportedError
from .grkan import (
    DEFAULT_BLOCK_SIZE,
    STRATEGY_BLOCKED,
    STRATEGY_NAIVE,
    ActivationTensor,
    ExecutionPlan,
    GradBundle,
    GroupLayout,
    GroupRationalParams,
    _device,
    _exact,
)
from .presets import preset_row


@dataclass
class GrKanLayer:
    """Layer parameters: group coefficients plus the linear map (layer.py:45-70)."""

    params: GroupRationalParams
    layout: GroupLayout
    weight: np.ndarray
    bias: np.ndarray | None = None

    def __post_init__(self):
        self.weight = np.ascontiguousarray(np.asarray(self.weight, dtype=np.float64))
        if self.weight.ndim != 2:
            raise ValueError("weight must be a (d_out, d_in) matrix")
        if self.weight.shape[1] != self.layout.feature_dim:
            raise LayoutMismatchError("layout mismatch: weight d_in %d vs layout %d"
                                      % (self.weight.shape[1], self.layout.feature_dim))
        if self.params.num_groups != self.layout.num_groups:
            raise LayoutMismatchError("layout mismatch: params groups vs layout groups")
        if self.bias is None:
            self.bias = np.zeros(self.weight.shape[0])
        self.bias = np.ascontiguousarray(np.asarray(self.bias, dtype=np.float64))
        if self.bias.shape != (self.weight.shape[0],):
            raise ValueError("bias must have length d_out")
        if not (np.all(np.isfinite(self.weight)) and np.all(np.isfinite(self.bias))):
            raise ValueError("layer parameters must be finite")

    d_in = property(lambda self: self.weight.shape[1])
    d_out = property(lambda self: self.weight.shape[0])


def make_layer(d_in: int, d_out: int, num_groups: int, target: str = "identity", degrees=(5, 4),
               weight: np.ndarray | None = None) -> GrKanLayer:
    """Every group set to the same activation-mimicking row (layer.py:265-279).  The
    built-in presets only (identity at any degree; swish / gelu at (5, 4)): fitting new
    rows (fit_activation_coeffs) is outside the hot path."""
    layout = GroupLayout(d_in, num_groups)
    try:
        num, den = preset_row(target, tuple(degrees))
    except ValueError as exc:
        raise UnsupportedError("no built-in preset for %r at degrees %r (coefficient fitting is not "
                               "part of the B200 path)" % (target, tuple(degrees))) from exc
    params = GroupRationalParams.from_row(num, den, num_groups)
    if weight is None:
        weight = np.zeros((d_out, d_in))
    return GrKanLayer(params=params, layout=layout, weight=weight)


@contextlib.contextmanager
def _ieee_matmul():
    """fp32 GEMMs in fp32 (no TF32), as NumPy computes them."""
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        yield
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def _dev_coeffs(params: GroupRationalParams, tdt, dev):
    return (torch.from_numpy(params.numerator).to(device=dev, dtype=tdt).contiguous(),
            torch.from_numpy(params.denominator).to(device=dev, dtype=tdt).contiguous())


def layer_forward(layer: GrKanLayer, x: ActivationTensor, validate: bool = True,
                  exact: bool | None = None) -> ActivationTensor:
    """y[b, s, :] = W @ F(x[b, s, :]) + bias, in the input precision (layer.py:318-325)."""
    if x.feature != layer.layout.feature_dim:
        raise LayoutMismatchError("layout mismatch: tensor feature dim %d vs layout %d"
                                  % (x.feature, layer.layout.feature_dim))
    dev = _device()
    xd = torch.from_numpy(x.data).to(dev)
    a, b = _dev_coeffs(layer.params, xd.dtype, dev)
    check = validate and not x.validated
    f = ops.rational_forward(xd, a, b, exact=_exact(exact), check_finite=check)
    if check:
        x.validated = True
    w = torch.from_numpy(layer.weight).to(device=dev, dtype=xd.dtype)
    bias = torch.from_numpy(layer.bias).to(device=dev, dtype=xd.dtype)
    with _ieee_matmul():
        y = torch.addmm(bias, f.reshape(-1, x.feature), w.t())
    return ActivationTensor(y.reshape(x.batch, x.seq, layer.d_out).cpu().numpy())


def layer_backward(layer: GrKanLayer, x: ActivationTensor, upstream_y: ActivationTensor,
                   strategy: str = STRATEGY_BLOCKED, block_size: int = DEFAULT_BLOCK_SIZE, workers: int = 1,
                   validate: bool = True, exact: bool | None = None):
    """(GradBundle, d_weight, d_bias) of the layer (layer.py:328-379).  The rational stage
    receives uy W per position and runs the blocked (K2 + K3) or the naive (Alg. 1)
    backward; d_weight = uy^T F(x) and d_bias = sum(uy), returned as float64."""
    if upstream_y.feature != layer.d_out:
        raise LayoutMismatchError("layout mismatch: upstream feature %d vs d_out %d"
                                  % (upstream_y.feature, layer.d_out))
    if (upstream_y.batch, upstream_y.seq) != (x.batch, x.seq):
        raise LayoutMismatchError("layout mismatch: upstream batch/seq differ from input")
    if x.feature != layer.layout.feature_dim:
        raise LayoutMismatchError("layout mismatch: tensor feature dim %d vs layout %d"
                                  % (x.feature, layer.layout.feature_dim))
    plan_fn = ExecutionPlan.naive if strategy == STRATEGY_NAIVE else ExecutionPlan.blocked
    plan_fn(x.batch, x.seq, layer.layout, block_size).validate_for(x)
    if validate:
        x.check_finite()
        upstream_y.check_finite()
    dev = _device()
    xd = torch.from_numpy(x.data).to(dev)
    tdt = xd.dtype
    uy = torch.from_numpy(upstream_y.data).to(device=dev, dtype=tdt).reshape(-1, layer.d_out)
    w = torch.from_numpy(layer.weight).to(device=dev, dtype=tdt)
    a, b = _dev_coeffs(layer.params, tdt, dev)
    ex = _exact(exact)
    with _ieee_matmul():
        up = (uy @ w).reshape(xd.shape).contiguous()
        if strategy == STRATEGY_NAIVE:
            dx, da, db = ops.rational_backward_atomic(xd, up, a, b, exact=ex, check_overflow=True)
        else:
            dx, da, db = ops.rational_backward(xd, up, a, b, exact=ex, check_overflow=True)
        f = ops.rational_forward(xd, a, b, exact=ex).reshape(-1, layer.d_in)
        d_w = uy.t() @ f
        d_bias = uy.sum(0)
    bundle = GradBundle(d_x=ActivationTensor(dx.cpu().numpy()), d_a=da.cpu().numpy(), d_b=db.cpu().numpy(),
                        strategy=STRATEGY_NAIVE if strategy == STRATEGY_NAIVE else STRATEGY_BLOCKED,
                        precision=x.precision, combine_mode="deterministic_ordered")
    return bundle, d_w.double().cpu().numpy(), d_bias.double().cpu().numpy()
