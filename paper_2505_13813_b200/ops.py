"""Torch-facing entry points onto the C ABI (include/grkan_b200.h).

PyTorch supplies device memory, the current CUDA stream and the caching
allocator (for the backward workspace); all arithmetic happens in the sm_100a
kernels of ``_lib/libgrkan_b200.so``.  Nothing here computes on the CPU and
there is no fallback: a CPU tensor or a missing library raises.

Public functions
  rational_forward(x, a, b)            -> y        (grkan_fwd)
  rational_backward(x, dy, a, b)       -> dx, da, db (grkan_bwd: K2 + K3)
  rational_backward_atomic(x, dy, a, b)-> dx, da, db (grkan_bwd_atomic, Alg. 1 comparator)
  rational_backward(..., deterministic=True)   row-sharding-invariant da/db
  rational_forward_backward(x, dy, a, b) -> y, dx, da, db in one pass (grkan_fwd_bwd)
  backward_partials(x, dy, a, b)       -> dx, per-block partials (grkan_bwd_partials)
  reduce_partials(part, ...)           -> da, db (grkan_reduce_partials)
  linear_backward_fused(dy, w, x, a, b)-> dx, da, db (grkan_linear_bwd: tcgen05 dY.W + rational
                                        backward epilogue, dF never in HBM)
and the torch.library ops ``grkan_b200::rational_fwd`` / ``rational_bwd``
(graph-capturable, torch.compile-traceable through their fake kernels).
"""

from __future__ import annotations

import torch

from . import _native as N
from .errors import LayoutMismatchError, UnsupportedError, raise_for_status

STATUS_WORDS = 4  # grkan_device_status: nonfinite_input, accum_overflow, peer_timeout, reserved
STATUS_BYTES = 4 * STATUS_WORDS
_DT = {torch.float32: N.DT_F32, torch.bfloat16: N.DT_BF16, torch.float64: N.DT_F64}


def coeff_dtype(x_dtype: torch.dtype) -> torch.dtype:
    """Coefficient / gradient dtype for a tensor dtype (fp64 for fp64, else fp32)."""
    return torch.float64 if x_dtype == torch.float64 else torch.float32


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream(dev):
    return torch.cuda.current_stream(dev).cuda_stream


def _validate(x: torch.Tensor, a: torch.Tensor, b: torch.Tensor):
    if x.dtype not in _DT:
        raise UnsupportedError("tensor dtype %s not supported (float32, bfloat16, float64)" % x.dtype)
    if not x.is_cuda:
        raise UnsupportedError("GR-KAN B200 kernels need CUDA tensors (got %s); there is no CPU path"
                               % x.device)
    if x.dim() < 1:
        raise LayoutMismatchError("layout mismatch: tensor needs a feature dimension")
    if a.dim() != 2 or b.dim() != 2 or a.shape[0] != b.shape[0]:
        raise LayoutMismatchError("layout mismatch: a must be [groups, m+1], b [groups, n]")
    cd = coeff_dtype(x.dtype)
    if a.dtype != cd or b.dtype != cd:
        raise UnsupportedError("coefficients must be %s for %s tensors" % (cd, x.dtype))
    if a.device != x.device or b.device != x.device:
        raise UnsupportedError("coefficients must live on %s" % x.device)
    d = x.shape[-1]
    ng = a.shape[0]
    if d < 1 or ng < 1 or d % ng:
        raise LayoutMismatchError("layout mismatch: feature_dim %d not divisible by num_groups %d"
                                  % (d, ng))
    rows = x.numel() // d if d else 0
    return rows, d, ng, a.shape[1], b.shape[1]


def _flags(exact: bool, check_finite: bool, deterministic: bool = False) -> int:
    return ((N.FLAG_EXACT if exact else N.FLAG_FAST) | (N.FLAG_CHECK_FINITE if check_finite else 0)
            | (N.FLAG_DETERMINISTIC if deterministic else 0))


def _raise(rc):
    if rc != N.OK:
        raise_for_status(rc, N.last_error())


def read_status(status: torch.Tensor) -> None:
    """Synchronise and raise NonFiniteInputError / AccumulationOverflowError if flagged."""
    host = N.DeviceStatus()
    rc = N.lib().grkan_read_status(status.data_ptr(), _stream(status.device), host)
    _raise(rc)


def rational_forward(x: torch.Tensor, a: torch.Tensor, b: torch.Tensor, exact: bool = False,
                     check_finite: bool = False, out: torch.Tensor | None = None) -> torch.Tensor:
    """y = P(x)/(1+|A(x)|) per group (forward_tensor, pkg/src/grkan/rational.py:325-345).

    With ``check_finite`` the kernel flags NaN/Inf inputs and this call
    synchronises to raise NonFiniteInputError (the reference's validate=True).
    """
    rows, d, ng, m1, n = _validate(x, a, b)
    x = x.contiguous()
    a = a.contiguous()
    b = b.contiguous()
    y = torch.empty_like(x) if out is None else out
    if y.shape != x.shape or y.dtype != x.dtype or not y.is_contiguous():
        raise ValueError("out must be a contiguous tensor like x")
    status = torch.zeros(STATUS_WORDS, dtype=torch.int32, device=x.device) if check_finite else None
    with torch.cuda.device(x.device):
        rc = N.lib().grkan_fwd(x.data_ptr(), y.data_ptr(), a.data_ptr(), _ptr(b), rows, d, ng, m1, n,
                               _DT[x.dtype], _flags(exact, check_finite), _ptr(status),
                               _stream(x.device))
        _raise(rc)
        if check_finite:
            read_status(status)
    return y


def workspace_bytes(rows: int, d: int, ng: int, m1: int, n: int, dtype: torch.dtype) -> int:
    nbytes = N.lib().grkan_bwd_workspace_bytes(rows, d, ng, m1, n, _DT[dtype])
    if nbytes == 0:
        raise LayoutMismatchError("layout mismatch: cannot size workspace for d=%d groups=%d" % (d, ng))
    return nbytes


def rational_backward(x: torch.Tensor, dy: torch.Tensor, a: torch.Tensor, b: torch.Tensor,
                      exact: bool = False, check_finite: bool = False, check_overflow: bool = False,
                      workspace: torch.Tensor | None = None, da_out: torch.Tensor | None = None,
                      db_out: torch.Tensor | None = None, dx_out: torch.Tensor | None = None,
                      deterministic: bool = False):
    """(dx, da, db) with per-CTA partials and a deterministic second pass.

    ``deterministic`` folds one partial per global row block
    (det_block_rows) instead of one per CTA: da/db are then bitwise what any
    block-aligned row sharding gives through backward_partials +
    reduce_partials (parallel.deterministic_backward).

    Mirrors backward_blocked (pkg/src/grkan/backward.py:275-372).  da/db are
    in the coefficient dtype (fp32 for fp32/bf16 tensors).  ``check_overflow``
    synchronises and raises AccumulationOverflowError for non-finite da/db
    (_check_accumulators, backward.py:182-184); ``check_finite`` also flags
    NaN/Inf in x / dy (validate=True).  ``da_out``/``db_out`` may be views of
    one flat buffer (parallel.coeff_grad_buffer) so the all-reduce needs no copy.
    """
    rows, d, ng, m1, n = _validate(x, a, b)
    if dy.shape != x.shape:
        from .errors import GridGeometryError
        raise GridGeometryError("grid geometry invalid: x and upstream shapes differ")
    if dy.dtype != x.dtype or dy.device != x.device:
        raise UnsupportedError("upstream must match x in dtype and device")
    x = x.contiguous()
    dy = dy.contiguous()
    a = a.contiguous()
    b = b.contiguous()
    dx = torch.empty_like(x) if dx_out is None else dx_out
    if dx.shape != x.shape or dx.dtype != x.dtype or not dx.is_contiguous():
        raise ValueError("dx_out must be a contiguous tensor like x")
    da = torch.empty((ng, m1), dtype=a.dtype, device=x.device) if da_out is None else da_out
    db = torch.empty((ng, n), dtype=a.dtype, device=x.device) if db_out is None else db_out
    for t, shp in ((da, (ng, m1)), (db, (ng, n))):
        if tuple(t.shape) != shp or t.dtype != a.dtype or not t.is_contiguous():
            raise ValueError("gradient output must be a contiguous %s tensor of shape %s" % (a.dtype, shp))
    nbytes = workspace_bytes(rows, d, ng, m1, n, x.dtype)
    if workspace is None or workspace.numel() < nbytes:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
    with torch.cuda.device(x.device):
        rc = N.lib().grkan_bwd(x.data_ptr(), dy.data_ptr(), a.data_ptr(), _ptr(b), dx.data_ptr(),
                               da.data_ptr(), _ptr(db), workspace.data_ptr(), workspace.numel(),
                               rows, d, ng, m1, n, _DT[x.dtype], _flags(exact, check_finite, deterministic),
                               _stream(x.device))
        _raise(rc)
        if check_finite or check_overflow:
            read_status(workspace[:STATUS_BYTES])
    return dx, da, db


def rational_forward_backward(x: torch.Tensor, dy: torch.Tensor, a: torch.Tensor, b: torch.Tensor,
                              exact: bool = False, check_finite: bool = False, check_overflow: bool = False,
                              workspace: torch.Tensor | None = None):
    """(y, dx, da, db): forward_tensor and backward_blocked of the same x in one pass
    (grkan_fwd_bwd: x read once, y from the backward's own P and 1/Q).  Same results as
    rational_forward + rational_backward -- EXACT y / dx bitwise the reference's; bf16
    FAST within the FAST tolerances (rational_backward's x-factor table body rounds the
    terms differently)."""
    rows, d, ng, m1, n = _validate(x, a, b)
    if dy.shape != x.shape:
        from .errors import GridGeometryError
        raise GridGeometryError("grid geometry invalid: x and upstream shapes differ")
    if dy.dtype != x.dtype or dy.device != x.device:
        raise UnsupportedError("upstream must match x in dtype and device")
    x, dy, a, b = x.contiguous(), dy.contiguous(), a.contiguous(), b.contiguous()
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    da = torch.empty((ng, m1), dtype=a.dtype, device=x.device)
    db = torch.empty((ng, n), dtype=a.dtype, device=x.device)
    nbytes = workspace_bytes(rows, d, ng, m1, n, x.dtype)
    if workspace is None or workspace.numel() < nbytes:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
    with torch.cuda.device(x.device):
        rc = N.lib().grkan_fwd_bwd(x.data_ptr(), dy.data_ptr(), a.data_ptr(), _ptr(b), y.data_ptr(), dx.data_ptr(),
                                   da.data_ptr(), _ptr(db), workspace.data_ptr(), workspace.numel(), rows, d, ng,
                                   m1, n, _DT[x.dtype], _flags(exact, check_finite, False), _stream(x.device))
        _raise(rc)
        if check_finite or check_overflow:
            read_status(workspace[:STATUS_BYTES])
    return y, dx, da, db


def det_block_rows(d: int, ng: int, dtype: torch.dtype) -> int:
    """Rows per global block of the deterministic mode (shard boundaries must be multiples)."""
    rb = N.lib().grkan_det_block_rows(d, ng, _DT[dtype])
    if rb <= 0:
        raise LayoutMismatchError("layout mismatch: feature_dim %d not divisible by num_groups %d" % (d, ng))
    return rb


def backward_partials(x: torch.Tensor, dy: torch.Tensor, a: torch.Tensor, b: torch.Tensor,
                      exact: bool = False, check_finite: bool = False, part_out: torch.Tensor | None = None,
                      dx_out: torch.Tensor | None = None):
    """dx and this shard's per-block coefficient partials, [n_blocks, ng, m1 + n] (no reduction).

    The shard must start on a multiple of det_block_rows() rows of the global
    tensor; concatenating every shard's partials in row order and calling
    reduce_partials gives bitwise the single-GPU deterministic da/db.
    """
    rows, d, ng, m1, n = _validate(x, a, b)
    if dy.shape != x.shape or dy.dtype != x.dtype or dy.device != x.device:
        from .errors import GridGeometryError
        raise GridGeometryError("grid geometry invalid: x and upstream differ in shape, dtype or device")
    x, dy, a, b = x.contiguous(), dy.contiguous(), a.contiguous(), b.contiguous()
    dx = torch.empty_like(x) if dx_out is None else dx_out
    n_blocks = -(-rows // det_block_rows(d, ng, x.dtype))
    part = (torch.empty((n_blocks, ng, m1 + n), dtype=a.dtype, device=x.device)
            if part_out is None else part_out)
    if part.shape != (n_blocks, ng, m1 + n) or part.dtype != a.dtype or not part.is_contiguous():
        raise ValueError("part_out must be a contiguous %s tensor of shape %s"
                         % (a.dtype, (n_blocks, ng, m1 + n)))
    status = torch.zeros(STATUS_WORDS, dtype=torch.int32, device=x.device) if check_finite else None
    with torch.cuda.device(x.device):
        rc = N.lib().grkan_bwd_partials(x.data_ptr(), dy.data_ptr(), a.data_ptr(), _ptr(b), dx.data_ptr(),
                                        part.data_ptr(), part.numel() * part.element_size(), rows, d, ng,
                                        m1, n, _DT[x.dtype], _flags(exact, check_finite), _ptr(status),
                                        _stream(x.device))
        _raise(rc)
        if check_finite:
            read_status(status)
    return dx, part


def reduce_partials(part: torch.Tensor, m1: int, n: int, check_overflow: bool = False,
                    da_out: torch.Tensor | None = None, db_out: torch.Tensor | None = None):
    """Fixed-order fp64 fold of [n_blocks, ng, m1 + n] partials -> (da, db) (combine_partials)."""
    if part.dim() != 3 or part.shape[2] != m1 + n:
        raise LayoutMismatchError("layout mismatch: partials must be [blocks, groups, m1 + n]")
    if not part.is_cuda or not part.is_contiguous() or part.dtype not in (torch.float32, torch.float64):
        raise UnsupportedError("partials must be a contiguous CUDA float32/float64 tensor")
    nb, ng = part.shape[0], part.shape[1]
    da = torch.empty((ng, m1), dtype=part.dtype, device=part.device) if da_out is None else da_out
    db = torch.empty((ng, n), dtype=part.dtype, device=part.device) if db_out is None else db_out
    status = torch.zeros(STATUS_WORDS, dtype=torch.int32, device=part.device)
    dt = N.DT_F64 if part.dtype == torch.float64 else N.DT_F32
    with torch.cuda.device(part.device):
        rc = N.lib().grkan_reduce_partials(part.data_ptr(), nb, ng, m1, n, da.data_ptr(), _ptr(db), dt,
                                           status.data_ptr(), _stream(part.device))
        _raise(rc)
        if check_overflow:
            read_status(status)
    return da, db


def rational_backward_atomic(x, dy, a, b, exact: bool = False, check_overflow: bool = False):
    """The paper's Alg. 1 (per-element global atomicAdd): comparator only, not the product path."""
    rows, d, ng, m1, n = _validate(x, a, b)
    x = x.contiguous()
    dy = dy.contiguous()
    dx = torch.empty_like(x)
    da = torch.empty((ng, m1), dtype=a.dtype, device=x.device)
    db = torch.empty((ng, n), dtype=a.dtype, device=x.device)
    status = torch.zeros(STATUS_WORDS, dtype=torch.int32, device=x.device)
    with torch.cuda.device(x.device):
        rc = N.lib().grkan_bwd_atomic(x.data_ptr(), dy.data_ptr(), a.contiguous().data_ptr(),
                                      _ptr(b.contiguous()), dx.data_ptr(), da.data_ptr(), _ptr(db),
                                      rows, d, ng, m1, n, _DT[x.dtype], _flags(exact, False),
                                      status.data_ptr(), _stream(x.device))
        _raise(rc)
        if check_overflow:
            read_status(status)
    return dx, da, db


# ---------------------------------------------------------------------------
# torch.library registration (CUDA graphs / torch.compile see opaque ops)
# ---------------------------------------------------------------------------

@torch.library.custom_op("grkan_b200::rational_fwd", mutates_args=(), device_types="cuda")
def rational_fwd_op(x: torch.Tensor, a: torch.Tensor, b: torch.Tensor, exact: bool) -> torch.Tensor:
    return rational_forward(x, a, b, exact=exact)


@rational_fwd_op.register_fake
def _(x, a, b, exact):
    return torch.empty_like(x)


@torch.library.custom_op("grkan_b200::rational_bwd", mutates_args=(), device_types="cuda")
def rational_bwd_op(x: torch.Tensor, dy: torch.Tensor, a: torch.Tensor, b: torch.Tensor,
                    exact: bool) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    return rational_backward(x, dy, a, b, exact=exact)


@rational_bwd_op.register_fake
def _(x, dy, a, b, exact):
    return torch.empty_like(x), a.new_empty(a.shape), b.new_empty(b.shape)


def linear_backward_fused(dy: torch.Tensor, w: torch.Tensor, x: torch.Tensor, a: torch.Tensor, b: torch.Tensor,
                          check_overflow: bool = False):
    """Backward of  Y = R(X) W^T  through W and R in one kernel.

    dy [..., K], w [K, F] (torch Linear weight [out, in]), x [..., F]: bf16 CUDA
    tensors; a [ng, 6], b [ng, 4] fp32.  Returns (dx like x, da, db) where
    dx = R'(x, dy @ w) and da/db the coefficient gradients -- what
    rational_backward(x, dy @ w, a, b) gives, without materialising dy @ w.
    (dW = dy^T R(x) is a plain GEMM and stays with the caller.)
    """
    if x.dtype != torch.bfloat16 or dy.dtype != torch.bfloat16 or w.dtype != torch.bfloat16:
        raise UnsupportedError("fused linear backward takes bf16 dy, w and x")
    if not (x.is_cuda and dy.is_cuda and w.is_cuda):
        raise UnsupportedError("fused linear backward needs CUDA tensors; there is no CPU path")
    feat = x.shape[-1]
    k = dy.shape[-1]
    if w.dim() != 2 or tuple(w.shape) != (k, feat):
        raise LayoutMismatchError("layout mismatch: w must be [K=%d, F=%d], got %s" % (k, feat, tuple(w.shape)))
    rows = x.numel() // feat if feat else 0
    if dy.numel() // k != rows:
        from .errors import GridGeometryError
        raise GridGeometryError("grid geometry invalid: dy and x disagree on the row count")
    if a.dtype != torch.float32 or b.dtype != torch.float32 or a.shape[1] != 6 or b.shape[1] != 4:
        raise UnsupportedError("fused linear backward: fp32 coefficients of degrees (5, 4)")
    ng = a.shape[0]
    x, dy, w, a, b = x.contiguous(), dy.contiguous(), w.contiguous(), a.contiguous(), b.contiguous()
    dx = torch.empty_like(x)
    da = torch.empty((ng, 6), dtype=torch.float32, device=x.device)
    db = torch.empty((ng, 4), dtype=torch.float32, device=x.device)
    nbytes = N.lib().grkan_linear_bwd_workspace_bytes(rows, feat, k, ng)
    if nbytes == 0:
        raise UnsupportedError("fused linear backward: unsupported shape (F=%d, groups=%d, K=%d)" % (feat, ng, k))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
    with torch.cuda.device(x.device):
        rc = N.lib().grkan_linear_bwd(dy.data_ptr(), w.data_ptr(), x.data_ptr(), a.data_ptr(), b.data_ptr(),
                                      dx.data_ptr(), da.data_ptr(), db.data_ptr(), ws.data_ptr(), ws.numel(),
                                      rows, feat, k, ng, N.FLAG_FAST, _stream(x.device))
        _raise(rc)
        if check_overflow:
            read_status(ws[:STATUS_BYTES])
    return dx, da, db


