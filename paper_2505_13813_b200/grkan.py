"""Reference-API shim: the ``grkan`` functional interface, executed on the B200.

Same names, argument meaning and error behaviour as the reference package
(/root/reference/pkg/src/grkan), so code and tests written against
``grkan.forward_tensor`` / ``grkan.backward_blocked`` run unchanged on the GPU:

    from paper_2505_13813_b200 import grkan
    y = grkan.forward_tensor(x, params, layout)            # rational.py:325
    bundle = grkan.backward_blocked(x, up, params, plan)   # backward.py:275

Host NumPy arrays in, host NumPy arrays out (the CPU path's contract); every
element is computed by the sm_100a kernels.  By default the shim runs the
EXACT policy (reference op order, IEEE-rounded ops), so ``y`` and ``d_x`` are
bitwise identical to the reference; ``d_a``/``d_b`` come from the device
tree reduction (more accurate than either reference strategy, not bitwise).
Pass ``exact=False`` (or ``set_default_exact(False)``) for the FMA policy.

Differences, all deliberate: ``workers`` is accepted and ignored (the GPU is
the pool); ``counter``/``coverage`` run the kernels' counting instantiations
(grkan_bwd_instrumented), so the tallies are the B200 kernels' own accesses in the
reference's units, not the reference's model; ``backward_naive`` runs the
paper's Alg. 1 (global atomicAdd), the algorithm the reference's naive
strategy models, so its d_a/d_b are not bit-reproducible.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field
from typing import Iterator

import numpy as np
import torch

from . import ops
from .errors import raise_for_status
from .errors import (  # noqa: F401  (re-exported like grkan/__init__.py)
    AccumulationOverflowError,
    ActivationFitError,
    DegenerateAlphaError,
    GridGeometryError,
    GrkanError,
    LayoutMismatchError,
    NonFiniteInputError,
    PartialCoverageError,
    TailNotCoveredError,
    UnsupportedError,
)

STRATEGY_NAIVE = "naive_atomic"           # backward.py:44
STRATEGY_BLOCKED = "blocked_reduction"    # backward.py:45
COMBINE_ORDERED = "deterministic_ordered"  # backward.py:46
COMBINE_UNORDERED = "unordered_scatter"   # backward.py:47
DEFAULT_BLOCK_SIZE = 256                  # backward.py:48

PRECISION_DTYPES = {"single": np.float32, "double": np.float64}
DTYPE_PRECISIONS = {np.dtype(np.float32): "single", np.dtype(np.float64): "double"}

_DEFAULT_EXACT = True


def set_default_exact(flag: bool) -> None:
    """Choose the policy used when a call does not pass ``exact=``."""
    global _DEFAULT_EXACT
    _DEFAULT_EXACT = bool(flag)


def _exact(flag):
    return _DEFAULT_EXACT if flag is None else bool(flag)


def _device():
    if not torch.cuda.is_available():
        raise UnsupportedError("the GR-KAN B200 shim needs a CUDA device; there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


# ---------------------------------------------------------------------------
# Types (rational.py:31-183, backward.py:51-110)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class GroupLayout:
    """Equal contiguous groups over the feature dim (rational.py:31-55)."""

    feature_dim: int
    num_groups: int

    def __post_init__(self):
        if self.feature_dim < 1 or self.num_groups < 1:
            raise LayoutMismatchError("layout mismatch: dimensions must be positive")
        if self.feature_dim % self.num_groups != 0:
            raise LayoutMismatchError("layout mismatch: feature_dim %d not divisible by num_groups %d"
                                      % (self.feature_dim, self.num_groups))

    @property
    def group_width(self) -> int:
        return self.feature_dim // self.num_groups

    def group_slices(self) -> Iterator[tuple[int, int, int]]:
        w = self.group_width
        for g in range(self.num_groups):
            yield g, g * w, (g + 1) * w


@dataclass(frozen=True)
class GroupRationalParams:
    """numerator (G, m+1) = a_0..a_m; denominator (G, n) = b_1..b_n; stored fp64 (rational.py:58-129)."""

    numerator: np.ndarray
    denominator: np.ndarray

    def __post_init__(self):
        num = np.ascontiguousarray(np.atleast_2d(np.asarray(self.numerator, dtype=np.float64)))
        den = np.asarray(self.denominator, dtype=np.float64)
        if den.ndim == 1:
            den = den.reshape(num.shape[0], -1)
        den = np.ascontiguousarray(den)
        if num.ndim != 2 or den.ndim != 2:
            raise ValueError("coefficient arrays must be 2-D")
        if num.shape[1] < 1:
            raise ValueError("numerator needs at least the constant coefficient")
        if den.shape[0] != num.shape[0]:
            raise ValueError("numerator and denominator group counts differ")
        if not (np.isfinite(num).all() and np.isfinite(den).all()):
            raise NonFiniteInputError("non-finite input: coefficients must be finite")
        object.__setattr__(self, "numerator", num)
        object.__setattr__(self, "denominator", den)

    num_groups = property(lambda self: self.numerator.shape[0])
    num_coeffs = property(lambda self: self.numerator.shape[1])
    den_coeffs = property(lambda self: self.denominator.shape[1])
    degrees = property(lambda self: (self.numerator.shape[1] - 1, self.denominator.shape[1]))
    total_coeffs = property(lambda self: self.numerator.shape[1] + self.denominator.shape[1])

    def group_row(self, g: int):
        return self.numerator[g], self.denominator[g]

    @classmethod
    def identity(cls, num_groups: int, degrees=(5, 4)) -> "GroupRationalParams":
        m, n = degrees
        if m < 1:
            raise ValueError("identity needs numerator degree >= 1")
        num = np.zeros((num_groups, m + 1))
        num[:, 1] = 1.0
        return cls(num, np.zeros((num_groups, n)))

    @classmethod
    def from_row(cls, numerator_row, denominator_row, num_groups: int) -> "GroupRationalParams":
        num = np.tile(np.asarray(numerator_row, dtype=np.float64), (num_groups, 1))
        den = np.tile(np.asarray(denominator_row, dtype=np.float64).reshape(1, -1), (num_groups, 1))
        return cls(num, den)


@dataclass
class ActivationTensor:
    """Dense (batch, seq, feature) host tensor, f32 or f64 (rational.py:132-183)."""

    data: np.ndarray
    validated: bool = field(default=False, repr=False)

    def __post_init__(self):
        arr = np.ascontiguousarray(self.data)
        if arr.ndim != 3:
            raise ValueError("activation tensor must be rank 3 (batch, seq, feature)")
        if arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(np.float64)
        self.data = arr

    @classmethod
    def from_array(cls, arr, validate: bool = True) -> "ActivationTensor":
        t = cls(np.asarray(arr))
        if validate:
            t.check_finite()
        return t

    batch = property(lambda self: self.data.shape[0])
    seq = property(lambda self: self.data.shape[1])
    feature = property(lambda self: self.data.shape[2])
    num_elements = property(lambda self: self.data.size)
    precision = property(lambda self: DTYPE_PRECISIONS[self.data.dtype])

    def check_finite(self) -> "ActivationTensor":
        """Checked mode, evaluated on the device by the forward kernel's finiteness flag."""
        if not self.validated:
            if self.data.size:
                x = torch.from_numpy(self.data).to(_device())
                a, b = _coeffs(GroupRationalParams.identity(1, (1, 0)), x.dtype, x.device)
                ops.rational_forward(x.reshape(-1, 1), a, b, exact=False, check_finite=True)
            self.validated = True
        return self

    def rows(self) -> np.ndarray:
        return self.data.reshape(self.batch * self.seq, self.feature)


@dataclass(frozen=True)
class ExecutionPlan:
    """Grid geometry of one backward pass (backward.py:51-98).

    On the GPU the kernel picks its own tiling; the plan is validated exactly
    as the reference does so the same inputs raise the same errors.
    """

    strategy: str
    block_size: int
    layout: GroupLayout
    grid_rows: int
    grid_cols: int

    def __post_init__(self):
        if self.strategy not in (STRATEGY_NAIVE, STRATEGY_BLOCKED):
            raise ValueError("unknown strategy %r" % (self.strategy,))
        if self.block_size < 1 or self.grid_rows < 1 or self.grid_cols < 1:
            raise GridGeometryError("grid geometry invalid: non-positive dimension")

    @classmethod
    def naive(cls, batch, seq, layout, block_size=DEFAULT_BLOCK_SIZE) -> "ExecutionPlan":
        total = batch * seq * layout.feature_dim
        return cls(STRATEGY_NAIVE, block_size, layout, -(-total // block_size), 1)

    @classmethod
    def blocked(cls, batch, seq, layout, block_size=DEFAULT_BLOCK_SIZE) -> "ExecutionPlan":
        return cls(STRATEGY_BLOCKED, block_size, layout, -(-(batch * seq) // block_size),
                   layout.num_groups)

    def validate_for(self, x: ActivationTensor) -> None:
        if self.strategy == STRATEGY_NAIVE:
            want = (-(-(x.batch * x.seq * x.feature) // self.block_size), 1)
        else:
            want = (-(-(x.batch * x.seq) // self.block_size), self.layout.num_groups)
        if (self.grid_rows, self.grid_cols) != want:
            raise GridGeometryError("grid geometry invalid: plan %dx%d does not tile tensor (want %dx%d)"
                                    % (self.grid_rows, self.grid_cols, want[0], want[1]))


@dataclass
class GradBundle:
    """Backward outputs with provenance (backward.py:101-110)."""

    d_x: ActivationTensor
    d_a: np.ndarray
    d_b: np.ndarray
    strategy: str
    precision: str
    combine_mode: str


@dataclass(frozen=True)
class ElementGrads:
    d_x: float
    d_a: np.ndarray
    d_b: np.ndarray


# ---------------------------------------------------------------------------
# Device plumbing
# ---------------------------------------------------------------------------

def _coeffs(params: GroupRationalParams, tdtype: torch.dtype, device):
    """Coefficients rounded to the tensor dtype, as the reference casts at use (rational.py:220)."""
    np_dt = np.float64 if tdtype == torch.float64 else np.float32
    a = torch.from_numpy(np.ascontiguousarray(params.numerator.astype(np_dt))).to(device)
    b = torch.from_numpy(np.ascontiguousarray(params.denominator.astype(np_dt))).to(device)
    return a, b


_STAGE_BYTES = 32 << 20
# per thread (the reference's functions are safe from concurrent callers):
# device index -> (two pinned staging chunks, copy stream, two events)
_stage_local = threading.local()


def _download(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> a fresh NumPy array, through two pinned staging chunks.

    ``t.cpu()`` into fresh pageable memory runs at ~2 GB/s on the B200 host
    (driver staging + first-touch page faults); here the D2H of chunk k+1
    (56 GB/s pinned) overlaps the host copy of chunk k, so the cost is about the
    host's own first-touch copy rate (~5 GB/s measured, tools/pcie_bw.py).
    """
    nb = t.numel() * t.element_size()
    if nb <= 2 * _STAGE_BYTES:
        return t.cpu().numpy()
    bufs, stream, evs = _stage(t.device)
    dev = t.device
    src = t.contiguous().reshape(-1).view(torch.uint8)
    out = np.empty(t.shape, dtype=torch.empty(0, dtype=t.dtype).numpy().dtype)
    dst = out.reshape(-1).view(np.uint8)
    views = [b.numpy() for b in bufs]
    n = -(-nb // _STAGE_BYTES)
    stream.wait_stream(torch.cuda.current_stream(dev))

    def issue(k):
        lo = k * _STAGE_BYTES
        hi = min(nb, lo + _STAGE_BYTES)
        with torch.cuda.stream(stream):
            bufs[k & 1][: hi - lo].copy_(src[lo:hi], non_blocking=True)
            evs[k & 1].record(stream)

    issue(0)
    for k in range(n):
        if k + 1 < n:
            issue(k + 1)  # its buffer's previous chunk (k - 1) was copied out last iteration
        evs[k & 1].synchronize()
        lo = k * _STAGE_BYTES
        hi = min(nb, lo + _STAGE_BYTES)
        np.copyto(dst[lo:hi], views[k & 1][: hi - lo])
    return out


def check_compatible(x: ActivationTensor, params: GroupRationalParams, layout: GroupLayout) -> None:
    """rational.py:313-322."""
    if x.feature != layout.feature_dim:
        raise LayoutMismatchError("layout mismatch: tensor feature dim %d vs layout %d"
                                  % (x.feature, layout.feature_dim))
    if params.num_groups != layout.num_groups:
        raise LayoutMismatchError("layout mismatch: params have %d groups, layout %d"
                                  % (params.num_groups, layout.num_groups))


def _stage(dev):
    cache = getattr(_stage_local, "by_device", None)
    if cache is None:
        cache = _stage_local.by_device = {}
    if dev.index not in cache:
        cache[dev.index] = ([torch.empty(_STAGE_BYTES, dtype=torch.uint8, pin_memory=True) for _ in range(2)],
                            torch.cuda.Stream(dev), [torch.cuda.Event() for _ in range(2)])
    return cache[dev.index]


def _to_device(t: ActivationTensor):
    """Host array -> device tensor; large arrays go through the pinned staging chunks
    (host copy of chunk k+1 overlaps the H2D of chunk k), small ones directly."""
    dev = _device()
    arr = t.data
    if arr.nbytes <= 2 * _STAGE_BYTES:
        return torch.from_numpy(arr).to(dev, non_blocking=False)
    bufs, stream, evs = _stage(dev)
    out = torch.empty(arr.shape, dtype=torch.from_numpy(arr[:0].reshape(-1)).dtype, device=dev)
    dst = out.reshape(-1).view(torch.uint8)
    src = arr.reshape(-1).view(np.uint8)
    views = [b.numpy() for b in bufs]
    nb = arr.nbytes
    n = -(-nb // _STAGE_BYTES)
    stream.wait_stream(torch.cuda.current_stream(dev))  # `out`'s memory may be reused from that stream
    for k in range(n):
        lo = k * _STAGE_BYTES
        hi = min(nb, lo + _STAGE_BYTES)
        evs[k & 1].synchronize()  # whatever last read this staging chunk (this call or an earlier one) is done
        np.copyto(views[k & 1][: hi - lo], src[lo:hi])
        with torch.cuda.stream(stream):
            dst[lo:hi].copy_(bufs[k & 1][: hi - lo], non_blocking=True)
            evs[k & 1].record(stream)
    torch.cuda.current_stream(dev).wait_stream(stream)
    out.record_stream(stream)
    return out


# ---------------------------------------------------------------------------
# Hot path (rational.py:325-345, backward.py:187-395)
# ---------------------------------------------------------------------------

def _host_ctx():
    """This thread's native host pipeline on the current device (grkan_host_create)."""
    import ctypes

    from . import _native as N

    dev = _device()
    cache = getattr(_stage_local, "host_ctx", None)
    if cache is None:
        cache = _stage_local.host_ctx = {}
    ctx = cache.get(dev.index)
    if ctx is None:
        h = ctypes.c_void_p()
        rc = N.lib().grkan_host_create(dev.index, 0, 0, ctypes.byref(h))
        if rc:
            raise_for_status(rc, N.lib().grkan_host_last_error().decode())
        ctx = cache[dev.index] = _HostCtx(h)
    return ctx.handle


class _HostCtx:
    """Owns one grkan_host_ctx; released with the thread's cache."""

    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        try:
            from . import _native as N

            N.lib().grkan_host_destroy(self.handle)
        except Exception:  # interpreter teardown
            pass


def _host_check(rc: int) -> None:
    if rc:
        from . import _native as N

        raise_for_status(rc, N.lib().grkan_host_last_error().decode())


def _host_flags(exact, check: bool) -> int:
    from . import _native as N

    return (N.FLAG_EXACT if _exact(exact) else N.FLAG_FAST) | (N.FLAG_CHECK_FINITE if check else 0)


_PINNED_MIN_BYTES = 1 << 20


def _output_like(arr: np.ndarray) -> np.ndarray:
    """A fresh output array shaped like ``arr``.  Large ones live in page-locked memory
    from torch's caching host allocator: the pipeline DMAs results straight into them
    (no staging copy, no first-touch page faults), and a dropped output's block is
    reused by the next call."""
    if arr.nbytes < _PINNED_MIN_BYTES:
        return np.empty_like(arr)
    t = torch.empty(arr.shape, dtype=torch.from_numpy(arr.reshape(-1)[:1]).dtype, pin_memory=True)
    return t.numpy()


def _host_coeffs(params: GroupRationalParams, dtype) -> tuple[np.ndarray, np.ndarray]:
    """Coefficients rounded to the tensor dtype, as the reference casts at use (rational.py:220)."""
    return (np.ascontiguousarray(params.numerator, dtype=dtype),
            np.ascontiguousarray(params.denominator, dtype=dtype))


def forward_tensor(x: ActivationTensor, params: GroupRationalParams, layout: GroupLayout,
                   validate: bool = True, exact: bool | None = None) -> ActivationTensor:
    """Group-wise rational of every element; same shape and precision (rational.py:325-345).

    Host arrays in and out through the native pipeline (grkan_host_fwd): host copies,
    PCIe transfers and the sm_100a kernel overlap chunk by chunk."""
    from . import _native as N

    check_compatible(x, params, layout)
    check = validate and not x.validated
    arr = x.data
    y = _output_like(arr)
    a, b = _host_coeffs(params, arr.dtype)
    dt = N.DT_F64 if arr.dtype == np.float64 else N.DT_F32
    rows = x.batch * x.seq
    _host_check(N.lib().grkan_host_fwd(_host_ctx(), arr.ctypes.data, y.ctypes.data, a.ctypes.data,
                                       b.ctypes.data, rows, x.feature, params.num_groups, params.num_coeffs,
                                       params.den_coeffs, dt, _host_flags(exact, check)))
    if check:
        x.validated = True
    return ActivationTensor(y, validated=False)


def _prepare_bwd(x, upstream, params, plan, default_plan):
    layout = plan.layout if plan is not None else GroupLayout(x.feature, params.num_groups)
    if plan is None:
        plan = default_plan(x.batch, x.seq, layout)
    check_compatible(x, params, layout)
    if x.data.shape != upstream.data.shape:
        raise GridGeometryError("grid geometry invalid: x and upstream shapes differ")
    plan.validate_for(x)
    return layout, plan


def _instrumented(x, upstream, params, naive: bool, exact, counter, coverage):
    """counter= / coverage= (backward.py:230-236, 335-351): the same kernels in their
    counting instantiations (grkan_bwd_instrumented).  The kernels tally the accesses
    they perform and mark every element they visit; both are added to the caller's
    counter / coverage array, as the reference's workers do."""
    from . import _native as N

    dev = _device()
    xd, ud = torch.from_numpy(x.data).to(dev), torch.from_numpy(upstream.data).to(dev)
    a, b = _coeffs(params, xd.dtype, xd.device)
    rows, d = x.batch * x.seq, x.feature
    ng, m1, n = params.num_groups, params.num_coeffs, params.den_coeffs
    dx = torch.empty_like(xd)
    da = torch.empty((ng, m1), dtype=a.dtype, device=dev)
    db = torch.empty((ng, n), dtype=a.dtype, device=dev)
    ws = torch.empty(max(256, ops.workspace_bytes(rows, d, ng, m1, n, xd.dtype)), dtype=torch.uint8, device=dev)
    cov = torch.zeros(max(1, rows * d), dtype=torch.int32, device=dev)
    cnt = torch.zeros(3, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        rc = N.lib().grkan_bwd_instrumented(
            xd.data_ptr(), ud.data_ptr(), a.data_ptr(), b.data_ptr() if b.numel() else None, dx.data_ptr(),
            da.data_ptr(), db.data_ptr() if db.numel() else None, ws.data_ptr(), ws.numel(), cov.data_ptr(),
            cnt.data_ptr(), rows, d, ng, m1, n, N.DT_F64 if xd.dtype == torch.float64 else N.DT_F32,
            N.FLAG_EXACT if _exact(exact) else N.FLAG_FAST, 1 if naive else 0,
            torch.cuda.current_stream(dev).cuda_stream)
    if rc:
        raise_for_status(rc, N.last_error())
    ops.read_status(ws[:ops.STATUS_BYTES])  # AccumulationOverflowError (backward.py:182-184)
    if counter is not None:
        r, w, m = (int(v) for v in cnt.cpu().tolist())
        counter.add(reads=r, writes=w, rmw=m)
    if coverage is not None:
        view = coverage.reshape(rows, d)
        view += cov[:rows * d].cpu().numpy().reshape(rows, d).astype(view.dtype)
    return dx.cpu().numpy(), da.cpu().numpy(), db.cpu().numpy()


def backward_blocked(x: ActivationTensor, upstream: ActivationTensor, params: GroupRationalParams,
                     plan: ExecutionPlan | None = None, workers: int = 1,
                     combine_mode: str = COMBINE_ORDERED, validate: bool = True, counter=None,
                     coverage=None, exact: bool | None = None) -> GradBundle:
    """Alg. 2 on the B200: dx in one pass, per-CTA partials, fixed-order fold (backward.py:275-372)."""
    if combine_mode not in (COMBINE_ORDERED, COMBINE_UNORDERED):
        raise ValueError("unknown combine mode %r" % (combine_mode,))
    _prepare_bwd(x, upstream, params, plan, ExecutionPlan.blocked)
    from . import _native as N

    if upstream.data.dtype != x.data.dtype:
        upstream = ActivationTensor(upstream.data.astype(x.data.dtype))
    check = validate and not (x.validated and upstream.validated)
    if counter is not None or coverage is not None:
        if check:
            x.check_finite()
            upstream.check_finite()
        dx, da, db = _instrumented(x, upstream, params, False, exact, counter, coverage)
        return GradBundle(d_x=ActivationTensor(dx), d_a=da, d_b=db, strategy=STRATEGY_BLOCKED,
                          precision=x.precision, combine_mode=combine_mode)
    arr = x.data
    dx = _output_like(arr)
    a, b = _host_coeffs(params, arr.dtype)
    da = np.empty((params.num_groups, params.num_coeffs), dtype=arr.dtype)
    db = np.empty((params.num_groups, params.den_coeffs), dtype=arr.dtype)
    dt = N.DT_F64 if arr.dtype == np.float64 else N.DT_F32
    _host_check(N.lib().grkan_host_bwd(_host_ctx(), arr.ctypes.data, upstream.data.ctypes.data,
                                       a.ctypes.data, b.ctypes.data, dx.ctypes.data, da.ctypes.data,
                                       db.ctypes.data, x.batch * x.seq, x.feature, params.num_groups,
                                       params.num_coeffs, params.den_coeffs, dt, _host_flags(exact, check)))
    if check:
        x.validated = upstream.validated = True
    return GradBundle(d_x=ActivationTensor(dx), d_a=da, d_b=db, strategy=STRATEGY_BLOCKED,
                      precision=x.precision, combine_mode=combine_mode)


def backward_naive(x: ActivationTensor, upstream: ActivationTensor, params: GroupRationalParams,
                   plan: ExecutionPlan | None = None, validate: bool = True, counter=None,
                   coverage=None, exact: bool | None = None) -> GradBundle:
    """The paper's Alg. 1 (per-element atomicAdd), which the reference's naive strategy models
    (backward.py:187-246).  Comparator only; d_x is identical to backward_blocked's."""
    _prepare_bwd(x, upstream, params, plan, ExecutionPlan.naive)
    if validate and not (x.validated and upstream.validated):
        x.check_finite()
        upstream.check_finite()
    if counter is not None or coverage is not None:
        if upstream.data.dtype != x.data.dtype:
            upstream = ActivationTensor(upstream.data.astype(x.data.dtype))
        dx, da, db = _instrumented(x, upstream, params, True, exact, counter, coverage)
        return GradBundle(d_x=ActivationTensor(dx), d_a=da, d_b=db, strategy=STRATEGY_NAIVE,
                          precision=x.precision, combine_mode=COMBINE_ORDERED)
    xd, ud = _to_device(x), _to_device(upstream).to(dtype=torch.float64 if x.precision == "double"
                                                     else torch.float32)
    a, b = _coeffs(params, xd.dtype, xd.device)
    dx, da, db = ops.rational_backward_atomic(xd, ud, a, b, exact=_exact(exact), check_overflow=True)
    return GradBundle(d_x=ActivationTensor(_download(dx)), d_a=da.cpu().numpy(),
                      d_b=db.cpu().numpy(), strategy=STRATEGY_NAIVE, precision=x.precision,
                      combine_mode=COMBINE_ORDERED)


def run_backward(x, upstream, params, plan: ExecutionPlan, workers: int = 1,
                 combine_mode: str = COMBINE_ORDERED, validate: bool = True, counter=None,
                 coverage=None, exact: bool | None = None) -> GradBundle:
    """Dispatch on the plan's strategy tag (backward.py:375-395)."""
    if plan.strategy == STRATEGY_NAIVE:
        return backward_naive(x, upstream, params, plan, validate=validate, counter=counter,
                              coverage=coverage, exact=exact)
    return backward_blocked(x, upstream, params, plan, workers=workers, combine_mode=combine_mode,
                            validate=validate, counter=counter, coverage=coverage, exact=exact)


def combine_partials(partials, num_groups: int, mode: str = COMBINE_ORDERED):
    """Fold per-block partials into per-group totals (backward.py:142-179), on the GPU.

    ``partials``: (block_id, numerator_partials, denominator_partials) with
    block_id = row_block * num_groups + group; every id in 0..len-1 exactly once
    (else PartialCoverageError, as the reference).  The fold is the reference's own:
    ``d_a[g] += pa`` from zeros in ascending block id (``deterministic_ordered``) or
    in the order given (``unordered_scatter``), in the partials' dtype with
    separately rounded adds (grkan_combine_partials) -- bitwise the reference's
    totals, absorption of tiny partials included (test_backward.py:193-209).
    """
    from . import _native as N

    if mode not in (COMBINE_ORDERED, COMBINE_UNORDERED):
        raise ValueError("unknown combine mode %r" % (mode,))
    if not partials:
        raise PartialCoverageError("partial coverage violation: no partials")
    ids = [int(p[0]) for p in partials]
    if sorted(ids) != list(range(len(partials))):
        raise PartialCoverageError("partial coverage violation")
    first_a = np.asarray(partials[0][1])
    first_b = np.asarray(partials[0][2])
    num_w, den_w = first_a.shape[0], first_b.shape[0]
    for _, pa, pb in partials:
        if np.asarray(pa).shape != (num_w,) or np.asarray(pb).shape != (den_w,):
            raise PartialCoverageError("partial coverage violation: inconsistent shapes")
    dtype = first_a.dtype if first_a.dtype in (np.float32, np.float64) else np.dtype(np.float64)
    ordered = sorted(partials, key=lambda p: int(p[0])) if mode == COMBINE_ORDERED else list(partials)
    host = np.zeros((len(ordered), num_w + den_w), dtype=dtype)
    group_of = np.empty(len(ordered), dtype=np.int32)
    for i, (bid, pa, pb) in enumerate(ordered):
        host[i, :num_w] = pa
        host[i, num_w:] = pb
        group_of[i] = int(bid) % num_groups
    dev = _device()
    part = torch.from_numpy(host).to(dev)
    gid = torch.from_numpy(group_of).to(dev)
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    da = torch.empty((num_groups, num_w), dtype=tdt, device=dev)
    db = torch.empty((num_groups, den_w), dtype=tdt, device=dev)
    with torch.cuda.device(dev):
        rc = N.lib().grkan_combine_partials(part.data_ptr(), gid.data_ptr(), len(ordered), num_groups, num_w,
                                            den_w, da.data_ptr() if da.numel() else None,
                                            db.data_ptr() if db.numel() else None,
                                            N.DT_F64 if dtype == np.float64 else N.DT_F32,
                                            torch.cuda.current_stream(dev).cuda_stream)
    if rc:
        raise_for_status(rc, N.last_error())
    return da.cpu().numpy(), db.cpu().numpy()


# ---------------------------------------------------------------------------
# Scalar entry points (rational.py:285-310): one-element fp64 tensors on the GPU
# ---------------------------------------------------------------------------

def _scalar_params(numerator, denominator):
    num = np.asarray(numerator, dtype=np.float64).reshape(1, -1)
    den = np.asarray(denominator, dtype=np.float64).reshape(1, -1)
    return GroupRationalParams(num, den)


def eval_rational(x: float, numerator, denominator, validate: bool = True) -> float:
    if validate and not np.isfinite(x):
        raise NonFiniteInputError("non-finite input")
    t = ActivationTensor(np.array([[[x]]], dtype=np.float64), validated=True)
    y = forward_tensor(t, _scalar_params(numerator, denominator), GroupLayout(1, 1), validate=False,
                       exact=True)
    return float(y.data.reshape(-1)[0])


def elementwise_grads(x: float, upstream: float, numerator, denominator,
                      validate: bool = True) -> ElementGrads:
    if validate and not (np.isfinite(x) and np.isfinite(upstream)):
        raise NonFiniteInputError("non-finite input")
    params = _scalar_params(numerator, denominator)
    t = ActivationTensor(np.array([[[x]]], dtype=np.float64), validated=True)
    u = ActivationTensor(np.array([[[upstream]]], dtype=np.float64), validated=True)
    xd, ud = _to_device(t), _to_device(u)
    a, b = _coeffs(params, xd.dtype, xd.device)
    dx, da, db = ops.rational_backward(xd, ud, a, b, exact=True)
    return ElementGrads(d_x=float(dx.reshape(-1)[0]), d_a=da.cpu().numpy().reshape(-1),
                        d_b=db.cpu().numpy().reshape(-1))


# ---------------------------------------------------------------------------
# Array-level helpers for one coefficient row (rational.py:218-278)
# ---------------------------------------------------------------------------

def _row_arrays(x, numerator, denominator):
    x = np.asarray(x)
    if x.dtype not in (np.float32, np.float64):
        x = x.astype(np.float64)
    dev = _device()
    flat = torch.from_numpy(np.ascontiguousarray(x).reshape(1, -1)).to(dev)
    cd = ops.coeff_dtype(flat.dtype)
    a = torch.as_tensor(np.asarray(numerator, dtype=x.dtype).reshape(1, -1), dtype=cd, device=dev)
    b = torch.as_tensor(np.asarray(denominator, dtype=x.dtype).reshape(1, -1), dtype=cd, device=dev)
    return x, flat, a, b


def rational_values(x: np.ndarray, numerator, denominator, exact: bool | None = None) -> np.ndarray:
    """P(x) / Q(x) for one coefficient row, in x.dtype (rational.py:218-224)."""
    x, flat, a, b = _row_arrays(x, numerator, denominator)
    if flat.numel() == 0:
        return np.empty_like(x)
    y = ops.rational_forward(flat, a, b, exact=_exact(exact))
    return _download(y).reshape(x.shape)


def gradient_terms(x: np.ndarray, upstream: np.ndarray, numerator, denominator, exact: bool | None = None):
    """(d_x, da_terms, db_terms) per element for one coefficient row (rational.py:227-278).

    Unreduced: da_terms[i] = u x^i / Q, db_terms[j] = -u sign(A) x^(j+1) P / Q^2,
    in x.dtype.  EXACT (the shim's default) gives the reference's terms bit for
    bit (grkan_bwd_terms).
    """
    x, flat, a, b = _row_arrays(x, numerator, denominator)
    up = np.asarray(upstream, dtype=x.dtype)
    if up.shape != x.shape:
        raise GridGeometryError("grid geometry invalid: x and upstream shapes differ")
    m1, n = a.shape[1], b.shape[1]
    if flat.numel() == 0:
        return np.empty_like(x), [np.empty_like(x) for _ in range(m1)], [np.empty_like(x) for _ in range(n)]
    u = torch.from_numpy(np.ascontiguousarray(up).reshape(1, -1)).to(flat.device)
    dx = torch.empty_like(flat)
    terms = torch.empty((m1 + n, flat.numel()), dtype=a.dtype, device=flat.device)
    from . import _native as N
    with torch.cuda.device(flat.device):
        rc = N.lib().grkan_bwd_terms(flat.data_ptr(), u.data_ptr(), a.data_ptr(), b.data_ptr(), dx.data_ptr(),
                                     terms.data_ptr(), 1, flat.numel(), 1, m1, n, ops._DT[flat.dtype],
                                     N.FLAG_EXACT if _exact(exact) else N.FLAG_FAST,
                                     ops._stream(flat.device))
        ops._raise(rc)
    t = terms.cpu().numpy().astype(x.dtype, copy=False)
    shape = x.shape
    return (dx.cpu().numpy().reshape(shape), [t[i].reshape(shape) for i in range(m1)],
            [t[m1 + j].reshape(shape) for j in range(n)])


# ---------------------------------------------------------------------------
# GRKB dumps (cli.py:104-129)
# ---------------------------------------------------------------------------

def write_tensor_dump(path: str, tensor: ActivationTensor) -> None:
    from . import grkb
    grkb.save(path, tensor.data)


def read_tensor_dump(path: str) -> ActivationTensor:
    from . import grkb
    return ActivationTensor(grkb.load(path))

