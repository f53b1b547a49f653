"""Error taxonomy, mirroring the reference's (pkg/src/grkan/errors.py:4-37).

Same class names and hierarchy, so code written against ``grkan`` catches the
same exceptions.  ``raise_for_status`` maps C-ABI status codes onto them.
"""

from __future__ import annotations


class GrkanError(Exception):
    """Base class for all package-specific errors (errors.py:4)."""


class LayoutMismatchError(GrkanError):
    """Tensor feature dimension does not match the group layout (errors.py:8)."""


class GridGeometryError(GrkanError):
    """Execution plan grid does not tile the tensor it was applied to (errors.py:12)."""


class PartialCoverageError(GrkanError):
    """A block partial is missing or duplicated in a combine step (errors.py:16)."""


class AccumulationOverflowError(GrkanError):
    """A coefficient-gradient accumulator became non-finite (errors.py:20)."""


class NonFiniteInputError(GrkanError):
    """A checked-mode input contained NaN or infinity (errors.py:24)."""


class DegenerateAlphaError(GrkanError):
    """Kept for API parity (errors.py:28); raised by no hot-path function."""


class TailNotCoveredError(GrkanError):
    """Kept for API parity (errors.py:32); raised by no hot-path function."""


class ActivationFitError(GrkanError):
    """Kept for API parity (errors.py:36); raised by no hot-path function."""


class UnsupportedError(GrkanError):
    """A dtype / degree / device this B200 build does not provide."""


class CudaError(GrkanError):
    """A CUDA runtime call inside the library failed."""


class PeerExchangeTimeoutError(CudaError):
    """grkan_bwd_p2p: a peer rank never arrived at the da/db exchange (bounded wait expired)."""


def raise_for_status(code: int, message: str = "") -> None:
    from . import _native as N

    if code == N.OK:
        return
    cls = {
        N.ERR_LAYOUT: LayoutMismatchError,
        N.ERR_GRID: GridGeometryError,
        N.ERR_NONFINITE_INPUT: NonFiniteInputError,
        N.ERR_ACCUM_OVERFLOW: AccumulationOverflowError,
        N.ERR_UNSUPPORTED: UnsupportedError,
        N.ERR_CUDA: CudaError,
        N.ERR_INVALID: ValueError,
        N.ERR_PEER_TIMEOUT: PeerExchangeTimeoutError,
    }.get(code, GrkanError)
    raise cls(message or "grkan status %d" % code)
