"""B200-native GR-KAN group-rational activation (FlashKAT hot path, arXiv 2505.13813).

Layers:
  csrc/               sm_100a CUDA kernels + the C ABI (include/grkan_b200.h)
  _native             ctypes binding of _lib/libgrkan_b200.so (no fallback)
  ops                 torch entry points + torch.library ops
  module              GroupRationalFn (autograd) and GroupRational (nn.Module)
  grkan               reference-API shim (forward_tensor / backward_blocked / ...)
  layer               the layer around it (GrKanLayer, layer_forward / layer_backward)
  parallel            data-parallel glue: row sharding + da/db all-reduce
"""

from . import _native  # noqa: F401
from .errors import (  # noqa: F401
    AccumulationOverflowError,
    GridGeometryError,
    GrkanError,
    LayoutMismatchError,
    NonFiniteInputError,
    PartialCoverageError,
    UnsupportedError,
)

__version__ = "0.1.0"


def __getattr__(name):
    # torch-dependent modules load lazily so `import paper_2505_13813_b200` stays cheap
    if name in ("ops", "module", "grkan", "layer", "parallel", "presets"):
        import importlib

        return importlib.import_module("." + name, __name__)
    if name in ("GroupRational", "GroupRationalFn", "group_rational"):
        from . import module

        return getattr(module, name)
    if name in ("rational_forward", "rational_backward", "rational_backward_atomic"):
        from . import ops

        return getattr(ops, name)
    raise AttributeError(name)
