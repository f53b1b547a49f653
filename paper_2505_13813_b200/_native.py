"""Loader for the in-tree C-ABI library ``_lib/libgrkan_b200.so`` (include/grkan_b200.h).

The library is the product: there is no Python or CPU fallback.  If it is
missing or fails to load, every entry point raises ``NativeLibraryError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# GRKAN_LIB points at an alternative build (tuning variants from tools/build_variant.py)
LIB_PATH = os.environ.get("GRKAN_LIB") or os.path.join(HERE, "_lib", "libgrkan_b200.so")

# Status codes and flags (include/grkan_b200.h)
OK = 0
ERR_LAYOUT = 1
ERR_GRID = 2
ERR_NONFINITE_INPUT = 3
ERR_ACCUM_OVERFLOW = 4
ERR_UNSUPPORTED = 5
ERR_CUDA = 6
ERR_INVALID = 7
ERR_PEER_TIMEOUT = 8

DT_F32 = 0
DT_F64 = 1
DT_BF16 = 2

FLAG_FAST = 0
FLAG_EXACT = 1
FLAG_CHECK_FINITE = 2
FLAG_DETERMINISTIC = 4

MAX_M1 = 12
MAX_N = 12

EXPORTS = (
    "grkan_version", "grkan_status_string", "grkan_last_error", "grkan_fwd",
    "grkan_bwd_workspace_bytes", "grkan_bwd", "grkan_bwd_atomic", "grkan_read_status",
    "grkan_plan", "grkan_det_block_rows", "grkan_det_partials_bytes", "grkan_bwd_partials",
    "grkan_reduce_partials", "grkan_linear_bwd_workspace_bytes", "grkan_linear_bwd",
    "grkan_p2p_buffer_bytes", "grkan_p2p_alloc", "grkan_p2p_free", "grkan_ipc_get_handle",
    "grkan_ipc_open_handle", "grkan_ipc_close_handle", "grkan_bwd_p2p", "grkan_bwd_terms",
    "grkan_host_create", "grkan_host_destroy", "grkan_host_threads", "grkan_host_last_error",
    "grkan_host_fwd", "grkan_host_bwd", "grkan_combine_partials", "grkan_bwd_instrumented",
    "grkan_launch_ctas", "grkan_fwd_bwd",
)
IPC_HANDLE_BYTES = 64


class NativeLibraryError(RuntimeError):
    """The CUDA extension is missing or unusable (no fallback exists)."""


class DeviceStatus(ctypes.Structure):
    _fields_ = [("nonfinite_input", ctypes.c_int32), ("accum_overflow", ctypes.c_int32),
                ("peer_timeout", ctypes.c_int32), ("reserved", ctypes.c_int32)]


_lib = None
_lock = threading.Lock()


def _declare(L):
    p, i32, i64, u32, sz = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32,
                            ctypes.c_size_t)
    L.grkan_version.argtypes = []
    L.grkan_version.restype = ctypes.c_char_p
    L.grkan_status_string.argtypes = [ctypes.c_int]
    L.grkan_status_string.restype = ctypes.c_char_p
    L.grkan_last_error.argtypes = []
    L.grkan_last_error.restype = ctypes.c_char_p
    L.grkan_fwd.argtypes = [p, p, p, p, i64, i32, i32, i32, i32, i32, u32, p, p]
    L.grkan_fwd.restype = ctypes.c_int
    L.grkan_bwd_workspace_bytes.argtypes = [i64, i32, i32, i32, i32, i32]
    L.grkan_bwd_workspace_bytes.restype = sz
    L.grkan_bwd.argtypes = [p, p, p, p, p, p, p, p, sz, i64, i32, i32, i32, i32, i32, u32, p]
    L.grkan_bwd.restype = ctypes.c_int
    L.grkan_bwd_atomic.argtypes = [p, p, p, p, p, p, p, i64, i32, i32, i32, i32, i32, u32, p, p]
    L.grkan_bwd_atomic.restype = ctypes.c_int
    L.grkan_read_status.argtypes = [p, p, ctypes.POINTER(DeviceStatus)]
    L.grkan_read_status.restype = ctypes.c_int
    L.grkan_plan.argtypes = [i64, i32, i32, i32, i32, i32, ctypes.POINTER(ctypes.c_int64)]
    L.grkan_plan.restype = ctypes.c_int
    L.grkan_det_block_rows.argtypes = [i32, i32, i32]
    L.grkan_det_block_rows.restype = i64
    L.grkan_det_partials_bytes.argtypes = [i64, i32, i32, i32, i32, i32]
    L.grkan_det_partials_bytes.restype = sz
    L.grkan_bwd_partials.argtypes = [p, p, p, p, p, p, sz, i64, i32, i32, i32, i32, i32, u32, p, p]
    L.grkan_bwd_partials.restype = ctypes.c_int
    L.grkan_reduce_partials.argtypes = [p, i64, i32, i32, i32, p, p, i32, p, p]
    L.grkan_reduce_partials.restype = ctypes.c_int
    L.grkan_linear_bwd_workspace_bytes.argtypes = [i64, i32, i32, i32]
    L.grkan_linear_bwd_workspace_bytes.restype = sz
    L.grkan_linear_bwd.argtypes = [p, p, p, p, p, p, p, p, p, sz, i64, i32, i32, i32, u32, p]
    L.grkan_linear_bwd.restype = ctypes.c_int
    L.grkan_p2p_buffer_bytes.argtypes = [i32, i32, i32, i32]
    L.grkan_p2p_buffer_bytes.restype = sz
    L.grkan_p2p_alloc.argtypes = [sz, ctypes.POINTER(ctypes.c_void_p)]
    L.grkan_p2p_alloc.restype = ctypes.c_int
    L.grkan_p2p_free.argtypes = [p]
    L.grkan_p2p_free.restype = ctypes.c_int
    L.grkan_ipc_get_handle.argtypes = [p, p]
    L.grkan_ipc_get_handle.restype = ctypes.c_int
    L.grkan_ipc_open_handle.argtypes = [p, ctypes.POINTER(ctypes.c_void_p)]
    L.grkan_ipc_open_handle.restype = ctypes.c_int
    L.grkan_ipc_close_handle.argtypes = [p]
    L.grkan_ipc_close_handle.restype = ctypes.c_int
    L.grkan_bwd_p2p.argtypes = [p, p, p, p, p, p, p, p, sz, i64, i32, i32, i32, i32, i32, u32, p, i32, i32,
                                ctypes.c_uint64, p]
    L.grkan_bwd_p2p.restype = ctypes.c_int
    L.grkan_bwd_terms.argtypes = [p, p, p, p, p, p, i64, i32, i32, i32, i32, i32, u32, p]
    L.grkan_bwd_terms.restype = ctypes.c_int
    L.grkan_bwd_instrumented.argtypes = [p, p, p, p, p, p, p, p, sz, p, p, i64, i32, i32, i32, i32, i32, u32, i32, p]
    L.grkan_bwd_instrumented.restype = ctypes.c_int
    L.grkan_fwd_bwd.argtypes = [p, p, p, p, p, p, p, p, p, sz, i64, i32, i32, i32, i32, i32, u32, p]
    L.grkan_fwd_bwd.restype = ctypes.c_int
    L.grkan_launch_ctas.argtypes = [i64, i32, i32, i32, i32, i32, i32]
    L.grkan_launch_ctas.restype = i64
    L.grkan_combine_partials.argtypes = [p, p, i64, i32, i32, i32, p, p, i32, p]
    L.grkan_combine_partials.restype = ctypes.c_int
    L.grkan_host_create.argtypes = [i32, sz, i32, ctypes.POINTER(ctypes.c_void_p)]
    L.grkan_host_create.restype = ctypes.c_int
    L.grkan_host_destroy.argtypes = [p]
    L.grkan_host_destroy.restype = ctypes.c_int
    L.grkan_host_threads.argtypes = [p]
    L.grkan_host_threads.restype = ctypes.c_int
    L.grkan_host_last_error.argtypes = []
    L.grkan_host_last_error.restype = ctypes.c_char_p
    L.grkan_host_fwd.argtypes = [p, p, p, p, p, i64, i32, i32, i32, i32, i32, u32]
    L.grkan_host_fwd.restype = ctypes.c_int
    L.grkan_host_bwd.argtypes = [p, p, p, p, p, p, p, p, i64, i32, i32, i32, i32, i32, u32]
    L.grkan_host_bwd.restype = ctypes.c_int


def lib():
    """The loaded library (loads on first use; raises NativeLibraryError if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryError(
                    "GR-KAN CUDA library not built: %s is missing "
                    "(run `python -c 'import __graft_entry__ as g; g.build()'`)" % LIB_PATH)
            try:
                L = ctypes.CDLL(LIB_PATH)
            except OSError as exc:
                raise NativeLibraryError("cannot load %s: %s" % (LIB_PATH, exc)) from exc
            for sym in EXPORTS:
                if not hasattr(L, sym):
                    raise NativeLibraryError("%s does not export %s" % (LIB_PATH, sym))
            _declare(L)
            _lib = L
    return _lib


def version() -> str:
    return lib().grkan_version().decode()


def status_string(code: int) -> str:
    return lib().grkan_status_string(code).decode()


def last_error() -> str:
    return lib().grkan_last_error().decode()


def plan(rows, d, n_groups, m1, n, dtype_code):
    out = (ctypes.c_int64 * 6)()
    rc = lib().grkan_plan(rows, d, n_groups, m1, n, dtype_code, out)
    if rc:
        from .errors import raise_for_status
        raise_for_status(rc, last_error())
    return {"vector_width": out[0], "threads": out[1], "rows_per_unit": out[2],
            "partials_per_group": out[3], "ctas": out[4], "staged": bool(out[5])}
