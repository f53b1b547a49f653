"""ctypes wrapper for the C oracle (oracle/grkan_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use it.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        p = ctypes.c_void_p
        i64, i32 = ctypes.c_int64, ctypes.c_int32
        for suf in ("f", "dbl"):
            fwd = getattr(L, "orc_fwd_" + suf)
            fwd.argtypes = [p, p, p, p, i64, i32, i32, i32, i32]
            fwd.restype = None
            bwd = getattr(L, "orc_bwd_" + suf)
            bwd.argtypes = [p, p, p, p, i64, i32, i32, i32, i32, i64] + [p] * 9
            bwd.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def _suffix(dtype):
    if dtype == np.float32:
        return "f"
    if dtype == np.float64:
        return "dbl"
    raise TypeError("oracle supports float32/float64, got %s" % dtype)


def forward(x: np.ndarray, num: np.ndarray, den: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x)
    num = np.ascontiguousarray(num, dtype=np.float64)
    den = np.ascontiguousarray(den, dtype=np.float64).reshape(num.shape[0], -1)
    y = np.empty_like(x)
    d = x.shape[-1]
    getattr(lib(), "orc_fwd_" + _suffix(x.dtype))(
        _ptr(x), _ptr(y), _ptr(num), _ptr(den), x.size // d, d, num.shape[0], num.shape[1],
        den.shape[1])
    return y


def backward(x, u, num, den, block_size=256, want=("dx", "blocked", "naive", "ref64", "true64")):
    """Returns a dict with any of: dx, blocked_da/db, naive_da/db, ref64_da/db, true64_da/db,
    and 'overflow' (True when the reference would raise AccumulationOverflowError)."""
    x = np.ascontiguousarray(x)
    u = np.ascontiguousarray(u, dtype=x.dtype)
    num = np.ascontiguousarray(num, dtype=np.float64)
    den = np.ascontiguousarray(den, dtype=np.float64).reshape(num.shape[0], -1)
    ng, m1, n = num.shape[0], num.shape[1], den.shape[1]
    d = x.shape[-1]
    out = {}
    if "dx" in want:
        out["dx"] = np.empty_like(x)
    for k, dt in (("blocked", x.dtype), ("naive", x.dtype), ("ref64", np.float64),
                  ("true64", np.float64)):
        if k in want:
            out[k + "_da"] = np.zeros((ng, m1), dtype=dt)
            out[k + "_db"] = np.zeros((ng, n), dtype=dt)
    g = out.get
    bad = getattr(lib(), "orc_bwd_" + _suffix(x.dtype))(
        _ptr(x), _ptr(u), _ptr(num), _ptr(den), x.size // d, d, ng, m1, n, int(block_size),
        _ptr(g("dx")), _ptr(g("blocked_da")), _ptr(g("blocked_db")), _ptr(g("naive_da")),
        _ptr(g("naive_db")), _ptr(g("ref64_da")), _ptr(g("ref64_db")), _ptr(g("true64_da")),
        _ptr(g("true64_db")))
    out["overflow"] = bool(bad)
    return out
