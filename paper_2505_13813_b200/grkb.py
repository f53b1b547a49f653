"""GRKB tensor dumps: the reference CLI's wire format for cross-checking results.

Format (pkg/src/grkan/cli.py:52-54, 104-129): 4-byte magic ``GRKB``, u32
version 1, u8 dtype code (0 = float32, 1 = float64), three u64 dims
(batch, seq, feature), then the little-endian row-major element stream.
``grkan bench --dump`` writes dx in this format; ``save``/``load`` let GPU
results be written and compared byte for byte.
"""

from __future__ import annotations

import struct

import numpy as np

MAGIC = b"GRKB"
VERSION = 1
CODES = {np.dtype(np.float32): 0, np.dtype(np.float64): 1}
DTYPES = {0: "<f4", 1: "<f8"}


def dumps(arr) -> bytes:
    """Serialise a rank-3 float32/float64 array (numpy, or a torch tensor on any device)."""
    if hasattr(arr, "detach"):  # torch.Tensor
        arr = arr.detach().cpu().numpy()
    arr = np.asarray(arr)
    if arr.ndim != 3:
        raise ValueError("GRKB dumps hold rank-3 (batch, seq, feature) tensors")
    if arr.dtype not in CODES:
        raise ValueError("GRKB dumps hold float32 or float64, got %s" % arr.dtype)
    code = CODES[arr.dtype]
    head = struct.pack("<4sIB", MAGIC, VERSION, code) + struct.pack("<3Q", *arr.shape)
    return head + np.ascontiguousarray(arr, dtype=DTYPES[code]).tobytes(order="C")


def loads(blob: bytes) -> np.ndarray:
    magic, version, code = struct.unpack("<4sIB", blob[:9])
    if magic != MAGIC:
        raise ValueError("not a tensor dump (bad magic %r)" % (magic,))
    if version != VERSION:
        raise ValueError("unsupported dump version %d" % version)
    if code not in DTYPES:
        raise ValueError("unknown dtype code %d" % code)
    dims = struct.unpack("<3Q", blob[9:33])
    data = np.frombuffer(blob[33:], dtype=DTYPES[code])
    if data.size != dims[0] * dims[1] * dims[2]:
        raise ValueError("payload holds %d elements, header says %s" % (data.size, dims))
    return data.reshape(dims).astype(data.dtype.newbyteorder("="))


def save(path: str, arr) -> None:
    with open(path, "wb") as fh:
        fh.write(dumps(arr))


def load(path: str) -> np.ndarray:
    with open(path, "rb") as fh:
        return loads(fh.read())
