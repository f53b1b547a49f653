"""Global-memory access model of the B200 path, next to the reference's.

The reference models the backward's cost as element-sized global accesses
(`pkg/src/grkan/access.py:1-18`): an element load or store counts 1, an atomic
add counts a read plus a write.  Its closed forms:

* naive (Alg. 1):  3 * (m_c + 1) * E                              (access.py:89-94)
* blocked (Alg. 2): 3 * E + 3 * m_c * grid_rows * n_groups         (access.py:97-126)

with E = rows * d and m_c = m1 + n coefficients per group.  This module
restates them (same names, same argument checks) and adds what the B200
kernels actually move, in BYTES, so the ncu DRAM counters can be read against
both (`tools/access_ncu.py` -> `profiles/r1/access_model_vs_ncu.json`):

* K1 forward:   read x, write y                                    2 s E
* K2 + K3:      read x, dy; write dx                               3 s E
                + per-(warp-partial, coefficient) fp32 partials written by
                K2 and read once by K3, + m_c * n_groups results;
                coefficients are read once per CTA (L2 hits).
* K4 (Alg. 1 comparator): the same 3 s E of tensor traffic, plus m_c * E
                atomic adds that resolve in L2 (they are RMWs in the
                reference's model, but not DRAM bytes on the device).

Host-side arithmetic only; no kernels run here.
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

from . import _native as N

_DT = {"fp32": (N.DT_F32, 4, 4), "bf16": (N.DT_BF16, 2, 4), "fp64": (N.DT_F64, 8, 8)}


class TailNotCoveredError(ValueError):
    """The blocked closed form needs exact tiling (access.py:110-111)."""


def _require_positive(**kwargs: int) -> None:
    for name, value in kwargs.items():
        if int(value) != value or value < 1:
            raise ValueError("%s must be a positive integer, got %r" % (name, value))


def predict_accesses_naive(batch: int, seq: int, feature: int, m_coeffs: int) -> int:
    """Reference naive model (access.py:89-94): 3 * (m_coeffs + 1) * E."""
    _require_positive(batch=batch, seq=seq, feature=feature)
    if m_coeffs < 0:
        raise ValueError("m_coeffs must be non-negative")
    return 3 * (m_coeffs + 1) * batch * seq * feature


def predict_accesses_blocked(batch: int, seq: int, feature: int, block_size: int, group_width: int,
                             m_coeffs: int) -> int:
    """Reference blocked model under exact tiling (access.py:97-116)."""
    _require_positive(batch=batch, seq=seq, feature=feature, block_size=block_size, group_width=group_width)
    if m_coeffs < 0:
        raise ValueError("m_coeffs must be non-negative")
    if feature % group_width != 0 or (batch * seq) % block_size != 0:
        raise TailNotCoveredError("tail not covered by closed form")
    e = batch * seq * feature
    exact = 3 * e + 3 * m_coeffs * ((batch * seq) // block_size) * (feature // group_width)
    assert 3 * (Fraction(m_coeffs, block_size * group_width) + 1) * e == exact
    return exact


def predicted_total_for_plan(batch: int, seq: int, feature: int, block_size: int, num_groups: int,
                             m_coeffs: int, naive: bool = False) -> int:
    """Tail-aware reference prediction (access.py:119-126); `block_size` is the plan's."""
    if naive:
        return predict_accesses_naive(batch, seq, feature, m_coeffs)
    grid_rows = -(-(batch * seq) // block_size)
    return 3 * batch * seq * feature + 3 * m_coeffs * grid_rows * num_groups


@dataclass(frozen=True)
class DeviceTraffic:
    """Modelled global traffic of one B200 pass, in bytes (and L2 atomics)."""

    kernel: str
    tensor_bytes: int      # x / dy / y / dx streams
    partial_bytes: int     # K2 partial stores + K3 partial loads + da/db stores
    atomics: int           # element atomic adds (K4 only; resolve in L2)
    reference_accesses: int  # the reference model's count for the same pass
    reference_bytes: int     # reference_accesses x element size

    @property
    def total_bytes(self) -> int:
        return self.tensor_bytes + self.partial_bytes


def device_traffic(rows: int, d: int, n_groups: int, dtype: str = "fp32", kernel: str = "bwd",
                   m1: int = 6, n: int = 4, block_size: int = 256) -> DeviceTraffic:
    """Bytes the B200 kernels move for one pass, with the reference model beside them.

    kernel: "fwd" (K1), "bwd" (K2 + K3) or "bwd_atomic" (K4).  `block_size` is
    the reference plan's row block for its blocked prediction.
    """
    if kernel not in ("fwd", "bwd", "bwd_atomic"):
        raise ValueError("kernel must be fwd, bwd or bwd_atomic")
    if dtype not in _DT:
        raise ValueError("dtype must be one of %s" % sorted(_DT))
    _require_positive(rows=rows, d=d, n_groups=n_groups)
    code, es, acc = _DT[dtype]
    e = rows * d
    mc = m1 + n
    if kernel == "fwd":
        # the reference's forward reads x and writes y once (rational.py:325-345)
        return DeviceTraffic("fwd", 2 * es * e, 0, 0, 2 * e, 2 * es * e)
    if kernel == "bwd_atomic":
        ref = predict_accesses_naive(1, rows, d, mc)
        return DeviceTraffic("bwd_atomic", 3 * es * e, 0, mc * e, ref, ref * es)
    p = N.plan(rows, d, n_groups, m1, n, code)
    parts = p["partials_per_group"] * n_groups * mc
    partial_bytes = 2 * parts * acc + n_groups * mc * acc  # K2 store, K3 load, da/db store
    ref = predicted_total_for_plan(1, rows, d, block_size, n_groups, mc)
    return DeviceTraffic("bwd", 3 * es * e, partial_bytes, 0, ref, ref * es)
