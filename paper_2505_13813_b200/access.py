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

``AccessCounter`` / ``AccessReport`` / ``instrumented_backward`` mirror the
reference's instrumentation (access.py:36-80, 129-161) on the device: the counts
and the per-element coverage come from the kernels themselves
(grkan_bwd_instrumented), and the prediction is the B200 closed form
``predicted_device_accesses`` (one coefficient-row load per CTA, one partial per
CTA or warp, K3's fold), next to the reference's own model for the same pass.
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


@dataclass
class AccessCounter:
    """Mutable tally of modelled accesses (access.py:36-52)."""

    reads: int = 0
    writes: int = 0
    rmw_atomic: int = 0

    def add(self, reads: int = 0, writes: int = 0, rmw: int = 0) -> None:
        self.reads += reads
        self.writes += writes
        self.rmw_atomic += rmw

    @property
    def total(self) -> int:
        return self.reads + self.writes


@dataclass(frozen=True)
class AccessReport:
    """Instrumented access counts next to the closed-form prediction (access.py:55-80).

    ``predicted_total`` is the B200 kernels' closed form (predicted_device_accesses);
    ``reference_predicted_total`` the reference's model of the same plan."""

    reads: int
    writes: int
    rmw_atomic: int
    total: int
    predicted_total: int
    strategy: str
    reference_predicted_total: int = 0

    @property
    def matches_prediction(self) -> bool:
        return self.total == self.predicted_total

    def to_dict(self) -> dict:
        return {"reads": self.reads, "writes": self.writes, "rmw_atomic": self.rmw_atomic, "total": self.total,
                "predicted_total": self.predicted_total, "strategy": self.strategy,
                "reference_predicted_total": self.reference_predicted_total}


def predicted_device_accesses(rows: int, d: int, n_groups: int, m1: int = 6, n: int = 4, dtype: str = "fp32",
                              naive: bool = False) -> tuple[int, int, int]:
    """(reads, writes, rmw) element accesses of one B200 backward, in the reference's units.

    blocked (K2 + K3): x, dy read and dx written once per element; one coefficient-row
    load per K2 CTA; m_c partial stores per partial slot (one per CTA, or per consumer
    warp in the staged kernel), all read back once by K3, which stores m_c * n_groups
    results.  naive (K4, Alg. 1): x, dy, dx per element plus m_c atomic adds per
    element (1 read + 1 write + 1 rmw each), one coefficient-row load per CTA.
    """
    code = _DT[dtype][0]
    mc = m1 + n
    e = rows * d
    if naive:
        ctas = N.lib().grkan_launch_ctas(rows, d, n_groups, m1, n, code, 2)
        return e * (2 + mc) + mc * ctas, e * (1 + mc), e * mc
    ctas = N.lib().grkan_launch_ctas(rows, d, n_groups, m1, n, code, 1)
    parts = N.plan(rows, d, n_groups, m1, n, code)["partials_per_group"] * n_groups
    return 2 * e + mc * ctas + mc * parts, e + mc * parts + mc * n_groups, 0


def instrumented_backward(x, upstream, params, plan, workers: int = 1, combine_mode: str = "deterministic_ordered",
                          validate: bool = True, exact: bool | None = None):
    """Run the plan's strategy on the GPU while the kernels count every modelled global
    access and mark every element they visit (access.py:129-161).  Raises
    PartialCoverageError unless every element was visited exactly once."""
    import numpy as np

    from . import grkan as G
    from .errors import PartialCoverageError

    counter = AccessCounter()
    coverage = np.zeros((x.batch * x.seq, x.feature), dtype=np.int16)
    bundle = G.run_backward(x, upstream, params, plan, workers=workers, combine_mode=combine_mode,
                            validate=validate, counter=counter, coverage=coverage, exact=exact)
    if not np.all(coverage == 1):
        raise PartialCoverageError("partial coverage violation: element visited != 1 times")
    naive = plan.strategy == G.STRATEGY_NAIVE
    dt = "fp64" if x.data.dtype == np.float64 else "fp32"
    if x.batch * x.seq == 0:
        predicted = 0
    else:
        predicted = sum(predicted_device_accesses(x.batch * x.seq, x.feature, params.num_groups, params.num_coeffs,
                                                  params.den_coeffs, dt, naive)[:2])
    ref = predicted_total_for_plan(x.batch, x.seq, x.feature, plan.block_size, params.num_groups,
                                   params.total_coeffs, naive=naive) if x.batch * x.seq else 0
    report = AccessReport(reads=counter.reads, writes=counter.writes, rmw_atomic=counter.rmw_atomic,
                          total=counter.total, predicted_total=predicted, strategy=plan.strategy,
                          reference_predicted_total=ref)
    return bundle, report


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
