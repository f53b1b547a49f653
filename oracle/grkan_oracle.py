"""CPU oracle for the GR-KAN group-rational hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in NumPy, the reference algorithm of the FlashKAT
artifact (``grkan``; /root/reference/pkg/src/grkan).  It is the *checker*:
only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` leg of ``bench.py`` may import it.  Nothing in the
product package (``paper_2505_13813_b200``) imports or calls it, and the
product path never falls back to it.

Parity pinning: every public function here is checked bit-for-bit against the
golden fixtures that ``tests/golden/make_golden.py`` recorded from the real
reference (``tests/test_oracle_golden.py``).

Op order is the reference's: every ``*``, ``+``, ``/``
is a separate NumPy ufunc call, so each is rounded on its own in the tensor
dtype (no FMA contraction); coefficients are rounded fp64 -> tensor dtype
before use.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

DEFAULT_BLOCK_SIZE = 256  # pkg/src/grkan/backward.py:48


# ---------------------------------------------------------------------------
# Elementwise math (pkg/src/grkan/rational.py:195-278)
# ---------------------------------------------------------------------------

def horner(coeffs: np.ndarray, x: np.ndarray) -> np.ndarray:
    """sum_k c_k x^k, top coefficient first; rational.py:195-200."""
    out = np.full(x.shape, coeffs[-1], dtype=x.dtype)
    for k in range(coeffs.shape[0] - 2, -1, -1):
        out = out * x
        out = out + coeffs[k]
    return out


def derivative(coeffs: np.ndarray) -> np.ndarray:
    """[1*c_1, 2*c_2, ...] in the coefficient dtype; rational.py:203-208."""
    if coeffs.shape[0] < 2:
        return np.zeros(1, dtype=coeffs.dtype)
    return coeffs[1:] * np.arange(1, coeffs.shape[0], dtype=coeffs.dtype)


def series(den: np.ndarray, x: np.ndarray) -> np.ndarray:
    """A(x) = (b_1 + b_2 x + ...) * x, zero for n == 0; rational.py:211-215."""
    if den.shape[0] == 0:
        return np.zeros(x.shape, dtype=x.dtype)
    return horner(den, x) * x


def rational(x: np.ndarray, num, den) -> np.ndarray:
    """y = P(x) / (1 + |A(x)|); rational.py:218-224."""
    a = np.asarray(num, dtype=x.dtype)
    b = np.asarray(den, dtype=x.dtype)
    return horner(a, x) / (1.0 + np.abs(series(b, x)))


def element_terms(x: np.ndarray, u: np.ndarray, num, den):
    """(dx, [m+1 numerator terms], [n denominator terms]); rational.py:227-278."""
    a = np.asarray(num, dtype=x.dtype)
    b = np.asarray(den, dtype=x.dtype)
    p = horner(a, x)
    s = series(b, x)
    q = 1.0 + np.abs(s)
    sg = np.sign(s)
    iq = 1.0 / q
    dp = horner(derivative(a), x)
    if b.shape[0]:
        ds = horner(derivative(np.concatenate(([x.dtype.type(0)], b))), x)
    else:
        ds = np.zeros(x.shape, dtype=x.dtype)
    pq = p * iq
    dx = u * (dp * iq - (sg * ds) * pq * iq)
    ta = [u * iq]
    while len(ta) < a.shape[0]:
        ta.append(ta[-1] * x)
    tb = []
    if b.shape[0]:
        w = -(sg * u) * pq * iq
        tb.append(w * x)
        while len(tb) < b.shape[0]:
            tb.append(tb[-1] * x)
    return dx, ta, tb


# ---------------------------------------------------------------------------
# Whole-tensor passes (rational.py:325-345, backward.py:113-372)
# ---------------------------------------------------------------------------

def _group_cols(d: int, n_groups: int):
    if d % n_groups:
        raise ValueError("feature dim %d not divisible by %d groups" % (d, n_groups))
    w = d // n_groups
    return [(g, g * w, (g + 1) * w) for g in range(n_groups)]


def forward(x: np.ndarray, num: np.ndarray, den: np.ndarray) -> np.ndarray:
    """forward_tensor: per-group rational on strided column slices; rational.py:325-345."""
    rows = x.reshape(-1, x.shape[-1])
    y = np.empty_like(rows)
    for g, lo, hi in _group_cols(rows.shape[1], num.shape[0]):
        y[:, lo:hi] = rational(rows[:, lo:hi], num[g], den[g])
    return y.reshape(x.shape)


def _seq_total(v: np.ndarray):
    """Strict left-to-right fold starting from the first element; backward.py:113-119."""
    return np.add.accumulate(v)[-1]


def _block_totals(t2: np.ndarray, block: int) -> np.ndarray:
    """Per-row-block strict folds, rows outer / features inner; backward.py:122-139."""
    nrow, width = t2.shape
    full = nrow // block
    out = []
    if full:
        out.append(np.add.accumulate(t2[: full * block].reshape(full, block * width), axis=1)[:, -1])
    if nrow > full * block:
        out.append(np.add.accumulate(t2[full * block:].reshape(-1))[-1:])
    return np.concatenate(out)


def backward_blocked(x, u, num, den, block_size=DEFAULT_BLOCK_SIZE, workers=1):
    """Alg. 2 on the CPU: returns (dx, da, db) in the tensor dtype.

    Mirrors backward_blocked (backward.py:275-372): per (row-block, group)
    partials, tasks of contiguous row-block runs (backward.py:320-325), and an
    ascending block-id fold from zero (combine_partials, backward.py:142-179).
    Raises FloatingPointError("accumulation overflow") for non-finite da/db
    (backward.py:182-184).
    """
    rows = x.reshape(-1, x.shape[-1])
    urows = u.reshape(-1, u.shape[-1])
    nrow = rows.shape[0]
    groups = _group_cols(rows.shape[1], num.shape[0])
    ng = len(groups)
    m1, n = num.shape[1], den.shape[1]
    grid_rows = -(-nrow // block_size)
    dx = np.empty_like(rows)
    per_task = max(1, math.ceil(grid_rows / max(1, workers) / 4))
    tasks = [(g, lo, hi, t0, min(t0 + per_task, grid_rows))
             for g, lo, hi in groups for t0 in range(0, grid_rows, per_task)]

    def task(t):
        g, lo, hi, t0, t1 = t
        r0, r1 = t0 * block_size, min(t1 * block_size, nrow)
        d, ta, tb = element_terms(rows[r0:r1, lo:hi], urows[r0:r1, lo:hi], num[g], den[g])
        dx[r0:r1, lo:hi] = d
        pa = np.stack([_block_totals(t2, block_size) for t2 in ta], axis=1)
        pb = (np.stack([_block_totals(t2, block_size) for t2 in tb], axis=1) if tb
              else np.zeros((pa.shape[0], 0), dtype=pa.dtype))
        return t, pa, pb

    if workers > 1 and len(tasks) > 1:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            results = list(pool.map(task, tasks))
    else:
        results = [task(t) for t in tasks]
    # ordered combine: ascending block_id = row_block * n_groups + group
    parts = []
    for (g, _, _, t0, _), pa, pb in results:
        for k in range(pa.shape[0]):
            parts.append(((t0 + k) * ng + g, g, pa[k], pb[k]))
    parts.sort(key=lambda p: p[0])
    da = np.zeros((ng, m1), dtype=rows.dtype)
    db = np.zeros((ng, n), dtype=rows.dtype)
    for _, g, pa, pb in parts:
        da[g] += pa
        if n:
            db[g] += pb
    if not (np.all(np.isfinite(da)) and np.all(np.isfinite(db))):
        raise FloatingPointError("accumulation overflow")
    return dx.reshape(x.shape), da, db


def combine_partials(partials, num_groups, ordered=True):
    """The reference's fold of (block_id, pa, pb) partials (backward.py:142-179):
    d_a[g] += pa from zeros in ascending block id (or the given order), in the
    partials' dtype."""
    first_a = np.asarray(partials[0][1])
    first_b = np.asarray(partials[0][2])
    seq = sorted(partials, key=lambda p: p[0]) if ordered else list(partials)
    d_a = np.zeros((num_groups, first_a.shape[0]), dtype=first_a.dtype)
    d_b = np.zeros((num_groups, first_b.shape[0]), dtype=first_a.dtype)
    for bid, pa, pb in seq:
        g = bid % num_groups
        d_a[g] += pa
        if first_b.shape[0]:
            d_b[g] += pb
    return d_a, d_b


def backward_naive(x, u, num, den):
    """Alg. 1 model: one long fold per coefficient in tensor precision; backward.py:187-246."""
    rows = x.reshape(-1, x.shape[-1])
    urows = u.reshape(-1, u.shape[-1])
    groups = _group_cols(rows.shape[1], num.shape[0])
    dx = np.empty_like(rows)
    da = np.empty((len(groups), num.shape[1]), dtype=rows.dtype)
    db = np.empty((len(groups), den.shape[1]), dtype=rows.dtype)
    for g, lo, hi in groups:
        d, ta, tb = element_terms(rows[:, lo:hi], urows[:, lo:hi], num[g], den[g])
        dx[:, lo:hi] = d
        for i, t in enumerate(ta):
            da[g, i] = _seq_total(t.reshape(-1))
        for j, t in enumerate(tb):
            db[g, j] = _seq_total(t.reshape(-1))
    if not (np.all(np.isfinite(da)) and np.all(np.isfinite(db))):
        raise FloatingPointError("accumulation overflow")
    return dx.reshape(x.shape), da, db


def ref64_coeff_grads(x, u, num, den):
    """fp64 sequential fold of the run-precision terms; verification.py:318-341."""
    rows = x.reshape(-1, x.shape[-1])
    urows = u.reshape(-1, u.shape[-1])
    groups = _group_cols(rows.shape[1], num.shape[0])
    da = np.zeros((len(groups), num.shape[1]))
    db = np.zeros((len(groups), den.shape[1]))
    for g, lo, hi in groups:
        _, ta, tb = element_terms(rows[:, lo:hi], urows[:, lo:hi], num[g], den[g])
        for i, t in enumerate(ta):
            da[g, i] = np.add.accumulate(t.reshape(-1).astype(np.float64))[-1]
        for j, t in enumerate(tb):
            db[g, j] = np.add.accumulate(t.reshape(-1).astype(np.float64))[-1]
    return da, db


def true64_grads(x, u, num_run, den_run, chunk_rows=1 << 14):
    """fp64 oracle: terms *computed* in fp64 from the run-precision inputs.

    ``num_run``/``den_run`` are the coefficients rounded to the run dtype (the
    values the run actually used, rational.py:243-244) and are widened back to
    fp64 here.  Chunked over rows with pairwise ``np.sum`` per chunk and
    ``math.fsum`` across chunks.
    Returns (dx64, da64, db64).
    """
    rows = x.reshape(-1, x.shape[-1]).astype(np.float64, copy=False)
    urows = u.reshape(-1, u.shape[-1]).astype(np.float64, copy=False)
    groups = _group_cols(rows.shape[1], num_run.shape[0])
    num64 = np.asarray(num_run, dtype=np.float64)
    den64 = np.asarray(den_run, dtype=np.float64)
    dx = np.empty(rows.shape)
    acc_a = [[[] for _ in range(num64.shape[1])] for _ in groups]
    acc_b = [[[] for _ in range(den64.shape[1])] for _ in groups]
    for r0 in range(0, rows.shape[0], chunk_rows):
        r1 = min(r0 + chunk_rows, rows.shape[0])
        for g, lo, hi in groups:
            d, ta, tb = element_terms(rows[r0:r1, lo:hi], urows[r0:r1, lo:hi], num64[g], den64[g])
            dx[r0:r1, lo:hi] = d
            for i, t in enumerate(ta):
                acc_a[g][i].append(float(np.sum(t)))
            for j, t in enumerate(tb):
                acc_b[g][j].append(float(np.sum(t)))
    da = np.array([[math.fsum(v) for v in row] for row in acc_a]).reshape(len(groups), -1)
    db = np.array([[math.fsum(v) for v in row] for row in acc_b]).reshape(len(groups), -1)
    return dx.reshape(x.shape), da, db


# ---------------------------------------------------------------------------
# Error metrics (verification.py:497-510) and the run_bench input generator
# ---------------------------------------------------------------------------

def matrix_rel(a, b) -> float:
    """max|a-b| / max(max|a|, max|b|, 1e-30); verification.py:497-510."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if not a.size:
        return 0.0
    scale = max(float(np.max(np.abs(a))), float(np.max(np.abs(b))), 1e-30)
    return float(np.max(np.abs(a - b))) / scale


def mae(a, b) -> float:
    return float(np.mean(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))))


def bench_inputs(batch, seq, dim, groups, m1=6, n=4, seed=0, dtype=np.float32):
    """run_bench's draw order: x, upstream, numerator, denominator; cli.py:143-158."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((batch, seq, dim)).astype(dtype)
    u = rng.standard_normal((batch, seq, dim)).astype(dtype)
    num = rng.standard_normal((groups, m1))
    den = rng.standard_normal((groups, n))
    return x, u, num, den


def cpu_step(x, u, num, den, block_size=DEFAULT_BLOCK_SIZE, workers=None):
    """One reference-style fwd+bwd pass (run_bench --include-forward, cli.py:178-185)."""
    workers = workers or os.cpu_count() or 1
    y = forward(x, num, den)
    dx, da, db = backward_blocked(x, u, num, den, block_size, workers)
    return y, dx, da, db


# ---------------------------------------------------------------------------
# The layer around the hot path (pkg/src/grkan/layer.py:318-379)
# ---------------------------------------------------------------------------

def layer_forward(x, num, den, weight, bias):
    """y = F(x) W^T + bias in the input precision; layer.py:318-325."""
    rows = forward(x, num, den).reshape(-1, x.shape[-1])
    w = weight.astype(rows.dtype, copy=False)
    b = bias.astype(rows.dtype, copy=False)
    return (rows @ w.T + b).reshape(x.shape[0], x.shape[1], weight.shape[0])


def layer_backward(x, uy, num, den, weight, block_size=DEFAULT_BLOCK_SIZE, naive=False):
    """(d_x, d_a, d_b, d_weight, d_bias); layer.py:328-379: the rational stage gets
    uy W per position; d_weight / d_bias fold per-row-block products in ascending
    block order, returned as float64."""
    dt = x.dtype
    uy_rows = uy.reshape(-1, uy.shape[-1]).astype(dt, copy=False)
    w = weight.astype(dt, copy=False)
    up = (uy_rows @ w).reshape(x.shape)
    if naive:
        dx, da, db = backward_naive(x, up, num, den)
    else:
        dx, da, db = backward_blocked(x, up, num, den, block_size)
    act = forward(x, num, den).reshape(-1, x.shape[-1])
    d_w = np.zeros(weight.shape, dtype=dt)
    d_bias = np.zeros(weight.shape[0], dtype=dt)
    for start in range(0, act.shape[0], block_size):
        stop = min(start + block_size, act.shape[0])
        d_w += uy_rows[start:stop].T @ act[start:stop]
        d_bias += uy_rows[start:stop].sum(axis=0)
    return dx, da, db, d_w.astype(np.float64), d_bias.astype(np.float64)
