"""Config 5 stress sweep: token count 1e5..1e9 x groups {1, 8, 16, 64}.

    python tools/stress_sweep.py [--max-e 1e9] [--cpu-max-e 1e8] [--passes 20] [--max-passes-e 1e8] > sweep.jsonl

Per case (d = 3072, rows = ceil(E / d), seeded N(0,1) x, dy and coefficients):
  * device da/db: FAST, EXACT and the Alg.-1 atomic comparator;
  * true fp64 da/db from a plain-PyTorch fp64 evaluation on the GPU of the
    fp32-rounded inputs and coefficients (chunked; independent of this
    package's kernels) -- the same definition as oracle.true64_grads;
  * the fp64 sum of the reference's own fp32 terms (terms64: accumulation-only
  truth; the fp64 values above also carry fp32 term-evaluation error, e.g. an
  element whose fp32 sign(A) differs from the fp64 one near a root of A --
  shared by every fp32 method including the reference);
* for E <= --cpu-max-e also the reference's own blocked and naive fp32
    strategies through the C oracle (bitwise the reference), so the paper's
    rounding claim is shown on the same instance.
Errors: MAE (the paper's metric) and max-scaled, vs the fp64 values.
With --passes P (20 passes, as the reference's
rounding_experiment, verification.py:352-420) every case is repeated on fresh
inputs per pass and the line reports the mean over passes and the normal-
approximation CI95 half-width of the MAE (verification.py:344-349); cases
above --max-passes-e run 3 passes.  The CPU reference runs on pass 0 only.
Test infrastructure: the oracle is the checker, never the thing measured.
"""
import argparse
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_13813_b200 import ops  # noqa: E402


def true64_torch(x, u, a32, b32, ng, chunk_rows=1 << 14):
    """fp64 da/db of the fp32 inputs x, u [rows, d] and coefficients (GPU, chunked, fp64 sums)."""
    rows, d = x.shape
    dg = d // ng
    a = a32.double()
    b = b32.double()
    da = torch.zeros(ng, 6, dtype=torch.float64, device=x.device)
    db = torch.zeros(ng, 4, dtype=torch.float64, device=x.device)
    for r0 in range(0, rows, chunk_rows):
        xc = x[r0:r0 + chunk_rows].double().view(-1, ng, dg)
        uc = u[r0:r0 + chunk_rows].double().view(-1, ng, dg)
        ag = a.view(1, ng, 6, 1)
        bg = b.view(1, ng, 4, 1)
        p = torch.zeros_like(xc)
        for k in range(5, -1, -1):
            p = p * xc + ag[:, :, k]
        h = torch.zeros_like(xc)
        for k in range(3, -1, -1):
            h = h * xc + bg[:, :, k]
        s = h * xc
        q = 1.0 + s.abs()
        t0 = uc / q
        w = -torch.sign(s) * t0 * p / q
        xp = torch.ones_like(xc)
        for i in range(6):
            da[:, i] += (t0 * xp).sum(dim=(0, 2))
            xp = xp * xc
            if i < 4:
                db[:, i] += (w * xp).sum(dim=(0, 2))
    return da, db


def terms64(x, u, a32, b32, ng, chunk_rows=1 << 13):
    """fp64 sums of the reference's own fp32 terms (EXACT grkan_bwd_terms: bitwise the
    reference's gradient_terms) -- the paper-style accumulation-only truth
    (reference_coeff_grads, verification.py:318-341).  Unlike true64_torch it shares
    the fp32 sign(A) of every element with the reference, so it isolates the
    accumulation error from fp32 term evaluation."""
    from paper_2505_13813_b200 import _native as N
    rows, d = x.shape
    dg = d // ng
    acc = torch.zeros(10, ng, dtype=torch.float64, device=x.device)
    dx = torch.empty(min(chunk_rows, rows), d, dtype=x.dtype, device=x.device)
    t = torch.empty(10 * min(chunk_rows, rows) * d, dtype=torch.float32, device=x.device)  # [10][r][d] per chunk
    for r0 in range(0, rows, chunk_rows):
        r = min(chunk_rows, rows - r0)
        rc = N.lib().grkan_bwd_terms(x[r0].data_ptr(), u[r0].data_ptr(), a32.data_ptr(), b32.data_ptr(),
                                     dx.data_ptr(), t.data_ptr(), r, d, ng, 6, 4, N.DT_F32, N.FLAG_EXACT,
                                     torch.cuda.current_stream().cuda_stream)
        assert rc == 0, N.last_error()
        acc += t[:10 * r * d].view(10, r, ng, dg).double().sum(dim=(1, 3))
    return acc[:6].T.contiguous(), acc[6:].T.contiguous()


def errs(got, ref):
    g = got.double().cpu().numpy()
    r = ref.double().cpu().numpy()
    return {"mae": float(np.mean(np.abs(g - r))), "maxrel": float(np.max(np.abs(g - r)) / max(np.max(np.abs(r)), 1e-300))}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--max-e", type=float, default=1e9)
    p.add_argument("--cpu-max-e", type=float, default=1e8)
    p.add_argument("--groups", default="1,8,16,64")
    p.add_argument("--passes", type=int, default=1)
    p.add_argument("--max-passes-e", type=float, default=1e8)
    args = p.parse_args()
    dev = torch.device("cuda", 0)
    d = 3072
    for e in (1e5, 1e6, 1e7, 1e8, 1e9):
        if e > args.max_e:
            break
        for ng in (int(g) for g in args.groups.split(",")):
            rows = math.ceil(e / d)
            passes = args.passes if e <= args.max_passes_e else min(args.passes, 3)
            line = {"elements": rows * d, "rows": rows, "d": d, "groups": ng, "passes": passes}
            per = {}
            for pss in range(passes):
                gen = torch.Generator(device=dev).manual_seed(int(e) * 131 + ng + 1000003 * pss)
                x = torch.randn(rows, d, device=dev, generator=gen)
                u = torch.randn(rows, d, device=dev, generator=gen)
                a = torch.randn(ng, 6, device=dev, generator=gen)
                b = torch.randn(ng, 4, device=dev, generator=gen)
                ta, tb = true64_torch(x, u, a, b, ng)
                sa, sb = terms64(x, u, a, b, ng)
                for name, fn in (("b200_fast", lambda: ops.rational_backward(x, u, a, b)),
                                 ("b200_exact", lambda: ops.rational_backward(x, u, a, b, exact=True)),
                                 ("b200_deterministic", lambda: ops.rational_backward(x, u, a, b, deterministic=True)),
                                 ("b200_atomic_alg1", lambda: ops.rational_backward_atomic(x, u, a, b))):
                    _, da, db = fn()
                    ea, eb = errs(da, ta), errs(db, tb)
                    fa, fb = errs(da, sa), errs(db, sb)
                    per.setdefault(name, []).append((ea["mae"], eb["mae"], ea["maxrel"], eb["maxrel"],
                                                     fa["mae"], fb["mae"], fa["maxrel"], fb["maxrel"]))
                if pss == 0 and rows * d <= args.cpu_max_e:
                    from oracle import c_oracle
                    xn = x.cpu().numpy()[None]
                    un = u.cpu().numpy()[None]
                    r = c_oracle.backward(xn, un, a.double().cpu().numpy(), b.double().cpu().numpy(), 256,
                                          want=("blocked", "naive"))
                    for name in ("blocked", "naive"):
                        ga = torch.from_numpy(np.asarray(r[name + "_da"]))
                        gb = torch.from_numpy(np.asarray(r[name + "_db"]))
                        ea, eb = errs(ga, ta), errs(gb, tb)
                        fa, fb = errs(ga, sa), errs(gb, sb)
                        line["reference_" + name] = {"mae_da": ea["mae"], "mae_db": eb["mae"],
                                                     "maxrel_da": ea["maxrel"], "maxrel_db": eb["maxrel"],
                                                     "acc_mae_da": fa["mae"], "acc_mae_db": fb["mae"],
                                                     "acc_maxrel_da": fa["maxrel"], "acc_maxrel_db": fb["maxrel"]}
                del x, u
                torch.cuda.empty_cache()
            for name, vals in per.items():
                v = np.asarray(vals)
                ci = (1.96 * v.std(axis=0, ddof=1) / math.sqrt(len(v))) if len(v) > 1 else [None] * 4
                line[name] = {"mae_da": float(v[:, 0].mean()), "mae_db": float(v[:, 1].mean()),
                              "maxrel_da": float(v[:, 2].max()), "maxrel_db": float(v[:, 3].max()),
                              "mae_da_ci95": None if ci[0] is None else float(ci[0]),
                              "mae_db_ci95": None if ci[1] is None else float(ci[1]),
                              # vs the fp64 sum of the reference's fp32 terms (accumulation only)
                              "acc_mae_da": float(v[:, 4].mean()), "acc_mae_db": float(v[:, 5].mean()),
                              "acc_maxrel_da": float(v[:, 6].max()), "acc_maxrel_db": float(v[:, 7].max()),
                              # pass 0 alone: the instance the CPU reference also ran
                              "p0_mae_da": float(v[0, 0]), "p0_mae_db": float(v[0, 1]),
                              "p0_acc_mae_da": float(v[0, 4]), "p0_acc_mae_db": float(v[0, 5])}
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
