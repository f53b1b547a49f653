"""Config 5 stress sweep: token count 1e5..1e9 x groups {1, 8, 16, 64}.

    python tools/stress_sweep.py [--max-e 1e9] [--cpu-max-e 1e8] > sweep.jsonl

Per case (d = 3072, rows = ceil(E / d), seeded N(0,1) x, dy and coefficients):
  * device da/db: FAST, EXACT and the Alg.-1 atomic comparator;
  * true fp64 da/db from a plain-PyTorch fp64 evaluation on the GPU of the
    fp32-rounded inputs and coefficients (chunked; independent of this
    package's kernels) -- the same definition as oracle.true64_grads;
  * for E <= --cpu-max-e also the reference's own blocked and naive fp32
    strategies through the C oracle (bitwise the reference), so the paper's
    rounding claim is shown on the same instance.
Errors: MAE (the paper's metric) and max-scaled, vs the fp64 values.
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


def errs(got, ref):
    g = got.double().cpu().numpy()
    r = ref.double().cpu().numpy()
    return {"mae": float(np.mean(np.abs(g - r))), "maxrel": float(np.max(np.abs(g - r)) / max(np.max(np.abs(r)), 1e-300))}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--max-e", type=float, default=1e9)
    p.add_argument("--cpu-max-e", type=float, default=1e8)
    p.add_argument("--groups", default="1,8,16,64")
    args = p.parse_args()
    dev = torch.device("cuda", 0)
    d = 3072
    for e in (1e5, 1e6, 1e7, 1e8, 1e9):
        if e > args.max_e:
            break
        for ng in (int(g) for g in args.groups.split(",")):
            rows = math.ceil(e / d)
            gen = torch.Generator(device=dev).manual_seed(int(e) * 131 + ng)
            x = torch.randn(rows, d, device=dev, generator=gen)
            u = torch.randn(rows, d, device=dev, generator=gen)
            a = torch.randn(ng, 6, device=dev, generator=gen)
            b = torch.randn(ng, 4, device=dev, generator=gen)
            ta, tb = true64_torch(x, u, a, b, ng)
            line = {"elements": rows * d, "rows": rows, "d": d, "groups": ng}
            for name, fn in (("b200_fast", lambda: ops.rational_backward(x, u, a, b)),
                             ("b200_exact", lambda: ops.rational_backward(x, u, a, b, exact=True)),
                             ("b200_deterministic", lambda: ops.rational_backward(x, u, a, b, deterministic=True)),
                             ("b200_atomic_alg1", lambda: ops.rational_backward_atomic(x, u, a, b))):
                _, da, db = fn()
                ea, eb = errs(da, ta), errs(db, tb)
                line[name] = {"mae_da": ea["mae"], "mae_db": eb["mae"], "maxrel_da": ea["maxrel"],
                              "maxrel_db": eb["maxrel"]}
            if rows * d <= args.cpu_max_e:
                from oracle import c_oracle
                xn = x.cpu().numpy()[None]
                un = u.cpu().numpy()[None]
                r = c_oracle.backward(xn, un, a.double().cpu().numpy(), b.double().cpu().numpy(), 256,
                                      want=("blocked", "naive"))
                for name in ("blocked", "naive"):
                    ea = errs(torch.from_numpy(np.asarray(r[name + "_da"])), ta)
                    eb = errs(torch.from_numpy(np.asarray(r[name + "_db"])), tb)
                    line["reference_" + name] = {"mae_da": ea["mae"], "mae_db": eb["mae"],
                                                 "maxrel_da": ea["maxrel"], "maxrel_db": eb["maxrel"]}
            print(json.dumps(line), flush=True)
            del x, u
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
