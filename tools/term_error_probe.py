"""Where does the fp32 da/db error vs fp64 come from on the stress sweep's worst instances?

    python tools/term_error_probe.py [--e 1e8] [--groups 1] [--passes 20]

For each pass (the stress sweep's seeds) it evaluates the reference's fp32
terms (EXACT grkan_bwd_terms, bitwise the reference's gradient_terms) and the
fp64 terms of the same fp32 inputs, and reports for the worst db coefficient:
the share of its fp32-vs-fp64 error carried by elements whose fp32 sign(A)
differs from the fp64 sign(A), and how many such elements there are.
Test infrastructure / evidence only.
"""
import argparse
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_13813_b200 import _native as N  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--e", type=float, default=1e8)
    p.add_argument("--groups", type=int, default=1)
    p.add_argument("--passes", type=int, default=20)
    args = p.parse_args()
    dev = torch.device("cuda", 0)
    d, ng = 3072, args.groups
    rows = math.ceil(args.e / d)
    dg = d // ng
    chunk = 4096
    for pss in range(args.passes):
        gen = torch.Generator(device=dev).manual_seed(int(args.e) * 131 + ng + 1000003 * pss)
        x = torch.randn(rows, d, device=dev, generator=gen)
        u = torch.randn(rows, d, device=dev, generator=gen)
        a = torch.randn(ng, 6, device=dev, generator=gen)
        b = torch.randn(ng, 4, device=dev, generator=gen)
        s32 = torch.zeros(4, ng, dtype=torch.float64, device=dev)   # fp64 sum of fp32 db terms
        s64 = torch.zeros(4, ng, dtype=torch.float64, device=dev)   # fp64 terms
        flip_err = torch.zeros(4, ng, dtype=torch.float64, device=dev)
        nflip = 0
        dx = torch.empty(chunk, d, device=dev)
        t = torch.empty(10 * chunk * d, device=dev)
        for r0 in range(0, rows, chunk):
            r = min(chunk, rows - r0)
            rc = N.lib().grkan_bwd_terms(x[r0].data_ptr(), u[r0].data_ptr(), a.data_ptr(), b.data_ptr(),
                                         dx.data_ptr(), t.data_ptr(), r, d, ng, 6, 4, N.DT_F32, N.FLAG_EXACT,
                                         torch.cuda.current_stream().cuda_stream)
            assert rc == 0, N.last_error()
            tb32 = t[6 * r * d:10 * r * d].view(4, r, ng, dg).double()
            xc = x[r0:r0 + r].double().view(r, ng, dg)
            uc = u[r0:r0 + r].double().view(r, ng, dg)
            a64, b64 = a.double(), b.double()
            pp = torch.zeros_like(xc)
            for k in range(5, -1, -1):
                pp = pp * xc + a64[:, k].view(1, ng, 1)
            h = torch.zeros_like(xc)
            for k in range(3, -1, -1):
                h = h * xc + b64[:, k].view(1, ng, 1)
            s = h * xc
            q = 1.0 + s.abs()
            w = -torch.sign(s) * (uc / q) * pp / q
            # fp32 sign(A) as the reference rounds it: h by separately rounded Horner in fp32, times x
            x32 = x[r0:r0 + r].view(r, ng, dg)
            h32 = torch.zeros_like(x32)
            for k in range(3, -1, -1):
                h32 = h32 * x32 + b[:, k].view(1, ng, 1)
            flip = torch.sign(h32 * x32).double() != torch.sign(s)
            nflip += int(flip.sum())
            xp = xc.clone()
            for j in range(4):
                t64 = w * xp
                s64[j] += t64.sum(dim=(0, 2))
                s32[j] += tb32[j].sum(dim=(0, 2))
                flip_err[j] += ((tb32[j] - t64) * flip).sum(dim=(0, 2))
                xp = xp * xc
        err = (s32 - s64).abs()
        j, g = divmod(int(err.argmax()), ng)
        scale = float(s64.abs().max())
        print(json.dumps({"pass": pss, "elements": rows * d, "groups": ng,
                          "db_maxrel": float(err.max()) / scale, "worst": [j + 1, g],
                          "err": float((s32 - s64)[j, g]), "err_from_sign_flips": float(flip_err[j, g]),
                          "sign_flips": nflip}), flush=True)
        del x, u
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
