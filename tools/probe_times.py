"""Where the staged backward's time goes at one shape: per-CTA %globaltimer stamps.

Needs a probe build:  python tools/build_variant.py probe GRKAN_PROBE_TIMES=1
    GRKAN_LIB=tools/variants/probe/libgrkan_b200.so python tools/probe_times.py --config kat-s --dtype bf16

Runs the backward (K2 + K3) as the bench does, then prints, relative to the
first CTA start: the spread of CTA starts, the first-stage arrival, the
distribution of CTA ends, K3's start / end, beside the CUDA-event time of the
same launch.  Diagnostic only; numbers under a probe build carry its stores.
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_13813_b200 import _native as N  # noqa: E402
from paper_2505_13813_b200 import ops  # noqa: E402

SHAPES = {"kat-t": (8, 197, 768), "kat-s": (128, 197, 1536), "kat-b": (256, 197, 3072)}
KPROBE = 4096


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="kat-s")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--groups", type=int, default=8)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--dump", default=None, help="per-CTA end / SM / rows of the last rep (JSON)")
    args = ap.parse_args()
    B, L, D = SHAPES[args.config]
    dt = {"bf16": torch.bfloat16, "fp32": torch.float32}[args.dtype]
    suf = {"bf16": "bf16", "fp32": "f32"}[args.dtype]
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(1)
    x = torch.randn(B * L, D, device=dev, generator=g).to(dt)
    u = torch.randn(B * L, D, device=dev, generator=g).to(dt)
    a = torch.randn(args.groups, 6, device=dev, generator=g) * 0.3
    b = torch.randn(args.groups, 4, device=dev, generator=g) * 0.3
    lib = N.lib()
    rd = getattr(lib, "grkan_probe_read_" + suf)
    clr = getattr(lib, "grkan_probe_clear_" + suf)
    rd.argtypes = [ctypes.c_void_p, ctypes.c_int]
    dx = torch.empty_like(x)
    for _ in range(5):
        ops.rational_backward(x, u, a, b, dx_out=dx)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = []
    last_rep = None
    buf = np.zeros(4 * KPROBE + 4, dtype=np.uint64)
    for _ in range(args.reps):
        clr()
        torch.cuda.synchronize()
        e0.record()
        ops.rational_backward(x, u, a, b, dx_out=dx)
        e1.record()
        torch.cuda.synchronize()
        rd(buf.ctypes.data, buf.size)
        t = buf[: 4 * KPROBE].reshape(KPROBE, 4).astype(np.int64)
        used = t[:, 0] > 0
        t = t[used]
        t0 = t[:, 0].min()
        rel = (t - t0) / 1e3
        k3s, k3e = (int(buf[4 * KPROBE]) - t0) / 1e3, (int(buf[4 * KPROBE + 1]) - t0) / 1e3
        ends = np.sort(rel[:, 3])
        meta = buf[: 4 * KPROBE].reshape(KPROBE, 4)[used, 2]
        sm, nr = (meta >> 32).astype(np.int64), (meta & 0xffffffff).astype(np.int64)
        last_rep = {"end": rel[:, 3].round(2).tolist(), "sm": sm.tolist(), "rows": nr.tolist()}
        out.append({
            "event_us": e0.elapsed_time(e1) * 1e3, "ctas": int(used.sum()),
            "start_max": rel[:, 0].max(), "first_stage_med": float(np.median(rel[:, 1])),
            "first_stage_max": rel[:, 1].max(), "end_min": ends[0], "end_p10": ends[len(ends) // 10],
            "end_med": float(np.median(ends)), "end_p90": ends[(9 * len(ends)) // 10], "end_max": ends[-1],
            "k3_start": k3s, "k3_end": k3e,
        })
    keys = out[0].keys()
    med = {k: round(float(np.median([o[k] for o in out])), 2) for k in keys}
    print(json.dumps({"config": args.config, "dtype": args.dtype, "groups": args.groups, "median_of_reps": med}))
    if args.dump:
        with open(args.dump, "w") as f:
            json.dump(last_rep, f)


if __name__ == "__main__":
    main()
