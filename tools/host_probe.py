"""Where the reference-API shim's time goes (KAT-B fp32, pageable NumPy in/out):
forward_tensor / backward_blocked separately, the native pipeline at several thread
counts and chunk sizes, host first-touch vs warm copies, and cudaHostRegister cost.

    python tools/host_probe.py  -> JSON lines
"""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_13813_b200 import _native as N  # noqa: E402
from paper_2505_13813_b200 import grkan as G  # noqa: E402


def wall(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


def main():
    torch.cuda.init()
    B, L, D, NG = 256, 197, 3072, 8
    rng = np.random.default_rng(0)
    x = rng.standard_normal((B, L, D), dtype=np.float32)
    u = rng.standard_normal((B, L, D), dtype=np.float32)
    num, den = rng.standard_normal((NG, 6)), rng.standard_normal((NG, 4))
    xt, ut = G.ActivationTensor(x), G.ActivationTensor(u)
    params = G.GroupRationalParams(num, den)
    layout = G.GroupLayout(D, NG)
    plan = G.ExecutionPlan.blocked(B, L, layout)
    out = {"fwd_ms": wall(lambda: G.forward_tensor(xt, params, layout, validate=False)),
           "bwd_ms": wall(lambda: G.backward_blocked(xt, ut, params, plan, validate=False))}
    print(json.dumps({"shim": out}), flush=True)

    a32, b32 = num.astype(np.float32), den.astype(np.float32)
    rows = B * L
    for threads in (4, 8, 16):
        for chunk_mb in (4, 16, 64):
            h = ctypes.c_void_p()
            assert N.lib().grkan_host_create(0, chunk_mb << 20, threads, ctypes.byref(h)) == 0
            y = np.empty_like(x)
            dx = np.empty_like(x)
            da = np.empty((NG, 6), np.float32)
            db = np.empty((NG, 4), np.float32)

            def f(fresh):
                yy = np.empty_like(x) if fresh else y
                return N.lib().grkan_host_fwd(h, x.ctypes.data, yy.ctypes.data, a32.ctypes.data, b32.ctypes.data,
                                              rows, D, NG, 6, 4, N.DT_F32, 0)

            def bw(fresh):
                dd = np.empty_like(x) if fresh else dx
                return N.lib().grkan_host_bwd(h, x.ctypes.data, u.ctypes.data, a32.ctypes.data, b32.ctypes.data,
                                              dd.ctypes.data, da.ctypes.data, db.ctypes.data, rows, D, NG, 6, 4,
                                              N.DT_F32, 0)
            r = {"threads": threads, "chunk_mb": chunk_mb,
                 "fwd_fresh_ms": wall(lambda: f(True)), "fwd_warm_ms": wall(lambda: f(False)),
                 "bwd_fresh_ms": wall(lambda: bw(True)), "bwd_warm_ms": wall(lambda: bw(False))}
            N.lib().grkan_host_destroy(h)
            print(json.dumps({"pipeline": r}), flush=True)

    # host-only copies (single thread numpy) and first touch
    dst = np.empty_like(x)
    warm = wall(lambda: np.copyto(dst, x))
    fresh = wall(lambda: np.copyto(np.empty_like(x), x))
    touch = wall(lambda: np.empty_like(x).fill(0))
    # pinning the caller's buffer in place instead of staging
    cr = torch.cuda.cudart()
    t0 = time.perf_counter()
    rc = cr.cudaHostRegister(x.ctypes.data, x.nbytes, 0)
    reg_ms = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    rc2 = cr.cudaHostUnregister(x.ctypes.data)
    unreg_ms = (time.perf_counter() - t0) * 1e3
    print(json.dumps({"host": {"bytes": x.nbytes, "copy_warm_ms_1t": warm, "copy_fresh_ms_1t": fresh,
                               "first_touch_fill_ms_1t": touch, "host_register_ms": reg_ms,
                               "host_unregister_ms": unreg_ms, "rc": [int(rc), int(rc2)]}}), flush=True)


if __name__ == "__main__":
    main()
