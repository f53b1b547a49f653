"""PCIe roofline for the e2e line: pinned host <-> device copy bandwidth, one way and both ways at once.

    python tools/pcie_bw.py  -> one JSON line (GB/s)
"""
import json
import time

import numpy as np
import torch


def main():
    dev = torch.device("cuda", 0)
    n = 256 << 20  # 1 GiB of fp32
    h_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d_in = torch.empty(n, dtype=torch.float32, device=dev)
    d_out = torch.empty(n, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    nbytes = n * 4

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps / 1e3

    def h2d():
        d_in.copy_(h_in, non_blocking=True)

    def d2h():
        h_out.copy_(d_out, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream(dev)
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t1, t2, t3 = timed(h2d), timed(d2h), timed(both)

    # pageable NumPy memory, as a caller of the reference-API shim holds it (wall clock,
    # synchronous): an existing array uploaded, and a download into a FRESH array (first
    # touch of its pages included, as .cpu().numpy() does)
    arr = np.ones(n, dtype=np.float32)

    def wall(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps

    t4 = wall(lambda: d_in.copy_(torch.from_numpy(arr)))
    t5 = wall(lambda: d_out.cpu().numpy())
    print(json.dumps({"h2d_gbs": nbytes / t1 / 1e9, "d2h_gbs": nbytes / t2 / 1e9,
                      "bidirectional_gbs_each_way": nbytes / t3 / 1e9, "bytes": nbytes,
                      "pageable_h2d_gbs": nbytes / t4 / 1e9, "pageable_d2h_fresh_gbs": nbytes / t5 / 1e9}))


if __name__ == "__main__":
    main()
