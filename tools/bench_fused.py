"""Fused vs unfused GR-KAN layer backward through the linear map.

    python tools/bench_fused.py [--reps 50]  -> one JSON line per KAT-B layer shape

backward  fused   : ops.linear_backward_fused  (one tcgen05 kernel + the K3 fold)
          unfused : dF = dy @ w (cuBLAS bf16, bf16 output) then ops.rational_backward(x, dF)
(The prologue-fused forward, K6, measured 0.42-0.71x of the unfused chain in round 1
and was removed; the forward is ops.rational_forward then cuBLAS.)
Both on the same synthetic bf16 tensors; CUDA events on the current stream,
inputs far larger than L2.  TFLOP/s counts the GEMM's 2*M*F*K only.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_13813_b200 import ops  # noqa: E402
from bench import ClockSampler  # noqa: E402


CLOCKS = {}  # label -> NVML clock summary of its timed loop


def timed(fn, reps, warm=5, label=None):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(0) if label else None
    if sampler:
        sampler.start()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    if sampler:
        sampler.stop()
        CLOCKS[label] = sampler.summary()
    return e0.elapsed_time(e1) / reps * 1e3  # us


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--reps", type=int, default=50)
    p.add_argument("--batch", type=int, default=256)
    args = p.parse_args()
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                            "MEASURED_PEAKS.json")))
    except OSError:
        pass
    tc_peak = peaks.get("bf16_tflops", 2250.0)
    dev = torch.device("cuda", 0)
    M = args.batch * 197
    for name, F, K in (("kat-b rational2 -> fc2 (F=3072, K=768)", 3072, 768),
                       ("kat-b rational1 -> fc1 (F=768, K=3072)", 768, 3072)):
        g = torch.Generator(device="cpu").manual_seed(0)
        x = torch.randn(M, F, generator=g).to(torch.bfloat16).to(dev)
        dy = torch.randn(M, K, generator=g).to(torch.bfloat16).to(dev)
        w = (torch.randn(K, F, generator=g) / K ** 0.5).to(torch.bfloat16).to(dev)
        a = torch.randn(8, 6, generator=g).to(dev)
        b = torch.randn(8, 4, generator=g).to(dev)
        t_fused = timed(lambda: ops.linear_backward_fused(dy, w, x, a, b), args.reps, label="bwd_fused")
        dF = torch.empty(M, F, dtype=torch.bfloat16, device=dev)
        t_gemm = timed(lambda: torch.matmul(dy, w, out=dF), args.reps, label="bwd_gemm")
        t_rat = timed(lambda: ops.rational_backward(x, dF, a, b), args.reps)
        flops = 2.0 * M * F * K
        print(json.dumps({"direction": "backward",
            "shape": name, "M": M, "F": F, "K": K, "groups": 8,
            "fused_us": t_fused, "fused_tflops": flops / t_fused / 1e6,
            "fused_frac_of_bf16_peak": flops / t_fused / 1e6 / tc_peak,
            "unfused_gemm_us": t_gemm, "unfused_rational_bwd_us": t_rat, "unfused_us": t_gemm + t_rat,
            "speedup": (t_gemm + t_rat) / t_fused, "bf16_peak_tflops": tc_peak,
            "hbm_bytes_fused": 2.0 * (M * K + K * F + 2 * M * F),
            "hbm_bytes_unfused": 2.0 * (M * K + K * F + M * F) + 2.0 * 3 * M * F,
            # NVML during the timed loops: tensor-core work runs the B200 into its power cap
            "fused_clocks": CLOCKS.get("bwd_fused"), "gemm_clocks": CLOCKS.get("bwd_gemm"),
        }), flush=True)


if __name__ == "__main__":
    main()
