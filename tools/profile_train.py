"""Where a KAT training step spends its GPU time (bench.py --config kat-*-train workload).

    python tools/profile_train.py [--model kat_b] [--batch 128] [--fused-mlp]

torch.profiler over two steps after warm-up; CUDA kernel time grouped into the
GR-KAN kernels of this package (k_fwd*, k_bwd*, k_linear_*), GEMMs, attention
and the rest.  Prints one JSON line.
"""
import argparse
import collections
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_13813_b200 import kat  # noqa: E402


def bucket(name):
    n = name.lower()
    if "grkan" in n or n.startswith("void k_") or "k_fwd" in n or "k_bwd" in n or "k_linear" in n:
        return "grkan (this package)"
    if "gemm" in n or "cutlass" in n or "nvjet" in n or "sm100_xmma" in n or "cublas" in n:
        return "gemm (cuBLAS)"
    if "flash" in n or "fmha" in n or "attention" in n or "sdpa" in n:
        return "attention"
    if "norm" in n:
        return "layernorm"
    if "adam" in n or "multi_tensor" in n or "foreach" in n:
        return "optimizer"
    return "other"


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--model", default="kat_b")
    p.add_argument("--batch", type=int, default=128)
    p.add_argument("--fused-mlp", action="store_true")
    args = p.parse_args()
    dev = torch.device("cuda", 0)
    model = getattr(kat, args.model)(fused_mlp=args.fused_mlp).to(dev)
    opt = torch.optim.AdamW(model.parameters(), lr=1e-4, weight_decay=0.05, fused=True)
    imgs = torch.randn(args.batch, 3, 224, 224, device=dev)
    labels = torch.randint(0, 1000, (args.batch,), device=dev)

    def step():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = torch.nn.functional.cross_entropy(model(imgs), labels)
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(2):
            step()
        torch.cuda.synchronize()
    per = collections.Counter()
    top = collections.Counter()
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            us = e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
            per[bucket(e.name)] += us / 2
            top[e.name[:80]] += us / 2
    total = sum(per.values())
    print(json.dumps({"model": args.model, "batch": args.batch, "fused_mlp": args.fused_mlp,
                      "gpu_ms_per_step": total / 1e3,
                      "share": {k: round(v / total, 4) for k, v in per.most_common()},
                      "ms": {k: round(v / 1e3, 3) for k, v in per.most_common()},
                      "top_kernels_ms": {k: round(v / 1e3, 3) for k, v in top.most_common(12)}}))


if __name__ == "__main__":
    main()
