"""Small fwd/bwd runs for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
Exercises every kernel family on small shapes: staged (fp32/bf16/fp64, fast/exact, checked),
register-direct (unaligned), generic degrees, the reduce, the atomic comparator, the
deterministic block partials and the fused tcgen05 layer backward.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_13813_b200 import ops  # noqa: E402

dev = torch.device("cuda", 0)
torch.manual_seed(0)
for dtype in (torch.float32, torch.bfloat16, torch.float64):
    cd = torch.float64 if dtype == torch.float64 else torch.float32
    for shape, g, m1, n in [((3, 37, 384), 8, 6, 4), ((2, 5, 48), 4, 6, 4), ((2, 3, 12), 4, 6, 4),
                            ((2, 9, 64), 2, 4, 2)]:
        x = torch.randn(shape, device=dev).to(dtype)
        u = torch.randn(shape, device=dev).to(dtype)
        a = torch.randn(g, m1, device=dev, dtype=cd)
        b = torch.randn(g, n, device=dev, dtype=cd)
        for exact in (False, True):
            ops.rational_forward(x, a, b, exact=exact, check_finite=True)
            ops.rational_backward(x, u, a, b, exact=exact, check_finite=True, check_overflow=True)
        ops.rational_backward_atomic(x, u, a, b)
        xs = torch.randn(x.numel() + 1, device=dev).to(dtype)[1:].view(shape)  # unaligned
        ops.rational_forward(xs, a, b)
        ops.rational_backward(xs, u, a, b)
        # deterministic mode: whole-tensor call and a two-shard partials + reduce
        if shape[0] * shape[1] > 1:
            ops.rational_backward(x, u, a, b, deterministic=True, check_overflow=True)
            rows = shape[0] * shape[1]
            x2, u2 = x.reshape(rows, -1), u.reshape(rows, -1)
            _, p0 = ops.backward_partials(x2, u2, a, b)
            ops.reduce_partials(p0, m1, n, check_overflow=True)
# fused tcgen05 layer backward: both B-atom swizzles, X staged and direct, M tail
for M, F, K, g in [(200, 256, 128, 2), (130, 768, 192, 8), (256, 256, 1536, 2), (130, 768, 3072, 8)]:
    x = torch.randn(M, F, device=dev).to(torch.bfloat16)
    dy = torch.randn(M, K, device=dev).to(torch.bfloat16)
    w = torch.randn(K, F, device=dev).to(torch.bfloat16)
    a = torch.randn(g, 6, device=dev)
    b = torch.randn(g, 4, device=dev)
    ops.linear_backward_fused(dy, w, x, a, b, check_overflow=True)
# the peer-memory reduce/exchange (one rank)
from paper_2505_13813_b200 import parallel  # noqa: E402
pex = parallel.PeerExchange(8, 6, 4, dev)
for _ in range(3):
    pex.backward(torch.randn(3, 37, 384, device=dev), torch.randn(3, 37, 384, device=dev),
                 torch.randn(8, 6, device=dev), torch.randn(8, 4, device=dev), check_overflow=True)
pex.close()
torch.cuda.synchronize()
print("sanitize run ok")
