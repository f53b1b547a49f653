"""Debug: locate FAST-mode dx mismatches at full size (GPU)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import grkan_oracle as orc, c_oracle
from paper_2505_13813_b200 import ops

for (B, L, D) in [(16, 197, 1536), (128, 197, 1536)]:
    x, u, num, den = orc.bench_inputs(B, L, D, 8, seed=0)
    r = c_oracle.backward(x, u, num, den, 256, want=("dx",))
    a = torch.from_numpy(num.astype(np.float32)).cuda(); b = torch.from_numpy(den.astype(np.float32)).cuda()
    xd = torch.from_numpy(x).cuda(); ud = torch.from_numpy(u).cuda()
    for mode in ("staged", "direct"):
        os.environ["GRKAN_STAGED"] = "1" if mode == "staged" else "0"
        dx, da, db = ops.rational_backward(xd, ud, a, b)
        y = ops.rational_forward(xd, a, b)
        dxh = dx.cpu().numpy(); ref = r["dx"]
        err = np.abs(dxh.astype(np.float64) - ref)
        yerr = orc.matrix_rel(y.cpu().numpy(), orc.forward(x, num, den)) if B == 16 else -1
        print(B, mode, "dx rel", err.max() / np.abs(ref).max(), "y rel", yerr, flush=True)
        idx = np.argsort(err.reshape(-1))[-5:]
        for i in idx:
            rr, cc = divmod(int(i), D)
            print("   row", rr, "col", cc, "g", cc // (D // 8), "x", x.reshape(-1)[i], "u", u.reshape(-1)[i],
                  "ref", ref.reshape(-1)[i], "got", dxh.reshape(-1)[i])
        bad = err.reshape(-1, D) > 1e-3 * np.abs(ref).max()
        print("   bad count", bad.sum(), "rows with bad", np.unique(np.nonzero(bad)[0])[:20], "cols", np.unique(np.nonzero(bad)[1])[:20])
