"""Host-buffer streaming: the GR-KAN unit over tensors that live in (pinned) host memory.

The CPU reference works on host arrays; a drop-in user therefore pays PCIe
for ``x``/``dy`` in and ``y``/``dx`` out every step.  ``HostPipeline`` hides
most of that: rows are processed in chunks, each chunk's host->device copy,
its fwd+bwd kernels and its device->host copy run on three streams with two
buffer slots, so copy-in of chunk i+1, compute of chunk i and copy-out of
chunk i-1 overlap (PCIe is full duplex).  Per-chunk da/db are summed on the
device in fixed chunk order (fp64), so results are run-to-run deterministic.

    pipe = HostPipeline(device, d=3072, n_groups=8)
    da, db = pipe.fwd_bwd(x_pinned, dy_pinned, a, b, y_pinned, dx_pinned)
"""

from __future__ import annotations

import torch

from . import ops


class HostPipeline:
    AUTO_CHUNK_BYTES = 32 << 20  # smaller chunks pay more per-chunk launch overhead than they overlap

    def __init__(self, device, d: int, n_groups: int, m1: int = 6, n: int = 4,
                 dtype: torch.dtype = torch.float32, chunk_rows: int | None = None):
        self.device = torch.device(device)
        self.d, self.ng, self.m1, self.n = d, n_groups, m1, n
        self.dtype = dtype
        row_bytes = d * torch.empty((), dtype=dtype).element_size()
        self.chunk_rows = int(chunk_rows) if chunk_rows else -(-self.AUTO_CHUNK_BYTES // row_bytes)
        shape = (self.chunk_rows, d)
        mk = lambda: torch.empty(shape, dtype=dtype, device=self.device)  # noqa: E731
        self.x = [mk(), mk()]
        self.dy = [mk(), mk()]
        self.y = [mk(), mk()]
        self.dx = [mk(), mk()]
        self.ws = [torch.empty(ops.workspace_bytes(self.chunk_rows, d, n_groups, m1, n, dtype),
                               dtype=torch.uint8, device=self.device) for _ in range(2)]
        self.h2d = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)
        self.ev_in = [torch.cuda.Event() for _ in range(2)]
        self.ev_comp = [torch.cuda.Event() for _ in range(2)]
        self.ev_out = [torch.cuda.Event() for _ in range(2)]

    def fwd_bwd(self, x_h: torch.Tensor, dy_h: torch.Tensor, a: torch.Tensor, b: torch.Tensor,
                y_h: torch.Tensor, dx_h: torch.Tensor, exact: bool = False):
        """Forward into ``y_h`` and backward into ``dx_h`` (all host tensors, [..., d]);
        returns (da, db) on the device (enqueued on the current stream)."""
        rows = x_h.numel() // self.d
        xr, dyr = x_h.reshape(rows, self.d), dy_h.reshape(rows, self.d)
        yr, dxr = y_h.reshape(rows, self.d), dx_h.reshape(rows, self.d)
        comp = torch.cuda.current_stream(self.device)
        n_chunks = max(1, -(-rows // self.chunk_rows))
        grads = torch.empty((n_chunks, self.ng * (self.m1 + self.n)), dtype=a.dtype, device=self.device)
        ng_m1 = self.ng * self.m1
        for i in range(n_chunks):
            s = i % 2
            r0, r1 = i * self.chunk_rows, min(rows, (i + 1) * self.chunk_rows)
            nr = r1 - r0
            with torch.cuda.stream(self.h2d):
                # The slot's inputs must be consumed before they are overwritten --
                # also across calls: chunks 0/1 of this call reuse the slots the
                # previous call's last chunks may still be reading.  An event that
                # was never recorded is already complete, so the first call is free.
                self.h2d.wait_event(self.ev_comp[s])
                self.x[s][:nr].copy_(xr[r0:r1], non_blocking=True)
                self.dy[s][:nr].copy_(dyr[r0:r1], non_blocking=True)
                self.ev_in[s].record(self.h2d)
            comp.wait_event(self.ev_in[s])
            comp.wait_event(self.ev_out[s])  # slot's outputs drained to the host (this or the previous call)
            ops.rational_forward(self.x[s][:nr], a, b, exact=exact, out=self.y[s][:nr])
            dx_s = self.dx[s][:nr]
            ops.rational_backward(self.x[s][:nr], self.dy[s][:nr], a, b, exact=exact,
                                  workspace=self.ws[s], dx_out=dx_s,
                                  da_out=grads[i, :ng_m1].view(self.ng, self.m1),
                                  db_out=grads[i, ng_m1:].view(self.ng, self.n))
            self.ev_comp[s].record(comp)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(self.ev_comp[s])
                yr[r0:r1].copy_(self.y[s][:nr], non_blocking=True)
                dxr[r0:r1].copy_(dx_s, non_blocking=True)
                self.ev_out[s].record(self.d2h)
        comp.wait_stream(self.d2h)
        tot = grads.to(torch.float64).sum(0).to(a.dtype)  # fixed chunk order
        return tot[:ng_m1].view(self.ng, self.m1), tot[ng_m1:].view(self.ng, self.n)
