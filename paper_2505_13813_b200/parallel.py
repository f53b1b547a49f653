"""Data-parallel glue for the GR-KAN unit.

Rows (B*L tokens) are independent in both directions, so each rank runs the
kernels on its own contiguous row shard with no communication on the data
path.  The one exchange is the sum over ranks of the per-group coefficient
gradients da || db (n_groups * (m1 + n) values, 320 bytes per layer at the
paper's shape): ``allreduce_coeff_grads`` does it with one NCCL all-reduce on a
single flat buffer (the backward writes da and db straight into views of it),
``CoeffGradBucket`` batches every rational layer of a model into one
collective, and ``deterministic_allreduce`` gives a rank-order fp64 sum that is
bitwise identical on every rank and independent of the NCCL algorithm.

The reference has no distributed layer; its analogue is worker-count
invariance of backward_blocked (pkg/tests/test_backward.py:128-138).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_rows(total_rows: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    """Contiguous [start, stop) row range of ``rank``; boundaries on multiples of ``align``.

    Strong scaling splits one batch; with align = seq_len every shard holds whole
    sequences.  Remainder rows go to the lowest ranks.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank %d / world %d" % (rank, world))
    if align < 1 or total_rows % align:
        raise ValueError("total_rows %d not a multiple of align %d" % (total_rows, align))
    units = total_rows // align
    base, extra = divmod(units, world)
    start = rank * base + min(rank, extra)
    stop = start + base + (1 if rank < extra else 0)
    return start * align, stop * align


def coeff_grad_buffer(n_groups: int, m1: int, n: int, device=None, dtype=torch.float32):
    """One flat buffer and the (da, db) views the backward writes into."""
    flat = torch.zeros(n_groups * (m1 + n), dtype=dtype, device=device)
    return flat, flat[: n_groups * m1].view(n_groups, m1), flat[n_groups * m1:].view(n_groups, n)


def allreduce_coeff_grads(flat: torch.Tensor, group=None, async_op: bool = False):
    """Sum da || db over ranks in place (NCCL over NVLink on the B200 box)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    return dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group, async_op=async_op)


def deterministic_allreduce(flat: torch.Tensor, group=None) -> torch.Tensor:
    """Rank-order fp64 sum of every rank's vector: bitwise identical on all ranks.

    All-gathers the (tiny) per-rank vectors, then folds them rank 0, 1, ... in
    float64 on the device and rounds once to ``flat``'s dtype.
    """
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return flat
    world = dist.get_world_size(group)
    parts = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(parts, flat.contiguous(), group=group)
    acc = torch.zeros(flat.shape, dtype=torch.float64, device=flat.device)
    for p in parts:  # fixed rank order
        acc += p.to(torch.float64)
    flat.copy_(acc.to(flat.dtype))
    return flat


class CoeffGradBucket:
    """Bucket the da/db of several rational layers into one all-reduce.

    ``views(i)`` returns layer i's (da, db) views; after every layer's backward
    has written them, ``reduce()`` issues one collective (optionally async on
    the caller's stream, returning the work handle to wait on before the
    optimizer step).
    """

    def __init__(self, shapes, device=None, dtype=torch.float32):
        self._offsets = []
        total = 0
        for n_groups, m1, n in shapes:
            self._offsets.append((total, n_groups, m1, n))
            total += n_groups * (m1 + n)
        self.flat = torch.zeros(total, dtype=dtype, device=device)

    def views(self, i: int):
        off, g, m1, n = self._offsets[i]
        da = self.flat[off: off + g * m1].view(g, m1)
        db = self.flat[off + g * m1: off + g * (m1 + n)].view(g, n)
        return da, db

    def reduce(self, group=None, async_op: bool = False, deterministic: bool = False):
        if deterministic:
            deterministic_allreduce(self.flat, group)
            return None
        return allreduce_coeff_grads(self.flat, group, async_op)
