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

``deterministic_backward`` goes one step further: da/db bitwise independent
of the NUMBER of ranks.  Each rank computes one partial per global row block
(ops.backward_partials), ``gather_blocks`` all-gathers them into global block
order, and every rank folds the same array in the same fixed order
(ops.reduce_partials) -- the multi-GPU analogue of the reference's
worker-count invariance (pkg/tests/test_acceptance.py:232-252).

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


def block_counts(total_rows: int, world: int, block_rows: int) -> list[int]:
    """Global row blocks owned by each rank under shard_rows(..., align=block_rows).

    The last block may be partial, so ``total_rows`` need not be a multiple of
    ``block_rows``: the tail rows go with the last non-empty shard.
    """
    full, tail = divmod(total_rows, block_rows)
    counts = []
    for r in range(world):
        start, stop = shard_rows(full * block_rows, world, r, align=block_rows)
        counts.append((stop - start) // block_rows)
    if tail:
        last = max(i for i in range(world) if counts[i] > 0 or i == 0) if full else 0
        counts[last] += 1
    return counts


def block_shard(total_rows: int, world: int, rank: int, block_rows: int) -> tuple[int, int]:
    """[start, stop) rows of ``rank`` for the deterministic path (block-aligned, tail on the last shard)."""
    counts = block_counts(total_rows, world, block_rows)
    start = min(total_rows, sum(counts[:rank]) * block_rows)
    stop = min(total_rows, start + counts[rank] * block_rows)
    return start, stop


def gather_blocks(local: torch.Tensor, counts: list[int], group=None) -> torch.Tensor:
    """All-gather per-rank [n_i, ...] block arrays into one [sum n_i, ...] array in rank order.

    Ranks pad to max(counts) for the collective (all_gather needs equal sizes);
    the padding is dropped so the result is exactly the rank-order concatenation.
    """
    world = len(counts)
    if not dist.is_initialized() or world == 1:
        return local
    rank = dist.get_rank(group)
    if local.shape[0] != counts[rank]:
        raise ValueError("rank %d holds %d blocks, expected %d" % (rank, local.shape[0], counts[rank]))
    width = max(counts)
    padded = local.new_zeros((width,) + tuple(local.shape[1:]))
    padded[: local.shape[0]] = local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)


def deterministic_backward(x_shard: torch.Tensor, dy_shard: torch.Tensor, a: torch.Tensor, b: torch.Tensor,
                           total_rows: int, group=None, exact: bool = False):
    """(dx_shard, da, db) with da/db bitwise independent of the world size.

    Each rank passes its rows [block_shard(total_rows, world, rank, det_block_rows)].
    One all-gather of the per-block partials (KAT-B fp32: 394 blocks x 80 values)
    replaces the 320-byte all-reduce; every rank then runs the same fixed-order
    fold, so da/db equal ops.rational_backward(x, dy, a, b, deterministic=True)
    on the unsharded tensor, bit for bit, for 1, 2, 4 or 8 ranks.
    """
    from . import ops

    d = x_shard.shape[-1]
    ng, m1, n = a.shape[0], a.shape[1], b.shape[1]
    rb = ops.det_block_rows(d, ng, x_shard.dtype)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    counts = block_counts(total_rows, world, rb)
    dx, part = ops.backward_partials(x_shard, dy_shard, a, b, exact=exact)
    full = gather_blocks(part, counts, group)
    da, db = ops.reduce_partials(full.contiguous(), m1, n)
    return dx, da, db


class PeerExchange:
    """da||db summed across ranks INSIDE the reduce kernel, over peer memory (no NCCL).

    Setup (once): every rank allocates a zeroed exchange buffer
    (grkan_p2p_alloc), the CUDA-IPC handles are all-gathered through the
    process group (any backend: only 64 bytes per rank) and opened, and the
    device array of the ``world`` mapped pointers is built.  Each
    ``backward(...)`` is then K2 + one fused reduce/exchange kernel
    (grkan_bwd_p2p) -- bitwise-identical da/db on every rank.  Ranks must call
    ``backward`` the same number of times (the epoch counter).
    """

    def __init__(self, n_groups: int, m1: int, n: int, device, group=None):
        import ctypes

        from . import _native as N

        self._N = N
        self.device = torch.device(device)
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        L = N.lib()
        nbytes = L.grkan_p2p_buffer_bytes(self.world, n_groups, m1, n)
        buf = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            self._check(L.grkan_p2p_alloc(nbytes, ctypes.byref(buf)))
        self._own = buf.value
        handle = (ctypes.c_char * N.IPC_HANDLE_BYTES)()
        self._check(L.grkan_ipc_get_handle(self._own, handle))
        handles = [bytes(handle)]
        if self.world > 1:
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(handle), group=group)
        self._opened = []
        ptrs = []
        with torch.cuda.device(self.device):
            for r, h in enumerate(handles):
                if r == self.rank:
                    ptrs.append(self._own)
                    continue
                p = ctypes.c_void_p()
                hb = (ctypes.c_char * N.IPC_HANDLE_BYTES).from_buffer_copy(h)
                self._check(L.grkan_ipc_open_handle(hb, ctypes.byref(p)))
                self._opened.append(p.value)
                ptrs.append(p.value)
        self.ptrs = torch.tensor(ptrs, dtype=torch.int64, device=self.device)
        self.epoch = 0
        if self.world > 1:
            dist.barrier(group=group)  # every buffer is zeroed before anyone writes into it

    def _check(self, rc):
        if rc != 0:
            from .errors import raise_for_status
            raise_for_status(rc, self._N.last_error())

    def backward(self, x, dy, a, b, exact: bool = False, check_overflow: bool = False):
        """(dx, da, db): dx for this rank's rows, da/db summed over every rank."""
        from . import ops

        rows, d, ng, m1, n = ops._validate(x, a, b)
        x, dy, a, b = x.contiguous(), dy.contiguous(), a.contiguous(), b.contiguous()
        dx = torch.empty_like(x)
        da = torch.empty((ng, m1), dtype=a.dtype, device=x.device)
        db = torch.empty((ng, n), dtype=a.dtype, device=x.device)
        ws = torch.empty(ops.workspace_bytes(max(rows, 1), d, ng, m1, n, x.dtype), dtype=torch.uint8,
                         device=x.device)
        self.epoch += 1
        N = self._N
        with torch.cuda.device(x.device):
            rc = N.lib().grkan_bwd_p2p(x.data_ptr(), dy.data_ptr(), a.data_ptr(), ops._ptr(b), dx.data_ptr(),
                                       da.data_ptr(), ops._ptr(db), ws.data_ptr(), ws.numel(), rows, d, ng, m1, n,
                                       ops._DT[x.dtype], ops._flags(exact, False), self.ptrs.data_ptr(),
                                       self.rank, self.world, self.epoch, ops._stream(x.device))
            self._check(rc)
            if check_overflow:
                ops.read_status(ws[:ops.STATUS_BYTES])
        return dx, da, db

    def close(self):
        L = self._N.lib()
        torch.cuda.synchronize(self.device)
        for p in self._opened:
            L.grkan_ipc_close_handle(p)
        self._opened = []
        if self._own:
            L.grkan_p2p_free(self._own)
            self._own = None
