"""Data-parallel glue on CPU with the gloo backend, world size 2.

The per-shard gradients come from the oracle (the CUDA kernels need a GPU);
what is under test is the sharding and the da/db exchange of
paper_2505_13813_b200.parallel: sharded + all-reduced == unsharded.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_13813_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import grkan_oracle as orc
        x, u, num, den = orc.bench_inputs(4, 9, 64, 8, seed=3)
        rows = x.reshape(-1, 64)
        urows = u.reshape(-1, 64)
        lo, hi = parallel.shard_rows(rows.shape[0], world, rank, align=9)
        num_run = num.astype(np.float32).astype(np.float64)
        den_run = den.astype(np.float32).astype(np.float64)
        _, da, db = orc.true64_grads(rows[lo:hi][None], urows[lo:hi][None], num_run, den_run)
        flat, dav, dbv = parallel.coeff_grad_buffer(8, 6, 4, dtype=torch.float64)
        dav.copy_(torch.from_numpy(da))
        dbv.copy_(torch.from_numpy(db))
        det = flat.clone()
        parallel.allreduce_coeff_grads(flat)
        parallel.deterministic_allreduce(det)
        bucket = parallel.CoeffGradBucket([(8, 6, 4), (8, 6, 4)], dtype=torch.float64)
        for i in range(2):
            ba, bb = bucket.views(i)
            ba.copy_(torch.from_numpy(da) * (i + 1))
            bb.copy_(torch.from_numpy(db) * (i + 1))
        bucket.reduce()
        q.put((rank, lo, hi, flat.numpy().copy(), det.numpy().copy(), bucket.flat.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_sharded_allreduce_matches_unsharded():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    from oracle import grkan_oracle as orc
    x, u, num, den = orc.bench_inputs(4, 9, 64, 8, seed=3)
    _, da, db = orc.true64_grads(x, u, num.astype(np.float32).astype(np.float64),
                                 den.astype(np.float32).astype(np.float64))
    want = np.concatenate([da.reshape(-1), db.reshape(-1)])
    assert res[0][1] == 0 and res[-1][2] == 36 and res[0][2] == res[1][1]
    for _, _, _, flat, det, bucket in res:
        assert orc.matrix_rel(flat, want) <= 1e-12
        assert orc.matrix_rel(det, want) <= 1e-12
        assert orc.matrix_rel(bucket, np.concatenate([want, 2 * want])) <= 1e-12
    # deterministic variant is bitwise identical on every rank
    assert res[0][4].tobytes() == res[1][4].tobytes()


@pytest.mark.parametrize("total,world,align", [(36, 2, 9), (50432, 8, 197), (10, 3, 1), (7, 4, 1)])
def test_shard_rows_partition(total, world, align):
    spans = [parallel.shard_rows(total, world, r, align) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == total
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert a1 == b0
    for s0, s1 in spans:
        assert s0 % align == 0 and s1 % align == 0 and s1 >= s0
    sizes = [s1 - s0 for s0, s1 in spans]
    assert max(sizes) - min(sizes) <= align


def test_shard_rows_rejects_bad_args():
    with pytest.raises(ValueError):
        parallel.shard_rows(10, 2, 2)
    with pytest.raises(ValueError):
        parallel.shard_rows(10, 2, 0, align=3)


# ---------------------------------------------------------------------------
# Deterministic (world-size-invariant) path: block-aligned shards + all-gather
# of per-block partials in rank order (parallel.gather_blocks).  The partials
# here are the oracle's fp64 per-block sums; on the GPU they come from
# grkan_bwd_partials (tests/test_gpu_deterministic.py).
# ---------------------------------------------------------------------------

def _block_partials(rows, urows, num, den, start, stop, rb):
    from oracle import grkan_oracle as orc
    out = []
    for r0 in range(start, stop, rb):
        r1 = min(stop, r0 + rb)
        _, da, db = orc.true64_grads(rows[r0:r1][None], urows[r0:r1][None], num, den)
        out.append(np.concatenate([da, db], axis=1))
    return np.stack(out) if out else np.zeros((0, num.shape[0], num.shape[1] + den.shape[1]))


def _gather_worker(rank, world, port, q, total, rb):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import grkan_oracle as orc
        x, u, num, den = orc.bench_inputs(1, total, 16, 2, seed=5)
        rows, urows = x.reshape(-1, 16), u.reshape(-1, 16)
        counts = parallel.block_counts(total, world, rb)
        lo, hi = parallel.block_shard(total, world, rank, rb)
        local = torch.from_numpy(_block_partials(rows, urows, num, den, lo, hi, rb))
        full = parallel.gather_blocks(local, counts)
        q.put((rank, lo, hi, full.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,total,rb", [(2, 40, 8), (3, 37, 8), (2, 5, 8)])
def test_gather_blocks_is_rank_order_concatenation(world, total, rb):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q, total, rb)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import grkan_oracle as orc
    x, u, num, den = orc.bench_inputs(1, total, 16, 2, seed=5)
    want = _block_partials(x.reshape(-1, 16), u.reshape(-1, 16), num, den, 0, total, rb)
    for _, _, _, full in res:
        # every rank holds the same global-order block array: bitwise the unsharded one
        assert full.shape == want.shape and full.tobytes() == want.tobytes()
    assert res[0][1] == 0 and res[-1][2] == total


@pytest.mark.parametrize("total", [0, 1, 127, 128, 129, 1000, 50432])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_block_shards_cover_rows_on_block_boundaries(total, world):
    rb = 128
    counts = parallel.block_counts(total, world, rb)
    spans = [parallel.block_shard(total, world, r, rb) for r in range(world)]
    assert sum(counts) == -(-total // rb)
    assert spans[0][0] == 0 and spans[-1][1] == total
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert a1 == b0
    for (s0, s1), c in zip(spans, counts):
        assert (s0 % rb == 0 or s1 == s0) and -(-(s1 - s0) // rb) == c
