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
