"""K3 fused with the da||db exchange over peer memory (parallel.PeerExchange, grkan_bwd_p2p).

Two processes share the one GPU of the test box (CUDA IPC works between
processes on one device; their kernels time-slice): each runs the backward on
its half of the rows through the fused reduce/exchange kernel.  Checks: da/db
bitwise identical on both ranks, equal to the rank-order fp64 sum, within
1e-5 (max-scaled) of the fp64 oracle of the whole batch, over three epochs
(slot parity reuse) with different upstream gradients.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(epoch):
    rng = np.random.default_rng(100 + epoch)
    x = rng.standard_normal((2, 101, 384)).astype(np.float32)
    u = rng.standard_normal((2, 101, 384)).astype(np.float32)
    a = rng.standard_normal((8, 6)).astype(np.float32)
    b = rng.standard_normal((8, 4)).astype(np.float32)
    return x, u, a, b


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2505_13813_b200 import parallel

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    ex = parallel.PeerExchange(8, 6, 4, dev)
    try:
        out = []
        for epoch in range(3):
            x, u, a, b = _inputs(epoch)
            xs = torch.from_numpy(x[rank]).to(dev)  # rank r owns batch row r
            us = torch.from_numpy(u[rank]).to(dev)
            _, da, db = ex.backward(xs, us, torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev),
                                    check_overflow=True)
            out.append((da.cpu().numpy(), db.cpu().numpy()))
        q.put((rank, out))
    finally:
        ex.close()
        dist.destroy_process_group()


def test_peer_exchange_two_ranks_on_one_gpu():
    from oracle import grkan_oracle as orc

    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for epoch in range(3):
        (da0, db0), (da1, db1) = res[0][epoch], res[1][epoch]
        assert da0.tobytes() == da1.tobytes() and db0.tobytes() == db1.tobytes()  # same bits on every rank
        x, u, a, b = _inputs(epoch)
        _, ta, tb = orc.true64_grads(x, u, a.astype(np.float64), b.astype(np.float64))
        assert orc.matrix_rel(da0, ta) <= 1e-5 and orc.matrix_rel(db0, tb) <= 1e-5


def test_peer_exchange_single_rank_matches_k3():
    from paper_2505_13813_b200 import ops, parallel

    dev = torch.device("cuda", 0)
    x, u, a, b = [torch.from_numpy(t).to(dev) for t in _inputs(0)]
    ex = parallel.PeerExchange(8, 6, 4, dev)
    try:
        for _ in range(3):
            dx, da, db = ex.backward(x, u, a, b)
            dx0, da0, db0 = ops.rational_backward(x, u, a, b)
            assert torch.equal(dx, dx0)
            # one rank: the fp64 fold of the same partials, rounded once -- K3's bits
            assert torch.equal(da, da0) and torch.equal(db, db0)
    finally:
        ex.close()


def test_peer_exchange_empty_shard():
    """A rank with no rows still joins the exchange and contributes zeros."""
    from paper_2505_13813_b200 import parallel
    dev = torch.device("cuda", 0)
    ex = parallel.PeerExchange(8, 6, 4, dev)
    try:
        x = torch.empty((0, 384), device=dev)
        a = torch.randn(8, 6, device=dev)
        b = torch.randn(8, 4, device=dev)
        for _ in range(2):
            dx, da, db = ex.backward(x, x, a, b, check_overflow=True)
            assert dx.shape == (0, 384)
            assert float(da.abs().sum()) == 0.0 and float(db.abs().sum()) == 0.0
    finally:
        ex.close()


def test_peer_exchange_more_columns_than_ctas():
    """192 groups x (5, 4) = 1920 columns: the fixed grid of <= 128 CTAs loops over
    them (no whole-grid co-residency needed); one rank == K2 + K3 bits."""
    from paper_2505_13813_b200 import ops, parallel

    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cpu").manual_seed(5)
    x = torch.randn(300, 1536, generator=g).to(dev)
    u = torch.randn(300, 1536, generator=g).to(dev)
    a = torch.randn(192, 6, generator=g).to(dev)
    b = torch.randn(192, 4, generator=g).to(dev)
    ex = parallel.PeerExchange(192, 6, 4, dev)
    try:
        for _ in range(2):
            dx, da, db = ex.backward(x, u, a, b, check_overflow=True)
            dx0, da0, db0 = ops.rational_backward(x, u, a, b)
            assert torch.equal(dx, dx0) and torch.equal(da, da0) and torch.equal(db, db0)
    finally:
        ex.close()


def _timeout_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2505_13813_b200 import parallel
    from paper_2505_13813_b200.errors import PeerExchangeTimeoutError

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["GRKAN_P2P_TIMEOUT_MS"] = "1500"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    ex = parallel.PeerExchange(8, 6, 4, dev)
    outcome = "no-call"
    try:
        if rank == 0:  # rank 1 "fails before launching": it never joins the exchange
            x, u, a, b = [torch.from_numpy(t[0] if t.ndim == 3 else t).to(dev) for t in _inputs(0)]
            try:
                ex.backward(x, u, a, b, check_overflow=True)
                outcome = "returned"
            except PeerExchangeTimeoutError:
                outcome = "timeout"
        dist.barrier()  # rank 1 keeps its buffer mapped until rank 0 is done
        q.put((rank, outcome))
    finally:
        ex.close()
        dist.destroy_process_group()


def test_peer_exchange_missing_rank_times_out_instead_of_hanging():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_timeout_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == "timeout" and res[1] == "no-call"
