"""World-size-2 (gloo, CPU) coverage of the data-parallel plumbing of fit.fit_distributed:
per-rank shards' unnormalised [mu | r] buffers are all-reduced (sum) and theta is broadcast from
rank 0.  The per-rank moments here come from the oracle (CPU), so the test exercises exactly the
collective logic the GPU path uses (paper_2509_02649_b200.fit.reduce_moments / broadcast_theta)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, m, q):
    import sys

    sys.path.insert(0, ROOT)
    import datagen
    import oracle
    from paper_2509_02649_b200.fit import broadcast_theta, reduce_moments

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = n * rank // world, n * (rank + 1) // world
    X, Y = datagen.dataset(hi - lo, i0=lo, seed=5)
    nmu, nr = 4 * m + 1, 2 * m + 1
    buf = torch.zeros(nmu + nr, dtype=torch.complex128)
    buf[:nmu] = torch.from_numpy(oracle.moments(X, 1.0, m))
    buf[nmu:] = torch.from_numpy(oracle.rhs(X, Y, 1.0, m))
    reduce_moments(buf)
    theta = torch.zeros(nr, dtype=torch.complex128)
    if rank == 0:
        theta[:] = torch.from_numpy(oracle.solve(buf[:nmu].numpy(), buf[nmu:].numpy(), n, 1, m, 1e-4, "sobolev", 2.0))
    broadcast_theta(theta)
    q.put((rank, buf.numpy(), theta.numpy()))
    dist.destroy_process_group()


def test_allreduce_and_broadcast_world2(oracle):
    import datagen

    n, m, world = 9_001, 12, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    X, Y = datagen.dataset(n, seed=5)
    full = np.concatenate([oracle.moments(X, 1.0, m), oracle.rhs(X, Y, 1.0, m)])
    th = oracle.solve(full[: 4 * m + 1], full[4 * m + 1:], n, 1, m, 1e-4, "sobolev", 2.0)
    for rank, buf, theta in res:
        assert np.max(np.abs(buf - full)) / np.max(np.abs(full)) < 1e-12
        assert np.max(np.abs(theta - th)) / np.max(np.abs(th)) < 1e-10
