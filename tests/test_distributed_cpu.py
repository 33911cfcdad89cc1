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


def _grid_worker(rank, world, port, n, nv, m, lams, q):
    import sys

    sys.path.insert(0, ROOT)
    import datagen
    import oracle
    from paper_2509_02649_b200.fit import broadcast_best, reduce_grid_inputs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nmu, nr = 4 * m + 1, 2 * m + 1

    def shard_buf(N, seed):
        lo, hi = N * rank // world, N * (rank + 1) // world
        X, Y = datagen.dataset(hi - lo, i0=lo, seed=seed)
        b = torch.zeros(nmu + nr, dtype=torch.complex128)
        b[:nmu] = torch.from_numpy(oracle.moments(X, 1.0, m))
        b[nmu:] = torch.from_numpy(oracle.rhs(X, Y, 1.0, m))
        return b, Y

    buf, _ = shard_buf(n, 6)
    buf_v, Yv = shard_buf(nv, 7)
    sy2 = torch.tensor([float(np.dot(Yv.astype(np.float64), Yv.astype(np.float64)))], dtype=torch.float64)
    reduce_grid_inputs(buf, buf_v, sy2)
    best = torch.zeros(1, dtype=torch.int64)
    theta = torch.zeros(nr, dtype=torch.complex128)
    if rank == 0:  # the oracle stands in for fk_solve_path / fk_path_validate (same formulas, DESIGN R11)
        mu, r, mu_v, r_v = (t.numpy() for t in (buf[:nmu], buf[nmu:], buf_v[:nmu], buf_v[nmu:]))
        risks = []
        for lam in lams:
            th = oracle.solve(mu, r, n, 1, m, lam, "sobolev", 2.0)
            T = oracle.toeplitz_from_moments(mu_v, 1, m) / nv
            risks.append(float(sy2[0]) / nv - 2 * np.real(np.vdot(th, r_v)) / nv + np.real(np.vdot(th, T @ th)))
        best[0] = int(np.argmin(risks))
        theta[:] = torch.from_numpy(oracle.solve(mu, r, n, 1, m, lams[int(best[0])], "sobolev", 2.0))
    broadcast_best(theta, best)
    q.put((rank, int(best[0]), theta.numpy(), float(sy2[0])))
    dist.destroy_process_group()


def test_grid_search_plumbing_world2(oracle):
    """Data-parallel grid search: training + validation moment buffers and the validation sum of
    Y^2 are all-reduced, rank 0 picks lambda, the chosen index and theta reach every rank."""
    import datagen

    n, nv, m, world = 6_001, 3_001, 10, 2
    lams = [1e-7, 1e-5, 1e-3, 1e-1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grid_worker, args=(r, world, port, n, nv, m, lams, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    Xv, Yv = datagen.dataset(nv, seed=7)
    X, Y = datagen.dataset(n, seed=6)
    mu, r = oracle.moments(X, 1.0, m), oracle.rhs(X, Y, 1.0, m)
    direct = [np.mean((Yv - oracle.predict(oracle.solve(mu, r, n, 1, m, lam, "sobolev", 2.0), Xv, 1.0, m).real) ** 2) for lam in lams]
    b = int(np.argmin(direct))
    th = oracle.solve(mu, r, n, 1, m, lams[b], "sobolev", 2.0)
    sy2 = float(np.dot(Yv.astype(np.float64), Yv.astype(np.float64)))
    for rank, best, theta, s in res:
        assert best == b
        assert np.max(np.abs(theta - th)) / np.max(np.abs(th)) < 1e-10
        assert abs(s - sy2) / sy2 < 1e-12
