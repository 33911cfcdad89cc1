"""World-size-2 runs of the REAL data-parallel fits on the GPU (verdict r01 #4/#5): two processes,
both on cuda:0 (the boxes have one GPU), joined by a gloo process group over CUDA tensors.  Each
rank spreads its shard with libfk, the [mu | r (| G)] buffers are all-reduced, rank 0 solves, theta
is broadcast -- fit_distributed, fit_additive_distributed and grid_search_distributed against the
one-process fits of the whole dataset.  No kernel waits on another process (the exchange is the
gloo collective on the host), so two ranks may share the GPU.  Also runs bench.py's distributed
branch once under torchrun with --backend gloo."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = dict(
    sobolev=dict(n=3_000_017, d=1, m=300, lam=1e-5, s=2.0),
    additive=dict(n=400_003, d=4, m=20, lam=1e-4),
    grid=dict(n=600_001, nv=200_003, d=1, m=80, lams=[1e-7, 1e-6, 1e-5, 1e-4, 1e-3]),
)


def _shard(case, rank, world, dev, nkey="n", seed=0):
    from datagen.device import gen_dataset

    c = CASES[case]
    n, d = c[nkey], c["d"]
    lo, hi = n * rank // world, n * (rank + 1) // world
    Y = torch.empty(hi - lo, device=dev)
    if d == 1:
        X = torch.empty(hi - lo, device=dev)
        gen_dataset(X, Y, hi - lo, 1, i0=lo, seed=seed)
    else:
        Xs = torch.empty((d, hi - lo), device=dev)
        gen_dataset(Xs, Y, hi - lo, d, i0=lo, ykind=2, seed=seed, stride_n=1, stride_d=hi - lo)
        X = Xs.t()
    return X, Y


def _worker(rank, world, port, case, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2509_02649_b200 import fit

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = CASES[case]
    try:
        if case == "sobolev":
            X, Y = _shard(case, rank, world, dev)
            res = fit.fit_distributed(X, Y, c["n"], 1.0, c["m"], c["lam"], "sobolev", c["s"]).check()
            out = res.theta.cpu().numpy()
        elif case == "additive":
            X, Y = _shard(case, rank, world, dev)
            res = fit.fit_additive_distributed(X, Y, c["n"], 1.0, c["m"], c["lam"]).check()
            out = res.theta.cpu().numpy()
        else:
            X, Y = _shard(case, rank, world, dev)
            Xv, Yv = _shard(case, rank, world, dev, "nv", seed=1)
            g = fit.grid_search_distributed(X, Y, c["n"], Xv, Yv, c["nv"], 1.0, c["m"], c["lams"], "sobolev", 2.0)
            out = (g.best, g.theta.cpu().numpy())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _run_world2(case):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def _rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


def test_fit_distributed_world2_matches_single():
    sys.path.insert(0, ROOT)
    from paper_2509_02649_b200 import build, fit

    build.build()
    res = _run_world2("sobolev")
    c = CASES["sobolev"]
    X, Y = _shard("sobolev", 0, 1, torch.device("cuda"))
    ref = fit.fit(X, Y, 1.0, c["m"], c["lam"], "sobolev", c["s"]).check().theta.cpu().numpy()
    assert np.array_equal(res[0], res[1])  # theta broadcast from rank 0
    e = _rel(res[0], ref)
    print(f"world-2 fit_distributed vs one process: {e:.2e}")
    assert e < 1e-6  # the shards' fp32 rhs use their own per-CTA scales (rounding-level)


def test_fit_additive_distributed_world2_matches_single():
    sys.path.insert(0, ROOT)
    from paper_2509_02649_b200.fit import fit_additive_distributed

    res = _run_world2("additive")
    c = CASES["additive"]
    X, Y = _shard("additive", 0, 1, torch.device("cuda"))
    ref = fit_additive_distributed(X, Y, c["n"], 1.0, c["m"], c["lam"]).check().theta.cpu().numpy()
    assert np.array_equal(res[0], res[1])
    e = _rel(res[0], ref)
    print(f"world-2 additive vs one process: {e:.2e}")
    assert e < 1e-6


def test_grid_search_distributed_world2_matches_single():
    sys.path.insert(0, ROOT)
    from paper_2509_02649_b200 import fit

    res = _run_world2("grid")
    c = CASES["grid"]
    X, Y = _shard("grid", 0, 1, torch.device("cuda"))
    Xv, Yv = _shard("grid", 0, 1, torch.device("cuda"), "nv", seed=1)
    g = fit.grid_search(X, Y, Xv, Yv, 1.0, c["m"], c["lams"], "sobolev", 2.0)
    assert res[0][0] == res[1][0] == g.best
    assert _rel(res[0][1], g.theta.cpu().numpy()) < 1e-6


def test_bench_distributed_branch_gloo():
    """bench.py's N > 1 branch (sample shards, all-reduce, rank-0 solve, broadcast, max-over-ranks
    timing) executed once: two ranks on the one GPU over gloo."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--config", "c1", "--backend", "gloo", "--no-e2e", "--no-cpu"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["fit_status_ok"]
