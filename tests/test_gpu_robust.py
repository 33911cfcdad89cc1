"""Robustness of the boundary (verdict r01 #6/#7, advisor r01): failures reported through the
device status word even on the asynchronous solve path, the condition estimate of the solve
report, calls on a caller's side stream, the native host-streaming entry point, and a reused
host streamer."""
import os

import numpy as np
import pytest

import datagen
from gpu_util import check_mu, check_r, dev, fk, gen_dataset, host, rel

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def F():
    assert torch.cuda.is_available()
    return fk()


def test_solve_not_spd_sets_device_status(F, oracle):
    """A = T(-mu)/n + lambda R is negative definite: the dense path's factorisation fails.  With
    report=False (no synchronisation) the device ORs FK_DSTATUS_NOT_SPD into d_status; with a
    report the call returns FK_E_SOLVE."""
    n, m = 5_000, 30
    X, Y = datagen.dataset(n, seed=61)
    mu, r = oracle.moments(X, 1.0, m), oracle.rhs(X, Y, 1.0, m)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    F.fk_solve(dev(-mu.reshape(-1)), dev(r.reshape(-1)), n, 1, m, 1.0, 1e-6, "sobolev", 2.0, report=False, d_status=st)
    assert int(st.item()) & F.FK_DSTATUS_NOT_SPD
    with pytest.raises(F.FkError):
        F.fk_solve(dev(-mu.reshape(-1)), dev(r.reshape(-1)), n, 1, m, 1.0, 1e-6, "sobolev", 2.0)
    # a healthy system leaves the word untouched
    st.zero_()
    F.fk_solve(dev(mu.reshape(-1)), dev(r.reshape(-1)), n, 1, m, 1.0, 1e-6, "sobolev", 2.0, report=False, d_status=st)
    assert int(st.item()) == 0


def test_fit_result_check_raises_on_range(F):
    from paper_2509_02649_b200 import fit

    X = torch.tensor([0.1, 1.5, -0.2, 0.3], device="cuda")
    Y = torch.ones(4, device="cuda")
    res = fit.fit(X, Y, 1.0, 5, 1e-3, "sobolev", 2.0)
    with pytest.raises(fk().FkError):
        res.check()


@pytest.mark.parametrize("m,lam,s", [(50, 1e-4, 2.0), (1000, 1e10 ** (-2 / 3), 1.0)])
def test_rcond_estimate(F, oracle, m, lam, s):
    """rcond_est of the report: an estimate of 1/cond_2 of the solved real-symmetric system from
    its factor (power / inverse iteration converge from one side, so it over-estimates rcond).
    The real form P*AP uses non-normalised pair columns (e_k +- e_-k), so its spectrum matches the
    oracle's Hermitian A only up to a factor <= 2 per end: bracket [true / 4, 10 true]."""
    n = 20_000
    X, Y = datagen.dataset(n, seed=62)
    mu, r = oracle.moments(X, 1.0, m), oracle.rhs(X, Y, 1.0, m)
    _, rep = F.fk_solve(dev(mu.reshape(-1)), dev(r.reshape(-1)), n, 1, m, 1.0, lam, "sobolev", s)
    A = oracle.assemble(mu, n, 1, m, lam, "sobolev", s)
    ev = np.linalg.eigvalsh(A)
    true = ev[0] / ev[-1]
    print(f"m={m}: rcond_est {rep['rcond_est']:.3e} true {true:.3e}")
    assert true / 4 <= rep["rcond_est"] <= 10 * true


def test_calls_on_a_side_stream(F):
    """Outputs allocated (zeroed) on the current stream, the call on another stream: the library
    call must be ordered after the zero-fill (fk._On) -- repeated under load, results identical
    to the default-stream call."""
    n, m = 2_000_000, 500
    X = torch.empty(n, device="cuda")
    Y = torch.empty(n, device="cuda")
    gen_dataset(X, Y, n, 1, seed=63)
    r0, mu0 = F.fk_rhs_type1(X, Y, 1.0, m, 1e-6)
    side = torch.cuda.Stream()
    for _ in range(5):
        torch.cuda._sleep(20_000_000)  # keep the current stream busy so a missing wait would show
        r1, mu1 = F.fk_rhs_type1(X, Y, 1.0, m, 1e-6, stream=side)
        side.synchronize()
        torch.cuda.synchronize()
        assert torch.equal(mu1, mu0) and torch.equal(r1, r0)
    th0, _ = F.fk_solve(mu0.reshape(-1), r0.reshape(-1), n, 1, m, 1.0, 1e-6, "sobolev", 2.0, report=False)
    torch.cuda._sleep(20_000_000)
    th1, _ = F.fk_solve(mu0.reshape(-1), r0.reshape(-1), n, 1, m, 1.0, 1e-6, "sobolev", 2.0, report=False, stream=side)
    side.synchronize()
    torch.cuda.synchronize()
    assert torch.equal(th0, th1)


def test_pcg_large_block_on_side_stream(F):
    """CG path with a preconditioner block above the tile-Cholesky limit (Dl > 4600: cuSOLVER
    potrf inside pcg_run) on a non-default stream (advisor r01: the cuSOLVER handle must be bound
    to the call's stream): theta matches the dense path."""
    n, d, m, lam = 1_000_000, 2, 64, 1e-7
    X = torch.empty(n, 2, device="cuda")
    Y = torch.empty(n, device="cuda")
    gen_dataset(X, Y, n, d, xkind=0, ykind=1, seed=64)
    r, mu = F.fk_rhs_type1(X, Y, 1.0, m, 1e-6)
    old = os.environ.get("FK_SOLVER")
    try:
        os.environ["FK_SOLVER"] = "dense"
        th_d, _ = F.fk_solve(mu.reshape(-1), r.reshape(-1), n, d, m, 1.0, lam, "sobolev", 2.0)
        os.environ["FK_SOLVER"] = "pcg"
        side = torch.cuda.Stream()
        torch.cuda._sleep(50_000_000)
        th_c, rep = F.fk_solve(mu.reshape(-1), r.reshape(-1), n, d, m, 1.0, lam, "sobolev", 2.0, stream=side)
        side.synchronize()
    finally:
        if old is None:
            os.environ.pop("FK_SOLVER", None)
        else:
            os.environ["FK_SOLVER"] = old
    print(f"pcg large block: iters {rep['iters']} backward {rep['backward_err']:.1e} rel {rel(host(th_c), host(th_d)):.1e}")
    assert rep["iters"] > 0
    assert rel(host(th_c), host(th_d)) < 1e-8


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_rhs_type1_host_matches_device(F, oracle, dt):
    """fk_rhs_type1_host (native chunked H2D overlapped with the spreading) == fk_rhs_type1 on
    the same data up to the chunking's rounding (moments: exact fixed-point sums per chunk), and
    both within the gates of the oracle on a subsample-sized case."""
    n, m = 3_000_011, 300
    X = torch.empty(n, device="cuda")
    Y = torch.empty(n, device="cuda")
    gen_dataset(X, Y, n, 1, seed=65)
    X, Y = X.to(dt), Y.to(dt)
    eps = 1e-6 if dt == torch.float32 else 1e-10
    r_d, mu_d = F.fk_rhs_type1(X, Y, 1.0, m, eps)
    Xh, Yh = X.cpu().pin_memory(), Y.cpu().pin_memory()
    r_h, mu_h = F.fk_rhs_type1_host(Xh, Yh, 1.0, m, eps, chunk=1 << 20)
    torch.cuda.synchronize()
    assert float(mu_h[2 * m].real) == n
    assert rel(host(mu_h), host(mu_d)) < 1e-12
    assert rel(host(r_h), host(r_d)) < (1e-7 if dt == torch.float32 else 1e-12)
    # small case against the oracle (pageable host memory: the copies serialise but stay correct)
    Xs, Ys = datagen.dataset(40_001, seed=66)
    Xs, Ys = Xs.reshape(-1).astype(np.float32 if dt == torch.float32 else np.float64), Ys.astype(np.float32 if dt == torch.float32 else np.float64)
    r_s, mu_s = F.fk_rhs_type1_host(torch.from_numpy(Xs), torch.from_numpy(Ys), 1.0, 200, eps, chunk=7_000)
    tol = 1e-5 if dt == torch.float32 else 1e-10
    check_mu(host(mu_s), oracle.moments(Xs, 1.0, 200), tol, eps)
    check_r(host(r_s), oracle.rhs(Xs, Ys, 1.0, 200), Ys, tol, eps)


def test_host_streamer_reused_without_sync(F):
    """advisor r01: a reused HostStreamer must not refill a staging buffer the previous call's
    kernels may still read -- two back-to-back calls with no synchronisation in between give the
    same moments as the device-resident pass."""
    from paper_2509_02649_b200.fit import HostStreamer, _moment_buffers

    n, m = 5_000_000, 200
    X = torch.empty(n, device="cuda")
    Y = torch.empty(n, device="cuda")
    gen_dataset(X, Y, n, 1, seed=67)
    r_d, mu_d = F.fk_rhs_type1(X, Y, 1.0, m, 1e-6)
    Xh, Yh = X.cpu().pin_memory(), Y.cpu().pin_memory()
    st = HostStreamer(1 << 20, 1, torch.float32, torch.device("cuda"))
    outs = []
    for _ in range(3):
        _, mu, r = _moment_buffers(1, m, torch.device("cuda"))
        st.moments(Xh, Yh, 1.0, m, 1e-6, mu, r)
        outs.append((mu, r))
    torch.cuda.synchronize()
    for mu, r in outs:
        assert rel(host(mu), host(mu_d)) < 1e-12 and rel(host(r), host(r_d)) < 1e-7
