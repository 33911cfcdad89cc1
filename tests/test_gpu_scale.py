"""Full-size and structural GPU checks (BASELINE-scale launch configurations) that do not need
the oracle to sum 1e9-1e10 terms: exact totals, shard additivity, sampled prediction outputs,
a 2-D lattice closed form (product of the 1-D equispaced closed forms, pin P1), the
host-streamed fit, and the large-m fallback path."""
import numpy as np
import pytest

import datagen
from gpu_util import dev, fk, gen_dataset, host, rel, check_mu, check_r

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def F():
    assert torch.cuda.is_available()
    return fk()


def _free_gb():
    free, _ = torch.cuda.mem_get_info()
    return free / 1e9


def _closed_mu1(N, q):
    q = np.asarray(q)
    out = np.zeros(q.shape, dtype=np.complex128)
    odd = np.abs(q) % 2 == 1
    qa = np.abs(q[odd])
    out[odd] = (-1.0) ** ((qa - 1) // 2) / np.sin(qa * np.pi / (2 * N))
    out[q == 0] = N
    return out


def test_full_size_gaussian_shard_additivity(F):
    """C2 (ii) workload (truncated-Gaussian X, n = 4e9 here): mu_0 = n exactly, and the moments
    of the whole set equal the sum over two shards (the fine grids are exact fixed-point sums; only
    the two FFTs' fp64 rounding differs)."""
    n = 4_000_000_000
    if _free_gb() < n * 8 / 1e9 + 4:
        pytest.skip("not enough device memory")
    X = torch.empty(n, dtype=torch.float32, device="cuda")
    Y = torch.empty(n, dtype=torch.float32, device="cuda")
    gen_dataset(X, Y, n, 1, xkind=1, ykind=0, seed=3)
    r, mu = F.fk_rhs_type1(X, Y, 1.0, 1000, 1e-6)
    h = 1_234_567_891
    r2, mu2 = F.fk_rhs_type1(X[:h], Y[:h], 1.0, 1000, 1e-6)
    F.fk_rhs_type1(X[h:], Y[h:], 1.0, 1000, 1e-6, r_out=r2, mu_out=mu2, accumulate=True)
    torch.cuda.synchronize()
    del X, Y
    mu, mu2, r, r2 = host(mu), host(mu2), host(r), host(r2)
    assert mu[2000] == n
    assert rel(mu2, mu) < 1e-13
    assert rel(r2, r) < 1e-7  # per-CTA rhs scales differ between the two launches: fixed-point rounding noise only
    # Hermitian symmetry of the fp64 outputs
    assert np.max(np.abs(mu[::-1] - np.conj(mu))) / abs(mu[2000]) < 1e-12


def test_full_size_predict_sampled(F, oracle):
    """Prediction at 2^30 query points (the bench's launch shape) checked on 2000 sampled outputs."""
    nq, m = 1 << 30, 1000
    if _free_gb() < nq * 8 / 1e9 + 2:
        pytest.skip("not enough device memory")
    rng = np.random.default_rng(5)
    k = np.arange(-m, m + 1)
    th = (rng.normal(size=2 * m + 1) + 1j * rng.normal(size=2 * m + 1)) / (1.0 + np.abs(k)) ** 1.5
    Xq = torch.empty(nq, dtype=torch.float32, device="cuda")
    gen_dataset(Xq, None, nq, 1, xkind=0, seed=9)
    out = F.fk_predict_type2(dev(th), 1, m, 1.0, Xq, 1e-6)
    idx = np.sort(rng.choice(nq, size=2000, replace=False))
    xs = host(Xq[torch.from_numpy(idx).cuda()])
    got = host(out[torch.from_numpy(idx).cuda()])
    ref = oracle.predict(th, xs.astype(np.float64), 1.0, m)
    assert rel(got, ref) <= 1e-5


def test_2d_lattice_closed_form(F):
    """C3-scale d = 2 pass on the N x N lattice of equispaced points (N = 2^15, n ~ 1.07e9):
    mu_{q0,q1} = mu1(q0) mu1(q1) with the 1-D closed form of pin P1."""
    N, m = 1 << 15, 64
    n = N * N
    if _free_gb() < n * 8 / 1e9 + 4:
        pytest.skip("not enough device memory")
    x = ((2 * torch.arange(N, device="cuda", dtype=torch.int64) + 1 - N).to(torch.float32) / N)
    X = torch.empty((n, 2), dtype=torch.float32, device="cuda")
    X[:, 0] = x.repeat_interleave(N)
    X[:, 1] = x.repeat(N)
    mu = host(F.fk_moments_type1(X, 1.0, m, 1e-6))
    del X
    q = np.arange(-2 * m, 2 * m + 1)
    c = _closed_mu1(N, q)
    closed = np.outer(c, c)
    assert rel(mu, closed) <= 1e-5


def test_host_streamed_fit_matches_device_fit(F):
    """fit.fit_host (pinned host buffers, chunked H2D on a copy stream) == the on-device fit."""
    from paper_2509_02649_b200 import fit

    n, m = 3_000_001, 200
    X, Y = datagen.dataset(n, seed=31)
    Xh = torch.from_numpy(X.reshape(-1)).pin_memory()
    Yh = torch.from_numpy(Y).pin_memory()
    th_host = fit.fit_host(Xh, Yh, 1.0, m, 1e-4, "sobolev", 2.0, chunk=1 << 20)
    res = fit.fit(Xh.cuda(), Yh.cuda(), 1.0, m, 1e-4, "sobolev", 2.0)
    assert rel(th_host, host(res.theta)) < 1e-6


def test_large_m_fallback_path(F, oracle):
    """m = 2500: the B-spline grids exceed one CTA's shared memory, so the plan falls back to the
    ES window with fp64 global accumulation -- still within tolerance of the oracle."""
    n, m = 3_000, 2500
    X, Y = datagen.dataset(n, seed=32)
    r, mu = F.fk_rhs_type1(dev(X.reshape(-1)), dev(Y), 1.0, m, 1e-6)
    check_mu(host(mu), oracle.moments(X, 1.0, m), 1e-5)
    check_r(host(r), oracle.rhs(X, Y, 1.0, m), Y, 1e-5)


def test_workspace_too_small_is_reported(F):
    import ctypes

    X = torch.zeros(10, device="cuda")
    mu = torch.zeros(41, dtype=torch.complex128, device="cuda")
    ws = torch.zeros(256, dtype=torch.uint8, device="cuda")
    st = F.lib().fk_moments_type1(F._points(X), 1.0, 10, 1e-6, mu.data_ptr(), 0, ws.data_ptr(), 256, None,
                                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == F.FK_E_WORKSPACE
    assert b"workspace" in F.lib().fk_last_error()


@pytest.mark.parametrize("eps", [1e-6, 1e-10])
def test_identical_samples_many_drains(F, eps):
    """2^29 identical samples: in every CTA each touched cell overflows its fixed-point range many
    times over (int32 cells at eps = 1e-6; the high words of the 64-bit fixed point at eps = 1e-10),
    so the drains into the fp64 carry grids carry the result.  Closed form mu_q = n e^{-i q t0},
    r_k = 1.5 n e^{-i k t0}."""
    n, m, x0 = 1 << 29, 300, 0.3
    X = torch.full((n,), x0, dtype=torch.float32, device="cuda")
    Y = torch.full((n,), 1.5, dtype=torch.float32, device="cuda")
    r, mu = F.fk_rhs_type1(X, Y, 1.0, m, eps)
    t0 = np.pi * np.float64(np.float32(x0)) / 2
    q = np.arange(-2 * m, 2 * m + 1)
    k = np.arange(-m, m + 1)
    mu_cf = n * np.exp(-1j * q * t0)
    r_cf = 1.5 * n * np.exp(-1j * k * t0)
    tol = 1e-5 if eps >= 1e-7 else 1e-10
    e_mu, e_r = rel(host(mu), mu_cf), rel(host(r), r_cf)
    print(f"identical n=2^29 eps={eps}: mu {e_mu:.2e} r {e_r:.2e}")
    assert e_mu <= tol and e_r <= tol
    del X, Y
