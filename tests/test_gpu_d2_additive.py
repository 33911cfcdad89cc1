"""GPU parity of the d = 2 pass (C3/C4 shapes), the physics-informed and Sobolev d = 2 solves,
2-D prediction, and the additive model (cross moments, block solve, additive prediction)."""
import numpy as np
import pytest

import datagen
from gpu_util import dev, fk, host, rel, check_mu, check_r

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def F():
    assert torch.cuda.is_available()
    return fk()


HEAT = dict(alpha=[[1, 0], [0, 2]], a_alpha=[1.0, -1.0], box=[[-1.0, 1.0], [-1.0, 1.0]])  # d_tau f - d_xx f (DESIGN R6)


@pytest.mark.parametrize("n,m,eps,dt", [(20_001, 8, 1e-6, "f32"), (20_000, 32, 1e-6, "f32"), (6_000, 64, 1e-6, "f32"),
                                        (5_000, 16, 1e-10, "f64"), (4_001, 12, 1e-6, "f64")])
def test_type1_2d_matches_oracle(F, oracle, n, m, eps, dt):
    X, Y = datagen.dataset(n, d=2, ykind="expcos", seed=21)
    t = torch.float32 if dt == "f32" else torch.float64
    if dt == "f64":
        X = X.astype(np.float64) * (1 - 2.0 ** -31)
        Y = Y.astype(np.float64)
    r, mu = F.fk_rhs_type1(dev(X, t), dev(Y, t), 1.0, m, eps)
    mu_o, r_o = oracle.moments(X, 1.0, m), oracle.rhs(X, Y, 1.0, m)
    tol = 1e-5 if eps >= 1e-7 else 1e-10
    e_mu, em_mu = check_mu(host(mu), mu_o, tol, eps)
    e_r, em_r = check_r(host(r), r_o, Y, tol, eps)
    print(f"d=2 n={n} m={m} eps={eps} {dt}: mu {e_mu:.2e} (elem {em_mu:.1e}) r {e_r:.2e} (elem {em_r:.1e})")


def test_2d_edges_and_views(F, oracle):
    m = 10
    X = np.array([[1.0, 1.0], [-1.0, -1.0], [1.0, -1.0], [-1.0, 1.0], [0.3, -0.7]] * 300, dtype=np.float32)
    Y = np.linspace(-1, 2, X.shape[0]).astype(np.float32)
    r, mu = F.fk_rhs_type1(dev(X), dev(Y), 1.0, m, 1e-6)
    check_mu(host(mu), oracle.moments(X, 1.0, m), 1e-5)
    check_r(host(r), oracle.rhs(X, Y, 1.0, m), Y, 1e-5)
    # SoA view (column pitch != d) and general L
    X2, Y2 = datagen.dataset(7_003, d=2, seed=22, L=1.9)
    soa = dev(np.ascontiguousarray(X2.T))  # (2, n)
    mu2 = F.fk_moments_type1(soa.t(), 1.9, m, 1e-6)
    check_mu(host(mu2), oracle.moments(X2, 1.9, m), 1e-5)


@pytest.mark.parametrize("kind,m", [("sobolev", 16), ("pik_box", 12)])
def test_solve_2d_matches_oracle(F, oracle, kind, m):
    X, Y = datagen.dataset(20_000, d=2, ykind="expcos", seed=23)
    mu, r = oracle.moments(X, 1.0, m), oracle.rhs(X, Y, 1.0, m)
    kw = dict(mu_pde=1.0, L=1.0, **HEAT) if kind == "pik_box" else {}
    th_o = oracle.solve(mu, r, 20_000, 2, m, 1e-6, kind, 2.0, **kw)
    kw2 = dict(mu_pde=1.0, **HEAT) if kind == "pik_box" else {}
    th, rep = F.fk_solve(dev(mu.reshape(-1)), dev(r.reshape(-1)), 20_000, 2, m, 1.0, 1e-6, kind, 2.0, **kw2)
    print(f"solve d=2 {kind} m={m}: {rel(host(th), th_o):.2e} backward {rep['backward_err']:.1e} ms {rep['ms']:.1f}")
    assert rep["backward_err"] < 1e-11
    assert rel(host(th), th_o) < 1e-6


@pytest.mark.parametrize("m,eps", [(20, 1e-6), (64, 1e-6), (16, 1e-10)])
def test_predict_2d_matches_oracle(F, oracle, m, eps):
    rng = np.random.default_rng(4)
    k = oracle.mode_grid(2, m)
    D = k.shape[0]
    th = (rng.normal(size=D) + 1j * rng.normal(size=D)) / (1.0 + np.sum(k * k, 1))
    Xq = datagen.dataset(5_001, d=2, seed=24)[0]
    t = torch.float32 if eps >= 1e-7 else torch.float64
    out = host(F.fk_predict_type2(dev(th), 2, m, 1.0, dev(Xq, t), eps))
    err = rel(out, oracle.predict(th, Xq, 1.0, m))
    print(f"predict d=2 m={m} eps={eps}: {err:.2e}")
    assert err <= (1e-5 if eps >= 1e-7 else 1e-10)


def test_pi_fit_end_to_end(F, oracle):
    """C4 shape (PI space-time heat equation, d = 2, m = 16 here): GPU fit vs oracle fit."""
    n, m, s, lam = 30_000, 16, 2.0, 30_000 ** (-2 / 3)
    X, Y = datagen.dataset(n, d=2, ykind="expcos", seed=25)
    Xq = datagen.dataset(3_000, d=2, seed=26)[0]
    th_o, _, _ = oracle.fit(X, Y, 1.0, m, lam, "pik_box", s, mu_pde=1.0, **HEAT)
    r, mu = F.fk_rhs_type1(dev(X), dev(Y), 1.0, m, 1e-6)
    th, rep = F.fk_solve(mu.reshape(-1), r.reshape(-1), n, 2, m, 1.0, lam, "pik_box", s, mu_pde=1.0, **HEAT)
    f = host(F.fk_predict_type2(th, 2, m, 1.0, dev(Xq), 1e-6))
    f_o = oracle.predict(th_o, Xq, 1.0, m)
    print(f"PI fit: pred {rel(f, f_o):.2e}")
    assert rel(f, f_o) <= 1e-4


@pytest.mark.parametrize("d,m,n,eps", [(3, 10, 20_000, 1e-6), (10, 50, 2_000, 1e-6), (4, 8, 5_000, 1e-10),
                                        (3, 131, 3_001, 1e-6), (3, 90, 2_001, 1e-10)])  # last two: a pair grid exceeds a CTA (per-pair 2-D passes)
def test_cross_moments_match_oracle(F, oracle, d, m, n, eps):
    X, _ = datagen.dataset(n, d=d, ykind="additive", seed=27)
    t = torch.float32 if eps >= 1e-7 else torch.float64
    Xs = X if eps >= 1e-7 else X.astype(np.float64)
    G = host(F.fk_additive_cross_moments(dev(Xs, t), 1.0, m, eps))
    G_o = oracle.cross_moments(Xs, 1.0, m)
    errs = [check_mu(G[p], G_o[p], 1e-5 if eps >= 1e-7 else 1e-10, eps, f"pair {p}") for p in range(G.shape[0])]
    print(f"cross d={d} m={m} n={n} eps={eps}: max pair err {max(e[0] for e in errs):.2e} elem {max(e[1] for e in errs):.1e}")


def test_additive_fit_end_to_end(F, oracle):
    """C5 shape (d = 10 features, m = 20 here): per-feature moments/rhs (fk_rhs_type1 on column
    views), cross moments, block solve, additive prediction vs the oracle."""
    n, d, m, lam = 10_000, 10, 20, 10_000 ** (-0.8)
    X, Y = datagen.dataset(n, d=d, ykind="additive", seed=28)
    Xq = datagen.dataset(2_000, d=d, seed=29)[0]
    Xd, Yd = dev(X), dev(Y)
    mus = torch.zeros((d, 4 * m + 1), dtype=torch.complex128, device="cuda")
    rs = torch.zeros((d, 2 * m + 1), dtype=torch.complex128, device="cuda")
    for l in range(d):
        F.fk_rhs_type1(Xd[:, l], Yd, 1.0, m, 1e-6, r_out=rs[l], mu_out=mus[l])
    G = F.fk_additive_cross_moments(Xd, 1.0, m, 1e-6)
    th, rep = F.fk_solve(mus, rs, n, d, m, 1.0, lam, "additive", cross=G)
    mu_l = [oracle.moments(X[:, l], 1.0, m) for l in range(d)]
    r_l = [oracle.rhs(X[:, l], Y, 1.0, m) for l in range(d)]
    th_o = oracle.solve_additive(mu_l, r_l, oracle.cross_moments(X, 1.0, m), n, d, m, lam)
    f = host(F.fk_predict_type2(th, d, m, 1.0, dev(Xq), 1e-6, additive=True))
    f_o = oracle.predict_additive(th_o, Xq, 1.0, m)
    print(f"additive fit: theta {rel(host(th), th_o):.2e} pred {rel(f, f_o):.2e} backward {rep['backward_err']:.1e}")
    assert rel(f, f_o) <= 1e-4
    # theta itself through the same (oracle) inputs: the block solve
    th2, _ = F.fk_solve(dev(np.stack(mu_l)), dev(np.stack(r_l)), n, d, m, 1.0, lam, "additive", cross=dev(oracle.cross_moments(X, 1.0, m)))
    assert rel(host(th2), th_o) < 1e-8
    # additive prediction alone
    f2 = host(F.fk_predict_type2(dev(th_o), d, m, 1.0, dev(Xq), 1e-6, additive=True))
    assert rel(f2, f_o) <= 1e-5


@pytest.mark.parametrize("x0", [(0.3141, -0.777), (1.0, -1.0)])
def test_identical_samples_drain_2d(F, x0):
    """2^20 identical samples: every CTA's 1024 threads hammer the same w^2 cells, so the int32
    cells cross the drain threshold many times concurrently (overflow regression).  Closed form:
    mu_q = n e^{-i pi <q, x0>/2}, r_k = (sum Y) e^{-i pi <k, x0>/2}; cross moments of the pair
    (x0_0, x0_1): n e^{-i pi (a x0_0 - b x0_1)/2}."""
    n, m = 1 << 20, 24
    X = torch.tensor(x0, dtype=torch.float32, device="cuda").repeat(n, 1)
    Y = torch.linspace(-1.0, 2.0, n, dtype=torch.float32, device="cuda")
    r, mu = F.fk_rhs_type1(X, Y, 1.0, m, 1e-6)
    q = np.arange(-2 * m, 2 * m + 1)
    ph = lambda k: np.exp(-1j * np.pi * k * np.float64(np.float32(x0[0])) / 2)[:, None] * \
        np.exp(-1j * np.pi * k * np.float64(np.float32(x0[1])) / 2)[None, :]
    mu_cf = n * ph(q)
    k = np.arange(-m, m + 1)
    r_cf = float(Y.double().sum()) * ph(k)
    assert rel(host(mu), mu_cf) <= 1e-5
    assert rel(host(r), r_cf) <= 1e-5
    G = host(F.fk_additive_cross_moments(X, 1.0, m, 1e-6))
    a = np.exp(-1j * np.pi * k * np.float64(np.float32(x0[0])) / 2)[:, None]
    b = np.exp(+1j * np.pi * k * np.float64(np.float32(x0[1])) / 2)[None, :]
    assert rel(G[0], n * a * b) <= 1e-5


@pytest.mark.parametrize("d,m,eps", [(1, 200, 1e-6), (1, 60, 1e-12), (2, 24, 1e-6), (2, 12, 1e-11)])
def test_type1_type2_adjoint(F, d, m, eps):
    """SURVEY P9 across the two GPU transforms: for Hermitian theta, <theta, r> = sum_k conj(theta_k)
    r_k = sum_j Y_j conj(f_theta(X_j)) = sum_j Y_j f_theta(X_j) (f real), with r from fk_rhs_type1
    and f from fk_predict_type2 at the same points."""
    n = 200_000
    X, Y = datagen.dataset(n, d=d, ykind="expcos" if d == 2 else "sin", seed=95)
    X = X.reshape(-1) if d == 1 else X
    t = torch.float32 if eps >= 1e-7 else torch.float64
    Xd, Yd = dev(X, t), dev(Y, t)
    rng = np.random.default_rng(7)
    D = (2 * m + 1) ** d
    th = rng.normal(size=D) + 1j * rng.normal(size=D)
    th = (th + np.conj(th[::-1])) / 2  # Hermitian: theta_{-k} = conj theta_k (lexicographic reversal)
    r, _ = F.fk_rhs_type1(Xd, Yd, 1.0, m, eps)
    f = F.fk_predict_type2(dev(th), d, m, 1.0, Xd, eps)
    lhs = np.sum(np.conj(th) * host(r).reshape(-1))
    rhs = float(torch.dot(Yd.double(), f.double()))
    scale = np.sum(np.abs(th)) * float(Yd.abs().sum())
    print(f"adjoint d={d} m={m} eps={eps}: |lhs-rhs|/scale {abs(lhs - rhs) / scale:.2e}, imag {abs(lhs.imag) / scale:.1e}")
    tol = 1e-6 if eps >= 1e-7 else 1e-11
    assert abs(lhs - rhs) <= tol * scale


def test_host_streamed_additive_matches_device(F):
    """fit.HostStreamerAdditive (pinned SoA host columns, chunked H2D) reproduces the device-resident
    per-feature moments / rhs and the cross moments (same fixed-point sums, chunked)."""
    from paper_2509_02649_b200 import fit

    n, d, m, chunk = 300_001, 4, 12, 1 << 16
    X, Y = datagen.dataset(n, d=d, ykind="additive", seed=96)
    Xs = torch.from_numpy(np.ascontiguousarray(X.T)).pin_memory()
    Yh = torch.from_numpy(Y).pin_memory()
    _, mus, rs, G = fit.additive_buffers(d, m, "cuda")
    fit.HostStreamerAdditive(chunk, d, torch.device("cuda")).moments(Xs, Yh, 1.0, m, 1e-6, mus, rs, G)
    torch.cuda.synchronize()
    Xd = dev(np.ascontiguousarray(X.T)).t()
    Yd = dev(Y)
    G2 = F.fk_additive_cross_moments(Xd, 1.0, m, 1e-6)
    assert rel(host(G), host(G2)) < 1e-12
    for l in range(d):
        r2, mu2 = F.fk_rhs_type1(Xd[:, l], Yd, 1.0, m, 1e-6)
        assert rel(host(mus[l]), host(mu2)) < 1e-12 and rel(host(rs[l]), host(r2)) < 1e-6


@pytest.mark.parametrize("n", [37, 149, 5_003])
def test_cross_moments_balanced_split(F, oracle, n):
    """One pair per CTA spreads an even share of the npairs x n sample-pair units (segments cross
    pair boundaries; with npairs x n < resident CTAs some CTAs get nothing): oracle parity and
    bitwise reproducibility."""
    d, m = 4, 50
    X, _ = datagen.dataset(n, d=d, ykind="additive", seed=29)
    Xd = dev(np.ascontiguousarray(X.T)).t()  # SoA columns, as the bench lays them out
    G1 = host(F.fk_additive_cross_moments(Xd, 1.0, m, 1e-6))
    G2 = host(F.fk_additive_cross_moments(Xd, 1.0, m, 1e-6))
    assert np.array_equal(G1, G2)
    Go = oracle.cross_moments(X, 1.0, m)
    for p in range(G1.shape[0]):
        check_mu(G1[p], Go[p], 1e-5, what=f"pair {p}")


@pytest.mark.parametrize("eps,dt", [(1e-6, "f32"), (1e-10, "f64")])
@pytest.mark.parametrize("what", ["type1_2d", "cross", "cross_large_m"])
def test_range_flag_2d_and_cross(F, oracle, what, eps, dt):
    """A coordinate outside [-L, L] (or NaN) sets FK_E_RANGE in d_status; the sample is skipped
    (d = 2: everywhere; cross moments: in the pairs that use that coordinate) and the other
    samples' sums are unaffected."""
    t = torch.float32 if dt == "f32" else torch.float64
    X, Y = datagen.dataset(301, d=3, ykind="additive", seed=33)
    X = X.astype(np.float64)
    X[17, 1] = 1.5
    X[200, 0] = np.nan
    good = np.ones(301, bool)
    good[[17, 200]] = False
    ds = torch.zeros(1, dtype=torch.int32, device="cuda")
    if what == "type1_2d":
        m = 12
        X2 = X[:, :2]
        Xd = dev(X2, t)
        r, mu = F.fk_rhs_type1(Xd, dev(Y, t), 1.0, m, eps, d_status=ds)
        check_mu(host(mu), oracle.moments(X2[good], 1.0, m), (1e-5 if dt == "f32" else 1e-10))
        check_r(host(r), oracle.rhs(X2[good], Y[good].astype(np.float64), 1.0, m), Y[good].astype(np.float64), (1e-5 if dt == "f32" else 1e-10))
    else:
        m = 10 if what == "cross" else 130
        G = host(F.fk_additive_cross_moments(dev(X, t), 1.0, m, eps, d_status=ds))
        # a bad coordinate removes the sample from the pairs that use that coordinate only
        # (as the per-feature 1-D passes skip it only in their own column)
        for p, (l1, l2) in enumerate([(0, 1), (0, 2), (1, 2)]):
            ok = np.all(np.isfinite(X[:, [l1, l2]]) & (np.abs(X[:, [l1, l2]]) <= 1.0), axis=1)
            Go = oracle.cross_moments(X[ok][:, [l1, l2]], 1.0, m)[0]
            check_mu(G[p], Go, 1e-5 if dt == "f32" else 1e-10, eps, f"pair {p}")
    assert int(ds.item()) & F.FK_E_RANGE
    with pytest.raises(F.FkError):
        if what == "type1_2d":
            F.fk_moments_type1(dev(X[:, :2], t), 1.0, 12, eps)
        else:
            F.fk_additive_cross_moments(dev(X, t), 1.0, 10, eps)


@pytest.mark.parametrize("eps", [1e-6, 1e-10])
@pytest.mark.parametrize("d,additive", [(1, False), (2, False), (3, True)])
def test_predict_range_flag(F, oracle, d, additive, eps):
    """A NaN query flags FK_E_RANGE and yields NaN at that query only.  A query outside [-L, L]
    either does the same or -- when it still lies on the grid (within the window's halo; the
    type-2 sum is 4L-periodic, so the value is exact there) -- equals the oracle's sum."""
    m = 9
    t = torch.float32 if eps >= 1e-7 else torch.float64
    rng = np.random.default_rng(d)
    D = d * (2 * m + 1) if additive else (2 * m + 1) ** d
    th = rng.normal(size=D) + 1j * rng.normal(size=D)
    Xq = datagen.dataset(257, d=d, seed=34)[0].astype(np.float64)
    Xq[5, 0] = -1.25
    Xq[100, d - 1] = np.nan
    Xq = Xq.reshape(-1) if d == 1 else Xq
    ds = torch.zeros(1, dtype=torch.int32, device="cuda")
    f = host(F.fk_predict_type2(dev(th), d, m, 1.0, dev(Xq, t), eps, additive=additive, d_status=ds))
    assert int(ds.item()) & F.FK_E_RANGE
    assert np.isnan(f[100])
    ok = np.ones(257, bool)
    ok[100] = False
    if np.isnan(f[5]):
        ok[5] = False
    fo = oracle.predict_additive(th, Xq[ok], 1.0, m) if additive else oracle.predict(th, Xq[ok], 1.0, m)
    assert rel(f[ok], np.real(fo)) <= (1e-5 if eps >= 1e-7 else 1e-10)
