"""GPU parity of the regularisation path (§8(f) NEXT-1): fk_solve_path returns
theta(lambda) for many lambda from one eigendecomposition; each row must match the oracle's dense
solve at that lambda (oracle.solve / oracle.solve_additive), and the Cholesky fk_solve."""
import numpy as np
import pytest

import datagen
from gpu_util import dev, fk, host, rel

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

HEAT = dict(alpha=[[1, 0], [0, 2]], a_alpha=[1.0, -1.0])
LAMS = list(np.logspace(-8, 0, 9))


@pytest.fixture(scope="module")
def F():
    assert torch.cuda.is_available()
    return fk()


@pytest.mark.parametrize("d,m,kind,s", [(1, 40, "sobolev", 2.0), (1, 25, "lowbias", 1.0), (2, 8, "sobolev", 2.0),
                                        (2, 6, "pik_box", 2.0)])
def test_path_matches_oracle(F, oracle, d, m, kind, s):
    n = 20_000
    X, Y = datagen.dataset(n, d=d, ykind="expcos" if d == 2 else "sin", seed=61)
    mu, r = oracle.moments(X, 1.0, m), oracle.rhs(X, Y, 1.0, m)
    kw = dict(mu_pde=1.0, box=[[-1.0, 0.5], [-0.5, 1.0]], **HEAT) if kind == "pik_box" else {}
    th = host(F.fk_solve_path(dev(mu.reshape(-1)), dev(r.reshape(-1)), n, d, m, 1.0, LAMS, kind, s, **kw))
    assert th.shape == (len(LAMS), (2 * m + 1) ** d)
    kw_o = dict(kw, L=1.0) if kind == "pik_box" else {}
    errs = [rel(th[l], oracle.solve(mu, r, n, d, m, lam, kind, s, **kw_o)) for l, lam in enumerate(LAMS)]
    print(f"path d={d} m={m} {kind}: max err {max(errs):.2e}")
    assert max(errs) < 1e-6


def test_path_additive(F, oracle):
    n, d, m = 8_000, 4, 10
    X, Y = datagen.dataset(n, d=d, ykind="additive", seed=62)
    mu_l = [oracle.moments(X[:, l], 1.0, m) for l in range(d)]
    r_l = [oracle.rhs(X[:, l], Y, 1.0, m) for l in range(d)]
    G = oracle.cross_moments(X, 1.0, m)
    lams = [1e-6, 1e-4, 1e-2]
    th = host(F.fk_solve_path(dev(np.stack(mu_l)), dev(np.stack(r_l)), n, d, m, 1.0, lams, "additive", cross=dev(G)))
    errs = [rel(th[l], oracle.solve_additive(mu_l, r_l, G, n, d, m, lam)) for l, lam in enumerate(lams)]
    print(f"path additive: max err {max(errs):.2e}")
    assert max(errs) < 1e-6


def test_path_agrees_with_cholesky_and_colloc(F, oracle):
    """PIK collocation system along the path vs fk_solve (Cholesky) at each lambda."""
    n, nr, d, m = 20_000, 4_000, 2, 8
    X, Y = datagen.dataset(n, d=d, ykind="expcos", seed=63)
    Xr = datagen.dataset(nr, d=d, seed=64)[0]
    mu, r, mur = dev(oracle.moments(X, 1.0, m).reshape(-1)), dev(oracle.rhs(X, Y, 1.0, m).reshape(-1)), dev(
        oracle.moments(Xr, 1.0, m).reshape(-1))
    lams = [1e-7, 1e-5, 1e-3]
    kw = dict(mu_pde=1.0, colloc_moments=mur, n_colloc=nr, **HEAT)
    th = host(F.fk_solve_path(mu, r, n, d, m, 1.0, lams, "pik_colloc", 2.0, **kw))
    for l, lam in enumerate(lams):
        ch, _ = F.fk_solve(mu, r, n, d, m, 1.0, lam, "pik_colloc", 2.0, **kw)
        assert rel(th[l], host(ch)) < 1e-7


def test_path_rejects_bad_lambda(F):
    mu = torch.zeros(4 * 3 + 1, dtype=torch.complex128, device="cuda")
    r = torch.zeros(2 * 3 + 1, dtype=torch.complex128, device="cuda")
    with pytest.raises(F.FkError):
        F.fk_solve_path(mu, r, 10, 1, 3, 1.0, [1e-3, 0.0])


@pytest.mark.parametrize("d,m,kind", [(1, 30, "sobolev"), (2, 6, "sobolev"), (4, 8, "additive"), (2, 6, "pik_box")])
def test_path_validate_matches_direct_prediction(F, oracle, d, m, kind):
    """Held-out risk from validation moments == mean (Y - f(x))^2 by direct prediction (oracle)."""
    n, nv = 10_000, 3_000
    yk = "additive" if kind == "additive" else ("expcos" if d == 2 else "sin")
    X, Y = datagen.dataset(n, d=d, ykind=yk, seed=65)
    Xv, Yv = datagen.dataset(nv, d=d, ykind=yk, seed=66)
    lams = [1e-7, 1e-5, 1e-3, 1e-1]
    if kind == "additive":
        args = [dev(np.stack([oracle.moments(X[:, l], 1.0, m) for l in range(d)])),
                dev(np.stack([oracle.rhs(X[:, l], Y, 1.0, m) for l in range(d)]))]
        kw = dict(cross=dev(oracle.cross_moments(X, 1.0, m)))
        mu_v = dev(np.stack([oracle.moments(Xv[:, l], 1.0, m) for l in range(d)]))
        r_v = dev(np.stack([oracle.rhs(Xv[:, l], Yv, 1.0, m) for l in range(d)]))
        kv = dict(cross_v=dev(oracle.cross_moments(Xv, 1.0, m)))
    else:
        args = [dev(oracle.moments(X, 1.0, m).reshape(-1)), dev(oracle.rhs(X, Y, 1.0, m).reshape(-1))]
        kw = dict(mu_pde=1.0, box=[[-1.0, 0.5], [-0.5, 1.0]], **HEAT) if kind == "pik_box" else {}
        kv = {}
        mu_v, r_v = dev(oracle.moments(Xv, 1.0, m).reshape(-1)), dev(oracle.rhs(Xv, Yv, 1.0, m).reshape(-1))
    th = F.fk_solve_path(*args, n, d, m, 1.0, lams, kind, 2.0, **kw)
    yy = float(np.dot(Yv.astype(np.float64), Yv.astype(np.float64)))
    risk = host(F.fk_path_validate(th, mu_v, r_v, nv, d, m, 1.0, kind, yy, **kv))
    thh = host(th)
    pred = oracle.predict_additive if kind == "additive" else oracle.predict
    direct = np.array([np.mean((Yv.astype(np.float64) - np.real(pred(thh[l], Xv, 1.0, m))) ** 2) for l in range(len(lams))])
    print(f"validate d={d} {kind}: {risk} vs {direct}")
    assert np.max(np.abs(risk - direct) / direct) < 1e-9


def test_grid_search_end_to_end(F, oracle):
    from paper_2509_02649_b200 import fit

    X, Y = datagen.dataset(20_000, d=1, ykind="sin", seed=67)
    Xv, Yv = datagen.dataset(5_000, d=1, ykind="sin", seed=68)
    lams = list(np.logspace(-9, 0, 40))
    g = fit.grid_search(dev(X.reshape(-1)), dev(Y), dev(Xv.reshape(-1)), dev(Yv), 1.0, 30, lams, "sobolev", 2.0)
    direct = [np.mean((Yv - oracle.predict(host(g.thetas[l]), Xv, 1.0, 30).real) ** 2) for l in range(len(lams))]
    # fp32 type-1 moments (eps 1e-6): the chosen lambda is optimal up to that accuracy
    assert direct[g.best] <= min(direct) * (1 + 1e-4)
    assert abs(float(g.risk[g.best]) - direct[g.best]) / direct[g.best] < 1e-3


@pytest.mark.parametrize("kind,d", [("sobolev", 1), ("additive", 3)])
def test_grid_search_distributed_single_rank(F, kind, d):
    """fit.grid_search_distributed on one rank (no process group) = fit.grid_search."""
    from paper_2509_02649_b200 import fit

    yk = "additive" if kind == "additive" else "sin"
    X, Y = datagen.dataset(30_000, d=d, ykind=yk, seed=97)
    Xv, Yv = datagen.dataset(8_000, d=d, ykind=yk, seed=98)
    Xd = dev(X.reshape(-1) if d == 1 else X)
    Xvd = dev(Xv.reshape(-1) if d == 1 else Xv)
    lams = list(np.logspace(-8, -1, 12))
    g1 = fit.grid_search(Xd, dev(Y), Xvd, dev(Yv), 1.0, 12, lams, kind, 2.0)
    g2 = fit.grid_search_distributed(Xd, dev(Y), 30_000, Xvd, dev(Yv), 8_000, 1.0, 12, lams, kind, 2.0)
    assert g1.best == g2.best
    assert torch.allclose(g1.theta, g2.theta, rtol=0, atol=1e-12 * float(g1.theta.abs().max()))
    assert torch.allclose(g1.risk, g2.risk, rtol=1e-12, atol=0)
