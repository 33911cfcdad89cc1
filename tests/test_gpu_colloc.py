"""GPU parity of the collocation physics-informed estimator (§8(f) NEXT-2): the
collocation points' moments come from the same type-1 pass (fk_moments_type1), the solve adds
mu_pde n_r^{-1} D^* T(mu_r) D."""
import numpy as np
import pytest

import datagen
from gpu_util import dev, fk, host, rel

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

HEAT = dict(alpha=[[1, 0], [0, 2]], a_alpha=[1.0, -1.0])


@pytest.fixture(scope="module")
def F():
    assert torch.cuda.is_available()
    return fk()


@pytest.mark.parametrize("d,m", [(1, 40), (2, 12)])
def test_colloc_solve_matches_oracle(F, oracle, d, m):
    n, nr, s, lam = 20_000, 5_000, 2.0, 1e-5
    X, Y = datagen.dataset(n, d=d, ykind="expcos" if d == 2 else "sin", seed=51)
    Xr = datagen.dataset(nr, d=d, seed=52)[0] * np.float32(0.8)  # collocation points in a sub-domain
    pde = HEAT if d == 2 else dict(alpha=[[1], [0]], a_alpha=[1.0, -1.0])  # d=1: f' - f
    mu, r, mur = oracle.moments(X, 1.0, m), oracle.rhs(X, Y, 1.0, m), oracle.moments(Xr, 1.0, m)
    th_o = oracle.solve(mu, r, n, d, m, lam, "pik_colloc", s, mu_pde=1.0, L=1.0, mu_colloc=mur, n_colloc=nr, **pde)
    th, rep = F.fk_solve(dev(mu.reshape(-1)), dev(r.reshape(-1)), n, d, m, 1.0, lam, "pik_colloc", s, mu_pde=1.0,
                         colloc_moments=dev(mur.reshape(-1)), n_colloc=nr, **pde)
    print(f"colloc d={d} m={m}: {rel(host(th), th_o):.2e} backward {rep['backward_err']:.1e}")
    assert rep["backward_err"] < 1e-11
    assert rel(host(th), th_o) < 1e-6


def test_colloc_fit_end_to_end(F, oracle):
    """Whole GPU path: moments of data and collocation points by the type-1 kernel, collocation-PI
    solve, prediction -- against the oracle's fit (predictions within 1e-4)."""
    n, nr, m, s = 40_000, 8_000, 14, 2.0
    lam = n ** (-2 / 3)
    X, Y = datagen.dataset(n, d=2, ykind="expcos", seed=53)
    Xr = datagen.dataset(nr, d=2, seed=54)[0]
    Xq = datagen.dataset(2_000, d=2, seed=55)[0]
    th_o, _, _ = oracle.fit(X, Y, 1.0, m, lam, "pik_colloc", s, mu_pde=1.0, X_colloc=Xr, **HEAT)
    r, mu = F.fk_rhs_type1(dev(X), dev(Y), 1.0, m, 1e-6)
    mur = F.fk_moments_type1(dev(Xr), 1.0, m, 1e-6)
    th, _ = F.fk_solve(mu.reshape(-1), r.reshape(-1), n, 2, m, 1.0, lam, "pik_colloc", s, mu_pde=1.0, colloc_moments=mur.reshape(-1),
                       n_colloc=nr, **HEAT)
    f = host(F.fk_predict_type2(th, 2, m, 1.0, dev(Xq), 1e-6))
    assert rel(f, oracle.predict(th_o, Xq, 1.0, m)) <= 1e-4
