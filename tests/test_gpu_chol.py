"""The tile dataflow Cholesky (csrc/chol.cu) against cuSOLVER potrf and the oracle's dense solve:
the same fit systems solved with FK_CHOL=tiles and FK_CHOL=cusolver."""
import os

import numpy as np
import pytest

import datagen
from gpu_util import dev, fk, host, rel

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
HEAT = dict(alpha=[[1, 0], [0, 2]], a_alpha=[1.0, -1.0], box=[[-1.0, 1.0], [-1.0, 1.0]])


@pytest.fixture(scope="module")
def F():
    assert torch.cuda.is_available()
    return fk()


def _solve(F, how, *args, **kw):
    old = os.environ.get("FK_CHOL")
    os.environ["FK_CHOL"] = how
    try:
        th, rep = F.fk_solve(*args, **kw)
    finally:
        if old is None:
            del os.environ["FK_CHOL"]
        else:
            os.environ["FK_CHOL"] = old
    return host(th), rep


@pytest.mark.parametrize("d,m,kind,s,lam", [(1, 3, "sobolev", 2.0, 1e-3), (1, 50, "sobolev", 2.0, 1e-4), (1, 1000, "sobolev", 1.0, 2.15e-7),
                                            (1, 700, "lowbias", 1.0, 1e-6), (2, 32, "pik_box", 2.0, 1e-5), (2, 20, "sobolev", 2.0, 1e-6)])
def test_tiles_match_cusolver_and_oracle(F, oracle, d, m, kind, s, lam):
    n = 50_000
    X, Y = datagen.dataset(n, d=d, ykind="expcos" if d == 2 else "sin", seed=81)
    mu, r = oracle.moments(X, 1.0, m), oracle.rhs(X, Y, 1.0, m)
    kw = dict(mu_pde=1.0, **HEAT) if kind == "pik_box" else {}
    args = (dev(mu.reshape(-1)), dev(r.reshape(-1)), n, d, m, 1.0, lam, kind, s)
    th_t, rep_t = _solve(F, "tiles", *args, **kw)
    th_c, rep_c = _solve(F, "cusolver", *args, **kw)
    print(f"d={d} m={m} {kind}: tiles {rep_t['ms']:.3f} ms  cusolver {rep_c['ms']:.3f} ms  diff {rel(th_t, th_c):.2e} "
          f"backward {rep_t['backward_err']:.1e} / {rep_c['backward_err']:.1e}")
    assert rep_t["info"] == 0
    assert rep_t["backward_err"] <= max(10 * rep_c["backward_err"], 1e-14)
    if (2 * m + 1) ** d <= 4225:
        kw_o = dict(kw, L=1.0) if kind == "pik_box" else {}
        th_o = oracle.solve(mu, r, n, d, m, lam, kind, s, **kw_o)
        assert rel(th_t, th_o) <= max(10 * rel(th_c, th_o), 1e-12)


def test_tiles_additive(F, oracle):
    n, d, m, lam = 20_000, 6, 40, 1e-5
    X, Y = datagen.dataset(n, d=d, ykind="additive", seed=82)
    mu_l = np.stack([oracle.moments(X[:, l], 1.0, m) for l in range(d)])
    r_l = np.stack([oracle.rhs(X[:, l], Y, 1.0, m) for l in range(d)])
    G = oracle.cross_moments(X, 1.0, m)
    th_t, rep_t = _solve(F, "tiles", dev(mu_l), dev(r_l), n, d, m, 1.0, lam, "additive", cross=dev(G))
    th_o = oracle.solve_additive(list(mu_l), list(r_l), G, n, d, m, lam)
    assert rep_t["backward_err"] < 1e-13
    assert rel(th_t, th_o) < 1e-8


def test_tiles_report_not_spd(F):
    """A system that is not positive definite (negative moments) reports FK_E_SOLVE with the pivot."""
    m = 40
    mu = torch.zeros(4 * m + 1, dtype=torch.complex128, device="cuda")
    mu[2 * m] = -1000.0  # mu_0 < 0: A = -I*1000/n + lambda R is indefinite
    r = torch.ones(2 * m + 1, dtype=torch.complex128, device="cuda")
    os.environ["FK_CHOL"] = "tiles"
    try:
        with pytest.raises(F.FkError):
            F.fk_solve(mu, r, 1000, 1, m, 1.0, 1e-6, "sobolev", 1.0)
    finally:
        del os.environ["FK_CHOL"]


def test_tiles_report_not_spd_with_partial_tasks(F):
    """N >= 3200 runs the partial-accumulation (U) tasks; an indefinite system still reports."""
    m = 1700  # D = 3401, N = 3402: 107 tile columns
    mu = torch.zeros(4 * m + 1, dtype=torch.complex128, device="cuda")
    mu[2 * m] = -1000.0
    r = torch.ones(2 * m + 1, dtype=torch.complex128, device="cuda")
    os.environ["FK_CHOL"] = "tiles"
    try:
        with pytest.raises(F.FkError):
            F.fk_solve(mu, r, 1000, 1, m, 1.0, 1e-9, "sobolev", 1.0)
    finally:
        del os.environ["FK_CHOL"]


@pytest.mark.parametrize("m", [14, 15, 16, 30, 31, 47, 63, 1278, 1279, 1280])
def test_tiles_size_sweep(F, oracle, m):
    """Tile-boundary sizes of the dataflow Cholesky (N = 2m + 2: partial last tile, exact multiples
    of 32, the one-tile-column-per-step structure of the diagonal task with its trailing TRSM warp,
    and the switch to the partial-accumulation tasks at 80 tile columns, N = 2560) against
    cuSOLVER potrf on the same d = 1 fit system."""
    n = 3000
    X, Y = datagen.dataset(n, d=1, ykind="sin", seed=90 + m)
    mu, r = oracle.moments(X, 1.0, m), oracle.rhs(X, Y, 1.0, m)
    args = (dev(mu.reshape(-1)), dev(r.reshape(-1)), n, 1, m, 1.0, 1e-5, "sobolev", 1.0)
    th_t, rep_t = _solve(F, "tiles", *args)
    th_c, rep_c = _solve(F, "cusolver", *args)
    assert rep_t["info"] == 0
    assert rep_t["backward_err"] <= max(10 * rep_c["backward_err"], 1e-14)
    assert rel(th_t, th_c) <= 1e-9
