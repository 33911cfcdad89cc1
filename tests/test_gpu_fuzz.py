"""Randomised parity (hypothesis): type-1 moments / rhs for d = 1, 2, cross moments and type-2
predictions at random shapes, sample counts (incl. ragged tails and n < one CTA's threads),
accuracy modes and input precisions, against the fp64 oracle."""
import numpy as np
import pytest

import datagen
from gpu_util import dev, fk, host, rel, check_mu, check_r

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
hyp = pytest.importorskip("hypothesis")
from hypothesis import given, settings, strategies as st  # noqa: E402


@pytest.fixture(scope="module")
def F():
    assert torch.cuda.is_available()
    return fk()


def _tol(eps):
    return 10 * eps  # reading R7: requested relative l2 accuracy eps, gate 10 eps


@settings(max_examples=80, deadline=None, derandomize=True)
@given(d=st.sampled_from([1, 2]), m=st.integers(1, 48), n=st.integers(1, 6000), eps=st.sampled_from([1e-6, 1e-9, 1e-11]),
       xkind=st.sampled_from(["uniform", "gaussian"]), f64=st.booleans(), seed=st.integers(0, 10_000))
def test_type1_random_shapes(F, oracle, d, m, n, eps, xkind, f64, seed):
    X, Y = datagen.dataset(n, d=d, xkind=xkind, ykind="expcos" if d == 2 else "sin", seed=seed)
    if f64:
        X, Y = X.astype(np.float64), Y.astype(np.float64)
    Xc = X.reshape(-1) if d == 1 else X
    r, mu = F.fk_rhs_type1(dev(Xc), dev(Y), 1.0, m, eps)
    check_mu(host(mu), oracle.moments(Xc, 1.0, m), _tol(eps), eps)
    check_r(host(r), oracle.rhs(Xc, Y.astype(np.float64), 1.0, m), Y.astype(np.float64), _tol(eps), eps)


@settings(max_examples=50, deadline=None, derandomize=True)
@given(d=st.integers(2, 5), m=st.integers(1, 30), n=st.integers(1, 3000), eps=st.sampled_from([1e-6, 1e-10]),
       seed=st.integers(0, 10_000))
def test_cross_random_shapes(F, oracle, d, m, n, eps, seed):
    X, _ = datagen.dataset(n, d=d, ykind="additive", seed=seed)
    Xc = X if eps >= 1e-7 else X.astype(np.float64)
    G = host(F.fk_additive_cross_moments(dev(Xc), 1.0, m, eps))
    Go = oracle.cross_moments(Xc, 1.0, m)
    for p in range(G.shape[0]):
        check_mu(G[p], Go[p], _tol(eps), eps, f"pair {p}")


@settings(max_examples=50, deadline=None, derandomize=True)
@given(d=st.sampled_from([1, 2, 3]), m=st.integers(1, 40), nq=st.integers(1, 4000), eps=st.sampled_from([1e-6, 1e-10]),
       seed=st.integers(0, 10_000))
def test_predict_random_shapes(F, oracle, d, m, nq, eps, seed):
    additive = d == 3
    rng = np.random.default_rng(seed)
    D = d * (2 * m + 1) if additive else (2 * m + 1) ** d
    th = rng.normal(size=D) + 1j * rng.normal(size=D)
    Xq = datagen.dataset(nq, d=d, seed=seed + 1)[0]
    Xq = Xq.reshape(-1) if d == 1 else Xq
    Xq = Xq if eps >= 1e-7 else Xq.astype(np.float64)
    f = host(F.fk_predict_type2(dev(th), d, m, 1.0, dev(Xq), eps, additive=additive))
    fo = oracle.predict_additive(th, Xq, 1.0, m) if additive else oracle.predict(th, Xq, 1.0, m)
    assert rel(f, np.real(fo)) <= _tol(eps)


HEAT = dict(alpha=[[1, 0], [0, 2]], a_alpha=[1.0, -1.0], box=[[-1.0, 1.0], [-1.0, 1.0]])


@settings(max_examples=40, deadline=None, derandomize=True)
@given(d=st.sampled_from([1, 2]), m=st.integers(1, 24), n=st.integers(3, 3000), kind=st.sampled_from(["sobolev", "lowbias", "pik_box"]),
       loglam=st.floats(-9, -1), s=st.sampled_from([1.0, 1.5, 2.0]), seed=st.integers(0, 10_000))
def test_solve_random_systems(F, oracle, d, m, n, kind, loglam, s, seed):
    """fk_solve on the oracle's moments at random shapes, penalties and lambdas: the backward error
    in the oracle's own system (which tracks conditioning-independent accuracy, reading R8)."""
    if kind == "pik_box" and d != 2:
        kind = "sobolev"
    lam = 10.0 ** loglam
    X, Y = datagen.dataset(n, d=d, ykind="expcos" if d == 2 else "sin", seed=seed)
    Xc = X.reshape(-1) if d == 1 else X
    mu, r = oracle.moments(Xc, 1.0, m), oracle.rhs(Xc, Y, 1.0, m)
    kw = dict(mu_pde=1.0, **HEAT) if kind == "pik_box" else {}
    th, rep = F.fk_solve(dev(mu.reshape(-1)), dev(r.reshape(-1)), n, d, m, 1.0, lam, kind, s, **kw)
    A = oracle.assemble(mu, n, d, m, lam, kind, s, **(dict(kw, L=1.0) if kw else {}))
    assert rep["info"] == 0
    assert oracle.backward_error(A, host(th), r.reshape(-1) / n) < 1e-11
