"""Degenerate small truncation levels (m = 1..3, the rate experiments' first points): every
type-1 / cross / type-2 path against the oracle.  Regression test: at m <= 2 the sigma = 2 ES
grids were smaller than their own tile (nf/2 + w + 4 cells) and lost accuracy (5e-3)."""
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


def _tol(eps):
    return 1e-5 if eps >= 1e-7 else 1e-10


@pytest.mark.parametrize("m", [1, 2, 3])
@pytest.mark.parametrize("eps", [1e-6, 1e-12])
def test_small_m_type1(F, oracle, m, eps):
    t = torch.float32 if eps >= 1e-7 else torch.float64
    X1, Y1 = datagen.dataset(3_000, d=1, seed=71)
    X2, Y2 = datagen.dataset(3_000, d=2, ykind="expcos", seed=72)
    X3, _ = datagen.dataset(3_000, d=3, ykind="additive", seed=73)
    for X, Y in ((X1.reshape(-1), Y1), (X2, Y2)):
        Xc = X if t == torch.float32 else X.astype(np.float64)
        Yc = Y if t == torch.float32 else Y.astype(np.float64)
        r, mu = F.fk_rhs_type1(dev(Xc), dev(Yc), 1.0, m, eps)
        check_mu(host(mu), oracle.moments(Xc, 1.0, m), _tol(eps))
        check_r(host(r), oracle.rhs(Xc, Yc, 1.0, m), Yc, _tol(eps))
    X3c = X3 if t == torch.float32 else X3.astype(np.float64)
    G = host(F.fk_additive_cross_moments(dev(X3c), 1.0, m, eps))
    Go = oracle.cross_moments(X3c, 1.0, m)
    for p in range(3):
        check_mu(G[p], Go[p], _tol(eps), what=f"pair {p}")


@pytest.mark.parametrize("m", [1, 2, 3])
@pytest.mark.parametrize("eps", [1e-6, 1e-12])
def test_small_m_predict(F, oracle, m, eps):
    rng = np.random.default_rng(m)
    t = torch.float32 if eps >= 1e-7 else torch.float64
    for d, additive in ((1, False), (2, False), (4, True)):
        D = d * (2 * m + 1) if additive else (2 * m + 1) ** d
        th = rng.normal(size=D) + 1j * rng.normal(size=D)
        Xq = datagen.dataset(2_001, d=d, seed=74)[0]
        Xq = Xq.reshape(-1) if d == 1 else Xq
        Xqc = Xq if t == torch.float32 else Xq.astype(np.float64)
        f = host(F.fk_predict_type2(dev(th), d, m, 1.0, dev(Xqc), eps, additive=additive))
        fo = oracle.predict_additive(th, Xqc, 1.0, m) if additive else oracle.predict(th, Xqc, 1.0, m)
        assert rel(f, np.real(fo)) <= _tol(eps), (d, additive)
