"""Pins of the CPU oracle against facts fixed by the paper and by mathematics (not by itself).

Each test names the pin of DESIGN.md §Oracle pins (P1..P9) and the passage it follows.  A
plausible mistake in the oracle (sign of the exponent, 1/n vs n lambda, Toeplitz index order,
conjugate-transposed additive block, PDE symbol sign, box integral order) fails at least one.
"""
import math
import os

import numpy as np
import pytest

import datagen

RNG = np.random.default_rng(12345)


def rel(a, b):
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# --------------------------------------------------------------------------------------------
# P5: special cases and invariants of the exponential sums
# --------------------------------------------------------------------------------------------
def test_single_point_at_origin(oracle):
    """n=1, X=0: every moment is exp(0) = 1 and r_k = Y."""
    mu = oracle.moments(np.zeros((1, 2)), 1.0, 3)
    assert np.all(mu == 1.0)
    r = oracle.rhs(np.zeros((1, 1)), [2.5], 1.0, 4)
    assert np.allclose(r, 2.5, rtol=0, atol=0)


def test_zero_mode_counts_samples(oracle):
    """mu_0 = n and r_0 = sum Y (the q=0 term of the sums)."""
    X, Y = datagen.dataset(3000, d=2, seed=3)
    mu = oracle.moments(X, 1.0, 5)
    r = oracle.rhs(X, Y, 1.0, 5)
    assert abs(mu[10, 10] - 3000) < 1e-9
    assert abs(r[5, 5] - np.sum(Y.astype(np.float64))) < 1e-9


def test_hermitian_symmetry(oracle):
    """mu_{-q} = conj(mu_q) for real points (every q is summed independently by the oracle)."""
    X, Y = datagen.dataset(2000, d=2, seed=5)
    mu = oracle.moments(X, 1.0, 6)
    assert np.max(np.abs(mu[::-1, ::-1] - np.conj(mu))) < 1e-10
    r = oracle.rhs(X, Y, 1.0, 6)
    assert np.max(np.abs(r[::-1, ::-1] - np.conj(r))) < 1e-10


def test_shift_theorem(oracle):
    """X -> X + delta multiplies mu_q by exp(-i pi q delta / 2L): pins the sign and the pi/2L scale."""
    L = 1.7
    X = RNG.uniform(-1.0, 1.0, size=500)
    delta = 0.3125
    m = 7
    a = oracle.moments(X, L, m)
    b = oracle.moments(X + delta, L, m)
    q = np.arange(-2 * m, 2 * m + 1)
    assert rel(b, a * np.exp(-1j * np.pi * q * delta / (2 * L))) < 1e-12


def test_linearity_and_shard_additivity(oracle):
    """Unnormalised sums add over shards (the multi-GPU reduction relies on it)."""
    X, Y = datagen.dataset(1500, seed=9)
    full = oracle.rhs(X, Y, 1.0, 9)
    parts = oracle.rhs(X[:700], Y[:700], 1.0, 9) + oracle.rhs(X[700:], Y[700:], 1.0, 9)
    assert rel(parts, full) < 1e-13
    assert rel(oracle.rhs(X, 3.0 * Y.astype(np.float64), 1.0, 9), 3.0 * full) < 1e-14


# --------------------------------------------------------------------------------------------
# P1 / P2: closed forms for equispaced-replicated points (geometric series)
# --------------------------------------------------------------------------------------------
def _closed_mu(N, r, q):
    q = np.asarray(q)
    out = np.zeros(q.shape, dtype=np.complex128)
    odd = (np.abs(q) % 2) == 1
    qa = np.abs(q[odd])
    out[odd] = r * (-1.0) ** ((qa - 1) // 2) / np.sin(qa * np.pi / (2 * N))
    out[q == 0] = r * N
    return out


def _closed_r01(N, r, k):
    k = np.asarray(k)
    out = np.zeros(k.shape, dtype=np.complex128)
    odd = (np.abs(k) % 2) == 1
    ko = k[odd].astype(np.float64)
    out[odd] = r * np.exp(1j * ko * np.pi / 2) * np.exp(-1j * ko * np.pi / (2 * N)) * 2.0 / (1 - np.exp(-2j * np.pi * ko / N))
    out[k == 0] = r * N / 2
    return out


@pytest.mark.parametrize("N,r,m", [(64, 3, 20), (256, 2, 100)])
def test_equispaced_closed_form(oracle, N, r, m):
    """P1: mu_q = r N (q=0), 0 (q even), r (-1)^((|q|-1)/2) / sin(|q| pi / 2N) (q odd), for
    x_i = -1 + (2i+1)/N each repeated r times, in a scrambled order (L = 1)."""
    n = N * r
    X, Y = datagen.equispaced(n, 0, n, a=2 * 7 + 1 if math.gcd(15, n) == 1 else 17, b=5, N=N)
    assert sorted(np.round((X.ravel() + 1) * N / 2 - 0.5).astype(int).tolist()) == sorted(list(range(N)) * r)
    mu = oracle.moments(X, 1.0, m)
    q = np.arange(-2 * m, 2 * m + 1)
    assert rel(mu, _closed_mu(N, r, q)) < 1e-13
    rr = oracle.rhs(X, Y, 1.0, m)
    k = np.arange(-m, m + 1)
    assert rel(rr, _closed_r01(N, r, k)) < 1e-13


# --------------------------------------------------------------------------------------------
# P4: moments / rhs against the dense design matrix
# --------------------------------------------------------------------------------------------
@pytest.mark.parametrize("d,m", [(1, 5), (2, 3)])
def test_toeplitz_equals_dense_gram(oracle, d, m):
    """Phi = (phi(X_1)|...|phi(X_n))^*, phi_k(x) = exp(-i pi <k,x>/2L).
    Phi^* Phi must equal the d-level Toeplitz matrix T[k1,k2] = mu_{k1-k2} and
    Phi^* Y must equal r."""
    L = 1.3
    X = RNG.uniform(-L, L, size=(80, d))
    Y = RNG.normal(size=80)
    k = oracle.mode_grid(d, m)
    phi = np.exp(-1j * np.pi * (X @ k.T) / (2 * L))  # row j = phi(X_j)^T
    Phi = np.conj(phi)  # row j = phi(X_j)^*
    gram = Phi.conj().T @ Phi
    T = oracle.toeplitz_from_moments(oracle.moments(X, L, m), d, m)
    assert np.max(np.abs(gram - T)) < 1e-11
    assert np.max(np.abs(Phi.conj().T @ Y - oracle.rhs(X, Y, L, m).ravel())) < 1e-11


def test_cross_moments_identities(oracle):
    """P6: a duplicated column gives G_{a,b} = mu_{a-b}; a zero column gives G_{a,b} = mu_a;
    and the block equals Phi_{l1}^* Phi_{l2} built from the feature map."""
    m = 4
    n = 300
    x = RNG.uniform(-1, 1, size=n)
    X = np.stack([x, x, np.zeros(n), RNG.uniform(-1, 1, size=n)], axis=1)
    G = oracle.cross_moments(X, 1.0, m)  # pairs (0,1),(0,2),(0,3),(1,2),(1,3),(2,3)
    mu = oracle.moments(x, 1.0, m)
    a = np.arange(-m, m + 1)
    assert np.max(np.abs(G[0] - mu[(a[:, None] - a[None, :]) + 2 * m])) < 1e-11
    assert np.max(np.abs(G[1] - mu[a + 2 * m][:, None] * np.ones((1, 2 * m + 1)))) < 1e-11
    Phi = [np.exp(1j * np.pi * np.outer(X[:, l], a) / 2) for l in range(4)]  # (Phi_l)_{j,a} = e^{+i a t_jl}
    assert np.max(np.abs(Phi[0].conj().T @ Phi[3] - G[2])) < 1e-11
    assert np.max(np.abs(Phi[2].conj().T @ Phi[3] - G[5])) < 1e-11


# --------------------------------------------------------------------------------------------
# P3: brute-force kernel ridge regression reproduces the Fourier estimator
# --------------------------------------------------------------------------------------------
def _krr_predict(X, Y, Xq, L, m, lam, Rk):
    """f(x) = k(x)^T (K + n lam I)^{-1} Y with K(x,x') = sum_k R_k^{-1} cos<k, t(x) - t(x')> (reading R2)."""
    d = X.shape[1]
    import itertools

    k = np.array(list(itertools.product(range(-m, m + 1), repeat=d)), dtype=np.float64)
    t = np.pi * X / (2 * L)
    tq = np.pi * Xq / (2 * L)
    w = 1.0 / Rk

    def kern(A, B):
        ph = (A @ k.T)[:, None, :] - (B @ k.T)[None, :, :]
        return np.cos(ph) @ w

    K = kern(t, t)
    n = X.shape[0]
    alpha = np.linalg.solve(K + n * lam * np.eye(n), Y)
    return kern(tq, t) @ alpha


@pytest.mark.parametrize("d,m,kind,s,lam", [(1, 6, "sobolev", 2.0, 1e-3), (1, 8, "lowbias", 1.0, 1e-2), (2, 3, "sobolev", 1.5, 1e-3)])
def test_krr_twin(oracle, d, m, kind, s, lam):
    L = 1.0
    n = 150
    X = RNG.uniform(-1.0, 0.3, size=(n, d))  # asymmetric on purpose
    Y = np.sin(3 * X[:, 0]) + 0.1 * RNG.normal(size=n)
    Xq = RNG.uniform(-1, 1, size=(40, d))
    theta, mu, r = oracle.fit(X, Y, L, m, lam, kind, s)
    f_fourier = oracle.predict(theta, Xq, L, m)
    Rk = oracle.sobolev_weights(d, m, s) if kind == "sobolev" else np.ones((2 * m + 1) ** d)
    f_krr = _krr_predict(X, Y, Xq, L, m, lam, Rk)
    assert rel(f_fourier, f_krr) < 1e-9
    # theta is Hermitian for real Y, so the imaginary part of the model vanishes
    th = theta.reshape((2 * m + 1,) * d)
    assert np.max(np.abs(th[(slice(None, None, -1),) * d] - np.conj(th))) < 1e-9


def test_krr_rejects_literal_paper_sign(oracle):
    """Reading R1: with the literal +i of P:206 in v (and Sigma_{k1,k2} = c_{k2-k1}) the
    estimator is NOT kernel ridge regression; this is why the oracle uses -i."""
    n, m, lam = 150, 6, 1e-3
    X = RNG.uniform(-1.0, 0.3, size=(n, 1))
    Y = np.sin(3 * X[:, 0])
    Xq = RNG.uniform(-1, 1, size=(40, 1))
    mu = oracle.moments(X, 1.0, m)
    r_wrong = np.conj(oracle.rhs(X, Y, 1.0, m))  # sum Y exp(+i k t)
    th = oracle.solve(mu, r_wrong, n, 1, m, lam, "sobolev", 2.0)
    f_wrong = oracle.predict(th, Xq, 1.0, m)
    f_krr = _krr_predict(X, Y, Xq, 1.0, m, lam, oracle.sobolev_weights(1, m, 2.0))
    assert rel(f_wrong, f_krr) > 1e-2


# --------------------------------------------------------------------------------------------
# P8: the solve
# --------------------------------------------------------------------------------------------
def test_single_sample_sherman_morrison(oracle):
    """n = 1: A = u u^* + lam R with u_k = exp(-i k t_1), b = Y u, so
    theta = Y (lam R)^{-1} u / (1 + u^* (lam R)^{-1} u) (Sherman-Morrison)."""
    m, lam, s = 9, 0.37, 1.0
    x, y = 0.4217, -1.3
    theta, _, _ = oracle.fit(np.array([[x]]), np.array([y]), 1.0, m, lam, "sobolev", s)
    k = np.arange(-m, m + 1)
    u = np.exp(-1j * k * np.pi * x / 2)
    Rinv = 1.0 / (lam * (1 + np.abs(k) ** (2 * s)))
    expect = y * Rinv * u / (1 + np.sum(np.abs(u) ** 2 * Rinv))
    assert rel(theta, expect) < 1e-13


def test_large_lambda_limit(oracle):
    """lam -> infinity: theta -> r / (n lam R)."""
    X, Y = datagen.dataset(400, seed=2)
    m, lam = 10, 1e8
    theta, mu, r = oracle.fit(X, Y, 1.0, m, lam, "sobolev", 1.0)
    approx = r.ravel() / (400 * lam * oracle.sobolev_weights(1, m, 1.0))
    assert rel(theta, approx) < 1e-6


def test_sobolev_diagonal_values(oracle):
    """S_kk = sqrt(1 + ||k||_2^{2s}): k=0 -> 1, s=1, k=2 -> sqrt 5; d=2, s=2, k=(1,1) -> sqrt 5."""
    w1 = oracle.sobolev_weights(1, 3, 1.0)
    assert w1[3] == 1.0 and abs(np.sqrt(w1[5]) - np.sqrt(5)) < 1e-15
    w2 = oracle.sobolev_weights(2, 2, 2.0).reshape(5, 5)
    assert abs(np.sqrt(w2[3, 3]) - np.sqrt(5)) < 1e-15


# --------------------------------------------------------------------------------------------
# P7: physics-informed penalty, by quadrature of (4L)^{-d} int_Omega |D f_theta|^2
# --------------------------------------------------------------------------------------------
def _f_theta(theta, k, x, L):
    return np.exp(1j * np.pi * (x @ k.T) / (2 * L)) @ theta


def _fd(fun, x, axis, order, h):
    e = np.zeros_like(x)
    e[:, axis] = h
    if order == 1:
        return (-fun(x + 2 * e) + 8 * fun(x + e) - 8 * fun(x - e) + fun(x - 2 * e)) / (12 * h)
    return (-fun(x + 2 * e) + 16 * fun(x + e) - 30 * fun(x) + 16 * fun(x - e) - fun(x - 2 * e)) / (12 * h * h)


@pytest.mark.parametrize("case", ["ode1d", "heat2d"])
def test_pi_penalty_quadrature(oracle, case):
    if case == "ode1d":  # Omega = ]0,1[, L = pi/2, D f = f' - f
        d, m, L = 1, 6, np.pi / 2
        alpha, a_alpha, box = [[1], [0]], [1.0, -1.0], [[0.0, 1.0]]
    else:  # space-time heat equation d_tau f - d_xx f on a sub-box of [-1,1]^2 (C4)
        d, m, L = 2, 3, 1.0
        alpha, a_alpha, box = [[1, 0], [0, 2]], [1.0, -1.0], [[-0.5, 0.8], [-1.0, 0.3]]
    k = oracle.mode_grid(d, m).astype(np.float64)
    theta = RNG.normal(size=k.shape[0]) + 1j * RNG.normal(size=k.shape[0])
    dk = oracle.pde_symbol(d, m, L, alpha, a_alpha)
    B = oracle.box_fourier_matrix(d, m, L, box)
    pen = np.real(np.conj(theta * dk) @ B @ (theta * dk))
    # quadrature: Gauss-Legendre tensor grid; D f by 4th-order finite differences of f itself
    g, w = np.polynomial.legendre.leggauss(40)
    pts, wts = [], []
    for l in range(d):
        a, b = box[l]
        pts.append(0.5 * (b - a) * g + 0.5 * (b + a))
        wts.append(0.5 * (b - a) * w)
    P = np.stack(np.meshgrid(*pts, indexing="ij"), -1).reshape(-1, d)
    W = np.prod(np.stack(np.meshgrid(*wts, indexing="ij"), -1).reshape(-1, d), axis=1)
    fun = lambda x: _f_theta(theta, k, x, L)
    Df = np.zeros(P.shape[0], dtype=np.complex128)
    for al, a in zip(alpha, a_alpha):
        term = fun(P)
        nz = [l for l in range(d) if al[l] > 0]
        if nz:
            assert len(nz) == 1
            term = _fd(fun, P, nz[0], al[nz[0]], 1e-3)
        Df += a * term
    quad = np.sum(W * np.abs(Df) ** 2) / (4 * L) ** d
    assert abs(pen - quad) / quad < 1e-7


def test_pi_zero_weight_is_sobolev(oracle):
    """mu = 0 reduces the physics-informed system to the Sobolev one."""
    X, Y = datagen.dataset(500, d=2, seed=4)
    m = 3
    mu = oracle.moments(X, 1.0, m)
    r = oracle.rhs(X, Y, 1.0, m)
    a = oracle.solve(mu, r, 500, 2, m, 1e-3, "pik_box", 2.0, mu_pde=0.0, L=1.0, alpha=[[1, 0], [0, 2]], a_alpha=[1, -1], box=[[-1, 1], [-1, 1]])
    b = oracle.solve(mu, r, 500, 2, m, 1e-3, "sobolev", 2.0)
    assert rel(a, b) < 1e-14


# --------------------------------------------------------------------------------------------
# P6: additive model
# --------------------------------------------------------------------------------------------
def test_additive_matches_explicit_ridge(oracle):
    """theta = (Phi^*Phi/n + lam I)^{-1} Phi^*Y/n with Phi = [Phi_1 .. Phi_d] built explicitly
     equals the oracle's block assembly from moments / cross moments / rhs."""
    n, d, m, lam = 400, 3, 4, 1e-3
    X, Y = datagen.dataset(n, d=d, ykind="additive", seed=8)
    a = np.arange(-m, m + 1)
    Phi = np.concatenate([np.exp(1j * np.pi * np.outer(X[:, l].astype(np.float64), a) / 2) for l in range(d)], axis=1)
    A = Phi.conj().T @ Phi / n + lam * np.eye(d * (2 * m + 1))
    theta_ref = np.linalg.solve(A, Phi.conj().T @ Y.astype(np.float64) / n)
    mu_l = [oracle.moments(X[:, l], 1.0, m) for l in range(d)]
    r_l = [oracle.rhs(X[:, l], Y, 1.0, m) for l in range(d)]
    G = oracle.cross_moments(X, 1.0, m)
    theta = oracle.solve_additive(mu_l, r_l, G, n, d, m, lam)
    assert rel(theta, theta_ref) < 1e-10
    # predictions: additive kernel ridge twin, K(x,x') = sum_l sum_a cos(a (t_l - t'_l))
    Xq = RNG.uniform(-1, 1, size=(30, d))
    t, tq = np.pi * X.astype(np.float64) / 2, np.pi * Xq / 2

    def kern(A_, B_):
        return sum(np.cos(np.subtract.outer(A_[:, l], B_[:, l])[..., None] * a).sum(-1) for l in range(d))

    alpha = np.linalg.solve(kern(t, t) + n * lam * np.eye(n), Y.astype(np.float64))
    f_krr = kern(tq, t) @ alpha
    assert rel(oracle.predict_additive(theta, Xq, 1.0, m), f_krr) < 1e-8


def test_additive_d1_is_lowbias(oracle):
    """d = 1 additive equals the low-bias estimator."""
    X, Y = datagen.dataset(300, seed=6)
    m, lam = 5, 1e-2
    mu = oracle.moments(X, 1.0, m)
    r = oracle.rhs(X, Y, 1.0, m)
    a = oracle.solve_additive([mu], [r], np.zeros((0, 11, 11)), 300, 1, m, lam)
    b = oracle.solve(mu, r, 300, 1, m, lam, "lowbias")
    assert rel(a, b) < 1e-13


# --------------------------------------------------------------------------------------------
# P9: prediction
# --------------------------------------------------------------------------------------------
def test_predict_basis_functions(oracle):
    m = 5
    x = RNG.uniform(-1, 1, size=(50, 1))
    th = np.zeros(2 * m + 1, dtype=np.complex128)
    th[m] = 2.5
    assert np.allclose(oracle.predict(th, x, 1.0, m), 2.5, atol=1e-14)
    th[:] = 0
    th[m + 3] = 1.0  # k = 3: f = Re exp(+i 3 t)
    assert np.allclose(oracle.predict(th, x, 1.0, m), np.cos(3 * np.pi * x[:, 0] / 2), atol=1e-14)
    th[m + 3] = 1j  # Re(i e^{i 3 t}) = -sin(3t): pins the +i of the model
    assert np.allclose(oracle.predict(th, x, 1.0, m), -np.sin(3 * np.pi * x[:, 0] / 2), atol=1e-14)


def test_schedules_golden(oracle):
    """tests/golden/schedules.txt: m = n^{1/(2s+d)}, lambda = n^{-2s/(2s+d)}."""
    path = os.path.join(os.path.dirname(__file__), "golden", "schedules.txt")
    rows = [l.split() for l in open(path) if l.strip() and not l.startswith("#")]
    assert rows
    for n, s, d, m, lam in rows:
        mm, ll = oracle.schedule(float(n), float(s), int(d))
        assert mm == int(m)
        assert abs(ll - float(lam)) / float(lam) < 1e-3


# --------------------------------------------------------------------------------------------
# P7': physics-informed penalty by collocation
# --------------------------------------------------------------------------------------------
def test_pi_collocation_quadratic_form(oracle):
    """theta^* D^* T(mu_r) D theta / n_r == n_r^{-1} sum_i |D f_theta(X^r_i)|^2, with
    D f evaluated by finite differences of f itself (independent of the symbol d_k)."""
    d, m, L = 2, 3, 1.0
    alpha, a_alpha = [[1, 0], [0, 2]], [1.0, -1.0]
    Xr = RNG.uniform(-0.8, 0.9, size=(400, d))
    k = oracle.mode_grid(d, m).astype(np.float64)
    theta = RNG.normal(size=k.shape[0]) + 1j * RNG.normal(size=k.shape[0])
    dk = oracle.pde_symbol(d, m, L, alpha, a_alpha)
    Tr = oracle.toeplitz_from_moments(oracle.moments(Xr, L, m), d, m)
    form = np.real(np.conj(theta * dk) @ Tr @ (theta * dk)) / Xr.shape[0]
    fun = lambda x: _f_theta(theta, k, x, L)
    Df = _fd(fun, Xr, 0, 1, 1e-3) - _fd(fun, Xr, 1, 2, 1e-3)
    direct = np.mean(np.abs(Df) ** 2)
    assert abs(form - direct) / direct < 1e-7


def test_pi_collocation_matches_box_penalty(oracle):
    """Collocation on a fine midpoint grid of the box Omega approximates the box penalty:
    mu' n_r^{-1} sum |Df|^2 ~ mu' |Omega|^{-1} int |Df|^2, i.e. pik_colloc(mu') == pik_box(mu) for
    mu' = mu |Omega| (4L)^{-d} (P:398-404 vs P:410-413)."""
    d, m, L, s, lam = 2, 4, 1.0, 2.0, 1e-4
    alpha, a_alpha = [[1, 0], [0, 2]], [1.0, -1.0]
    box = [[-0.6, 0.7], [-0.9, 0.5]]
    X, Y = datagen.dataset(3000, d=2, ykind="expcos", seed=41)
    mu, r = oracle.moments(X, L, m), oracle.rhs(X, Y, L, m)
    g = 200
    ax = [np.linspace(a, b, g, endpoint=False) + (b - a) / (2 * g) for a, b in box]
    Xr = np.stack(np.meshgrid(*ax, indexing="ij"), -1).reshape(-1, d)
    vol = np.prod([b - a for a, b in box])
    th_box = oracle.solve(mu, r, 3000, d, m, lam, "pik_box", s, mu_pde=1.0, L=L, alpha=alpha, a_alpha=a_alpha, box=box)
    th_col = oracle.solve(mu, r, 3000, d, m, lam, "pik_colloc", s, mu_pde=vol / (4 * L) ** d, L=L, alpha=alpha, a_alpha=a_alpha,
                          mu_colloc=oracle.moments(Xr, L, m), n_colloc=Xr.shape[0])
    assert rel(th_col, th_box) < 1e-3
