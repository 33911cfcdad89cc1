"""CPU oracle of the fast-kernel-regression fit path (arXiv 2509.02649).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The product path
(``paper_2509_02649_b200``) never imports it, and the two share no code: the direct sums
live in ``oracle/direct.c`` (plain fp64 C), the linear algebra below is plain numpy in
complex128.  Each function cites the PAPER.md passage it follows ("P:<line>") and the
DESIGN.md reading ("R<n>") where the paper is ambiguous.

Conventions (R1-R4):
    t(x)  = pi x / (2L)
    f(x)  = sum_{|k|<=m} theta_k exp(+i <k, t(x)>)
    mu_q  = sum_j exp(-i <q, t_j>),  |q|_inf <= 2m          P:212-220 (unnormalised, R1)
    r_k   = sum_j Y_j exp(-i <k, t_j>), |k|_inf <= m        P:203-208 (unnormalised, R1)
    A     = T(mu)/n + lambda M*M (+ mu_pde D* C D),  A theta = r / n
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "direct.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle/direct.c with gcc (-O2, OpenMP, no fast-math) into oracle/liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _get():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            dp = ctypes.POINTER(ctypes.c_double)
            lib.oracle_type1.argtypes = [dp, dp, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_int, dp]
            lib.oracle_cross.argtypes = [dp, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_int, dp]
            lib.oracle_type2.argtypes = [dp, ctypes.c_int, ctypes.c_int, ctypes.c_double, dp, ctypes.c_int64, dp]
            lib.oracle_type2_additive.argtypes = [dp, ctypes.c_int, ctypes.c_int, ctypes.c_double, dp, ctypes.c_int64, dp]
            lib.oracle_num_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def num_threads() -> int:
    return int(_get().oracle_num_threads())


def _points(X) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)  # fp32 inputs are exact in fp64 (R6)
    if X.ndim == 1:
        X = X[:, None]
    return np.ascontiguousarray(X)


# ---------------------------------------------------------------------------------------------
# Exponential sums (direct, fp64)
# ---------------------------------------------------------------------------------------------
def type1(X, w, L: float, K: int) -> np.ndarray:
    """sum_j w_j exp(-i <k, pi X_j/2L>) for k in {-K..K}^d, shape (2K+1,)*d, complex128.

    P:203-220 (v and the first row of Sigma-hat as exponential sums); sign per R1."""
    X = _points(X)
    n, d = X.shape
    out = np.zeros((2 * K + 1) ** d * 2, dtype=np.float64)
    wp = None
    if w is not None:
        w = np.ascontiguousarray(np.asarray(w, dtype=np.float64).reshape(-1))
        assert w.shape[0] == n
        wp = _dp(w)
    _get().oracle_type1(_dp(X), wp, n, d, float(L), int(K), _dp(out))
    return out.view(np.complex128).reshape((2 * K + 1,) * d)


def moments(X, L: float, m: int) -> np.ndarray:
    """mu_q = sum_j exp(-i <q, t_j>), |q|_inf <= 2m (first row of n Sigma-hat)."""
    return type1(X, None, L, 2 * m)


def rhs(X, Y, L: float, m: int) -> np.ndarray:
    """r_k = sum_j Y_j exp(-i <k, t_j>), |k|_inf <= m (n v = Phi* Y)."""
    return type1(X, Y, L, m)


def cross_moments(X, L: float, m: int) -> np.ndarray:
    """G[p, a, b] = sum_j exp(-i (a t_{j,l1} - b t_{j,l2})) for pairs l1 < l2."""
    X = _points(X)
    n, d = X.shape
    npairs = d * (d - 1) // 2
    side = 2 * m + 1
    out = np.zeros(npairs * side * side * 2, dtype=np.float64)
    _get().oracle_cross(_dp(X), n, d, float(L), int(m), _dp(out))
    return out.view(np.complex128).reshape(npairs, side, side)


def predict(theta, Xq, L: float, m: int) -> np.ndarray:
    """f(x) = Re sum_k theta_k exp(+i <k, pi x/2L>) by direct summation."""
    Xq = _points(Xq)
    nq, d = Xq.shape
    th = np.ascontiguousarray(np.asarray(theta, dtype=np.complex128).reshape(-1)).view(np.float64)
    assert th.size == 2 * (2 * m + 1) ** d
    out = np.zeros(nq, dtype=np.float64)
    _get().oracle_type2(_dp(th), d, int(m), float(L), _dp(Xq), nq, _dp(out))
    return out


def predict_additive(theta, Xq, L: float, m: int) -> np.ndarray:
    """f(x) = Re sum_l sum_a theta_{l,a} exp(+i a t(x_l))."""
    Xq = _points(Xq)
    nq, d = Xq.shape
    th = np.ascontiguousarray(np.asarray(theta, dtype=np.complex128).reshape(-1)).view(np.float64)
    assert th.size == 2 * d * (2 * m + 1)
    out = np.zeros(nq, dtype=np.float64)
    _get().oracle_type2_additive(_dp(th), d, int(m), float(L), _dp(Xq), nq, _dp(out))
    return out


# ---------------------------------------------------------------------------------------------
# Mode grid and regularisers
# ---------------------------------------------------------------------------------------------
def mode_grid(d: int, m: int) -> np.ndarray:
    """All k in {-m..m}^d, lexicographic with the last coordinate fastest; shape (D, d)."""
    axes = [np.arange(-m, m + 1)] * d
    return np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, d)


def sobolev_weights(d: int, m: int, s: float) -> np.ndarray:
    """(S^2)_kk = 1 + ||k||_2^{2s} (Sobolev matrix S)."""
    k = mode_grid(d, m).astype(np.float64)
    return 1.0 + np.sum(k * k, axis=1) ** s


def toeplitz_from_moments(mu: np.ndarray, d: int, m: int) -> np.ndarray:
    """Dense T[k1, k2] = mu_{k1 - k2} over the model grid (Sigma-hat is d-level Toeplitz)."""
    k = mode_grid(d, m)
    diff = k[:, None, :] - k[None, :, :] + 2 * m  # index into {-2m..2m}^d
    return mu[tuple(diff[..., l] for l in range(d))]


def pde_symbol(d: int, m: int, L: float, alpha, a_alpha) -> np.ndarray:
    """d_k = sum_alpha a_alpha prod_l (i pi k_l / 2L)^{alpha_l}: symbol of D on exp(+i<k,t(x)>).

    PAPER.md:384 defines D = sum a_alpha d^alpha; :403 writes the symbol with (-i pi/2L), the
    conjugate convention; under f = sum theta exp(+ikt) the derivative gives (+i pi/2L)
    (reading R3)."""
    k = mode_grid(d, m).astype(np.float64)
    out = np.zeros(k.shape[0], dtype=np.complex128)
    for al, a in zip(np.asarray(alpha, dtype=np.int64).reshape(-1, d), np.asarray(a_alpha, dtype=np.float64)):
        term = np.full(k.shape[0], complex(a))
        for l in range(d):
            term = term * (1j * np.pi * k[:, l] / (2.0 * L)) ** int(al[l])
        out += term
    return out


def box_fourier_matrix(d: int, m: int, L: float, box) -> np.ndarray:
    """B[k1, k2] = (4L)^{-d} int_Omega exp(+i <k2 - k1, pi x / 2L>) dx for the box Omega = prod [a_l, b_l].

    P:398-400 (Fourier matrix C of Omega), with the index order of reading R3."""
    box = np.asarray(box, dtype=np.float64).reshape(d, 2)
    k = mode_grid(d, m)
    q = k[None, :, :] - k[:, None, :]  # k2 - k1
    B = np.ones(q.shape[:2], dtype=np.complex128)
    c = np.pi / (2.0 * L)
    for l in range(d):
        a, b = box[l]
        ql = q[..., l].astype(np.float64)
        with np.errstate(divide="ignore", invalid="ignore"):
            val = (np.exp(1j * c * ql * b) - np.exp(1j * c * ql * a)) / (1j * c * ql)
        val = np.where(ql == 0, b - a, val)
        B = B * val / (4.0 * L)
    return B


# ---------------------------------------------------------------------------------------------
# The regularised Fourier system and its solve
# ---------------------------------------------------------------------------------------------
def assemble(mu, n_total: float, d: int, m: int, lam: float, kind: str = "sobolev", s: float = 1.0,
             mu_pde: float = 0.0, L: float = 1.0, alpha=None, a_alpha=None, box=None, mu_colloc=None,
             n_colloc: float = 0.0) -> np.ndarray:
    """A = T(mu)/n + lam * M*M (+ mu_pde * D* B D) (P:107 eq. kenrel_reg; P:252 Sobolev M=S;
    P:316 low-bias M=I; P:396 physics-informed, tractable box domain; P:413 physics-informed,
    collocation: + mu_pde n_r^{-1} D* (Phi^r)* Phi^r D with (Phi^r)* Phi^r = T(mu_colloc), the
    Toeplitz matrix of the collocation points' moments)."""
    A = toeplitz_from_moments(np.asarray(mu), d, m) / float(n_total)
    if kind in ("sobolev", "pik_box", "pik_colloc"):
        A = A + lam * np.diag(sobolev_weights(d, m, s))
    elif kind == "lowbias":
        A = A + lam * np.eye(A.shape[0])
    else:
        raise ValueError(kind)
    if kind == "pik_box":
        dk = pde_symbol(d, m, L, alpha, a_alpha)
        A = A + mu_pde * (np.conj(dk)[:, None] * box_fourier_matrix(d, m, L, box) * dk[None, :])
    if kind == "pik_colloc":
        dk = pde_symbol(d, m, L, alpha, a_alpha)
        Tr = toeplitz_from_moments(np.asarray(mu_colloc), d, m) / float(n_colloc)
        A = A + mu_pde * (np.conj(dk)[:, None] * Tr * dk[None, :])
    return A


def solve(mu, r, n_total: float, d: int, m: int, lam: float, kind: str = "sobolev", s: float = 1.0, **pi) -> np.ndarray:
    """theta = A^{-1} r / n, complex128 dense solve (numpy / LAPACK)."""
    A = assemble(mu, n_total, d, m, lam, kind, s, **pi)
    b = np.asarray(r, dtype=np.complex128).reshape(-1) / float(n_total)
    return np.linalg.solve(A, b)


def assemble_additive(mu_l, G, n_total: float, d: int, m: int, lam: float) -> np.ndarray:
    """Sigma-hat + lam I for the additive model: diagonal blocks are the 1-D Toeplitz
    moments of feature l, block (l1, l2), l1 < l2, is G^{(l1,l2)}/n, block (l2, l1) its conjugate
    transpose (Sigma-hat is Hermitian)."""
    side = 2 * m + 1
    A = np.zeros((d * side, d * side), dtype=np.complex128)
    for l in range(d):
        A[l * side:(l + 1) * side, l * side:(l + 1) * side] = toeplitz_from_moments(np.asarray(mu_l[l]), 1, m) / n_total
    p = 0
    for l1 in range(d):
        for l2 in range(l1 + 1, d):
            blk = np.asarray(G[p]) / n_total
            A[l1 * side:(l1 + 1) * side, l2 * side:(l2 + 1) * side] = blk
            A[l2 * side:(l2 + 1) * side, l1 * side:(l1 + 1) * side] = blk.conj().T
            p += 1
    return A + lam * np.eye(d * side)


def solve_additive(mu_l, r_l, G, n_total: float, d: int, m: int, lam: float) -> np.ndarray:
    """theta = (Sigma-hat + lam I)^{-1} (Phi_l* Y / n)_l (low-bias additive)."""
    A = assemble_additive(mu_l, G, n_total, d, m, lam)
    b = np.concatenate([np.asarray(r_l[l]).reshape(-1) for l in range(d)]) / float(n_total)
    return np.linalg.solve(A, b)


def backward_error(A: np.ndarray, theta: np.ndarray, b: np.ndarray) -> float:
    """||A theta - b|| / ||b|| (reading R8: the solve gate in fp32 mode)."""
    return float(np.linalg.norm(A @ theta - b) / np.linalg.norm(b))


# ---------------------------------------------------------------------------------------------
# Schedules
# ---------------------------------------------------------------------------------------------
def schedule(n: float, s: float, d: int):
    """m = n^{1/(2s+d)} (rounded), lambda = n^{-2s/(2s+d)}."""
    return int(round(n ** (1.0 / (2 * s + d)))), float(n ** (-2.0 * s / (2 * s + d)))


def fit(X, Y, L: float, m: int, lam: float, kind: str = "sobolev", s: float = 1.0, **pi):
    """Whole oracle fit: moments + rhs + dense solve.  Returns (theta, mu, r)."""
    X = _points(X)
    d = X.shape[1]
    mu = moments(X, L, m)
    r = rhs(X, Y, L, m)
    if kind in ("pik_box", "pik_colloc"):
        pi = dict(pi, L=L)
    if kind == "pik_colloc":  # collocation points -> their moments
        Xr = _points(pi.pop("X_colloc"))
        pi = dict(pi, mu_colloc=moments(Xr, L, m), n_colloc=Xr.shape[0])
    theta = solve(mu, r, X.shape[0], d, m, lam, kind, s, **pi)
    return theta, mu, r
