"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only turns (seed, stream, sample id)
into sample values.  Both the numpy implementation below and the CUDA kernels in
``datagen/gen.cu`` (``libfkgen.so``) implement the same counter-based generator with the
same fp32 operation order, so a sample is bit-identical whichever side produced it
(checked by tests/test_datagen_gpu.py).  Random numbers are never drawn by the method.

Recipe:
  z(i, stream)   = splitmix64((seed << 48) ^ (stream << 40) ^ i)
  u24            = z >> 40  (and (z >> 16) & 0xFFFFFF as a second draw)
  uniform X      = (2 u24 + 1 - 2^24) * 2^-24            in (-1, 1), exact in fp32
  unit X         = u24 * 2^-24                           in [0, 1) (the rate experiment)
  gaussian X     = clip(IH4 * 0.6928203f, -1, 1): Irwin-Hall of 4 draws (sd 0.577) rescaled
                   to sd 0.4 and truncated to the box
  noise          = (sum of 12 draws - 6 * 2^24) * 2^-24   (Irwin-Hall approx. of N(0,1))
  equispaced     = v = ((a i + b) mod n) mod N, X = (2 v + 1 - N) / N, Y = [v even]
                   (N = 2^24, n = r N: the closed-form pin P1/P2 of SURVEY.md §8(c))
  f*             = fp32 polynomials (sin-like, exp*cos-like, additive exp-like), explicit
                   rounding order, see _fstar_*.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
XKIND = {"uniform": 0, "gaussian": 1, "equispaced": 2, "unit": 3}
YKIND = {"sin": 0, "expcos": 1, "additive": 2, "pattern01": 3, "zero": 4, "exp": 5}
EQ_N = 1 << 24


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        z = x
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _z(idx: np.ndarray, stream: int, seed: int) -> np.ndarray:
    key = (np.uint64(seed & 0xFFFF) << np.uint64(48)) ^ (np.uint64(stream & 0xFF) << np.uint64(40))
    return _splitmix64(idx.astype(np.uint64) ^ key)


def _u24pair(idx, stream, seed):
    z = _z(idx, stream, seed)
    return (z >> np.uint64(40)).astype(np.int64), ((z >> np.uint64(16)) & np.uint64(0xFFFFFF)).astype(np.int64)


def _uniform(idx, stream, seed) -> np.ndarray:
    u, _ = _u24pair(idx, stream, seed)
    return ((2 * u + 1 - (1 << 24)).astype(np.float32) * np.float32(2.0 ** -24)).astype(np.float32)


def _unit(idx, stream, seed) -> np.ndarray:
    u, _ = _u24pair(idx, stream, seed)
    return (u.astype(np.float32) * np.float32(2.0 ** -24)).astype(np.float32)


def _gaussian(idx, stream, seed) -> np.ndarray:
    a, b = _u24pair(idx, stream, seed)
    c, e = _u24pair(idx, stream + 64, seed)
    s = (a + b + c + e - (2 << 24)).astype(np.float32) * np.float32(2.0 ** -24)  # int->fp32 round-to-nearest-even
    x = (s * np.float32(0.6928203)).astype(np.float32)
    return np.clip(x, np.float32(-1.0), np.float32(1.0)).astype(np.float32)


def _noise(idx, seed) -> np.ndarray:
    s = np.zeros(idx.shape, dtype=np.int64)
    for k in range(6):
        a, b = _u24pair(idx, 128 + k, seed)
        s += a + b
    return ((s - 6 * (1 << 24)).astype(np.float32) * np.float32(2.0 ** -24)).astype(np.float32)


def _equispaced_v(idx, n: int, a: int, b: int, N: int) -> np.ndarray:
    i = idx.astype(object) if n >= (1 << 31) else idx.astype(np.int64)
    j = (a * i + b) % n
    return np.asarray(j % N, dtype=np.int64)


def _fstar_sin(x):
    f = np.float32
    x2 = f(x * x)
    t = f(f(1.0) - f(x2 * f(0.05)))
    t = f(f(x2 * t) * f(1.0 / 6.0))
    return f(x * f(f(1.0) - t))


def _expm1_poly(z):
    f = np.float32
    # z + z^2/2 + z^3/6 + z^4/24, Horner in fp32
    p = f(f(z * f(1.0 / 24.0)) + f(1.0 / 6.0))
    p = f(f(z * p) + f(0.5))
    p = f(f(z * p) + f(1.0))
    return f(z * p)


def _fstar_expcos(x1, x2):
    f = np.float32
    e = f(_expm1_poly(x1) + f(1.0))
    y2 = f(x2 * x2)
    c = f(f(1.0) - f(y2 * f(f(0.5) - f(y2 * f(1.0 / 24.0)))))
    return f(e * c)


def dataset(n: int, d: int = 1, i0: int = 0, xkind: str = "uniform", ykind: str = "sin", seed: int = 0,
            L: float = 1.0, noise: bool = True):
    """Samples i0 .. i0+n-1 of the seeded synthetic dataset.  Returns (X float32 (n,d), Y float32 (n,)).

    X lies in [-L, L]^d (L multiplies the unit-box value in fp32)."""
    idx = np.arange(i0, i0 + n, dtype=np.int64)
    X = np.empty((n, d), dtype=np.float32)
    f = np.float32
    gen = {"uniform": _uniform, "gaussian": _gaussian, "unit": _unit}
    if xkind not in gen:
        raise ValueError("xkind must be 'uniform', 'gaussian' or 'unit' (use equispaced() for the pin data)")
    for l in range(d):
        X[:, l] = gen[xkind](idx, l, seed)
    Y = _response(X, idx, d, ykind, seed, noise)
    if L != 1.0:
        X = (X * f(L)).astype(np.float32)
    return X, Y


def _response(Xu, idx, d, ykind, seed, noise):
    f = np.float32
    n = Xu.shape[0]
    if ykind == "sin":
        Y = _fstar_sin(Xu[:, 0])
    elif ykind == "expcos":
        Y = _fstar_expcos(Xu[:, 0], Xu[:, 1] if d > 1 else np.zeros(n, np.float32))
    elif ykind == "additive":
        Y = np.zeros(n, dtype=np.float32)
        for l in range(d):
            Y = f(Y + _expm1_poly(f(Xu[:, l] * f(1.0 / (l + 1)))))
    elif ykind == "exp":  # e^x, as the 4-term polynomial + 1
        Y = f(_expm1_poly(Xu[:, 0]) + f(1.0))
    elif ykind == "zero":
        Y = np.zeros(n, dtype=np.float32)
    else:
        raise ValueError(ykind)
    Y = np.asarray(Y, dtype=np.float32)
    if noise:
        Y = (Y + _noise(idx, seed)).astype(np.float32)
    return Y


def equispaced(n_total: int, i0: int, count: int, a: int, b: int, N: int = EQ_N):
    """Equispaced-replicated, permuted points (pin P1/P2): sample i has grid value
    v = ((a i + b) mod n_total) mod N, X = (2v + 1 - N) / N, Y = 1 if v is even else 0.
    N is a power of two <= 2^24 (so X is exact in fp32), n_total a multiple of N and
    gcd(a, n_total) = 1 (the affine map is then a bijection of the sample ids)."""
    assert N & (N - 1) == 0 and N <= EQ_N and n_total % N == 0
    idx = np.arange(i0, i0 + count, dtype=np.int64)
    v = _equispaced_v(idx, n_total, a, b, N)
    X = ((2 * v + 1 - N).astype(np.float32) * np.float32(1.0 / N)).astype(np.float32)
    Y = (v % 2 == 0).astype(np.float32)
    return X.reshape(-1, 1), Y
