"""Helpers shared by the GPU parity tests (no method arithmetic here)."""
import ctypes
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b) -> float:
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def fk():
    from paper_2509_02649_b200 import build, fk as _fk

    build.build()
    return _fk


def dev(a, dtype=None):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def host(t):
    return t.detach().cpu().numpy()


_gen = None


def gen_lib():
    """datagen/libfkgen.so: the on-device twin of datagen (seeded inputs only)."""
    global _gen
    if _gen is None:
        fk()  # builds libfkgen.so too
        L = ctypes.CDLL(os.path.join(ROOT, "datagen", "libfkgen.so"))
        L.fkgen_dataset.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_uint32, ctypes.c_float, ctypes.c_int,
                                    ctypes.c_void_p]
        L.fkgen_equispaced.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                       ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
        _gen = L
    return _gen


def gen_dataset(X, Y, n, d, i0=0, xkind=0, ykind=0, seed=0, L=1.0, noise=True, stride_n=None, stride_d=None):
    import torch

    s = torch.cuda.current_stream().cuda_stream
    sn = d if stride_n is None else stride_n
    sd = 1 if stride_d is None else stride_d
    rc = gen_lib().fkgen_dataset(X.data_ptr() if X is not None else None, Y.data_ptr() if Y is not None else None, n, d, sn, sd, i0,
                                 xkind, ykind, seed, L, 1 if noise else 0, ctypes.c_void_p(s))
    assert rc == 0


def gen_equispaced(X, Y, count, i0, n_total, a, b, log2N=24):
    import torch

    s = torch.cuda.current_stream().cuda_stream
    rc = gen_lib().fkgen_equispaced(X.data_ptr() if X is not None else None, Y.data_ptr() if Y is not None else None, count, i0,
                                    n_total, a, b, log2N, ctypes.c_void_p(s))
    assert rc == 0
