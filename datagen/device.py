"""ctypes wrapper of datagen/libfkgen.so: the on-device twin of the numpy generator.

Writes seeded synthetic samples straight into CUDA tensors (inputs of 80 GB cannot be
generated on the host).  Holds none of the method's arithmetic."""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libfkgen.so")
_gen = None


def lib():
    global _gen
    if _gen is None:
        if not os.path.exists(_LIB):
            from paper_2509_02649_b200 import build

            build.build()
        L = ctypes.CDLL(_LIB)
        L.fkgen_dataset.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_uint32, ctypes.c_float, ctypes.c_int,
                                    ctypes.c_void_p]
        L.fkgen_equispaced.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                       ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
        _gen = L
    return _gen


def gen_dataset(X, Y, n, d, i0=0, xkind=0, ykind=0, seed=0, L=1.0, noise=True, stride_n=None, stride_d=None):
    """Samples i0..i0+n-1 into X (n x d, element strides stride_n / stride_d) and Y (n)."""
    import torch

    s = torch.cuda.current_stream().cuda_stream
    sn = d if stride_n is None else stride_n
    sd = 1 if stride_d is None else stride_d
    rc = lib().fkgen_dataset(X.data_ptr() if X is not None else None, Y.data_ptr() if Y is not None else None, n, d, sn, sd, i0,
                             xkind, ykind, seed, L, 1 if noise else 0, ctypes.c_void_p(s))
    if rc != 0:
        raise RuntimeError(f"fkgen_dataset failed ({rc})")


def gen_equispaced(X, Y, count, i0, n_total, a, b, log2N=24):
    import torch

    s = torch.cuda.current_stream().cuda_stream
    rc = lib().fkgen_equispaced(X.data_ptr() if X is not None else None, Y.data_ptr() if Y is not None else None, count, i0,
                                n_total, a, b, log2N, ctypes.c_void_p(s))
    if rc != 0:
        raise RuntimeError(f"fkgen_equispaced failed ({rc})")
