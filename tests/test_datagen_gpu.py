"""The on-device generator (datagen/gen.cu) is bit-identical to the numpy one (datagen)."""
import numpy as np
import pytest

import datagen
from gpu_util import gen_dataset, gen_equispaced, host

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("d,xkind,ykind", [(1, "uniform", "sin"), (1, "gaussian", "sin"), (2, "uniform", "expcos"), (10, "uniform", "additive"),
                                            (1, "unit", "exp")])
def test_generator_bit_identical(d, xkind, ykind):
    n, i0 = 50_000, 123_456_789
    X = torch.empty((n, d), dtype=torch.float32, device="cuda")
    Y = torch.empty(n, dtype=torch.float32, device="cuda")
    gen_dataset(X, Y, n, d, i0=i0, xkind=datagen.XKIND[xkind], ykind=datagen.YKIND[ykind], seed=7)
    Xh, Yh = datagen.dataset(n, d=d, i0=i0, xkind=xkind, ykind=ykind, seed=7)
    assert np.array_equal(host(X), Xh)
    assert np.array_equal(host(Y), Yh)


def test_equispaced_bit_identical():
    n_total = 596 << 24
    X = torch.empty(4096, dtype=torch.float32, device="cuda")
    Y = torch.empty(4096, dtype=torch.float32, device="cuda")
    gen_equispaced(X, Y, 4096, n_total - 5000, n_total, 1000003, 12345)
    Xh, Yh = datagen.equispaced(n_total, n_total - 5000, 4096, 1000003, 12345)
    assert np.array_equal(host(X), Xh.ravel()) and np.array_equal(host(Y), Yh)
