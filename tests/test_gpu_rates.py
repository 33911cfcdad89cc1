"""Statistical sanity of the whole GPU path (SURVEY.md §8(c) pin P12, NEXT-4): the paper's Fig. 1
 reports a test error decaying at the Sobolev minimax rate n^{-2/3} for s = 1,
lambda = n^{-2/3}, m = n^{1/3}, X ~ U(0,1), Y = e^X + N(0,1).  A dropped term or a wrong sign
anywhere in moments / rhs / solve / predict destroys the slope (the estimator stops converging)."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


def test_fig1_rate_slope():
    assert torch.cuda.is_available()
    from paper_2509_02649_b200 import build

    build.build()
    import rates

    rows, sl = rates.run([10 ** e for e in range(3, 8)], resamples=6)
    print("rates:", [(r["n"], f"{r['test_mse']:.3e}") for r in rows], f"slope {sl:.3f}")
    assert all(b["test_mse"] < a["test_mse"] for a, b in zip(rows, rows[1:]))
    assert -0.85 < sl < -0.5


def test_fig5_additive_rate_slope():
    """Fig. 5: low-bias additive, d = 5, s = 2, lambda = n^{-0.8}; paper slope -0.8."""
    import rates

    rows, sl = rates.run([10 ** e for e in range(3, 8)], resamples=4, additive=True)
    print("additive rates:", [(r["n"], f"{r['test_mse']:.3e}") for r in rows], f"slope {sl:.3f}")
    assert all(b["test_mse"] < a["test_mse"] for a, b in zip(rows, rows[1:]))
    assert -1.0 < sl < -0.65
