#!/usr/bin/env python
"""Statistical rate experiment of the paper's Fig. 1 on the GPU
path: X ~ U(0, 1), Y = e^X + N(0, 1) (datagen xkind "unit", ykind "exp"), Sobolev s = 1,
lambda = n^{-2/3}, m = n^{1/3}; test error E ||f_theta - f*||^2_{L2(P_X)} on a separate noise-free
test set of 1e4 samples, averaged over resamples.  The paper reports the minimax slope -2/3.

The fit and the prediction run through libfk (fit.fit -> fk_rhs_type1 + fk_solve,
fk_predict_type2); only the evaluation (mean squared difference, slope) is done here in torch /
numpy -- it is the experiment's measurement, not part of the method.

    python tools/rates.py [--max-exp 9] [--resamples 20] [--additive]   -> JSON lines + fitted slope
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_error(n: int, seed: int, test_n: int = 10_000, s: float = 1.0, eps: float = 1e-6, chunk: int = 1 << 28) -> float:
    import torch

    from datagen.device import gen_dataset
    from paper_2509_02649_b200 import fit, fk

    m = max(1, int(round(n ** (1.0 / 3.0))))
    lam = n ** (-2.0 / 3.0)
    dev = torch.device("cuda")
    buf, mu, r = fit._moment_buffers(1, m, dev)
    c = min(n, chunk)
    X = torch.empty(c, dtype=torch.float32, device=dev)
    Y = torch.empty(c, dtype=torch.float32, device=dev)
    for i0 in range(0, n, c):  # FK_ACCUMULATE over chunks keeps memory bounded at any n
        k = min(c, n - i0)
        gen_dataset(X[:k], Y[:k], k, 1, i0=i0, xkind=3, ykind=5, seed=seed)
        fk.fk_rhs_type1(X[:k], Y[:k], 1.0, m, eps, r_out=r, mu_out=mu, accumulate=i0 > 0, check=False)
    theta, _ = fk.fk_solve(mu.reshape(-1), r.reshape(-1), n, 1, m, 1.0, lam, "sobolev", s, report=False)
    Xt = torch.empty(test_n, dtype=torch.float32, device=dev)
    ft = torch.empty(test_n, dtype=torch.float32, device=dev)
    gen_dataset(Xt, ft, test_n, 1, i0=0, xkind=3, ykind=5, seed=seed + 10_000, noise=False)
    f = fk.fk_predict_type2(theta, 1, m, 1.0, Xt, eps)
    return float(torch.mean((f.double() - ft.double()) ** 2))


def test_error_additive(n: int, seed: int, d: int = 5, test_n: int = 10_000, eps: float = 1e-6, chunk: int = 1 << 26) -> float:
    """Fig. 5: X ~ U(0,1)^5, Y = sum_l (e^{X_l/(l+1)} - 1) + N(0,1), low-bias additive,
    s = 2, lambda = n^{-2s/(2s+1)}, m = 1 + floor(n^{1/(2s+1)} / d) (reading of P:530)."""
    import torch

    from datagen.device import gen_dataset
    from paper_2509_02649_b200 import fit, fk

    m = 1 + int(n ** (1.0 / 5.0) / d)
    lam = n ** (-0.8)
    dev = torch.device("cuda")
    buf, mus, rs, G = fit.additive_buffers(d, m, dev)
    c = min(n, chunk)
    X = torch.empty(d, c, dtype=torch.float32, device=dev)  # SoA columns
    Y = torch.empty(c, dtype=torch.float32, device=dev)
    for i0 in range(0, n, c):
        k = min(c, n - i0)
        Xk = X[:, :k].t()
        gen_dataset(Xk, Y[:k], k, d, i0=i0, xkind=3, ykind=2, seed=seed, stride_n=1, stride_d=c)
        acc = i0 > 0
        for l in range(d):
            fk.fk_rhs_type1(Xk[:, l], Y[:k], 1.0, m, eps, r_out=rs[l], mu_out=mus[l], accumulate=acc, check=False)
        fk.fk_additive_cross_moments(Xk, 1.0, m, eps, G_out=G, accumulate=acc, check=False)
    theta, _ = fk.fk_solve(mus, rs, n, d, m, 1.0, lam, "additive", cross=G, report=False)
    Xt = torch.empty(test_n, d, dtype=torch.float32, device=dev)
    ft = torch.empty(test_n, dtype=torch.float32, device=dev)
    gen_dataset(Xt, ft, test_n, d, i0=0, xkind=3, ykind=2, seed=seed + 10_000, noise=False)
    f = fk.fk_predict_type2(theta, d, m, 1.0, Xt, eps, additive=True)
    return float(torch.mean((f.double() - ft.double()) ** 2))


def slope(ns, errs) -> float:
    import numpy as np

    return float(np.polyfit(np.log10(ns), np.log10(errs), 1)[0])


def run(ns, resamples: int, test_n: int = 10_000, additive: bool = False):
    import numpy as np

    rows = []
    for n in ns:
        fn = test_error_additive if additive else test_error
        e = [fn(int(n), seed=1 + 97 * k + int(math.log10(n)) * 7919, test_n=test_n) for k in range(resamples)]
        m = 1 + int(n ** 0.2 / 5) if additive else max(1, int(round(n ** (1 / 3))))
        rows.append({"n": int(n), "m": m, "test_mse": float(np.mean(e)), "std": float(np.std(e)), "resamples": resamples})
    return rows, slope([r["n"] for r in rows], [r["test_mse"] for r in rows])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-exp", type=int, default=3)
    ap.add_argument("--max-exp", type=int, default=9)
    ap.add_argument("--resamples", type=int, default=20)
    ap.add_argument("--additive", action="store_true", help="Fig. 5: low-bias additive d=5, s=2 (paper slope -0.8)")
    a = ap.parse_args()
    import torch

    from paper_2509_02649_b200 import build

    build.build()
    torch.cuda.set_device(0)
    rows, sl = run([10 ** e for e in range(a.min_exp, a.max_exp + 1)], a.resamples, additive=a.additive)
    for r in rows:
        print(json.dumps(r), flush=True)
    if a.additive:
        print(json.dumps({"experiment": "Fig. 5 (P:516-540) low-bias additive d=5, s=2, lambda=n^-0.8", "fitted_slope": sl,
                          "paper_slope": -0.8}))
    else:
        print(json.dumps({"experiment": "Fig. 1 (P:274-287) Sobolev s=1, lambda=n^-2/3, m=n^1/3", "fitted_slope": sl,
                          "paper_slope": -2 / 3}))


if __name__ == "__main__":
    main()
