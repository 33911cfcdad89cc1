"""fk_solve_path for 16 lambdas at D = 4225 / 9409 / 16641 against one fk_solve per lambda (the
library picks the eigendecomposition or per-lambda solves by cost; before the per-lambda branch the
path took 99 / 661 / 2708 ms here, all by eigendecomposition)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_02649_b200 import build, fk
from datagen.device import gen_dataset
build.build()
n, d = 4_000_000, 2
for m in (32, 48, 64):
    X, Y = torch.empty(n, 2, device="cuda"), torch.empty(n, device="cuda")
    gen_dataset(X, Y, n, d, xkind=0, ykind=2, seed=0)
    r, mu = fk.fk_rhs_type1(X, Y, 1.0, m, 1e-6)
    lams = list(np.logspace(-9, -3, 16))
    fk.fk_solve_path(mu, r, n, d, m, 1.0, lams[:2], "sobolev", 2.0)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    th = fk.fk_solve_path(mu, r, n, d, m, 1.0, lams, "sobolev", 2.0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    cg = []
    for lam in lams:
        torch.cuda.synchronize(); a = time.perf_counter()
        t, rep = fk.fk_solve(mu, r, n, d, m, 1.0, lam, "sobolev", 2.0)
        torch.cuda.synchronize(); cg.append((time.perf_counter() - a) * 1e3)
    print(f"m={m} D={(2*m+1)**2}: fk_solve_path 16 lambdas {1e3*(t1-t0):.1f} ms; fk_solve per lambda (ms): "
          + " ".join(f"{c:.1f}" for c in cg), flush=True)
