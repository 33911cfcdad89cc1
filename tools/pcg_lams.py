"""CG vs dense fk_solve over a lambda sweep (iterations, time, agreement) -- cost-model check."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_02649_b200 import build, fk
from datagen.device import gen_dataset
build.build()
n, d = 4_000_000, 2
for m in (48, 64):
    X, Y = torch.empty(n, 2, device="cuda"), torch.empty(n, device="cuda")
    gen_dataset(X, Y, n, d, xkind=0, ykind=2, seed=0)
    r, mu = fk.fk_rhs_type1(X, Y, 1.0, m, 1e-6)
    for lam in np.logspace(-8, -4, 9):
        out = []
        for how in ("dense", "pcg"):
            os.environ["FK_SOLVER"] = how
            best = 1e9
            for _ in range(2):
                th, rep = fk.fk_solve(mu, r, n, d, m, 1.0, float(lam), "sobolev", 2.0)
                best = min(best, rep["ms"])
            out.append((best, rep["iters"], th))
        del os.environ["FK_SOLVER"]
        diff = ((out[1][2] - out[0][2]).abs().norm() / out[0][2].abs().norm()).item()
        print(f"m={m} lam={lam:.1e}: dense {out[0][0]:.2f} ms  pcg {out[1][0]:.2f} ms ({out[1][1]} it)  diff {diff:.1e}", flush=True)
