"""One C3-size fk_solve through the CG path after a warm-up (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_02649_b200 import build, fk
from datagen.device import gen_dataset
build.build()
n, d, m = 4_000_000, 2, 64
X, Y = torch.empty(n, 2, device="cuda"), torch.empty(n, device="cuda")
gen_dataset(X, Y, n, d, xkind=0, ykind=2, seed=0)
r, mu = fk.fk_rhs_type1(X, Y, 1.0, m, 1e-6)
for _ in range(2):
    th, rep = fk.fk_solve(mu, r, n, d, m, 1.0, 1e-6, "sobolev", 2.0)
torch.cuda.synchronize()
print(rep)
