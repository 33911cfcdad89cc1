"""fk_solve on C3-size Sobolev systems: conjugate gradients (FK_SOLVER=pcg) against dense Cholesky
(FK_SOLVER=dense): time, iterations, backward error and the difference of theta."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_02649_b200 import build, fk
from datagen.device import gen_dataset
build.build()


def run(how, mu, r, n, d, m, lam, s, reps=3):
    os.environ["FK_SOLVER"] = how
    best = 1e9
    for _ in range(reps):
        th, rep = fk.fk_solve(mu, r, n, d, m, 1.0, lam, "sobolev", s)
        best = min(best, rep["ms"])
    del os.environ["FK_SOLVER"]
    return best, th, rep


cases = [(2, 64, 2.0, 1e-6, 0), (2, 64, 2.0, 1e-6, 1), (2, 40, 2.0, 1e-6, 0), (1, 3000, 1.0, 2.15e-7, 0), (1, 3000, 2.0, 1e-8, 0),
         (2, 90, 2.0, 1e-7, 0)]
sel = os.environ.get("CASES")
if sel:
    cases = [cases[int(i)] for i in sel.split(",")]
for d, m, s, lam, xk in cases:
    n = 20_000_000
    X = torch.empty(n, d, device="cuda") if d == 2 else torch.empty(n, device="cuda")
    Y = torch.empty(n, device="cuda")
    gen_dataset(X, Y, n, d, xkind=xk, ykind=2 if d == 2 else 0, seed=0)
    r, mu = fk.fk_rhs_type1(X, Y, 1.0, m, 1e-6)
    ms_d, th_d, rep_d = run("dense", mu, r, n, d, m, lam, s)
    ms_p, th_p, rep_p = run("pcg", mu, r, n, d, m, lam, s)
    diff = ((th_p - th_d).abs().norm() / th_d.abs().norm()).item()
    print(f"d={d} m={m} s={s} lam={lam} xkind={xk}: dense {ms_d:.2f} ms (bw {rep_d['backward_err']:.1e})  "
          f"pcg {ms_p:.2f} ms, {rep_p['iters']} it (bw {rep_p['backward_err']:.1e})  rel diff {diff:.1e}", flush=True)
