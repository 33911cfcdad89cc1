"""Device time of fk_solve (report.ms = CUDA events around assembly + factorisation + solves)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_02649_b200 import fk
import datagen

def main():
    for d, m, kind in [(1, 50, "sobolev"), (1, 80, "sobolev"), (1, 1000, "sobolev"), (2, 32, "pik_box"), (10, 50, "additive")]:
        n = 100000
        if kind == "additive":
            X, Y = datagen.dataset(n, d=d, ykind="additive")
            Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
            mus = torch.zeros((d, 4 * m + 1), dtype=torch.complex128, device="cuda")
            rs = torch.zeros((d, 2 * m + 1), dtype=torch.complex128, device="cuda")
            for l in range(d):
                fk.fk_rhs_type1(Xd[:, l], Yd, 1.0, m, 1e-6, r_out=rs[l], mu_out=mus[l])
            G = fk.fk_additive_cross_moments(Xd, 1.0, m, 1e-6)
            args = (mus, rs, n, d, m, 1.0, 1e-5, "additive")
            kw = dict(cross=G)
        else:
            X, Y = datagen.dataset(n, d=d, ykind="expcos" if d == 2 else "sin")
            Xd = torch.from_numpy(X.reshape(-1) if d == 1 else X).cuda()
            r, mu = fk.fk_rhs_type1(Xd, torch.from_numpy(Y).cuda(), 1.0, m, 1e-6)
            args = (mu.reshape(-1), r.reshape(-1), n, d, m, 1.0, 1e-5, kind, 2.0)
            kw = dict(mu_pde=1.0, alpha=[[1, 0], [0, 2]], a_alpha=[1.0, -1.0], box=[[-1, 1], [-1, 1]]) if kind == "pik_box" else {}
        for _ in range(3):
            fk.fk_solve(*args, **kw)
        torch.cuda.synchronize()
        ms = []
        for _ in range(10):
            _, rep = fk.fk_solve(*args, **kw)
            ms.append(rep["ms"])
        t0 = time.perf_counter()
        for _ in range(20):
            fk.fk_solve(*args, report=False, **kw)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / 20 * 1e3
        print(f"d={d} m={m} {kind}: D={rep['n_unknowns']} device {np.median(ms):.3f} ms  wall/call {wall:.3f} ms  backward {rep['backward_err']:.1e}")

main()
