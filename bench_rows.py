#!/usr/bin/env python
"""Per-row measurements of the hot path (SURVEY.md §8(a) rows not timed by bench.py's fit step
on their own), each against its roofline and beside the CPU oracle:

  A12 predict (type-2 gather)     queries/s and GB/s of Xq in + f out (8 B/query fp32) vs HBM peak
  A10/A11 solve                   GFLOP/s of the real Cholesky (D^3/3) vs the fp64 FMA peak
  A7/A8 DFT + deconvolution       post-spread time of fk_rhs_type1 (reduce + hand-written DFT + deconv)
  NEXT-1 lambda path              fk_solve_path over 300 lambdas vs 300 fk_solve calls
  NEXT-1 large path (path_large)  16 lambdas at D = 4225 / 9409 / 16641: path vs one fk_solve per lambda
  NEXT-3 CG vs dense (cg)         fk_solve with FK_SOLVER=pcg / dense on C3-size Sobolev systems
  library reference (libref)      cuBLAS DGEMM and cuSOLVER potrf rates (context for the solve rows)

    python bench_rows.py [--rows predict,solve,post,path]     -> one JSON line per measurement
    (cg, path_large and libref run only when named)
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# fp64 FMA peak from unit counts and clock: 148 SMs x 64 FP64 FMA/clk x 2 flop x 1.965 GHz
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


def hbm_peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except (OSError, ValueError, KeyError):
        return 6650.0


def timed(fn, reps=10, warm=3):
    import torch

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def row_predict(out):
    import numpy as np
    import torch

    import oracle
    from datagen.device import gen_dataset
    from paper_2509_02649_b200 import fk

    for d, m, nq, eps, dt in [(1, 1000, 1 << 30, 1e-6, torch.float32), (1, 1000, 1 << 27, 1e-10, torch.float64),
                              (2, 64, 1 << 28, 1e-6, torch.float32),
                              (2, 64, 1 << 26, 1e-10, torch.float64), (10, 50, 1 << 26, 1e-6, torch.float32)]:
        additive = d > 2
        rng = np.random.default_rng(0)
        D = d * (2 * m + 1) if additive else (2 * m + 1) ** d
        th = torch.from_numpy((rng.normal(size=D) + 1j * rng.normal(size=D)) / np.sqrt(D)).cuda()
        Xq32 = torch.empty((nq, d) if d > 1 else (nq,), dtype=torch.float32, device="cuda")
        gen_dataset(Xq32, None, nq, d, xkind=0, seed=1)
        Xq = Xq32.to(dt) if dt != torch.float32 else Xq32
        del Xq32
        res = torch.empty(nq, dtype=dt, device="cuda")
        ms = timed(lambda: fk.fk_predict_type2(th, d, m, 1.0, Xq, eps, additive=additive, out=res, check=False))
        bpq = (d + 1) * (4 if dt == torch.float32 else 8)
        gbs = nq * bpq / (ms * 1e-3) / 1e9
        # oracle beside it: direct sum on a bounded sample of queries
        ns = 2000 if d == 1 else 500
        xs = Xq[:ns].double().cpu().numpy()
        t0 = time.perf_counter()
        if additive:
            oracle.predict_additive(th.cpu().numpy(), xs, 1.0, m)
        else:
            oracle.predict(th.cpu().numpy(), xs, 1.0, m)
        tcpu = time.perf_counter() - t0
        out.append({"row": "A12 predict (type-2)", "d": d, "m": m, "additive": additive, "eps": eps, "dtype": str(dt).split(".")[-1],
                    "queries": nq, "ms": ms, "queries_per_s": nq / (ms * 1e-3),
                    "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm_peak(), "unit": "GB/s", "frac": gbs / hbm_peak(),
                                 "bytes_per_query": bpq},
                    "cpu_oracle": {"queries_per_s": ns / tcpu, "sample": ns, "threads": oracle.num_threads()}})
        del Xq, res


def row_solve(out):
    import numpy as np
    import torch

    import datagen
    import oracle
    from paper_2509_02649_b200 import fk

    HEAT = dict(alpha=[[1, 0], [0, 2]], a_alpha=[1.0, -1.0], box=[[-1.0, 1.0], [-1.0, 1.0]])
    for d, m, kind in [(1, 1000, "sobolev"), (2, 32, "pik_box"), (10, 50, "additive"), (2, 64, "sobolev")]:
        n = 200_000
        if kind == "additive":
            X, Y = datagen.dataset(n, d=d, ykind="additive")
            Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
            mus = torch.zeros((d, 4 * m + 1), dtype=torch.complex128, device="cuda")
            rs = torch.zeros((d, 2 * m + 1), dtype=torch.complex128, device="cuda")
            for l in range(d):
                fk.fk_rhs_type1(Xd[:, l], Yd, 1.0, m, 1e-6, r_out=rs[l], mu_out=mus[l])
            G = fk.fk_additive_cross_moments(Xd, 1.0, m, 1e-6)
            args, kw = (mus, rs, n, d, m, 1.0, 1e-5, "additive"), dict(cross=G)
        else:
            X, Y = datagen.dataset(n, d=d, ykind="expcos" if d == 2 else "sin")
            Xd = torch.from_numpy(X.reshape(-1) if d == 1 else X).cuda()
            r, mu = fk.fk_rhs_type1(Xd, torch.from_numpy(Y).cuda(), 1.0, m, 1e-6)
            args = (mu.reshape(-1), r.reshape(-1), n, d, m, 1.0, 1e-6, kind, 2.0)
            kw = dict(mu_pde=1.0, **HEAT) if kind == "pik_box" else {}
        for _ in range(2):
            fk.fk_solve(*args, **kw)
        reps = []
        for _ in range(5):
            _, rep = fk.fk_solve(*args, **kw)
            reps.append(rep["ms"])
        ms = float(np.median(reps))
        D = rep["n_unknowns"]
        gflops = (D + 1) ** 3 / 3.0 / (ms * 1e-3) / 1e9
        cpu = None
        if D <= 4225:  # numpy / LAPACK complex solve of the same system (the oracle's solve)
            A = np.eye(D, dtype=np.complex128) + 0.01
            b = np.ones(D, dtype=np.complex128)
            t0 = time.perf_counter()
            np.linalg.solve(A, b)
            cpu = {"ms": 1e3 * (time.perf_counter() - t0), "what": "numpy.linalg.solve complex128 (the oracle's dense solve)"}
        if rep["iters"] > 0:  # the CG path: the N^3/3 Cholesky model does not describe it
            roof = {"bound": "latency", "note": f"conjugate gradients, {rep['iters']} iterations of FFT-Toeplitz products "
                    "(5 own kernels + cuFFT each) after a dense-block inverse; dense Cholesky of the same system: "
                    f"(N^3/3 = {(D + 1) ** 3 / 3.0:.3g} flops) see profiles/r01_pcg_c3_launches.txt"}
        else:
            roof = {"bound": "alu", "achieved": gflops / 1e3, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                    "frac": gflops / 1e3 / FP64_PEAK_TFLOPS, "flops": (D + 1) ** 3 / 3.0,
                    "peak_source": "148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz"}
        out.append({"row": "A10/A11 assemble + solve", "d": d, "m": m, "kind": kind, "D": D, "ms": ms, "iters": rep["iters"],
                    "backward_err": rep["backward_err"], "roofline": roof, "cpu_oracle": cpu})


def row_post(out):
    import torch

    from datagen.device import gen_dataset
    from paper_2509_02649_b200 import fk

    for d, m, n in [(1, 1000, 1 << 24), (1, 50, 1 << 24), (2, 64, 1 << 24), (2, 32, 1 << 24)]:
        X = torch.empty((n, d) if d > 1 else (n,), dtype=torch.float32, device="cuda")
        Y = torch.empty(n, dtype=torch.float32, device="cuda")
        gen_dataset(X, Y, n, d, xkind=0, ykind=1 if d == 2 else 0, seed=2)
        r = torch.zeros((2 * m + 1,) * d, dtype=torch.complex128, device="cuda")
        mu = torch.zeros((4 * m + 1,) * d, dtype=torch.complex128, device="cuda")
        fk.profile_read()
        fk.profile_enable(True)
        ms = timed(lambda: fk.fk_rhs_type1(X, Y, 1.0, m, 1e-6, r_out=r, mu_out=mu, check=False), reps=10, warm=3)
        fk.profile_enable(False)
        sp, nl, _ = fk.profile_read()
        spread = sp / max(1, nl)
        out.append({"row": "A7/A8 reduce + FFT + deconvolution (post-spread part of fk_rhs_type1)", "d": d, "m": m, "n": n,
                    "total_ms": ms, "spread_ms": spread, "post_spread_ms": ms - spread,
                    "roofline": {"bound": "latency", "note": "fixed cost per fit: tiny grids (<= 1 MB), a handful of launches"}})
        del X, Y


def row_path(out):
    import numpy as np
    import torch

    import datagen
    from paper_2509_02649_b200 import fk

    lams = list(np.logspace(-9, -1, 300))
    for d, m, kind in [(1, 1000, "sobolev"), (10, 50, "additive"), (2, 32, "sobolev")]:
        n = 200_000
        X, Y = datagen.dataset(n, d=d, ykind="additive" if kind == "additive" else ("expcos" if d == 2 else "sin"))
        Xd, Yd = torch.from_numpy(X.reshape(-1) if d == 1 else X).cuda(), torch.from_numpy(Y).cuda()
        kw = {}
        if kind == "additive":
            mu = torch.zeros((d, 4 * m + 1), dtype=torch.complex128, device="cuda")
            r = torch.zeros((d, 2 * m + 1), dtype=torch.complex128, device="cuda")
            for l in range(d):
                fk.fk_rhs_type1(Xd[:, l], Yd, 1.0, m, 1e-6, r_out=r[l], mu_out=mu[l])
            kw["cross"] = fk.fk_additive_cross_moments(Xd, 1.0, m, 1e-6)
        else:
            r, mu = fk.fk_rhs_type1(Xd, Yd, 1.0, m, 1e-6)
            mu, r = mu.reshape(-1), r.reshape(-1)
        th = torch.empty(len(lams), d * (2 * m + 1) if kind == "additive" else (2 * m + 1) ** d, dtype=torch.complex128, device="cuda")
        ms_path = timed(lambda: fk.fk_solve_path(mu, r, n, d, m, 1.0, lams, kind, 2.0, theta_out=th, check=False, **kw), reps=3, warm=1)
        one = th[0].clone()
        ms_chol = timed(lambda: [fk.fk_solve(mu, r, n, d, m, 1.0, lam, kind, 2.0, theta_out=one, report=False, **kw) for lam in lams],
                        reps=1, warm=1)
        # agreement of the two methods at the median lambda
        l = len(lams) // 2
        ch, _ = fk.fk_solve(mu, r, n, d, m, 1.0, lams[l], kind, 2.0, **kw)
        err = float(torch.linalg.norm(th[l] - ch) / torch.linalg.norm(ch))
        out.append({"row": "NEXT-1 lambda path (one eigendecomposition, P:542-548)", "d": d, "m": m, "kind": kind,
                    "D": th.shape[1], "n_lambda": len(lams), "path_ms": ms_path, "cholesky_per_lambda_ms": ms_chol,
                    "speedup": ms_chol / ms_path, "rel_diff_vs_cholesky": err})
        del Xd, Yd


def _device_data(n, d, m, xkind=0, seed=0):
    import torch

    from datagen.device import gen_dataset
    from paper_2509_02649_b200 import fk

    X = torch.empty(n, d, device="cuda") if d == 2 else torch.empty(n, device="cuda")
    Y = torch.empty(n, device="cuda")
    gen_dataset(X, Y, n, d, xkind=xkind, ykind=2 if d == 2 else 0, seed=seed)
    r, mu = fk.fk_rhs_type1(X, Y, 1.0, m, 1e-6)
    del X, Y
    return r, mu


def row_cg(out):
    """CG (FK_SOLVER=pcg) against dense Cholesky (FK_SOLVER=dense) on C3-size Sobolev systems: time,
    iterations, backward error, agreement of theta -- the data behind fk_solve's cost model."""
    from paper_2509_02649_b200 import fk

    def run(how, mu, r, n, d, m, lam, s, reps=3):
        os.environ["FK_SOLVER"] = how
        try:
            best = 1e9
            for _ in range(reps):
                th, rep = fk.fk_solve(mu, r, n, d, m, 1.0, lam, "sobolev", s)
                best = min(best, rep["ms"])
        finally:
            del os.environ["FK_SOLVER"]
        return best, th, rep

    n = 20_000_000
    for d, m, s, lam, xk in [(2, 64, 2.0, 1e-6, 0), (2, 64, 2.0, 1e-6, 1), (2, 40, 2.0, 1e-6, 0), (1, 3000, 1.0, 2.15e-7, 0),
                             (2, 90, 2.0, 1e-7, 0), (2, 64, 2.0, 1e-8, 0), (2, 64, 2.0, 1e-4, 0)]:
        r, mu = _device_data(n, d, m, xkind=xk)
        ms_d, th_d, rep_d = run("dense", mu, r, n, d, m, lam, s)
        ms_p, th_p, rep_p = run("pcg", mu, r, n, d, m, lam, s)
        diff = ((th_p - th_d).abs().norm() / th_d.abs().norm()).item()
        out.append({"row": "NEXT-3 CG vs dense solve", "d": d, "m": m, "s": s, "lambda": lam, "xkind": xk, "D": rep_d["n_unknowns"],
                    "dense_ms": ms_d, "dense_backward_err": rep_d["backward_err"], "cg_ms": ms_p, "cg_iters": rep_p["iters"],
                    "cg_backward_err": rep_p["backward_err"], "rel_diff": diff})


def row_path_large(out):
    """fk_solve_path for 16 lambdas at D = 4225 / 9409 / 16641 against one fk_solve per lambda (the
    library picks the eigendecomposition or per-lambda solves by cost)."""
    import numpy as np
    import torch

    from paper_2509_02649_b200 import fk

    n, d = 4_000_000, 2
    lams = list(np.logspace(-9, -3, 16))
    for m in (32, 48, 64):
        r, mu = _device_data(n, d, m)
        fk.fk_solve_path(mu, r, n, d, m, 1.0, lams[:2], "sobolev", 2.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fk.fk_solve_path(mu, r, n, d, m, 1.0, lams, "sobolev", 2.0)
        torch.cuda.synchronize()
        path_ms = 1e3 * (time.perf_counter() - t0)
        per = []
        for lam in lams:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fk.fk_solve(mu, r, n, d, m, 1.0, lam, "sobolev", 2.0)
            torch.cuda.synchronize()
            per.append(1e3 * (time.perf_counter() - t0))
        out.append({"row": "NEXT-1 lambda path, large D", "d": d, "m": m, "D": (2 * m + 1) ** 2, "n_lambda": len(lams),
                    "path_ms": path_ms, "solve_per_lambda_ms": per, "solve_all_ms": sum(per)})


def row_libref(out):
    """Library reference rates on this GPU (context for the solve rows): cuBLAS DGEMM and the cuSOLVER
    Cholesky behind torch.linalg.cholesky at the C3 system size."""
    import torch

    def t(f, r=5):
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        best = 1e9
        for _ in range(r):
            e0.record()
            f()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    for N in (4096, 8192, 16384):
        a = torch.randn(N, N, dtype=torch.float64, device="cuda")
        b = torch.randn_like(a)
        ms = t(lambda: a @ b)
        out.append({"row": "library reference: cuBLAS DGEMM", "N": N, "ms": ms, "tflops": 2 * N ** 3 / ms / 1e9})
        del a, b
    N = 16641
    A = torch.randn(N, N, dtype=torch.float64, device="cuda")
    A = A @ A.T / N + torch.eye(N, dtype=torch.float64, device="cuda")
    ms = t(lambda: torch.linalg.cholesky(A), 3)
    out.append({"row": "library reference: cuSOLVER potrf (torch.linalg.cholesky)", "N": N, "ms": ms, "tflops": N ** 3 / 3 / ms / 1e9})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="predict,solve,post,path")
    a = ap.parse_args()
    import torch

    from paper_2509_02649_b200 import build

    build.build()
    torch.cuda.set_device(0)
    out = []
    rows = {"predict": row_predict, "solve": row_solve, "post": row_post, "path": row_path, "cg": row_cg,
            "path_large": row_path_large, "libref": row_libref}
    for r in a.rows.split(","):
        rows[r](out)
    for o in out:
        print(json.dumps(o), flush=True)


if __name__ == "__main__":
    main()
