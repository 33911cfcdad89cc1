#!/usr/bin/env python
"""Benchmark of the fit path (moments + rhs in one pass over the samples, then the solve).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl fk|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one process per GPU, NCCL)

A step = one whole fit over the configuration's n samples, which are generated on the device
(seeded, counter-based: datagen/gen.cu) BEFORE the timed region and stay resident in HBM.
Multi-GPU is strong scaling: rank r owns samples [r n/N, (r+1) n/N) of the same global dataset,
spreads them, the small complex128 [mu | r (| G)] vector is all-reduced over NCCL, rank 0 solves,
theta is broadcast.  Time = CUDA events on the launching stream between barriers, max over ranks.
Default workload: BASELINE config C2 (d=1, m=1000, n=1e10), which fits one B200 (80 GB).

Rank 0 prints ONE JSON line (DESIGN.md §6 explains every key).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples/sec fit (moments+solve) at 1/2/4/8 B200; HBM GB/s vs 8 TB/s"
HEAT = dict(alpha=[[1, 0], [0, 2]], a_alpha=[1.0, -1.0], box=[[-1.0, 1.0], [-1.0, 1.0]])

# BASELINE.json configs C1..C5; s, lambda, mu, PDE per the paper's schedules (reading R6)
CONFIGS = {
    "c1": dict(d=1, m=50, n=100_000, s=2.0, lam=1e5 ** -0.8, kind="sobolev", xkind=0, ykind=0,
               desc="C1 Sobolev d=1 s=2 m=50 n=1e5 uniform X on [-1,1], Y=sin-like+N(0,1)"),
    "c2": dict(d=1, m=1000, n=10_000_000_000, s=1.0, lam=1e10 ** (-2.0 / 3.0), kind="sobolev", xkind=0, ykind=0,
               desc="C2 Sobolev d=1 s=1 m=1000 n=1e10 uniform X on [-1,1], Y=sin-like+N(0,1)"),
    "c3": dict(d=2, m=64, n=1_000_000_000, s=2.0, lam=1e-6, kind="sobolev", xkind=0, ykind=1,
               desc="C3 Sobolev d=2 s=2 m=64 (129^2 modes, 257^2 moments) n=1e9 uniform X, Y=exp(x1)cos(x2)-like+N(0,1)"),
    "c4": dict(d=2, m=32, n=100_000_000, s=2.0, lam=1e8 ** (-2.0 / 3.0), kind="pik_box", xkind=0, ykind=1, mu_pde=1.0,
               desc="C4 physics-informed d=2 space-time heat penalty d_t f - d_xx f on [-1,1]^2, mu=1, s=2, m=32, n=1e8"),
    "c5": dict(d=10, m=50, n=1_000_000_000, s=2.0, lam=1e9 ** -0.8, kind="additive", xkind=0, ykind=2,
               desc="C5 low-bias additive d=10 m=50 n=1e9 (10 1-D moment/rhs passes + 45 pairwise 2-D cross moments), X SoA"),
}
NOMINAL_HBM_GBS = 8000.0
# measured int32 shared-memory ATOMS.ADD lane-ops/s, chip-wide (profiles/r01_microbench_spread.log):
ATOMS_RANDOM_PEAK = 2.604e12     # random addresses (3.5-way bank conflicts: what a random scatter can reach)
ATOMS_CFREE_PEAK = 9.065e12      # conflict-free (one wavefront per instruction: the hardware ceiling)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="fk", choices=["fk", "reference"])
    ap.add_argument("--n", type=float, default=None, help="override n (profiling runs only)")
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--xkind", default=None, choices=[None, "uniform", "gaussian"])
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the fit as one CUDA graph (auto: one GPU and n <= 1e7, the launch-bound configs)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-n", type=float, default=float(1 << 30))
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: exercise the distributed branch on one GPU / CPU transport)")
    ap.add_argument("--no-paper-precision", action="store_true",
                    help="skip the fp64-mode (eps = 1e-10, the paper's complex-128 arithmetic) record of the d = 1 configs")
    ap.add_argument("--pp-steps", type=int, default=3)
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the compact records of C1, C3, C4, C5 appended to the default (C2, one GPU) line")
    return ap.parse_args()


def pi_kwargs(cfg):
    return dict(mu_pde=cfg["mu_pde"], **HEAT) if cfg["kind"] == "pik_box" else {}


# ---------------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg and --impl reference); the only place bench runs oracle/
# ---------------------------------------------------------------------------------------------
def oracle_fit_rate(cfg, target_s: float):
    """(samples/s, sample size, seconds, threads, note) of the fp64 oracle on a bounded sample."""
    import datagen
    import oracle

    oracle.build()
    d, m = cfg["d"], cfg["m"]
    xk = "uniform" if cfg["xkind"] == 0 else "gaussian"
    yk = {0: "sin", 1: "expcos", 2: "additive"}[cfg["ykind"]]
    D = d * (2 * m + 1) if cfg["kind"] == "additive" else (2 * m + 1) ** d
    with_solve = D <= 5000
    note = "moments+rhs by fp64 direct sum" + (" + dense solve" if with_solve else "; the dense solve (D=%d) is not timed on CPU" % D)

    def one(n):
        X, Y = datagen.dataset(n, d=d, xkind=xk, ykind=yk, seed=0)
        t0 = time.perf_counter()
        if cfg["kind"] == "additive":
            mu_l = [oracle.moments(X[:, l], 1.0, m) for l in range(d)]
            r_l = [oracle.rhs(X[:, l], Y, 1.0, m) for l in range(d)]
            G = oracle.cross_moments(X, 1.0, m)
            if with_solve:
                oracle.solve_additive(mu_l, r_l, G, n, d, m, cfg["lam"])
        else:
            mu = oracle.moments(X, 1.0, m)
            r = oracle.rhs(X, Y, 1.0, m)
            if with_solve:
                kw = dict(pi_kwargs(cfg), L=1.0) if cfg["kind"] == "pik_box" else {}
                oracle.solve(mu, r, n, d, m, cfg["lam"], cfg["kind"], cfg["s"], **kw)
        return time.perf_counter() - t0

    n, t = 256, one(256)
    while t < target_s / 4 and n < 20_000_000:
        n *= 4
        t = one(n)
    if t < target_s * 0.6:
        n = int(n * target_s / max(t, 1e-3))
        t = one(n)
    return n / t, n, t, oracle.num_threads(), note


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return 0
    rates = []
    n_s = cores = note = None
    target = max(2.0, min(10.0, 150.0 / max(1, args.steps + args.warmup)))
    for i in range(args.warmup + args.steps):
        rate, n_s, t, cores, note = oracle_fit_rate(cfg, target)
        if i >= args.warmup:
            rates.append(rate)
    v = statistics.median(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * n_s / v, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "n": cfg["n"], "d": cfg["d"], "m": cfg["m"], "s": cfg["s"], "lambda": cfg["lam"],
                   "sample_per_step": n_s, "note": "CPU oracle (oracle/direct.c OpenMP + numpy) on a bounded sample: " + note},
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "oracle",
                         "sample": f"{n_s} samples of the same workload per step ({cpu_model()}); {note}"},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return

        def rd():
            for line in self.proc.stdout:
                self.rows.append([c.strip() for c in line.split(",")])

        self.thread = threading.Thread(target=rd, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
                for nm, v in zip(names, r[2:6]):
                    if v.lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def ncu_traffic(config: str):
    """dram bytes per sample of the spreading kernel from the committed ncu --set full capture."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(config)
    except (OSError, ValueError):
        return None


def es_width(eps):
    """Taps per dimension of the d = 2 spreading window (csrc/spread2d.cu es_width, sigma = 2):
    fp32 fixed-point path 5..8, fp64 mode (eps < 1e-7) 9..16."""
    import math

    if eps >= 1e-7:
        return min(8, max(5, int(math.ceil(math.log10(1.0 / eps))) + 1))
    return min(16, max(9, int(math.ceil(math.log10(1.0 / eps))) + 2))


def spread2d_width(eps):
    """Taps per dimension of the d = 2 type-1 pass (csrc/spread2d.cu make_plan2): sigma = 2, or
    sigma = 4 with one tap fewer on the fp32 path when FK_SPREAD2D_SIGMA=4 (measurement)."""
    w = es_width(eps)
    if eps >= 1e-7 and os.environ.get("FK_SPREAD2D_SIGMA", "2") == "4":
        return max(5, w - 1)
    return w


def cross_width(eps, m):
    """Taps per dimension of the cross-moment window: sigma = 4 with one tap fewer when one pair
    grid fits a CTA (csrc/spread2d.cu make_planx, fp32 path only), else the sigma = 2 width."""
    w = es_width(eps)
    if eps < 1e-7:
        return w
    w4 = max(5, w - 1)
    nf4 = 4 * (2 * m + 1)
    nf4 = next(v for v in range(nf4, 8 * nf4 + 64) if v % 8 == 0 and _smooth(v))
    g4 = nf4 // 2 + w4 + 4
    return w4 if g4 * g4 * 4 <= 232448 - 2048 else w


def _smooth(v):
    for p in (2, 3, 5):
        while v % p == 0:
            v //= p
    return v == 1


# ---------------------------------------------------------------------------------------------
# the GPU arm
# ---------------------------------------------------------------------------------------------
def main():
    args = parse()
    cfg = dict(CONFIGS[args.config])
    if args.n is not None:
        cfg["n"] = int(args.n)
    if args.xkind is not None:
        cfg["xkind"] = 0 if args.xkind == "uniform" else 1
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    import torch
    import torch.distributed as dist

    from datagen.device import gen_dataset
    from paper_2509_02649_b200 import build, fk
    from paper_2509_02649_b200.fit import _moment_buffers, additive_buffers, fit_additive_distributed, fit_distributed

    if not os.path.exists(fk.LIB_PATH):
        build.build()
    local = local % max(1, torch.cuda.device_count())  # gloo runs may place several ranks on one GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    d, m, n = cfg["d"], cfg["m"], cfg["n"]
    L, eps = 1.0, args.eps
    lo = n * rank // world
    hi = n * (rank + 1) // world
    n_loc = hi - lo
    additive = cfg["kind"] == "additive"
    Y = torch.empty(n_loc, dtype=torch.float32, device=dev)
    if additive:  # SoA: one contiguous column per feature
        Xsoa = torch.empty((d, n_loc), dtype=torch.float32, device=dev)
        gen_dataset(Xsoa, Y, n_loc, d, i0=lo, xkind=cfg["xkind"], ykind=cfg["ykind"], seed=0, stride_n=1, stride_d=n_loc)
        X = Xsoa.t()
        buffers = additive_buffers(d, m, dev)
        theta = torch.empty(d * (2 * m + 1), dtype=torch.complex128, device=dev)
    else:
        X = torch.empty((n_loc,) if d == 1 else (n_loc, d), dtype=torch.float32, device=dev)
        gen_dataset(X, Y, n_loc, d, i0=lo, xkind=cfg["xkind"], ykind=cfg["ykind"], seed=0)
        buffers = _moment_buffers(d, m, dev)
        theta = torch.empty((2 * m + 1) ** d, dtype=torch.complex128, device=dev)
    pik = pi_kwargs(cfg)
    status = torch.zeros(1, dtype=torch.int32, device=dev)  # FK_DSTATUS_* bits of every fit (read after timing)

    # small fits are launch-latency bound: one CUDA graph per fit (type-1 pass + solve), one GPU only
    use_graph = args.graph == "on" or (args.graph == "auto" and world == 1 and not additive and n <= 10_000_000)
    graph = None
    if use_graph:
        from paper_2509_02649_b200.fit import FitGraph

        graph = FitGraph(X, Y, L, m, cfg["lam"], cfg["kind"], cfg["s"], eps, **pik)

    def step():
        if graph is not None:
            graph.replay()
        elif additive:
            fit_additive_distributed(X, Y, n, L, m, cfg["lam"], eps, buffers=buffers, theta_out=theta, status=status)
        else:
            fit_distributed(X, Y, n, L, m, cfg["lam"], cfg["kind"], cfg["s"], eps, buffers=buffers, theta_out=theta, status=status,
                            **pik)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    fk.profile_read()
    fk.profile_enable(True)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    fk.profile_enable(False)
    spread_ms, spread_launches, kernels = fk.profile_read()
    if graph is not None:  # replays launch the captured kernels; the spread time comes from a timed eager pass
        kernels = graph.launches * args.steps
        fk.profile_enable(True)
        fit_distributed(X, Y, n, L, m, cfg["lam"], cfg["kind"], cfg["s"], eps, buffers=buffers, theta_out=theta, **pik)
        torch.cuda.synchronize()
        fk.profile_enable(False)
        sp1, nl1, _ = fk.profile_read()
        spread_ms, spread_launches = sp1 * args.steps, nl1 * args.steps
    if graph is not None:
        graph.check()
    fit_ok = int(status.item()) == 0  # no skipped coordinate, factorisation SPD, no watchdog
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    value = n / (ms_step * 1e-3)

    peaks = measured_peaks()
    spread_per_step_ms = spread_ms / args.steps
    bytes_step = n_loc * (d + 1) * 4 if not additive else n_loc * (d + 1) * 4
    if d == 1:
        # dominant kernel = the one-pass spread: algorithmic 8 B per local sample
        avg = spread_ms / max(1, spread_launches)
        achieved = n_loc * 8 / (avg * 1e-3) / 1e9
        peak = peaks.get("hbm_gbs", 6650.0)
        tr = ncu_traffic(args.config)
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": None if tr is None else tr["dram_bytes_per_sample"] * n_loc,
                "kernel": "k_spread1d_bs3 (one pass over X, Y)",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s",
                "frac_of_nominal_8tbs": achieved / NOMINAL_HBM_GBS, "spread_ms_avg": avg, "bytes_per_launch": n_loc * 8,
                "spread_share_of_step": spread_per_step_ms / ms_step,
                # the resource that binds this kernel: 8 int32 shared-memory atomics per sample (4 cubic
                # B-spline taps x 2 channels) against the measured random-address ATOMS.ADD rate --
                # ~9.5 lane-ops/clk/SM for ANY non-consecutive address pattern, bank-conflict-free ones
                # included (profiles/r02_microbench_atoms_patterns.log)
                "atomics": {"bound": "alu", "achieved": 8 * n_loc / (avg * 1e-3) / 1e9, "peak": ATOMS_RANDOM_PEAK / 1e9,
                            "unit": "Gatomic/s", "frac": 8 * n_loc / (avg * 1e-3) / ATOMS_RANDOM_PEAK,
                            "peak_source": "measured random-address int32 ATOMS.ADD, profiles/r01_microbench_spread.log"}}
    else:
        # d >= 2 / additive: bound by random-address shared-memory atomics (2 w^2 per sample for d = 2,
        # npairs w^2 + 2 d x 4 per sample for the additive model); peak = the measured random ATOMS rate
        # fp64 mode: 64-bit fixed point as int32 pairs, up to 2 ATOMS per tap (pair_add: low word, and
        # the high word when the tap's high part or the carry is non-zero -- counted as 2, an upper bound)
        w = spread2d_width(eps)
        per_tap = 2 if eps < 1e-7 else 1
        d1 = 8 if eps >= 1e-7 else 2 * 8 * 2  # per-feature 1-D pass: 2 channels x 4 taps (fp32); 2 x 8 septic taps x 2 words
        if additive:
            wc = cross_width(eps, m)
            atoms = n_loc * (d * (d - 1) // 2 * wc * wc * per_tap + d * d1)
        else:
            atoms = n_loc * 2 * w * w * per_tap
        achieved = atoms / (spread_per_step_ms * 1e-3) / 1e9
        tr = ncu_traffic(args.config)
        roof = {"bound": "alu", "achieved": achieved, "peak": ATOMS_CFREE_PEAK / 1e9, "unit": "Gatomic/s",
                "frac": achieved * 1e9 / ATOMS_CFREE_PEAK, "traffic": None if tr is None else tr["dram_bytes_per_sample"] * n_loc,
                "frac_of_random_atoms": achieved * 1e9 / ATOMS_RANDOM_PEAK,
                "kernel": "spreading kernels (shared-memory int32 atomics)",
                "peak_source": "measured conflict-free int32 ATOMS.ADD rate (9.07e12/s); frac_of_random_atoms: vs the measured "
                               "random-address rate (2.60e12/s), profiles/r01_microbench_spread.log",
                "atomics_counted": f"{'2 w^2' if not additive else 'npairs w^2 + d x (1-D pass)'} per sample, w = {w}"
                                   + (f", cross w = {cross_width(eps, m)}" if additive else "")
                                   + (", x2 int32 words per tap (fp64 mode, upper bound)" if eps < 1e-7 else ""),
                "hbm_gbs": bytes_step / (spread_per_step_ms * 1e-3) / 1e9, "spread_ms_per_step": spread_per_step_ms,
                "spread_share_of_step": spread_per_step_ms / ms_step, "atomics_per_step": atoms}

    pp = None
    if d == 1 and eps >= 1e-7 and not args.no_paper_precision and graph is None:
        pp = paper_precision(args, cfg, X, Y, n, n_loc, world, dev, buffers, theta, pik, peaks)
    others = None
    rows = None
    if args.config == "c2" and args.n is None and world == 1 and not args.no_other_configs:
        rows = c2_rows(args, cfg, buffers, theta, n, peaks, dev)
        del X, Y, buffers
        torch.cuda.empty_cache()
        others = other_configs(args, dev)
    e2e = None
    if not args.no_e2e and rank == 0:
        e2e = run_e2e_additive(args, cfg, dev, eps) if additive else run_e2e(args, cfg, dev, eps)
    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:
        rate, n_s, t_s, cores, note = oracle_fit_rate(cfg, args.cpu_seconds)
        cpu = {"value": rate, "unit": "samples/s", "cores": cores, "kind": "oracle",
               "sample": f"{n_s} samples of {args.config} in {t_s:.1f} s on {cpu_model()}: {note}"}
    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if eps < 1e-7 else "f32",  # fp64 mode: fp64 taps, 64-bit fixed-point sums
            "data": "synthetic",
            "config": {"workload": cfg["desc"], "n": n, "d": d, "m": m, "s": cfg["s"], "lambda": cfg["lam"], "eps": eps, "L": L,
                       "kind": cfg["kind"], "xkind": "uniform" if cfg["xkind"] == 0 else "gaussian",
                       "parallelism": f"dp{world}: sample shards, NCCL all-reduce of the moment vector, solve on rank 0",
                       "cache": (f"inputs {bytes_step / 1e9:.1f} GB/GPU >> 126 MB L2 (no flush needed)" if bytes_step > 2e8 else
                                 f"inputs {bytes_step / 1e6:.1f} MB/GPU: L2-resident across steps (launch-bound config)"),
                       "cuda_graph": graph is not None},
            "roofline": roof,
            "fit_status_ok": fit_ok,
            "paper_precision": pp,
            "other_configs": others,
            "rows": rows,
            "hbm_gbs_fit": n_loc * (d + 1) * 4 / (ms_step * 1e-3) / 1e9,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": kernels,
            "clocks": clk,
            "paper_context": "paper: n=1e10 d=1 Sobolev fit in ~1 min on NVIDIA T4, complex128, m=n^(1/3)=2154 (P:286) ~ 1.7e8 samples/s",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def paper_precision(args, cfg, X, Y, n, n_loc, world, dev, buffers, theta, pik, peaks):
    """The same fit at the paper's arithmetic (sec. 3.1: complex-128): the fp64 mode,
    eps = 1e-10 (septic B-spline window, 64-bit fixed-point sums), on the same resident fp32 X, Y.
    Timed like the main line (CUDA events between barriers, max over ranks), with its own clocks,
    the spreading kernels' roofline and the moment checks available at this size."""
    import torch
    import torch.distributed as dist

    from paper_2509_02649_b200 import fk
    from paper_2509_02649_b200.fit import _moment_buffers, fit_distributed

    eps = 1e-10
    bufs = _moment_buffers(1, cfg["m"], dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)

    def step():
        fit_distributed(X, Y, n, 1.0, cfg["m"], cfg["lam"], cfg["kind"], cfg["s"], eps, buffers=bufs, theta_out=theta, status=st, **pik)

    step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    fk.profile_read()
    fk.profile_enable(True)
    clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clocks.start()
    time.sleep(0.3)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.pp_steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.pp_steps
    clk = clocks.stop()
    fk.profile_enable(False)
    sp_ms, sp_launches, kernels = fk.profile_read()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    # one pass per channel (X read twice): algorithmic 8 B per sample over the two passes of a fit
    sp_step = sp_ms / args.pp_steps
    achieved = n_loc * 8 / (sp_step * 1e-3) / 1e9
    peak = peaks.get("hbm_gbs", 6650.0)
    _, mu64, r64 = bufs
    _, mu32, r32 = buffers  # the main line's last fit (fp32 mode) of the same data
    mu64h, mu32h, r64h, r32h = (v.reshape(-1).cpu().numpy() for v in (mu64, mu32, r64, r32))
    import numpy as np

    K = 2 * cfg["m"]
    herm = float(np.max(np.abs(mu64h[::-1] - np.conj(mu64h))) / abs(mu64h[K]))
    return {
        "value": n / (ms * 1e-3), "unit": "samples/s", "ms_per_step": ms, "steps": args.pp_steps, "dtype": "f64",
        "config": {"workload": cfg["desc"], "eps": eps, "n": n, "storage": "fp32 X, Y (as the main line)",
                   "window": "septic B-spline (8 taps, sigma ~ 11), 64-bit fixed point, one pass per channel"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "kernel": "k_spread1d_bs7 (2 launches per fit: moments, rhs)",
                     "spread_ms_per_step": sp_step, "spread_share_of_step": sp_step / ms,
                     "note": "algorithmic 8 B/sample per fit; the kernel is bound by its shared-memory pair atomics (DESIGN.md §5)"},
        "clocks": clk, "gpu_launches": kernels,
        "moment_checks": {"mu0_exact": bool(mu64h[K].real == n and mu64h[K].imag == 0.0), "hermitian_rel": herm,
                          "rel_l2_vs_fp32_mode_mu": float(np.linalg.norm(mu64h - mu32h) / np.linalg.norm(mu64h)),
                          "rel_l2_vs_fp32_mode_r": float(np.linalg.norm(r64h - r32h) / np.linalg.norm(r64h)),
                          "oracle_parity": "tests/test_gpu_d1.py::test_type1_fp64_matches_oracle, test_fit_c2_shape_end_to_end[*-fp64] "
                                           "(<= 1e-10 l2 and 1e-9 n per element vs the fp64 direct sums)"},
        "fit_status_ok": int(st.item()) == 0,
    }


def c2_rows(args, cfg, buffers, theta, n, peaks, dev):
    """The two other timed rows of the C2 path, on the fit's own moments and theta, so the driver's
    default run sees them (bench_rows.py has the full set): the solve (A10/A11: assembly, tile
    Cholesky, back substitution; CUDA events inside fk_solve, median of 7) and the type-2 prediction
    (A12) of 2^30 resident fp32 queries, against the HBM roofline of its 8 B per query."""
    import torch

    from paper_2509_02649_b200 import fk

    d, m, L = cfg["d"], cfg["m"], 1.0
    _, mu, r = buffers
    ms = []
    for _ in range(9):
        _, rep_ = fk.fk_solve(mu.reshape(-1), r.reshape(-1), n, d, m, L, cfg["lam"], cfg["kind"], cfg["s"], report=True)
        ms.append(rep_["ms"])
    ms = sorted(ms[2:])
    solve = {"row": "A10/A11 assemble + solve", "D": rep_["n_unknowns"], "ms": ms[len(ms) // 2], "backward_err": rep_["backward_err"],
             "rcond_est": rep_["rcond_est"], "method": "tile dataflow Cholesky + multi-SM back substitution (fp64)"}
    nq = 1 << 30
    Xq = torch.rand(nq, device=dev, dtype=torch.float32) * 2.0 - 1.0
    out = torch.empty(nq, device=dev, dtype=torch.float32)
    for _ in range(3):
        fk.fk_predict_type2(theta, d, m, L, Xq, args.eps, out=out)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        fk.fk_predict_type2(theta, d, m, L, Xq, args.eps, out=out)
    e1.record(s)
    torch.cuda.synchronize()
    pms = e0.elapsed_time(e1) / reps
    gbs = nq * 8 / (pms * 1e-3) / 1e9
    peak = peaks.get("hbm_gbs", 6650.0)
    pred = {"row": "A12 predict (type-2)", "queries": nq, "ms": pms, "queries_per_s": nq / (pms * 1e-3),
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak, "bytes_per_query": 8}}
    del Xq, out
    return {"solve": solve, "predict": pred}


def other_configs(args, dev):
    """Compact records of the other BASELINE configurations (C1, C3, C4, C5) at their full n, so the
    driver's default run sees every configuration: the same fit step (type-1 passes + solve; C1 as
    one CUDA graph), CUDA events over the timed steps, the spreading kernels' share and their
    atomic-unit roofline (d >= 2), the fit status word."""
    import torch

    from datagen.device import gen_dataset
    from paper_2509_02649_b200 import fk
    from paper_2509_02649_b200.fit import FitGraph, _moment_buffers, additive_buffers, fit_additive_distributed, fit_distributed

    out = {}
    for name in ("c1", "c3", "c4", "c5"):
        cfg = dict(CONFIGS[name])
        d, m, n, eps = cfg["d"], cfg["m"], cfg["n"], 1e-6
        additive = cfg["kind"] == "additive"
        pik = pi_kwargs(cfg)
        st = torch.zeros(1, dtype=torch.int32, device=dev)
        Y = torch.empty(n, dtype=torch.float32, device=dev)
        if additive:
            Xs = torch.empty((d, n), dtype=torch.float32, device=dev)
            gen_dataset(Xs, Y, n, d, xkind=cfg["xkind"], ykind=cfg["ykind"], seed=0, stride_n=1, stride_d=n)
            X = Xs.t()
            bufs = additive_buffers(d, m, dev)
            theta = torch.empty(d * (2 * m + 1), dtype=torch.complex128, device=dev)
        else:
            X = torch.empty((n,) if d == 1 else (n, d), dtype=torch.float32, device=dev)
            gen_dataset(X, Y, n, d, xkind=cfg["xkind"], ykind=cfg["ykind"], seed=0)
            bufs = _moment_buffers(d, m, dev)
            theta = torch.empty((2 * m + 1) ** d, dtype=torch.complex128, device=dev)
        graph = FitGraph(X, Y, 1.0, m, cfg["lam"], cfg["kind"], cfg["s"], eps, **pik) if name == "c1" else None

        def step():
            if graph is not None:
                graph.replay()
            elif additive:
                fit_additive_distributed(X, Y, n, 1.0, m, cfg["lam"], eps, buffers=bufs, theta_out=theta, status=st)
            else:
                fit_distributed(X, Y, n, 1.0, m, cfg["lam"], cfg["kind"], cfg["s"], eps, buffers=bufs, theta_out=theta, status=st, **pik)

        steps = 20 if name == "c1" else (3 if name == "c5" else 5)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        fk.profile_read()
        fk.profile_enable(True)
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(steps):
            step()
        e1.record(s)
        torch.cuda.synchronize()
        fk.profile_enable(False)
        sp_ms, _, _ = fk.profile_read()
        ms = e0.elapsed_time(e1) / steps
        if graph is not None:
            graph.check()
        rec = {"workload": cfg["desc"], "value": n / (ms * 1e-3), "unit": "samples/s", "ms_per_step": ms, "steps": steps,
               "fit_status_ok": int(st.item()) == 0, "cuda_graph": graph is not None}
        if d >= 2:
            w = spread2d_width(eps)
            atoms = n * (d * (d - 1) // 2 * cross_width(eps, m) ** 2 + d * 8) if additive else n * 2 * w * w
            sp = sp_ms / steps
            rec["roofline"] = {"bound": "alu", "unit": "Gatomic/s", "achieved": atoms / (sp * 1e-3) / 1e9,
                               "peak": ATOMS_CFREE_PEAK / 1e9, "frac": atoms / (sp * 1e-3) / ATOMS_CFREE_PEAK,
                               "frac_of_random_atoms": atoms / (sp * 1e-3) / ATOMS_RANDOM_PEAK,
                               "spread_share_of_step": sp / ms}
        out[name] = rec
        del X, Y, bufs, theta, graph
        if additive:
            del Xs
        torch.cuda.empty_cache()
    return out


def run_e2e_additive(args, cfg, dev, eps):
    """Additive model end to end: pinned host X (SoA columns) and Y -> chunked H2D on two copy
    streams overlapped with the per-feature passes and the cross moments -> block solve -> theta D2H."""
    import torch

    from datagen.device import gen_dataset
    from paper_2509_02649_b200 import fk
    from paper_2509_02649_b200.fit import HostStreamerAdditive, additive_buffers

    d, m = cfg["d"], cfg["m"]
    n = int(min(args.e2e_n / 4, cfg["n"]))  # 44 B per sample: a quarter of the d = 1 sample count
    chunk = 1 << 24
    Xh = torch.empty((d, n), dtype=torch.float32, pin_memory=True)
    Yh = torch.empty(n, dtype=torch.float32, pin_memory=True)
    tx = torch.empty((d, chunk), dtype=torch.float32, device=dev)
    ty = torch.empty(chunk, dtype=torch.float32, device=dev)
    for lo in range(0, n, chunk):
        c = min(chunk, n - lo)
        gen_dataset(tx[:, :c].t(), ty[:c], c, d, i0=lo, xkind=cfg["xkind"], ykind=cfg["ykind"], seed=0, stride_n=1, stride_d=chunk)
        Xh[:, lo:lo + c].copy_(tx[:, :c])
        Yh[lo:lo + c].copy_(ty[:c])
    del tx, ty
    st = HostStreamerAdditive(chunk, d, dev)
    _, mus, rs, G = additive_buffers(d, m, dev)
    D = d * (2 * m + 1)
    theta_h = torch.empty(D, dtype=torch.complex128, pin_memory=True)

    def step():
        st.moments(Xh, Yh, 1.0, m, eps, mus, rs, G)
        th, _ = fk.fk_solve(mus, rs, n, d, m, 1.0, cfg["lam"], "additive", report=False, cross=G)
        theta_h.copy_(th, non_blocking=True)

    step()
    torch.cuda.synchronize()
    steps = max(2, min(3, args.steps))
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        step()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return {"value": n / (ms * 1e-3), "unit": "samples/s", "h2d_bytes_per_step": n * (d + 1) * 4, "d2h_bytes_per_step": D * 16,
            "n": n, "ms_per_step": ms,
            "path": "fit.HostStreamerAdditive + fk_solve: pinned host SoA X and Y -> chunked H2D on two copy streams overlapped with "
                    "the per-feature passes and the cross moments; theta D2H"}


def run_e2e(args, cfg, dev, eps):
    """Same metric through the public API from pinned HOST buffers: chunked H2D (copy stream,
    overlapped with the spreading of the previous chunk) + fk_solve + theta D2H, every step."""
    import torch

    from datagen.device import gen_dataset
    from paper_2509_02649_b200 import fk
    from paper_2509_02649_b200.fit import _moment_buffers

    d, m = cfg["d"], cfg["m"]
    n = int(min(args.e2e_n, cfg["n"]))
    chunk = 1 << 26
    Xh = torch.empty((n,) if d == 1 else (n, d), dtype=torch.float32, pin_memory=True)
    Yh = torch.empty(n, dtype=torch.float32, pin_memory=True)
    tmpx = torch.empty((chunk,) if d == 1 else (chunk, d), dtype=torch.float32, device=dev)
    tmpy = torch.empty(chunk, dtype=torch.float32, device=dev)
    for lo in range(0, n, chunk):
        c = min(chunk, n - lo)
        gen_dataset(tmpx, tmpy, c, d, i0=lo, xkind=cfg["xkind"], ykind=cfg["ykind"], seed=0)
        Xh[lo:lo + c].copy_(tmpx[:c])
        Yh[lo:lo + c].copy_(tmpy[:c])
    del tmpx, tmpy
    _, mu, r = _moment_buffers(d, m, dev)
    D = (2 * m + 1) ** d
    theta_h = torch.empty(D, dtype=torch.complex128, pin_memory=True)
    pik = pi_kwargs(cfg)

    def step():  # the library's native host-streaming entry point (chunked H2D overlapped with the spread)
        fk.fk_rhs_type1_host(Xh, Yh, 1.0, m, eps, r_out=r, mu_out=mu, chunk=chunk, check=False, device=dev)
        th, _ = fk.fk_solve(mu.reshape(-1), r.reshape(-1), n, d, m, 1.0, cfg["lam"], cfg["kind"], cfg["s"], report=False, **pik)
        theta_h.copy_(th, non_blocking=True)

    step()
    torch.cuda.synchronize()
    steps = max(2, min(5, args.steps))
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        step()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return {"value": n / (ms * 1e-3), "unit": "samples/s", "h2d_bytes_per_step": n * (d + 1) * 4, "d2h_bytes_per_step": D * 16,
            "n": n, "ms_per_step": ms,
            "path": "fk_rhs_type1_host (C ABI: pinned host X, Y -> chunked H2D on the library's copy stream overlapped with the "
                    "spreading of the previous chunk) + fk_solve; theta D2H; bound by the PCIe link (~55 GB/s); n = 2^30 bounded sample "
                    "(the rate is PCIe-bound and independent of n)"}


if __name__ == "__main__":
    sys.exit(main())
