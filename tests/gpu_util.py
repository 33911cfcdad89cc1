"""Helpers shared by the GPU parity tests (no method arithmetic here)."""
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b) -> float:
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def fk():
    from paper_2509_02649_b200 import build, fk as _fk

    build.build()
    return _fk


def dev(a, dtype=None):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def host(t):
    return t.detach().cpu().numpy()


from datagen.device import gen_dataset, gen_equispaced  # noqa: E402,F401


# ---------------------------------------------------------------------------------------------
# type-1 parity gates (verdict r01 #1): the relative l2 gate of north_star AND a per-element bound
#   max_q |out_q - ref_q| <= 10 eps * scale,  scale = n (moments, cross moments: = |ref_0|) or
#   sum_j |Y_j| (rhs),
# so an error confined to a few modes (e.g. the high modes |q| ~ 2m where the window deconvolution
# is largest) cannot hide under mu_0 = n in the l2 norm.  eps = the accuracy the call requested.
# ---------------------------------------------------------------------------------------------
def _eps_of(tol):
    return tol / 10.0 if tol >= 1e-7 else 1e-10


def elem_err(out, ref, scale) -> float:
    out = np.asarray(out).ravel()
    ref = np.asarray(ref).ravel()
    if out.size == 0:
        return 0.0
    return float(np.max(np.abs(out - ref)) / max(float(scale), 1e-300))


def check_type1(out, ref, tol, scale, eps=None, what=""):
    eps = _eps_of(tol) if eps is None else eps
    e2, em = rel(out, ref), elem_err(out, ref, scale)
    assert e2 <= tol and em <= 10 * eps, f"{what}: rel l2 {e2:.3e} (gate {tol:.0e}), max elem/scale {em:.3e} (gate {10 * eps:.0e})"
    return e2, em


def check_mu(out, ref, tol, eps=None, what="moments"):
    """Moments / cross moments: scale = the exact zero mode (= number of summed samples)."""
    ref = np.asarray(ref)
    return check_type1(out, ref, tol, abs(ref.ravel()[ref.size // 2]), eps, what)


def check_r(out, ref, Y, tol, eps=None, what="rhs"):
    """Right-hand side: scale = sum_j |Y_j| over the summed samples."""
    return check_type1(out, ref, tol, float(np.sum(np.abs(np.asarray(Y, dtype=np.float64)))), eps, what)
