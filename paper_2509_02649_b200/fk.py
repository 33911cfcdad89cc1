"""Thin Python binding of libfk (include/fk.h): argument marshalling only.

Every step of the fit path runs in libfk's CUDA kernels; this module turns torch CUDA tensors
into the C ABI's plain pointers / sizes / strides, allocates outputs and the workspace with
torch (device memory plumbing), calls the C entry point on the current torch stream and turns a
non-zero status into an exception.  The names are the C names.  There is no fallback: importing
this module on a box without the built library raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfk.so")

FK_OK, FK_E_ARG, FK_E_RANGE, FK_E_EPS, FK_E_CUDA, FK_E_WORKSPACE, FK_E_SOLVE, FK_E_UNSUPPORTED = range(8)
FK_F32, FK_F64 = 0, 1
FK_ACCUMULATE = 1
FK_DSTATUS_RANGE, FK_DSTATUS_NOT_SPD, FK_DSTATUS_WATCHDOG = 2, 0x10, 0x20
FK_SOBOLEV, FK_LOWBIAS, FK_PIK_BOX, FK_ADDITIVE, FK_PIK_COLLOC = 0, 1, 2, 3, 4
KINDS = {"sobolev": FK_SOBOLEV, "lowbias": FK_LOWBIAS, "pik_box": FK_PIK_BOX, "additive": FK_ADDITIVE, "pik_colloc": FK_PIK_COLLOC}
(FK_ENTRY_MOMENTS, FK_ENTRY_RHS, FK_ENTRY_CROSS, FK_ENTRY_SOLVE, FK_ENTRY_PREDICT, FK_ENTRY_SOLVE_PATH,
 FK_ENTRY_PATH_VALIDATE, FK_ENTRY_RHS_HOST) = range(8)
_STATUS = {1: "FK_E_ARG", 2: "FK_E_RANGE", 3: "FK_E_EPS", 4: "FK_E_CUDA", 5: "FK_E_WORKSPACE", 6: "FK_E_SOLVE", 7: "FK_E_UNSUPPORTED"}


class FkError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class fk_points(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("d", ctypes.c_int32), ("n", ctypes.c_int64),
                ("stride_n", ctypes.c_int64), ("stride_d", ctypes.c_int64)]


class fk_problem(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("m", ctypes.c_int32), ("kind", ctypes.c_int32), ("n_terms", ctypes.c_int32),
                ("n_total", ctypes.c_double), ("L", ctypes.c_double), ("s", ctypes.c_double), ("lam", ctypes.c_double),
                ("mu_pde", ctypes.c_double), ("alpha", ctypes.POINTER(ctypes.c_int32)), ("a_alpha", ctypes.POINTER(ctypes.c_double)),
                ("box", ctypes.POINTER(ctypes.c_double)), ("mu_moments", ctypes.c_void_p), ("rhs", ctypes.c_void_p),
                ("cross", ctypes.c_void_p), ("colloc_moments", ctypes.c_void_p), ("n_colloc", ctypes.c_double),
                ("d_status", ctypes.c_void_p)]


class fk_solve_report(ctypes.Structure):
    _fields_ = [("backward_err", ctypes.c_double), ("ms", ctypes.c_double), ("info", ctypes.c_int32), ("n_unknowns", ctypes.c_int32),
                ("iters", ctypes.c_int32), ("reserved", ctypes.c_int32), ("rcond_est", ctypes.c_double)]


_lib = None


def lib():
    """Load libfk.so (raises if it was not built: there is no CPU path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libfk.so not found at {LIB_PATH}; build it with `python -m paper_2509_02649_b200.build`")
        L = ctypes.CDLL(os.environ.get("FK_LIB_OVERRIDE", LIB_PATH))  # override: A/B measurements only
        vp, dp, ip, sz = ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_size_t
        L.fk_moments_type1.argtypes = [fk_points, dp, ip, dp, vp, ip, vp, sz, vp, vp]
        L.fk_rhs_type1.argtypes = [fk_points, vp, dp, ip, dp, vp, vp, ip, vp, sz, vp, vp]
        L.fk_rhs_type1_host.argtypes = [fk_points, vp, dp, ip, dp, vp, vp, ip, ctypes.c_int64, vp, sz, vp, vp]
        L.fk_additive_cross_moments.argtypes = [fk_points, dp, ip, dp, vp, ip, vp, sz, vp, vp]
        L.fk_solve.argtypes = [ctypes.POINTER(fk_problem), vp, ctypes.POINTER(fk_solve_report), vp, sz, vp]
        L.fk_solve_path.argtypes = [ctypes.POINTER(fk_problem), vp, ip, vp, vp, vp, sz, vp]
        L.fk_path_validate.argtypes = [ctypes.POINTER(fk_problem), vp, ip, dp, vp, vp, sz, vp]
        L.fk_predict_type2.argtypes = [vp, ip, ip, dp, ip, fk_points, dp, vp, vp, sz, vp, vp]
        L.fk_workspace_bytes.argtypes = [ip, ip, ip, dp, ip, ctypes.c_int64, ip]
        L.fk_workspace_bytes.restype = ctypes.c_size_t
        L.fk_last_error.restype = ctypes.c_char_p
        L.fk_version.restype = ctypes.c_char_p
        for f in ("fk_moments_type1", "fk_rhs_type1", "fk_rhs_type1_host", "fk_additive_cross_moments", "fk_solve", "fk_solve_path", "fk_path_validate",
                  "fk_predict_type2"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(status: int):
    if status != FK_OK:
        raise FkError(status, lib().fk_last_error().decode())


def _stream(stream: Optional[torch.cuda.Stream]) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class _On:
    """Stream plumbing of one call on `stream` (default: torch's current stream).  Outputs, the
    status word and the workspace are allocated / zeroed on the current stream, so a different
    `stream` first waits for the current one; afterwards the tensors the library wrote are marked
    as used on `stream` (record_stream) so the caching allocator does not recycle them early."""

    def __init__(self, stream, device):
        self.cur = torch.cuda.current_stream(device)
        self.s = stream if stream is not None else self.cur
        self.other = self.s != self.cur
        if self.other:
            self.s.wait_stream(self.cur)

    @property
    def handle(self):
        return ctypes.c_void_p(self.s.cuda_stream)

    def done(self, *tensors):
        if self.other:
            for t in tensors:
                if t is not None:
                    t.record_stream(self.s)

    def sync(self):
        self.s.synchronize()


def _points(X: torch.Tensor) -> fk_points:
    if not X.is_cuda:
        raise ValueError("points must be a CUDA tensor")
    if X.dtype not in (torch.float32, torch.float64):
        raise ValueError("points must be float32 or float64")
    if X.dim() == 1:
        n, d, sn, sd = X.shape[0], 1, X.stride(0), 1
    elif X.dim() == 2:
        n, d = X.shape
        sn, sd = X.stride()
    else:
        raise ValueError("points must be (n,) or (n, d)")
    return fk_points(X.data_ptr(), FK_F32 if X.dtype == torch.float32 else FK_F64, d, n, sn, sd)


_ws_cache = {}


def _workspace(nbytes: int, device, stream=None) -> torch.Tensor:
    """Scratch for a call, cached per (device, stream): calls on different streams may run
    concurrently and must not share scratch; calls on one stream are ordered, so they can.  A grown
    buffer replaces the old one, which is freed only after the work queued on that stream so far
    (record_stream when the stream is not the allocating one)."""
    dev = device.index if device.index is not None else torch.cuda.current_device()
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    key = (dev, s.cuda_stream)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        if buf is not None and s != torch.cuda.current_stream(dev):
            buf.record_stream(s)
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
        _ws_cache[key] = buf
    return buf


def fk_workspace_bytes(entry: int, d: int, m: int, eps: float, dtype: int = FK_F32, n: int = 0, kind: int = 0) -> int:
    """Workspace bytes for a call; 0 when the arguments are invalid (the call itself then returns
    the precise status, so callers pass a minimal buffer and let the entry point report it)."""
    return int(lib().fk_workspace_bytes(entry, d, m, eps, dtype, n, kind))


def _dstatus(d_status, device):
    if d_status is None:
        d_status = torch.zeros(1, dtype=torch.int32, device=device)
    return d_status


def raise_on_status(d_status: torch.Tensor):
    v = int(d_status.item())
    if v & FK_E_RANGE:
        raise FkError(FK_E_RANGE, "a coordinate outside [-L, L] (or NaN) was skipped")


def fk_moments_type1(X: torch.Tensor, L: float, m: int, eps: float = 1e-6, mu_out: Optional[torch.Tensor] = None,
                     accumulate: bool = False, d_status: Optional[torch.Tensor] = None, stream=None, check: bool = True) -> torch.Tensor:
    """mu_q = sum_j exp(-i pi <q, X_j>/2L), |q|_inf <= 2m (complex128, shape (4m+1,)*d)."""
    P = _points(X)
    if mu_out is None:
        mu_out = torch.zeros((4 * m + 1,) * P.d, dtype=torch.complex128, device=X.device)
    nb = fk_workspace_bytes(FK_ENTRY_MOMENTS, P.d, m, eps, P.dtype, P.n)
    ds = _dstatus(d_status, X.device)
    on = _On(stream, X.device)
    ws = _workspace(nb, X.device, on.s)
    _check(lib().fk_moments_type1(P, L, m, eps, mu_out.data_ptr(), FK_ACCUMULATE if accumulate else 0, ws.data_ptr(), ws.numel(),
                                  ds.data_ptr(), on.handle))
    on.done(mu_out, ds, X)
    if check and d_status is None:
        on.sync()
        raise_on_status(ds)
    return mu_out


def fk_rhs_type1(X: torch.Tensor, Y: torch.Tensor, L: float, m: int, eps: float = 1e-6, r_out: Optional[torch.Tensor] = None,
                 mu_out: Optional[torch.Tensor] = None, with_moments: bool = True, accumulate: bool = False,
                 d_status: Optional[torch.Tensor] = None, stream=None, check: bool = True):
    """(r, mu): r_k = sum_j Y_j exp(-i pi <k, X_j>/2L), |k| <= m, and (same pass) the moments."""
    P = _points(X)
    if Y.dtype != X.dtype or not Y.is_cuda or Y.dim() != 1 or Y.shape[0] != P.n or (P.n > 1 and Y.stride(0) != 1):
        raise ValueError("Y must be a contiguous CUDA vector of X's dtype and length")
    if r_out is None:
        r_out = torch.zeros((2 * m + 1,) * P.d, dtype=torch.complex128, device=X.device)
    if with_moments and mu_out is None:
        mu_out = torch.zeros((4 * m + 1,) * P.d, dtype=torch.complex128, device=X.device)
    entry = FK_ENTRY_RHS
    nb = fk_workspace_bytes(entry, P.d, m, eps, P.dtype, P.n)
    ds = _dstatus(d_status, X.device)
    on = _On(stream, X.device)
    ws = _workspace(nb, X.device, on.s)
    _check(lib().fk_rhs_type1(P, Y.data_ptr(), L, m, eps, r_out.data_ptr(), mu_out.data_ptr() if mu_out is not None else None,
                              FK_ACCUMULATE if accumulate else 0, ws.data_ptr(), ws.numel(), ds.data_ptr(), on.handle))
    on.done(r_out, mu_out, ds, X, Y)
    if check and d_status is None:
        on.sync()
        raise_on_status(ds)
    return r_out, mu_out


def fk_rhs_type1_host(Xh: torch.Tensor, Yh: torch.Tensor, L: float, m: int, eps: float = 1e-6, r_out: Optional[torch.Tensor] = None,
                      mu_out: Optional[torch.Tensor] = None, with_moments: bool = True, accumulate: bool = False, chunk: int = 0,
                      d_status: Optional[torch.Tensor] = None, stream=None, check: bool = True, device=None):
    """fk_rhs_type1 from HOST tensors (pinned for overlap): the library streams chunks to the device
    through two staging buffers on its own copy stream, overlapped with the spreading."""
    if Xh.is_cuda or Yh.is_cuda:
        raise ValueError("fk_rhs_type1_host takes host tensors")
    if Xh.dtype not in (torch.float32, torch.float64) or Yh.dtype != Xh.dtype:
        raise ValueError("X, Y must share a float dtype")
    Xh, Yh = Xh.contiguous(), Yh.contiguous()
    d = 1 if Xh.dim() == 1 else Xh.shape[1]
    n = Xh.shape[0]
    if Yh.dim() != 1 or Yh.shape[0] != n:
        raise ValueError("Y must be a vector of X's length")
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    P = fk_points(Xh.data_ptr(), FK_F32 if Xh.dtype == torch.float32 else FK_F64, d, n, d, 1)
    if r_out is None:
        r_out = torch.zeros((2 * m + 1,) * d, dtype=torch.complex128, device=dev)
    if with_moments and mu_out is None:
        mu_out = torch.zeros((4 * m + 1,) * d, dtype=torch.complex128, device=dev)
    nb = fk_workspace_bytes(FK_ENTRY_RHS_HOST, d, m, eps, P.dtype, chunk)
    ds = _dstatus(d_status, dev)
    on = _On(stream, dev)
    ws = _workspace(nb, dev, on.s)
    _check(lib().fk_rhs_type1_host(P, Yh.data_ptr(), L, m, eps, r_out.data_ptr(), mu_out.data_ptr() if mu_out is not None else None,
                                   FK_ACCUMULATE if accumulate else 0, int(chunk), ws.data_ptr(), ws.numel(), ds.data_ptr(), on.handle))
    on.done(r_out, mu_out, ds)
    if check and d_status is None:
        on.sync()
        raise_on_status(ds)
    return r_out, mu_out


def fk_additive_cross_moments(X: torch.Tensor, L: float, m: int, eps: float = 1e-6, G_out: Optional[torch.Tensor] = None,
                              accumulate: bool = False, d_status: Optional[torch.Tensor] = None, stream=None,
                              check: bool = True) -> torch.Tensor:
    """G[p, a, b] = sum_j exp(-i pi (a X_{j,l1} - b X_{j,l2})/2L) for pairs l1 < l2."""
    P = _points(X)
    npairs = P.d * (P.d - 1) // 2
    if G_out is None:
        G_out = torch.zeros((npairs, 2 * m + 1, 2 * m + 1), dtype=torch.complex128, device=X.device)
    nb = fk_workspace_bytes(FK_ENTRY_CROSS, P.d, m, eps, P.dtype, P.n)
    ds = _dstatus(d_status, X.device)
    on = _On(stream, X.device)
    ws = _workspace(nb, X.device, on.s)
    _check(lib().fk_additive_cross_moments(P, L, m, eps, G_out.data_ptr(), FK_ACCUMULATE if accumulate else 0, ws.data_ptr(),
                                           ws.numel(), ds.data_ptr(), on.handle))
    on.done(G_out, ds, X)
    if check and d_status is None:
        on.sync()
        raise_on_status(ds)
    return G_out


def fk_solve(mu: torch.Tensor, r: torch.Tensor, n_total: float, d: int, m: int, L: float, lam: float, kind: str = "sobolev",
             s: float = 1.0, mu_pde: float = 0.0, alpha: Optional[Sequence] = None, a_alpha: Optional[Sequence[float]] = None,
             box: Optional[Sequence] = None, cross: Optional[torch.Tensor] = None, theta_out: Optional[torch.Tensor] = None,
             report: bool = True, stream=None, colloc_moments: Optional[torch.Tensor] = None, n_colloc: float = 0.0,
             d_status: Optional[torch.Tensor] = None):
    """theta = A^{-1} r/n (dense fp64 Cholesky, or CG for large Sobolev systems).  Returns (theta
    complex128, report dict or None).  d_status (device int32, optional): FK_DSTATUS_NOT_SPD /
    FK_DSTATUS_WATCHDOG are ORed into it by the device, also when report=False (no sync)."""
    k = KINDS[kind] if isinstance(kind, str) else int(kind)
    D = d * (2 * m + 1) if k == FK_ADDITIVE else (2 * m + 1) ** d
    if theta_out is None:
        theta_out = torch.empty(D, dtype=torch.complex128, device=mu.device)
    prob, keep = _problem(mu, r, n_total, d, m, L, lam, k, s, mu_pde, alpha, a_alpha, box, cross, colloc_moments, n_colloc)
    if d_status is not None:
        prob.d_status = d_status.data_ptr()
    nb = fk_workspace_bytes(FK_ENTRY_SOLVE, d, m, 1e-6, FK_F64, 0, k)
    on = _On(stream, mu.device)
    ws = _workspace(nb, mu.device, on.s)
    rep = fk_solve_report()
    _check(lib().fk_solve(ctypes.byref(prob), theta_out.data_ptr(), ctypes.byref(rep) if report else None, ws.data_ptr(), ws.numel(),
                          on.handle))
    on.done(theta_out, d_status, *[t for t in keep if isinstance(t, torch.Tensor)])
    del keep
    out = None
    if report:
        out = {"backward_err": rep.backward_err, "ms": rep.ms, "info": rep.info, "n_unknowns": rep.n_unknowns, "iters": rep.iters,
               "rcond_est": rep.rcond_est}
    return theta_out, out


def solve_status(d_status: torch.Tensor) -> None:
    """Raise if the device status word of fk_solve calls reports a failed factorisation (syncs)."""
    v = int(d_status.item())
    if v & FK_DSTATUS_WATCHDOG:
        raise FkError(FK_E_SOLVE, "a dataflow wait of the factorisation hit its watchdog: theta is not valid")
    if v & FK_DSTATUS_NOT_SPD:
        raise FkError(FK_E_SOLVE, "the system is not numerically positive definite")


def fk_solve_path(mu: torch.Tensor, r: torch.Tensor, n_total: float, d: int, m: int, L: float, lambdas: Sequence[float],
                  kind: str = "sobolev", s: float = 1.0, mu_pde: float = 0.0, alpha: Optional[Sequence] = None,
                  a_alpha: Optional[Sequence[float]] = None, box: Optional[Sequence] = None, cross: Optional[torch.Tensor] = None,
                  theta_out: Optional[torch.Tensor] = None, check: bool = True, stream=None,
                  colloc_moments: Optional[torch.Tensor] = None, n_colloc: float = 0.0) -> torch.Tensor:
    """theta(lambda_l) for every lambda in `lambdas` from ONE eigendecomposition (regularisation path,
    P:542-548).  Returns a (nlam, D) complex128 tensor."""
    k = KINDS[kind] if isinstance(kind, str) else int(kind)
    D = d * (2 * m + 1) if k == FK_ADDITIVE else (2 * m + 1) ** d
    lams = (ctypes.c_double * len(lambdas))(*[float(v) for v in lambdas])
    if theta_out is None:
        theta_out = torch.empty(len(lambdas), D, dtype=torch.complex128, device=mu.device)
    prob, keep = _problem(mu, r, n_total, d, m, L, 0.0, k, s, mu_pde, alpha, a_alpha, box, cross, colloc_moments, n_colloc)
    nb = fk_workspace_bytes(FK_ENTRY_SOLVE_PATH, d, m, 1e-6, FK_F64, len(lambdas), k)
    on = _On(stream, mu.device)
    ws = _workspace(nb, mu.device, on.s)
    info = ctypes.c_int(0)
    _check(lib().fk_solve_path(ctypes.byref(prob), lams, len(lambdas), theta_out.data_ptr(), ctypes.byref(info) if check else None,
                               ws.data_ptr(), ws.numel(), on.handle))
    on.done(theta_out, *[t for t in keep if isinstance(t, torch.Tensor)])
    del keep
    return theta_out


def fk_path_validate(theta: torch.Tensor, mu_v: torch.Tensor, r_v: torch.Tensor, n_v: float, d: int, m: int, L: float,
                     kind: str = "sobolev", sum_y2: float = 0.0, cross_v: Optional[torch.Tensor] = None,
                     risk_out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Held-out mean squared error of each row of theta (nlam x D) on a validation set given by its
    type-1 moments mu_v / rhs r_v (and cross moments for the additive model), n_v samples and
    sum_y2 = sum Y_v^2 (P:542-548 grid search; R11).  Returns nlam float64 (device)."""
    k = KINDS[kind] if isinstance(kind, str) else int(kind)
    if k in (FK_PIK_BOX, FK_PIK_COLLOC):  # the risk needs only the data part of the system
        k = FK_SOBOLEV
    theta = theta.contiguous()
    nlam = theta.shape[0] if theta.dim() == 2 else 1
    if risk_out is None:
        risk_out = torch.empty(nlam, dtype=torch.float64, device=theta.device)
    prob, keep = _problem(mu_v, r_v, n_v, d, m, L, 0.0, k, 1.0, 0.0, None, None, None, cross_v, None, 0.0)
    nb = fk_workspace_bytes(FK_ENTRY_PATH_VALIDATE, d, m, 1e-6, FK_F64, nlam, k)
    on = _On(stream, theta.device)
    ws = _workspace(nb, theta.device, on.s)
    _check(lib().fk_path_validate(ctypes.byref(prob), theta.data_ptr(), nlam, float(sum_y2), risk_out.data_ptr(), ws.data_ptr(),
                                  ws.numel(), on.handle))
    on.done(risk_out, theta, *[t for t in keep if isinstance(t, torch.Tensor)])
    del keep
    return risk_out


def _problem(mu, r, n_total, d, m, L, lam, k, s, mu_pde, alpha, a_alpha, box, cross, colloc_moments, n_colloc):
    prob = fk_problem()
    prob.d, prob.m, prob.kind = d, m, k
    prob.n_total, prob.L, prob.s, prob.lam, prob.mu_pde = float(n_total), float(L), float(s), float(lam), float(mu_pde)
    keep = []
    if k in (FK_PIK_BOX, FK_PIK_COLLOC):
        al = (ctypes.c_int32 * (len(alpha) * d))(*[int(v) for row in alpha for v in row])
        aa = (ctypes.c_double * len(a_alpha))(*[float(v) for v in a_alpha])
        keep += [al, aa]
        prob.n_terms = len(a_alpha)
        prob.alpha = ctypes.cast(al, ctypes.POINTER(ctypes.c_int32))
        prob.a_alpha = ctypes.cast(aa, ctypes.POINTER(ctypes.c_double))
        if box is not None:
            bx = (ctypes.c_double * (2 * d))(*[float(v) for row in box for v in row])
            keep.append(bx)
            prob.box = ctypes.cast(bx, ctypes.POINTER(ctypes.c_double))
    if k == FK_PIK_COLLOC:
        colloc_moments = colloc_moments.contiguous()
        keep.append(colloc_moments)
        prob.colloc_moments = colloc_moments.data_ptr()
        prob.n_colloc = float(n_colloc)
    mu = mu.contiguous()
    r = r.contiguous()
    prob.mu_moments = mu.data_ptr()
    prob.rhs = r.data_ptr()
    if cross is not None:
        cross = cross.contiguous()
        keep.append(cross)
        prob.cross = cross.data_ptr()
    keep += [mu, r]
    return prob, keep


def fk_predict_type2(theta: torch.Tensor, d: int, m: int, L: float, Xq: torch.Tensor, eps: float = 1e-6, additive: bool = False,
                     out: Optional[torch.Tensor] = None, d_status: Optional[torch.Tensor] = None, stream=None,
                     check: bool = True) -> torch.Tensor:
    """f(x) = Re sum_k theta_k exp(+i pi <k, x>/2L) at the rows of Xq (additive: sum over features)."""
    P = _points(Xq)
    if out is None:
        out = torch.empty(P.n, dtype=Xq.dtype, device=Xq.device)
    nb = fk_workspace_bytes(FK_ENTRY_PREDICT, d, m, eps, P.dtype, P.n, 1 if additive else 0)
    ds = _dstatus(d_status, Xq.device)
    theta = theta.contiguous()
    on = _On(stream, Xq.device)
    ws = _workspace(nb, Xq.device, on.s)
    _check(lib().fk_predict_type2(theta.data_ptr(), d, m, L, 1 if additive else 0, P, eps, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                  ds.data_ptr(), on.handle))
    on.done(out, ds, theta, Xq)
    if check and d_status is None:
        on.sync()
        raise_on_status(ds)
    return out


def version() -> str:
    return lib().fk_version().decode()


def profile_enable(on: bool = True):
    """Bracket every spreading-kernel launch with CUDA events on its stream (diagnostics)."""
    lib().fk_profile_enable(1 if on else 0)


def profile_read():
    """(spread_ms_total, spread_launches, kernel_launches) since the last read; resets them."""
    ms = ctypes.c_double(0.0)
    nl = ctypes.c_int64(0)
    nk = ctypes.c_int64(0)
    lib().fk_profile_read(ctypes.byref(ms), ctypes.byref(nl), ctypes.byref(nk))
    return ms.value, nl.value, nk.value


fk_profile_enable = profile_enable
fk_profile_read = profile_read


def fk_version() -> str:
    return version()


def fk_last_error() -> str:
    return lib().fk_last_error().decode()
