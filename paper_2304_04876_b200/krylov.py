"""Right-preconditioned restarted GMRES on the GPU (mirrors schwarzdd.krylov,
krylov.py:1-370).

Both variants of the reference run in libgdsw's native loop (gdsw_gmres):
vectors, the operator SpMV, the preconditioner and the fused reductions on
the device; the Hessenberg/Givens bookkeeping on the host from the one
reduced block copied back per iteration.

* single_reduce (krylov.py:260-361): ONE fused block reduction
  [V[:j]; v]^T [v, z] per iteration, delayed normalization, Pythagorean
  delta, delayed reorthogonalization, speculative M/A on the unnormalized
  candidate -- the reference's algebra step for step.
* classic (krylov.py:179-257): MGS or CGS2 Arnoldi.

Convergence is confirmed on the true residual, counters and history follow
the reference's accounting (SolveReport).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .sparse_core import CsrMatrix

VARIANTS = ("classic", "single_reduce")
ORTHOGONALIZATIONS = ("mgs", "cgs2")
BREAKDOWN_REL = 1e-14


@dataclass(frozen=True)
class KrylovConfig:
    restart: int = 30
    rel_tol: float = 1e-7
    max_iters: int = 500
    variant: str = "classic"
    orthogonalization: str = "mgs"

    def __post_init__(self):
        if self.restart < 1:
            raise ValueError("restart must be at least 1")
        if not 0.0 < self.rel_tol < 1.0:
            raise ValueError("rel_tol must lie strictly between 0 and 1")
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}")
        if self.orthogonalization not in ORTHOGONALIZATIONS:
            raise ValueError(f"unknown orthogonalization {self.orthogonalization!r}")


@dataclass
class Timings:
    symbolic: float = 0.0
    numeric: float = 0.0
    solve: float = 0.0


@dataclass
class SolveReport:
    iterations: int
    converged: bool
    residual_history: np.ndarray
    timings: Timings
    reduction_count: int
    iteration_reductions: int
    residual_reductions: int
    restarts: int
    true_residuals: list


def _host_operator(obj):
    """The reference's fallbacks (krylov.py:93-98): `.apply` objects, then
    callables; they run on the host, called with float64 numpy vectors."""
    if hasattr(obj, "apply") and callable(obj.apply):
        return obj.apply
    if callable(obj):
        return obj
    raise TypeError("operator must be a CsrMatrix, expose .apply, or be callable")


_IDENTITY: dict = {}


def _identity(n: int) -> CsrMatrix:
    eye = _IDENTITY.get(n)
    if eye is None:
        _IDENTITY.clear()
        idx = np.arange(n, dtype=np.int64)
        eye = _IDENTITY[n] = CsrMatrix(n, n, np.arange(n + 1, dtype=np.int64), idx,
                                       np.ones(n, dtype=np.float64))
    return eye


def _device_operators(a, m, n: int):
    """Resolve (A, M) with the reference's duck typing (krylov.py:88-100):
    CsrMatrix / DeviceCsr / TwoLevelPreconditioner run on the GPU; other
    `.apply` objects and callables become host operators.
    Returns (a_dev, a_fn, m_pre, m_csr, m_fn)."""
    from . import device
    from .schwarz import TwoLevelPreconditioner
    a_fn = m_fn = a_dev = None
    if a is None:
        # the reference's _operator(None) is the identity (krylov.py:89-90)
        a_dev = device.device_csr(_identity(n))
    elif isinstance(a, CsrMatrix):
        if a.nrows != n or a.ncols != n:
            raise ValueError("operator dimensions do not match the vector")
        a_dev = device.device_csr(a)
    elif isinstance(a, device.DeviceCsr):
        if a.nrows != n or a.ncols != n:
            raise ValueError("operator dimensions do not match the vector")
        a_dev = a
    else:
        a_fn = _host_operator(a)
    m_pre = m_csr = None
    if m is None:
        pass
    elif isinstance(m, TwoLevelPreconditioner):
        if m.n != n:
            raise ValueError("operator dimensions do not match the vector")
        m_pre = m._dev
    elif isinstance(m, CsrMatrix):
        if m.nrows != n or m.ncols != n:
            raise ValueError("operator dimensions do not match the vector")
        m_csr = device.device_csr(m)
    elif isinstance(m, device.DeviceCsr):
        m_csr = m
    else:
        m_fn = _host_operator(m)
    return a_dev, a_fn, m_pre, m_csr, m_fn


def _report(out: dict, solve_s: float) -> SolveReport:
    return SolveReport(iterations=out["iterations"], converged=out["converged"],
                       residual_history=np.asarray(out["history"]),
                       timings=Timings(solve=solve_s),
                       reduction_count=out["reduction_count"],
                       iteration_reductions=out["iteration_reductions"],
                       residual_reductions=out["residual_reductions"],
                       restarts=out["restarts"], true_residuals=out["true_residuals"])


def gmres(a, m, b, cfg: KrylovConfig = KrylovConfig(), x0=None):
    """Solve A x = b with right preconditioner M (krylov.py:141-161).
    Returns (x, SolveReport); x is a numpy array for numpy input, a device
    tensor for device-tensor input. timings.solve covers the whole call,
    host<->device copies included."""
    from . import device
    t = device.torch()
    on_device = isinstance(b, t.Tensor) and b.is_cuda
    host_tensor = isinstance(b, t.Tensor) and not b.is_cuda
    t0 = time.perf_counter()
    if on_device:
        bd = b.to(t.float64).contiguous()
        n = bd.shape[0]
    elif host_tensor:
        # (pinned) host tensor: async H2D copy, result returned on the host
        bd = b.to(device="cuda", dtype=t.float64, non_blocking=True)
        n = bd.shape[0]
        on_device = True
    else:
        bh = np.ascontiguousarray(b, dtype=np.float64)
        n = bh.shape[0]
    a_dev, a_fn, m_pre, m_csr, m_fn = _device_operators(a, m, n)
    if x0 is None:
        xd = t.zeros(n, dtype=t.float64, device="cuda")
        nonzero = False
    else:
        if isinstance(x0, t.Tensor):
            xd = x0.to(device="cuda", dtype=t.float64).clone()
        else:
            xh = np.array(x0, dtype=np.float64)
            if xh.shape != (n,):
                raise ValueError("x0 length does not match b")
            xd = t.from_numpy(xh).cuda()
        if tuple(xd.shape) != (n,):
            raise ValueError("x0 length does not match b")
        nonzero = bool((xd != 0).any().item())
    if not on_device:
        bd = t.from_numpy(bh).cuda()
    if a_fn is None and m_fn is None:
        out = device.gmres_device(a_dev, m_pre, m_csr, bd, xd, nonzero, cfg)
    else:
        out = device.gmres_host_ops(a_dev, a_fn, m_pre, m_csr, m_fn, n, bd, xd, nonzero, cfg)
    if host_tensor:
        x = device.to_host(xd)
    else:
        x = xd if on_device else device.to_host(xd).numpy()
    return x, _report(out, time.perf_counter() - t0)
