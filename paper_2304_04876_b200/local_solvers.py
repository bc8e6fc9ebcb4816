"""Subdomain solvers: orderings and symbolic phase on the host, numeric
phase and solves on the GPU (mirrors schwarzdd.local_solvers).

* Orderings (local_solvers.py:37-151): natural and the BFS-median nested
  dissection, bit-exact (libgdsw_host.so).
* Symbolic (local_solvers.py:158-243): exact no-pivot fill via the
  elimination tree and ILU(k) level-of-fill, level schedules for the
  triangular solves, and the same sha256 `structure_hash`.
* Numeric: `fast_ilu` runs its fixed-point sweeps on the GPU (batched over
  subdomains, see schwarz.setup_numeric / device.Precond.fastilu);
  `exact_lu` and `ilu_k` run the reference's pattern-restricted IKJ kernel
  (local_solvers.py:306-340) on the GPU, every block in one launch and
  bit-identical to the host kernel (separator chains factored by the whole
  CTA per row; schwarz._gpu_lu_pays).
* Solves: inside the preconditioner every block is solved in one launch --
  Jacobi FastSpTRSV for fast_ilu, the TMA-streamed level-set SpTRSV for
  ILU(k), supernodal partitioned inverses for exact factors (coarse_factor.py)
  when the blocks fit twice over the SMs. `LocalFactorization.solve`
  (`trisolve_levelset`, `fast_trisolve`) runs the same kernels through a
  one-subdomain context.

L has a unit diagonal (not stored); U stores its diagonal first per row.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

from . import _host
from .sparse_core import CsrMatrix, permute_symmetric

LOCAL_SOLVER_METHODS = ("exact_lu", "ilu_k", "fast_ilu")


@dataclass
class Ordering:
    kind: str
    perm: np.ndarray           # new position -> original index
    inverse_perm: np.ndarray

    def __post_init__(self):
        self.perm = np.asarray(self.perm, dtype=np.int64)
        self.inverse_perm = np.asarray(self.inverse_perm, dtype=np.int64)
        if not np.array_equal(self.perm[self.inverse_perm], np.arange(self.perm.size)):
            raise ValueError("perm and inverse_perm are not inverses")


def _invert(perm: np.ndarray) -> np.ndarray:
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size, dtype=np.int64)
    return inv


def order_natural(n: int) -> Ordering:
    ident = np.arange(n, dtype=np.int64)
    return Ordering("natural", ident, ident.copy())


def order_nested_dissection(a: CsrMatrix, leaf_size: int = 32) -> Ordering:
    """Recursive BFS-median bisection of the symmetrized pattern, separator
    last, natural order below `leaf_size` (local_solvers.py:72-143)."""
    if a.nrows != a.ncols:
        raise ValueError("ordering needs a square operator")
    perm = _host.nested_dissection(a.nrows, a.row_ptr, a.col_idx, leaf_size)
    return Ordering("nested_dissection", perm, _invert(perm))


def make_ordering(a: CsrMatrix, kind: str) -> Ordering:
    if kind == "natural":
        return order_natural(a.nrows)
    if kind == "nested_dissection":
        return order_nested_dissection(a)
    raise ValueError(f"unknown ordering kind {kind!r}")


# ---------------------------------------------------------------------------
# symbolic phase
# ---------------------------------------------------------------------------

@dataclass
class SymbolicFactorization:
    n: int
    kind: str                  # "exact" | "ilu"
    fill_level: int | None
    ordering: Ordering
    l_ptr: np.ndarray
    l_idx: np.ndarray
    u_ptr: np.ndarray
    u_idx: np.ndarray
    l_level_ptr: np.ndarray
    l_level_rows: np.ndarray
    u_level_ptr: np.ndarray
    u_level_rows: np.ndarray
    structure_hash: str

    @property
    def fill_nnz(self) -> int:
        return int(self.l_idx.size + self.u_idx.size)

    @property
    def n_levels(self):
        return (self.l_level_ptr.size - 1, self.u_level_ptr.size - 1)


def _finish_symbolic(n, kind, fill_level, ordering, l_ptr, l_idx, u_ptr, u_idx):
    l_level_ptr, l_level_rows = _host.level_schedule(n, l_ptr, l_idx, upper=False)
    u_level_ptr, u_level_rows = _host.level_schedule(n, u_ptr, u_idx, upper=True)
    h = hashlib.sha256()
    h.update(f"{n}|{kind}|{fill_level}|{ordering.kind}".encode())
    for arr in (ordering.perm, l_ptr, l_idx, u_ptr, u_idx):
        h.update(np.ascontiguousarray(arr, dtype=np.int64).tobytes())
    return SymbolicFactorization(n, kind, fill_level, ordering, l_ptr, l_idx, u_ptr,
                                 u_idx, l_level_ptr, l_level_rows, u_level_ptr,
                                 u_level_rows, h.hexdigest())


def symbolic_lu(a: CsrMatrix, ordering: Ordering | None = None) -> SymbolicFactorization:
    """Exact no-pivot fill of the symmetrized permuted pattern
    (local_solvers.py:205-225)."""
    if a.nrows != a.ncols:
        raise ValueError("factorization needs a square operator")
    ordering = ordering or order_natural(a.nrows)
    l_ptr, l_idx, u_ptr, u_idx = _host.symbolic_lu(a.nrows, a.row_ptr, a.col_idx,
                                                   ordering.perm)
    return _finish_symbolic(a.nrows, "exact", None, ordering, l_ptr, l_idx, u_ptr, u_idx)


def symbolic_ilu_k(a: CsrMatrix, fill_level: int,
                   ordering: Ordering | None = None) -> SymbolicFactorization:
    """Level-of-fill ILU(k) pattern (local_solvers.py:228-243)."""
    if a.nrows != a.ncols:
        raise ValueError("factorization needs a square operator")
    if fill_level < 0:
        raise ValueError("fill level must be nonnegative")
    ordering = ordering or order_natural(a.nrows)
    l_ptr, l_idx, u_ptr, u_idx = _host.symbolic_iluk(a.nrows, a.row_ptr, a.col_idx,
                                                     ordering.perm, fill_level)
    return _finish_symbolic(a.nrows, "ilu", fill_level, ordering, l_ptr, l_idx, u_ptr, u_idx)


# ---------------------------------------------------------------------------
# numeric phase
# ---------------------------------------------------------------------------

@dataclass
class LocalFactorization:
    """Factor values on a symbolic pattern. Values may live on the device
    (batched arena of a preconditioner); `l_values`/`u_values` download on
    first access. `solve` runs on the GPU."""

    symbolic: SymbolicFactorization
    method: str
    _l_values: np.ndarray | None = None
    _u_values: np.ndarray | None = None
    sweep_residuals: list | None = None
    trisolve_iters: int = 5
    _source: object = field(default=None, repr=False)   # (precond, subdomain)
    _solver: object = field(default=None, repr=False)

    @property
    def l_values(self) -> np.ndarray:
        if self._l_values is None:
            pre, s = self._source
            self._l_values, self._u_values = pre.download_factors(s)
        return self._l_values

    @property
    def u_values(self) -> np.ndarray:
        if self._u_values is None:
            _ = self.l_values
        return self._u_values

    @property
    def dtype(self):
        if self._l_values is None and self._source is not None:
            return self._source[0].value_dtype
        return self.l_values.dtype

    @property
    def fill_nnz(self) -> int:
        return self.symbolic.fill_nnz

    def _device_solver(self):
        if self._solver is None:
            from .device import SingleBlockSolver
            self._solver = SingleBlockSolver(self)
        return self._solver

    def solve(self, b: np.ndarray) -> np.ndarray:
        """x = (LU)^-1 b in the factor's element type, through the GPU
        (local_solvers.py:263-278)."""
        return self._device_solver().solve(b, self.trisolve_iters)

    def solve_many(self, b: np.ndarray) -> np.ndarray:
        b = np.asarray(b)
        return np.stack([self.solve(np.ascontiguousarray(b[:, c]))
                         for c in range(b.shape[1])], axis=1)


def _norm_inf(p: CsrMatrix) -> float:
    if p.values.size == 0:
        return 0.0
    sums = np.zeros(p.nrows)
    np.add.at(sums, p.row_ids(), np.abs(p.values.astype(np.float64)))
    return float(sums.max())


def _pivot_error(sym: SymbolicFactorization, rc: int) -> np.linalg.LinAlgError:
    row = int(sym.ordering.perm[rc - 1])
    return np.linalg.LinAlgError(
        f"pivot too small at row {row} (|u_ii| <= 1e-14 * ||A||_inf); "
        "the operator is singular or needs a different ordering")


def host_numeric(a: CsrMatrix, sym: SymbolicFactorization, diag_shift: float = 0.0):
    """IKJ numeric LU/ILU on the symbolic pattern (local_solvers.py:306-327,
    _kernels.py:429-466). Returns (l_values, u_values)."""
    if a.nrows != sym.n:
        raise ValueError("matrix size does not match the symbolic phase")
    p = permute_symmetric(a, sym.ordering.perm)
    vals = p.values
    if diag_shift:
        vals = vals.copy()
        vals[p.col_idx == p.row_ids()] += vals.dtype.type(diag_shift)
    tol = 1e-14 * _norm_inf(p)
    rc, l_values, u_values = _host.lu_numeric(sym.n, sym.l_ptr, sym.l_idx, sym.u_ptr,
                                              sym.u_idx, p.row_ptr, p.col_idx, vals, tol)
    if rc:
        raise _pivot_error(sym, rc)
    return l_values, u_values


def numeric_lu(a: CsrMatrix, sym: SymbolicFactorization) -> LocalFactorization:
    if sym.kind != "exact":
        raise ValueError("numeric_lu needs an exact symbolic phase")
    lv, uv = host_numeric(a, sym, 0.0)
    return LocalFactorization(sym, "exact_lu", lv, uv)


def numeric_ilu(a: CsrMatrix, sym: SymbolicFactorization,
                diag_shift: float = 0.0) -> LocalFactorization:
    if sym.kind != "ilu":
        raise ValueError("numeric_ilu needs an ilu symbolic phase")
    lv, uv = host_numeric(a, sym, diag_shift)
    return LocalFactorization(sym, "ilu_k", lv, uv)


def fast_ilu_numeric(a: CsrMatrix, sym: SymbolicFactorization, factor_sweeps: int = 3,
                     trisolve_iters: int = 5) -> LocalFactorization:
    """Fixed-point ILU sweeps on the GPU (local_solvers.py:343-397) for one
    block; the batched path lives in schwarz.setup_numeric."""
    if sym.kind != "ilu":
        raise ValueError("fast_ilu_numeric needs an ilu symbolic phase")
    if factor_sweeps < 1:
        raise ValueError("factor_sweeps must be at least 1")
    if trisolve_iters < 1:
        raise ValueError("trisolve_iters must be at least 1")
    from .device import single_block_fastilu
    return single_block_fastilu(a, sym, factor_sweeps, trisolve_iters)


# ---------------------------------------------------------------------------
# solve entry points
# ---------------------------------------------------------------------------

def trisolve_levelset(fac: LocalFactorization, b: np.ndarray) -> np.ndarray:
    """Level-scheduled forward/backward substitution (bit-identical to the
    sequential substitution; local_solvers.py:404-410)."""
    if fac.method == "fast_ilu":
        raise ValueError("fast_ilu factors are solved with fast_trisolve")
    return fac.solve(b)


def fast_trisolve(fac: LocalFactorization, b: np.ndarray, iters: int) -> np.ndarray:
    """Jacobi triangular iteration with `iters` iterates on L then U
    (local_solvers.py:413-427)."""
    if iters < 1:
        raise ValueError("iters must be at least 1")
    return fac._device_solver().solve(b, iters, force_jacobi=True)


# ---------------------------------------------------------------------------
# configuration-driven dispatch
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class SolverSpec:
    method: str = "exact_lu"
    fill_level: int = 0
    factor_sweeps: int = 3
    trisolve_iters: int = 5
    diag_shift: float = 0.0

    def __post_init__(self):
        if self.method not in LOCAL_SOLVER_METHODS:
            raise ValueError(f"unknown local solver method {self.method!r}")


def build_symbolic(a: CsrMatrix, spec: SolverSpec,
                   ordering: Ordering | None = None) -> SymbolicFactorization:
    if spec.method == "exact_lu":
        return symbolic_lu(a, ordering)
    return symbolic_ilu_k(a, spec.fill_level, ordering)


def build_numeric(a: CsrMatrix, sym: SymbolicFactorization,
                  spec: SolverSpec) -> LocalFactorization:
    if spec.method == "exact_lu":
        return numeric_lu(a, sym)
    if spec.method == "ilu_k":
        return numeric_ilu(a, sym, spec.diag_shift)
    return fast_ilu_numeric(a, sym, spec.factor_sweeps, spec.trisolve_iters)
