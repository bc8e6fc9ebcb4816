"""ORACLE -- test infrastructure, NOT the product (see oracle/__init__.py).

Sequential CPU restatement of the reference's numeric and solve phases:

* kernels: oracle_kernels.c (bit-identical restatements of
  _kernels.py:23-31, 429-466, 473-522, 547-656);
* `OracleSchwarz`: setup_numeric + apply of schwarz.py:213-327 with exact
  interior LU for the harmonic extension (coarse_space.py:106-179), the
  Galerkin product by scipy.sparse, and the sparse-LU coarse solve;
* `gmres`: _gmres_single_reduce / _gmres_classic of krylov.py:179-361.

Index-level inputs (overlap sets, orderings, fill patterns, level
schedules, interface components) come from the product's host layer, which
tests pin bit-exact against the reference's own (tests/golden).
"""

from __future__ import annotations

import ctypes as C
import math
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_SO = HERE / "_build" / "liboracle.so"


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return _SO


def _load():
    if not _SO.exists() or _SO.stat().st_mtime < (HERE / "oracle_kernels.c").stat().st_mtime:
        build()
    lib = C.CDLL(str(_SO))
    lib.or_lu_numeric_f64.restype = C.c_int64
    lib.or_lu_numeric_f32.restype = C.c_int64
    lib.or_fastilu_sweep_f64.restype = C.c_int
    lib.or_fastilu_sweep_f32.restype = C.c_int
    lib.or_fastilu_residual_f64.restype = C.c_double
    lib.or_fastilu_residual_f32.restype = C.c_double
    return lib


_lib = _load()


def _p(a):
    return C.c_void_p(a.ctypes.data)


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _sfx(dt) -> str:
    return "f32" if np.dtype(dt) == np.float32 else "f64"


def _scalar(dt, v):
    return C.c_float(v) if np.dtype(dt) == np.float32 else C.c_double(v)


# ---------------------------------------------------------------------------
# kernels
# ---------------------------------------------------------------------------

def spmv(ptr, idx, val, x, y=None, alpha=1.0, beta=0.0):
    """y <- alpha*A x + beta*y in A's element type (_kernels.py:23-31)."""
    val = np.ascontiguousarray(val)
    dt = val.dtype
    x = np.ascontiguousarray(x, dtype=dt)
    n = len(ptr) - 1
    if y is None:
        y = np.zeros(n, dtype=dt)
        beta = 0.0
    getattr(_lib, f"or_spmv_{_sfx(dt)}")(C.c_int64(n), _p(_i(ptr)), _p(_i(idx)), _p(val), _p(x),
                                         _p(y), _scalar(dt, alpha), _scalar(dt, beta))
    return y


def csr_spmv(a, x):
    return spmv(a.row_ptr, a.col_idx, a.values, x)


def levelset_solve(sym, lv, uv, b):
    """LocalFactorization.solve for exact/ILU factors (local_solvers.py:263-278)."""
    dt = lv.dtype
    x = np.ascontiguousarray(np.asarray(b)[sym.ordering.perm].astype(dt))
    s = _sfx(dt)
    getattr(_lib, f"or_trisolve_lower_{s}")(_p(_i(sym.l_ptr)), _p(_i(sym.l_idx)), _p(lv),
                                            C.c_int64(sym.l_level_ptr.size - 1),
                                            _p(_i(sym.l_level_ptr)), _p(_i(sym.l_level_rows)),
                                            _p(x))
    getattr(_lib, f"or_trisolve_upper_{s}")(_p(_i(sym.u_ptr)), _p(_i(sym.u_idx)), _p(uv),
                                            C.c_int64(sym.u_level_ptr.size - 1),
                                            _p(_i(sym.u_level_ptr)), _p(_i(sym.u_level_rows)),
                                            _p(x))
    out = np.empty_like(x)
    out[sym.ordering.perm] = x
    return out


def jacobi_solve(sym, lv, uv, b, iters):
    """fast_trisolve / fast_ilu solve (local_solvers.py:413-427)."""
    dt = lv.dtype
    n = sym.n
    bb = np.ascontiguousarray(np.asarray(b)[sym.ordering.perm].astype(dt))
    x, w = np.empty(n, dtype=dt), np.empty(n, dtype=dt)
    s = _sfx(dt)
    getattr(_lib, f"or_jacobi_lower_{s}")(C.c_int64(n), _p(_i(sym.l_ptr)), _p(_i(sym.l_idx)),
                                          _p(lv), _p(bb), C.c_int64(iters), _p(x), _p(w))
    y = np.empty(n, dtype=dt)
    getattr(_lib, f"or_jacobi_upper_{s}")(C.c_int64(n), _p(_i(sym.u_ptr)), _p(_i(sym.u_idx)),
                                          _p(uv), _p(x), C.c_int64(iters), _p(y), _p(w))
    out = np.empty_like(y)
    out[sym.ordering.perm] = y
    return out


def _norm_inf(ptr, vals) -> float:
    if vals.size == 0:
        return 0.0
    sums = np.zeros(len(ptr) - 1)
    np.add.at(sums, np.repeat(np.arange(len(ptr) - 1), np.diff(ptr)),
              np.abs(vals.astype(np.float64)))
    return float(sums.max())


def _permuted(block, perm):
    if np.array_equal(perm, np.arange(len(perm))):
        return block    # natural ordering (reference_setup: no product import)
    from paper_2304_04876_b200.sparse_core import permute_symmetric
    return permute_symmetric(block, perm)


def lu_numeric(block, sym, diag_shift: float = 0.0):
    """Numeric LU/ILU on the symbolic pattern (local_solvers.py:306-327)."""
    p = _permuted(block, sym.ordering.perm)
    vals = p.values
    if diag_shift:
        vals = vals.copy()
        vals[p.col_idx == p.row_ids()] += vals.dtype.type(diag_shift)
    tol = 1e-14 * _norm_inf(p.row_ptr, p.values)
    dt = vals.dtype
    lv = np.zeros(sym.l_idx.size, dtype=dt)
    uv = np.zeros(sym.u_idx.size, dtype=dt)
    rc = getattr(_lib, f"or_lu_numeric_{_sfx(dt)}")(
        C.c_int64(sym.n), _p(_i(sym.l_ptr)), _p(_i(sym.l_idx)), _p(_i(sym.u_ptr)),
        _p(_i(sym.u_idx)), _p(p.row_ptr), _p(p.col_idx), _p(np.ascontiguousarray(vals)),
        _p(lv), _p(uv), C.c_double(tol))
    if rc:
        raise np.linalg.LinAlgError(f"pivot too small at row {int(sym.ordering.perm[rc - 1])}")
    return lv, uv


def _align(a_ptr, a_idx, f_ptr, f_idx):
    out = np.full(len(f_idx), -1, dtype=np.int64)
    for i in range(len(a_ptr) - 1):
        cols = a_idx[a_ptr[i]:a_ptr[i + 1]]
        fc = f_idx[f_ptr[i]:f_ptr[i + 1]]
        pos = np.searchsorted(cols, fc)
        ok = (pos < cols.size) & (cols[np.minimum(pos, max(cols.size - 1, 0))] == fc) \
            if cols.size else np.zeros(fc.size, bool)
        out[f_ptr[i]:f_ptr[i + 1]] = np.where(ok, a_ptr[i] + pos, -1)
    return out


def _transpose_pattern(n, ptr, idx):
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ptr))
    order = np.lexsort((rows, idx))
    t_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(t_ptr, idx + 1, 1)
    return np.cumsum(t_ptr), rows[order], order.astype(np.int64)


def fast_ilu(block, sym, sweeps: int = 3):
    """Fixed-point ILU sweeps (local_solvers.py:343-397). Returns
    (l_values, u_values, residuals)."""
    p = _permuted(block, sym.ordering.perm)
    vals = np.ascontiguousarray(p.values)
    dt = vals.dtype
    n = sym.n
    a_of_l = _align(p.row_ptr, p.col_idx, sym.l_ptr, sym.l_idx)
    a_of_u = _align(p.row_ptr, p.col_idx, sym.u_ptr, sym.u_idx)
    l_of_a = _align(sym.l_ptr, sym.l_idx, p.row_ptr, p.col_idx)
    u_of_a = _align(sym.u_ptr, sym.u_idx, p.row_ptr, p.col_idx)
    ucp, ucr, ucs = _transpose_pattern(n, _i(sym.u_ptr), _i(sym.u_idx))
    zero = dt.type(0)
    u_old = np.where(a_of_u >= 0, vals[np.maximum(a_of_u, 0)], zero).astype(dt)
    diag = u_old[sym.u_ptr[:-1]]
    l_old = np.where(a_of_l >= 0, vals[np.maximum(a_of_l, 0)], zero).astype(dt)
    with np.errstate(divide="ignore", invalid="ignore"):
        l_old = (l_old / diag[sym.l_idx]).astype(dt)
    l_new, u_new = np.empty_like(l_old), np.empty_like(u_old)
    s = _sfx(dt)
    args_pat = [_p(_i(sym.l_ptr)), _p(_i(sym.l_idx))]
    residuals = []
    for _ in range(sweeps):
        bad = getattr(_lib, f"or_fastilu_sweep_{s}")(
            C.c_int64(n), *args_pat, _p(l_old), _p(l_new), _p(_i(sym.u_ptr)), _p(_i(sym.u_idx)),
            _p(u_old), _p(u_new), _p(ucp), _p(ucr), _p(ucs), _p(a_of_l), _p(a_of_u), _p(vals))
        if bad:
            raise FloatingPointError("fixed-point factorization produced nonfinite entries")
        l_old, l_new = l_new, l_old
        u_old, u_new = u_new, u_old
        residuals.append(float(getattr(_lib, f"or_fastilu_residual_{s}")(
            C.c_int64(n), *args_pat, _p(l_old), _p(_i(sym.u_ptr)), _p(_i(sym.u_idx)), _p(u_old),
            _p(ucp), _p(ucr), _p(ucs), _p(l_of_a), _p(u_of_a), _p(p.row_ptr), _p(p.col_idx),
            _p(vals))))
    if not (np.isfinite(l_old).all() and np.isfinite(u_old).all()):
        raise FloatingPointError("fixed-point factorization produced nonfinite entries")
    return l_old.copy(), u_old.copy(), residuals


# ---------------------------------------------------------------------------
# two-level preconditioner (schwarz.py:213-327)
# ---------------------------------------------------------------------------

class OracleSchwarz:
    """CPU restatement of setup_numeric + apply. `symbolics` are the
    product's host SymbolicFactorizations of the overlap blocks."""

    def __init__(self, a, dec, config, nullspace=None, symbolics=None, threads: int = 1,
                 coarse_parts=None):
        """coarse_parts=(phi, a0): take a ready coarse basis (timing samples
        only) instead of the exact-LU harmonic extension."""
        from paper_2304_04876_b200 import local_solvers as L
        from paper_2304_04876_b200.sparse_core import (CsrMatrix, convert_precision,
                                                       extract_submatrix)
        self.n = a.nrows
        self.sets = [np.asarray(s, np.int64) for s in dec.overlap.sets]
        self.single = config.precision == "single"
        spec = config.local
        if self.single:
            a32 = convert_precision(a, np.float32)
            local_src = a32
            coarse_src = CsrMatrix(a.nrows, a.ncols, a.row_ptr, a.col_idx,
                                   a32.values.astype(np.float64))
        else:
            local_src = coarse_src = a
        if symbolics is None:
            symbolics = []
            for dofs in self.sets:
                blk = extract_submatrix(a, dofs, dofs)
                symbolics.append(L.build_symbolic(blk, spec, L.make_ordering(blk, config.ordering)))
        self.symbolics = symbolics
        self.method = spec.method
        self.iters = spec.trisolve_iters
        # apply: subdomain solves on a thread pool like the reference's
        # `threads` option (schwarz.py:111-127, 310-324); the C kernels run
        # without the GIL, the sum stays in subdomain order
        self.threads = max(1, threads)
        self._pool = ThreadPoolExecutor(max_workers=self.threads) if self.threads > 1 else None

        def one(i):
            blk = extract_submatrix(local_src, self.sets[i], self.sets[i])
            if spec.method == "fast_ilu":
                return fast_ilu(blk, symbolics[i], spec.factor_sweeps)
            shift = spec.diag_shift if spec.method == "ilu_k" else 0.0
            lv, uv = lu_numeric(blk, symbolics[i], shift)
            return lv, uv, None

        with ThreadPoolExecutor(max_workers=max(1, threads)) as ex:
            self.factors = list(ex.map(one, range(len(self.sets))))
        self.coarse = None
        if config.use_coarse and coarse_parts is not None:
            self.coarse = _coarse_from_parts(*coarse_parts, config)
        elif config.use_coarse:
            self.coarse = _oracle_coarse(coarse_src, dec, nullspace, config, self.single, threads)

    def local_solve(self, i, b):
        lv, uv, _ = self.factors[i]
        if self.method == "fast_ilu":
            return jacobi_solve(self.symbolics[i], lv, uv, b, self.iters)
        return levelset_solve(self.symbolics[i], lv, uv, b)

    def apply(self, r):
        """z = Phi A0^-1 Phi^T r + sum_i R_i^T A_i^-1 R_i r, contributions in
        subdomain order (schwarz.py:290-327)."""
        r = np.ascontiguousarray(r, dtype=np.float64)
        rw = r.astype(np.float32) if self.single else r
        zc = None
        if self.coarse is not None:
            phi, phi_t, a0_sym, a0_l, a0_u = self.coarse
            u = csr_spmv(phi_t, rw)
            v = levelset_solve(a0_sym, a0_l, a0_u, u)
            zc = csr_spmv(phi, v)
        z = np.zeros(self.n, dtype=rw.dtype)
        if self._pool is not None:
            ys = list(self._pool.map(lambda i: self.local_solve(i, rw[self.sets[i]]),
                                     range(len(self.sets))))
        else:
            ys = (self.local_solve(i, rw[dofs]) for i, dofs in enumerate(self.sets))
        for dofs, y in zip(self.sets, ys):
            z[dofs] += y
        if zc is not None:
            z = zc + z
        return z.astype(np.float64) if self.single else z


def _coarse_from_parts(phi, a0, config):
    import scipy.sparse as sp
    from paper_2304_04876_b200 import local_solvers as L
    from paper_2304_04876_b200.sparse_core import CsrMatrix
    a0_sym = L.symbolic_lu(a0, L.make_ordering(a0, config.ordering))
    a0_l, a0_u = lu_numeric(a0, a0_sym)
    pt = sp.csr_matrix((phi.values, phi.col_idx, phi.row_ptr), shape=phi.shape).T.tocsr()
    pt.sort_indices()
    phi_t = CsrMatrix(phi.ncols, phi.nrows, pt.indptr, pt.indices, pt.data)
    return phi, phi_t, a0_sym, a0_l, a0_u


def _oracle_coarse(a, dec, nullspace, config, single, threads):
    """Phi by exact interior LU (coarse_space.py:106-179), A0 = Phi^T A Phi,
    A0 sparse LU (schwarz.py:241-272)."""
    import scipy.sparse as sp
    from paper_2304_04876_b200 import coarse_space as CS
    from paper_2304_04876_b200 import local_solvers as L
    from paper_2304_04876_b200.sparse_core import CsrMatrix, convert_precision, extract_submatrix
    structure = dec.structure
    basis = CS.interface_basis(nullspace, structure)
    column_map, pg = CS.coarse_columns(structure, basis)
    n_cols = len(column_map)
    if n_cols == 0:
        raise ValueError("coarse space is empty")
    gamma = structure.interface
    isets = CS.interior_sets(dec.partition, structure)
    rows = [gamma[pg.row_ids()]]
    cols = [pg.col_idx]
    vals = [pg.values]
    pgd = sp.csr_matrix((pg.values, pg.col_idx, pg.row_ptr), shape=(gamma.size, n_cols))

    def one(s):
        dofs = isets[s]
        if dofs.size == 0:
            return None
        blk = extract_submatrix(a, dofs, dofs)
        sym = L.symbolic_lu(blk, L.make_ordering(blk, "nested_dissection"))
        lv, uv = lu_numeric(blk, sym)
        cpl = extract_submatrix(a, dofs, gamma)
        need = np.unique(pgd[np.unique(cpl.col_idx)].indices)
        if need.size == 0:
            return None
        dense_g = np.ascontiguousarray(pgd[:, need].toarray())
        rhs = np.empty((dofs.size, need.size))
        _lib.or_csr_matmat_dense_f64(C.c_int64(dofs.size), _p(cpl.row_ptr), _p(cpl.col_idx),
                                     _p(cpl.values), _p(dense_g), C.c_int64(need.size), _p(rhs))
        rhs = -rhs
        x = np.ascontiguousarray(rhs[sym.ordering.perm])
        _lib.or_trisolve_lower_multi_f64(_p(_i(sym.l_ptr)), _p(_i(sym.l_idx)), _p(lv),
                                         C.c_int64(sym.l_level_ptr.size - 1),
                                         _p(_i(sym.l_level_ptr)), _p(_i(sym.l_level_rows)),
                                         _p(x), C.c_int64(need.size))
        _lib.or_trisolve_upper_multi_f64(_p(_i(sym.u_ptr)), _p(_i(sym.u_idx)), _p(uv),
                                         C.c_int64(sym.u_level_ptr.size - 1),
                                         _p(_i(sym.u_level_ptr)), _p(_i(sym.u_level_rows)),
                                         _p(x), C.c_int64(need.size))
        sol = np.empty_like(x)
        sol[sym.ordering.perm] = x
        rr, cc = np.nonzero(sol)
        return dofs[rr], need[cc], sol[rr, cc]

    with ThreadPoolExecutor(max_workers=max(1, threads)) as ex:
        for part in ex.map(one, range(len(isets))):
            if part is not None:
                rows.append(part[0])
                cols.append(part[1])
                vals.append(part[2])
    phi = CsrMatrix.from_coo(a.nrows, n_cols, np.concatenate(rows), np.concatenate(cols),
                             np.concatenate(vals))
    P = sp.csr_matrix((phi.values, phi.col_idx, phi.row_ptr), shape=phi.shape)
    A = sp.csr_matrix((a.values, a.col_idx, a.row_ptr), shape=a.shape)
    a0s = (P.T @ (A @ P)).tocsr()
    a0s.sort_indices()
    a0 = CsrMatrix(n_cols, n_cols, a0s.indptr, a0s.indices, a0s.data)
    if single:
        phi = convert_precision(phi, np.float32)
        a0 = convert_precision(a0, np.float32)
    a0_sym = L.symbolic_lu(a0, L.make_ordering(a0, config.ordering))
    a0_l, a0_u = lu_numeric(a0, a0_sym)
    pt = sp.csr_matrix((phi.values, phi.col_idx, phi.row_ptr), shape=phi.shape).T.tocsr()
    pt.sort_indices()
    phi_t = CsrMatrix(phi.ncols, phi.nrows, pt.indptr, pt.indices, pt.data)
    return phi, phi_t, a0_sym, a0_l, a0_u


# ---------------------------------------------------------------------------
# GMRES (krylov.py:111-361)
# ---------------------------------------------------------------------------

def _rotation(a, b):
    r = math.hypot(a, b)
    return (1.0, 0.0) if r == 0.0 else (a / r, b / r)


def _givens_column(h, cs, sn, g, j):
    for i in range(j):
        t = cs[i] * h[i, j] + sn[i] * h[i + 1, j]
        h[i + 1, j] = -sn[i] * h[i, j] + cs[i] * h[i + 1, j]
        h[i, j] = t
    cs[j], sn[j] = _rotation(h[j, j], h[j + 1, j])
    h[j, j] = cs[j] * h[j, j] + sn[j] * h[j + 1, j]
    h[j + 1, j] = 0.0
    g[j + 1] = -sn[j] * g[j]
    g[j] = cs[j] * g[j]
    return abs(g[j + 1])


def _back_solve(h, g, m):
    y = np.zeros(m)
    for i in range(m - 1, -1, -1):
        y[i] = (g[i] - h[i, i + 1:m] @ y[i + 1:m]) / h[i, i]
    return y


def gmres(a_op, m_op, b, restart=30, rel_tol=1e-7, max_iters=500, variant="single_reduce",
          orthogonalization="mgs", x0=None, reject_checks=0):
    """Returns (x, dict(iterations, converged, history, true_residuals,
    iteration_reductions, residual_reductions, restarts)).
    reject_checks (test hook, mirrors libgdsw's GDSW_DEBUG_REJECT_CHECKS):
    the first k true-residual confirmations count as failed."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(b.size) if x0 is None else np.array(x0, dtype=np.float64)
    m_op = m_op or (lambda v: v)
    st = dict(it=0, res=0, itr=0, restarts=0, history=[1.0], true=[], reject=reject_checks)
    if variant == "single_reduce":
        x, conv = _sr(a_op, m_op, b, x, restart, rel_tol, max_iters, st)
    else:
        x, conv = _classic(a_op, m_op, b, x, restart, rel_tol, max_iters, orthogonalization, st)
    return x, dict(iterations=st["it"], converged=conv, history=np.array(st["history"]),
                   true_residuals=st["true"], iteration_reductions=st["itr"],
                   residual_reductions=st["res"], restarts=st["restarts"])


def _rejected(st) -> bool:
    if st["reject"] > 0:
        st["reject"] -= 1
        return True
    return False


def _bnorm(b, x, beta, st):
    if not np.any(x):
        return beta
    st["res"] += 1
    return float(np.linalg.norm(b))


def _sr(A, M, b, x, R, tol, maxit, st):
    n = b.size
    V, Z = np.zeros((R, n)), np.zeros((R, n))
    h, g = np.zeros((R + 1, R)), np.zeros(R + 1)
    cs, sn = np.zeros(R), np.zeros(R)
    denom = bnorm = None
    while True:
        vc = b - A(x)
        st["restarts"] += 1
        mc = M(vc)
        zc = A(mc)
        g[:] = 0.0
        for j in range(R + 1):
            last = j == R
            basis = np.concatenate([V[:j], vc[None, :]])
            if last:
                blk = basis @ vc
                a, b2 = blk[:j], float(blk[j])
            else:
                blk = basis @ np.stack([vc, zc], axis=1)
                a, b2, p, q = blk[:j, 0], float(blk[j, 0]), blk[:j, 1], float(blk[j, 1])
            st["res" if j == 0 else "itr"] += 1
            d2 = b2 - float(a @ a)
            d = math.sqrt(d2) if d2 > 0.0 else 0.0
            if j == 0:
                if denom is None:
                    denom, bnorm = d, _bnorm(b, x, d, st)
                    if d <= 1e-14 * bnorm:
                        return x, True
                else:
                    st["true"].append((st["it"], d / denom))
                if d / denom <= tol:
                    return x, True
                g[0] = d
            else:
                h[:j, j - 1] += a
                h[j, j - 1] = d
                st["it"] += 1
                est = _givens_column(h, cs, sn, g, j - 1)
                st["history"].append(est / denom)
                brk = d <= 1e-14 * bnorm
                if brk or est / denom <= tol or st["it"] >= maxit:
                    xc = x + _back_solve(h, g, j) @ Z[:j]
                    st["res"] += 1
                    tr = float(np.linalg.norm(b - A(xc)))
                    st["true"].append((st["it"], tr / denom))
                    if tr / denom <= tol and not _rejected(st):
                        return xc, True
                    if brk or st["it"] >= maxit:
                        return xc, False
            if last:
                break
            V[j] = (vc - a @ V[:j]) / d
            Z[j] = (mc - a @ Z[:j]) / d
            corr = (q - float(a @ p)) / (d * d)
            h[:j, j] = p / d
            h[j, j] = corr
            vc = zc / d - (p / d) @ V[:j] - corr * V[j]
            if j + 1 <= R - 1:
                mc = M(vc)
                zc = A(mc)
        x = x + _back_solve(h, g, R) @ Z[:R]


def _classic(A, M, b, x, R, tol, maxit, orth, st):
    n = b.size
    V, Z = np.zeros((R + 1, n)), np.zeros((R, n))
    h, g = np.zeros((R + 1, R)), np.zeros(R + 1)
    cs, sn = np.zeros(R), np.zeros(R)
    denom = bnorm = None
    while True:
        r0 = b - A(x)
        beta = float(np.linalg.norm(r0))
        st["res"] += 1
        st["restarts"] += 1
        if denom is None:
            denom, bnorm = beta, _bnorm(b, x, beta, st)
            if beta <= 1e-14 * bnorm:
                return x, True
        else:
            st["true"].append((st["it"], beta / denom))
        if beta / denom <= tol:
            return x, True
        V[0] = r0 / beta
        g[:] = 0.0
        g[0] = beta
        for j in range(R):
            Z[j] = M(V[j])
            w = A(Z[j])
            if orth == "mgs":
                for i in range(j + 1):
                    hij = float(V[i] @ w)
                    st["itr"] += 1
                    w -= hij * V[i]
                    h[i, j] = hij
            else:
                c1 = V[:j + 1] @ w
                w -= c1 @ V[:j + 1]
                c2 = V[:j + 1] @ w
                w -= c2 @ V[:j + 1]
                st["itr"] += 2
                h[:j + 1, j] = c1 + c2
            nrm = float(np.linalg.norm(w))
            st["itr"] += 1
            h[j + 1, j] = nrm
            st["it"] += 1
            est = _givens_column(h, cs, sn, g, j)
            st["history"].append(est / denom)
            brk = nrm <= 1e-14 * bnorm
            if brk or est / denom <= tol or st["it"] >= maxit:
                xc = x + _back_solve(h, g, j + 1) @ Z[:j + 1]
                st["res"] += 1
                tr = float(np.linalg.norm(b - A(xc)))
                st["true"].append((st["it"], tr / denom))
                if tr / denom <= tol and not _rejected(st):
                    return xc, True
                if brk or st["it"] >= maxit:
                    return xc, False
            if j + 1 < R:
                V[j + 1] = w / nrm
        x = x + _back_solve(h, g, R) @ Z
