"""Coarse basis (Phi) and Galerkin coarse operator (mirrors
schwarzdd.coarse_space, coarse_space.py:1-237).

* `interface_basis` (host, tiny): null space restricted to each interface
  component, scaled by the partition-of-unity weights, dependent / vanishing
  columns dropped (coarse_space.py:64-103). Bitwise identical.
* Harmonic extension (GPU): Phi_I = -A_II^-1 A_IG Phi_G for only the k_s
  coarse columns that touch subdomain s, solved as one batched CG on the
  device into dense column-major interior panels
  (csrc/extension.cuh; reference: coarse_space.py:130-179, which factors
  every interior exactly and solves all n_c columns densely). The reference's
  residual check (coarse_space.py:182-202) is applied unchanged.
* `coarse_matrix`: A0 = Phi^T (A Phi) on the host (setup-only SpGEMM,
  coarse_space.py:205-207).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

from .decomposition import InterfaceStructure, Partition
from .sparse_core import CsrMatrix, extract_with_source, spgemm, transpose

EXTENSION_TOL = 1e-13       # relative CG residual per column
EXTENSION_MAX_ITERS = 20000


@dataclass
class InterfaceBasis:
    blocks: list
    kept: list
    n_nullspace: int
    coeffs: list = None


@dataclass
class InteriorBlocks:
    sets: list
    factors: list = None


@dataclass
class CoarseBasis:
    phi: CsrMatrix
    a0: CsrMatrix
    column_map: list

    @property
    def n_coarse(self) -> int:
        return self.phi.ncols


def interface_basis(nullspace: np.ndarray, structure: InterfaceStructure) -> InterfaceBasis:
    """Weights x restricted null space per component; keep/drop decided by
    an orthonormal scratch basis, kept columns copied unmodified
    (coarse_space.py:64-103)."""
    z = np.asarray(nullspace, dtype=np.float64)
    if z.ndim != 2:
        raise ValueError("nullspace must be a 2-D column block")
    col_scale = np.linalg.norm(z, axis=0)
    blocks, kept, coeffs = [], [], []
    for t, comp in enumerate(structure.components):
        vals = comp.weights[:, None] * z[comp.dofs, :]
        norms = np.linalg.norm(vals, axis=0)
        keep = []
        q = np.zeros((vals.shape[0], 0))
        for j in range(z.shape[1]):
            if norms[j] <= 1e-12 * col_scale[j]:
                continue
            r = vals[:, j] - q @ (q.T @ vals[:, j])
            r -= q @ (q.T @ r)
            rnorm = np.linalg.norm(r)
            if rnorm > 1e-8 * norms[j]:
                q = np.hstack([q, (r / rnorm)[:, None]])
                keep.append(j)
        if not keep:
            warnings.warn(f"interface component {t} has no nonzero null-space restriction; "
                          "it contributes no coarse functions")
            coeffs.append(np.zeros((0, z.shape[1])))
        else:
            coeffs.append(np.linalg.lstsq(vals[:, keep], vals, rcond=None)[0])
        blocks.append(vals[:, keep])
        kept.append(keep)
    return InterfaceBasis(blocks, kept, z.shape[1], coeffs)


def interior_sets(part: Partition, structure: InterfaceStructure, subdomains=None) -> list:
    """I_s = dofs owned by s and not on the interface (schwarz.py:177-181);
    `subdomains`: only those, in that order (sharded setups)."""
    on_iface = np.zeros(structure.n, dtype=bool)
    on_iface[structure.interface] = True
    subs = range(part.n_parts) if subdomains is None else subdomains
    return [np.flatnonzero((part.owner == s) & ~on_iface) for s in subs]


def coarse_columns(structure: InterfaceStructure, basis: InterfaceBasis):
    """Column map and the interface rows of Phi as CSR over interface
    positions (coarse_space.py:139-157)."""
    gamma = structure.interface
    column_map, rows, cols, vals = [], [], [], []
    for t, comp in enumerate(structure.components):
        start = len(column_map)
        column_map.extend((t, j) for j in basis.kept[t])
        ids = np.arange(start, len(column_map), dtype=np.int64)
        if ids.size == 0:
            continue
        pos = np.searchsorted(gamma, comp.dofs)
        rows.append(np.repeat(pos, ids.size))
        cols.append(np.tile(ids, pos.size))
        vals.append(np.asarray(basis.blocks[t], dtype=np.float64).ravel())
    n_cols = len(column_map)
    if rows:
        pg = CsrMatrix.from_coo(gamma.size, max(n_cols, 1), np.concatenate(rows),
                                np.concatenate(cols), np.concatenate(vals))
    else:
        pg = CsrMatrix.from_coo(gamma.size, max(n_cols, 1), [], [], np.zeros(0))
    return column_map, pg


def _row_entries(ptr: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """Entry positions of the given CSR rows, concatenated."""
    lens = ptr[rows + 1] - ptr[rows]
    total = int(lens.sum())
    if total == 0:
        return np.zeros(0, dtype=np.int64)
    starts = np.repeat(ptr[rows] - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens)
    return starts + np.arange(total, dtype=np.int64)


def coarse_desc(a: CsrMatrix, structure: InterfaceStructure, pg: CsrMatrix, n_cols: int,
                sets: list, gamma: np.ndarray | None = None) -> dict:
    """Device descriptor of the coarse structure: interface rows of Phi,
    per-subdomain interior rows and touching coarse columns, and the A_II /
    A_IG patterns with their A.values positions. `gamma` overrides the
    interface row list (a rank's owned interface rows, sharded solve)."""
    if gamma is None:
        gamma = structure.interface
    int_ptr = np.zeros(len(sets) + 1, dtype=np.int64)
    col_lists, aii, aig = [], [], []
    for s, dofs in enumerate(sets):
        int_ptr[s + 1] = int_ptr[s] + dofs.size
        blk, src = extract_with_source(a, dofs, dofs)
        aii.append((blk.row_ptr, blk.col_idx, src))
        cpl, csrc = extract_with_source(a, dofs, gamma)
        aig.append((cpl.row_ptr, cpl.col_idx, csrc))
        g = np.unique(cpl.col_idx)
        cols = np.unique(pg.col_idx[_row_entries(pg.row_ptr, g)])
        col_lists.append(cols[cols < n_cols])

    def cat_csr(parts):
        ptr = [np.zeros(1, dtype=np.int64)]
        off = 0
        for p, _, _ in parts:
            ptr.append(p[1:] + off)
            off += p[-1]
        return (np.concatenate(ptr), np.concatenate([c for _, c, _ in parts] or [np.zeros(0)]),
                np.concatenate([s for _, _, s in parts] or [np.zeros(0)]))

    aii_ptr, aii_col, aii_src = cat_csr(aii)
    aig_ptr, aig_col, aig_src = cat_csr(aig)
    col_ptr = np.concatenate([[0], np.cumsum([c.size for c in col_lists])]).astype(np.int64)
    return dict(n_c=n_cols, n_gamma=gamma.size, gamma_rows=gamma, pg_ptr=pg.row_ptr,
                pg_col=pg.col_idx, pg_val=pg.values, int_ptr=int_ptr,
                int_rows=np.concatenate(sets) if sets else np.zeros(0, dtype=np.int64),
                col_ptr=col_ptr,
                col_ids=np.concatenate(col_lists) if col_lists else np.zeros(0, dtype=np.int64),
                aii_ptr=aii_ptr, aii_col=aii_col, aii_src=aii_src, aig_ptr=aig_ptr,
                aig_col=aig_col, aig_src=aig_src)


def check_extension_residual(a: CsrMatrix, desc: dict, pg: CsrMatrix, col_resid: np.ndarray):
    """Reference check (coarse_space.py:182-202): interior rows of A Phi must
    vanish to 1e-10 * ||A||_inf * max|phi_Gamma column|."""
    n_cols = desc["n_c"]
    if n_cols == 0:
        return
    resid = np.zeros(n_cols)
    np.maximum.at(resid, desc["col_ids"], col_resid)
    row_sums = np.zeros(a.nrows)
    np.add.at(row_sums, a.row_ids(), np.abs(a.values))
    anorm = row_sums.max() if a.nrows else 0.0
    gnorm = np.zeros(n_cols)
    if pg.nnz:
        np.maximum.at(gnorm, pg.col_idx, np.abs(pg.values))
    bad = np.flatnonzero(resid > 1e-10 * anorm * np.maximum(gnorm, 1e-300))
    if bad.size:
        raise ArithmeticError(
            f"energy-minimizing extension failed the residual check for "
            f"column {int(bad[0])} ({resid[bad[0]]:.3e})")


def assemble_phi(n: int, desc: dict, pg: CsrMatrix, panels: np.ndarray) -> CsrMatrix:
    """Host CsrMatrix of Phi: interface rows bitwise from the basis, interior
    rows from the device panels with exact zeros pruned (coarse_space.py:164-176)."""
    n_cols = desc["n_c"]
    rows = [desc["gamma_rows"][pg.row_ids()]]
    cols = [pg.col_idx]
    vals = [pg.values]
    int_ptr, col_ptr = desc["int_ptr"], desc["col_ptr"]
    off = 0
    for s in range(int_ptr.size - 1):
        ni = int(int_ptr[s + 1] - int_ptr[s])
        k = int(col_ptr[s + 1] - col_ptr[s])
        if ni == 0 or k == 0:
            continue
        blk = panels[off:off + ni * k].reshape(k, ni)   # column-major panel
        off += ni * k
        cc, rr = np.nonzero(blk)
        rows.append(desc["int_rows"][int_ptr[s] + rr])
        cols.append(desc["col_ids"][col_ptr[s] + cc])
        vals.append(blk[cc, rr])
    return CsrMatrix.from_coo(n, n_cols, np.concatenate(rows), np.concatenate(cols),
                              np.concatenate(vals))


def coarse_matrix(a: CsrMatrix, phi: CsrMatrix) -> CsrMatrix:
    """Galerkin product Phi^T A Phi via two sparse products (coarse_space.py:205-207)."""
    return spgemm(transpose(phi), spgemm(a, phi))


def reproduction_coefficients(column_map, n_nullspace: int, coeffs=None) -> np.ndarray:
    """Coefficients c with Phi @ c[:, j] reproducing null-space column j
    (coarse_space.py:210-227)."""
    c = np.zeros((len(column_map), n_nullspace))
    if coeffs is None:
        for i, (_, j) in enumerate(column_map):
            c[i, j] = 1.0
        return c
    row = 0
    for block in coeffs:
        c[row:row + block.shape[0], :] = block
        row += block.shape[0]
    if row != len(column_map):
        raise ValueError("coefficient blocks do not match the column map")
    return c


def extend_on_device(pre, a_dev, a: CsrMatrix, structure, basis, sets, lazy_phi: bool = False):
    """Bind the coarse structure to a device preconditioner, run the batched
    extension, check it, and return (phi, column_map, desc); with lazy_phi,
    phi is a thunk assembling the host CsrMatrix on demand (the solve path
    only uses the device panels)."""
    column_map, pg = coarse_columns(structure, basis)
    if not column_map:
        raise ValueError("coarse space is empty; use use_coarse=False")
    desc = coarse_desc(a, structure, pg, len(column_map), sets)
    pre.set_coarse(desc)
    _, col_resid = pre.extend(a_dev, int(desc["col_ptr"][-1]), EXTENSION_TOL,
                              EXTENSION_MAX_ITERS)
    check_extension_residual(a, desc, pg, col_resid)
    if lazy_phi:
        return (lambda: assemble_phi(structure.n, desc, pg, pre.panels())), column_map, desc
    phi = assemble_phi(structure.n, desc, pg, pre.panels())
    return phi, column_map, desc


def harmonic_extension(a: CsrMatrix, structure: InterfaceStructure, basis: InterfaceBasis,
                       interiors: InteriorBlocks):
    """Phi on the GPU (coarse_space.py:130-179). Returns (phi, column_map)."""
    from . import device
    from .schwarz import empty_local_plan
    plan = device.Plan(empty_local_plan(structure.n, len(interiors.sets)))
    pre = device.Precond(plan, np.float64, 1)
    a64 = a if a.dtype == np.float64 else CsrMatrix(a.nrows, a.ncols, a.row_ptr, a.col_idx,
                                                    a.values.astype(np.float64))
    phi, column_map, _ = extend_on_device(pre, device.DeviceCsr(a64), a64, structure, basis,
                                          interiors.sets)
    return phi, column_map


def factor_interiors(a: CsrMatrix, part: Partition, structure: InterfaceStructure,
                     ordering_kind: str = "nested_dissection") -> InteriorBlocks:
    """Interior index sets; the GPU extension needs no interior factors."""
    return InteriorBlocks(interior_sets(part, structure), None)


def build_coarse_basis(a: CsrMatrix, part: Partition, structure: InterfaceStructure,
                       nullspace: np.ndarray,
                       ordering_kind: str = "nested_dissection") -> CoarseBasis:
    basis = interface_basis(nullspace, structure)
    phi, column_map = harmonic_extension(a, structure, basis,
                                         factor_interiors(a, part, structure, ordering_kind))
    return CoarseBasis(phi, coarse_matrix(a, phi), column_map)
