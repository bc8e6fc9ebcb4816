"""Sharded solve: one process per GPU, subdomains split over ranks
(SURVEY.md §8(e)).

The subdomain boxes are split into z-slabs; with the x-fastest node
numbering every rank then owns a contiguous global row range and a
contiguous range of subdomain ids (decomposition.py:118-136). A rank's
vectors live in an extended local layout [e0, e1): its owned rows plus the
halo rows its operator rows, overlapped subdomains and scatter touch (one
node plane per neighbour for overlap 1). Everything else is the single-GPU
machinery on that layout; libgdsw's peer-memory collectives (gdsw_dist)
refresh halos, return overlapped partial sums to their owners in subdomain
order, and all-reduce the coarse right-hand side and the fused GMRES block.

Host bootstrap (IPC handle exchange, the small dense A0 partial sums) goes
through torch.distributed (gloo); no NCCL is needed on the data path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _host
from .coarse_space import (
    EXTENSION_MAX_ITERS,
    EXTENSION_TOL,
    assemble_phi,
    coarse_columns,
    coarse_desc,
    interface_basis,
    interior_sets,
)
from .local_solvers import LocalFactorization, build_symbolic, host_numeric, make_ordering
from .local_solvers import _pivot_error, numeric_lu, symbolic_lu
from .sparse_core import CsrMatrix, convert_precision, extract_submatrix


@dataclass
class Shard:
    rank: int
    nranks: int
    n: int
    g0: int
    g1: int
    e0: int
    e1: int
    subs: np.ndarray
    nbrs: list = field(default_factory=list)  # (rank, send_lo, send_hi, recv_lo, recv_hi), ext-local

    @property
    def n_ext(self) -> int:
        return self.e1 - self.e0

    @property
    def n_own(self) -> int:
        return self.g1 - self.g0

    @property
    def own_off(self) -> int:
        return self.g0 - self.e0


def slab_subdomains(part, nranks: int) -> list:
    """Contiguous z-layers of boxes per rank (ids s = sx + px*(sy + py*sz))."""
    if not part.boxes:
        raise ValueError("sharding needs a box partition")
    zr = sorted({b[2] for b in part.boxes})
    pz = len(zr)
    if pz < nranks:
        raise ValueError(f"cannot split {pz} subdomain layers over {nranks} ranks")
    per_layer = part.n_parts // pz
    out = []
    for r in range(nranks):
        l0, l1 = r * pz // nranks, (r + 1) * pz // nranks
        out.append(np.arange(l0 * per_layer, l1 * per_layer, dtype=np.int64))
    return out


def plan_shards(a: CsrMatrix, dec, nranks: int) -> list:
    """Every rank's layout (computed identically on every rank)."""
    part = dec.partition
    subs_by_rank = slab_subdomains(part, nranks)
    sets = dec.overlap.sets
    own, ext = [], []
    for subs in subs_by_rank:
        rows = np.flatnonzero(np.isin(part.owner, subs))
        if rows.size == 0 or rows[-1] - rows[0] + 1 != rows.size:
            raise ValueError("a rank's rows are not contiguous (shard along z only)")
        g0, g1 = int(rows[0]), int(rows[-1]) + 1
        lo = min([g0] + [int(sets[s][0]) for s in subs])
        hi = max([g1] + [int(sets[s][-1]) + 1 for s in subs])
        cols = a.col_idx[a.row_ptr[g0]:a.row_ptr[g1]]
        if cols.size:
            lo, hi = min(lo, int(cols.min())), max(hi, int(cols.max()) + 1)
        own.append((g0, g1))
        ext.append((lo, hi))
    return [Shard(r, nranks, a.nrows, own[r][0], own[r][1], ext[r][0], ext[r][1], subs_by_rank[r],
                  _neighbours(r, own, ext)) for r in range(nranks)]


def _neighbours(r: int, own: list, ext: list) -> list:
    """Halo exchange ranges of rank r from every rank's owned / extended row
    ranges (one global numbering): (q, send_lo, send_hi, recv_lo, recv_hi)
    relative to r's extended start."""
    (g0, g1), (e0, e1) = own[r], ext[r]
    nbrs = []
    for q in range(len(own)):
        if q == r:
            continue
        (q0, q1), (f0, f1) = own[q], ext[q]
        recv = (max(e0, q0), min(e1, q1))   # rows q owns in my halo
        send = (max(g0, f0), min(g1, f1))   # rows I own in q's halo
        if recv[1] > recv[0] or send[1] > send[0]:
            if send[1] <= send[0]:
                send = (g0, g0)
            if recv[1] <= recv[0]:
                recv = (e0, e0)
            nbrs.append((q, send[0] - e0, send[1] - e0, recv[0] - e0, recv[1] - e0))
    return nbrs


def plan_slab_shard(sp, nranks: int, rank: int, gather=None) -> Shard:
    """This rank's layout from its slab problem (slab.py), in the window's
    numbering; the neighbour ranges come from every rank's (global) row
    ranges, exchanged by `gather` (default: all_gather_object)."""
    a, sets = sp.a, sp.dec.overlap.sets
    g0, g1 = sp.g0, sp.g1
    lo = min([g0] + [int(sets[s][0]) for s in sp.subs])
    hi = max([g1] + [int(sets[s][-1]) + 1 for s in sp.subs])
    cols = a.col_idx[a.row_ptr[g0]:a.row_ptr[g1]]
    if cols.size:
        lo, hi = min(lo, int(cols.min())), max(hi, int(cols.max()) + 1)
    mine = (g0 + sp.offset, g1 + sp.offset, lo + sp.offset, hi + sp.offset)
    if gather is None and nranks > 1:
        import torch.distributed as tdist

        def gather(x):
            out = [None] * nranks
            tdist.all_gather_object(out, x)
            return out
    allr = gather(mine) if gather is not None else [mine]
    own = [(t[0], t[1]) for t in allr]
    ext = [(t[2], t[3]) for t in allr]
    return Shard(rank, nranks, a.nrows, g0, g1, lo, hi, np.asarray(sp.subs), _neighbours(rank, own, ext))


def _range_rows(lo, hi):
    return np.arange(lo, hi, dtype=np.int64)


class DistPreconditioner:
    """This rank's share of the two-level preconditioner on the GPU."""

    def __init__(self, a: CsrMatrix, dec, config, nullspace, shard: Shard, pg_group=None,
                 slab=None):
        """`slab` (slab.SlabProblem): a, dec, nullspace and shard are the
        rank's window (window numbering); coarse columns and the residual
        check scales are global (the slab's column ids, max-reductions)."""
        self.slab = slab
        import torch.distributed as tdist

        from . import device
        from .schwarz import _gpu_lu_pays, _install_local_factor, _local_factor_pays
        self.shard = sh = shard
        spec = config.local
        single = config.precision == "single"
        ext = _range_rows(sh.e0, sh.e1)
        if single:
            a32 = convert_precision(a, np.float32)
            local_src = a32
            coarse_src = CsrMatrix(a.nrows, a.ncols, a.row_ptr, a.col_idx,
                                   a32.values.astype(np.float64))
        else:
            local_src = coarse_src = a
        a_ext = extract_submatrix(coarse_src, ext, ext)          # f64 values for setup
        loc_ext = extract_submatrix(local_src, ext, ext)
        sets = [dec.overlap.sets[s] - sh.e0 for s in sh.subs]
        syms = []
        for d in sets:
            blk = extract_submatrix(loc_ext, d, d)
            syms.append(build_symbolic(blk, spec, make_ordering(blk, config.ordering)))
        self.local_symbolics = syms
        from .schwarz import local_plan_arrays
        self.plan = device.Plan(local_plan_arrays(sh.n_ext, sets, syms, spec.method, a_ext))
        vdt = np.float32 if single else np.float64
        self.pre = device.Precond(self.plan, vdt, spec.trisolve_iters)
        self.layout = device.DistLayout(sh.rank, sh.nranks, sh.n_ext, sh.own_off,
                                        sh.own_off + sh.n_own, sh.nbrs)
        handles = [None] * sh.nranks
        tdist.all_gather_object(handles, self.layout.ipc_handle(), group=pg_group)
        self.layout.open_peers(handles)
        a_ext_dev = device.DeviceCsr(a_ext)
        if spec.method == "fast_ilu":
            self.sweep_residuals = self.pre.fastilu(a_ext_dev, spec.factor_sweeps, len(sets))
        elif self.plan.has_block_pattern and _gpu_lu_pays(spec, syms):
            # the single-GPU numeric LU / ILU(k) kernel on this rank's blocks
            shift = spec.diag_shift if spec.method == "ilu_k" else 0.0
            fail = self.pre.lu_numeric(a_ext_dev, shift, len(sets))
            bad = np.flatnonzero(fail)
            if bad.size:
                i = int(bad[0])
                err = _pivot_error(syms[i], int(fail[i]))
                raise np.linalg.LinAlgError(
                    f"local matrix of subdomain {int(sh.subs[i])} failed to factor: {err}")
        else:
            lvs, uvs = [], []
            shift = spec.diag_shift if spec.method == "ilu_k" else 0.0
            for i, (d, sym) in enumerate(zip(sets, syms)):
                try:
                    lv, uv = host_numeric(extract_submatrix(loc_ext, d, d), sym, shift)
                except np.linalg.LinAlgError as err:
                    raise np.linalg.LinAlgError(
                        f"local matrix of subdomain {int(sh.subs[i])} failed to factor: {err}"
                    ) from err
                lvs.append(lv)
                uvs.append(uv)
            self.pre.set_factors(np.concatenate(lvs).astype(vdt), np.concatenate(uvs).astype(vdt))
        if spec.method == "exact_lu" and _local_factor_pays(syms):
            _install_local_factor(self.pre, self.plan, syms,
                                  on_device=self.plan.has_block_pattern and _gpu_lu_pays(spec, syms))
        self.coarse_n = 0
        if config.use_coarse:
            self._coarse(a, coarse_src, a_ext, a_ext_dev, dec, nullspace, config, single,
                         pg_group)
        device.precond_set_dist(self.pre, self.layout)
        own = _range_rows(sh.g0, sh.g1)
        self.a_own = device.DeviceCsr(extract_submatrix(a, own, ext))

    @property
    def a0_factorization(self):
        """The reference's sparse LU of A0, built on first access when the
        device solve uses the factored partitioned inverse."""
        if callable(self._a0_fac):
            self._a0_fac = self._a0_fac()
        return self._a0_fac

    def _coarse(self, a, coarse_src, a_ext, a_ext_dev, dec, nullspace, config, single, group):
        sh = self.shard
        structure = dec.structure
        basis = interface_basis(nullspace, structure)
        column_map, pg = coarse_columns(structure, basis)
        if not column_map:
            raise ValueError("coarse space is empty; use use_coarse=False")
        n_c = len(column_map)
        if self.slab is not None:
            # the window's components carry their GLOBAL coarse columns (one
            # per component: scalar null space)
            if any(len(k) != 1 for k in basis.kept):
                raise ValueError("slab setup supports one null-space column per component")
            col = np.asarray(self.slab.comp_col, dtype=np.int64)
            if np.any(col < 0):
                raise ValueError("slab setup: a window component has no global coarse column")
            n_c = int(self.slab.n_c)
            pg = CsrMatrix(pg.nrows, n_c, pg.row_ptr, col[pg.col_idx], pg.values)
        gamma = structure.interface
        mine = (gamma >= sh.g0) & (gamma < sh.g1)
        in_ext = (gamma >= sh.e0) & (gamma < sh.e1)
        pg_rows = np.flatnonzero(mine)
        pg_own = extract_submatrix(pg, pg_rows, np.arange(pg.ncols))
        isets = [d - sh.e0 for d in interior_sets(dec.partition, structure, sh.subs)]
        g_own = gamma[mine] - sh.e0
        g_ext = gamma[in_ext] - sh.e0
        for d in isets:   # interiors only couple to interface rows this rank owns
            if extract_submatrix(a_ext, d, g_ext).nnz != extract_submatrix(a_ext, d, g_own).nnz:
                raise ValueError("an interior couples to an interface row of another rank")
        desc = coarse_desc(a_ext, structure, pg_own, n_c, isets, gamma=g_own)
        self.pre.set_coarse(desc)
        _, col_resid = self.pre.extend(a_ext_dev, int(desc["col_ptr"][-1]), EXTENSION_TOL,
                                       EXTENSION_MAX_ITERS)
        # residual check against the GLOBAL operator / basis scales
        resid = np.zeros(n_c)
        np.maximum.at(resid, desc["col_ids"], col_resid)
        rs = np.zeros(a.nrows)
        np.add.at(rs, a.row_ids(), np.abs(coarse_src.values))
        gnorm = np.zeros(n_c)
        np.maximum.at(gnorm, pg.col_idx, np.abs(pg.values))
        rs_max = rs.max()
        if self.slab is not None and sh.nranks > 1:
            import torch
            import torch.distributed as tdist
            red = torch.from_numpy(np.concatenate([[rs_max], gnorm]))
            tdist.all_reduce(red, op=tdist.ReduceOp.MAX, group=group)
            rs_max, gnorm = float(red[0]), red[1:].numpy()
        bad = np.flatnonzero(resid > 1e-10 * rs_max * np.maximum(gnorm, 1e-300))
        if bad.size:
            raise ArithmeticError(
                f"energy-minimizing extension failed the residual check for column "
                f"{int(bad[0])} ({resid[bad[0]]:.3e})")
        # Phi on the extended rows: my panels + every interface row in range
        phi_own = assemble_phi(sh.n_ext, desc, pg_own, self.pre.panels())
        halo_g = np.flatnonzero(in_ext & ~mine)
        if halo_g.size:
            pgh = extract_submatrix(pg, halo_g, np.arange(pg.ncols))
            r1 = np.concatenate([phi_own.row_ids(), gamma[halo_g][pgh.row_ids()] - sh.e0])
            c1 = np.concatenate([phi_own.col_idx, pgh.col_idx])
            v1 = np.concatenate([phi_own.values, pgh.values])
            phi_ext = CsrMatrix.from_coo(sh.n_ext, n_c, r1, c1, v1)
        else:
            phi_ext = phi_own
        # A0 = Phi^T A Phi on the GPU: my owned rows' share, summed over ranks
        # in rank order by the peer-memory all-reduce (identical everywhere)
        own = _range_rows(sh.g0, sh.g1)
        from . import device
        a_own_src = device.DeviceCsr(extract_submatrix(coarse_src, own, _range_rows(sh.e0, sh.e1)))
        a0 = self.pre.coarse_galerkin(a_own_src, n_c, self.layout)
        if single:
            a0 = convert_precision(a0, np.float32)
        from .coarse_factor import install as _install_coarse
        from .coarse_factor import use_factor
        order = config.ordering
        self._a0_fac = lambda: numeric_lu(a0, symbolic_lu(a0, make_ordering(a0, order)))
        try:
            if not use_factor(a0.nrows):  # the reference's pivot check
                self._a0_fac = self._a0_fac()
            _install_coarse(self.pre, a0)
        except np.linalg.LinAlgError as err:
            raise np.linalg.LinAlgError(f"coarse matrix is singular: {err}") from err
        self.a0 = a0
        self.phi_local = phi_ext
        self.column_map = column_map
        self.coarse_n = n_c

    def solve(self, b_own, cfg, x0_own=None):
        """Sharded native GMRES on device vectors of this rank's owned rows."""
        from . import device
        t = device.torch()
        x = t.zeros_like(b_own) if x0_own is None else x0_own.clone()
        nonzero = x0_own is not None and bool((x0_own != 0).any().item())
        out = device.gmres_dist(self.a_own, self.pre, b_own, x, nonzero, cfg, self.layout)
        return x, out


def build_sharded_problem(n_xy: int, n_z_per_rank: int, boxes_xy: int, boxes_z_per_rank: int,
                          nranks: int):
    """Weak-scaling Laplace problem: (n_xy, n_xy, n_z_per_rank*nranks) nodes,
    (boxes_xy, boxes_xy, boxes_z_per_rank*nranks) boxes."""
    from .decomposition import box_partition, build_components, classify_interface
    from .decomposition import Decomposition, extend_overlap
    from .model_problems import Grid3D, assemble_laplace3d
    prob = assemble_laplace3d(Grid3D(n_xy, n_xy, n_z_per_rank * nranks))
    part = box_partition(prob.grid, boxes_xy, boxes_xy, boxes_z_per_rank * nranks)
    overlap = extend_overlap(prob.a, part, 1)
    structure = build_components(classify_interface(prob.a, part), "rgdsw")
    return prob, Decomposition(part, overlap, structure)


__all__ = ["Shard", "plan_shards", "plan_slab_shard", "slab_subdomains", "DistPreconditioner",
           "build_sharded_problem", "_host"]
