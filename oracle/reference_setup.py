"""ORACLE -- test infrastructure, NOT the product (see oracle/__init__.py).

Self-contained CPU restatement of the reference's SETUP for box-partitioned
3D Laplace problems (numpy + scipy + liboracle only; nothing from the
product package or its host runtime is imported), so that
`bench.py --impl reference` times the reference's CPU path on inputs it
built itself:

* assemble_laplace3d        -- model_problems.py:90-124 (7-point, Dirichlet,
                               1/h^2 = (n_a - 1)^2 per axis, z = 1/sqrt(n))
* box_partition             -- decomposition.py:114-137 (remainders to the
                               leading boxes, s = sx + px (sy + py sz))
* extend_overlap            -- decomposition.py:152-167 (graph layers)
* classify_interface        -- decomposition.py:174-251 (closure sets,
                               connected classes, vertex/edge/face kinds)
* build_components("rgdsw") -- decomposition.py:254-300
* interface_basis           -- coarse_space.py:64-103 (one null-space column)
* harmonic_extension        -- coarse_space.py:130-179 (exact interior solves:
                               here scipy's SuperLU, pruned exact zeros)
* coarse_matrix             -- coarse_space.py:205-207 (Phi^T (A Phi))
* ILU(0) natural-ordering patterns for fast_ilu (local_solvers.py:205-243)

Pinned in tests/test_oracle_golden.py: the decomposition hashes equal the
reference's (golden dec_hash of tests/golden/configs) and the apply agrees
with the pinned oracle.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from types import SimpleNamespace

import numpy as np
import scipy.sparse as sp
import scipy.sparse.csgraph as csg
import scipy.sparse.linalg as spla

from . import oracle as O


class Csr:
    """Minimal CSR value (the fields the oracle kernels read)."""

    def __init__(self, m: sp.csr_matrix):
        m = m.tocsr()
        m.sort_indices()
        self.nrows, self.ncols = m.shape
        self.row_ptr = m.indptr.astype(np.int64)
        self.col_idx = m.indices.astype(np.int64)
        self.values = np.ascontiguousarray(m.data, dtype=np.float64)
        self.scipy = m

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    def row_ids(self):
        return np.repeat(np.arange(self.nrows, dtype=np.int64), np.diff(self.row_ptr))

    def __matmul__(self, x):
        return O.csr_spmv(self, np.ascontiguousarray(x, dtype=np.float64))


def assemble_laplace3d(nx: int, ny: int, nz: int):
    """(A, nullspace) of the reference's Dirichlet 7-point Laplacian."""
    n = nx * ny * nz
    idx = np.arange(n, dtype=np.int64).reshape(nz, ny, nx)
    scale = [float((nx - 1) ** 2), float((ny - 1) ** 2), float((nz - 1) ** 2)]
    rows, cols, vals = [], [], []
    for axis, s in enumerate(scale):
        a = np.moveaxis(idx, 2 - axis, 0)
        lo, hi = a[:-1].ravel(), a[1:].ravel()
        rows += [lo, hi]
        cols += [hi, lo]
        vals += [np.full(lo.size, -s), np.full(lo.size, -s)]
    rows.append(np.arange(n, dtype=np.int64))
    cols.append(np.arange(n, dtype=np.int64))
    vals.append(np.full(n, 2.0 * sum(scale)))
    m = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n)).tocsr()
    return Csr(m), np.full((n, 1), 1.0 / np.sqrt(n))


def _splits(n: int, p: int) -> np.ndarray:
    base, rem = divmod(n, p)
    return np.concatenate([[0], np.cumsum([base + 1] * rem + [base] * (p - rem))])


def box_partition(nx, ny, nz, px, py, pz) -> np.ndarray:
    ix = np.searchsorted(_splits(nx, px), np.arange(nx), side="right") - 1
    iy = np.searchsorted(_splits(ny, py), np.arange(ny), side="right") - 1
    iz = np.searchsorted(_splits(nz, pz), np.arange(nz), side="right") - 1
    return (ix[None, None, :] + px * (iy[None, :, None] + py * iz[:, None, None])).ravel()


def _graph(a: Csr) -> sp.csr_matrix:
    g = sp.csr_matrix((np.ones(a.col_idx.size, dtype=np.int8), a.col_idx, a.row_ptr),
                      shape=a.shape)
    g.setdiag(0)
    g.eliminate_zeros()
    return g


def extend_overlap(a: Csr, owner: np.ndarray, n_parts: int, layers: int = 1) -> list:
    g = _graph(a)
    sets = []
    for s in range(n_parts):
        mask = owner == s
        for _ in range(layers):
            mask = mask | (g @ mask.astype(np.int8) > 0)
        sets.append(np.flatnonzero(mask).astype(np.int64))
    return sets


def classify_interface(a: Csr, owner: np.ndarray):
    """Interior / interface dofs, multiplicities and the raw classes
    (dofs, kind, subdomain set), sorted by first dof."""
    g = _graph(a)
    n = owner.size
    deg = np.diff(g.indptr)
    width = int(deg.max(initial=0)) + 1
    own = np.full((n, width), -1, dtype=np.int64)
    own[:, 0] = owner
    rows = np.repeat(np.arange(n), deg)
    slot = np.arange(g.indices.size) - np.repeat(g.indptr[:-1], deg) + 1
    own[rows, slot] = owner[g.indices]
    own.sort(axis=1)
    dup = np.zeros_like(own, dtype=bool)
    dup[:, 1:] = own[:, 1:] == own[:, :-1]
    own[dup] = -1
    own.sort(axis=1)                       # unique owners, -1 padding first
    card = (own >= 0).sum(axis=1)
    iface = np.flatnonzero(card >= 2)
    keys, cls = np.unique(own[iface], axis=0, return_inverse=True)
    cls = cls.ravel()
    # connected pieces of each class over graph edges inside the class
    cls_of = np.full(n, -1, dtype=np.int64)
    cls_of[iface] = cls
    gi = g.tocoo()
    same = (cls_of[gi.row] >= 0) & (cls_of[gi.row] == cls_of[gi.col])
    sub = sp.coo_matrix((np.ones(int(same.sum())), (gi.row[same], gi.col[same])), shape=(n, n))
    _, lab = csg.connected_components(sub, directed=False)
    piece_key = cls_of * (n + 1) + lab
    pk, piece = np.unique(piece_key[iface], return_inverse=True)
    piece = piece.ravel()
    npieces = pk.size
    piece_of = np.full(n, -1, dtype=np.int64)
    piece_of[iface] = piece
    pcls = np.empty(npieces, dtype=np.int64)
    pcls[piece] = cls
    # adjacency between pieces (maximality clause)
    pr, pc = piece_of[gi.row], piece_of[gi.col]
    m = (pr >= 0) & (pc >= 0) & (pr != pc)
    adj = sp.coo_matrix((np.ones(int(m.sum())), (pr[m], pc[m])), shape=(npieces, npieces)).tocsr()
    sets = [frozenset(int(v) for v in keys[c] if v >= 0) for c in range(keys.shape[0])]
    comps = []
    order = np.argsort(piece, kind="stable")
    bounds = np.searchsorted(piece[order], np.arange(npieces + 1))
    for q in range(npieces):
        nodes = np.sort(iface[order[bounds[q]:bounds[q + 1]]])
        key = sets[pcls[q]]
        if len(key) == 2:
            kind = "face"
        elif len(key) >= 5:
            kind = "vertex"
        else:
            nb = adj.indices[adj.indptr[q]:adj.indptr[q + 1]]
            kind = "edge" if any(key < sets[pcls[t]] for t in nb) else "vertex"
        comps.append(SimpleNamespace(dofs=nodes.astype(np.int64), kind=kind,
                                     weights=np.ones(nodes.size), subdomains=key))
    comps.sort(key=lambda c: int(c.dofs[0]))
    mask = np.zeros(n, dtype=bool)
    mask[iface] = True
    return SimpleNamespace(n=n, interior=np.flatnonzero(~mask).astype(np.int64),
                           interface=iface.astype(np.int64), multiplicity=card[iface].astype(np.int64),
                           components=comps)


def build_rgdsw(st):
    vertices = [c for c in st.components if c.kind == "vertex"]
    gathered = [[] for _ in vertices]
    for c in st.components:
        parents = [t for t, v in enumerate(vertices) if c.subdomains <= v.subdomains]
        if not parents:
            raise ValueError("interface class covered by no vertex class")
        w = 1.0 / len(parents)
        for t in parents:
            gathered[t].append((c.dofs, w))
    comps = []
    for v, chunks in zip(vertices, gathered):
        dofs = np.concatenate([d for d, _ in chunks])
        weights = np.concatenate([np.full(d.size, w) for d, w in chunks])
        o = np.argsort(dofs)
        comps.append(SimpleNamespace(dofs=dofs[o], kind="vertex", weights=weights[o],
                                     subdomains=v.subdomains))
    comps.sort(key=lambda c: int(c.dofs[0]))
    return SimpleNamespace(n=st.n, interior=st.interior, interface=st.interface,
                           multiplicity=st.multiplicity, components=comps)


def harmonic_extension(a: Csr, owner, st, nullspace, threads: int = 1):
    """Phi (scipy CSR) with one column per component (null space of one
    column: Laplace), interior rows by exact interior solves."""
    z = np.asarray(nullspace, dtype=np.float64)
    gamma = st.interface
    n_cols = len(st.components)
    rows, cols, vals = [], [], []
    pg_r, pg_c, pg_v = [], [], []
    for t, c in enumerate(st.components):
        v = c.weights * z[c.dofs, 0]
        rows.append(c.dofs)
        cols.append(np.full(c.dofs.size, t))
        vals.append(v)
        pg_r.append(np.searchsorted(gamma, c.dofs))
        pg_c.append(np.full(c.dofs.size, t))
        pg_v.append(v)
    phi_g = sp.csr_matrix((np.concatenate(pg_v), (np.concatenate(pg_r), np.concatenate(pg_c))),
                          shape=(gamma.size, n_cols))
    on_g = np.zeros(st.n, dtype=bool)
    on_g[gamma] = True
    global _EXT
    _EXT = (a.scipy, owner, on_g, gamma, phi_g)
    # SuperLU holds the GIL: subdomains in forked worker processes
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    nsub = int(owner.max()) + 1
    if threads > 1:
        ex = ProcessPoolExecutor(max_workers=threads, mp_context=mp.get_context("fork"))
    else:
        ex = ThreadPoolExecutor(max_workers=1)
    with ex:
        for part in ex.map(_extend_one, range(nsub)):
            if part is not None:
                rows.append(part[0])
                cols.append(part[1])
                vals.append(part[2])
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(st.n, n_cols)).tocsr()


_EXT = None


def _extend_one(s):
    """Interior rows of Phi for subdomain s: A_II phi_I = -A_IG Phi_G."""
    A, owner, on_g, gamma, phi_g = _EXT
    dofs = np.flatnonzero((owner == s) & ~on_g)
    if dofs.size == 0:
        return None
    rhs = -(A[dofs][:, gamma] @ phi_g).toarray()
    need = np.flatnonzero(np.abs(rhs).sum(axis=0) > 0)
    if need.size == 0:
        return None
    lu = spla.splu(A[dofs][:, dofs].tocsc(), permc_spec="MMD_AT_PLUS_A")
    sol = lu.solve(np.ascontiguousarray(rhs[:, need]))
    rr, cc = np.nonzero(sol)
    return dofs[rr], need[cc], sol[rr, cc]


_LOCAL = None


def _local_one(i):
    """FastILU(0) factors of overlap block i (natural ordering)."""
    A, sets, sweeps = _LOCAL
    d = sets[i]
    blk = Csr(A[d][:, d])
    sym = ilu0_natural(blk)
    lv, uv, _ = O.fast_ilu(blk, sym, sweeps)
    return sym, lv, uv


def ilu0_natural(block: Csr):
    """Symbolic ILU(0), natural ordering: L strictly lower, U with the
    diagonal first in each row (local_solvers.py:18-20)."""
    n = block.nrows
    r = block.row_ids()
    c = block.col_idx
    lo = c < r
    up = c > r
    l_ptr = np.concatenate([[0], np.cumsum(np.bincount(r[lo], minlength=n))]).astype(np.int64)
    u_cnt = np.bincount(r[up], minlength=n) + 1
    u_ptr = np.concatenate([[0], np.cumsum(u_cnt)]).astype(np.int64)
    u_idx = np.empty(u_ptr[-1], dtype=np.int64)
    u_idx[u_ptr[:-1]] = np.arange(n)
    rest = np.ones(u_ptr[-1], dtype=bool)
    rest[u_ptr[:-1]] = False
    u_idx[rest] = c[up]
    return SimpleNamespace(n=n, l_ptr=l_ptr, l_idx=c[lo].astype(np.int64), u_ptr=u_ptr,
                           u_idx=u_idx, ordering=SimpleNamespace(perm=np.arange(n, dtype=np.int64)))


class IndependentSchwarz:
    """Two-level rGDSW with fast_ilu(0, sweeps, iters) local solves and the
    natural ordering (C2's configuration), built without the product."""

    def __init__(self, nx, ny, nz, px, py, pz, sweeps=3, iters=5, threads=1):
        self.a, self.z = assemble_laplace3d(nx, ny, nz)
        self.owner = box_partition(nx, ny, nz, px, py, pz)
        nparts = px * py * pz
        self.sets = extend_overlap(self.a, self.owner, nparts, 1)
        self.structure = build_rgdsw(classify_interface(self.a, self.owner))
        self.iters = iters
        A = self.a.scipy
        global _LOCAL
        _LOCAL = (A, self.sets, sweeps)
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor
        if threads > 1:   # numpy work between the C sweeps holds the GIL
            ex = ProcessPoolExecutor(max_workers=threads, mp_context=mp.get_context("fork"))
        else:
            ex = ThreadPoolExecutor(max_workers=1)
        with ex:
            self.local = list(ex.map(_local_one, range(nparts)))
        phi = harmonic_extension(self.a, self.owner, self.structure, self.z, threads)
        self.phi = Csr(phi)
        self.phi_t = Csr(phi.T.tocsr())
        self.a0 = (phi.T @ (A @ phi)).tocsc()
        self.a0_lu = spla.splu(self.a0)
        self.threads = max(1, threads)
        self._pool = ThreadPoolExecutor(max_workers=self.threads) if self.threads > 1 else None

    def local_solve(self, i, b):
        sym, lv, uv = self.local[i]
        return O.jacobi_solve(sym, lv, uv, b, self.iters)

    def apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        zc = O.csr_spmv(self.phi, self.a0_lu.solve(O.csr_spmv(self.phi_t, r)))
        z = np.zeros_like(r)
        if self._pool is not None:
            ys = list(self._pool.map(lambda i: self.local_solve(i, r[self.sets[i]]),
                                     range(len(self.sets))))
        else:
            ys = (self.local_solve(i, r[d]) for i, d in enumerate(self.sets))
        for d, y in zip(self.sets, ys):
            z[d] += y
        return zc + z


def decomposition_hash(sets, st) -> str:
    """tests/cases.decomposition_hash over these structures."""
    import hashlib
    h = hashlib.sha256()
    for s in sets:
        h.update(np.asarray(s, np.int64).tobytes())
    for arr in (st.interior, st.interface, st.multiplicity):
        h.update(np.asarray(arr, np.int64).tobytes())
    for c in st.components:
        h.update(np.asarray(c.dofs, np.int64).tobytes())
        h.update(np.asarray(c.weights, np.float64).tobytes())
        h.update(c.kind.encode())
        h.update(np.array(sorted(c.subdomains), np.int64).tobytes())
    return h.hexdigest()
