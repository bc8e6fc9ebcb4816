"""Per-rank setup of the sharded weak-scaling problem from the rank's own
z-window: no rank assembles or decomposes the global
N x 2M system.

The global problem is the reference's 7-point Dirichlet Laplacian on an
n_xy x n_xy x (n_z_per_rank * N) grid with boxes_xy^2 x (boxes_z_per_rank * N)
boxes (model_problems.py:90-124, decomposition.py:114-137), sharded in
z-slabs of whole box layers (dist.slab_subdomains). Rank r builds only the
node planes [W0, W1) around its slab: its own box layers plus a margin of
two box layers and three planes on each side. That margin makes every object
the rank needs identical to the global one:

* operator rows, overlap sets (one node layer) and interior sets of the
  rank's subdomains -- a node layer away from the slab;
* the raw interface classes (closure sets need the neighbours' owners, one
  plane) and the rGDSW components touching the rank's extended rows: a
  component gathers the classes around one vertex class, so it reaches at
  most one box layer beyond the vertex, and a vertex whose component touches
  the slab's halo lies at most one box layer away from it;
* classes touching the untrusted window planes (the three next to a window
  edge that is not a global boundary) are dropped before the rGDSW gather,
  and only components inside the trusted planes are kept.

Global coarse-column numbering (components sorted by first dof, ties in
vertex-class order: decomposition.py:243, 292): each rank contributes the
keys (first dof, vertex-class first dof) of the components whose first dof
it owns; one all-gather gives the global order, the rank's components look
their column up by key.

Window row w has global id w + offset (x-fastest numbering: a z-window is a
contiguous row range). The setup work and memory per rank depend only on
the slab size, not on N.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .decomposition import (Decomposition, InterfaceComponent, InterfaceStructure,
                            OverlapSets, Partition, _axis_bounds, classify_interface,
                            extend_overlap)
from .sparse_core import CsrMatrix


@dataclass
class SlabProblem:
    a: CsrMatrix               # window operator (window-local numbering)
    nullspace: np.ndarray      # window rows of the global null space
    dec: Decomposition         # window-local; overlap sets of the rank's subdomains only
    offset: int                # global id of window row 0
    n_global: int
    subs: np.ndarray           # the rank's subdomains (global ids)
    g0: int                    # owned rows [g0, g1), window-local
    g1: int
    comp_col: np.ndarray       # global coarse column of each kept component
    n_c: int                   # global coarse dimension


def _window_laplace(nx, ny, nz_global, w0, w1):
    """Rows of the global Dirichlet 7-point Laplacian for the node planes
    [w0, w1) (same values as model_problems.assemble_laplace3d on the full
    grid; neighbours outside the window are cut)."""
    nzw = w1 - w0
    n = nx * ny * nzw
    scale = [float((nx - 1) ** 2), float((ny - 1) ** 2), float((nz_global - 1) ** 2)]
    idx = np.arange(n, dtype=np.int64).reshape(nzw, ny, nx)
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
    return CsrMatrix.from_coo(n, n, np.concatenate(rows), np.concatenate(cols),
                              np.concatenate(vals))


def _partition(owner: np.ndarray, n_parts: int) -> Partition:
    """A window's partition: global subdomain ids, most of them absent (the
    global Partition's every-subdomain-present check does not apply)."""
    p = object.__new__(Partition)
    p.n_parts, p.owner, p.dofs_per_node, p.boxes = n_parts, owner.astype(np.int64), 1, None
    return p


def _rgdsw(components: list) -> list:
    """decomposition.build_components(..., "rgdsw") on a list of raw classes
    (no global partition-of-unity assertion: dropped window-edge classes)."""
    vertices = [c for c in components if c.kind == "vertex"]
    gathered = [[] for _ in vertices]
    for c in components:
        parents = [t for t, v in enumerate(vertices) if c.subdomains <= v.subdomains]
        if not parents:
            continue        # only possible next to a dropped window-edge class
        w = 1.0 / len(parents)
        for t in parents:
            gathered[t].append((c.dofs, w))
    out = []
    for v, chunks in zip(vertices, gathered):
        dofs = np.concatenate([d for d, _ in chunks])
        weights = np.concatenate([np.full(d.size, w) for d, w in chunks])
        o = np.argsort(dofs)
        out.append((InterfaceComponent(dofs[o], "vertex", weights[o], v.subdomains),
                    int(v.dofs[0])))
    # sorted by first dof, ties in vertex-class order (the reference's stable
    # sort): the pair (first dof, vertex-class first dof) is the global key
    out.sort(key=lambda cv: (int(cv[0].dofs[0]), cv[1]))
    return out


def build_slab_problem(n_xy: int, n_z_per_rank: int, boxes_xy: int, boxes_z_per_rank: int,
                       nranks: int, rank: int, group=None, gather=None) -> SlabProblem:
    """`gather(list) -> list of every rank's list` (default: all_gather_object
    over torch.distributed when initialized)."""
    import torch.distributed as tdist

    nx = ny = n_xy
    nz = n_z_per_rank * nranks
    pz = boxes_z_per_rank * nranks
    n_parts = boxes_xy * boxes_xy * pz
    bz = _axis_bounds(nz, pz)
    l0, l1 = rank * pz // nranks, (rank + 1) * pz // nranks
    z0, z1 = int(bz[l0]), int(bz[l1])
    h = int(np.diff(bz).max())
    margin = 2 * h + 3
    w0, w1 = max(0, z0 - margin), min(nz, z1 + margin)
    plane = nx * ny
    offset = w0 * plane
    a = _window_laplace(nx, ny, nz, w0, w1)
    # owners of the window nodes (global box ids)
    bx = _axis_bounds(nx, boxes_xy)
    ix = np.searchsorted(bx, np.arange(nx), side="right") - 1
    iy = np.searchsorted(bx, np.arange(ny), side="right") - 1
    iz = np.searchsorted(bz, np.arange(w0, w1), side="right") - 1
    owner = (ix[None, None, :] + boxes_xy * (iy[None, :, None] + boxes_xy * iz[:, None, None])).ravel()
    part = _partition(owner, n_parts)
    per_layer = boxes_xy * boxes_xy
    subs = np.arange(l0 * per_layer, l1 * per_layer, dtype=np.int64)
    overlap = extend_overlap(a, part, 1, subdomains=subs)
    raw = classify_interface(a, part)
    # trusted planes: three planes inside each window edge that is not a
    # global boundary (closure sets there miss neighbours)
    t0 = (w0 + 3 if w0 > 0 else 0) - w0
    t1 = (w1 - 3 if w1 < nz else nz) - w0
    lo_row, hi_row = t0 * plane, t1 * plane

    def inside(d):
        return d.size > 0 and d[0] >= lo_row and d[-1] < hi_row

    g0, g1 = (z0 - w0) * plane, (z1 - w0) * plane
    band0, band1 = max(0, g0 - 2 * plane), g1 + 2 * plane

    def touches_band(d):
        return bool(np.any((d >= band0) & (d < band1)))

    # components touching the slab (+ two planes) are complete in the
    # trusted planes; farther ones may miss dropped window-edge classes
    classes = [c for c in raw.components if inside(c.dofs)]
    kept = [(c, vf) for c, vf in _rgdsw(classes) if inside(c.dofs) and touches_band(c.dofs)]
    comps = [c for c, _ in kept]
    iface = raw.interface
    keep_if = (iface >= lo_row) & (iface < hi_row)
    structure = InterfaceStructure(a.nrows, raw.interior, iface[keep_if], raw.multiplicity[keep_if],
                                   comps, "rgdsw")
    # global coarse columns: the first dofs of the components this rank owns
    keys = [(int(c.dofs[0]) + offset, vf + offset) for c, vf in kept]
    mine = [k for k in keys if g0 + offset <= k[0] < g1 + offset]
    if gather is None and tdist.is_available() and tdist.is_initialized() and nranks > 1:
        def gather(x):
            out = [None] * nranks
            tdist.all_gather_object(out, x, group=group)
            return out
    lists = gather(mine) if gather is not None else [mine]
    allkeys = sorted(tuple(k) for v in lists for k in v)
    col_of = {k: i for i, k in enumerate(allkeys)}
    comp_col = np.array([col_of.get(k, -1) for k in keys], dtype=np.int64)
    n_global = nx * ny * nz
    nullspace = np.full((a.nrows, 1), 1.0 / np.sqrt(n_global))
    return SlabProblem(a, nullspace, Decomposition(part, overlap, structure), offset, n_global,
                       subs, g0, g1, comp_col, len(allkeys))
