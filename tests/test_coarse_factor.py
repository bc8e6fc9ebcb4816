"""Factored coarse solve (coarse_factor.py): the supernodal partitioned
inverse of the nested-dissection LU of A0, restated level by level on the
host (`solve_host`, the device algorithm's exact task order) against a dense
solve, plus its structural invariants. The device kernels are compared with
the dense A0^-1 path in tests/test_gpu_parity.py."""

import numpy as np
import pytest

from paper_2304_04876_b200.coarse_factor import build_coarse_factor, solve_host
from paper_2304_04876_b200.sparse_core import CsrMatrix


def _grid_matrix(nx, ny, nz, dpn, seed, sym=True):
    """Block 7-point operator on an nx x ny x nz node grid with dpn dofs per
    node (the shape of rGDSW coarse matrices), diagonally dominant."""
    rng = np.random.default_rng(seed)
    nn = nx * ny * nz
    n = nn * dpn
    rows, cols = [], []
    idx = np.arange(nn).reshape(nz, ny, nx)
    pairs = [(idx.ravel(), idx.ravel())]
    for ax in range(3):
        a = np.moveaxis(idx, 2 - ax, 0)
        pairs.append((a[1:].ravel(), a[:-1].ravel()))
        pairs.append((a[:-1].ravel(), a[1:].ravel()))
    for p, q in pairs:
        for i in range(dpn):
            for j in range(dpn):
                rows.append(p * dpn + i)
                cols.append(q * dpn + j)
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = rng.uniform(-1.0, 0.0, rows.size)
    a = np.zeros((n, n))
    np.add.at(a, (rows, cols), vals)
    if sym:
        a = 0.5 * (a + a.T)
    a[np.diag_indices(n)] = np.abs(a).sum(axis=1) + 1.0
    return CsrMatrix.from_dense(a)


@pytest.mark.parametrize("dims,dpn,sym", [((6, 6, 5), 2, True), ((7, 5, 4), 3, False),
                                          ((9, 9, 4), 1, True)])
def test_partitioned_inverse_matches_dense_solve(dims, dpn, sym):
    a0 = _grid_matrix(*dims, dpn, seed=sum(dims), sym=sym)
    f = build_coarse_factor(a0)
    dense = a0.to_dense()
    for k in range(3):
        u = np.random.default_rng(k).standard_normal(a0.nrows)
        x = solve_host(f, u)
        ref = np.linalg.solve(dense, u)
        assert np.abs(x - ref).max() <= 1e-12 * np.abs(ref).max()


def test_structure_invariants():
    a0 = _grid_matrix(8, 7, 6, 2, seed=5)
    f = build_coarse_factor(a0)
    n = a0.nrows
    # every column belongs to exactly one supernode
    assert np.array_equal(np.sort(f.col_ids), np.arange(n))
    # supernode levels: a supernode's rows below belong to supernodes on
    # strictly higher levels (processed later forward, earlier backward)
    level = np.repeat(np.arange(f.n_levels), np.diff(f.level_ptr))
    sn_of_col = np.empty(n, dtype=np.int64)
    sn_of_col[f.col_ids] = np.repeat(np.arange(f.n_sn), f.sn_s)
    for k in range(f.n_sn):
        rows = f.row_ids[f.row_ptr[k]:f.row_ptr[k + 1]]
        assert np.all(level[sn_of_col[rows]] > level[k])
    # extend-add: every update slot except the root's is consumed exactly
    # once, by its parent (as a column it subtracts or an update row it adds)
    used = np.sort(np.concatenate([f.in_idx, f.out_idx]))
    roots = [k for k in range(f.n_sn) if f.sn_r[k] == 0]
    assert np.array_equal(used, np.arange(f.row_ptr[-1]))
    assert len(roots) >= 1
    # fewer levels and values than the dense inverse
    assert f.n_levels < 40 and f.values.size < n * n


def test_singular_coarse_matrix_raises():
    a = np.eye(6)
    a[3, 3] = 0.0
    with pytest.raises(np.linalg.LinAlgError, match="pivot too small at row"):
        build_coarse_factor(CsrMatrix.from_dense(a))


@pytest.mark.parametrize("name", ["lap9_exact_nd", "ela7_exact"])
def test_block_factors_match_levelset_solves(name):
    """Batched partitioned inverses of the exact local factors (every
    subdomain in one batch, supernodes merged by tree level) against the
    oracle's level-set substitution, block by block (1e-12 relative)."""
    from cases import CASES, build
    from oracle import oracle as O
    from paper_2304_04876_b200 import decomposition as dd
    from paper_2304_04876_b200 import local_solvers as ls
    from paper_2304_04876_b200 import model_problems as mp
    from paper_2304_04876_b200 import schwarz as sw
    from paper_2304_04876_b200.coarse_factor import build_block_factors
    from paper_2304_04876_b200.sparse_core import extract_submatrix
    prob, dec, cfg = build((mp, dd, sw, ls), CASES[name])
    blocks, syms, facs, base = [], [], [], 0
    for dofs in dec.overlap.sets:
        blk = extract_submatrix(prob.a, dofs, dofs)
        sym = ls.build_symbolic(blk, cfg.local, ls.make_ordering(blk, cfg.ordering))
        lv, uv = O.lu_numeric(blk, sym)
        blocks.append((base, sym.l_ptr, sym.l_idx, lv, sym.u_ptr, sym.u_idx, uv))
        syms.append(sym)
        facs.append((lv, uv))
        base += dofs.size
    f = build_block_factors(blocks, threads=2)
    assert f.n == base
    # the host runtime's build equals the numpy restatement
    from paper_2304_04876_b200.coarse_factor import build_block_factors_py
    fp = build_block_factors_py(blocks, threads=2)
    for k in ("level_ptr", "sn_s", "sn_r", "col_ptr", "col_ids", "row_ptr", "row_ids", "d_off",
              "m_off", "n_off", "in_ptr", "in_idx", "out_ptr", "out_idx"):
        assert np.array_equal(getattr(f, k), getattr(fp, k)), k
    assert np.abs(f.values - fp.values).max() <= 1e-12 * np.abs(fp.values).max()
    # structure-only build (the device computes the blocks): same structure
    fs = build_block_factors(blocks, threads=2, values=False)
    for k in ("level_ptr", "sn_s", "sn_r", "col_ptr", "col_ids", "row_ptr", "row_ids", "d_off",
              "m_off", "n_off", "in_ptr", "in_idx", "out_ptr", "out_idx"):
        assert np.array_equal(getattr(f, k), getattr(fs, k)), k
    assert fs.values.size == 0 and fs.n_values == f.values.size
    rng = np.random.default_rng(7)
    b = rng.standard_normal(base)
    x = solve_host(f, b)
    for (b0, *_), sym, (lv, uv), dofs in zip(blocks, syms, facs, dec.overlap.sets):
        nb = dofs.size
        bp = b[b0:b0 + nb]
        # the oracle solves in the original block order; the factor in ND order
        ref = O.levelset_solve(sym, lv, uv, bp[np.argsort(sym.ordering.perm)])[sym.ordering.perm]
        got = x[b0:b0 + nb]
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    # far fewer sequential steps than the level schedule
    assert f.n_levels < max(s.n_levels[0] for s in syms)
