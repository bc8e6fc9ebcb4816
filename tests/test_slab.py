"""Per-rank slab setup (slab.py) against the global sharded problem
(dist.build_sharded_problem): every object a rank's DistPreconditioner reads
-- operator rows, overlap and interior sets of its subdomains, the rGDSW
components touching its extended rows with their weights and GLOBAL coarse
columns, the coarse dimension -- is identical, for 2 and 3 ranks."""

import numpy as np
import pytest

from paper_2304_04876_b200.coarse_space import interior_sets
from paper_2304_04876_b200.dist import build_sharded_problem, plan_shards
from paper_2304_04876_b200.slab import build_slab_problem
from paper_2304_04876_b200.sparse_core import extract_submatrix


def _slabs(args, nranks):
    mine = []
    for r in range(nranks):     # each rank's own keys, as the all-gather would deliver them
        def grab(x):
            mine.append(x)
            return [x]
        build_slab_problem(*args, nranks, r, gather=grab)
    return [build_slab_problem(*args, nranks, r, gather=lambda x: mine) for r in range(nranks)]


@pytest.mark.parametrize("args,nranks", [((10, 8, 2, 2), 2), ((9, 6, 3, 1), 3), ((8, 12, 2, 3), 2),
                                         ((6, 4, 2, 1), 8), ((7, 3, 3, 1), 10)])
def test_slab_setup_matches_global(args, nranks):
    prob, dec = build_sharded_problem(*args, nranks)
    shards = plan_shards(prob.a, dec, nranks)
    gcomps = dec.structure.components
    gfirst = np.array([int(c.dofs[0]) for c in gcomps])
    gis = interior_sets(dec.partition, dec.structure)
    slabs = _slabs(args, nranks)
    if nranks >= 8:   # the windows really are windows
        assert max(sp.a.nrows for sp in slabs) < prob.a.nrows
    for sp, sh in zip(slabs, shards):
        off = sp.offset
        assert sp.n_c == len(gcomps)
        assert sp.g0 + off == sh.g0 and sp.g1 + off == sh.g1
        assert np.array_equal(sp.subs, sh.subs)
        # operator rows of the extended layout
        ext_w = np.arange(sh.e0 - off, sh.e1 - off)
        want = extract_submatrix(prob.a, np.arange(sh.e0, sh.e1), np.arange(sh.e0, sh.e1))
        got = extract_submatrix(sp.a, ext_w, ext_w)
        own = slice(sh.g0 - sh.e0, sh.g1 - sh.e0)
        for m in (want, got):
            m.rp = m.row_ptr
        assert np.array_equal(want.row_ptr[own.start:own.stop + 1] - want.row_ptr[own.start],
                              got.row_ptr[own.start:own.stop + 1] - got.row_ptr[own.start])
        sl = slice(want.row_ptr[own.start], want.row_ptr[own.stop])
        assert np.array_equal(want.col_idx[sl], got.col_idx[slice(got.row_ptr[own.start],
                                                                  got.row_ptr[own.stop])])
        assert np.array_equal(want.values[sl], got.values[slice(got.row_ptr[own.start],
                                                                got.row_ptr[own.stop])])
        wis = interior_sets(sp.dec.partition, sp.dec.structure)
        for s in sh.subs:
            assert np.array_equal(sp.dec.overlap.sets[s] + off, dec.overlap.sets[s])
            assert np.array_equal(wis[s] + off, gis[s])
        # every global component touching the extended rows, with its column
        byfirst = {(int(c.dofs[0]) + off, c.subdomains): (c, col) for c, col in
                   zip(sp.dec.structure.components, sp.comp_col)}
        for t, c in enumerate(gcomps):
            if not np.any((c.dofs >= sh.e0) & (c.dofs < sh.e1)):
                continue
            wc, col = byfirst[(int(c.dofs[0]), c.subdomains)]
            assert col == t
            assert np.array_equal(wc.dofs + off, c.dofs)
            assert np.array_equal(wc.weights, c.weights)
            assert wc.subdomains == c.subdomains
        assert np.array_equal(np.sort(gfirst), gfirst)
