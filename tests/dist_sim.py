"""Host simulation of the sharded apply (test infrastructure).

Runs the exact data movement of the sharded GPU path -- forward halo of the
input, local solves of owned subdomains on the extended layout, partial
sums of halo rows sent back to their owners, the ordered combination
(lower-rank partial, own contributions in subdomain order, higher-rank
partial), and the coarse right-hand side summed over ranks in rank order --
with the ORACLE's kernels, so the shard plan (row ranges, halo ranges,
combination order) is checked against the global oracle apply on CPU.
`exchange` abstracts the transport: in-process (all ranks in one loop) or
torch.distributed gloo (one process per rank).
"""

from __future__ import annotations

import numpy as np

from oracle import oracle as O


def local_apply(sh, ore, r_ext, coarse_u_allreduce, exchange_rev):
    """One rank's apply. r_ext: input on the extended layout with halo rows
    filled. Returns z on the owned rows."""
    n_ext = sh.n_ext
    z_loc = np.zeros(n_ext)
    contrib = [[] for _ in range(n_ext)]          # per ext row: y values in subdomain order
    for s in sh.subs:                              # ascending subdomain ids
        dofs = ore.sets[s] - sh.e0
        y = ore.local_solve(int(s), r_ext[dofs])
        for d, v in zip(dofs, y):
            contrib[d].append(v)

    def ordered(vals, start=0.0):
        acc = start
        for v in vals:
            acc = acc + v
        return acc
    part = np.zeros(n_ext)
    for (q, slo, shi, rlo, rhi) in sh.nbrs:
        for g in range(rlo, rhi):
            part[g] = ordered(contrib[g], 0.0)
    recv = exchange_rev(part)                      # partials for my send ranges
    pre = post = None
    for (q, slo, shi, rlo, rhi) in sh.nbrs:
        if q < sh.rank:
            pre = (slo, shi)
        else:
            post = (slo, shi)
    zc = None
    if ore.coarse is not None:
        phi, phi_t, a0_sym, a0_l, a0_u = ore.coarse
        own = np.arange(sh.g0, sh.g1)
        # partial restriction over owned rows, then the rank-order sum
        u_part = O.spmv(phi_t.row_ptr, phi_t.col_idx, phi_t.values,
                        _masked(r_ext, sh, phi_t.ncols))
        u = coarse_u_allreduce(u_part)
        v = O.levelset_solve(a0_sym, a0_l, a0_u, u)
        zc = O.csr_spmv(phi, v)[own]
    out = np.zeros(sh.n_own)
    for k in range(sh.n_own):
        g = sh.own_off + k
        acc = recv[g] if pre and pre[0] <= g < pre[1] else 0.0
        acc = ordered(contrib[g], acc)
        if post and post[0] <= g < post[1]:
            acc = acc + recv[g]
        out[k] = acc if zc is None else zc[k] + acc
    return out


def _masked(r_ext, sh, n):
    """Global-length vector holding only this rank's owned entries."""
    full = np.zeros(n)
    full[sh.g0:sh.g1] = r_ext[sh.own_off:sh.own_off + sh.n_own]
    return full


def simulate_all(shards, ore, r):
    """All ranks in one process; exchanges by direct slicing."""
    r_ext = []
    for sh in shards:
        x = np.zeros(sh.n_ext)
        x[sh.own_off:sh.own_off + sh.n_own] = r[sh.g0:sh.g1]
        r_ext.append(x)
    for sh, x in zip(shards, r_ext):               # forward halo from the owners
        for (q, slo, shi, rlo, rhi) in sh.nbrs:
            src = shards[q]
            mine = next(t for t in src.nbrs if t[0] == sh.rank)
            x[rlo:rhi] = r_ext[q][mine[1]:mine[2]]
    parts = {}

    def make_rev(sh):
        def rev(part):
            parts[sh.rank] = part
            return part
        return rev
    u_parts = {}
    # two passes: first collect every rank's partials, then combine
    for sh in shards:
        def u_all(up, sh=sh):
            u_parts[sh.rank] = up
            return up
        local_apply(sh, ore, r_ext[sh.rank], u_all, make_rev(sh))
    u = np.zeros_like(next(iter(u_parts.values()))) if u_parts else None
    if u_parts:
        for q in range(len(shards)):
            u = u + u_parts[q]
    z = np.zeros(r.size)
    for sh in shards:
        def rev_in(part, sh=sh):
            recv = np.zeros(sh.n_ext)
            for (q, slo, shi, rlo, rhi) in sh.nbrs:
                theirs = next(t for t in shards[q].nbrs if t[0] == sh.rank)
                recv[slo:shi] = parts[q][theirs[3]:theirs[4]]
            return recv
        z[sh.g0:sh.g1] = local_apply(sh, ore, r_ext[sh.rank], lambda up: u, rev_in)
    return z
