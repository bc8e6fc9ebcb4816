"""Sharded-solve plan on CPU: layout invariants, and the
sharded apply's data movement (halo, reverse partial sums in subdomain
order, rank-order coarse sum) reproducing the global apply -- in one
process and over torch.distributed gloo with world_size 2."""

import os
import socket

import numpy as np
import pytest

from dist_sim import local_apply, simulate_all
from oracle import oracle as O
from paper_2304_04876_b200.dist import build_sharded_problem, plan_shards
from paper_2304_04876_b200.local_solvers import SolverSpec
from paper_2304_04876_b200.schwarz import SchwarzConfig


def _problem(nranks, method="fast_ilu"):
    prob, dec = build_sharded_problem(10, 6, 2, 2, nranks)
    cfg = SchwarzConfig(local=SolverSpec(method, 0, 3, 5), ordering="natural")
    return prob, dec, cfg


@pytest.mark.parametrize("nranks", [2, 3])
def test_shard_layout_invariants(nranks):
    prob, dec, cfg = _problem(nranks)
    shards = plan_shards(prob.a, dec, nranks)
    assert shards[0].g0 == 0 and shards[-1].g1 == prob.a.nrows
    for a, b in zip(shards, shards[1:]):
        assert a.g1 == b.g0
    for sh in shards:
        assert sh.e0 <= sh.g0 < sh.g1 <= sh.e1
        for s in sh.subs:                        # overlap sets inside the layout
            assert dec.overlap.sets[s][0] >= sh.e0 and dec.overlap.sets[s][-1] < sh.e1
        rows = slice(prob.a.row_ptr[sh.g0], prob.a.row_ptr[sh.g1])
        assert prob.a.col_idx[rows].min() >= sh.e0 and prob.a.col_idx[rows].max() < sh.e1
        for (q, slo, shi, rlo, rhi) in sh.nbrs:  # symmetric neighbour ranges
            back = next(t for t in shards[q].nbrs if t[0] == sh.rank)
            assert shi - slo == back[4] - back[3]
            assert rhi - rlo == back[2] - back[1]
            assert sh.e0 + rlo == shards[q].e0 + back[1]


@pytest.mark.parametrize("method", ["fast_ilu", "ilu_k"])
def test_sharded_apply_matches_global_in_process(method):
    prob, dec, cfg = _problem(2, method)
    ore = O.OracleSchwarz(prob.a, dec, cfg, prob.nullspace)
    shards = plan_shards(prob.a, dec, 2)
    r = np.random.default_rng(4).standard_normal(prob.a.nrows)
    want = ore.apply(r)
    got = simulate_all(shards, ore, r)
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, q):
    import torch
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prob, dec, cfg = _problem(world)
        ore = O.OracleSchwarz(prob.a, dec, cfg, prob.nullspace)
        sh = plan_shards(prob.a, dec, world)[rank]
        r = np.random.default_rng(4).standard_normal(prob.a.nrows)
        x = np.zeros(sh.n_ext)
        x[sh.own_off:sh.own_off + sh.n_own] = r[sh.g0:sh.g1]
        # forward halo over gloo
        reqs = []
        for (qr, slo, shi, rlo, rhi) in sh.nbrs:
            reqs.append(tdist.isend(torch.from_numpy(x[slo:shi].copy()), qr))
        for (qr, slo, shi, rlo, rhi) in sh.nbrs:
            buf = torch.zeros(rhi - rlo, dtype=torch.float64)
            tdist.recv(buf, qr)
            x[rlo:rhi] = buf.numpy()
        for rq in reqs:
            rq.wait()

        def u_all(up):
            parts = [torch.zeros(up.size, dtype=torch.float64) for _ in range(world)]
            tdist.all_gather(parts, torch.from_numpy(up))
            u = np.zeros(up.size)
            for p in parts:
                u = u + p.numpy()
            return u

        def rev(part):
            reqs = [tdist.isend(torch.from_numpy(part[rlo:rhi].copy()), qr)
                    for (qr, slo, shi, rlo, rhi) in sh.nbrs]
            recv = np.zeros(sh.n_ext)
            for (qr, slo, shi, rlo, rhi) in sh.nbrs:
                buf = torch.zeros(shi - slo, dtype=torch.float64)
                tdist.recv(buf, qr)
                recv[slo:shi] = buf.numpy()
            for rq in reqs:
                rq.wait()
            return recv

        z = local_apply(sh, ore, x, u_all, rev)
        want = ore.apply(r)[sh.g0:sh.g1]
        q.put((rank, float(np.abs(z - want).max() / np.abs(want).max())))
    finally:
        tdist.destroy_process_group()


def test_sharded_apply_over_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for rank, rel in res:
        assert rel <= 1e-13, (rank, rel)
