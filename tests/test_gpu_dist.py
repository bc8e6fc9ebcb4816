"""Sharded solve on the GPU with 2 ranks (2 processes sharing one device;
IPC mailboxes + device-side flags): the peer-memory collectives, and the
sharded GMRES against the single-GPU solve of the same global system."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(world, method):
    from paper_2304_04876_b200.dist import build_sharded_problem
    from paper_2304_04876_b200.local_solvers import SolverSpec
    from paper_2304_04876_b200.schwarz import SchwarzConfig
    prob, dec = build_sharded_problem(14, 8, 2, 2, world)
    spec = SolverSpec(method, 0, 3, 5)
    cfg = SchwarzConfig(local=spec, ordering="natural")
    return prob, dec, cfg


def _rank_main(rank, world, port, method, q):
    import torch
    import torch.distributed as tdist

    from paper_2304_04876_b200 import device
    from paper_2304_04876_b200.dist import DistPreconditioner, plan_shards
    from paper_2304_04876_b200.krylov import KrylovConfig
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prob, dec, cfg = _problem(world, method)
        sh = plan_shards(prob.a, dec, world)[rank]
        # collectives: rank-ordered all-reduce and the forward halo
        lay = device.DistLayout(sh.rank, sh.nranks, sh.n_ext, sh.own_off, sh.own_off + sh.n_own,
                                sh.nbrs)
        hs = [None] * world
        tdist.all_gather_object(hs, lay.ipc_handle())
        lay.open_peers(hs)
        v = torch.arange(5, dtype=torch.float64, device="cuda") * (rank + 1)
        out = torch.zeros_like(v)
        lay.allreduce(v, out)
        red_ok = bool(torch.equal(out.cpu(), torch.arange(5, dtype=torch.float64) * 3))
        glob = torch.arange(prob.a.nrows, dtype=torch.float64)
        xe = torch.full((sh.n_ext,), -1.0, dtype=torch.float64, device="cuda")
        xe[sh.own_off:sh.own_off + sh.n_own] = glob[sh.g0:sh.g1].cuda()
        lay.halo(xe)
        torch.cuda.synchronize()
        halo_ok = True
        for (qr, slo, shi, rlo, rhi) in sh.nbrs:
            halo_ok &= bool(torch.equal(xe[rlo:rhi].cpu(), glob[sh.e0 + rlo:sh.e0 + rhi]))
        # the sharded solve
        pre = DistPreconditioner(prob.a, dec, cfg, prob.nullspace, sh)
        b = prob.a @ np.random.default_rng(0).standard_normal(prob.a.nrows)
        bo = torch.from_numpy(b[sh.g0:sh.g1].copy()).cuda()
        x, rep = pre.solve(bo, KrylovConfig(variant="single_reduce"))
        x, rep = pre.solve(bo, KrylovConfig(variant="single_reduce"))   # replayed pass graphs
        os.environ["GDSW_NO_GRAPH"] = "1"
        xe, _ = pre.solve(bo, KrylovConfig(variant="single_reduce"))
        del os.environ["GDSW_NO_GRAPH"]
        torch.cuda.synchronize()
        graph_ok = bool(torch.equal(x, xe))
        q.put((rank, red_ok, halo_ok, sh.g0, x.cpu().numpy(), rep["iterations"], rep["converged"],
               list(rep["history"]), graph_ok, pre.a0.to_dense().astype(np.float64),
               pre.a0.row_ptr.copy(), pre.a0.col_idx.copy()))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("method", ["fast_ilu", "ilu_k", "exact_lu"])
def test_sharded_gmres_two_ranks_one_gpu(method):
    """Sharded solve (GPU numeric LU / FastILU per rank, GPU Galerkin A0 summed
    over ranks on the device, graphed passes with device-sequenced
    collectives, the coarse side stream) == the single-GPU solve."""
    import torch.multiprocessing as mp

    from paper_2304_04876_b200.decomposition import decompose
    from paper_2304_04876_b200.krylov import KrylovConfig, gmres
    from paper_2304_04876_b200.schwarz import setup_numeric, setup_symbolic
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, method, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = sorted([q.get(timeout=600) for _ in procs], key=lambda t: t[0])
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert all(r[1] for r in res), "rank-ordered all-reduce"
    assert all(r[2] for r in res), "forward halo"
    prob, dec, cfg = _problem(world, method)
    # the same global system on one GPU
    skel = setup_symbolic(prob.a, decompose(prob.a, dec.partition, 1, "rgdsw"), cfg)
    pre = setup_numeric(skel, prob.a, prob.nullspace)
    b = prob.a @ np.random.default_rng(0).standard_normal(prob.a.nrows)
    x1, rep1 = gmres(prob.a, pre, b, KrylovConfig(variant="single_reduce"))
    xs = np.concatenate([r[4] for r in res])
    assert all(r[6] for r in res)
    assert res[0][5] == res[1][5]
    assert abs(res[0][5] - rep1.iterations) <= 1
    assert np.allclose(res[0][7][:5], rep1.residual_history[:5], rtol=1e-8)
    assert np.abs(xs - x1).max() <= 1e-6 * np.abs(x1).max()
    assert all(r[8] for r in res), "graphed sharded passes == eager, bitwise"
    a0 = pre.coarse.a0
    for r in res:   # every rank: the single-GPU A0 (values; the reference's SpGEMM pattern)
        assert np.array_equal(r[10], a0.row_ptr) and np.array_equal(r[11], a0.col_idx)
        assert np.abs(r[9] - a0.to_dense()).max() <= 1e-12 * np.abs(a0.to_dense()).max()
    assert np.array_equal(res[0][9], res[1][9])
    assert np.linalg.norm(b - prob.a @ xs) <= 1e-7 * np.linalg.norm(b) * 1.0001


def _slab_rank_main(rank, world, port, method, q):
    import torch
    import torch.distributed as tdist

    from paper_2304_04876_b200.dist import DistPreconditioner, plan_slab_shard
    from paper_2304_04876_b200.krylov import KrylovConfig
    from paper_2304_04876_b200.local_solvers import SolverSpec
    from paper_2304_04876_b200.schwarz import SchwarzConfig
    from paper_2304_04876_b200.slab import build_slab_problem
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sp = build_slab_problem(14, 8, 2, 2, world, rank)
        sh = plan_slab_shard(sp, world, rank)
        cfg = SchwarzConfig(local=SolverSpec(method, 0, 3, 5), ordering="natural")
        pre = DistPreconditioner(sp.a, sp.dec, cfg, sp.nullspace, sh, slab=sp)
        x_star = np.random.default_rng(0).standard_normal(sp.n_global)
        b = sp.a @ x_star[sp.offset:sp.offset + sp.a.nrows]
        bo = torch.from_numpy(b[sh.g0:sh.g1].copy()).cuda()
        x, rep = pre.solve(bo, KrylovConfig(variant="single_reduce"))
        torch.cuda.synchronize()
        q.put((rank, x.cpu().numpy(), rep["iterations"], rep["converged"], list(rep["history"]),
               pre.a0.to_dense().astype(np.float64), sp.a.nrows, sp.n_global))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("method", ["fast_ilu", "exact_lu"])
def test_sharded_gmres_slab_setup_two_ranks(method):
    """Every rank builds only its z-window (slab.py) -- the sharded solve
    still equals the single-GPU solve of the global system: iterations,
    residual history, solution, and the coarse matrix A0 (global columns)."""
    import torch.multiprocessing as mp

    from paper_2304_04876_b200.decomposition import decompose
    from paper_2304_04876_b200.krylov import KrylovConfig, gmres
    from paper_2304_04876_b200.schwarz import setup_numeric, setup_symbolic
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_rank_main, args=(r, world, port, method, q))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = sorted([q.get(timeout=600) for _ in procs], key=lambda t: t[0])
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    prob, dec, cfg = _problem(world, method)
    skel = setup_symbolic(prob.a, decompose(prob.a, dec.partition, 1, "rgdsw"), cfg)
    pre = setup_numeric(skel, prob.a, prob.nullspace)
    b = prob.a @ np.random.default_rng(0).standard_normal(prob.a.nrows)
    x1, rep1 = gmres(prob.a, pre, b, KrylovConfig(variant="single_reduce"))
    assert all(r[7] == prob.a.nrows for r in res)
    assert all(r[3] for r in res)
    assert res[0][2] == res[1][2] and abs(res[0][2] - rep1.iterations) <= 1
    assert np.allclose(res[0][4][:5], rep1.residual_history[:5], rtol=1e-8)
    xs = np.concatenate([r[1] for r in res])
    assert np.abs(xs - x1).max() <= 1e-6 * np.abs(x1).max()
    a0 = pre.coarse.a0.to_dense()
    for r in res:
        assert np.abs(r[5] - a0).max() <= 1e-12 * np.abs(a0).max()
