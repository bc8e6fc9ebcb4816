"""CUDA path vs the oracle (and the reference's golden vectors), through the
C ABI. Sequential kernels (SpMV, level-set and Jacobi trisolves, FastILU
sweeps, gather/scatter) must be bit-identical; the coarse correction
(batched-CG extension + dense A0^-1) within the north star's tolerances:
1e-10 relative (fp64 apply), 1e-5 (fp32 apply vs fp64), GMRES iterations
within +-1 of the reference."""

import json

import numpy as np
import pytest

from cases import BIG, CASES, build, probes, rhs
from oracle import oracle as O
from paper_2304_04876_b200 import decomposition as dd
from paper_2304_04876_b200 import local_solvers as ls
from paper_2304_04876_b200 import model_problems as mp
from paper_2304_04876_b200 import schwarz as sw
from paper_2304_04876_b200.krylov import KrylovConfig, gmres
from paper_2304_04876_b200.sparse_core import CsrMatrix

pytestmark = pytest.mark.gpu
PKG = (mp, dd, sw, ls)
APPLY_TOL64 = 1e-10
APPLY_TOL32 = 1e-5


@pytest.fixture(scope="module")
def golden(golden_dir):
    return json.loads((golden_dir / "golden.json").read_text())


_CACHE = {}


def setup_case(name, table=CASES):
    if name not in _CACHE:
        prob, dec, cfg = build(PKG, table[name])
        skel = sw.setup_symbolic(prob.a, dec, cfg)
        pre = sw.setup_numeric(skel, prob.a, prob.nullspace if cfg.use_coarse else None)
        _CACHE[name] = (prob, dec, cfg, skel, pre)
    return _CACHE[name]


def _torch():
    import torch
    return torch


# ---------------------------------------------------------------------------
def test_spmv_bitwise_against_oracle():
    torch = _torch()
    from paper_2304_04876_b200.device import DeviceCsr
    rng = np.random.default_rng(0)
    mats = [mp.assemble_laplace3d(mp.Grid3D(13, 12, 11)).a,
            mp.assemble_elasticity3d(mp.Grid3D(6, 6, 5)).a]
    d = (rng.random((70, 50)) < 0.1) * rng.standard_normal((70, 50))
    mats.append(CsrMatrix.from_dense(d))
    for a in mats:
        x = rng.standard_normal(a.ncols)
        want = O.spmv(a.row_ptr, a.col_idx, a.values, x)
        dev = DeviceCsr(a)
        y = torch.zeros(a.nrows, dtype=torch.float64, device="cuda")
        dev.spmv(torch.from_numpy(x).cuda(), y)
        assert np.array_equal(y.cpu().numpy(), want)
        yy = torch.from_numpy(want.copy()).cuda()
        dev.spmv(torch.from_numpy(x).cuda(), yy, -1.0, 1.0)   # b - A x
        assert np.array_equal(yy.cpu().numpy(), want - want)


def _banded(n, offsets_of_slice, rng, p_keep):
    """Random matrix whose rows draw their columns from a per-slice offset set
    (ragged rows, empty rows, clipping at the matrix edges)."""
    rows, cols = [], []
    for i in range(n):
        offs = offsets_of_slice(i // 32)
        for o in sorted(offs):
            j = i + o
            if 0 <= j < n and rng.random() < p_keep:
                rows.append(i)
                cols.append(j)
    d = np.zeros((n, n))
    d[rows, cols] = rng.standard_normal(len(rows))
    return CsrMatrix.from_dense(d)


@pytest.mark.parametrize("no_mask", [False, True])
def test_spmv_offset_mask_layout_bitwise(no_mask, monkeypatch):
    """The offset-mask column layout (sparse.cuh SellMaskCols): slices with up
    to eight distinct offsets, ragged and empty rows, non-uniform slice widths
    (the sell_row chunk loop), a slice set with nine offsets (fallback to
    per-entry columns); GDSW_NO_SELL_MASK=1 forces the per-entry layout. The
    SpMV must be bit-identical to the oracle either way."""
    torch = _torch()
    from paper_2304_04876_b200.device import DeviceCsr
    if no_mask:
        monkeypatch.setenv("GDSW_NO_SELL_MASK", "1")
    rng = np.random.default_rng(7)
    base8 = [-300, -41, -7, -1, 0, 2, 33, 290]
    mats = [
        _banded(700, lambda s: base8, rng, 0.6),                                   # <= 8 per slice
        _banded(700, lambda s: [o + (s % 3) for o in base8], rng, 0.9),            # slice-dependent
        _banded(650, lambda s: base8[:3] if s % 2 else base8, rng, 0.35),          # sparse, ragged
        _banded(500, lambda s: base8 + [97] if s == 5 else base8, rng, 0.8),       # one slice has 9
    ]
    for a in mats:
        x = rng.standard_normal(a.ncols)
        want = O.spmv(a.row_ptr, a.col_idx, a.values, x)
        dev = DeviceCsr(a)
        y = torch.zeros(a.nrows, dtype=torch.float64, device="cuda")
        dev.spmv(torch.from_numpy(x).cuda(), y)
        assert np.array_equal(y.cpu().numpy(), want)


TS_CHAIN = 128   # tristream.cuh TR_SEG: rows up to this length keep the sequential order
LONG_ROW_TOL = 1e-13


def _max_row_len(sym):
    lu = np.diff(sym.u_ptr) - 1
    ll = np.diff(sym.l_ptr)
    return int(max(ll.max(initial=0), lu.max(initial=0)))


@pytest.mark.parametrize("name", sorted(CASES))
def test_local_solves_bitwise_against_oracle(name):
    """Bit-identical to sequential substitution for the Jacobi sweeps and
    ILU(k) factors whose rows have <= TS_CHAIN entries; exact-LU factors
    (warp-tree rows, supernodal dense blocks) are compared at 1e-13
    relative."""
    torch = _torch()
    prob, dec, cfg, skel, pre = setup_case(name)
    ore = O.OracleSchwarz(prob.a, dec, cfg, prob.nullspace if cfg.use_coarse else None,
                          symbolics=skel.local_symbolics)
    r = probes(prob.a.nrows, ks=(5,))[0]
    dt = torch.float32 if cfg.precision == "single" else torch.float64
    y = torch.empty(skel._local_plan["n_loc"], dtype=dt, device="cuda")
    pre._dev.local_solve(torch.from_numpy(r).cuda(), y)
    y = y.cpu().numpy()
    off = 0
    rw = r.astype(np.float32) if cfg.precision == "single" else r
    for i, (dofs, sym) in enumerate(zip(skel.sets, skel.local_symbolics)):
        want = ore.local_solve(i, rw[dofs])
        got = np.empty_like(want)
        got[sym.ordering.perm] = y[off:off + dofs.size]
        off += dofs.size
        if cfg.local.method == "fast_ilu" or (cfg.local.method == "ilu_k"
                                              and _max_row_len(sym) <= TS_CHAIN):
            assert np.array_equal(got, want), f"subdomain {i}"
        else:
            assert np.abs(got - want).max() <= LONG_ROW_TOL * np.abs(want).max(), f"subdomain {i}"


@pytest.mark.parametrize("name", [n for n in sorted(CASES) if CASES[n][4] != "fast_ilu"])
def test_gpu_numeric_lu_bitwise_against_host_ikj(name):
    """The GPU IKJ factorization (every block in one launch) reproduces the
    reference's lu_numeric bit for bit (host restatement and oracle)."""
    from paper_2304_04876_b200.sparse_core import convert_precision, extract_submatrix
    prob, dec, cfg, skel, pre = setup_case(name)
    src = convert_precision(prob.a, np.float32) if cfg.precision == "single" else prob.a
    shift = cfg.local.diag_shift if cfg.local.method == "ilu_k" else 0.0
    for dofs, sym, fac in zip(skel.sets, skel.local_symbolics, pre.local_factorizations):
        lv, uv = ls.host_numeric(extract_submatrix(src, dofs, dofs), sym, shift)
        assert np.array_equal(fac.l_values, lv)
        assert np.array_equal(fac.u_values, uv)


@pytest.mark.parametrize("dims,method,fill", [((42, 42, 40), "ilu_k", 0), ((42, 42, 40), "ilu_k", 2),
                                              ((32, 32, 30), "ilu_k", 0), ((32, 32, 30), "ilu_k", 1)])
def test_large_block_streamed_sptrsv_bitwise(dims, method, fill):
    """A single large block: the iterate in global memory with previous-chunk
    forwarding through shared memory (the C2-like layout of the streamed
    SpTRSV), 32-bit block columns above 65,536 rows, 16-bit below; ILU(k)
    rows stay bit-identical to the oracle."""
    torch = _torch()
    prob = mp.assemble_laplace3d(mp.Grid3D(*dims))
    dec = dd.decompose(prob.a, dd.box_partition(prob.grid, 1, 1, 1), 1, None)
    cfg = sw.SchwarzConfig(local=ls.SolverSpec(method, fill), use_coarse=False,
                           ordering="natural")
    skel = sw.setup_symbolic(prob.a, dec, cfg)
    pre = sw.setup_numeric(skel, prob.a, None)
    assert skel.sets[0].size > 65536 or dims[0] < 42
    ore = O.OracleSchwarz(prob.a, dec, cfg, None, symbolics=skel.local_symbolics)
    r = probes(prob.a.nrows, ks=(3,))[0]
    y = torch.empty(skel._local_plan["n_loc"], dtype=torch.float64, device="cuda")
    pre._dev.local_solve(torch.from_numpy(r).cuda(), y)
    want = ore.local_solve(0, r[skel.sets[0]])
    got = np.empty_like(want)
    got[skel.local_symbolics[0].ordering.perm] = y.cpu().numpy()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("name", [n for n in sorted(CASES) if CASES[n][4] == "fast_ilu"])
def test_fastsptrsv_layout_and_apply_overlap_variants(name):
    """The plain-loop FastSpTRSV rows (GDSW_JACOBI_UNI=0) and the L2-hinted
    iterates are bit-identical to the default uniform-width sweeps; the apply
    with and without the side-stream coarse overlap is bit-identical too."""
    import os
    torch = _torch()
    prob, dec, cfg, skel, pre = setup_case(name)
    r = torch.from_numpy(probes(prob.a.nrows, ks=(5,))[0]).cuda()
    dt = torch.float32 if cfg.precision == "single" else torch.float64
    n_loc = skel._local_plan["n_loc"]
    y0 = torch.empty(n_loc, dtype=dt, device="cuda")
    pre._dev.local_solve(r, y0)
    for var, val in (("GDSW_L2HINT", "1"),):
        try:
            os.environ[var] = val
            for _ in range(2):
                y1 = torch.full((n_loc,), float("nan"), dtype=dt, device="cuda")
                pre._dev.local_solve(r, y1)
                assert torch.equal(y0, y1), var
        finally:
            del os.environ[var]
    z0 = torch.empty_like(r)
    pre._dev.apply(r, z0)
    try:
        os.environ["GDSW_NO_OVERLAP"] = "1"
        z1 = torch.empty_like(r)
        pre._dev.apply(r, z1)
    finally:
        del os.environ["GDSW_NO_OVERLAP"]
    assert torch.equal(z0, z1)


@pytest.mark.parametrize("name", [n for n in sorted(CASES) if CASES[n][4] == "fast_ilu"])
def test_fastilu_factors_bitwise_against_oracle(name):
    prob, dec, cfg, skel, pre = setup_case(name)
    ore = O.OracleSchwarz(prob.a, dec, cfg, prob.nullspace if cfg.use_coarse else None,
                          symbolics=skel.local_symbolics)
    for i, fac in enumerate(pre.local_factorizations):
        lv, uv, res = ore.factors[i]
        assert np.array_equal(fac.l_values, lv)
        assert np.array_equal(fac.u_values, uv)
        assert np.allclose(fac.sweep_residuals, res, rtol=1e-10, atol=0)


@pytest.mark.parametrize("name", sorted(CASES))
def test_apply_against_reference_golden(golden_dir, name):
    prob, dec, cfg, skel, pre = setup_case(name)
    g = np.load(golden_dir / f"golden_{name}.npz")
    tol = APPLY_TOL32 if cfg.precision == "single" else APPLY_TOL64
    for k, r in enumerate(probes(prob.a.nrows)):
        z = pre.apply(r)
        want = g[f"apply_{k}"]
        assert z.dtype == np.float64
        assert np.abs(z - want).max() <= tol * np.abs(want).max()
        if cfg.precision == "single":
            # against the reference's own fp32 apply the gap is far tighter
            assert np.abs(z - want).max() <= 1e-5 * np.abs(want).max()


@pytest.mark.parametrize("name", [n for n in sorted(CASES) if CASES[n][3] == "none"])
def test_one_level_apply_bitwise(golden_dir, name):
    prob, dec, cfg, skel, pre = setup_case(name)
    g = np.load(golden_dir / f"golden_{name}.npz")
    for k, r in enumerate(probes(prob.a.nrows)):
        assert np.array_equal(pre.apply(r), g[f"apply_{k}"])


@pytest.mark.parametrize("name", [n for n in sorted(CASES) if CASES[n][3] != "none"])
def test_coarse_basis_and_a0(golden_dir, name):
    prob, dec, cfg, skel, pre = setup_case(name)
    g = np.load(golden_dir / f"golden_{name}.npz")
    phi = pre.coarse.phi.to_dense().astype(np.float64)
    want = g["phi_dense"]
    tol = 1e-6 if cfg.precision == "single" else 1e-10
    assert phi.shape == want.shape
    assert np.abs(phi - want).max() <= tol * np.abs(want).max()
    a0 = pre.coarse.a0.to_dense().astype(np.float64)
    assert np.abs(a0 - g["a0_dense"]).max() <= tol * np.abs(g["a0_dense"]).max()
    # the reference's SpGEMM pattern, computed zeros included (coarse_space.py:205-207)
    assert np.array_equal(pre.coarse.a0.row_ptr, g["a0_row_ptr"])
    assert np.array_equal(pre.coarse.a0.col_idx, g["a0_col_idx"])


@pytest.mark.parametrize("name", sorted(CASES))
def test_gmres_matches_reference(golden, golden_dir, name):
    prob, dec, cfg, skel, pre = setup_case(name)
    g = np.load(golden_dir / f"golden_{name}.npz")
    x_star, b = rhs(prob)
    for variant, orth in (("single_reduce", "mgs"), ("classic", "mgs"), ("classic_cgs2", "cgs2")):
        x, rep = gmres(prob.a, pre, b, KrylovConfig(variant=variant.split("_cgs2")[0],
                                                    orthogonalization=orth))
        want = golden["cases"][name][variant]
        assert rep.converged
        assert abs(rep.iterations - want["iterations"]) <= 1
        assert rep.true_residuals[-1][1] <= 1e-7
        r = b - prob.a @ x
        assert np.linalg.norm(r) <= 1e-7 * np.linalg.norm(b) * 1.0001
        if rep.iterations == want["iterations"]:
            assert rep.residual_reductions == want["residual_reductions"]
            assert rep.restarts == want["restarts"]
            assert rep.iteration_reductions == want["iteration_reductions"]
            assert [i for i, _ in rep.true_residuals] == [i for i, _ in want["true_residuals"]]
        if variant == "single_reduce" and rep.iterations == want["iterations"]:
            assert rep.iteration_reductions == rep.iterations
            # fp32 preconditioners round differently in the coarse sums
            rtol = 1e-4 if cfg.precision == "single" else 1e-6
            assert np.allclose(rep.residual_history, g[f"hist_{variant}"], rtol=rtol,
                               atol=1e-12)


@pytest.mark.parametrize("graphs", [True, False])
def test_gmres_drift_confirmation_failures(golden, graphs, monkeypatch):
    """Failed true-residual confirmations (krylov.py:331-342): a nonlinear
    host operator A makes the Givens estimate pass rtol while the true
    residual does not, for ten iterations in a row, then the cycle restarts.
    The pipelined single-reduce loop must keep the queued pass's scalars and
    block intact across each failed check (candidate y and the true-residual
    norm have their own buffers), so iterations, restarts and every true
    residual follow the reference."""
    from cases import DRIFT_EPS, drift_operator
    if not graphs:
        monkeypatch.setenv("GDSW_NO_GRAPH", "1")
    prob, dec, cfg, skel, pre = setup_case("lap10_fast_nat")
    _, b = rhs(prob)
    want = golden["drift"]["lap10_fast_nat"]
    x, rep = gmres(drift_operator(prob.a, DRIFT_EPS), pre, b,
                   KrylovConfig(variant="single_reduce", max_iters=60))
    assert rep.converged == want["converged"]
    assert rep.iterations == want["iterations"]
    assert rep.restarts == want["restarts"]
    assert rep.residual_reductions == want["residual_reductions"]
    assert [i for i, _ in rep.true_residuals] == [i for i, _ in want["true_residuals"]]
    assert np.allclose([v for _, v in rep.true_residuals],
                       [v for _, v in want["true_residuals"]], rtol=1e-5)
    assert np.allclose(rep.residual_history, want["residual_history"], rtol=1e-5, atol=1e-14)


@pytest.mark.parametrize("variant", ["single_reduce", "classic"])
def test_gmres_rejected_confirmations_device_operators(variant, monkeypatch):
    """Device A and M, graphed passes: the test hook
    GDSW_DEBUG_REJECT_CHECKS=3 makes the first three true-residual
    confirmations count as failed, so the solve keeps iterating with a pass
    already queued behind each check (krylov.py:331-342). The pipelined
    state must survive: iterations, checks and history follow the oracle
    run with the same rule, and graphed == eager bitwise."""
    prob, dec, cfg, skel, pre = setup_case("lap10_fast_nat")
    _, b = rhs(prob)
    ore = O.OracleSchwarz(prob.a, dec, cfg, prob.nullspace, symbolics=skel.local_symbolics)
    xo, ro = O.gmres(lambda v: O.csr_spmv(prob.a, v), ore.apply, b, variant=variant,
                     reject_checks=3)
    monkeypatch.setenv("GDSW_DEBUG_REJECT_CHECKS", "3")
    x, rep = gmres(prob.a, pre, b, KrylovConfig(variant=variant))
    assert len(ro["true_residuals"]) == 4
    assert rep.converged and rep.iterations == ro["iterations"]
    assert [i for i, _ in rep.true_residuals] == [i for i, _ in ro["true_residuals"]]
    assert np.allclose([v for _, v in rep.true_residuals], [v for _, v in ro["true_residuals"]],
                       rtol=1e-6)
    assert np.allclose(rep.residual_history, ro["history"], rtol=1e-6, atol=1e-14)
    assert np.abs(x - xo).max() <= 1e-8 * np.abs(xo).max()
    monkeypatch.setenv("GDSW_NO_GRAPH", "1")
    x2, rep2 = gmres(prob.a, pre, b, KrylovConfig(variant=variant))
    assert np.array_equal(rep2.residual_history, rep.residual_history)
    assert np.array_equal(x2, x)


def test_gmres_identity_operator_none():
    """gmres(None, M, b): A is the identity (krylov.py:89-90)."""
    prob, dec, cfg, skel, pre = setup_case("lap9_onelevel_ilu0")
    b = probes(prob.a.nrows, ks=(4,))[0]
    x, rep = gmres(None, None, b)
    assert rep.converged and rep.iterations == 1
    assert np.allclose(x, b, rtol=1e-12)


def test_gmres_solve_and_apply_on_two_threads():
    """A solve and standalone applies of the same preconditioner from two
    threads: the solve holds the preconditioner for its duration, each
    thread has its own Krylov workspace, results are bit-identical to the
    sequential ones."""
    from concurrent.futures import ThreadPoolExecutor
    prob, dec, cfg, skel, pre = setup_case("lap10_fast_nat")
    _, b = rhs(prob)
    vecs = probes(prob.a.nrows, ks=range(20, 28))
    want_z = [pre.apply(r) for r in vecs]
    want_x, _ = gmres(prob.a, pre, b)

    def solve(_):
        return gmres(prob.a, pre, b)[0]
    with ThreadPoolExecutor(max_workers=3) as ex:
        fx = [ex.submit(solve, k) for k in range(3)]
        fz = [ex.submit(pre.apply, r) for r in vecs]
        got_x = [f.result() for f in fx]
        got_z = [f.result() for f in fz]
    for g in got_x:
        assert np.array_equal(g, want_x)
    for g, w in zip(got_z, want_z):
        assert np.array_equal(g, w)


def test_gmres_stale_operator_values_rejected():
    """The device copy of A is keyed on its values array, which is made
    read-only while cached: an in-place edit raises instead of silently
    solving with stale values."""
    a = mp.assemble_laplace3d(mp.Grid3D(6, 6, 6)).a
    a = CsrMatrix(a.nrows, a.ncols, a.row_ptr, a.col_idx, a.values.copy())
    b = probes(a.nrows, ks=(2,))[0]
    x1, _ = gmres(a, None, b)
    with pytest.raises(ValueError):
        a.values *= 2.0
    a2 = CsrMatrix(a.nrows, a.ncols, a.row_ptr, a.col_idx, a.values * 2.0)
    x2, _ = gmres(a2, None, b)
    assert np.allclose(x2, 0.5 * x1, rtol=1e-6)


def test_gmres_against_oracle_identical_iterations():
    """The oracle builds the reference's preconditioner independently (exact
    interior LU); the coarse bases agree to ~1e-13, so the iteration counts
    match exactly."""
    prob, dec, cfg, skel, pre = setup_case("lap10_fast_nat")
    _, b = rhs(prob)
    ore = O.OracleSchwarz(prob.a, dec, cfg, prob.nullspace, symbolics=skel.local_symbolics)
    xo, ro = O.gmres(lambda v: O.csr_spmv(prob.a, v), ore.apply, b)
    x, rep = gmres(prob.a, pre, b, KrylovConfig(variant="single_reduce"))
    assert rep.iterations == ro["iterations"]
    assert np.abs(x - xo).max() <= 1e-8 * np.abs(xo).max()


@pytest.mark.parametrize("name", ["C1_lap30_exact", "lap24_fast_4x4x4", "lap17_exact_3x3x3",
                                  "ela12_fast_2x2x2", "lap20_single_fast"])
def test_iteration_counts_at_size(golden, name):
    prob, dec, cfg, skel, pre = setup_case(name, BIG)
    _, b = rhs(prob)
    x, rep = gmres(prob.a, pre, b, KrylovConfig(variant="single_reduce"))
    assert rep.converged
    assert abs(rep.iterations - golden["big"][name]["iterations"]) <= 1
    assert np.linalg.norm(b - prob.a @ x) <= 1e-7 * np.linalg.norm(b) * 1.0001


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["lap9_exact_nd", "ela7_exact"])
def test_local_partitioned_inverse_device_build_matches_host(monkeypatch, name):
    """Exact-LU local solves through partitioned inverses whose blocks the
    device computes (k_pinv_fill / k_pinv_blocks, from its own factors)
    against the host runtime's blocks (1e-13 relative per block), and both
    against the streamed level-set substitution."""
    torch = _torch()
    out = {}
    for mode, env in (("device", {}), ("host", {"GDSW_PINV_HOST": "1"}),
                      ("stream", {"GDSW_LOCAL_FACTOR": "0"})):
        for k in ("GDSW_PINV_HOST", "GDSW_LOCAL_FACTOR"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        prob, dec, cfg = build(PKG, CASES[name])
        skel = sw.setup_symbolic(prob.a, dec, cfg)
        pre = sw.setup_numeric(skel, prob.a, prob.nullspace if cfg.use_coarse else None)
        r = probes(prob.a.nrows, ks=(5,))[0]
        y = torch.empty(skel._local_plan["n_loc"], dtype=torch.float64, device="cuda")
        pre._dev.local_solve(torch.from_numpy(r).cuda(), y)
        out[mode] = y.cpu().numpy()
    scale = np.abs(out["stream"]).max()
    assert np.abs(out["device"] - out["host"]).max() <= 1e-13 * scale
    assert np.abs(out["device"] - out["stream"]).max() <= LONG_ROW_TOL * scale


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["double", "single"])
def test_factored_coarse_solve_matches_dense_inverse(monkeypatch, precision):
    """The factored coarse solve (supernodal partitioned inverse, one launch
    per tree level) against the dense A0^-1 GEMV on the same preconditioner:
    8x8x8 boxes, n_c = 2,744 (fp64 1e-12, fp32 1e-5 relative)."""
    prob = mp.assemble_laplace3d(mp.Grid3D(32, 32, 32))
    dec = dd.decompose(prob.a, dd.box_partition(prob.grid, 8, 8, 8), 1, "rgdsw")
    cfg = sw.SchwarzConfig(local=ls.SolverSpec("fast_ilu", 0, 3, 5), ordering="natural",
                           precision=precision)
    skel = sw.setup_symbolic(prob.a, dec, cfg)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("GDSW_COARSE_FACTOR", mode)
        pre = sw.setup_numeric(skel, prob.a, prob.nullspace)
        assert pre.coarse.a0.nrows == 2744
        out[mode] = [pre.apply(r) for r in probes(prob.a.nrows, ks=(1, 2))]
        if mode == "1":
            x_star, b = rhs(prob)
            _, rep = gmres(prob.a, pre, b, KrylovConfig(variant="single_reduce"))
            out["its"] = rep.iterations
    tol = 1e-12 if precision == "double" else 1e-5
    for z0, z1 in zip(out["0"], out["1"]):
        assert np.abs(z1 - z0).max() <= tol * np.abs(z0).max()
    assert out["its"] > 0


# ---------------------------------------------------------------------------
# properties and error paths (tests/test_schwarz.py:122-308 of the reference)
# ---------------------------------------------------------------------------
def test_apply_linearity_and_symmetry():
    prob, dec, cfg, skel, pre = setup_case("lap9_exact_nd")
    rng = np.random.default_rng(11)
    r = rng.standard_normal(prob.a.nrows)
    z1, z2 = pre.apply(2.5 * r), 2.5 * pre.apply(r)
    assert np.abs(z1 - z2).max() <= 1e-12 * np.abs(z2).max()
    s = rng.standard_normal(prob.a.nrows)
    assert abs(s @ pre.apply(r) - r @ pre.apply(s)) <= 1e-10 * abs(s @ pre.apply(r))


def test_apply_deterministic_and_threadsafe():
    from concurrent.futures import ThreadPoolExecutor
    prob, dec, cfg, skel, pre = setup_case("lap10_fast_nat")
    vecs = probes(prob.a.nrows, ks=range(10, 18))
    want = [pre.apply(r) for r in vecs]
    with ThreadPoolExecutor(max_workers=4) as ex:
        got = list(ex.map(pre.apply, vecs))
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


def test_apply_rejects_wrong_length():
    prob, dec, cfg, skel, pre = setup_case("lap9_onelevel_ilu0")
    with pytest.raises(ValueError, match="length"):
        pre.apply(np.zeros(5))


def test_refactorization_on_kept_skeleton_is_bitwise():
    prob, dec, cfg, skel, pre = setup_case("lap10_fast_nat")
    pre2 = sw.setup_numeric(skel, prob.a, prob.nullspace)
    r = probes(prob.a.nrows, ks=(3,))[0]
    assert np.array_equal(pre.apply(r), pre2.apply(r))
    a2 = CsrMatrix(prob.a.nrows, prob.a.ncols, prob.a.row_ptr, prob.a.col_idx, 2.0 * prob.a.values)
    pre3 = sw.setup_numeric(skel, a2, prob.nullspace)
    assert np.abs(pre3.apply(r) - 0.5 * pre.apply(r)).max() <= 1e-12 * np.abs(pre.apply(r)).max()


def test_singular_local_names_subdomain():
    a = CsrMatrix.from_dense(np.diag([1.0, 1.0, 1.0, 1.0, 1.0, 0.0]))
    part = dd.Partition(2, [0, 0, 0, 1, 1, 1])
    skel = sw.setup_symbolic(a, dd.decompose(a, part, 0), sw.SchwarzConfig(use_coarse=False))
    with pytest.raises(np.linalg.LinAlgError, match="subdomain 1"):
        sw.setup_numeric(skel, a)


def test_singular_coarse_named():
    n = 6
    d = np.full(n, 2.0)
    d[0] = d[-1] = 1.0
    t = np.diag(d) + np.diag(np.full(n - 1, -1.0), 1) + np.diag(np.full(n - 1, -1.0), -1)
    a = CsrMatrix.from_dense(t)
    part = dd.Partition(2, [0, 0, 0, 1, 1, 1])
    skel = sw.setup_symbolic(a, dd.decompose(a, part, 1, "gdsw"), sw.SchwarzConfig())
    with pytest.raises(np.linalg.LinAlgError, match="coarse matrix"):
        sw.setup_numeric(skel, a, np.ones((6, 1)))


def test_pattern_mismatch_and_missing_nullspace():
    prob, dec, cfg, skel, pre = setup_case("lap9_exact_nd")
    other = CsrMatrix.identity(prob.a.nrows)
    with pytest.raises(ValueError, match="pattern"):
        sw.setup_numeric(skel, other, prob.nullspace)
    with pytest.raises(ValueError, match="null space"):
        sw.setup_numeric(skel, prob.a, None)


def test_gmres_identity_zero_rhs_and_breakdown():
    n = 10
    ident = CsrMatrix.identity(n)
    b = np.random.default_rng(0).standard_normal(n)
    for variant in ("classic", "single_reduce"):
        x, rep = gmres(ident, None, b, KrylovConfig(variant=variant))
        assert rep.converged and rep.iterations == 1
        assert np.allclose(x, b, atol=1e-13)
        x, rep = gmres(ident, None, np.zeros(n), KrylovConfig(variant=variant))
        assert rep.converged and rep.iterations == 0 and list(rep.residual_history) == [1.0]
        dg = CsrMatrix.from_dense(np.diag([2.0, 3.0, 4.0]))
        x, rep = gmres(dg, None, np.array([5.0, 0.0, 0.0]), KrylovConfig(variant=variant))
        assert rep.converged and rep.iterations == 1
        assert np.allclose(x, [2.5, 0, 0], atol=1e-14)


def test_gmres_max_iters_reports_failure():
    prob = mp.assemble_laplace3d(mp.Grid3D(10, 10, 10))
    _, b = rhs(prob)
    x, rep = gmres(prob.a, None, b, KrylovConfig(variant="single_reduce", max_iters=37))
    assert not rep.converged and rep.iterations == 37
    assert len(rep.residual_history) == 38


def test_block_dot_matches_numpy():
    torch = _torch()
    from paper_2304_04876_b200.device import block_dot
    rng = np.random.default_rng(1)
    n, j = 100_003, 21
    V = rng.standard_normal((j, n))
    v, z = rng.standard_normal(n), rng.standard_normal(n)
    out = block_dot(torch.from_numpy(V).cuda(), j, torch.from_numpy(v).cuda(),
                    torch.from_numpy(z).cuda(), n)
    want = np.concatenate([V @ v, [v @ v], V @ z, [v @ z]])
    assert np.allclose(out, want, rtol=1e-12, atol=1e-9)


def test_sr_update_matches_reference_algebra():
    """gdsw_sr_update against krylov.py:346-351 in numpy, with and without
    the preconditioned basis."""
    torch = _torch()
    from paper_2304_04876_b200.device import sr_update
    rng = np.random.default_rng(2)
    n, j = 50_001, 7
    V = rng.standard_normal((j + 1, n))
    Zm = rng.standard_normal((j + 1, n))
    w, mc, zc = (rng.standard_normal(n) for _ in range(3))
    a, p = rng.standard_normal(j), rng.standard_normal(j)
    delta, corr = 1.7, 0.3
    coef = np.concatenate([a, p / delta, [delta, corr]])
    vj = (w - a @ V[:j]) / delta
    zj = (mc - a @ Zm[:j]) / delta
    wn = zc / delta - (p / delta) @ V[:j] - corr * vj
    for keep in (True, False):
        Vd, Zd = torch.from_numpy(V.copy()).cuda(), torch.from_numpy(Zm.copy()).cuda()
        wd = torch.from_numpy(w.copy()).cuda()
        sr_update(Vd, Zd if keep else None, j, torch.from_numpy(coef).cuda(), wd,
                  torch.from_numpy(mc).cuda(), torch.from_numpy(zc).cuda(), n)
        assert np.allclose(Vd[j].cpu().numpy(), vj, rtol=1e-12, atol=1e-12)
        assert np.allclose(wd.cpu().numpy(), wn, rtol=1e-12, atol=1e-12)
        if keep:
            assert np.allclose(Zd[j].cpu().numpy(), zj, rtol=1e-12, atol=1e-12)
        else:
            assert np.array_equal(Zd[j].cpu().numpy(), Zm[j])   # untouched


def test_supernodal_chunks_on_dense_and_arrow_blocks():
    """Exact factors with strictly nested row patterns take the streamed
    SpTRSV's supernodal chunks (GEMV over the shared external pattern,
    32-row diagonal tiles, panel updates): a dense block (one supernode, no
    external pattern) and an arrow block (a dense separator coupled to every
    earlier row), against the oracle's sequential substitution and a dense
    solve."""
    rng = np.random.default_rng(4)
    n, m1 = 150, 90
    d = rng.standard_normal((n, n))
    dense = d @ d.T + n * np.eye(n)
    arrow = np.zeros((n, n))
    for i in range(m1):
        arrow[i, i] = 4.0
        if i + 1 < m1:
            arrow[i, i + 1] = arrow[i + 1, i] = -1.0
    c = rng.standard_normal((n - m1, m1))
    arrow[m1:, :m1] = c
    arrow[:m1, m1:] = c.T
    s = rng.standard_normal((n - m1, n - m1))
    arrow[m1:, m1:] = s @ s.T + 4 * n * np.eye(n - m1)
    for mat in (dense, arrow):
        a = CsrMatrix.from_dense(mat)
        sym = ls.symbolic_lu(a, ls.order_natural(n))
        fac = ls.numeric_lu(a, sym)
        b = rng.standard_normal(n)
        x = fac.solve(b)
        want = O.levelset_solve(sym, fac.l_values, fac.u_values, b)
        assert np.abs(x - want).max() <= 1e-12 * np.abs(want).max()
        assert np.abs(mat @ x - b).max() <= 1e-10 * np.abs(b).max()
