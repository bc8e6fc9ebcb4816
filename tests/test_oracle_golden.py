"""Pin the ORACLE against the reference: golden vectors produced by running
the reference itself (tests/golden/make_golden.py). The oracle's kernels
are sequential restatements compiled without FMA contraction, so apply
vectors, local factors and GMRES histories match bit for bit. CPU only."""

import json

import numpy as np
import pytest

from cases import CASES, build, probes, rhs
from oracle import oracle as O
from paper_2304_04876_b200 import decomposition as dd
from paper_2304_04876_b200 import local_solvers as ls
from paper_2304_04876_b200 import model_problems as mp
from paper_2304_04876_b200 import schwarz as sw
from paper_2304_04876_b200.sparse_core import extract_submatrix

PKG = (mp, dd, sw, ls)


@pytest.fixture(scope="module")
def golden(golden_dir):
    return json.loads((golden_dir / "golden.json").read_text())


def _oracle(name):
    prob, dec, cfg = build(PKG, CASES[name])
    return prob, dec, cfg, O.OracleSchwarz(prob.a, dec, cfg,
                                           prob.nullspace if cfg.use_coarse else None)


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_apply_matches_reference(golden_dir, name):
    prob, dec, cfg, ore = _oracle(name)
    g = np.load(golden_dir / f"golden_{name}.npz")
    for k, r in enumerate(probes(prob.a.nrows)):
        z = ore.apply(r)
        want = g[f"apply_{k}"]
        # the oracle forms A0 with scipy (different SpGEMM summation order);
        # everything else is the reference's own operation sequence
        assert np.abs(z - want).max() <= 1e-13 * np.abs(want).max()


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_local_factor_and_solve_bitwise(golden_dir, name):
    prob, dec, cfg, ore = _oracle(name)
    g = np.load(golden_dir / f"golden_{name}.npz")
    lv, uv, res = ore.factors[0]
    assert np.array_equal(lv, g["fac0_l"])
    assert np.array_equal(uv, g["fac0_u"])
    if res is not None:
        assert np.allclose(res, g["fac0_sweep_res"], rtol=1e-12, atol=0)
    b0 = probes(len(dec.overlap.sets[0]), ks=(7,))[0]
    sol = ore.local_solve(0, b0.astype(lv.dtype))
    assert np.array_equal(sol, g["fac0_solve"])


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_gmres_matches_reference(golden, golden_dir, name):
    prob, dec, cfg, ore = _oracle(name)
    g = np.load(golden_dir / f"golden_{name}.npz")
    _, b = rhs(prob)
    for variant, orth in (("single_reduce", "mgs"), ("classic", "mgs"), ("classic_cgs2", "cgs2")):
        x, rep = O.gmres(lambda v: O.csr_spmv(prob.a, v), ore.apply, b,
                         variant=variant.split("_cgs2")[0], orthogonalization=orth)
        want = golden["cases"][name][variant]
        assert rep["iterations"] == want["iterations"]
        assert rep["converged"] == want["converged"]
        assert rep["iteration_reductions"] == want["iteration_reductions"]
        assert rep["residual_reductions"] == want["residual_reductions"]
        assert np.allclose(rep["history"], g[f"hist_{variant}"], rtol=1e-9, atol=1e-15)
        assert np.abs(x - g[f"x_{variant}"]).max() <= 1e-9 * np.abs(x).max()


@pytest.mark.parametrize("name", ["lap10_fast_nat"])
def test_oracle_gmres_drift_matches_reference(golden, name):
    """Nonlinear operator: failed true-residual confirmations, then a restart
    (krylov.py:331-342) -- the oracle follows the reference's path."""
    from cases import DRIFT_EPS, drift_operator
    prob, dec, cfg, ore = _oracle(name)
    _, b = rhs(prob)
    x, rep = O.gmres(drift_operator(prob.a, DRIFT_EPS), ore.apply, b, max_iters=60)
    want = golden["drift"][name]
    assert rep["iterations"] == want["iterations"]
    assert rep["converged"] == want["converged"]
    assert len(want["true_residuals"]) > 2
    assert [i for i, _ in rep["true_residuals"]] == [i for i, _ in want["true_residuals"]]
    assert np.allclose([v for _, v in rep["true_residuals"]],
                       [v for _, v in want["true_residuals"]], rtol=1e-6)


def test_oracle_coarse_basis_matches_reference(golden_dir):
    for name in ("lap9_exact_nd", "ela7_ilu0"):
        prob, dec, cfg, ore = _oracle(name)
        g = np.load(golden_dir / f"golden_{name}.npz")
        phi = ore.coarse[0].to_dense()
        want = g["phi_dense"]
        assert phi.shape == want.shape
        assert np.abs(phi - want).max() <= 1e-14 * np.abs(want).max()


def test_oracle_kernels_on_dense_oracles():
    """Independent dense checks of the restated kernels (the reference's own
    test strategy: tests/test_local_solvers.py:549-565, 634-659)."""
    prob = mp.assemble_laplace3d(mp.Grid3D(6, 5, 4))
    a = prob.a
    sym = ls.symbolic_lu(a, ls.make_ordering(a, "nested_dissection"))
    lv, uv = O.lu_numeric(a, sym)
    rng = np.random.default_rng(3)
    b = rng.standard_normal(a.nrows)
    x = O.levelset_solve(sym, lv, uv, b)
    assert np.abs(a.to_dense() @ x - b).max() <= 1e-10 * np.abs(b).max()
    # Jacobi on exact factors reaches the exact solve at the dependency depth
    depth = max(sym.n_levels)
    xj = O.jacobi_solve(sym, lv, uv, b, depth + 1)
    assert np.abs(xj - x).max() <= 1e-9 * np.abs(x).max()
    y = O.spmv(a.row_ptr, a.col_idx, a.values, x)
    assert np.array_equal(y, a @ x)
    blk = extract_submatrix(a, np.arange(10), np.arange(10))
    assert blk.nrows == 10


# ---------------------------------------------------------------------------
# the reference arm's own setup (oracle/reference_setup.py): pinned against
# the reference's decomposition hashes and apply, independent of the product
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,n,p", [("lap64_fast_p4", 64, 4), ("lap64_fast_p8", 64, 8)])
def test_reference_setup_decomposition_matches_reference(golden_dir, name, n, p):
    import json

    from oracle import reference_setup as R
    want = json.loads((golden_dir / "configs" / f"{name}.json").read_text())
    a, _ = R.assemble_laplace3d(n, n, n)
    owner = R.box_partition(n, n, n, p, p, p)
    sets = R.extend_overlap(a, owner, p ** 3, 1)
    st = R.build_rgdsw(R.classify_interface(a, owner))
    assert R.decomposition_hash(sets, st) == want["dec_hash"]
    assert len(st.components) == want["n_coarse"]


def test_reference_setup_apply_and_solve_match_reference(golden_dir):
    """64^3, 4x4x4, fast_ilu(0,3,5): the independently built preconditioner
    applies like the reference (1e-10) and GMRES takes its iteration count;
    the build loads nothing of the product."""
    import json
    import subprocess
    import sys
    code = (
        "import sys, json, numpy as np\n"
        f"sys.path.insert(0, {str(golden_dir.parents[1])!r})\n"
        "from oracle import reference_setup as R\n"
        "from oracle import oracle as O\n"
        "S = R.IndependentSchwarz(64, 64, 64, 4, 4, 4, threads=4)\n"
        "r = np.random.default_rng(1).standard_normal(64 ** 3)\n"
        f"zr = np.load({str(golden_dir / 'configs' / 'lap64_fast_p4.npz')!r})['apply_probe1']\n"
        "rel = float(np.abs(S.apply(r) - zr).max() / np.abs(zr).max())\n"
        "b = S.a @ np.random.default_rng(0).standard_normal(64 ** 3)\n"
        "_, rep = O.gmres(lambda v: O.csr_spmv(S.a, v), S.apply, b)\n"
        "mods = sorted(m for m in sys.modules if m.startswith('paper_2304'))\n"
        "print(json.dumps(dict(rel=rel, its=rep['iterations'], mods=mods)))\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=600, check=True).stdout
    got = json.loads(out.strip().splitlines()[-1])
    want = json.loads((golden_dir / "configs" / "lap64_fast_p4.json").read_text())
    assert got["rel"] <= 1e-10
    assert got["its"] == want["iterations"]
    assert got["mods"] == []
