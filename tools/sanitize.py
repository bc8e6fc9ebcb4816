"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every kernel family of the solve path on tiny cases.

    compute-sanitizer --tool racecheck python tools/sanitize.py [case ...]

Cases: fast (FastILU setup + Jacobi FastSpTRSV, SELL SpMV, coarse restrict /
solve / prolong, block dot, sr_update, pass graphs), exact (GPU numeric LU +
TMA-streamed SpTRSV with its mbarrier ring, supernodal chunks), ilu1 (ILU(k)
level-set, fp32 preconditioner), classic (MGS and CGS2 GMRES), gdsw.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2304_04876_b200.decomposition import box_partition, decompose  # noqa: E402
from paper_2304_04876_b200.krylov import KrylovConfig, gmres  # noqa: E402
from paper_2304_04876_b200.local_solvers import SolverSpec  # noqa: E402
from paper_2304_04876_b200.model_problems import (Grid3D, assemble_elasticity3d,  # noqa: E402
                                                  assemble_laplace3d)
from paper_2304_04876_b200.schwarz import SchwarzConfig, setup_numeric, setup_symbolic  # noqa: E402

CASES = {
    "fast": ("laplace", (10, 9, 8), (2, 2, 2), "rgdsw", SolverSpec("fast_ilu", 0, 3, 5),
             "natural", "double", "single_reduce"),
    "exact": ("elasticity", (7, 6, 6), (2, 2, 2), "rgdsw", SolverSpec("exact_lu"),
              "nested_dissection", "double", "single_reduce"),
    "ilu1": ("laplace", (10, 9, 8), (2, 2, 2), "rgdsw", SolverSpec("ilu_k", 1), "natural",
             "single", "single_reduce"),
    "classic": ("laplace", (9, 9, 9), (2, 2, 2), "rgdsw", SolverSpec("exact_lu"),
                "nested_dissection", "double", "classic"),
    "gdsw": ("laplace", (12, 12, 12), (3, 3, 3), "gdsw", SolverSpec("fast_ilu", 0, 3, 5),
             "natural", "single", "single_reduce"),
}


def run(name):
    kind, dims, parts, coarse, spec, ordering, prec, variant = CASES[name]
    g = Grid3D(*dims)
    prob = assemble_laplace3d(g) if kind == "laplace" else assemble_elasticity3d(g)
    dec = decompose(prob.a, box_partition(prob.grid, *parts), 1, coarse)
    cfg = SchwarzConfig(local=spec, ordering=ordering, precision=prec)
    skel = setup_symbolic(prob.a, dec, cfg)
    pre = setup_numeric(skel, prob.a, prob.nullspace)
    b = prob.a @ np.random.default_rng(0).standard_normal(prob.a.nrows)
    z = pre.apply(b)
    its = []
    for orth in (("mgs", "cgs2") if variant == "classic" else (None,)):
        kc = KrylovConfig(variant=variant) if orth is None else KrylovConfig(
            variant=variant, orthogonalization=orth)
        for _ in range(3):  # third call replays the captured pass graphs
            x, rep = gmres(prob.a, pre, b, kc)
        assert rep.converged
        its.append(rep.iterations)
    print(f"{name}: |z| {np.linalg.norm(z):.6e} iterations {its}", flush=True)


if __name__ == "__main__":
    for name in (sys.argv[1:] or list(CASES)):
        run(name)
