"""Generate the golden fixtures by running the REFERENCE itself.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--big]

Only this script touches /root/reference (read-only import); the fixtures it
writes (golden_*.npz, golden.json) are committed and travel to the GPU box.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(1, "/root/reference/pkg/src")

import schwarzdd.decomposition as dd  # noqa: E402  (the reference)
import schwarzdd.krylov as kr  # noqa: E402
import schwarzdd.local_solvers as ls  # noqa: E402
import schwarzdd.model_problems as mp  # noqa: E402
import schwarzdd.schwarz as sw  # noqa: E402

from cases import BIG, CASES, DRIFT_CASES, build, decomposition_hash, probes, rhs, sha  # noqa: E402

PKG = (mp, dd, sw, ls)


def one(name, case):
    prob, dec, cfg = build(PKG, case)
    skel = sw.setup_symbolic(prob.a, dec, cfg)
    pre = sw.setup_numeric(skel, prob.a, prob.nullspace if cfg.use_coarse else None)
    n = prob.a.nrows
    out = {"a_hash": sha(prob.a.row_ptr, prob.a.col_idx, prob.a.values),
           "dec_hash": decomposition_hash(dec), "structure_hash": skel.structure_hash,
           "n": n}
    arrays = {}
    for k, r in enumerate(probes(n)):
        arrays[f"apply_{k}"] = pre.apply(r)
    f0 = pre.local_factorizations[0]
    arrays["fac0_l"] = f0.l_values
    arrays["fac0_u"] = f0.u_values
    b0 = probes(len(skel.sets[0]), ks=(7,))[0]
    arrays["fac0_solve"] = f0.solve(b0)
    if f0.sweep_residuals is not None:
        arrays["fac0_sweep_res"] = np.asarray(f0.sweep_residuals)
    if pre.coarse is not None:
        arrays["phi_dense"] = pre.coarse.phi.to_dense()
        arrays["a0_dense"] = pre.coarse.a0.to_dense()
        arrays["a0_row_ptr"] = pre.coarse.a0.row_ptr
        arrays["a0_col_idx"] = pre.coarse.a0.col_idx
        out["n_coarse"] = pre.coarse.a0.nrows
    x_star, b = rhs(prob)
    for variant, orth in (("single_reduce", "mgs"), ("classic", "mgs"), ("classic_cgs2", "cgs2")):
        kcfg = kr.KrylovConfig(variant=variant.split("_")[0] if variant.startswith("classic")
                               else variant, orthogonalization=orth)
        x, rep = kr.gmres(prob.a, pre, b, kcfg)
        arrays[f"hist_{variant}"] = rep.residual_history
        arrays[f"x_{variant}"] = x
        out[variant] = dict(iterations=rep.iterations, converged=rep.converged,
                            iteration_reductions=rep.iteration_reductions,
                            residual_reductions=rep.residual_reductions,
                            restarts=rep.restarts,
                            true_residuals=[(int(i), float(v)) for i, v in rep.true_residuals])
    np.savez_compressed(HERE / f"golden_{name}.npz", **arrays)
    return out


def drift(name, case):
    """A deliberately nonlinear host operator (tests/cases.py drift_operator):
    the Givens estimate passes rel_tol while the true residual does not, so
    the solve keeps iterating after failed confirmations and restarts
    (krylov.py:331-342)."""
    from cases import DRIFT_EPS, drift_operator
    prob, dec, cfg = build(PKG, case)
    skel = sw.setup_symbolic(prob.a, dec, cfg)
    pre = sw.setup_numeric(skel, prob.a, prob.nullspace if cfg.use_coarse else None)
    _, b = rhs(prob)
    x, rep = kr.gmres(drift_operator(prob.a, DRIFT_EPS), pre, b,
                      kr.KrylovConfig(variant="single_reduce", max_iters=60))
    return dict(iterations=rep.iterations, converged=rep.converged, restarts=rep.restarts,
                iteration_reductions=rep.iteration_reductions,
                residual_reductions=rep.residual_reductions,
                residual_history=[float(v) for v in rep.residual_history],
                true_residuals=[(int(i), float(v)) for i, v in rep.true_residuals])


def big(name, case):
    t0 = time.perf_counter()
    prob, dec, cfg = build(PKG, case)
    skel = sw.setup_symbolic(prob.a, dec, cfg)
    pre = sw.setup_numeric(skel, prob.a, prob.nullspace)
    _, b = rhs(prob)
    _, rep = kr.gmres(prob.a, pre, b, kr.KrylovConfig(variant="single_reduce"))
    r = probes(prob.a.nrows, ks=(1,))[0]
    z = pre.apply(r)
    return dict(iterations=rep.iterations, converged=rep.converged, n=prob.a.nrows,
                dec_hash=decomposition_hash(dec),
                local_structure_hashes=sha(*[np.frombuffer(bytes.fromhex(s.structure_hash),
                                                           np.uint8)
                                             for s in skel.local_symbolics]),
                apply_probe1_norm=float(np.linalg.norm(z)), seconds=time.perf_counter() - t0)


def main():
    path = HERE / "golden.json"
    data = json.loads(path.read_text()) if path.exists() else {}
    data.setdefault("cases", {})
    data.setdefault("big", {})
    for name, case in CASES.items():
        print("case", name, flush=True)
        data["cases"][name] = one(name, case)
    data.setdefault("drift", {})
    for name in DRIFT_CASES:
        print("drift", name, flush=True)
        data["drift"][name] = drift(name, CASES[name])
    if "--big" in sys.argv:
        for name, case in BIG.items():
            print("big", name, flush=True)
            data["big"][name] = big(name, case)
    data["generator"] = "tests/golden/make_golden.py against /root/reference/pkg/src (schwarzdd 0.1.0)"
    path.write_text(json.dumps(data, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
