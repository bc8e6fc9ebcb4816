"""Golden numbers at BASELINE.json scale, produced by running the REFERENCE here.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_configs.py NAME [NAME ...]

One reference run per NAME (see CONFIGS): assemble, box partition, decompose,
setup_symbolic / setup_numeric, one apply of probe k=1 and one single-reduce
GMRES solve of b = A x* (x* = default_rng(0).standard_normal(n)), exactly as
the reference's own harness does (schwarzdd/bench.py:307-358).  Each run
writes tests/golden/configs/NAME.json (iteration count, residual history,
reduction counters, true residuals, decomposition hash, the apply probe's norm
and a strided sample of it, reference wall-clock per phase) and, for the
configs in FULL_APPLY, NAME.npz with the full apply vector.  Only this script touches
/root/reference; the fixtures travel to the GPU box.
"""

from __future__ import annotations

import json
import platform
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
OUT = HERE / "configs"
sys.path.insert(0, str(HERE.parent))
sys.path.insert(1, "/root/reference/pkg/src")

import schwarzdd.decomposition as dd  # noqa: E402  (the reference)
import schwarzdd.krylov as kr  # noqa: E402
import schwarzdd.local_solvers as ls  # noqa: E402
import schwarzdd.model_problems as mp  # noqa: E402
import schwarzdd.schwarz as sw  # noqa: E402

from cases import CONFIGS, FULL_APPLY, build, decomposition_hash, probes, rhs  # noqa: E402

PKG = (mp, dd, sw, ls)
SAMPLE_STRIDE = 997

def run(name: str) -> dict:
    case = CONFIGS[name]
    t0 = time.perf_counter()
    prob, dec, cfg = build(PKG, case)
    t1 = time.perf_counter()
    skel = sw.setup_symbolic(prob.a, dec, cfg)
    t2 = time.perf_counter()
    pre = sw.setup_numeric(skel, prob.a, prob.nullspace if cfg.use_coarse else None)
    t3 = time.perf_counter()
    n = prob.a.nrows
    r = probes(n, ks=(1,))[0]
    z = pre.apply(r)
    x_star, b = rhs(prob)
    x, rep = kr.gmres(prob.a, pre, b, kr.KrylovConfig(variant="single_reduce"))
    true_rel = float(np.linalg.norm(b - prob.a @ x) / np.linalg.norm(b))
    out = dict(
        case=[case[0], list(case[1]), list(case[2])] + list(case[3:]),
        n=n, n_coarse=(pre.coarse.a0.nrows if pre.coarse is not None else 0),
        nnz_phi=(pre.coarse.phi.nnz if pre.coarse is not None else 0),
        dec_hash=decomposition_hash(dec),
        iterations=rep.iterations, converged=rep.converged,
        residual_history=[float(v) for v in rep.residual_history],
        iteration_reductions=rep.iteration_reductions,
        residual_reductions=rep.residual_reductions, restarts=rep.restarts,
        true_residuals=[(int(i), float(v)) for i, v in rep.true_residuals],
        true_rel_residual=true_rel,
        true_error=float(np.linalg.norm(x - x_star) / np.linalg.norm(x_star)),
        apply_probe1_norm=float(np.linalg.norm(z)),
        apply_probe1_sample_stride=SAMPLE_STRIDE,
        apply_probe1_sample=[float(v) for v in z[::SAMPLE_STRIDE]],
        x_sample=[float(v) for v in x[::SAMPLE_STRIDE]],
        reference_seconds=dict(build=t1 - t0, symbolic=t2 - t1, numeric=t3 - t2,
                               solve=rep.timings.solve),
        host=dict(cpu=platform.processor() or platform.machine(), python=platform.python_version()),
        generator="tests/golden/make_golden_configs.py against /root/reference/pkg/src",
    )
    if name in FULL_APPLY:
        np.savez_compressed(OUT / f"{name}.npz", apply_probe1=z)
        out["apply_probe1_full"] = f"{name}.npz"
    return out


def main():
    OUT.mkdir(exist_ok=True)
    for name in sys.argv[1:]:
        print("config", name, flush=True)
        rec = run(name)
        (OUT / f"{name}.json").write_text(json.dumps(rec, indent=1))
        print(name, "iterations", rec["iterations"], "seconds", rec["reference_seconds"],
              flush=True)


if __name__ == "__main__":
    main()
