"""Parity cases shared by the golden generator (run against the reference)
and the tests (run against the oracle and the CUDA path).

Each case is built the same way the reference's own tests and bench do
(tests/test_acceptance.py:64-75, bench.py:307-358): assemble, box
partition, decompose, setup_symbolic / setup_numeric, b = A x* with
x* = default_rng(seed).standard_normal(n), GMRES rtol 1e-7.
"""

from __future__ import annotations

import hashlib

import numpy as np

# name: (kind, dims, parts, coarse, method, fill, sweeps, iters, precision, ordering, overlap)
CASES = {
    "lap9_exact_nd": ("laplace3d", (9, 9, 9), (2, 2, 2), "rgdsw", "exact_lu", 0, 3, 5,
                      "double", "nested_dissection", 1),
    "lap10_fast_nat": ("laplace3d", (10, 9, 8), (2, 2, 2), "rgdsw", "fast_ilu", 0, 3, 5,
                       "double", "natural", 1),
    "lap10_ilu1_single": ("laplace3d", (10, 9, 8), (2, 2, 2), "rgdsw", "ilu_k", 1, 3, 5,
                          "single", "natural", 1),
    "lap12_fast_single_gdsw": ("laplace3d", (12, 12, 12), (3, 3, 3), "gdsw", "fast_ilu", 0, 3,
                               5, "single", "natural", 1),
    "lap9_onelevel_ilu0": ("laplace3d", (9, 9, 9), (2, 2, 1), "none", "ilu_k", 0, 3, 5,
                           "double", "nested_dissection", 1),
    "ela7_ilu0": ("elasticity3d", (7, 6, 6), (2, 2, 2), "rgdsw", "ilu_k", 0, 3, 5, "double",
                  "natural", 1),
    "ela7_exact": ("elasticity3d", (7, 6, 6), (2, 2, 2), "rgdsw", "exact_lu", 0, 3, 5,
                   "double", "nested_dissection", 1),
    "lap11_fast12_ovl2": ("laplace3d", (11, 11, 11), (2, 2, 2), "rgdsw", "fast_ilu", 1, 2, 7,
                          "double", "natural", 2),
}

# iteration-count goldens at larger sizes (single_reduce, rtol 1e-7), from
# running the reference here (make_golden.py --big); C1 is BASELINE config 0
BIG = {
    "C1_lap30_exact": ("laplace3d", (30, 30, 30), (2, 2, 2), "rgdsw", "exact_lu", 0, 3, 5,
                       "double", "nested_dissection", 1),
    "lap24_fast_4x4x4": ("laplace3d", (24, 24, 24), (4, 4, 4), "rgdsw", "fast_ilu", 0, 3, 5,
                         "double", "natural", 1),
    "lap17_exact_3x3x3": ("laplace3d", (17, 17, 17), (3, 3, 3), "rgdsw", "exact_lu", 0, 3, 5,
                          "double", "nested_dissection", 1),
    "ela12_fast_2x2x2": ("elasticity3d", (12, 12, 12), (2, 2, 2), "rgdsw", "fast_ilu", 0, 3, 5,
                         "double", "natural", 1),
    "lap20_single_fast": ("laplace3d", (20, 20, 20), (2, 2, 2), "rgdsw", "fast_ilu", 0, 3, 5,
                          "single", "natural", 1),
}


# name: (kind, dims, parts, coarse, method, fill, sweeps, iters, precision, ordering, overlap)
# BASELINE-scale configurations run by the reference (make_golden_configs.py)
CONFIGS = {
    # BASELINE configs[1] (C2) and its level-set companion
    "C2_fast": ("laplace3d", (128, 128, 128), (4, 4, 4), "rgdsw", "fast_ilu", 0, 3, 5,
                "double", "natural", 1),
    "C2_ilu0": ("laplace3d", (128, 128, 128), (4, 4, 4), "rgdsw", "ilu_k", 0, 3, 5,
                "double", "natural", 1),
    # BASELINE configs[2] (C3): elasticity 64^3, exact LU + ND, P=8
    "C3_ela64_exact_p8": ("elasticity3d", (64, 64, 64), (8, 8, 8), "rgdsw", "exact_lu", 0, 3,
                          5, "double", "nested_dissection", 1),
    # the subdomain sweep trend of configs[4] (C5) at 64^3
    "lap64_fast_p2": ("laplace3d", (64, 64, 64), (2, 2, 2), "rgdsw", "fast_ilu", 0, 3, 5,
                      "double", "natural", 1),
    "lap64_fast_p4": ("laplace3d", (64, 64, 64), (4, 4, 4), "rgdsw", "fast_ilu", 0, 3, 5,
                      "double", "natural", 1),
    "lap64_fast_p8": ("laplace3d", (64, 64, 64), (8, 8, 8), "rgdsw", "fast_ilu", 0, 3, 5,
                      "double", "natural", 1),
    "lap64_ilu0_p2": ("laplace3d", (64, 64, 64), (2, 2, 2), "rgdsw", "ilu_k", 0, 3, 5,
                      "double", "natural", 1),
    "lap64_ilu0_p4": ("laplace3d", (64, 64, 64), (4, 4, 4), "rgdsw", "ilu_k", 0, 3, 5,
                      "double", "natural", 1),
    "lap64_ilu0_p8": ("laplace3d", (64, 64, 64), (8, 8, 8), "rgdsw", "ilu_k", 0, 3, 5,
                      "double", "natural", 1),
    "lap64_fast_p4_single": ("laplace3d", (64, 64, 64), (4, 4, 4), "rgdsw", "fast_ilu", 0, 3,
                             5, "single", "natural", 1),
    "lap64_ilu0_p8_single": ("laplace3d", (64, 64, 64), (8, 8, 8), "rgdsw", "ilu_k", 0, 3, 5,
                             "single", "natural", 1),
    # elasticity with the rigid-body coarse space
    "ela24_exact_p4": ("elasticity3d", (24, 24, 24), (4, 4, 4), "rgdsw", "exact_lu", 0, 3, 5,
                       "double", "nested_dissection", 1),
    # BASELINE configs[3] (C4) shape at a size the reference's dense harmonic
    # extension can finish: fp32 preconditioner, fast_ilu, P=5
    "C4_lap100_single_p5": ("laplace3d", (100, 100, 100), (5, 5, 5), "rgdsw", "fast_ilu", 0, 3,
                            5, "single", "natural", 1),
}


# configs whose full apply vector is stored (the rest keep a strided sample)
FULL_APPLY = ("lap64_fast_p4", "lap64_fast_p4_single", "lap64_ilu0_p4", "ela24_exact_p4")

# cases re-solved with a deliberately nonlinear operator (drift_operator):
# the GMRES estimate passes rtol while the true residual does not
DRIFT_CASES = ("lap10_fast_nat",)
DRIFT_EPS = 0.02


def drift_operator(a, eps: float):
    """x -> A x + eps ||x|| u (u a fixed unit vector): not linear, so the
    Givens estimate drifts from the true residual ||b - A x|| and the
    true-residual confirmation fails (krylov.py:331-342)."""
    u = np.random.default_rng(11).standard_normal(a.nrows)
    u /= np.linalg.norm(u)

    def op(x):
        return a @ x + eps * np.linalg.norm(x) * u
    return op


def build(pkg, case, nullspace_needed=True):
    """Build (prob, dec, config) with module namespace `pkg` exposing
    model_problems, decomposition, schwarz, local_solvers."""
    kind, dims, parts, coarse, method, fill, sweeps, iters, prec, ordk, ovl = case
    mp, dd, sw, ls = pkg
    grid = mp.Grid3D(*dims)
    prob = mp.assemble_laplace3d(grid) if kind == "laplace3d" else mp.assemble_elasticity3d(grid)
    part = dd.box_partition(prob.grid, *parts)
    mode = None if coarse == "none" else coarse
    dec = dd.decompose(prob.a, part, ovl, mode)
    cfg = sw.SchwarzConfig(local=ls.SolverSpec(method, fill, sweeps, iters),
                           use_coarse=mode is not None, precision=prec, ordering=ordk)
    return prob, dec, cfg


def probes(n: int, ks=(1, 2)):
    return [np.random.default_rng(k).standard_normal(n) for k in ks]


def rhs(prob, seed: int = 0):
    x_star = np.random.default_rng(seed).standard_normal(prob.a.nrows)
    return x_star, prob.a @ x_star


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def decomposition_hash(dec) -> str:
    h = hashlib.sha256()
    for s in dec.overlap.sets:
        h.update(np.asarray(s, np.int64).tobytes())
    st = dec.structure
    if st is not None:
        for arr in (st.interior, st.interface, st.multiplicity):
            h.update(np.asarray(arr, np.int64).tobytes())
        for c in st.components:
            h.update(np.asarray(c.dofs, np.int64).tobytes())
            h.update(np.asarray(c.weights, np.float64).tobytes())
            h.update(c.kind.encode())
            h.update(np.array(sorted(c.subdomains), np.int64).tobytes())
    return h.hexdigest()
