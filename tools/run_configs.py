"""Run BASELINE.json's configs end to end on the GPU and print one JSON line
each (setup times, iterations, solve time, true residual).

    python tools/run_configs.py C1 C2ilu C3 C4
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2304_04876_b200.decomposition import box_partition, decompose  # noqa: E402
from paper_2304_04876_b200.krylov import KrylovConfig, gmres  # noqa: E402
from paper_2304_04876_b200.local_solvers import SolverSpec  # noqa: E402
from paper_2304_04876_b200.model_problems import (Grid3D, assemble_elasticity3d,  # noqa: E402
                                                  assemble_laplace3d)
from paper_2304_04876_b200.schwarz import SchwarzConfig, setup_numeric, setup_symbolic  # noqa: E402

CONFIGS = {
    # name: (kind, n, boxes (p or (px, py, pz)), solver, ordering, precision[, coarse])
    "C1": ("laplace", 30, 2, SolverSpec("exact_lu"), "nested_dissection", "double"),
    "C2": ("laplace", 128, 4, SolverSpec("fast_ilu", 0, 3, 5), "natural", "double"),
    "C2ilu": ("laplace", 128, 4, SolverSpec("ilu_k", 0), "natural", "double"),
    "C2single": ("laplace", 128, 4, SolverSpec("fast_ilu", 0, 3, 5), "natural", "single"),
    "C3": ("elasticity", 64, 8, SolverSpec("exact_lu"), "nested_dissection", "double"),
    "C4": ("laplace", 200, 5, SolverSpec("fast_ilu", 0, 3, 5), "natural", "single"),
    "C4double": ("laplace", 200, 5, SolverSpec("fast_ilu", 0, 3, 5), "natural", "double"),
    "C5_512": ("laplace", 128, 8, SolverSpec("fast_ilu", 0, 3, 5), "natural", "double"),
    # the paper's subdomains-per-GPU study at 2M dof (128^3), fast_ilu(0,3,5)
    "C5_1": ("laplace", 128, 1, SolverSpec("fast_ilu", 0, 3, 5), "natural", "double", None),
    "C5_8": ("laplace", 128, 2, SolverSpec("fast_ilu", 0, 3, 5), "natural", "double"),
    "C5_64": ("laplace", 128, 4, SolverSpec("fast_ilu", 0, 3, 5), "natural", "double"),
    "C5_216": ("laplace", 128, 6, SolverSpec("fast_ilu", 0, 3, 5), "natural", "double"),
    "C5_256": ("laplace", 128, (8, 8, 4), SolverSpec("fast_ilu", 0, 3, 5), "natural", "double"),
    # large coarse spaces on one GPU (n_c = 8 (P-1)^3 style growth): 2,744 and 12,600
    "C5_2048": ("laplace", 128, (16, 16, 8), SolverSpec("fast_ilu", 0, 3, 5), "natural", "double"),
}


def run(name):
    kind, n, p, spec, ordk, prec, *rest = CONFIGS[name]
    coarse = rest[0] if rest else "rgdsw"
    px, py, pz = p if isinstance(p, tuple) else (p, p, p)
    t0 = time.perf_counter()
    grid = Grid3D(n, n, n)
    prob = assemble_laplace3d(grid) if kind == "laplace" else assemble_elasticity3d(grid)
    dec = decompose(prob.a, box_partition(prob.grid, px, py, pz), 1, coarse)
    t_in = time.perf_counter() - t0
    cfg = SchwarzConfig(local=spec, ordering=ordk, precision=prec, use_coarse=coarse is not None)
    t0 = time.perf_counter()
    skel = setup_symbolic(prob.a, dec, cfg)
    t_sym = time.perf_counter() - t0
    t0 = time.perf_counter()
    pre = setup_numeric(skel, prob.a, prob.nullspace if coarse else None)
    torch.cuda.synchronize()
    t_num = time.perf_counter() - t0
    x_star = np.random.default_rng(0).standard_normal(prob.a.nrows)
    b = prob.a @ x_star
    bd = torch.from_numpy(b).cuda()
    kc = KrylovConfig(variant="single_reduce")
    gmres(prob.a, pre, bd, kc)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, rep = gmres(prob.a, pre, bd, kc)
    e1.record()
    torch.cuda.synchronize()
    solve_ms = e0.elapsed_time(e1)
    xh = x.cpu().numpy()
    # preconditioner apply alone (side-stream overlap on), then one profiled
    # pass (overlap off: every event interval is one kernel's own) for the
    # coarse phase's share of the apply
    from paper_2304_04876_b200 import device
    r = torch.from_numpy(np.random.default_rng(1).standard_normal(prob.a.nrows)).cuda()
    for _ in range(3):
        pre.apply(r)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        pre.apply(r)
    e1.record()
    torch.cuda.synchronize()
    apply_ms = e0.elapsed_time(e1) / 20
    device.prof_reset()
    device.prof_enable(True)
    for _ in range(5):
        pre.apply(r)
    torch.cuda.synchronize()
    device.prof_enable(False)
    ph = device.prof_read()
    coarse_keys = [k for k in ph if k.startswith(("restrict", "coarse"))]
    coarse_ms = sum(ph[k]["ms"] for k in coarse_keys) / 5
    apply_prof_ms = sum(v["ms"] for v in ph.values()) / 5
    out = dict(config=name, n=prob.a.nrows, subdomains=px * py * pz,
               n_coarse=pre.coarse.a0.nrows if pre.coarse else 0,
               setup_s=dict(inputs=t_in, symbolic=t_sym, numeric=t_num),
               iterations=rep.iterations, converged=rep.converged,
               solve_ms=solve_ms, ms_per_iteration=solve_ms / max(rep.iterations, 1),
               true_rel_residual=float(np.linalg.norm(b - prob.a @ xh) / np.linalg.norm(b)),
               fill_nnz=int(sum(s.fill_nnz for s in skel.local_symbolics)),
               apply_ms=apply_ms, apply_profiled_ms=apply_prof_ms, coarse_phase_ms=coarse_ms,
               coarse_share=coarse_ms / apply_prof_ms if apply_prof_ms else None,
               phases_ms={k: round(v["ms"] / 5, 4) for k, v in ph.items()})
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for name in sys.argv[1:]:
        try:
            run(name)
        except Exception as e:  # keep going through the list
            print(json.dumps(dict(config=name, error=f"{type(e).__name__}: {e}")), flush=True)
