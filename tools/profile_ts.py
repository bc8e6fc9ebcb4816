"""Time the batched local solve (streamed SpTRSV) alone on a config:
    python tools/profile_ts.py C1 | C3s | C2ilu  [reps]
C3s = elasticity 32^3 with 4x4x4 boxes (C3's block size, 64 blocks)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2304_04876_b200.decomposition import box_partition, decompose  # noqa: E402
from paper_2304_04876_b200.local_solvers import SolverSpec  # noqa: E402
from paper_2304_04876_b200.model_problems import Grid3D, assemble_elasticity3d, assemble_laplace3d  # noqa: E402
from paper_2304_04876_b200.schwarz import SchwarzConfig, setup_numeric, setup_symbolic  # noqa: E402

CFG = {
    "C1": ("laplace", 30, 2, SolverSpec("exact_lu"), "nested_dissection"),
    "C3s": ("elasticity", 32, 4, SolverSpec("exact_lu"), "nested_dissection"),
    "C3": ("elasticity", 64, 8, SolverSpec("exact_lu"), "nested_dissection"),
    "C2ilu": ("laplace", 128, 4, SolverSpec("ilu_k", 0), "natural"),
    "ela_ilu1": ("elasticity", 32, 4, SolverSpec("ilu_k", 1), "natural"),
}


def main():
    name = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    kind, n, p, spec, ordk = CFG[name]
    g = Grid3D(n, n, n)
    prob = assemble_laplace3d(g) if kind == "laplace" else assemble_elasticity3d(g)
    dec = decompose(prob.a, box_partition(prob.grid, p, p, p), 1, "rgdsw")
    cfg = SchwarzConfig(local=spec, ordering=ordk, use_coarse=False)
    skel = setup_symbolic(prob.a, dec, cfg)
    import os
    import time
    os.environ["GDSW_HOST_LU"] = "1"
    t0 = time.perf_counter()
    setup_numeric(skel, prob.a, None)
    t_host = time.perf_counter() - t0
    os.environ["GDSW_HOST_LU"] = "0"
    setup_numeric(skel, prob.a, None)   # warm-up (schedules, streams)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pre = setup_numeric(skel, prob.a, None)
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    del os.environ["GDSW_HOST_LU"]
    print(f"{name}: numeric setup host IKJ {t_host:.3f} s, GPU {t_gpu:.3f} s", flush=True)
    nloc = skel._local_plan["n_loc"]
    r = torch.from_numpy(np.random.default_rng(1).standard_normal(prob.a.nrows)).cuda()
    y = torch.empty(nloc, dtype=torch.float64, device="cuda")
    for _ in range(3):
        pre._dev.local_solve(r, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        pre._dev.local_solve(r, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fill = sum(s.fill_nnz for s in skel.local_symbolics)
    nlev = [s.n_levels for s in skel.local_symbolics]
    gb = (fill * 12 + nloc * 28) / 1e9
    print(f"{name}: blocks {len(skel.local_symbolics)} n_loc {nloc} fill {fill} levels max {max(nlev)} "
          f"-> local solve {ms:.3f} ms, {gb / ms * 1e3:.0f} GB/s algorithmic", flush=True)


if __name__ == "__main__":
    main()
