"""Coarse solve alone: apply of a 64^3 Laplace problem with 8x8x8 boxes
(n_c = 2,744) or 16x16x8 (n_c = 12,600) -- for ncu launch lists of the
factored vs dense coarse solve.
    GDSW_COARSE_FACTOR=1 python tools/profile_coarse.py 8 8 8 [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2304_04876_b200.decomposition import box_partition, decompose  # noqa: E402
from paper_2304_04876_b200.local_solvers import SolverSpec  # noqa: E402
from paper_2304_04876_b200.model_problems import Grid3D, assemble_laplace3d  # noqa: E402
from paper_2304_04876_b200.schwarz import SchwarzConfig, setup_numeric, setup_symbolic  # noqa: E402

px, py, pz = (int(v) for v in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
prob = assemble_laplace3d(Grid3D(64, 64, 64))
dec = decompose(prob.a, box_partition(prob.grid, px, py, pz), 1, "rgdsw")
cfg = SchwarzConfig(local=SolverSpec("fast_ilu", 0, 3, 5), ordering="natural")
pre = setup_numeric(setup_symbolic(prob.a, dec, cfg), prob.a, prob.nullspace)
r = torch.from_numpy(np.random.default_rng(1).standard_normal(prob.a.nrows)).cuda()
for _ in range(reps):
    pre.apply(r)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    pre.apply(r)
e1.record()
torch.cuda.synchronize()
print(f"n_c {pre.coarse.a0.nrows}: apply {e0.elapsed_time(e1) / 20:.3f} ms")
