"""Short C2 driver for ncu captures: set up the bench workload, then run
`--solves` GMRES solves inside cudaProfilerStart/Stop (use
`ncu --profile-from-start off`)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2304_04876_b200.krylov import KrylovConfig, gmres  # noqa: E402
from paper_2304_04876_b200.schwarz import setup_numeric, setup_symbolic  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=128)
p.add_argument("--parts", type=int, default=4)
p.add_argument("--solver", default="fast_ilu(0,3,5)")
p.add_argument("--ordering", default="natural")
p.add_argument("--precision", default="double")
p.add_argument("--solves", type=int, default=1)
p.add_argument("--max-iters", type=int, default=500)
a = p.parse_args()
a.gpus = 1
prob, dec, cfg = bench.build_problem(a)
pre = setup_numeric(setup_symbolic(prob.a, dec, cfg), prob.a, prob.nullspace)
b = torch.from_numpy(prob.a @ np.random.default_rng(0).standard_normal(prob.a.nrows)).cuda()
kc = KrylovConfig(variant="single_reduce", max_iters=a.max_iters)
gmres(prob.a, pre, b, kc)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(a.solves):
    x, rep = gmres(prob.a, pre, b, kc)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("iterations", rep.iterations)
