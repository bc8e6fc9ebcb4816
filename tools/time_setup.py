"""Break setup_numeric into its phases on the GPU box:
    python tools/time_setup.py C2|C4|C5_512"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2304_04876_b200.schwarz as sw  # noqa: E402
from paper_2304_04876_b200 import device  # noqa: E402
from tools.run_configs import CONFIGS  # noqa: E402
from paper_2304_04876_b200.decomposition import box_partition, decompose  # noqa: E402
from paper_2304_04876_b200.model_problems import Grid3D, assemble_laplace3d  # noqa: E402

T = {}


def wrap(mod, name):
    f = getattr(mod, name)

    def g(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        T[name] = T.get(name, 0.0) + time.perf_counter() - t0
        return r
    setattr(mod, name, g)


import paper_2304_04876_b200.coarse_space as cs  # noqa: E402
for nm in ("coarse_columns", "coarse_desc", "check_extension_residual", "assemble_phi"):
    wrap(cs, nm)
for nm in ("extend_on_device", "numeric_lu", "symbolic_lu", "interface_basis",
           "convert_precision"):
    wrap(sw, nm)
for nm in ("fastilu", "set_coarse_inverse", "lu_numeric", "set_coarse", "extend", "panels", "coarse_galerkin"):
    wrap(device.Precond, nm)
wrap(device, "DeviceCsr")
wrap(sw.np.linalg, "inv")

name = sys.argv[1]
kind, n, p, spec, ordk, prec, *rest = CONFIGS[name]
prob = assemble_laplace3d(Grid3D(n, n, n))
dec = decompose(prob.a, box_partition(prob.grid, p, p, p), 1, "rgdsw")
cfg = sw.SchwarzConfig(local=spec, ordering=ordk, precision=prec)
skel = sw.setup_symbolic(prob.a, dec, cfg)
_ = skel.device_plan()
torch.cuda.synchronize()
t0 = time.perf_counter()
pre = sw.setup_numeric(skel, prob.a, prob.nullspace)
torch.cuda.synchronize()
print(name, "setup_numeric", round(time.perf_counter() - t0, 3), {k: round(v, 3) for k, v in T.items()})
