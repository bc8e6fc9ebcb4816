"""B200-native rGDSW-preconditioned single-reduce GMRES (solve path of
arXiv 2304.04876), a drop-in for the schwarzdd Python API.

Host modules mirror the reference interface (model_problems,
decomposition, local_solvers, coarse_space, schwarz, krylov); the solve path
runs in hand-written sm_100a kernels behind the C ABI of include/gdsw.h.
"""

from .sparse_core import CsrMatrix

__version__ = "0.1.0"
__all__ = ["CsrMatrix"]
