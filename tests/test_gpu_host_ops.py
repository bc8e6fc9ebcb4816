"""gmres with host operators: the reference's duck-typed operands
(krylov.py:88-100) -- callables and objects with `.apply` -- for A and M,
through gdsw_gmres_host_ops (GMRES vectors on the device, each operator call
staged through pinned host buffers). Cases follow the reference's
tests/test_krylov.py:321-399."""

import numpy as np
import pytest

from paper_2304_04876_b200.krylov import KrylovConfig, gmres
from paper_2304_04876_b200.sparse_core import CsrMatrix

pytestmark = pytest.mark.gpu


def tridiag(n):
    d = 2.0 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    return CsrMatrix.from_dense(d), d


@pytest.mark.parametrize("variant", ["classic", "single_reduce"])
def test_exact_inverse_converges_in_at_most_two_iterations(variant):
    for trial in range(10):
        rng = np.random.default_rng(100 + trial)
        n = int(rng.integers(20, 101))
        ad = rng.standard_normal((n, n)) + n * np.eye(n)
        b = rng.standard_normal(n)
        x, rep = gmres(lambda v: ad @ v, lambda v: np.linalg.solve(ad, v), b,
                       KrylovConfig(variant=variant))
        assert rep.converged and rep.iterations <= 2
        assert np.linalg.norm(ad @ x - b) <= 1e-10 * np.linalg.norm(b)


def test_csr_callable_and_apply_agree():
    a, ad = tridiag(15)
    b = np.random.default_rng(2).standard_normal(15)

    class Op:
        def apply(self, v):
            return ad @ v

    cfg = KrylovConfig(rel_tol=1e-10)
    x1, r1 = gmres(a, None, b, cfg)
    x2, r2 = gmres(lambda v: ad @ v, None, b, cfg)
    x3, r3 = gmres(Op(), None, b, cfg)
    assert np.allclose(x1, x2, atol=1e-10) and np.allclose(x1, x3, atol=1e-10)
    assert r1.iterations == r2.iterations == r3.iterations


@pytest.mark.parametrize("variant", ["classic", "single_reduce"])
def test_device_operator_with_host_preconditioner(variant):
    """A on the device, M a host callable: same iterations and solution as
    the same M given as a device CsrMatrix."""
    from paper_2304_04876_b200.model_problems import Grid3D, assemble_laplace3d
    prob = assemble_laplace3d(Grid3D(9, 9, 9))
    dinv = 1.0 / prob.a.to_dense().diagonal()
    mcsr = CsrMatrix.from_dense(np.diag(dinv))
    b = prob.a @ np.random.default_rng(0).standard_normal(prob.a.nrows)
    cfg = KrylovConfig(variant=variant)
    xd, rd = gmres(prob.a, mcsr, b, cfg)
    xh, rh = gmres(prob.a, lambda v: dinv * v, b, cfg)
    assert rd.converged and rh.converged and rd.iterations == rh.iterations
    assert np.linalg.norm(xd - xh) <= 1e-10 * np.linalg.norm(xd)
    assert rh.iteration_reductions == (rh.iterations if variant == "single_reduce"
                                       else rh.iteration_reductions)


def test_operator_errors_surface():
    a, ad = tridiag(6)

    def boom(v):
        raise ValueError("boom from the operator")

    with pytest.raises(ValueError, match="boom from the operator"):
        gmres(boom, None, np.ones(6))
    with pytest.raises(ValueError, match="dimensions"):
        gmres(lambda v: np.ones(5), None, np.ones(6))
    with pytest.raises(TypeError):
        gmres(object(), None, np.ones(6))
    with pytest.raises(TypeError):
        gmres(a, object(), np.ones(6))
    x, rep = gmres(lambda v: ad @ v, None, np.ones(6))   # still usable afterwards
    assert rep.converged and np.allclose(ad @ x, 1.0, atol=1e-6)
