"""ctypes binding of libgdsw.so (include/gdsw.h) and the device-side objects.

This is the reference-side FFI shim: numpy descriptors and torch device
tensors in, the C ABI's opaque handles and status codes out. Status codes
are re-raised as the exception types the reference raises for the same
condition. There is no CPU fallback: importing this module without the
library, or calling it without a CUDA device, raises.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libgdsw.so"
_p64 = C.POINTER(C.c_int64)


class _LocalDesc(C.Structure):
    _fields_ = [("n", C.c_int64), ("n_sub", C.c_int32), ("method", C.c_int32),
                ("n_loc", C.c_int64)] + [
        (name, C.c_void_p) for name in (
            "sub_ptr", "gmap", "l_ptr", "l_idx", "u_ptr", "u_idx", "llev_sub", "llev_ptr",
            "llev_rows", "ulev_sub", "ulev_ptr", "ulev_rows", "a_of", "fi_ptr", "fi_pl",
            "fi_pu")] + [("n_res", C.c_int64)] + [
        (name, C.c_void_p) for name in (
            "res_sub_ptr", "res_a", "res_ptr", "res_pl", "res_pu", "res_tl", "res_tu")]


class _CoarseDesc(C.Structure):
    _fields_ = [("n_c", C.c_int32), ("n_gamma", C.c_int64)] + [
        (name, C.c_void_p) for name in (
            "gamma_rows", "pg_ptr", "pg_col", "pg_val", "int_ptr", "int_rows", "col_ptr",
            "col_ids", "aii_ptr", "aii_col", "aii_src", "aig_ptr", "aig_col", "aig_src")]


_CF_ARRAYS = ("level_ptr", "sn_s", "sn_r", "col_ptr", "col_ids", "row_ptr", "row_ids", "d_off",
              "m_off", "n_off", "in_ptr", "in_idx", "out_ptr", "out_idx")


class _CoarseFactor(C.Structure):
    _fields_ = ([("n", C.c_int32), ("n_sn", C.c_int32), ("n_levels", C.c_int32)] +
                [(k, C.c_void_p) for k in _CF_ARRAYS] +
                [("values", C.c_void_p), ("n_values", C.c_int64)])


class _KrylovCfg(C.Structure):
    _fields_ = [("restart", C.c_int32), ("rel_tol", C.c_double), ("max_iters", C.c_int32),
                ("variant", C.c_int32), ("orthogonalization", C.c_int32)]


class _Report(C.Structure):
    _fields_ = [(k, C.c_int32) for k in (
        "iterations", "converged", "reduction_count", "iteration_reductions",
        "residual_reductions", "restarts", "n_history", "n_true")]


_SIGS = {
    "gdsw_last_error": (C.c_char_p, []),
    "gdsw_abi_version": (C.c_int, []),
    "gdsw_csr_create": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_int]),
    "gdsw_csr_set_values": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gdsw_csr_spmv": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                                C.c_void_p]),
    "gdsw_csr_destroy": (C.c_int, [C.c_void_p]),
    "gdsw_plan_create": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gdsw_plan_destroy": (C.c_int, [C.c_void_p]),
    "gdsw_precond_create": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    "gdsw_precond_set_coarse": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gdsw_precond_set_factors": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "gdsw_precond_fastilu": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "gdsw_precond_get_factors": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "gdsw_plan_set_block_pattern": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gdsw_precond_lu_numeric": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, C.c_void_p]),
    "gdsw_precond_coarse_galerkin": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gdsw_dist_coarse_galerkin": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.c_void_p]),
    "gdsw_sr_update": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int32, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gdsw_precond_extend": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_void_p,
                                      C.c_void_p]),
    "gdsw_precond_panel_entries": (C.c_int64, [C.c_void_p]),
    "gdsw_precond_get_panels": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gdsw_precond_set_coarse_inverse": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gdsw_precond_set_coarse_factor": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gdsw_precond_set_local_factor": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gdsw_precond_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gdsw_precond_local_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                           C.c_void_p]),
    "gdsw_precond_destroy": (C.c_int, [C.c_void_p]),
    "gdsw_workspace_create": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32]),
    "gdsw_workspace_destroy": (C.c_int, [C.c_void_p]),
    "gdsw_gmres": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                             C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                             C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "gdsw_gmres_host_ops": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                      C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "gdsw_block_dot": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                                 C.c_int64, C.c_void_p, C.c_void_p]),
    "gdsw_dist_create": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                   C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_int64]),
    "gdsw_dist_ipc_handle": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gdsw_dist_open_peers": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gdsw_dist_allreduce": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "gdsw_dist_halo": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "gdsw_dist_destroy": (C.c_int, [C.c_void_p]),
    "gdsw_precond_set_dist": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gdsw_gmres_dist": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "gdsw_launch_count": (C.c_int64, []),
    "gdsw_prof_enable": (C.c_int, [C.c_int]),
    "gdsw_prof_reset": (C.c_int, []),
    "gdsw_prof_count": (C.c_int, []),
    "gdsw_prof_name": (C.c_char_p, [C.c_int]),
    "gdsw_prof_read": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
}

EXPORTED = tuple(_SIGS)


def load_library():
    if not _LIB_PATH.exists():
        raise ImportError(f"{_LIB_PATH} is missing; run `python -m "
                          "paper_2304_04876_b200.build` (no CPU fallback exists)")
    lib = C.CDLL(str(_LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = load_library()

F64, F32 = 0, 1
METHODS = {"exact_lu": 0, "ilu_k": 1, "fast_ilu": 2}


def _raise(code: int):
    msg = _lib.gdsw_last_error().decode()
    if code == 1:
        raise ValueError(msg)
    if code == 2:
        raise np.linalg.LinAlgError(msg)
    if code == 3:
        raise FloatingPointError(msg)
    if code == 4:
        raise ArithmeticError(msg)
    if code == 6:
        raise TypeError(msg)
    raise RuntimeError(msg)


def _ck(code: int):
    if code != 0:
        _raise(code)


def _ptr(a) -> C.c_void_p:
    if a is None:
        return C.c_void_p(0)
    if isinstance(a, np.ndarray):
        return C.c_void_p(a.ctypes.data)
    return C.c_void_p(a.data_ptr())   # torch tensor


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        if not t.cuda.is_available():
            raise RuntimeError("the B200 solve path needs a CUDA device (no CPU fallback)")
        _torch = t
    return _torch


def stream_handle():
    return C.c_void_p(torch().cuda.current_stream().cuda_stream)


def dtype_code(np_dtype) -> int:
    return F32 if np.dtype(np_dtype) == np.float32 else F64


# ---------------------------------------------------------------------------
class DeviceCsr:
    """A CsrMatrix resident on the GPU in SELL-32 layout."""

    def __init__(self, a):
        self.nrows, self.ncols = a.nrows, a.ncols
        self.nnz = a.nnz
        self.dtype = np.dtype(a.values.dtype)
        vals = np.ascontiguousarray(a.values)
        h = C.c_void_p()
        _ck(_lib.gdsw_csr_create(C.byref(h), a.nrows, a.ncols, _ptr(_i64(a.row_ptr)),
                                 _ptr(_i64(a.col_idx)), _ptr(vals), dtype_code(self.dtype)))
        self.handle = h

    def set_values(self, values: np.ndarray):
        _ck(_lib.gdsw_csr_set_values(self.handle, _ptr(np.ascontiguousarray(values, self.dtype))))

    def spmv(self, x, y, alpha=1.0, beta=0.0):
        _ck(_lib.gdsw_csr_spmv(self.handle, _ptr(x), _ptr(y), alpha, beta, stream_handle()))
        return y

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            _lib.gdsw_csr_destroy(h)
            self.handle = None


def to_host(xd):
    """Device tensor -> host tensor through the caching pinned allocator
    (a pageable .cpu() of a 16 MB vector costs ~5 ms, this ~0.3 ms)."""
    t = torch()
    out = t.empty(xd.shape, dtype=xd.dtype, pin_memory=True)
    out.copy_(xd, non_blocking=True)
    t.cuda.current_stream().synchronize()
    return out


def device_csr(a) -> DeviceCsr:
    """Cached float64 device copy of a host CsrMatrix (the GMRES operator is
    float64: a float32 matrix is lifted once and the lifted copy cached).

    The cache is keyed on the values array object, and that array is made
    read-only while it backs a device copy: an in-place edit
    (``a.values *= 2``) raises instead of silently solving with stale
    values (the reference reads the current values on every spmv); assign a
    new array, or build a new CsrMatrix, to change the operator."""
    cached = getattr(a, "_device_copy", None)
    if cached is not None and cached[0] is a.values:
        return cached[1]
    src = a
    if a.values.dtype != np.float64:
        from .sparse_core import CsrMatrix
        src = CsrMatrix(a.nrows, a.ncols, a.row_ptr, a.col_idx, a.values.astype(np.float64))
    d = DeviceCsr(src)
    try:
        a.values.flags.writeable = False
        object.__setattr__(a, "_device_copy", (a.values, d))
    except Exception:
        pass
    return d


class Plan:
    """Device symbolic plan (gdsw_plan_create)."""

    def __init__(self, local: dict):
        keep = []
        ld = _LocalDesc()
        ld.n, ld.n_sub, ld.method, ld.n_loc = (local["n"], local["n_sub"], local["method"],
                                               local["n_loc"])
        for name in ("sub_ptr", "gmap", "l_ptr", "l_idx", "u_ptr", "u_idx", "llev_sub",
                     "llev_ptr", "llev_rows", "ulev_sub", "ulev_ptr", "ulev_rows", "a_of",
                     "fi_ptr", "fi_pl", "fi_pu", "res_sub_ptr", "res_a", "res_ptr", "res_pl",
                     "res_pu", "res_tl", "res_tu"):
            if local.get(name) is not None:
                a = _i64(local[name])
                keep.append(a)
                setattr(ld, name, a.ctypes.data)
        ld.n_res = local.get("n_res", 0)
        h = C.c_void_p()
        _ck(_lib.gdsw_plan_create(C.byref(h), C.cast(C.pointer(ld), C.c_void_p)))
        self.handle = h
        self.n = local["n"]
        self.n_loc = local["n_loc"]
        self.n_sub = local["n_sub"]
        self.nnz_l = int(local["l_ptr"][-1])
        self.nnz_u = int(local["u_ptr"][-1])
        self.has_block_pattern = local.get("ab_ptr") is not None
        if self.has_block_pattern:
            ab = [_i64(local[k]) for k in ("ab_ptr", "ab_idx", "ab_src")]
            _ck(_lib.gdsw_plan_set_block_pattern(h, *[_ptr(x) for x in ab]))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            _lib.gdsw_plan_destroy(h)
            self.handle = None


class Precond:
    """Numeric preconditioner arena (gdsw_precond_*)."""

    def __init__(self, plan: Plan, value_dtype, trisolve_iters: int):
        self.plan = plan
        self.value_dtype = np.dtype(value_dtype)
        h = C.c_void_p()
        _ck(_lib.gdsw_precond_create(C.byref(h), plan.handle, dtype_code(self.value_dtype),
                                     int(trisolve_iters)))
        self.handle = h

    def set_coarse(self, coarse: dict):
        keep = []
        cd = _CoarseDesc()
        cd.n_c, cd.n_gamma = coarse["n_c"], coarse["n_gamma"]
        for name in ("gamma_rows", "pg_ptr", "pg_col", "int_ptr", "int_rows", "col_ptr",
                     "col_ids", "aii_ptr", "aii_col", "aii_src", "aig_ptr", "aig_col",
                     "aig_src"):
            a = _i64(coarse[name])
            keep.append(a)
            setattr(cd, name, a.ctypes.data)
        pv = np.ascontiguousarray(coarse["pg_val"], dtype=np.float64)
        keep.append(pv)
        cd.pg_val = pv.ctypes.data
        _ck(_lib.gdsw_precond_set_coarse(self.handle, C.cast(C.pointer(cd), C.c_void_p)))

    def set_factors(self, l_vals: np.ndarray, u_vals: np.ndarray):
        lv = np.ascontiguousarray(l_vals, dtype=self.value_dtype)
        uv = np.ascontiguousarray(u_vals, dtype=self.value_dtype)
        _ck(_lib.gdsw_precond_set_factors(self.handle, _ptr(lv), _ptr(uv)))

    def fastilu(self, a_dev: DeviceCsr, sweeps: int, n_sub: int) -> np.ndarray:
        res = np.zeros((sweeps, n_sub), dtype=np.float64)
        _ck(_lib.gdsw_precond_fastilu(self.handle, a_dev.handle, int(sweeps), _ptr(res)))
        return res

    def lu_numeric(self, a_dev: DeviceCsr, diag_shift: float, n_sub: int) -> np.ndarray:
        """GPU IKJ factorization of every block; returns 1 + the first failing
        row per block (0 = ok)."""
        fail = np.zeros(max(n_sub, 1), dtype=np.int64)
        _ck(_lib.gdsw_precond_lu_numeric(self.handle, a_dev.handle, float(diag_shift), _ptr(fail)))
        return fail[:n_sub]

    def coarse_galerkin(self, a_dev: DeviceCsr, n_c: int, layout=None):
        """A0 = Phi^T A Phi (float64) from the device coarse basis, as a
        CsrMatrix with the reference's SpGEMM pattern (computed zeros kept).
        layout: the rank's DistLayout on the sharded path (a_dev = its owned
        rows); the partial products are summed over ranks on the device."""
        from .sparse_core import CsrMatrix
        out = np.zeros((n_c, n_c), dtype=np.float64)
        pat = np.zeros((n_c, n_c), dtype=np.uint8)
        if layout is None:
            _ck(_lib.gdsw_precond_coarse_galerkin(self.handle, a_dev.handle, _ptr(out), _ptr(pat)))
        else:
            _ck(_lib.gdsw_dist_coarse_galerkin(self.handle, a_dev.handle, layout.handle, _ptr(out),
                                               _ptr(pat)))
        rows, cols = np.nonzero(pat)
        ptr = np.zeros(n_c + 1, dtype=np.int64)
        np.add.at(ptr, rows + 1, 1)
        return CsrMatrix(n_c, n_c, np.cumsum(ptr), cols.astype(np.int64), out[rows, cols])

    def factors(self, nnz_l: int, nnz_u: int):
        lv = np.empty(nnz_l, dtype=self.value_dtype)
        uv = np.empty(nnz_u, dtype=self.value_dtype)
        _ck(_lib.gdsw_precond_get_factors(self.handle, _ptr(lv), _ptr(uv)))
        return lv, uv

    def extend(self, a_dev: DeviceCsr, n_cols: int, tol: float, max_iters: int):
        it = C.c_int(0)
        resid = np.zeros(max(n_cols, 1), dtype=np.float64)
        _ck(_lib.gdsw_precond_extend(self.handle, a_dev.handle, tol, int(max_iters),
                                     C.byref(it), _ptr(resid)))
        return it.value, resid[:n_cols]

    def panels(self) -> np.ndarray:
        n = _lib.gdsw_precond_panel_entries(self.handle)
        out = np.empty(n, dtype=np.float64)
        _ck(_lib.gdsw_precond_get_panels(self.handle, _ptr(out)))
        return out

    def set_coarse_inverse(self, a0inv: np.ndarray):
        a = np.ascontiguousarray(a0inv, dtype=np.float64)
        _ck(_lib.gdsw_precond_set_coarse_inverse(self.handle, _ptr(a)))

    @staticmethod
    def _factor_desc(f):
        keep = {k: np.ascontiguousarray(getattr(f, k), dtype=np.int64) for k in _CF_ARRAYS}
        vals = np.ascontiguousarray(f.values, dtype=np.float64)
        # no values: a structure-only factor, the device computes its blocks
        d = _CoarseFactor(n=f.n, n_sn=f.n_sn, n_levels=f.n_levels,
                          values=vals.ctypes.data if vals.size else None,
                          n_values=f.n_values, **{k: v.ctypes.data for k, v in keep.items()})
        return d, (keep, vals)

    def set_coarse_factor(self, f):
        """Factored coarse solve (coarse_factor.CoarseFactor)."""
        d, _keep = self._factor_desc(f)
        _ck(_lib.gdsw_precond_set_coarse_factor(self.handle, C.byref(d)))

    def set_local_factor(self, f):
        """Factored exact-LU local solves (coarse_factor.build_block_factors),
        or None for the level-set path."""
        if f is None:
            _ck(_lib.gdsw_precond_set_local_factor(self.handle, None))
            return
        d, _keep = self._factor_desc(f)
        _ck(_lib.gdsw_precond_set_local_factor(self.handle, C.byref(d)))

    def apply(self, r, z):
        _ck(_lib.gdsw_precond_apply(self.handle, _ptr(r), _ptr(z), stream_handle()))
        return z

    def local_solve(self, r, y, jacobi_iters: int = 0):
        _ck(_lib.gdsw_precond_local_solve(self.handle, _ptr(r), _ptr(y), int(jacobi_iters),
                                          stream_handle()))
        return y

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            _lib.gdsw_precond_destroy(h)
            self.handle = None


class Workspace:
    def __init__(self, n: int, restart: int):
        h = C.c_void_p()
        _ck(_lib.gdsw_workspace_create(C.byref(h), int(n), int(restart)))
        self.handle, self.n, self.restart = h, n, restart

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            _lib.gdsw_workspace_destroy(h)
            self.handle = None


_WS = threading.local()


def workspace(n: int, restart: int) -> Workspace:
    """The calling thread's Krylov workspace (V, Zm, the block slots and
    pinned read-back buffers): per thread, so concurrent solves on different
    threads never share it; at most one per thread (it holds 2*restart
    vectors)."""
    key = (n, restart)
    cur = getattr(_WS, "ws", None)
    if cur is None or cur[0] != key:
        _WS.ws = None
        cur = _WS.ws = (key, Workspace(n, restart))
    return cur[1]


def gmres_device(a_dev: DeviceCsr, m_pre: Precond | None, m_csr: DeviceCsr | None, b, x,
                 x0_nonzero: bool, cfg) -> dict:
    """Run the native GMRES loop on device vectors b, x (x in: x0, out: x)."""
    ws = workspace(a_dev.nrows, cfg.restart)
    kc = _KrylovCfg(cfg.restart, cfg.rel_tol, cfg.max_iters,
                    1 if cfg.variant == "single_reduce" else 0,
                    1 if cfg.orthogonalization == "cgs2" else 0)
    rep = _Report()
    cap = 2 * cfg.max_iters + 8
    hist = np.zeros(cap, dtype=np.float64)
    tit = np.zeros(cap, dtype=np.int32)
    tres = np.zeros(cap, dtype=np.float64)
    _ck(_lib.gdsw_gmres(a_dev.handle, m_pre.handle if m_pre else None,
                        m_csr.handle if m_csr else None, _ptr(b), _ptr(x),
                        1 if x0_nonzero else 0, C.byref(kc), ws.handle, C.byref(rep),
                        _ptr(hist), _ptr(tit), _ptr(tres), cap, stream_handle()))
    return dict(iterations=rep.iterations, converged=bool(rep.converged),
                reduction_count=rep.reduction_count,
                iteration_reductions=rep.iteration_reductions,
                residual_reductions=rep.residual_reductions, restarts=rep.restarts,
                history=hist[:rep.n_history].copy(),
                true_residuals=[(int(tit[k]), float(tres[k])) for k in range(rep.n_true)])


HOST_OP = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64)


class _HostOp:
    """A Python operator (callable) as a gdsw_host_op. The first exception
    it raises is kept and re-raised after the native solve returns."""

    def __init__(self, fn):
        self.fn = fn
        self.error = None
        self.c = HOST_OP(self._call)

    def _call(self, _ctx, xp, yp, n):
        try:
            x = np.ctypeslib.as_array(xp, shape=(n,))
            y = np.asarray(self.fn(x.copy()), dtype=np.float64)
            if y.shape != (n,):
                raise ValueError("operator dimensions do not match the vector")
            np.ctypeslib.as_array(yp, shape=(n,))[:] = y
            return 0
        except BaseException as err:  # noqa: BLE001 -- surfaced after the native call
            if self.error is None:
                self.error = err
            return 1


def gmres_host_ops(a_dev, a_fn, m_pre, m_csr, m_fn, n: int, b, x, x0_nonzero: bool, cfg) -> dict:
    """The native GMRES loop with host-side A and/or M (the reference's
    callables and .apply objects); vectors b, x on the device."""
    ws = workspace(n, cfg.restart)
    kc = _KrylovCfg(cfg.restart, cfg.rel_tol, cfg.max_iters,
                    1 if cfg.variant == "single_reduce" else 0,
                    1 if cfg.orthogonalization == "cgs2" else 0)
    rep = _Report()
    cap = 2 * cfg.max_iters + 8
    hist = np.zeros(cap, dtype=np.float64)
    tit = np.zeros(cap, dtype=np.int32)
    tres = np.zeros(cap, dtype=np.float64)
    ops = [_HostOp(f) if f is not None else None for f in (a_fn, m_fn)]
    fn_ptr = [C.cast(o.c, C.c_void_p) if o else None for o in ops]
    code = _lib.gdsw_gmres_host_ops(a_dev.handle if a_dev else None, fn_ptr[0], None,
                                    m_pre.handle if m_pre else None, m_csr.handle if m_csr else None,
                                    fn_ptr[1], None, int(n), _ptr(b), _ptr(x), 1 if x0_nonzero else 0,
                                    C.byref(kc), ws.handle, C.byref(rep), _ptr(hist), _ptr(tit),
                                    _ptr(tres), cap, stream_handle())
    for o in ops:
        if o is not None and o.error is not None:
            raise o.error
    _ck(code)
    return dict(iterations=rep.iterations, converged=bool(rep.converged),
                reduction_count=rep.reduction_count,
                iteration_reductions=rep.iteration_reductions,
                residual_reductions=rep.residual_reductions, restarts=rep.restarts,
                history=hist[:rep.n_history].copy(),
                true_residuals=[(int(tit[k]), float(tres[k])) for k in range(rep.n_true)])


class DistLayout:
    """gdsw_dist: this rank's extended layout + peer-memory mailbox."""

    def __init__(self, rank, nranks, n_ext, own_lo, own_hi, nbrs, red_max=4096):
        nb = len(nbrs)
        ranks = np.array([q for q, *_ in nbrs] or [0], dtype=np.int32)
        cols = [np.array([t[k] for t in nbrs] or [0], dtype=np.int64) for k in range(1, 5)]
        h = C.c_void_p()
        _ck(_lib.gdsw_dist_create(C.byref(h), int(rank), int(nranks), int(n_ext), int(own_lo),
                                  int(own_hi), nb, _ptr(ranks), *[_ptr(c) for c in cols],
                                  int(red_max)))
        self.handle = h
        self.rank, self.nranks = rank, nranks
        self.n_ext, self.own_lo, self.own_hi = n_ext, own_lo, own_hi

    def ipc_handle(self) -> bytes:
        buf = (C.c_char * 64)()
        _ck(_lib.gdsw_dist_ipc_handle(self.handle, C.cast(buf, C.c_void_p)))
        return bytes(buf)

    def open_peers(self, handles: list):
        blob = b"".join(handles)
        buf = (C.c_char * len(blob)).from_buffer_copy(blob)
        _ck(_lib.gdsw_dist_open_peers(self.handle, C.cast(buf, C.c_void_p)))

    def allreduce(self, x_in, x_out):
        _ck(_lib.gdsw_dist_allreduce(self.handle, _ptr(x_in), _ptr(x_out), int(x_in.numel()),
                                     stream_handle()))
        return x_out

    def halo(self, x_ext):
        _ck(_lib.gdsw_dist_halo(self.handle, _ptr(x_ext), stream_handle()))
        return x_ext

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            _lib.gdsw_dist_destroy(h)
            self.handle = None


def precond_set_dist(pre: "Precond", layout: DistLayout | None):
    _ck(_lib.gdsw_precond_set_dist(pre.handle, layout.handle if layout else None))


def gmres_dist(a_own: DeviceCsr, m_pre, b_own, x_own, x0_nonzero: bool, cfg,
               layout: DistLayout) -> dict:
    """Sharded native GMRES: b_own/x_own are this rank's owned rows."""
    ws = workspace(layout.n_ext, cfg.restart)
    kc = _KrylovCfg(cfg.restart, cfg.rel_tol, cfg.max_iters,
                    1 if cfg.variant == "single_reduce" else 0,
                    1 if cfg.orthogonalization == "cgs2" else 0)
    rep = _Report()
    cap = 2 * cfg.max_iters + 8
    hist = np.zeros(cap, dtype=np.float64)
    tit = np.zeros(cap, dtype=np.int32)
    tres = np.zeros(cap, dtype=np.float64)
    _ck(_lib.gdsw_gmres_dist(a_own.handle, m_pre.handle if m_pre else None, None, _ptr(b_own),
                             _ptr(x_own), 1 if x0_nonzero else 0, C.byref(kc), ws.handle,
                             layout.handle, C.byref(rep), _ptr(hist), _ptr(tit), _ptr(tres), cap,
                             stream_handle()))
    return dict(iterations=rep.iterations, converged=bool(rep.converged),
                reduction_count=rep.reduction_count,
                iteration_reductions=rep.iteration_reductions,
                residual_reductions=rep.residual_reductions, restarts=rep.restarts,
                history=hist[:rep.n_history].copy(),
                true_residuals=[(int(tit[k]), float(tres[k])) for k in range(rep.n_true)])


def sr_update(V, Zm, j: int, coef, w, mc, zc, n: int):
    """In-place single-reduce update of device tensors (gdsw_sr_update)."""
    _ck(_lib.gdsw_sr_update(_ptr(V), _ptr(Zm), int(n), int(n), int(j), _ptr(coef), _ptr(w), _ptr(mc),
                            _ptr(zc), stream_handle()))


def block_dot(V, j: int, v, z, n: int) -> np.ndarray:
    out = np.zeros(2 * (j + 1), dtype=np.float64)
    _ck(_lib.gdsw_block_dot(_ptr(V), int(n), int(j), _ptr(v), _ptr(z), int(n), _ptr(out),
                            stream_handle()))
    return out


# ---------------------------------------------------------------------------
# instrumentation
# ---------------------------------------------------------------------------
def launch_count() -> int:
    return int(_lib.gdsw_launch_count())


def prof_enable(on: bool = True):
    _ck(_lib.gdsw_prof_enable(1 if on else 0))


def prof_reset():
    _ck(_lib.gdsw_prof_reset())


def prof_read() -> dict:
    out = {}
    for k in range(_lib.gdsw_prof_count()):
        ms, n, b = C.c_double(), C.c_int64(), C.c_double()
        _ck(_lib.gdsw_prof_read(k, C.byref(ms), C.byref(n), C.byref(b)))
        out[_lib.gdsw_prof_name(k).decode()] = dict(ms=ms.value, launches=n.value, bytes=b.value)
    return out


# ---------------------------------------------------------------------------
# single-block solver (LocalFactorization.solve on the GPU)
# ---------------------------------------------------------------------------
class SingleBlockSolver:
    """One-subdomain plan+precond around a LocalFactorization, so its solve
    runs through the same batched kernels (local_solvers.py:263-278)."""

    def __init__(self, fac):
        from .schwarz import local_plan_arrays
        sym = fac.symbolic
        n = sym.n
        local = local_plan_arrays(n, [np.arange(n, dtype=np.int64)], [sym], fac.method, None,
                                  None)
        self.plan = Plan(local)
        self.n = n
        self.dtype = np.dtype(fac.l_values.dtype)
        self.pre = Precond(self.plan, self.dtype, fac.trisolve_iters)
        self.pre.set_factors(fac.l_values, fac.u_values)
        self.perm = sym.ordering.perm
        self.method = fac.method

    def solve(self, b, iters: int, force_jacobi: bool = False) -> np.ndarray:
        t = torch()
        b = np.asarray(b)
        if b.shape != (self.n,):
            raise ValueError(f"right-hand side has length {b.shape}, block size {self.n}")
        r = t.from_numpy(np.ascontiguousarray(b, dtype=np.float64)).cuda()
        tdt = t.float32 if self.dtype == np.float32 else t.float64
        y = t.empty(self.n, dtype=tdt, device="cuda")
        jac = iters if (force_jacobi or self.method == "fast_ilu") else 0
        self.pre.local_solve(r, y, jac)
        x = y.cpu().numpy()
        out = np.empty_like(x)
        out[self.perm] = x
        return out


def single_block_fastilu(a, sym, factor_sweeps: int, trisolve_iters: int):
    """fast_ilu_numeric for one block on the GPU (local_solvers.py:343-397)."""
    from .local_solvers import LocalFactorization
    from .schwarz import local_plan_arrays
    n = sym.n
    dt = np.dtype(a.values.dtype)
    a64 = a if dt == np.float64 else type(a)(a.nrows, a.ncols, a.row_ptr, a.col_idx,
                                             a.values.astype(np.float64))
    local = local_plan_arrays(n, [np.arange(n, dtype=np.int64)], [sym], "fast_ilu",
                              a64, [np.arange(a.nnz, dtype=np.int64)])
    plan = Plan(local)
    pre = Precond(plan, dt, trisolve_iters)
    a_dev = DeviceCsr(a64)
    res = pre.fastilu(a_dev, factor_sweeps, 1)
    lv, uv = pre.factors(sym.l_idx.size, sym.u_idx.size)
    return LocalFactorization(sym, "fast_ilu", lv, uv, sweep_residuals=[float(x) for x in res[:, 0]],
                              trisolve_iters=trisolve_iters)
