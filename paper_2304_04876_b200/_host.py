"""ctypes binding of ``libgdsw_host.so`` (include/gdsw_host.h).

Host-side pattern work only: orderings, symbolic factorizations, level
schedules, gathers, the coarse Galerkin product and the setup-time numeric
LU. Loaded eagerly; a missing library raises instead of falling back to a
Python restatement.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libgdsw_host.so"

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_f32p = C.POINTER(C.c_float)
_u8p = C.POINTER(C.c_uint8)
_resp = C.POINTER(C.c_void_p)


def _load():
    if not _LIB_PATH.exists():
        raise ImportError(
            f"{_LIB_PATH} is missing; build it with "
            "`python -m paper_2304_04876_b200.build`")
    lib = C.CDLL(str(_LIB_PATH))
    lib.gh_last_error.restype = C.c_char_p
    lib.gh_result_count.restype = C.c_int64
    lib.gh_result_size.restype = C.c_int64
    lib.gh_result_size.argtypes = [C.c_void_p, C.c_int64]
    lib.gh_result_kind.argtypes = [C.c_void_p, C.c_int64]
    lib.gh_result_copy.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
    lib.gh_result_free.argtypes = [C.c_void_p]
    lib.gh_result_count.argtypes = [C.c_void_p]
    lib.gh_lu_numeric_f64.restype = C.c_int64
    lib.gh_lu_numeric_f32.restype = C.c_int64
    return lib


_lib = _load()


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _check(rc: int):
    if rc != 0:
        raise RuntimeError(_lib.gh_last_error().decode())


def _take(res: C.c_void_p) -> list:
    out = []
    try:
        for k in range(_lib.gh_result_count(res)):
            size = _lib.gh_result_size(res, k)
            kind = _lib.gh_result_kind(res, k)
            dtype = (np.int64, np.float64, np.float32)[kind]
            arr = np.empty(size, dtype=dtype)
            if size:
                _lib.gh_result_copy(res, k, _p(arr))
            out.append(arr)
    finally:
        _lib.gh_result_free(res)
    return out


def _call(fn, *args) -> list:
    res = C.c_void_p()
    _check(fn(*args, C.byref(res)))
    return _take(res)


# ---------------------------------------------------------------------------

def node_graph(ptr, idx, n_nodes: int, dpn: int):
    ptr, idx = _i64(ptr), _i64(idx)
    return _call(_lib.gh_node_graph, C.c_int64(n_nodes), C.c_int64(dpn), _p(ptr), _p(idx))


def expand_layers(g_ptr, g_idx, mask: np.ndarray, layers: int) -> np.ndarray:
    g_ptr, g_idx = _i64(g_ptr), _i64(g_idx)
    m = np.ascontiguousarray(mask, dtype=np.uint8).copy()
    _check(_lib.gh_expand_layers(C.c_int64(m.size), _p(g_ptr), _p(g_idx), _p(m),
                                 C.c_int64(layers)))
    return m.astype(bool)


def nested_dissection(n: int, ptr, idx, leaf_size: int = 32) -> np.ndarray:
    ptr, idx = _i64(ptr), _i64(idx)
    perm = np.empty(n, dtype=np.int64)
    _check(_lib.gh_nested_dissection(C.c_int64(n), _p(ptr), _p(idx),
                                     C.c_int64(leaf_size), _p(perm)))
    return perm


def symbolic_lu(n: int, ptr, idx, perm):
    ptr, idx, perm = _i64(ptr), _i64(idx), _i64(perm)
    return _call(_lib.gh_symbolic_lu, C.c_int64(n), _p(ptr), _p(idx), _p(perm))


def symbolic_iluk(n: int, ptr, idx, perm, fill_level: int):
    ptr, idx, perm = _i64(ptr), _i64(idx), _i64(perm)
    return _call(_lib.gh_symbolic_iluk, C.c_int64(n), _p(ptr), _p(idx), _p(perm),
                 C.c_int64(fill_level))


def level_schedule(n: int, ptr, idx, upper: bool):
    ptr, idx = _i64(ptr), _i64(idx)
    return _call(_lib.gh_level_schedule, C.c_int64(n), _p(ptr), _p(idx),
                 C.c_int(1 if upper else 0), C.c_void_p(0))


def csr_gather(ptr, idx, rows, col_map):
    ptr, idx, rows, col_map = _i64(ptr), _i64(idx), _i64(rows), _i64(col_map)
    return _call(_lib.gh_csr_gather, C.c_int64(rows.size), _p(ptr), _p(idx), _p(rows),
                 _p(col_map))


def transpose_pattern(n_rows: int, n_cols: int, ptr, idx):
    ptr, idx = _i64(ptr), _i64(idx)
    return _call(_lib.gh_transpose_pattern, C.c_int64(n_rows), C.c_int64(n_cols),
                 _p(ptr), _p(idx))


def spgemm(n_rows, n_cols, a_ptr, a_idx, a_val, b_ptr, b_idx, b_val):
    dt = np.dtype(a_val.dtype)
    fn = _lib.gh_spgemm_f64 if dt == np.float64 else _lib.gh_spgemm_f32
    a_ptr, a_idx, b_ptr, b_idx = _i64(a_ptr), _i64(a_idx), _i64(b_ptr), _i64(b_idx)
    a_val = np.ascontiguousarray(a_val, dtype=dt)
    b_val = np.ascontiguousarray(b_val, dtype=dt)
    return _call(fn, C.c_int64(n_rows), C.c_int64(n_cols), _p(a_ptr), _p(a_idx),
                 _p(a_val), _p(b_ptr), _p(b_idx), _p(b_val))


def lu_numeric(n, l_ptr, l_idx, u_ptr, u_idx, a_ptr, a_idx, a_val, pivot_tol):
    dt = np.dtype(a_val.dtype)
    l_val = np.zeros(len(l_idx), dtype=dt)
    u_val = np.zeros(len(u_idx), dtype=dt)
    fn = _lib.gh_lu_numeric_f64 if dt == np.float64 else _lib.gh_lu_numeric_f32
    arrs = [_i64(x) for x in (l_ptr, l_idx, u_ptr, u_idx, a_ptr, a_idx)]
    a_val = np.ascontiguousarray(a_val, dtype=dt)
    rc = fn(C.c_int64(n), *[_p(x) for x in arrs], _p(a_val), _p(l_val), _p(u_val),
            C.c_double(pivot_tol))
    return int(rc), l_val, u_val


def align_pattern(a_ptr, a_idx, f_ptr, f_idx) -> np.ndarray:
    a_ptr, a_idx, f_ptr, f_idx = _i64(a_ptr), _i64(a_idx), _i64(f_ptr), _i64(f_idx)
    out = np.empty(f_idx.size, dtype=np.int64)
    _check(_lib.gh_align_pattern(C.c_int64(a_ptr.size - 1), _p(a_ptr), _p(a_idx),
                                 _p(f_ptr), _p(f_idx), _p(out)))
    return out


def fastilu_plan(n, l_ptr, l_idx, u_ptr, u_idx, a_ptr, a_idx):
    arrs = [_i64(x) for x in (l_ptr, l_idx, u_ptr, u_idx, a_ptr, a_idx)]
    return _call(_lib.gh_fastilu_plan, C.c_int64(n), *[_p(x) for x in arrs])


def classify_interface(g_ptr, g_idx, node_owner):
    g_ptr, g_idx, node_owner = _i64(g_ptr), _i64(g_idx), _i64(node_owner)
    return _call(_lib.gh_classify_interface, C.c_int64(node_owner.size), _p(g_ptr),
                 _p(g_idx), _p(node_owner))


def spmv(ptr, idx, val, x, y, alpha, beta):
    dt = np.dtype(val.dtype)
    ptr, idx = _i64(ptr), _i64(idx)
    if dt == np.float64:
        _check(_lib.gh_spmv_f64(C.c_int64(ptr.size - 1), _p(ptr), _p(idx), _p(val), _p(x),
                                _p(y), C.c_double(alpha), C.c_double(beta)))
    else:
        _check(_lib.gh_spmv_f32(C.c_int64(ptr.size - 1), _p(ptr), _p(idx), _p(val), _p(x),
                                _p(y), C.c_float(alpha), C.c_float(beta)))
    return y


def overlap_sets(g_ptr, g_idx, node_owner, n_parts: int, subs, layers: int):
    g_ptr, g_idx, node_owner, subs = _i64(g_ptr), _i64(g_idx), _i64(node_owner), _i64(subs)
    ptr, nodes = _call(_lib.gh_overlap_sets, C.c_int64(node_owner.size), _p(g_ptr), _p(g_idx),
                       _p(node_owner), C.c_int64(n_parts), C.c_int64(subs.size), _p(subs),
                       C.c_int64(layers))
    return [nodes[ptr[k]:ptr[k + 1]] for k in range(subs.size)]


def partitioned_inverse(blocks, relax: int, zero_frac: float, threads: int,
                        with_values: bool = True):
    """Supernodal partitioned inverses of exact-LU blocks (gh_partitioned_inverse).
    blocks = [(base, l_ptr, l_idx, l_val, u_ptr, u_idx, u_val)]; returns the
    15 arrays of coarse_factor.CoarseFactor in ABI order."""
    nb = len(blocks)
    blk_n = _i64([b[1].size - 1 for b in blocks])
    base = _i64([b[0] for b in blocks])
    lp_off = _i64(np.concatenate([[0], np.cumsum([b[1].size for b in blocks])])[:-1])
    up_off = _i64(np.concatenate([[0], np.cumsum([b[4].size for b in blocks])])[:-1])
    lnz_off = _i64(np.concatenate([[0], np.cumsum([b[2].size for b in blocks])])[:-1])
    unz_off = _i64(np.concatenate([[0], np.cumsum([b[5].size for b in blocks])])[:-1])
    cat = (lambda k, dt: np.ascontiguousarray(np.concatenate([b[k] for b in blocks]), dtype=dt)
           if blocks else np.zeros(0, dtype=dt))
    lp, li, lv = cat(1, np.int64), cat(2, np.int64), cat(3, np.float64)
    up, ui, uv = cat(4, np.int64), cat(5, np.int64), cat(6, np.float64)
    return _call(_lib.gh_partitioned_inverse, C.c_int64(nb), _p(blk_n), _p(base), _p(lp_off),
                 _p(lnz_off), _p(up_off), _p(unz_off), _p(lp), _p(li), _p(lv), _p(up), _p(ui),
                 _p(uv), C.c_int64(relax), C.c_double(zero_frac), C.c_int64(threads),
                 C.c_int(1 if with_values else 0))
