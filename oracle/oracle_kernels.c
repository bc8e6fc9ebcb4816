/*
 * ORACLE -- test infrastructure, NOT the product.
 *
 * Plain-C restatement of the reference's sequential loop kernels on the
 * solve path (schwarzdd, /root/reference/pkg/src/schwarzdd/_kernels.py), used
 * only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg to
 * check / time the CUDA path. Compiled with -ffp-contract=off so every
 * product and sum is rounded separately, exactly like the numba loops
 * (_kernels.py:12-16, no fastmath): results are bit-identical to the
 * reference. Each function cites the reference lines it restates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;

/* _kernels.py:23-31  y <- alpha*A x + beta*y, rows in order */
#define SPMV(T, NAME)                                                                 \
  void NAME(i64 n, const i64* ptr, const i64* idx, const T* val, const T* x, T* y,   \
            T alpha, T beta) {                                                        \
    for (i64 i = 0; i < n; ++i) {                                                     \
      T acc = (T)0;                                                                   \
      for (i64 p = ptr[i]; p < ptr[i + 1]; ++p) acc += val[p] * x[idx[p]];           \
      y[i] = alpha * acc + beta * y[i];                                               \
    }                                                                                 \
  }
SPMV(double, or_spmv_f64)
SPMV(float, or_spmv_f32)

/* _kernels.py:473-484  L x = b (unit diagonal) over the level schedule */
#define TRI_L(T, NAME)                                                                \
  void NAME(const i64* lp, const i64* li, const T* lv, i64 nlev, const i64* lev_ptr, \
            const i64* lev_rows, T* x) {                                              \
    for (i64 l = 0; l < nlev; ++l)                                                    \
      for (i64 t = lev_ptr[l]; t < lev_ptr[l + 1]; ++t) {                             \
        i64 i = lev_rows[t];                                                          \
        T acc = x[i];                                                                 \
        for (i64 p = lp[i]; p < lp[i + 1]; ++p) acc -= lv[p] * x[li[p]];              \
        x[i] = acc;                                                                   \
      }                                                                               \
  }
TRI_L(double, or_trisolve_lower_f64)
TRI_L(float, or_trisolve_lower_f32)

/* _kernels.py:487-496  U x = b, diagonal first in each row */
#define TRI_U(T, NAME)                                                                \
  void NAME(const i64* up, const i64* ui, const T* uv, i64 nlev, const i64* lev_ptr, \
            const i64* lev_rows, T* x) {                                              \
    for (i64 l = 0; l < nlev; ++l)                                                    \
      for (i64 t = lev_ptr[l]; t < lev_ptr[l + 1]; ++t) {                             \
        i64 i = lev_rows[t];                                                          \
        T acc = x[i];                                                                 \
        for (i64 p = up[i] + 1; p < up[i + 1]; ++p) acc -= uv[p] * x[ui[p]];          \
        x[i] = acc / uv[up[i]];                                                       \
      }                                                                               \
  }
TRI_U(double, or_trisolve_upper_f64)
TRI_U(float, or_trisolve_upper_f32)

/* _kernels.py:620-636  x(1) = b ; x(m+1) = b - (L - I) x(m) ; `iters` iterates */
#define JAC_L(T, NAME)                                                                \
  void NAME(i64 n, const i64* lp, const i64* li, const T* lv, const T* b, i64 iters, \
            T* x, T* work) {                                                          \
    memcpy(x, b, n * sizeof(T));                                                      \
    T* cur = x;                                                                       \
    T* nxt = work;                                                                    \
    for (i64 it = 1; it < iters; ++it) {                                              \
      for (i64 i = 0; i < n; ++i) {                                                   \
        T acc = b[i];                                                                 \
        for (i64 p = lp[i]; p < lp[i + 1]; ++p) acc -= lv[p] * cur[li[p]];            \
        nxt[i] = acc;                                                                 \
      }                                                                               \
      T* t = cur; cur = nxt; nxt = t;                                                 \
    }                                                                                 \
    if (cur != x) memcpy(x, cur, n * sizeof(T));                                      \
  }
JAC_L(double, or_jacobi_lower_f64)
JAC_L(float, or_jacobi_lower_f32)

/* _kernels.py:639-656  x(1) = D^-1 b ; x(m+1) = D^-1 (b - (U - D) x(m)) */
#define JAC_U(T, NAME)                                                                \
  void NAME(i64 n, const i64* up, const i64* ui, const T* uv, const T* b, i64 iters, \
            T* x, T* work) {                                                          \
    for (i64 i = 0; i < n; ++i) x[i] = b[i] / uv[up[i]];                              \
    T* cur = x;                                                                       \
    T* nxt = work;                                                                    \
    for (i64 it = 1; it < iters; ++it) {                                              \
      for (i64 i = 0; i < n; ++i) {                                                   \
        T acc = b[i];                                                                 \
        for (i64 p = up[i] + 1; p < up[i + 1]; ++p) acc -= uv[p] * cur[ui[p]];        \
        nxt[i] = acc / uv[up[i]];                                                     \
      }                                                                               \
      T* t = cur; cur = nxt; nxt = t;                                                 \
    }                                                                                 \
    if (cur != x) memcpy(x, cur, n * sizeof(T));                                      \
  }
JAC_U(double, or_jacobi_upper_f64)
JAC_U(float, or_jacobi_upper_f32)

/* _kernels.py:429-466  IKJ numeric LU restricted to the pattern;
 * returns 0, or 1 + row of a tiny pivot */
#define LU(T, NAME)                                                                   \
  i64 NAME(i64 n, const i64* lp, const i64* li, const i64* up, const i64* ui,         \
           const i64* ap, const i64* ai, const T* av, T* lv, T* uv, double tol) {     \
    T* w = (T*)calloc(n > 0 ? n : 1, sizeof(T));                                      \
    i64* stamp = (i64*)malloc((n > 0 ? n : 1) * sizeof(i64));                         \
    for (i64 i = 0; i < n; ++i) stamp[i] = -1;                                        \
    i64 rc = 0;                                                                       \
    for (i64 i = 0; i < n && !rc; ++i) {                                              \
      for (i64 p = lp[i]; p < lp[i + 1]; ++p) { stamp[li[p]] = i; w[li[p]] = 0; }     \
      for (i64 p = up[i]; p < up[i + 1]; ++p) { stamp[ui[p]] = i; w[ui[p]] = 0; }     \
      for (i64 p = ap[i]; p < ap[i + 1]; ++p)                                         \
        if (stamp[ai[p]] == i) w[ai[p]] = av[p];                                      \
      for (i64 p = lp[i]; p < lp[i + 1]; ++p) {                                       \
        i64 k = li[p];                                                                \
        T l_ik = w[k] / uv[up[k]];                                                    \
        w[k] = l_ik;                                                                  \
        for (i64 q = up[k] + 1; q < up[k + 1]; ++q)                                   \
          if (stamp[ui[q]] == i) w[ui[q]] -= l_ik * uv[q];                            \
      }                                                                               \
      if (fabs((double)w[i]) <= tol) { rc = i + 1; break; }                           \
      for (i64 p = lp[i]; p < lp[i + 1]; ++p) lv[p] = w[li[p]];                       \
      for (i64 p = up[i]; p < up[i + 1]; ++p) uv[p] = w[ui[p]];                       \
    }                                                                                 \
    free(w); free(stamp);                                                             \
    return rc;                                                                        \
  }
LU(double, or_lu_numeric_f64)
LU(float, or_lu_numeric_f32)

/* _kernels.py:547-571  sum_{k<bound} L(i,k) U(k,j) by sorted merge */
#define SDOT(T, NAME)                                                                 \
  static T NAME(const i64* lp, const i64* li, const T* lv, i64 i, const i64* ucp,    \
                const i64* ucr, const i64* ucs, const T* uv, i64 j, i64 bound) {      \
    i64 p = lp[i], pe = lp[i + 1], q = ucp[j], qe = ucp[j + 1];                       \
    T s = (T)0;                                                                       \
    while (p < pe && q < qe) {                                                        \
      i64 kl = li[p];                                                                 \
      if (kl >= bound) break;                                                         \
      i64 ku = ucr[q];                                                                \
      if (ku >= bound) break;                                                         \
      if (kl == ku) { s += lv[p] * uv[ucs[q]]; ++p; ++q; }                            \
      else if (kl < ku) ++p;                                                          \
      else ++q;                                                                       \
    }                                                                                 \
    return s;                                                                         \
  }
SDOT(double, sdot_f64)
SDOT(float, sdot_f32)

/* _kernels.py:574-595  one synchronous FastILU sweep; returns 1 when a
 * zero pivot was hit (the reference raises ZeroDivisionError there) */
#define SWEEP(T, NAME, SD)                                                             \
  int NAME(i64 n, const i64* lp, const i64* li, const T* lo, T* ln, const i64* up,     \
           const i64* ui, const T* uo, T* un, const i64* ucp, const i64* ucr,          \
           const i64* ucs, const i64* a_of_l, const i64* a_of_u, const T* av) {        \
    for (i64 i = 0; i < n; ++i) {                                                      \
      for (i64 p = lp[i]; p < lp[i + 1]; ++p) {                                        \
        i64 j = li[p];                                                                 \
        T a = a_of_l[p] >= 0 ? av[a_of_l[p]] : (T)0;                                   \
        T s = SD(lp, li, lo, i, ucp, ucr, ucs, uo, j, j);                              \
        if (uo[up[j]] == (T)0) return 1;                                               \
        ln[p] = (a - s) / uo[up[j]];                                                   \
      }                                                                                \
      for (i64 p = up[i]; p < up[i + 1]; ++p) {                                        \
        i64 j = ui[p];                                                                 \
        T a = a_of_u[p] >= 0 ? av[a_of_u[p]] : (T)0;                                   \
        T s = SD(lp, li, lo, i, ucp, ucr, ucs, uo, j, i);                              \
        un[p] = a - s;                                                                 \
      }                                                                                \
    }                                                                                  \
    return 0;                                                                          \
  }
SWEEP(double, or_fastilu_sweep_f64, sdot_f64)
SWEEP(float, or_fastilu_sweep_f32, sdot_f32)

/* _kernels.py:598-617  sum over A's pattern of |A - LU| (accumulated in f64) */
#define RESID(T, NAME, SD)                                                             \
  double NAME(i64 n, const i64* lp, const i64* li, const T* lv, const i64* up,         \
              const i64* ui, const T* uv, const i64* ucp, const i64* ucr,              \
              const i64* ucs, const i64* l_of_a, const i64* u_of_a, const i64* ap,     \
              const i64* ai, const T* av) {                                            \
    double r = 0.0;                                                                    \
    for (i64 i = 0; i < n; ++i)                                                        \
      for (i64 p = ap[i]; p < ap[i + 1]; ++p) {                                        \
        i64 j = ai[p];                                                                 \
        i64 bound = i < j ? i : j;                                                     \
        T s = SD(lp, li, lv, i, ucp, ucr, ucs, uv, j, bound);                          \
        if (i > j) s += lv[l_of_a[p]] * uv[up[j]];                                     \
        else s += uv[u_of_a[p]];                                                       \
        T d = av[p] - s;                                                               \
        r += (double)(d < 0 ? -d : d);                                                 \
      }                                                                                \
    return r;                                                                          \
  }
RESID(double, or_fastilu_residual_f64, sdot_f64)
RESID(float, or_fastilu_residual_f32, sdot_f32)

/* _kernels.py:499-522 multi-RHS level-set solves on a row-major (n x m) block */
void or_trisolve_lower_multi_f64(const i64* lp, const i64* li, const double* lv, i64 nlev,
                                 const i64* lev_ptr, const i64* lev_rows, double* xb, i64 m) {
  for (i64 l = 0; l < nlev; ++l)
    for (i64 t = lev_ptr[l]; t < lev_ptr[l + 1]; ++t) {
      i64 i = lev_rows[t];
      for (i64 c = 0; c < m; ++c) {
        double acc = xb[i * m + c];
        for (i64 p = lp[i]; p < lp[i + 1]; ++p) acc -= lv[p] * xb[li[p] * m + c];
        xb[i * m + c] = acc;
      }
    }
}

void or_trisolve_upper_multi_f64(const i64* up, const i64* ui, const double* uv, i64 nlev,
                                 const i64* lev_ptr, const i64* lev_rows, double* xb, i64 m) {
  for (i64 l = 0; l < nlev; ++l)
    for (i64 t = lev_ptr[l]; t < lev_ptr[l + 1]; ++t) {
      i64 i = lev_rows[t];
      for (i64 c = 0; c < m; ++c) {
        double acc = xb[i * m + c];
        for (i64 p = up[i] + 1; p < up[i + 1]; ++p) acc -= uv[p] * xb[ui[p] * m + c];
        xb[i * m + c] = acc / uv[up[i]];
      }
    }
}

/* _kernels.py:34-48  out <- A @ B for a dense row-major B (k x m) */
void or_csr_matmat_dense_f64(i64 n, const i64* ptr, const i64* idx, const double* val,
                             const double* b, i64 m, double* out) {
  for (i64 i = 0; i < n; ++i) {
    for (i64 c = 0; c < m; ++c) out[i * m + c] = 0.0;
    for (i64 p = ptr[i]; p < ptr[i + 1]; ++p) {
      double v = val[p];
      const double* br = b + idx[p] * m;
      for (i64 c = 0; c < m; ++c) out[i * m + c] += v * br[c];
    }
  }
}
