// Sparse kernels of the solve path: SELL-32 SpMV, batched Jacobi
// (FastSpTRSV) sweeps, batched level-set SpTRSV, overlap gather and the
// owner-computes scatter fused with the coarse prolongation.
//
// Layout ("SELL-32"): rows are grouped in slices of 32 (one warp); slice s
// stores its entries column-major, entry k of row 32*s+lane at
// slice_off[s] + 32*k + lane. A warp's k-th load is one contiguous 32-entry
// run (fully coalesced 256 B for fp64 values, 128 B for int32 columns), while
// each thread still accumulates ITS row in the row's own column order with
// round-to-nearest mul/add -- the exact operation sequence of the
// reference's sequential loops (_kernels.py:23-31, 473-496, 620-656), so the
// results are bit-identical to them.
#pragma once
#include "common.cuh"

namespace gdsw {

struct SellDev {
  int32_t n_rows = 0;
  const int64_t* slice_off = nullptr;  // [n_slices + 1]
  const uint16_t* row_len = nullptr;   // [n_rows]
  const int32_t* col = nullptr;        // [padded nnz]
};

// host-side SELL pattern builder from a CSR pattern whose column indices are
// shifted by col_add (absolute positions in the concatenated vector)
struct SellPattern {
  int32_t n_rows = 0;
  int64_t padded = 0;
  DBuf<int64_t> slice_off;
  DBuf<uint16_t> row_len;
  DBuf<int32_t> col;
  DBuf<int64_t> csr_ptr;  // CSR row pointers, for value placement
  // rows_offdiag_skip: number of leading entries of each CSR row to drop
  // (1 = U's diagonal, stored first)
  void build(int64_t n, const int64_t* ptr, const int64_t* idx, const int64_t* col_add_per_row,
             int skip_first) {
    n_rows = (int32_t)n;
    int64_t ns = (n + 31) / 32;
    std::vector<int64_t> off(ns + 1, 0);
    std::vector<uint16_t> len(n);
    for (int64_t i = 0; i < n; ++i) {
      int64_t l = ptr[i + 1] - ptr[i] - skip_first;
      require(l >= 0 && l < 65536, "row too long for the SELL layout");
      len[i] = (uint16_t)l;
    }
    for (int64_t s = 0; s < ns; ++s) {
      int64_t w = 0;
      for (int64_t i = s * 32; i < std::min<int64_t>(n, s * 32 + 32); ++i) w = std::max<int64_t>(w, len[i]);
      off[s + 1] = off[s] + 32 * w;
    }
    padded = off[ns];
    std::vector<int32_t> c(padded, 0);
    for (int64_t i = 0; i < n; ++i) {
      int64_t base = off[i / 32] + (i % 32);
      for (int64_t k = 0; k < len[i]; ++k) {
        int64_t v = idx[ptr[i] + skip_first + k] + col_add_per_row[i];
        require(v >= 0 && v <= INT32_MAX, "column exceeds int32");
        c[base + 32 * k] = (int32_t)v;
      }
      // padding stays column 0 (never read: loops stop at row_len)
    }
    slice_off.upload(off);
    row_len.upload(len);
    col.upload(c);
    std::vector<int64_t> p(ptr, ptr + n + 1);
    csr_ptr.upload(p);
  }
  SellDev view() const {
    SellDev v;
    v.n_rows = n_rows;
    v.slice_off = slice_off.p;
    v.row_len = row_len.p;
    v.col = col.p;
    return v;
  }
};

// place CSR-ordered values (skipping `skip` leading entries per row) into
// SELL order; optionally extract the skipped leading entry (U's diagonal)
template <typename T, typename TS>
__global__ void k_csr_to_sell(int32_t n, const int64_t* __restrict__ ptr,
                              const int64_t* __restrict__ slice_off, const TS* __restrict__ src,
                              T* __restrict__ dst, int skip, T* __restrict__ diag_out) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t base = slice_off[i >> 5] + (i & 31);
  int64_t p0 = ptr[i], p1 = ptr[i + 1];
  if (skip && diag_out) diag_out[i] = (T)src[p0];
  for (int64_t p = p0 + skip, k = 0; p < p1; ++p, ++k) dst[base + 32 * k] = (T)src[p];
}

// ---------------------------------------------------------------------------
// SpMV: y = A x (mode 0), y = yin - A x (mode 1), y = alpha A x + beta yin (2)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) k_sell_spmv(SellDev A, const T* __restrict__ val,
                                                   const T* __restrict__ x,
                                                   const T* __restrict__ yin,
                                                   T* __restrict__ y, int mode, T alpha, T beta) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n_rows) return;
  const int64_t base = A.slice_off[i >> 5] + (i & 31);
  const int len = A.row_len[i];
  T acc = T(0);
  int k = 0;
  // 4 independent loads in flight per thread before the dependent gathers
  for (; k + 4 <= len; k += 4) {
    const int64_t q = base + 32 * (int64_t)k;
    int32_t c0 = ldg_stream(A.col + q), c1 = ldg_stream(A.col + q + 32);
    int32_t c2 = ldg_stream(A.col + q + 64), c3 = ldg_stream(A.col + q + 96);
    T v0 = ldg_stream(val + q), v1 = ldg_stream(val + q + 32);
    T v2 = ldg_stream(val + q + 64), v3 = ldg_stream(val + q + 96);
    T x0 = __ldg(x + c0), x1 = __ldg(x + c1), x2 = __ldg(x + c2), x3 = __ldg(x + c3);
    acc = rn_add(acc, rn_mul(v0, x0));
    acc = rn_add(acc, rn_mul(v1, x1));
    acc = rn_add(acc, rn_mul(v2, x2));
    acc = rn_add(acc, rn_mul(v3, x3));
  }
  for (; k < len; ++k) {
    const int64_t q = base + 32 * (int64_t)k;
    acc = rn_add(acc, rn_mul(ldg_stream(val + q), __ldg(x + ldg_stream(A.col + q))));
  }
  if (mode == 0) {
    y[i] = acc;
  } else if (mode == 1) {
    y[i] = rn_sub(yin[i], acc);
  } else {
    T t = rn_mul(alpha, acc);
    y[i] = (beta == T(0)) ? rn_add(t, T(0)) : rn_add(t, rn_mul(beta, yin[i]));
  }
}

// ---------------------------------------------------------------------------
// batched Jacobi triangular sweeps over all subdomains at once
// (jacobi_trisolve_lower_unit / _upper, _kernels.py:620-656)
// ---------------------------------------------------------------------------
// x_new = b - (L - I) x      (L strict lower in SELL)
template <typename T>
__global__ void __launch_bounds__(256) k_jacobi_lower(SellDev L, const T* __restrict__ lval,
                                                      const T* __restrict__ b,
                                                      const T* __restrict__ x,
                                                      T* __restrict__ xn) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L.n_rows) return;
  const int64_t base = L.slice_off[i >> 5] + (i & 31);
  const int len = L.row_len[i];
  T acc = b[i];
  for (int k = 0; k < len; ++k) {
    const int64_t q = base + 32 * (int64_t)k;
    acc = rn_sub(acc, rn_mul(ldg_stream(lval + q), x[ldg_stream(L.col + q)]));
  }
  xn[i] = acc;
}

// x_new = D^-1 (b - (U - D) x)  (U off-diagonal part in SELL, D separate)
template <typename T>
__global__ void __launch_bounds__(256) k_jacobi_upper(SellDev U, const T* __restrict__ uval,
                                                      const T* __restrict__ diag,
                                                      const T* __restrict__ b,
                                                      const T* __restrict__ x,
                                                      T* __restrict__ xn) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= U.n_rows) return;
  const int64_t base = U.slice_off[i >> 5] + (i & 31);
  const int len = U.row_len[i];
  T acc = b[i];
  for (int k = 0; k < len; ++k) {
    const int64_t q = base + 32 * (int64_t)k;
    acc = rn_sub(acc, rn_mul(ldg_stream(uval + q), x[ldg_stream(U.col + q)]));
  }
  xn[i] = rn_div(acc, diag[i]);
}

template <typename T>
__global__ void k_diag_solve(int32_t n, const T* __restrict__ diag, const T* __restrict__ b,
                             T* __restrict__ x) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = rn_div(b[i], diag[i]);
}

// overlap gather with the ordering folded in: xb[k] = T(r[gmap[k]])
// (schwarz.py:310-311 + local_solvers.py:266)
template <typename T>
__global__ void k_gather(int32_t n, const int32_t* __restrict__ gmap, const double* __restrict__ r,
                         T* __restrict__ xb) {
  int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) xb[k] = (T)r[ldg_stream(gmap + k)];
}

// gather fused with the first Jacobi L sweep: writes b = T(r[gmap]) and the
// second iterate b - (L - I) b in one pass over L
template <typename T>
__global__ void __launch_bounds__(256) k_gather_jacobi_lower(SellDev L,
                                                             const T* __restrict__ lval,
                                                             const int32_t* __restrict__ gmap,
                                                             const double* __restrict__ r,
                                                             T* __restrict__ b,
                                                             T* __restrict__ xn) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L.n_rows) return;
  const int64_t base = L.slice_off[i >> 5] + (i & 31);
  const int len = L.row_len[i];
  T acc = (T)r[gmap[i]];
  b[i] = acc;
  for (int k = 0; k < len; ++k) {
    const int64_t q = base + 32 * (int64_t)k;
    acc = rn_sub(acc, rn_mul(ldg_stream(lval + q), (T)r[__ldg(gmap + ldg_stream(L.col + q))]));
  }
  xn[i] = acc;
}

// ---------------------------------------------------------------------------
// batched level-set SpTRSV: one CTA per subdomain, gather + forward (unit L)
// + backward (U, diagonal first) over the host-computed level schedules
// (trisolve_forward_unit / trisolve_backward, _kernels.py:473-496). Rows of
// one level are independent, so each row's sequential accumulation
// reproduces sequential substitution bit for bit.
// ---------------------------------------------------------------------------
struct LevelSetDev {
  const int32_t* sub_ptr;
  const int32_t* gmap;
  const int64_t* l_ptr;
  const int32_t* l_col;
  const int64_t* u_ptr;
  const int32_t* u_col;
  const int32_t* llev_sub;
  const int32_t* llev_ptr;
  const int32_t* llev_rows;
  const int32_t* ulev_sub;
  const int32_t* ulev_ptr;
  const int32_t* ulev_rows;
};

template <typename T>
__global__ void __launch_bounds__(512) k_levelset(LevelSetDev P, const T* __restrict__ lval,
                                                  const T* __restrict__ uval,
                                                  const double* __restrict__ r,
                                                  T* __restrict__ x, int sub0, int do_gather) {
  const int s = sub0 + blockIdx.x;
  if (do_gather) {
    for (int32_t k = P.sub_ptr[s] + threadIdx.x; k < P.sub_ptr[s + 1]; k += blockDim.x)
      x[k] = (T)r[P.gmap[k]];
    __syncthreads();
  }
  for (int32_t lv = P.llev_sub[s]; lv < P.llev_sub[s + 1]; ++lv) {
    for (int32_t t = P.llev_ptr[lv] + threadIdx.x; t < P.llev_ptr[lv + 1]; t += blockDim.x) {
      const int32_t i = P.llev_rows[t];
      T acc = x[i];
      for (int64_t p = P.l_ptr[i]; p < P.l_ptr[i + 1]; ++p)
        acc = rn_sub(acc, rn_mul(lval[p], x[P.l_col[p]]));
      x[i] = acc;
    }
    __syncthreads();
  }
  for (int32_t lv = P.ulev_sub[s]; lv < P.ulev_sub[s + 1]; ++lv) {
    for (int32_t t = P.ulev_ptr[lv] + threadIdx.x; t < P.ulev_ptr[lv + 1]; t += blockDim.x) {
      const int32_t i = P.ulev_rows[t];
      const int64_t p0 = P.u_ptr[i];
      T acc = x[i];
      for (int64_t p = p0 + 1; p < P.u_ptr[i + 1]; ++p)
        acc = rn_sub(acc, rn_mul(uval[p], x[P.u_col[p]]));
      x[i] = rn_div(acc, uval[p0]);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// owner-computes scatter + coarse prolongation (schwarz.py:302-306, 322-327):
//   z[g] = double( (Phi v)[g] + (((0 + y_a) + y_b) + ...) )
// contributions y are summed in ascending subdomain order -- no atomics, the
// same order as the reference's `z[dofs] += y` loop.
// ---------------------------------------------------------------------------
struct ProlongDev {
  int enabled;
  const int64_t* pg_ptr;    // interface rows of Phi, CSR over all rows (empty for interior)
  const int32_t* pg_col;
  const int32_t* pi_sub;    // interior row -> subdomain (or -1)
  const int32_t* pi_row;    // row inside the subdomain's interior panel
  const int64_t* panel_off; // [n_sub] entry offset of the column-major panel
  const int32_t* n_int;     // [n_sub]
  const int32_t* col_ptr;   // [n_sub + 1]
  const int32_t* col_ids;   // coarse column of each panel column
};

template <typename T>
__global__ void __launch_bounds__(256) k_scatter_prolong(int32_t n, const int32_t* __restrict__ sc_ptr,
                                                         const int32_t* __restrict__ sc_pos,
                                                         const T* __restrict__ y, ProlongDev C,
                                                         const T* __restrict__ pg_val,
                                                         const T* __restrict__ panel,
                                                         const T* __restrict__ v,
                                                         double* __restrict__ z) {
  int32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  T acc = T(0);
  for (int32_t q = sc_ptr[g]; q < sc_ptr[g + 1]; ++q) acc = rn_add(acc, y[sc_pos[q]]);
  if (C.enabled) {
    T zc = T(0);
    const int64_t p0 = C.pg_ptr[g], p1 = C.pg_ptr[g + 1];
    if (p1 > p0) {
      for (int64_t p = p0; p < p1; ++p) zc = rn_add(zc, rn_mul(pg_val[p], v[C.pg_col[p]]));
    } else {
      const int32_t s = C.pi_sub[g];
      if (s >= 0) {
        const int32_t ni = C.n_int[s];
        const T* pr = panel + C.panel_off[s] + C.pi_row[g];
        for (int32_t c = C.col_ptr[s]; c < C.col_ptr[s + 1]; ++c, pr += ni)
          zc = rn_add(zc, rn_mul(ldg_stream(pr), v[C.col_ids[c]]));
      }
    }
    acc = rn_add(zc, acc);
  }
  z[g] = (double)acc;
}

}  // namespace gdsw
