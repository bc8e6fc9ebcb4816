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
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "common.cuh"

namespace gdsw {

struct SellDev {
  int32_t n_rows = 0;
  const int64_t* slice_off = nullptr;  // [n_slices + 1]
  const uint16_t* row_len = nullptr;   // [n_rows]
  const int32_t* col = nullptr;        // [padded nnz]
  const int16_t* d16 = nullptr;        // [padded nnz] col - row, when every |col - row| < 2^15
  int32_t uw = 0;                      // every slice padded to this width (<= SELL_UW), else 0
  // offset-mask columns (format 2): slice s lists the union of its rows'
  // column offsets (col - row, ascending, <= SELL_UW of them, padded to 8
  // int16 = one 16-byte load); row i keeps one bit per union entry. Values
  // stay in the plain SELL slots (k-th entry of the row in slot k); entry k's
  // column is row + the offset of the row's k-th set bit.
  const uint8_t* mask = nullptr;       // [n_rows]
  const int16_t* soff = nullptr;       // [n_slices * 8]
};

// column formats of the SELL kernels: absolute int32 columns, 16-bit
// row-relative offsets per entry, or the slot-mask layout (per-slice offset
// union + one byte per row: stencil-like patterns carry no per-entry index)
constexpr int SELL_COL32 = 0, SELL_D16 = 1, SELL_MASK = 2;
constexpr int SELL_UW = 8;  // widest pattern stored with uniform slice width

// first SELL slot of row i: arithmetic for uniform-width layouts (no
// dependent slice-offset load), else from slice_off
__device__ __forceinline__ int64_t sell_base(const SellDev& M, int32_t i) {
  if (M.uw) return (int64_t)(i >> 5) * 32 * M.uw + (i & 31);
  return M.slice_off[i >> 5] + (i & 31);
}

// column of SELL entry q of row i: 16-bit row-relative offsets when the
// pattern allows it (stencil-like and block-local factor patterns: 10 bytes
// per fp64 entry instead of 12), else absolute int32
template <int F>
__device__ __forceinline__ int32_t sell_col(const SellDev& M, int32_t i, int64_t q) {
  if (F == SELL_D16) return i + (int32_t)ldg_stream(M.d16 + q);
  return ldg_stream(M.col + q);
}

// offset-mask columns of row i, produced in entry order: the slice's offset
// union (one broadcast 16-byte load) and the row's mask byte
struct SellMaskCols {
  uint64_t lo = 0, hi = 0;
  unsigned mm = 0;
  int32_t i = 0;
  __device__ __forceinline__ SellMaskCols() {}
  __device__ __forceinline__ SellMaskCols(const SellDev& M, int32_t row) : i(row) {
    const int4 o = __ldg(reinterpret_cast<const int4*>(M.soff) + (row >> 5));
    lo = (uint64_t)(uint32_t)o.x | ((uint64_t)(uint32_t)o.y << 32);
    hi = (uint64_t)(uint32_t)o.z | ((uint64_t)(uint32_t)o.w << 32);
    mm = __ldg(M.mask + row);
  }
  __device__ __forceinline__ int len() const { return __popc(mm); }
  // column of the next entry (valid while entries remain)
  __device__ __forceinline__ int32_t next() {
    const int j = __ffs(mm) - 1;
    mm &= mm - 1;
    const uint64_t q = j < 4 ? lo : hi;
    return i + (int32_t)(int16_t)(uint16_t)(q >> (16 * (j & 3)));
  }
};

// entries of row i (format-independent count)
template <int F>
__device__ __forceinline__ int sell_len(const SellDev& M, int32_t i) {
  if constexpr (F == SELL_MASK) return __popc((unsigned)__ldg(M.mask + i));
  return (int)M.row_len[i];
}

// columns of entries [0, MW) of row i that exist (k < len); masked rows take
// them from the offset masks, the others from the per-entry index arrays
// (slots q = base + 32 k)
template <int F, int MW>
__device__ __forceinline__ void sell_cols(const SellDev& M, int32_t i, int64_t base, int len, int32_t* c) {
  if constexpr (F == SELL_MASK) {
    // branch-free: slots past the row's length get unused columns
    SellMaskCols mc(M, i);
#pragma unroll
    for (int k = 0; k < MW; ++k) c[k] = mc.next();
  } else {
#pragma unroll
    for (int k = 0; k < MW; ++k)
      if (k < len) c[k] = sell_col<F>(M, i, base + 32 * (int64_t)k);
  }
}

// host-side SELL pattern builder from a CSR pattern whose column indices are
// shifted by col_add (absolute positions in the concatenated vector)
struct SellPattern {
  int32_t n_rows = 0;
  int64_t padded = 0;
  DBuf<int64_t> slice_off;
  DBuf<uint16_t> row_len;
  DBuf<int32_t> col;
  DBuf<int16_t> d16;
  bool has16 = false;
  int32_t uw = 0;
  bool masked = false;
  DBuf<uint8_t> mask;
  DBuf<int16_t> soff;
  int fmt() const { return masked ? SELL_MASK : has16 ? SELL_D16 : SELL_COL32; }
  // stored index bytes per entry and per row (the roofline's algorithmic bytes)
  double idx_bytes_per_entry() const { return masked ? 0.0 : has16 ? 2.0 : 4.0; }
  double idx_bytes_per_row() const { return masked ? 1.5 : 2.0; }
  // offset masks feasible: every row's offsets strictly ascending and 16-bit,
  // at most SELL_UW distinct offsets per slice
  static bool mask_feasible(int64_t n, const int64_t* ptr, const int64_t* idx, const int64_t* col_add_per_row,
                            int skip_first, int32_t* width) {
    const int64_t ns = (n + 31) / 32;
    int32_t wmax = 0;
    int64_t nnz = 0;
    for (int64_t s = 0; s < ns; ++s) {
      int16_t u[SELL_UW];
      int nu = 0;
      for (int64_t i = s * 32; i < std::min<int64_t>(n, s * 32 + 32); ++i) {
        int64_t prev = INT64_MIN;
        const int64_t p0 = ptr[i] + skip_first, p1 = ptr[i + 1];
        nnz += p1 - p0;
        for (int64_t p = p0; p < p1; ++p) {
          const int64_t d = idx[p] + col_add_per_row[i] - i;
          if (d <= prev || d < -32768 || d > 32767) return false;
          prev = d;
          bool found = false;
          for (int k = 0; k < nu; ++k) found |= u[k] == (int16_t)d;
          if (!found) {
            if (nu == SELL_UW) return false;
            u[nu++] = (int16_t)d;
          }
        }
      }
      wmax = std::max(wmax, nu);
    }
    if (wmax == 0 || nnz == 0) return false;
    *width = wmax;
    return true;
  }
  void build_mask(int64_t n, const int64_t* ptr, const int64_t* idx, const int64_t* col_add_per_row,
                  int skip_first) {
    const int64_t ns = (n + 31) / 32;
    std::vector<int16_t> so(ns * 8, 0);
    std::vector<uint8_t> mk(n, 0);
    for (int64_t s = 0; s < ns; ++s) {
      std::vector<int16_t> u;
      const int64_t i1 = std::min<int64_t>(n, s * 32 + 32);
      for (int64_t i = s * 32; i < i1; ++i)
        for (int64_t p = ptr[i] + skip_first; p < ptr[i + 1]; ++p) u.push_back((int16_t)(idx[p] + col_add_per_row[i] - i));
      std::sort(u.begin(), u.end());
      u.erase(std::unique(u.begin(), u.end()), u.end());
      for (size_t k = 0; k < u.size(); ++k) so[s * 8 + k] = u[k];
      for (int64_t i = s * 32; i < i1; ++i) {
        unsigned m = 0;
        for (int64_t p = ptr[i] + skip_first; p < ptr[i + 1]; ++p) {
          const int16_t d = (int16_t)(idx[p] + col_add_per_row[i] - i);
          m |= 1u << (std::lower_bound(u.begin(), u.end(), d) - u.begin());
        }
        mk[i] = (uint8_t)m;
      }
    }
    masked = true;
    mask.upload(mk);
    soff.upload(so);
  }
  DBuf<int64_t> csr_ptr;  // CSR row pointers, for value placement
  // rows_offdiag_skip: number of leading entries of each CSR row to drop
  // (1 = U's diagonal, stored first)
  // allow_mask: use the slot-mask layout when feasible (callers that pair two
  // patterns in one kernel decide for both with mask_feasible)
  void build(int64_t n, const int64_t* ptr, const int64_t* idx, const int64_t* col_add_per_row,
             int skip_first, bool allow_mask = true) {
    n_rows = (int32_t)n;
    masked = false;
    mask.release();
    soff.release();
    int64_t ns = (n + 31) / 32;
    std::vector<int64_t> off(ns + 1, 0);
    std::vector<uint16_t> len(n);
    for (int64_t i = 0; i < n; ++i) {
      int64_t l = ptr[i + 1] - ptr[i] - skip_first;
      require(l >= 0 && l < 65536, "row too long for the SELL layout");
      len[i] = (uint16_t)l;
    }
    int64_t wmax = 0;
    for (int64_t s = 0; s < ns; ++s) {
      int64_t w = 0;
      for (int64_t i = s * 32; i < std::min<int64_t>(n, s * 32 + 32); ++i) w = std::max<int64_t>(w, len[i]);
      off[s + 1] = off[s] + 32 * w;
      wmax = std::max(wmax, w);
    }
    // uniform width when narrow and the extra padding is small: the slot of
    // a row is then computed, not loaded
    uw = 0;
    if (wmax > 0 && wmax <= SELL_UW && 32 * wmax * ns <= off[ns] + off[ns] / 8) {
      uw = (int32_t)wmax;
      for (int64_t s = 0; s <= ns; ++s) off[s] = 32 * wmax * s;
    }
    padded = off[ns];
    std::vector<int32_t> c(padded, 0);
    std::vector<int16_t> d(padded, 0);
    has16 = true;
    for (int64_t i = 0; i < n; ++i) {
      int64_t base = off[i / 32] + (i % 32);
      for (int64_t k = 0; k < len[i]; ++k) {
        int64_t v = idx[ptr[i] + skip_first + k] + col_add_per_row[i];
        require(v >= 0 && v <= INT32_MAX, "column exceeds int32");
        c[base + 32 * k] = (int32_t)v;
        const int64_t dl = v - i;
        if (dl < -32768 || dl > 32767) has16 = false;
        d[base + 32 * k] = (int16_t)dl;
      }
      // padding stays column 0 (never read: loops stop at row_len)
    }
    int32_t mw = 0;
    const char* nm = std::getenv("GDSW_NO_SELL_MASK");  // =1: per-entry columns (A/B switch)
    if (allow_mask && !(nm && nm[0] == '1') && mask_feasible(n, ptr, idx, col_add_per_row, skip_first, &mw)) {
      build_mask(n, ptr, idx, col_add_per_row, skip_first);
    }
    slice_off.upload(off);
    row_len.upload(len);
    if (masked) {  // no per-entry columns
      col.release();
      d16.release();
    } else {
      col.upload(c);
      if (has16) d16.upload(d);
      else d16.release();
    }
    std::vector<int64_t> p(ptr, ptr + n + 1);
    csr_ptr.upload(p);
  }
  SellDev view() const {
    SellDev v;
    v.n_rows = n_rows;
    v.slice_off = slice_off.p;
    v.row_len = row_len.p;
    v.col = col.p;
    v.d16 = has16 ? d16.p : nullptr;
    v.uw = uw;
    v.mask = masked ? mask.p : nullptr;
    v.soff = masked ? soff.p : nullptr;
    return v;
  }
};

// place CSR-ordered values (skipping `skip` leading entries per row) into
// SELL order; optionally extract the skipped leading entry (U's diagonal)
template <typename T, typename TS>
__global__ void k_csr_to_sell(int32_t n, const int64_t* __restrict__ ptr,
                              const int64_t* __restrict__ slice_off, const TS* __restrict__ src,
                              T* __restrict__ dst, int skip, T* __restrict__ diag_out, int32_t uw) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t base = uw ? (int64_t)(i >> 5) * 32 * uw + (i & 31) : slice_off[i >> 5] + (i & 31);
  int64_t p0 = ptr[i], p1 = ptr[i + 1];
  if (skip && diag_out) diag_out[i] = (T)src[p0];
  for (int64_t p = p0 + skip, k = 0; p < p1; ++p, ++k) dst[base + 32 * k] = (T)src[p];
}

// ---------------------------------------------------------------------------
// one SELL row, entries consumed in column order, loads issued SELL_U at a
// time: {columns, values} for SELL_U entries together, then the SELL_U x
// gathers together, then the ordered accumulation -- the dependent-load
// chain per row drops from 2*len round trips to 2*ceil(len/SELL_U)
// ---------------------------------------------------------------------------
constexpr int SELL_U = 4;

struct LdNc {  // read-only for the whole kernel: non-coherent path
  template <typename T>
  __device__ __forceinline__ static T ld(const T* p) { return __ldg(p); }
};
struct LdCg {  // written by other CTAs of the same kernel: L2 only
  template <typename T>
  __device__ __forceinline__ static T ld(const T* p) { return __ldcg(p); }
};

// SUB: acc -= v*x (triangular sweeps); else acc += v*x (SpMV)
// uniform-width row: every slot's column and value load is issued at once
// (no dependence on the row length), then the gathers of the row's own
// entries, then the ordered accumulation
template <typename T, typename TX, bool SUB, typename XL, int F, int MW = SELL_UW>
__device__ __forceinline__ T sell_row_uniform(T acc, int64_t base, int len, const T* __restrict__ val,
                                              const SellDev& M, int32_t i, const TX* x) {
  int32_t c[MW];
  T v[MW], xv[MW];
#pragma unroll
  for (int k = 0; k < MW; ++k) {
    if (k < M.uw) {
      const int64_t q = base + 32 * (int64_t)k;
      if constexpr (F != SELL_MASK) c[k] = sell_col<F>(M, i, q);
      v[k] = ldg_stream(val + q);
    }
  }
  if constexpr (F == SELL_MASK) sell_cols<F, MW>(M, i, base, len, c);
#pragma unroll
  for (int k = 0; k < MW; ++k)
    if (k < len) xv[k] = (T)XL::ld(x + c[k]);
#pragma unroll
  for (int k = 0; k < MW; ++k)
    if (k < len) acc = SUB ? rn_sub(acc, rn_mul(v[k], xv[k])) : rn_add(acc, rn_mul(v[k], xv[k]));
  return acc;
}

template <typename T, typename TX, bool SUB, typename XL, int F>
__device__ __forceinline__ T sell_row(T acc, int64_t base, int len, const T* __restrict__ val,
                                      const SellDev& M, int32_t i, const TX* x) {
  if (M.uw) return sell_row_uniform<T, TX, SUB, XL, F>(acc, base, len, val, M, i, x);
  [[maybe_unused]] SellMaskCols mc = F == SELL_MASK ? SellMaskCols(M, i) : SellMaskCols();
  for (int k0 = 0; k0 < len; k0 += SELL_U) {
    int32_t c[SELL_U];
    T v[SELL_U];
#pragma unroll
    for (int u = 0; u < SELL_U; ++u) {
      if (k0 + u < len) {
        const int64_t q = base + 32 * (int64_t)(k0 + u);
        if constexpr (F == SELL_MASK) c[u] = mc.next();
        else c[u] = sell_col<F>(M, i, q);
        v[u] = ldg_stream(val + q);
      }
    }
    T xv[SELL_U];
#pragma unroll
    for (int u = 0; u < SELL_U; ++u)
      if (k0 + u < len) xv[u] = (T)XL::ld(x + c[u]);
#pragma unroll
    for (int u = 0; u < SELL_U; ++u) {
      if (k0 + u < len) acc = SUB ? rn_sub(acc, rn_mul(v[u], xv[u])) : rn_add(acc, rn_mul(v[u], xv[u]));
    }
  }
  return acc;
}

// ---------------------------------------------------------------------------
// SpMV: y = A x (mode 0), y = yin - A x (mode 1), y = alpha A x + beta yin (2)
// ---------------------------------------------------------------------------
template <typename T, int F>
__global__ void __launch_bounds__(256) k_sell_spmv(SellDev A, const T* __restrict__ val,
                                                   const T* __restrict__ x,
                                                   const T* __restrict__ yin,
                                                   T* __restrict__ y, int mode, T alpha, T beta) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n_rows) return;
  const int64_t base = sell_base(A, i);
  const int len = sell_len<F>(A, i);
  const T acc = sell_row<T, T, false, LdNc, F>(T(0), base, len, val, A, i, x);
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
// HINT: iterate vectors read/written with L2 evict_last (they are re-read by
// the next sweep), factor values stream with evict_first
template <typename T, bool HINT>
struct VecIO {
  uint64_t pol;
  __device__ __forceinline__ VecIO() : pol(HINT ? l2_policy_last() : 0) {}
  __device__ __forceinline__ T ld(const T* p) const { return HINT ? ld_last(p, pol) : *p; }
  __device__ __forceinline__ void st(T* p, T v) const {
    if (HINT) st_last(p, v, pol); else *p = v;
  }
};

// sweep direction: rev = 1 runs the row blocks from the end, so a sweep that
// follows one in the other direction starts on the rows whose factor values
// and vectors the previous sweep left in L2 (the sweeps alternate)
__device__ __forceinline__ int32_t sweep_row(int rev) {
  const int32_t b = rev ? (int32_t)(gridDim.x - 1 - blockIdx.x) : (int32_t)blockIdx.x;
  return b * (int32_t)blockDim.x + (int32_t)threadIdx.x;
}

// factor values of the sweeps: evict-first (streamed) measured best with the
// alternating directions (C2 32.83 ms; default policy 33.61 ms; evict-first
// with forward-only sweeps 33.33 ms, tools/gpu_r2c_alt.sh); the vectors keep
// the default policy, so the next sweep's start hits them in L2
constexpr bool SWEEP_VAL_EF = true;
template <typename T>
__device__ __forceinline__ T ld_fval(const T* p) { return SWEEP_VAL_EF ? ldg_stream(p) : __ldg(p); }

// one Jacobi row: acc - sum_k val_k x[col_k] in column order. UNI (uniform
// slice width <= 4): every slot's column and value are loaded at once,
// independent of the row length, then the row's own gathers.
template <typename T, int F, bool UNI, typename IO>
__device__ __forceinline__ T jac_row(const SellDev& M, const T* __restrict__ val, int32_t i, int64_t base,
                                     int len, T acc, const T* x, const IO& io) {
  if (UNI) {
    int32_t c[4];
    T v[4], xv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < M.uw) {
        const int64_t q = base + 32 * (int64_t)k;
        if constexpr (F != SELL_MASK) c[k] = sell_col<F>(M, i, q);
        v[k] = ld_fval(val + q);
      }
    }
    if constexpr (F == SELL_MASK) sell_cols<F, 4>(M, i, base, len, c);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k < len) xv[k] = io.ld(x + c[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k < len) acc = rn_sub(acc, rn_mul(v[k], xv[k]));
  } else {
    [[maybe_unused]] SellMaskCols mc = F == SELL_MASK ? SellMaskCols(M, i) : SellMaskCols();
    for (int k = 0; k < len; ++k) {
      const int64_t q = base + 32 * (int64_t)k;
      int32_t c;
      if constexpr (F == SELL_MASK) c = mc.next();
      else c = sell_col<F>(M, i, q);
      acc = rn_sub(acc, rn_mul(ld_fval(val + q), io.ld(x + c)));
    }
  }
  return acc;
}

template <typename T, bool HINT, int F, bool UNI>
__global__ void __launch_bounds__(256) k_jacobi_lower(SellDev L, const T* __restrict__ lval,
                                                      const T* __restrict__ b,
                                                      const T* __restrict__ x,
                                                      T* __restrict__ xn, int rev) {
  const int32_t i = sweep_row(rev);
  if (i >= L.n_rows) return;
  const VecIO<T, HINT> io;
  const int64_t base = sell_base(L, i);
  const int len = sell_len<F>(L, i);
  const T acc = jac_row<T, F, UNI>(L, lval, i, base, len, io.ld(b + i), x, io);
  io.st(xn + i, acc);
}

// x_new = D^-1 (b - (U - D) x)  (U off-diagonal part in SELL, D separate)
template <typename T, bool HINT, int F, bool UNI>
__global__ void __launch_bounds__(256) k_jacobi_upper(SellDev U, const T* __restrict__ uval,
                                                      const T* __restrict__ diag,
                                                      const T* __restrict__ b,
                                                      const T* __restrict__ x,
                                                      T* __restrict__ xn, int rev) {
  const int32_t i = sweep_row(rev);
  if (i >= U.n_rows) return;
  const VecIO<T, HINT> io;
  const int64_t base = sell_base(U, i);
  const int len = sell_len<F>(U, i);
  const T acc = jac_row<T, F, UNI>(U, uval, i, base, len, io.ld(b + i), x, io);
  io.st(xn + i, rn_div(acc, io.ld(diag + i)));
}

// last L sweep fused with the first U iterate: writes both the L result F
// and y1 = F / diag (saves one pass over the vectors)
template <typename T, bool HINT, int F, bool UNI>
__global__ void __launch_bounds__(256) k_jacobi_lower_diag(SellDev L, const T* __restrict__ lval,
                                                           const T* __restrict__ b,
                                                           const T* __restrict__ x,
                                                           T* __restrict__ xn,
                                                           const T* __restrict__ diag,
                                                           T* __restrict__ y1, int rev) {
  const int32_t i = sweep_row(rev);
  if (i >= L.n_rows) return;
  const VecIO<T, HINT> io;
  const int64_t base = sell_base(L, i);
  const int len = sell_len<F>(L, i);
  const T f = jac_row<T, F, UNI>(L, lval, i, base, len, io.ld(b + i), x, io);
  io.st(xn + i, f);
  io.st(y1 + i, rn_div(f, io.ld(diag + i)));
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
template <typename T, bool HINT, int F, bool UNI>
__global__ void __launch_bounds__(256) k_gather_jacobi_lower(SellDev L,
                                                             const T* __restrict__ lval,
                                                             const int32_t* __restrict__ gmap,
                                                             const double* __restrict__ r,
                                                             T* __restrict__ b,
                                                             T* __restrict__ xn, int rev) {
  const int32_t i = sweep_row(rev);
  if (i >= L.n_rows) return;
  const int64_t base = sell_base(L, i);
  const int len = sell_len<F>(L, i);
  const VecIO<T, HINT> io;
  const T bi = (T)r[gmap[i]];
  io.st(b + i, bi);
  // x1 = b: neighbours' b read straight from r through gmap
  T acc = bi;
  constexpr int W = UNI ? 4 : SELL_U;
  const int kend = UNI ? 1 : len;  // UNI: one batch covers every slot
  [[maybe_unused]] SellMaskCols mc = F == SELL_MASK ? SellMaskCols(L, i) : SellMaskCols();
  for (int k0 = 0; k0 < kend; k0 += W) {
    int32_t c[W];
    T v[W];
#pragma unroll
    for (int u = 0; u < W; ++u) {
      if (F == SELL_MASK) c[u] = mc.next();
      if (UNI ? u < L.uw : k0 + u < len) {
        const int64_t q = base + 32 * (int64_t)(k0 + u);
        if constexpr (F != SELL_MASK) c[u] = sell_col<F>(L, i, q);
        v[u] = ld_fval(lval + q);
      }
    }
    int32_t g[W];
#pragma unroll
    for (int u = 0; u < W; ++u)
      if (k0 + u < len) g[u] = __ldg(gmap + c[u]);
#pragma unroll
    for (int u = 0; u < W; ++u)
      if (k0 + u < len) acc = rn_sub(acc, rn_mul(v[u], (T)__ldg(r + g[u])));
  }
  io.st(xn + i, acc);
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
