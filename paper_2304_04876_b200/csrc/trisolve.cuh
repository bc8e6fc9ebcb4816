// Scheduled batched SpTRSV for exact / ILU(k) factors (trisolve_levelset,
// local_solvers.py:404-410, over trisolve_forward_unit / trisolve_backward,
// _kernels.py:473-496): one CTA per subdomain walks the host level schedule
// of its L and U factors with the block's iterate resident in shared memory
// (global memory when it does not fit), one __syncthreads per level.
//
// Work inside a level is split by row length:
//  * short rows (<= TS_SHORT entries): one thread per row, entries stored
//    SELL-32 per level (entry k of the row in lane l of a 32-row slice at
//    slice_off + 32k + l: coalesced), accumulated sequentially in column
//    order with round-to-nearest mul/sub -- bit-identical to the reference;
//  * medium rows (<= TS_CHAIN): one warp per row; the products are formed in
//    parallel, the subtraction chain runs in column order (bit-identical);
//  * long rows (dense separator rows of exact LU factors): one warp per row,
//    lane-strided fused products and a fixed shuffle tree -- deterministic,
//    not bit-identical (within 1e-13 relative of sequential substitution).
// Every level's data is contiguous in the schedule-ordered value/column
// arrays, so a subdomain streams its factors front to back exactly once.
#pragma once
#include <algorithm>

#include "common.cuh"

namespace gdsw {

constexpr int TS_THREADS = 256;
constexpr int TS_SHORT = 32;
constexpr int TS_CHAIN = 128;

struct TriSchedDev {
  const int32_t* lev_sub = nullptr;   // [n_sub + 1] level range of each subdomain
  const int4* lev = nullptr;          // {warp task begin, #warp tasks, slice begin, #short rows}
  const int32_t* wt_row = nullptr;    // warp tasks: block-local row
  const int32_t* wt_len = nullptr;
  const int64_t* wt_off = nullptr;    // entry offset of the row's contiguous data
  const int32_t* st_row = nullptr;    // short rows, [slice * 32 + lane]
  const int32_t* st_len = nullptr;
  const int64_t* sl_off = nullptr;    // entry offset of each 32-row slice
  const int32_t* col = nullptr;       // block-local columns, schedule order
};

// host-side schedule of one factor over all subdomains
struct TriSched {
  int64_t entries = 0;       // schedule slots (incl. slice padding)
  int64_t n_levels = 0;
  int64_t max_rows = 0;      // largest block
  DBuf<int32_t> lev_sub, wt_row, wt_len, st_row, st_len, col;
  DBuf<int4> lev;
  DBuf<int64_t> wt_off, sl_off;
  // placement tasks (CSR position -> schedule slot), kept for value refills
  DBuf<int64_t> pl_src, pl_dst;
  DBuf<int32_t> pl_len, pl_stride;
  int64_t n_place = 0;

  // ptr/idx: concatenated CSR (block-local columns); skip: leading entries
  // of each row not in the schedule (1 = U's diagonal)
  void build(int32_t n_sub, const std::vector<int64_t>& sub_ptr, const std::vector<int64_t>& ptr,
             const std::vector<int64_t>& idx, int skip, const std::vector<int64_t>& lsub,
             const std::vector<int64_t>& lptr, const std::vector<int64_t>& lrows) {
    std::vector<int32_t> h_lev_sub(n_sub + 1), h_wt_row, h_wt_len, h_st_row, h_st_len;
    std::vector<int4> h_lev;
    std::vector<int64_t> h_wt_off, h_sl_off, p_src, p_dst;
    std::vector<int32_t> p_len, p_stride;
    int64_t cur = 0;
    max_rows = 0;
    for (int32_t s = 0; s < n_sub; ++s) {
      max_rows = std::max<int64_t>(max_rows, sub_ptr[s + 1] - sub_ptr[s]);
      h_lev_sub[s] = (int32_t)h_lev.size();
      const int64_t base = sub_ptr[s];
      for (int64_t lv = lsub[s]; lv < lsub[s + 1]; ++lv) {
        int4 d;
        d.x = (int32_t)h_wt_row.size();
        d.z = (int32_t)h_sl_off.size();
        std::vector<int64_t> shorts;
        for (int64_t t = lptr[lv]; t < lptr[lv + 1]; ++t) {
          const int64_t row = lrows[t];
          const int64_t g = base + row;
          const int64_t len = ptr[g + 1] - ptr[g] - skip;
          if (len > TS_SHORT) {
            h_wt_row.push_back((int32_t)row);
            h_wt_len.push_back((int32_t)len);
            h_wt_off.push_back(cur);
            p_src.push_back(ptr[g] + skip);
            p_dst.push_back(cur);
            p_len.push_back((int32_t)len);
            p_stride.push_back(1);
            cur += len;
          } else {
            shorts.push_back(row);
          }
        }
        d.y = (int32_t)h_wt_row.size() - d.x;
        d.w = (int32_t)shorts.size();
        for (size_t s0 = 0; s0 < shorts.size(); s0 += 32) {
          int64_t w = 0;
          for (size_t q = s0; q < std::min(shorts.size(), s0 + 32); ++q) {
            const int64_t g = base + shorts[q];
            w = std::max<int64_t>(w, ptr[g + 1] - ptr[g] - skip);
          }
          h_sl_off.push_back(cur);
          for (size_t l = 0; l < 32; ++l) {
            const size_t q = s0 + l;
            if (q < shorts.size()) {
              const int64_t g = base + shorts[q];
              const int64_t len = ptr[g + 1] - ptr[g] - skip;
              h_st_row.push_back((int32_t)shorts[q]);
              h_st_len.push_back((int32_t)len);
              if (len > 0) {
                p_src.push_back(ptr[g] + skip);
                p_dst.push_back(cur + (int64_t)l);
                p_len.push_back((int32_t)len);
                p_stride.push_back(32);
              }
            } else {
              h_st_row.push_back(0);
              h_st_len.push_back(0);
            }
          }
          cur += 32 * w;
        }
        h_lev.push_back(d);
      }
    }
    h_lev_sub[n_sub] = (int32_t)h_lev.size();
    entries = cur;
    n_levels = (int64_t)h_lev.size();
    lev_sub.upload(h_lev_sub);
    lev.upload(h_lev);
    wt_row.upload(h_wt_row);
    wt_len.upload(h_wt_len);
    wt_off.upload(h_wt_off);
    st_row.upload(h_st_row);
    st_len.upload(h_st_len);
    sl_off.upload(h_sl_off);
    pl_src.upload(p_src);
    pl_dst.upload(p_dst);
    pl_len.upload(p_len);
    pl_stride.upload(p_stride);
    n_place = (int64_t)p_src.size();
    // columns: block-local, placed from the host CSR
    std::vector<int32_t> c(std::max<int64_t>(entries, 1), 0);
    for (int64_t q = 0; q < n_place; ++q)
      for (int32_t k = 0; k < p_len[q]; ++k) c[p_dst[q] + (int64_t)k * p_stride[q]] = (int32_t)idx[p_src[q] + k];
    col.upload(c);
  }
  TriSchedDev view() const {
    TriSchedDev v;
    v.lev_sub = lev_sub.p;
    v.lev = lev.p;
    v.wt_row = wt_row.p;
    v.wt_len = wt_len.p;
    v.wt_off = wt_off.p;
    v.st_row = st_row.p;
    v.st_len = st_len.p;
    v.sl_off = sl_off.p;
    v.col = col.p;
    return v;
  }
};

// values CSR -> schedule order (padding slots stay zero)
template <typename T>
__global__ void k_sched_place(int64_t n_place, const int64_t* __restrict__ src, const int64_t* __restrict__ dst,
                              const int32_t* __restrict__ len, const int32_t* __restrict__ stride,
                              const T* __restrict__ csr_val, T* __restrict__ out) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
  if (q >= n_place) return;
  const int64_t s0 = src[q], d0 = dst[q];
  const int32_t n = len[q], st = stride[q];
  for (int32_t k = threadIdx.x; k < n; k += blockDim.x) out[d0 + (int64_t)k * st] = csr_val[s0 + k];
}

// U's diagonal (first entry of each CSR row) by concatenated row
template <typename T>
__global__ void k_extract_diag(int32_t n, const int64_t* __restrict__ ptr, const T* __restrict__ uval,
                               T* __restrict__ diag) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) diag[i] = uval[ptr[i]];
}

// Software pipeline over levels. Per thread, the FIRST warp task (warp w:
// task w) and the FIRST short row (thread t: row t) of a level are
// prefetched: at the compute stage of level lv the thread issues the data
// loads of lv+1 (first TS_PF entries of its items), the index loads of lv+2
// (row, length, data offset) and the descriptor of lv+3, so after each
// barrier only shared-memory gathers and arithmetic remain on the critical
// path. Further items of wide levels load on demand.
constexpr int TS_PF = 4;  // entries per lane prefetched (warp task: 128, short row: 4)

struct TsIdx {
  int32_t wrow, wlen, srow, slen;
  int64_t woff, soff;
};

template <typename T>
struct TsData {
  T wv[TS_PF], sv[TS_PF];
  int32_t wc[TS_PF], sc[TS_PF];
};

__device__ __forceinline__ int4 ts_desc(const TriSchedDev& S, int lv, int lv1) {
  return lv < lv1 ? S.lev[lv] : make_int4(0, 0, 0, 0);
}

__device__ __forceinline__ TsIdx ts_index(const TriSchedDev& S, int4 d, int warp) {
  TsIdx ix;
  ix.wrow = ix.wlen = ix.srow = ix.slen = 0;
  ix.woff = ix.soff = 0;
  if (warp < d.y) {
    const int q = d.x + warp;
    ix.wrow = S.wt_row[q];
    ix.wlen = S.wt_len[q];
    ix.woff = S.wt_off[q];
  }
  if ((int)threadIdx.x < d.w) {
    const int64_t g = (int64_t)d.z * 32 + threadIdx.x;
    ix.srow = S.st_row[g];
    ix.slen = S.st_len[g];
    ix.soff = S.sl_off[d.z + (threadIdx.x >> 5)] + (threadIdx.x & 31);
  }
  return ix;
}

template <typename T>
__device__ __forceinline__ void ts_data(const TriSchedDev& S, const T* __restrict__ val, const TsIdx& ix,
                                        TsData<T>& dt, int lane) {
#pragma unroll
  for (int u = 0; u < TS_PF; ++u) {
    const int k = lane + 32 * u;
    if (k < ix.wlen) {
      dt.wv[u] = val[ix.woff + k];
      dt.wc[u] = S.col[ix.woff + k];
    }
    if (u < ix.slen) {
      dt.sv[u] = val[ix.soff + 32 * u];
      dt.sc[u] = S.col[ix.soff + 32 * u];
    }
  }
}

// warp task: x[row] -= row . x (UP: then / diag). wv/wc hold entries
// lane + 32u for u < TS_PF.
template <typename T, bool UP>
__device__ __forceinline__ void ts_warp_row(const TriSchedDev& S, const T* __restrict__ val,
                                            const T* __restrict__ diag, T* x, int32_t row, int32_t len,
                                            int64_t off, const T* wv, const int32_t* wc, int lane) {
  T xi = x[row];
  if (len <= TS_CHAIN) {
    // products in parallel, subtraction chain in column order (bitwise)
    T p[TS_PF];
#pragma unroll
    for (int u = 0; u < TS_PF; ++u) {
      const int k = lane + 32 * u;
      p[u] = k < len ? rn_mul(wv[u], x[wc[u]]) : T(0);
    }
#pragma unroll
    for (int u = 0; u < TS_PF; ++u) {
      if (32 * u >= len) break;  // warp-uniform
#pragma unroll
      for (int l = 0; l < 32; ++l) {
        const T pk = __shfl_sync(0xffffffffu, p[u], l);
        if (32 * u + l < len) xi = rn_sub(xi, pk);
      }
    }
  } else {
    T acc = T(0);
#pragma unroll
    for (int u = 0; u < TS_PF; ++u) acc = fma(wv[u], x[wc[u]], acc);  // len > 128: all valid
#pragma unroll 4
    for (int k = lane + 32 * TS_PF; k < len; k += 32) acc = fma(val[off + k], x[S.col[off + k]], acc);
    xi = xi - warp_sum(acc);
  }
  if (UP) xi = rn_div(xi, diag[row]);
  if (lane == 0) x[row] = xi;
}

// short row: sequential in column order (bitwise); sv/sc hold the first
// TS_PF entries
template <typename T, bool UP>
__device__ __forceinline__ void ts_short_row(const TriSchedDev& S, const T* __restrict__ val,
                                             const T* __restrict__ diag, T* x, int32_t row, int32_t len,
                                             int64_t b, const T* sv, const int32_t* sc) {
  T acc = x[row];
  {
    T xv[TS_PF];
#pragma unroll
    for (int u = 0; u < TS_PF; ++u)
      if (u < len) xv[u] = x[sc[u]];
#pragma unroll
    for (int u = 0; u < TS_PF; ++u)
      if (u < len) acc = rn_sub(acc, rn_mul(sv[u], xv[u]));
  }
  for (int k0 = TS_PF; k0 < len; k0 += 4) {
    int32_t c[4];
    T v[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (k0 + u < len) {
        c[u] = S.col[b + 32 * (k0 + u)];
        v[u] = val[b + 32 * (k0 + u)];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (k0 + u < len) xv[u] = x[c[u]];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (k0 + u < len) acc = rn_sub(acc, rn_mul(v[u], xv[u]));
  }
  if (UP) acc = rn_div(acc, diag[row]);
  x[row] = acc;
}

template <typename T, bool UP>
__device__ __forceinline__ void ts_levels(const TriSchedDev& S, const T* __restrict__ val,
                                          const T* __restrict__ diag, T* x, int s) {
  constexpr int NW = TS_THREADS / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lv0 = S.lev_sub[s], lv1 = S.lev_sub[s + 1];
  // pipeline prologue: desc(lv0..lv0+2), index(lv0, lv0+1), data(lv0)
  int4 d0 = ts_desc(S, lv0, lv1), d1 = ts_desc(S, lv0 + 1, lv1), d2 = ts_desc(S, lv0 + 2, lv1);
  TsIdx i0 = ts_index(S, d0, warp), i1 = ts_index(S, d1, warp);
  TsData<T> t0;
  ts_data(S, val, i0, t0, lane);
  for (int lv = lv0; lv < lv1; ++lv) {
    // issue the loads of the next levels (independent of x)
    const int4 d3 = ts_desc(S, lv + 3, lv1);
    const TsIdx i2 = ts_index(S, d2, warp);
    TsData<T> t1;
    ts_data(S, val, i1, t1, lane);
    // this level: prefetched first items, then the rest on demand
    if (warp < d0.y)
      ts_warp_row<T, UP>(S, val, diag, x, i0.wrow, i0.wlen, i0.woff, t0.wv, t0.wc, lane);
    for (int t = warp + NW; t < d0.y; t += NW) {
      const int q = d0.x + t;
      const int32_t row = S.wt_row[q], len = S.wt_len[q];
      const int64_t off = S.wt_off[q];
      T wv[TS_PF];
      int32_t wc[TS_PF];
#pragma unroll
      for (int u = 0; u < TS_PF; ++u) {
        const int k = lane + 32 * u;
        wv[u] = k < len ? val[off + k] : T(0);
        wc[u] = k < len ? S.col[off + k] : 0;
      }
      ts_warp_row<T, UP>(S, val, diag, x, row, len, off, wv, wc, lane);
    }
    if ((int)threadIdx.x < d0.w)
      ts_short_row<T, UP>(S, val, diag, x, i0.srow, i0.slen, i0.soff, t0.sv, t0.sc);
    for (int t = threadIdx.x + TS_THREADS; t < d0.w; t += TS_THREADS) {
      const int64_t g = (int64_t)d0.z * 32 + t;
      const int32_t row = S.st_row[g], len = S.st_len[g];
      const int64_t b = S.sl_off[d0.z + (t >> 5)] + (t & 31);
      T sv[TS_PF];
      int32_t sc[TS_PF];
#pragma unroll
      for (int u = 0; u < TS_PF; ++u) {
        if (u < len) {
          sv[u] = val[b + 32 * u];
          sc[u] = S.col[b + 32 * u];
        }
      }
      ts_short_row<T, UP>(S, val, diag, x, row, len, b, sv, sc);
    }
    __syncthreads();
    d0 = d1;
    d1 = d2;
    d2 = d3;
    i0 = i1;
    i1 = i2;
    t0 = t1;
  }
}

// unpipelined variant (GDSW_TS_SIMPLE=1): every item loads its index and
// data after the level barrier
template <typename T, bool UP>
__device__ __forceinline__ void ts_levels_simple(const TriSchedDev& S, const T* __restrict__ val,
                                                 const T* __restrict__ diag, T* x, int s) {
  constexpr int NW = TS_THREADS / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lv0 = S.lev_sub[s], lv1 = S.lev_sub[s + 1];
  for (int lv = lv0; lv < lv1; ++lv) {
    const int4 d0 = S.lev[lv];
    for (int t = warp; t < d0.y; t += NW) {
      const int q = d0.x + t;
      const int32_t row = S.wt_row[q], len = S.wt_len[q];
      const int64_t off = S.wt_off[q];
      T wv[TS_PF];
      int32_t wc[TS_PF];
#pragma unroll
      for (int u = 0; u < TS_PF; ++u) {
        const int k = lane + 32 * u;
        wv[u] = k < len ? val[off + k] : T(0);
        wc[u] = k < len ? S.col[off + k] : 0;
      }
      ts_warp_row<T, UP>(S, val, diag, x, row, len, off, wv, wc, lane);
    }
    for (int t = threadIdx.x; t < d0.w; t += TS_THREADS) {
      const int64_t g = (int64_t)d0.z * 32 + t;
      const int32_t row = S.st_row[g], len = S.st_len[g];
      const int64_t b = S.sl_off[d0.z + (t >> 5)] + (t & 31);
      T sv[TS_PF];
      int32_t sc[TS_PF];
#pragma unroll
      for (int u = 0; u < TS_PF; ++u) {
        if (u < len) {
          sv[u] = val[b + 32 * u];
          sc[u] = S.col[b + 32 * u];
        }
      }
      ts_short_row<T, UP>(S, val, diag, x, row, len, b, sv, sc);
    }
    __syncthreads();
  }
}

// one CTA per subdomain: gather (ordering folded into gmap), L levels, U
// levels, block solution written to y (concatenated block layout)
template <typename T, bool SMEM, bool PIPE>
__global__ void __launch_bounds__(TS_THREADS, 2) k_trisolve_sched(TriSchedDev Ls, TriSchedDev Us,
                                                               const T* __restrict__ lval,
                                                               const T* __restrict__ uval,
                                                               const T* __restrict__ udiag,
                                                               const int32_t* __restrict__ sub_ptr,
                                                               const int32_t* __restrict__ gmap,
                                                               const double* __restrict__ r,
                                                               T* __restrict__ y) {
  extern __shared__ __align__(16) unsigned char ts_smem[];
  const int s = blockIdx.x;
  const int32_t base = sub_ptr[s], ns = sub_ptr[s + 1] - base;
  T* x = SMEM ? reinterpret_cast<T*>(ts_smem) : y + base;
  for (int32_t k = threadIdx.x; k < ns; k += TS_THREADS) x[k] = (T)r[gmap[base + k]];
  __syncthreads();
  if (PIPE) {
    ts_levels<T, false>(Ls, lval, nullptr, x, s);
    ts_levels<T, true>(Us, uval, udiag + base, x, s);
  } else {
    ts_levels_simple<T, false>(Ls, lval, nullptr, x, s);
    ts_levels_simple<T, true>(Us, uval, udiag + base, x, s);
  }
  if (SMEM)
    for (int32_t k = threadIdx.x; k < ns; k += TS_THREADS) y[base + k] = x[k];
}

}  // namespace gdsw
