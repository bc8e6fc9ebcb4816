// Dataflow FastSpTRSV: every Jacobi sweep of L and U over all subdomains in
// ONE persistent launch (jacobi_trisolve_lower_unit / _upper,
// _kernels.py:620-656; fast_trisolve, local_solvers.py:413-427).
//
// Work items are (subdomain group, sweep, row chunk), handed out in that
// order by a monotonic 64-bit atomic ticket. Chunk c of sweep t may start
// once sweep t-1 is done on chunks c-K..c+K of the same subdomain (K = the
// factor's reach in chunks): that covers the rows it reads and the rows
// whose readers it would overwrite. Completion is an epoch stamp per (sweep,
// chunk) written with st.release and polled with ld.acquire, so nothing is
// reset between launches. Items only wait on items with smaller tickets,
// which are already running, so the schedule cannot deadlock.
//
// Subdomains are grouped so that one group's factors and iterates (tens of
// MB) stay resident in the 126 MB L2 while all its sweeps run: each factor
// streams from HBM once per apply instead of once per sweep. Per-row
// arithmetic is the sequential kernels' (bit-identical to the reference);
// iterates written by other CTAs are read through L2 (ld.global.cg).
#pragma once
#include "common.cuh"
#include "sparse.cuh"

namespace gdsw {

constexpr int JF_THREADS = 256;
constexpr int JF_MAXSW = 32;
// RPT rows per thread (independent, loads interleaved); work item = 256*RPT
// rows; occupancy bound so that latency is hidden across warps

struct JfSweep {
  int kind;           // 0: gather + first L iterate, 1: L, 2: last L + y1 = F/D, 3: U
  const void* xin;    // previous iterate (kind 1..3)
  void* xout;
  const void* rhs;    // B (L sweeps) or F (U sweeps)
  void* out2;         // kind 0: B; kind 2: y1
};

constexpr int JF_MAXSUB = 1024;   // subdomain tables staged in shared memory
constexpr int JF_MAXGRP = 256;

struct JfPlan {
  SellDev L, U;
  const int32_t* sub_chunk0;   // [n_sub + 1] chunk range of each subdomain
  const int32_t* sub_row0;     // [n_sub + 1] row range (concatenated)
  const int32_t* sub_reach;    // [n_sub] K: rows of chunk c touch only chunks c-K..c+K
  const int32_t* group_sub0;   // [n_groups + 1] subdomain range of each group
  const int32_t* gmap;
  int32_t n_groups, n_sub, n_chunks, n_sweeps, rows_per_chunk;
  int64_t n_items;
  unsigned long long* ticket;  // monotonic across launches
  unsigned long long ticket_base;
  unsigned* done;              // [n_sweeps * n_chunks], = epoch when finished
  unsigned epoch;
  JfSweep sw[JF_MAXSW];
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// JF_RPT independent rows per thread, loads interleaved across the rows;
// each row still accumulates in its own column order (bit-identical)
template <typename T, bool D16, int MODE, int JF_RPT>  // MODE 0: x from r[gmap[]], 1: x iterate
__device__ __forceinline__ void jf_rows(const SellDev& M, const T* __restrict__ val, const int32_t* rows,
                                        const bool* ok, T* acc, const T* x, const double* __restrict__ r,
                                        const int32_t* __restrict__ gmap) {
  int64_t base[JF_RPT];
  int len[JF_RPT], lmax = 0;
#pragma unroll
  for (int u = 0; u < JF_RPT; ++u) {
    const int32_t i = rows[u];
    base[u] = ok[u] ? sell_base(M, i) : 0;
    len[u] = ok[u] ? (int)M.row_len[i] : 0;
  }
#pragma unroll
  for (int u = 0; u < JF_RPT; ++u) lmax = max(lmax, len[u]);
  for (int k = 0; k < lmax; ++k) {
    T v[JF_RPT], xv[JF_RPT];
    int32_t c[JF_RPT];
#pragma unroll
    for (int u = 0; u < JF_RPT; ++u) {
      if (k < len[u]) {
        const int64_t q = base[u] + 32 * (int64_t)k;
        v[u] = val[q];
        c[u] = sell_col<D16>(M, rows[u], q);
      }
    }
#pragma unroll
    for (int u = 0; u < JF_RPT; ++u) {
      if (k < len[u]) xv[u] = MODE == 0 ? (T)__ldg(r + __ldg(gmap + c[u])) : __ldcg(x + c[u]);
    }
#pragma unroll
    for (int u = 0; u < JF_RPT; ++u)
      if (k < len[u]) acc[u] = rn_sub(acc[u], rn_mul(v[u], xv[u]));
  }
}

template <typename T, bool D16, int JF_RPT>
__global__ void __launch_bounds__(JF_THREADS, 8 / JF_RPT) k_jacobi_flow(JfPlan P, const T* __restrict__ lval,
                                                                      const T* __restrict__ uval,
                                                                      const T* __restrict__ diag,
                                                                      const double* __restrict__ r) {
  __shared__ int32_t s_chunk0[JF_MAXSUB + 1], s_row0[JF_MAXSUB + 1], s_reach[JF_MAXSUB];
  __shared__ int32_t s_gsub0[JF_MAXGRP + 1];
  __shared__ int64_t s_gitem0[JF_MAXGRP + 1];
  __shared__ int64_t s_item;
  for (int k = threadIdx.x; k <= P.n_sub; k += JF_THREADS) {
    s_chunk0[k] = P.sub_chunk0[k];
    s_row0[k] = P.sub_row0[k];
    if (k < P.n_sub) s_reach[k] = P.sub_reach[k];
  }
  if (threadIdx.x == 0) {
    int64_t it = 0;
    for (int g = 0; g <= P.n_groups; ++g) {
      const int32_t sb = P.group_sub0[g];
      s_gsub0[g] = sb;
      if (g > 0) it += (int64_t)P.n_sweeps * (P.sub_chunk0[sb] - P.sub_chunk0[s_gsub0[g - 1]]);
      s_gitem0[g] = it;
    }
    s_item = (int64_t)(atomicAdd(P.ticket, 1ull) - P.ticket_base);
  }
  __syncthreads();
  for (;;) {
    const int64_t item = s_item;
    if (item >= P.n_items) break;
    __syncthreads();  // everyone has read s_item
    if (threadIdx.x == 0) s_item = (int64_t)(atomicAdd(P.ticket, 1ull) - P.ticket_base);
    // decode (group, sweep, chunk) from the shared tables
    int g = 0;
    while (g + 1 < P.n_groups && s_gitem0[g + 1] <= item) ++g;
    const int32_t gc0 = s_chunk0[s_gsub0[g]], gnc = s_chunk0[s_gsub0[g + 1]] - gc0;
    const int64_t rel = item - s_gitem0[g];
    const int t = (int)(rel / gnc);
    const int32_t c = gc0 + (int32_t)(rel % gnc);
    int lo_s = s_gsub0[g], hi_s = s_gsub0[g + 1] - 1;  // subdomain of chunk c
    while (lo_s < hi_s) {
      const int mid = (lo_s + hi_s + 1) >> 1;
      if (s_chunk0[mid] <= c) lo_s = mid; else hi_s = mid - 1;
    }
    const int32_t s = lo_s;
    const JfSweep sw = P.sw[t];
    const int32_t row0 = s_row0[s] + (c - s_chunk0[s]) * P.rows_per_chunk;
    const int32_t nrow = min(P.rows_per_chunk, s_row0[s + 1] - row0);
    int32_t rows[JF_RPT];
    bool ok[JF_RPT];
    T acc[JF_RPT];
#pragma unroll
    for (int u = 0; u < JF_RPT; ++u) {
      const int32_t k = threadIdx.x + u * JF_THREADS;
      ok[u] = k < nrow;
      rows[u] = row0 + (ok[u] ? k : 0);
    }
    if (t > 0) {
      // sweep t-1 done on the chunks this one reads (RAW) and on the chunks
      // reading the rows it overwrites (WAR)
      const int32_t K = s_reach[s];
      const int32_t lo = max(s_chunk0[s], c - K), hi = min(s_chunk0[s + 1] - 1, c + K);
      const int32_t w = lo + (int32_t)threadIdx.x;
      if (w <= hi) {
        const unsigned* d = P.done + (size_t)(t - 1) * P.n_chunks + w;
        while (ld_acquire_u32(d) != P.epoch) __nanosleep(32);
      }
      __syncthreads();
    }
    if (sw.kind == 0) {
      // x1 = b - (L - I) b with b = r[gmap] (neighbours read from r)
#pragma unroll
      for (int u = 0; u < JF_RPT; ++u) {
        acc[u] = ok[u] ? (T)r[P.gmap[rows[u]]] : T(0);
        if (ok[u]) ((T*)sw.out2)[rows[u]] = acc[u];
      }
      jf_rows<T, D16, 0, JF_RPT>(P.L, lval, rows, ok, acc, nullptr, r, P.gmap);
#pragma unroll
      for (int u = 0; u < JF_RPT; ++u)
        if (ok[u]) ((T*)sw.xout)[rows[u]] = acc[u];
    } else {
      const bool lower = sw.kind != 3;
#pragma unroll
      for (int u = 0; u < JF_RPT; ++u) acc[u] = ok[u] ? __ldcg((const T*)sw.rhs + rows[u]) : T(0);
      if (lower)
        jf_rows<T, D16, 1, JF_RPT>(P.L, lval, rows, ok, acc, (const T*)sw.xin, r, P.gmap);
      else
        jf_rows<T, D16, 1, JF_RPT>(P.U, uval, rows, ok, acc, (const T*)sw.xin, r, P.gmap);
#pragma unroll
      for (int u = 0; u < JF_RPT; ++u) {
        if (!ok[u]) continue;
        const int32_t i = rows[u];
        if (sw.kind == 1) {
          ((T*)sw.xout)[i] = acc[u];
        } else if (sw.kind == 2) {
          ((T*)sw.xout)[i] = acc[u];
          ((T*)sw.out2)[i] = rn_div(acc[u], diag[i]);
        } else {
          ((T*)sw.xout)[i] = rn_div(acc[u], diag[i]);
        }
      }
    }
    __syncthreads();  // orders every thread's stores before the release below
    if (threadIdx.x == 0) st_release_u32(P.done + (size_t)t * P.n_chunks + c, P.epoch);
  }
}

}  // namespace gdsw
