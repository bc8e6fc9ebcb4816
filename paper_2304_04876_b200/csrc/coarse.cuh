// Coarse correction of the two-level apply (schwarz.py:302-306):
//   u = Phi^T r  ->  v = A0^-1 u  ->  (Phi v fused into k_scatter_prolong)
//
// Phi is stored the B200 way: for each subdomain s the
// interior rows are one dense column-major panel n_I_s x k_s over a shared
// sorted coarse-column list (no per-entry indices, each panel column is a
// contiguous, coalesced vector), and the interface rows stay CSR. A0^-1 is a
// dense replicated n_c x n_c block.
#pragma once
#include "common.cuh"

namespace gdsw {

struct RestrictDev {
  int32_t n_c;
  const int32_t* colsub;     // [K] subdomain of each panel column
  const int32_t* col_ptr;    // [n_sub+1]
  const int64_t* panel_off;  // [n_sub]
  const int32_t* n_int;      // [n_sub]
  const int32_t* int_ptr;    // [n_sub+1] offsets into int_rows
  const int32_t* int_rows;   // interior rows (vector positions), per subdomain sorted
  const int64_t* pgt_ptr;    // [n_c+1] Phi_Gamma^T, coarse-major
  const int32_t* pgt_row;    // vector position of the interface row
  const int32_t* clist_ptr;  // [n_c+1] panel columns that map to coarse column c (ascending s)
  const int32_t* clist;      // panel column ids
};

// one CTA per panel column: pdot[col] = sum_row P[col][row] * r[int_rows[row]]
template <typename T>
__global__ void __launch_bounds__(256) k_restrict_panels(RestrictDev R, const T* __restrict__ panel,
                                                         const double* __restrict__ r,
                                                         T* __restrict__ pdot) {
  const int32_t col = blockIdx.x;
  const int32_t s = R.colsub[col];
  const int32_t c = col - R.col_ptr[s];
  const int32_t ni = R.n_int[s];
  const T* pc = panel + R.panel_off[s] + (int64_t)c * ni;
  const int32_t* rows = R.int_rows + R.int_ptr[s];
  T acc = T(0);
  for (int32_t i = threadIdx.x; i < ni; i += blockDim.x)
    acc += ldg_stream(pc + i) * (T)r[__ldg(rows + i)];
  __shared__ T red[32];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    T t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : T(0);
    t = warp_sum(t);
    if (threadIdx.x == 0) pdot[col] = t;
  }
}

// one warp per coarse column: u[c] = Phi_Gamma^T[c,:] r + sum of its panel dots
template <typename T>
__global__ void k_restrict_final(RestrictDev R, const T* __restrict__ pgt_val,
                                 const double* __restrict__ r, const T* __restrict__ pdot,
                                 T* __restrict__ u) {
  const int32_t c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= R.n_c) return;
  T acc = T(0);
  for (int64_t p = R.pgt_ptr[c] + lane; p < R.pgt_ptr[c + 1]; p += 32)
    acc += pgt_val[p] * (T)r[R.pgt_row[p]];
  acc = warp_sum(acc);
  if (lane == 0) {
    for (int32_t t = R.clist_ptr[c]; t < R.clist_ptr[c + 1]; ++t) acc += pdot[R.clist[t]];
    u[c] = acc;
  }
}

// ---------------------------------------------------------------------------
// partial sums received from other ranks (sharded solve). Rows owned by this
// rank that lower-ranked (= lower subdomain ids) ranks overlap start their
// ordered accumulation from the lower partial; rows overlapped by higher
// ranks add the higher partial after the own contributions -- the single-GPU
// order `z[dofs_i] += y_i` for ascending i. Empty ranges on one GPU.
// ---------------------------------------------------------------------------
struct RemoteAdd {
  const double* recv = nullptr;
  int64_t pre_lo = 0, pre_hi = 0, post_lo = 0, post_hi = 0;
  template <typename T>
  __device__ __forceinline__ T start(int64_t g) const {
    return (g >= pre_lo && g < pre_hi) ? (T)recv[g] : T(0);
  }
  template <typename T>
  __device__ __forceinline__ T finish(int64_t g, T acc) const {
    return (g >= post_lo && g < post_hi) ? rn_add(acc, (T)recv[g]) : acc;
  }
};

template <typename T>
__global__ void k_cast_to_f64(int64_t n, const T* __restrict__ a, double* __restrict__ b) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (double)a[i];
}
template <typename T>
__global__ void k_cast_from_f64(int64_t n, const double* __restrict__ a, T* __restrict__ b) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (T)a[i];
}

// one-level scatter over owned rows [lo, hi): z[g] = double(sum of y in
// ascending subdomain order), remote partials folded in order
template <typename T>
__global__ void k_scatter_owned(int64_t lo, int64_t hi, const int32_t* __restrict__ sc_ptr,
                                const int32_t* __restrict__ sc_pos, const T* __restrict__ y,
                                RemoteAdd RA, double* __restrict__ z) {
  const int64_t g = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= hi) return;
  T acc = RA.start<T>(g);
  for (int32_t q = sc_ptr[g]; q < sc_ptr[g + 1]; ++q) acc = rn_add(acc, y[sc_pos[q]]);
  z[g] = (double)RA.finish<T>(g, acc);
}

// this rank's contributions to rows owned by other ranks (its halo rows)
template <typename T>
__global__ void k_scatter_partial(int64_t lo, int64_t hi, const int32_t* __restrict__ sc_ptr,
                                  const int32_t* __restrict__ sc_pos, const T* __restrict__ y,
                                  double* __restrict__ part) {
  const int64_t g = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= hi) return;
  T acc = T(0);
  for (int32_t q = sc_ptr[g]; q < sc_ptr[g + 1]; ++q) acc = rn_add(acc, y[sc_pos[q]]);
  part[g] = (double)acc;
}

// ---------------------------------------------------------------------------
// chunked restriction / prolongation (chunks of <= 256 interior rows that
// never straddle a subdomain, shared with the extension solver)
// ---------------------------------------------------------------------------
struct ChunkDev {
  const int32_t* chunk_sub;
  const int32_t* chunk_row0;
  const int32_t* chunk_nrow;
  const int64_t* chunk_poff;  // partial offset of the chunk's first column
  const int32_t* int_ptr;
  const int32_t* int_rows;
  const int32_t* n_int;
  const int32_t* col_ptr;
  const int32_t* col_ids;
  const int64_t* panel_off;
  const int32_t* ch_g = nullptr;   // [chunk * CH_THREADS + t]: interior row
  const int32_t* ch_y0 = nullptr;  // its first local contribution (block position) or -1
  const int32_t* ch_ny = nullptr;  // number of local contributions
};

constexpr int CH_THREADS = 256;
constexpr int CH_MAXK = 128;

// partial[chunk_poff + c] = sum over the chunk's rows of P[c][row] r[row]
// (r is read once per row, each panel column streamed coalesced). Each of
// the RS_THREADS threads owns rows t and t + RS_THREADS of the chunk and
// adds its two products before the column's warp tree: half the shuffles
// per element (the kernel is shuffle-bound, most of all in fp32).
constexpr int RS_ROWS = 4;
constexpr int RS_THREADS = CH_THREADS / RS_ROWS;
template <typename T>
__global__ void __launch_bounds__(RS_THREADS) k_restrict_chunks(ChunkDev D, const T* __restrict__ panel,
                                                                const double* __restrict__ r,
                                                                T* __restrict__ partial) {
  __shared__ T red[RS_THREADS / 32][CH_MAXK];
  const int32_t ch = blockIdx.x;
  const int32_t s = D.chunk_sub[ch];
  const int32_t ni = D.n_int[s];
  const int k = D.col_ptr[s + 1] - D.col_ptr[s];
  const int32_t nrow = D.chunk_nrow[ch];
  T rv[RS_ROWS];
  bool on[RS_ROWS];
#pragma unroll
  for (int q = 0; q < RS_ROWS; ++q) {
    const int t = threadIdx.x + q * RS_THREADS;
    on[q] = t < nrow;
    rv[q] = on[q] ? (T)r[D.ch_g[(size_t)ch * CH_THREADS + t]] : T(0);
  }
  const T* pc = panel + D.panel_off[s] + D.chunk_row0[ch] + threadIdx.x;
  for (int c = 0; c < k; ++c) {
    const T* p = pc + (int64_t)c * ni;
    T v = T(0);
#pragma unroll
    for (int q = 0; q < RS_ROWS; ++q)
      if (on[q]) v += ldg_stream(p + q * RS_THREADS) * rv[q];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][c] = v;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    T acc = T(0);
#pragma unroll
    for (int w = 0; w < RS_THREADS / 32; ++w) acc += red[w][c];
    partial[D.chunk_poff[ch] + c] = acc;
  }
}

// one CTA per coarse column: u[c] = Phi_Gamma^T[c,:] r + sum of its panel
// partials (flattened list), both as fixed-shape block reductions
template <typename T>
__global__ void __launch_bounds__(256) k_restrict_columns(int32_t n_c, const int64_t* __restrict__ pgt_ptr,
                                                          const int32_t* __restrict__ pgt_row,
                                                          const T* __restrict__ pgt_val,
                                                          const double* __restrict__ r,
                                                          const int64_t* __restrict__ cpart_ptr,
                                                          const int64_t* __restrict__ cpart_idx,
                                                          const T* __restrict__ partial,
                                                          T* __restrict__ u) {
  const int32_t c = blockIdx.x;
  T acc = T(0);
  for (int64_t p = pgt_ptr[c] + threadIdx.x; p < pgt_ptr[c + 1]; p += blockDim.x)
    acc += pgt_val[p] * (T)r[pgt_row[p]];
  for (int64_t p = cpart_ptr[c] + threadIdx.x; p < cpart_ptr[c + 1]; p += blockDim.x)
    acc += partial[cpart_idx[p]];
  __shared__ T red[8];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    T t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : T(0);
    t = warp_sum(t);
    if (threadIdx.x == 0) u[c] = t;
  }
}

// interior rows: z[g] = double( (Phi v)[g] + (0 + y_a + ...) ), Phi row =
// dense panel row over the subdomain's sorted coarse columns (coalesced)
template <typename T>
__device__ __forceinline__ void prolong_interior_chunk(int32_t ch, const ChunkDev& D, const T* __restrict__ panel,
                                                       const T* __restrict__ v, const int32_t* __restrict__ sc_ptr,
                                                       const int32_t* __restrict__ sc_pos, const T* __restrict__ y,
                                                       const RemoteAdd& RA, double* __restrict__ z) {
  if (threadIdx.x >= D.chunk_nrow[ch]) return;
  const int32_t s = D.chunk_sub[ch];
  const int32_t ni = D.n_int[s];
  const int32_t row = D.chunk_row0[ch] + threadIdx.x;
  const size_t ft = (size_t)ch * CH_THREADS + threadIdx.x;
  const int32_t g = D.ch_g[ft];
  const int32_t y0 = D.ch_y0[ft], ny = D.ch_ny[ft];
  const T* pr = panel + D.panel_off[s] + row;
  T zc = T(0);
  // loads of 8 columns in flight (the additions stay in column order)
  const int32_t c0 = D.col_ptr[s], c1 = D.col_ptr[s + 1];
  int32_t c = c0;
  for (; c + 8 <= c1; c += 8, pr += 8 * (int64_t)ni) {
    T pv[8], vv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      pv[u] = ldg_stream(pr + u * (int64_t)ni);
      vv[u] = v[D.col_ids[c + u]];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) zc = rn_add(zc, rn_mul(pv[u], vv[u]));
  }
  for (; c < c1; ++c, pr += ni) zc = rn_add(zc, rn_mul(ldg_stream(pr), v[D.col_ids[c]]));
  T acc = RA.start<T>(g);
  if (ny > 0) acc = rn_add(acc, y[y0]);
  if (ny > 1)
    for (int32_t q = sc_ptr[g] + 1; q < sc_ptr[g + 1]; ++q) acc = rn_add(acc, y[sc_pos[q]]);
  z[g] = (double)rn_add(zc, RA.finish<T>(g, acc));
}

// interface rows: Phi_Gamma row (CSR by interface position) + scatter
struct ProlongGamma {
  int32_t n_gamma;
  const int32_t* gamma_rows;
  const int64_t* pg_ptr;
  const int32_t* pg_col;
};

template <typename T>
__device__ __forceinline__ void prolong_interface_row(int32_t t, const ProlongGamma& G, const T* __restrict__ pg_val,
                                                      const T* __restrict__ v, const int32_t* __restrict__ sc_ptr,
                                                      const int32_t* __restrict__ sc_pos, const T* __restrict__ y,
                                                      const RemoteAdd& RA, double* __restrict__ z) {
  if (t >= G.n_gamma) return;
  const int32_t* gamma_rows = G.gamma_rows;
  const int64_t* pg_ptr = G.pg_ptr;
  const int32_t* pg_col = G.pg_col;
  const int32_t g = gamma_rows[t];
  T zc = T(0);
  for (int64_t p = pg_ptr[t]; p < pg_ptr[t + 1]; ++p) zc = rn_add(zc, rn_mul(pg_val[p], v[pg_col[p]]));
  T acc = RA.start<T>(g);
  for (int32_t q = sc_ptr[g]; q < sc_ptr[g + 1]; ++q) acc = rn_add(acc, y[sc_pos[q]]);
  z[g] = (double)rn_add(zc, RA.finish<T>(g, acc));
}

// the whole prolongation + scatter in one launch: CTAs [0, n_chunks) take
// interior chunks (panel rows), the rest take interface rows
template <typename T>
__global__ void __launch_bounds__(CH_THREADS) k_prolong(int32_t n_chunks, ChunkDev D, const T* __restrict__ panel,
                                                        ProlongGamma G, const T* __restrict__ pg_val,
                                                        const T* __restrict__ v, const int32_t* __restrict__ sc_ptr,
                                                        const int32_t* __restrict__ sc_pos, const T* __restrict__ y,
                                                        RemoteAdd RA, double* __restrict__ z) {
  if ((int32_t)blockIdx.x < n_chunks)
    prolong_interior_chunk<T>(blockIdx.x, D, panel, v, sc_ptr, sc_pos, y, RA, z);
  else
    prolong_interface_row<T>((blockIdx.x - n_chunks) * CH_THREADS + threadIdx.x, G, pg_val, v, sc_ptr, sc_pos, y,
                             RA, z);
}

// dense replicated coarse solve: v = A0^-1 u, one warp per row
template <typename T>
__global__ void k_coarse_gemv(int32_t n_c, const T* __restrict__ ainv, const T* __restrict__ u,
                              T* __restrict__ v) {
  const int32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n_c) return;
  const T* row = ainv + (int64_t)i * n_c;
  // four independent partial sums: four row loads in flight per lane
  T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0);
  int32_t j = lane;
  for (; j + 96 < n_c; j += 128) {
    const T r0 = ldg_stream(row + j), r1 = ldg_stream(row + j + 32), r2 = ldg_stream(row + j + 64),
            r3 = ldg_stream(row + j + 96);
    a0 += r0 * u[j];
    a1 += r1 * u[j + 32];
    a2 += r2 * u[j + 64];
    a3 += r3 * u[j + 96];
  }
  for (; j < n_c; j += 32) a0 += ldg_stream(row + j) * u[j];
  const T acc = warp_sum((a0 + a1) + (a2 + a3));
  if (lane == 0) v[i] = acc;
}

}  // namespace gdsw
