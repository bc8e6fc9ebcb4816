// Factored coarse solve v = A0^-1 u for large coarse spaces: the supernodal
// partitioned inverse of the nested-dissection LU of A0 (built on the host by
// paper_2304_04876_b200/coarse_factor.py; replaces the reference's sparse LU
// + level-set solves, schwarz.py:267-272, 305, and the dense A0^-1 GEMV once
// n_c^2 values per apply stop being cheap).
//
// One launch per supernode-tree level and direction. A CTA takes one task =
// (supernode k, tile of CF_ROWS rows of its stacked block), stages the
// block's input vector in shared memory and computes its rows warp per row
// (coalesced row-major dense rows, fixed shuffle tree):
//  forward  (leaves first): bt = u[C_k] - the children's updates on C_k
//           (fixed order), rows < s: y[C_k] = L_kk^-1 bt (strict-lower part
//           of the diagonal block + the unit diagonal), rows >= s: the
//           update cbuf[R_k] = (L_{R_k,k} L_kk^-1) bt + the children's
//           updates on R_k (multifrontal extend-add)
//  backward (root first): x[C_k] = U_kk^-1 y[C_k] - (U_kk^-1 U_{k,R_k}) x[R_k]
#pragma once
#include "common.cuh"

namespace gdsw {

constexpr int CF_THREADS = 256;
constexpr int CF_ROWS = 16;  // rows of a block per CTA task

struct CoarseFactorDev {
  const int32_t* sn_s;
  const int32_t* sn_r;
  const int32_t* col_ptr;
  const int32_t* col_ids;
  const int32_t* row_ptr;
  const int32_t* row_ids;
  const int64_t* d_off;
  const int64_t* m_off;
  const int64_t* n_off;
  const int32_t* in_ptr;   // by flattened column position (col_ptr order)
  const int32_t* in_idx;
  const int32_t* out_ptr;  // by flattened update row (row_ptr order)
  const int32_t* out_idx;
};

// dot of a dense row segment [j0, j1) with a shared-memory vector: lanes
// over the columns, four independent partial sums (loads in flight)
template <typename T>
__device__ __forceinline__ T cf_dot(const T* __restrict__ row, const T* vec, int j0, int j1, int lane) {
  T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0);
  int j = j0 + lane;
  for (; j + 96 < j1; j += 128) {
    const T r0 = ldg_stream(row + j), r1 = ldg_stream(row + j + 32), r2 = ldg_stream(row + j + 64),
            r3 = ldg_stream(row + j + 96);
    a0 = fma(r0, vec[j], a0);
    a1 = fma(r1, vec[j + 32], a1);
    a2 = fma(r2, vec[j + 64], a2);
    a3 = fma(r3, vec[j + 96], a3);
  }
  for (; j < j1; j += 32) a0 = fma(ldg_stream(row + j), vec[j], a0);
  return warp_sum((a0 + a1) + (a2 + a3));
}

// input u indexed by the solve's own vector index, or through gmap (the
// local solves read the global residual r at gmap[k], rounded once to T)
template <typename T, typename TI>
__global__ void __launch_bounds__(CF_THREADS) k_cf_forward(CoarseFactorDev F, const int2* __restrict__ tasks,
                                                           const T* __restrict__ vals, const TI* __restrict__ u,
                                                           const int32_t* __restrict__ gmap, T* __restrict__ y,
                                                           T* __restrict__ cbuf) {
  extern __shared__ __align__(16) unsigned char cf_sm[];
  T* bt = reinterpret_cast<T*>(cf_sm);
  const int2 tk = tasks[blockIdx.x];
  const int k = tk.x, row0 = tk.y;
  const int s = F.sn_s[k], r = F.sn_r[k];
  const int32_t* cols = F.col_ids + F.col_ptr[k];
  const int32_t cb = F.col_ptr[k];
  for (int i = threadIdx.x; i < s; i += CF_THREADS) {
    const int32_t c = cols[i];
    T acc = (T)u[gmap ? gmap[c] : c];
    for (int32_t p = F.in_ptr[cb + i]; p < F.in_ptr[cb + i + 1]; ++p) acc -= cbuf[F.in_idx[p]];
    bt[i] = acc;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = warp; q < CF_ROWS; q += CF_THREADS / 32) {
    const int row = row0 + q;
    if (row >= s + r) break;
    if (row < s) {
      const T acc = cf_dot(vals + F.d_off[k] + (int64_t)row * s, bt, 0, row, lane);
      if (lane == 0) y[cols[row]] = acc + bt[row];
    } else {
      T acc = cf_dot(vals + F.m_off[k] + (int64_t)(row - s) * s, bt, 0, s, lane);
      if (lane == 0) {
        // extend-add: the children's updates on this row pass through
        const int32_t g = F.row_ptr[k] + row - s;
        for (int32_t p = F.out_ptr[g]; p < F.out_ptr[g + 1]; ++p) acc += cbuf[F.out_idx[p]];
        cbuf[g] = acc;
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(CF_THREADS) k_cf_backward(CoarseFactorDev F, const int2* __restrict__ tasks,
                                                            const T* __restrict__ vals, const T* __restrict__ y,
                                                            T* __restrict__ x) {
  extern __shared__ __align__(16) unsigned char cf_sm[];
  T* in = reinterpret_cast<T*>(cf_sm);
  const int2 tk = tasks[blockIdx.x];
  const int k = tk.x, row0 = tk.y;
  const int s = F.sn_s[k], r = F.sn_r[k];
  const int32_t* cols = F.col_ids + F.col_ptr[k];
  const int32_t* rows = F.row_ids + F.row_ptr[k];
  for (int i = threadIdx.x; i < s + r; i += CF_THREADS) in[i] = i < s ? y[cols[i]] : x[rows[i - s]];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = warp; q < CF_ROWS; q += CF_THREADS / 32) {
    const int row = row0 + q;
    if (row >= s) break;
    const T a = cf_dot(vals + F.d_off[k] + (int64_t)row * s, in, row, s, lane);
    const T b = cf_dot(vals + F.n_off[k] + (int64_t)row * r, in + s, 0, r, lane);
    if (lane == 0) x[cols[row]] = a - b;
  }
}

}  // namespace gdsw
