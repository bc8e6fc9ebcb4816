// Numeric exact LU / ILU(k) of every subdomain block on the GPU, bit-exact
// with the reference's IKJ kernel (lu_numeric, _kernels.py:429-466;
// local_solvers.py:306-340; host restatement gdsw_host.cpp lu_numeric).
//
// One CTA per subdomain walks the L level schedule (row i needs the U rows
// k in L(i), all in earlier levels); each warp factors one row of a level
// (levels of at most LU_COOP_ROWS rows -- separator chains -- use the whole
// CTA per row, the j updates of each k over all threads):
//   w[pattern(i)] = 0; w[j] = a_ij (+ shift on the diagonal) for j in A(i)
//   for k in L(i) ascending:  l = w[k] / u_kk;  w[k] = l;
//                             w[j] -= l * u_kj  for j in U(k) \ {k}, j in pattern(i)
// The k loop is sequential (as in the reference); the j updates of one k
// are independent (distinct j) and spread over the lanes, so every w[j]
// receives its subtractions in the reference's order with the same
// round-to-nearest operations. w and the pattern stamp are dense per warp
// (global scratch, L1-resident while the warp works on its row).
#pragma once
#include "common.cuh"

namespace gdsw {

constexpr int LU_WARPS = 8;
constexpr int LU_THREADS = 32 * LU_WARPS;
constexpr int LU_COOP_ROWS = 2;  // levels this small factor each row with the whole CTA

struct LuDev {
  const int32_t* sub_ptr;    // [n_sub + 1] block row ranges (concatenated)
  const int64_t* l_ptr;      // concatenated factor patterns, block-local columns
  const int32_t* l_idx;
  const int64_t* u_ptr;
  const int32_t* u_idx;
  const int32_t* lev_sub;    // [n_sub + 1] L level range of each block
  const int32_t* lev_ptr;    // [levels + 1] into lev_rows (concatenated positions)
  const int32_t* lev_rows;   // block-local rows
  const int64_t* ab_ptr;     // [n_loc + 1] permuted block pattern of A
  const int32_t* ab_idx;     // block-local columns
  const int64_t* ab_src;     // A.values position of each entry
  int32_t n_max;             // largest block
};

// ||P A_s P^T||_inf per block, rows summed in the permuted CSR order in
// float64 (_norm_inf, local_solvers.py; np.add.at over |values| as f64)
template <typename T>
__global__ void k_block_norm_inf(LuDev D, const double* __restrict__ aval, double* __restrict__ norm) {
  const int s = blockIdx.x;
  __shared__ double red[LU_THREADS];
  double mx = 0.0;
  for (int32_t r = D.sub_ptr[s] + threadIdx.x; r < D.sub_ptr[s + 1]; r += LU_THREADS) {
    double acc = 0.0;
    for (int64_t p = D.ab_ptr[r]; p < D.ab_ptr[r + 1]; ++p) acc += fabs((double)(T)aval[D.ab_src[p]]);
    mx = fmax(mx, acc);
  }
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int o = LU_THREADS / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) norm[s] = red[0];
}

template <typename T>
__global__ void __launch_bounds__(LU_THREADS) k_lu_numeric(LuDev D, const double* __restrict__ aval,
                                                          T shift, const double* __restrict__ norm,
                                                          T* __restrict__ lval, T* __restrict__ uval,
                                                          T* __restrict__ wbuf, int32_t* __restrict__ stamp_buf,
                                                          int64_t* __restrict__ fail) {
  const int s = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t base = D.sub_ptr[s];
  T* w = wbuf + ((size_t)s * LU_WARPS + warp) * D.n_max;
  int32_t* stamp = stamp_buf + ((size_t)s * LU_WARPS + warp) * D.n_max;
  const double tol = 1e-14 * norm[s];
  for (int32_t lv = D.lev_sub[s]; lv < D.lev_sub[s + 1]; ++lv) {
    const int32_t r0 = D.lev_ptr[lv], r1 = D.lev_ptr[lv + 1];
    if (r1 - r0 <= LU_COOP_ROWS) {
      // few rows in this level (nested-dissection separators: one row per
      // level): the whole CTA factors each row, the j updates of every k
      // spread over all threads, one barrier per k (the k order and every
      // w[j]'s subtraction order stay the reference's)
      T* wc = wbuf + (size_t)s * LU_WARPS * D.n_max;
      int32_t* sc = stamp_buf + (size_t)s * LU_WARPS * D.n_max;
      for (int32_t t = r0; t < r1; ++t) {
        const int32_t i = D.lev_rows[t];
        const int32_t g = base + i;
        const int64_t l0 = D.l_ptr[g], l1 = D.l_ptr[g + 1], u0 = D.u_ptr[g], u1 = D.u_ptr[g + 1];
        for (int64_t p = l0 + threadIdx.x; p < l1; p += LU_THREADS) {
          sc[D.l_idx[p]] = i;
          wc[D.l_idx[p]] = T(0);
        }
        for (int64_t p = u0 + threadIdx.x; p < u1; p += LU_THREADS) {
          sc[D.u_idx[p]] = i;
          wc[D.u_idx[p]] = T(0);
        }
        __syncthreads();
        for (int64_t p = D.ab_ptr[g] + threadIdx.x; p < D.ab_ptr[g + 1]; p += LU_THREADS) {
          const int32_t j = D.ab_idx[p];
          if (sc[j] == i) {
            T v = (T)aval[D.ab_src[p]];
            if (j == i && shift != T(0)) v = v + shift;
            wc[j] = v;
          }
        }
        __syncthreads();
        for (int64_t p = l0; p < l1; ++p) {
          const int32_t k = D.l_idx[p];
          const int64_t k0 = D.u_ptr[base + k], k1 = D.u_ptr[base + k + 1];
          // w[k] is final (its last update came from an earlier k, before
          // the barrier) and never updated again: l_ik goes straight to L
          const T lik = rn_div(wc[k], uval[k0]);
          if (threadIdx.x == 0) lval[p] = lik;
          for (int64_t q = k0 + 1 + threadIdx.x; q < k1; q += LU_THREADS) {
            const int32_t j = D.u_idx[q];
            if (sc[j] == i) wc[j] = rn_sub(wc[j], rn_mul(lik, uval[q]));
          }
          __syncthreads();
        }
        if (threadIdx.x == 0 && (double)fabs(wc[i]) <= tol)
          atomicMin((unsigned long long*)(fail + s), (unsigned long long)(i + 1));
        for (int64_t p = u0 + threadIdx.x; p < u1; p += LU_THREADS) uval[p] = wc[D.u_idx[p]];
        __syncthreads();
      }
      continue;
    }
    for (int32_t t = r0 + warp; t < r1; t += LU_WARPS) {
      const int32_t i = D.lev_rows[t];
      const int32_t g = base + i;
      const int64_t l0 = D.l_ptr[g], l1 = D.l_ptr[g + 1], u0 = D.u_ptr[g], u1 = D.u_ptr[g + 1];
      for (int64_t p = l0 + lane; p < l1; p += 32) {
        stamp[D.l_idx[p]] = i;
        w[D.l_idx[p]] = T(0);
      }
      for (int64_t p = u0 + lane; p < u1; p += 32) {
        stamp[D.u_idx[p]] = i;
        w[D.u_idx[p]] = T(0);
      }
      __syncwarp();
      for (int64_t p = D.ab_ptr[g] + lane; p < D.ab_ptr[g + 1]; p += 32) {
        const int32_t j = D.ab_idx[p];
        if (stamp[j] == i) {
          T v = (T)aval[D.ab_src[p]];
          if (j == i && shift != T(0)) v = v + shift;
          w[j] = v;
        }
      }
      __syncwarp();
      // k loop: the U row of k+1 (pointers, pivot, first 64 entries) is
      // loaded while k's updates run -- rows k are final, so the prefetch
      // never depends on this row's arithmetic
      int64_t nk0 = 0, nk1 = 0;
      T ndg = T(0), nu[2];
      int32_t nj[2] = {-1, -1};
      auto fetch = [&](int64_t p) {
        if (p >= l1) return;
        const int32_t gk = base + D.l_idx[p];
        nk0 = D.u_ptr[gk];
        nk1 = D.u_ptr[gk + 1];
        ndg = uval[nk0];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int64_t q = nk0 + 1 + lane + 32 * u;
          nj[u] = q < nk1 ? D.u_idx[q] : -1;
          nu[u] = q < nk1 ? uval[q] : T(0);
        }
      };
      fetch(l0);
      for (int64_t p = l0; p < l1; ++p) {
        const int32_t k = D.l_idx[p];
        const int64_t k0 = nk0, k1 = nk1;
        const T dg = ndg;
        const int32_t j0 = nj[0], j1 = nj[1];
        const T v0 = nu[0], v1 = nu[1];
        fetch(p + 1);
        const T lik = rn_div(w[k], dg);
        __syncwarp();
        if (lane == 0) w[k] = lik;
        if (j0 >= 0 && stamp[j0] == i) w[j0] = rn_sub(w[j0], rn_mul(lik, v0));
        if (j1 >= 0 && stamp[j1] == i) w[j1] = rn_sub(w[j1], rn_mul(lik, v1));
#pragma unroll 4
        for (int64_t q = k0 + 65 + lane; q < k1; q += 32) {
          const int32_t j = D.u_idx[q];
          if (stamp[j] == i) w[j] = rn_sub(w[j], rn_mul(lik, uval[q]));
        }
        __syncwarp();
      }
      if (lane == 0 && (double)fabs(w[i]) <= tol) atomicMin((unsigned long long*)(fail + s),
                                                           (unsigned long long)(i + 1));
      for (int64_t p = l0 + lane; p < l1; p += 32) lval[p] = w[D.l_idx[p]];
      for (int64_t p = u0 + lane; p < u1; p += 32) uval[p] = w[D.u_idx[p]];
      __syncwarp();
    }
    __syncthreads();  // rows of this level are final before the next level reads them
  }
}

}  // namespace gdsw
