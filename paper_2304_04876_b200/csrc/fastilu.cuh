// Batched FastILU numeric setup (fast_ilu_numeric, local_solvers.py:343-397;
// fastilu_sweep / fastilu_residual, _kernels.py:547-617).
//
// One thread per factor entry, all subdomains in one launch. The bounded
// sparse dot sum_{k<bound} L(i,k) U(k,j) is precomputed on the host as a
// flat list of (L position, U position) pairs in the reference's merge order
// (ascending k), so each thread performs exactly the reference's sequence of
// rounded multiply/adds: the factors are bit-identical to the sequential
// Jacobi sweeps.
#pragma once
#include "common.cuh"

namespace gdsw {

struct FastIluDev {
  int64_t nnz_l, nnz_u;
  const int64_t* a_of;      // [nnz_l + nnz_u] index into A.values or -1
  const int64_t* e_ptr;     // [nnz_l + nnz_u + 1] pair ranges
  const int32_t* pair_l;    // absolute L positions
  const int32_t* pair_u;    // absolute U positions
  const int32_t* ldiag;     // [nnz_l] U position of the diagonal of column j
};

// initial guess: U = upper(A) (fill 0), L = strict-lower(A) / diag(U)
template <typename T>
__global__ void k_fastilu_init_u(FastIluDev F, const double* __restrict__ a, T* __restrict__ u) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= F.nnz_u) return;
  int64_t s = F.a_of[F.nnz_l + p];
  u[p] = s >= 0 ? (T)a[s] : T(0);
}

template <typename T>
__global__ void k_fastilu_init_l(FastIluDev F, const double* __restrict__ a,
                                 const T* __restrict__ u, T* __restrict__ l) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= F.nnz_l) return;
  int64_t s = F.a_of[p];
  T v = s >= 0 ? (T)a[s] : T(0);
  l[p] = rn_div(v, u[F.ldiag[p]]);
}

// one synchronous sweep: reads only the previous iterate (double buffered)
template <typename T>
__global__ void __launch_bounds__(256) k_fastilu_sweep(FastIluDev F, const double* __restrict__ a,
                                                       const T* __restrict__ l_old,
                                                       const T* __restrict__ u_old,
                                                       T* __restrict__ l_new, T* __restrict__ u_new,
                                                       int* __restrict__ zero_div) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= F.nnz_l + F.nnz_u) return;
  const int64_t src = F.a_of[e];
  const T aij = src >= 0 ? (T)a[src] : T(0);
  T s = T(0);
  for (int64_t q = F.e_ptr[e]; q < F.e_ptr[e + 1]; ++q)
    s = rn_add(s, rn_mul(l_old[F.pair_l[q]], u_old[F.pair_u[q]]));
  if (e < F.nnz_l) {
    const T d = u_old[F.ldiag[e]];
    if (d == T(0)) *zero_div = 1;  // the reference raises ZeroDivisionError here
    l_new[e] = rn_div(rn_sub(aij, s), d);
  } else {
    u_new[e - F.nnz_l] = rn_sub(aij, s);
  }
}

struct FastIluResDev {
  int64_t n_terms;
  const int64_t* a_src;     // A.values index of the block entry
  const int64_t* r_ptr;
  const int32_t* r_l;
  const int32_t* r_u;
  const int32_t* tail_l;    // -1 when the tail is a plain U entry
  const int32_t* tail_u;
};

// per block-A entry |A_ij - (LU)_ij| (the nonlinear residual terms)
template <typename T>
__global__ void k_fastilu_residual_terms(FastIluResDev R, const double* __restrict__ a,
                                         const T* __restrict__ l, const T* __restrict__ u,
                                         double* __restrict__ terms) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= R.n_terms) return;
  T s = T(0);
  for (int64_t q = R.r_ptr[e]; q < R.r_ptr[e + 1]; ++q)
    s = rn_add(s, rn_mul(l[R.r_l[q]], u[R.r_u[q]]));
  const int32_t tl = R.tail_l[e];
  s = tl >= 0 ? rn_add(s, rn_mul(l[tl], u[R.tail_u[e]])) : rn_add(s, u[R.tail_u[e]]);
  T d = rn_sub((T)a[R.a_src[e]], s);
  terms[e] = (double)(d < T(0) ? -d : d);
}

// one CTA per segment: out[seg] = sum(terms[seg_ptr[seg] .. seg_ptr[seg+1]])
__global__ void k_segment_sum(const int64_t* __restrict__ seg_ptr, const double* __restrict__ terms,
                              double* __restrict__ out) {
  const int seg = blockIdx.x;
  double acc = 0.0;
  for (int64_t i = seg_ptr[seg] + threadIdx.x; i < seg_ptr[seg + 1]; i += blockDim.x) acc += terms[i];
  __shared__ double red[32];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) out[seg] = t;
  }
}

template <typename T>
__global__ void k_count_nonfinite(int64_t n, const T* __restrict__ x, int* __restrict__ flag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && !isfinite((double)x[i])) *flag = 1;
}

}  // namespace gdsw
