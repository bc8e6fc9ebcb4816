// Energy-minimizing (harmonic) extension of the coarse basis on the GPU
// (harmonic_extension, coarse_space.py:130-179):
//     A_{I_s I_s} Phi_{I_s} = -A_{I_s Gamma} Phi_Gamma     for every subdomain s
// solved for ONLY the k_s coarse columns that touch s (the reference solves
// all n_c columns densely, coarse_space.py:146, 161-163), as one batched
// Jacobi-preconditioned CG over every (subdomain, column) pair at once.
// Unknowns live in the same column-major interior panels the apply reads.
//
// Chunks of <= 256 interior rows never straddle a subdomain; per-column
// reductions go through per-chunk partials summed in fixed order.
#pragma once
#include "common.cuh"

namespace gdsw {

constexpr int EXT_THREADS = 256;
constexpr int EXT_MAXK = 128;

struct ExtDev {
  int32_t n_chunks;
  int32_t n_sub;
  int64_t n_int_total;
  const int32_t* chunk_sub;    // [n_chunks]
  const int32_t* chunk_row0;   // [n_chunks] first local interior row
  const int32_t* chunk_nrow;   // [n_chunks]
  const int64_t* chunk_poff;   // [n_chunks] offset into per-(chunk, column) partials
  const int32_t* int_ptr;      // [n_sub+1] concatenated interior row offsets
  const int32_t* n_int;        // [n_sub]
  const int32_t* col_ptr;      // [n_sub+1]
  const int32_t* col_ids;      // coarse column ids (sorted per subdomain)
  const int64_t* panel_off;    // [n_sub]
  // A_{II}: CSR over concatenated interior rows, columns = local interior row
  const int64_t* aii_ptr;
  const int32_t* aii_col;
  const double* aii_val;
  const double* dinv;          // 1 / diag(A_II) per interior row
  // A_{I Gamma}: CSR over concatenated interior rows, columns = gamma position
  const int64_t* aig_ptr;
  const int32_t* aig_col;
  const double* aig_val;
  // Phi_Gamma rows (CSR over gamma positions, columns = coarse ids)
  const int64_t* pgam_ptr;
  const int32_t* pgam_col;
  const double* pgam_val;
};

__device__ __forceinline__ int local_col(const int32_t* cols, int k, int32_t c) {
  int lo = 0, hi = k - 1;
  while (lo <= hi) {
    int mid = (lo + hi) >> 1;
    int32_t v = cols[mid];
    if (v == c) return mid;
    if (v < c) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

// rhs = -(A_{I Gamma} Phi_Gamma) restricted to the subdomain's columns,
// accumulated per (row, column) in A-row order with rounded mul/add (the
// reference's csr_matmat_dense order, _kernels.py:34-48), then negated.
__global__ void k_ext_rhs(ExtDev E, double* __restrict__ B) {
  const int32_t ch = blockIdx.x;
  const int32_t s = E.chunk_sub[ch];
  if (threadIdx.x >= E.chunk_nrow[ch]) return;
  const int32_t row = E.chunk_row0[ch] + threadIdx.x;
  const int32_t t = E.int_ptr[s] + row;
  const int32_t ni = E.n_int[s];
  const int k = E.col_ptr[s + 1] - E.col_ptr[s];
  const int32_t* cols = E.col_ids + E.col_ptr[s];
  double* b = B + E.panel_off[s] + row;
  for (int c = 0; c < k; ++c) b[(int64_t)c * ni] = 0.0;
  for (int64_t p = E.aig_ptr[t]; p < E.aig_ptr[t + 1]; ++p) {
    const int32_t g = E.aig_col[p];
    const double a = E.aig_val[p];
    for (int64_t q = E.pgam_ptr[g]; q < E.pgam_ptr[g + 1]; ++q) {
      int c = local_col(cols, k, E.pgam_col[q]);
      if (c >= 0) b[(int64_t)c * ni] = rn_add(b[(int64_t)c * ni], rn_mul(a, E.pgam_val[q]));
    }
  }
  for (int c = 0; c < k; ++c) b[(int64_t)c * ni] = -b[(int64_t)c * ni];
}

// block reduce of one value per column into partial[poff + c]
__device__ __forceinline__ void chunk_col_reduce(double v, int c, double (*red)[EXT_MAXK]) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][c] = v;
}

__device__ __forceinline__ void chunk_col_flush(int k, const double (*red)[EXT_MAXK],
                                                double* __restrict__ out) {
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < EXT_THREADS / 32; ++w) s += red[w][c];
    out[c] = s;
  }
}

// Y = A_II X ; optional partial dots (X . Y) per column
__global__ void __launch_bounds__(EXT_THREADS) k_ext_spmm(ExtDev E, const double* __restrict__ X,
                                                          double* __restrict__ Y,
                                                          double* __restrict__ partial) {
  __shared__ double red[EXT_THREADS / 32][EXT_MAXK];
  const int32_t ch = blockIdx.x;
  const int32_t s = E.chunk_sub[ch];
  const int32_t ni = E.n_int[s];
  const int k = E.col_ptr[s + 1] - E.col_ptr[s];
  const bool on = threadIdx.x < E.chunk_nrow[ch];
  const int32_t row = E.chunk_row0[ch] + threadIdx.x;
  const int32_t t = E.int_ptr[s] + (on ? row : 0);
  const int64_t off = E.panel_off[s];
  const int64_t p0 = on ? E.aii_ptr[t] : 0, p1 = on ? E.aii_ptr[t + 1] : 0;
  for (int c = 0; c < k; ++c) {
    double acc = 0.0, dot = 0.0;
    if (on) {
      const double* xc = X + off + (int64_t)c * ni;
      for (int64_t p = p0; p < p1; ++p) acc = fma(E.aii_val[p], xc[E.aii_col[p]], acc);
      Y[off + (int64_t)c * ni + row] = acc;
      dot = xc[row] * acc;
    }
    if (partial) chunk_col_reduce(dot, c, red);
  }
  if (partial) chunk_col_flush(k, red, partial + E.chunk_poff[ch]);
}

// per-column finalisation of a partial sum: out[col] = sum over the
// subdomain's chunks (ascending)
__global__ void k_ext_colsum(ExtDev E, const int32_t* __restrict__ colsub,
                             const int32_t* __restrict__ sub_chunk0,
                             const double* __restrict__ partial, double* __restrict__ out,
                             int K) {
  int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= K) return;
  int s = colsub[col];
  int c = col - E.col_ptr[s];
  double acc = 0.0;
  for (int ch = sub_chunk0[s]; ch < sub_chunk0[s + 1]; ++ch) acc += partial[E.chunk_poff[ch] + c];
  out[col] = acc;
}

// X += alpha P ; R -= alpha AP ; Z = Dinv R ; partial (R.Z, R.R)
__global__ void __launch_bounds__(EXT_THREADS) k_ext_update(ExtDev E, const double* __restrict__ alpha,
                                                            double* __restrict__ X,
                                                            double* __restrict__ R,
                                                            double* __restrict__ Z,
                                                            const double* __restrict__ P,
                                                            const double* __restrict__ AP,
                                                            double* __restrict__ part_rz,
                                                            double* __restrict__ part_rr) {
  __shared__ double red[EXT_THREADS / 32][EXT_MAXK];
  __shared__ double red2[EXT_THREADS / 32][EXT_MAXK];
  const int32_t ch = blockIdx.x;
  const int32_t s = E.chunk_sub[ch];
  const int32_t ni = E.n_int[s];
  const int k = E.col_ptr[s + 1] - E.col_ptr[s];
  const bool on = threadIdx.x < E.chunk_nrow[ch];
  const int32_t row = E.chunk_row0[ch] + threadIdx.x;
  const double di = on ? E.dinv[E.int_ptr[s] + row] : 0.0;
  const int64_t off = E.panel_off[s];
  for (int c = 0; c < k; ++c) {
    double rz = 0.0, rr = 0.0;
    if (on) {
      const int64_t q = off + (int64_t)c * ni + row;
      const double a = alpha ? alpha[E.col_ptr[s] + c] : 0.0;
      X[q] = fma(a, P[q], X[q]);
      const double r = fma(-a, AP[q], R[q]);
      R[q] = r;
      const double z = di * r;
      Z[q] = z;
      rz = r * z;
      rr = r * r;
    }
    chunk_col_reduce(rz, c, red);
    chunk_col_reduce(rr, c, red2);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < EXT_THREADS / 32; ++w) { a += red[w][c]; b += red2[w][c]; }
    part_rz[E.chunk_poff[ch] + c] = a;
    part_rr[E.chunk_poff[ch] + c] = b;
  }
}

// P = Z + beta P
__global__ void k_ext_pupdate(ExtDev E, const double* __restrict__ beta,
                              const double* __restrict__ Z, double* __restrict__ P) {
  const int32_t ch = blockIdx.x;
  const int32_t s = E.chunk_sub[ch];
  if (threadIdx.x >= E.chunk_nrow[ch]) return;
  const int32_t ni = E.n_int[s];
  const int k = E.col_ptr[s + 1] - E.col_ptr[s];
  const int32_t row = E.chunk_row0[ch] + threadIdx.x;
  const int64_t off = E.panel_off[s];
  for (int c = 0; c < k; ++c) {
    const int64_t q = off + (int64_t)c * ni + row;
    P[q] = fma(beta[E.col_ptr[s] + c], P[q], Z[q]);
  }
}

// per-column CG scalars: alpha = rz / pAp (0 once converged)
__global__ void k_ext_alpha(int K, const double* __restrict__ rz, const double* __restrict__ pap,
                            const int* __restrict__ active, double* __restrict__ alpha) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= K) return;
  alpha[c] = (active[c] && pap[c] != 0.0) ? rz[c] / pap[c] : 0.0;
}

__global__ void k_ext_beta(int K, double tol2, const double* __restrict__ bb,
                           double* __restrict__ rz, const double* __restrict__ rz_new,
                           const double* __restrict__ rr_new, int* __restrict__ active,
                           double* __restrict__ beta, int* __restrict__ n_active) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= K) return;
  int act = active[c] && rr_new[c] > tol2 * bb[c];
  beta[c] = (act && rz[c] != 0.0) ? rz_new[c] / rz[c] : 0.0;
  rz[c] = rz_new[c];
  active[c] = act;
  if (act) atomicAdd(n_active, 1);
}

// max |A_II X - B| per (chunk, column)  (_check_extension_residual,
// coarse_space.py:182-202)
__global__ void __launch_bounds__(EXT_THREADS) k_ext_resid_max(ExtDev E, const double* __restrict__ X,
                                                               const double* __restrict__ B,
                                                               double* __restrict__ partial) {
  __shared__ double red[EXT_THREADS / 32][EXT_MAXK];
  const int32_t ch = blockIdx.x;
  const int32_t s = E.chunk_sub[ch];
  const int32_t ni = E.n_int[s];
  const int k = E.col_ptr[s + 1] - E.col_ptr[s];
  const bool on = threadIdx.x < E.chunk_nrow[ch];
  const int32_t row = E.chunk_row0[ch] + threadIdx.x;
  const int32_t t = E.int_ptr[s] + (on ? row : 0);
  const int64_t off = E.panel_off[s];
  for (int c = 0; c < k; ++c) {
    double m = 0.0;
    if (on) {
      const double* xc = X + off + (int64_t)c * ni;
      double acc = 0.0;
      for (int64_t p = E.aii_ptr[t]; p < E.aii_ptr[t + 1]; ++p)
        acc = fma(E.aii_val[p], xc[E.aii_col[p]], acc);
      m = fabs(acc - B[off + (int64_t)c * ni + row]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][c] = m;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    double mm = 0.0;
    for (int w = 0; w < EXT_THREADS / 32; ++w) mm = fmax(mm, red[w][c]);
    partial[E.chunk_poff[ch] + c] = mm;
  }
}

__global__ void k_gather_vals(int64_t n, const int64_t* __restrict__ src, const double* __restrict__ a,
                              double* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[src[i]];
}

__global__ void k_make_dinv(int64_t n, const int64_t* __restrict__ diag_pos,
                            const double* __restrict__ val, double* __restrict__ dinv) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    double d = val[diag_pos[i]];
    dinv[i] = d != 0.0 ? 1.0 / d : 1.0;
  }
}

__global__ void k_init_active(int K, const double* __restrict__ bb, int* __restrict__ active) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < K) active[c] = bb[c] > 0.0;
}

__global__ void k_ext_colmax(ExtDev E, const int32_t* __restrict__ colsub,
                             const int32_t* __restrict__ sub_chunk0,
                             const double* __restrict__ partial, double* __restrict__ out, int K) {
  int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= K) return;
  int s = colsub[col];
  int c = col - E.col_ptr[s];
  double m = 0.0;
  for (int ch = sub_chunk0[s]; ch < sub_chunk0[s + 1]; ++ch) m = fmax(m, partial[E.chunk_poff[ch] + c]);
  out[col] = m;
}

__global__ void k_cast_f64_f32(int64_t n, const double* __restrict__ a, float* __restrict__ b) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (float)a[i];
}

}  // namespace gdsw
