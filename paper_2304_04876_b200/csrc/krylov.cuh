// GMRES vector kernels (krylov.py:260-361 single-reduce, 179-257 classic).
//
// * k_block_dot: the ONE fused reduction per single-reduce iteration,
//   [V[:j]; v]^T [v, z] (krylov.py:290-300). Each thread streams its
//   elements once, multiplying every basis row against both v and z, so the
//   block costs one pass over j+2 vectors. Deterministic two-stage reduction
//   (fixed grid, fixed tree, fixed-order second stage): bitwise
//   reproducible run to run.
// * k_sr_update: v[j], zm[j] and the speculative next candidate w in one
//   pass (krylov.py:346-351); V[:j] is read once for both a and p/delta.
#pragma once
#include "common.cuh"

namespace gdsw {

constexpr int KDOT_ROWS = 16;       // basis rows per block-dot launch
constexpr int KDOT_THREADS = 256;

// rows: V[r0 .. r0+nr) (stride ldv) then, if self, the vector v itself.
// partial[blk][2*(KDOT_ROWS+1)]: [row]*2 + {0: .v, 1: .z}
__global__ void __launch_bounds__(KDOT_THREADS) k_block_dot(int64_t n, const double* __restrict__ V,
                                                            int64_t ldv, int nr, int self,
                                                            const double* __restrict__ v,
                                                            const double* __restrict__ z,
                                                            double* __restrict__ partial,
                                                            double* __restrict__ out,
                                                            unsigned* __restrict__ counter) {
  double av[KDOT_ROWS + 1], az[KDOT_ROWS + 1];
#pragma unroll
  for (int r = 0; r <= KDOT_ROWS; ++r) av[r] = az[r] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double vi = ldg_stream(v + i);
    const double zi = z ? ldg_stream(z + i) : 0.0;
#pragma unroll
    for (int r = 0; r < KDOT_ROWS; ++r) {
      if (r < nr) {
        const double b = ldg_stream(V + r * ldv + i);
        av[r] = fma(b, vi, av[r]);
        az[r] = fma(b, zi, az[r]);
      }
    }
    if (self) {
      av[KDOT_ROWS] = fma(vi, vi, av[KDOT_ROWS]);
      az[KDOT_ROWS] = fma(vi, zi, az[KDOT_ROWS]);
    }
  }
  __shared__ double red[KDOT_THREADS / 32][2 * (KDOT_ROWS + 1)];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r <= KDOT_ROWS; ++r) {
    double a = warp_sum(av[r]);
    double c = warp_sum(az[r]);
    if (lane == 0) {
      red[warp][2 * r] = a;
      red[warp][2 * r + 1] = c;
    }
  }
  __syncthreads();
  constexpr int W2 = 2 * (KDOT_ROWS + 1);
  for (int k = threadIdx.x; k < W2; k += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < KDOT_THREADS / 32; ++w) s += red[w][k];
    partial[(int64_t)blockIdx.x * W2 + k] = s;
  }
  // last block to finish reduces all block partials in a fixed order (one
  // warp per value, lanes strided over blocks, fixed shuffle tree): the
  // second stage costs no extra launch and stays deterministic
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int k = warp; k < W2; k += KDOT_THREADS / 32) {
    double s = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) s += __ldcg(partial + (int64_t)b * W2 + k);
    s = warp_sum(s);
    if (lane == 0) out[k] = s;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// out[k] = sum over blocks (ascending) of partial[blk][k]
__global__ void k_reduce_partials(int nblk, int width, const double* __restrict__ partial,
                                  double* __restrict__ out) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= width) return;
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += partial[(int64_t)b * width + k];
  out[k] = s;
}

// single-reduce update (krylov.py:346-351). coef = [a(0..j), pd(0..j)],
// pd = p / delta.
__global__ void __launch_bounds__(256) k_sr_update(int64_t n, double* __restrict__ V,
                                                   double* __restrict__ Zm, int64_t ld, int j,
                                                   const double* __restrict__ coef, double delta,
                                                   double corr, double* __restrict__ W,
                                                   const double* __restrict__ Mc,
                                                   const double* __restrict__ Zc) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double va = 0.0, wp = 0.0, za = 0.0;
    for (int r = 0; r < j; ++r) {
      const double vr = ldg_stream(V + r * ld + i);
      const double zr = ldg_stream(Zm + r * ld + i);
      const double a = __ldg(coef + r), pd = __ldg(coef + j + r);
      va = fma(a, vr, va);
      wp = fma(pd, vr, wp);
      za = fma(a, zr, za);
    }
    const double vj = (W[i] - va) / delta;
    const double zj = (Mc[i] - za) / delta;
    V[(int64_t)j * ld + i] = vj;
    Zm[(int64_t)j * ld + i] = zj;
    W[i] = Zc[i] / delta - wp - corr * vj;
  }
}

// x_out = x + sum_r y[r] Zm[r]   (krylov.py:340, 361)
__global__ void __launch_bounds__(256) k_x_update(int64_t n, const double* __restrict__ x,
                                                  const double* __restrict__ Zm, int64_t ld, int m,
                                                  const double* __restrict__ y,
                                                  double* __restrict__ xo) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double acc = 0.0;
    for (int r = 0; r < m; ++r) acc = fma(__ldg(y + r), ldg_stream(Zm + r * ld + i), acc);
    xo[i] = x[i] + acc;
  }
}

// classic Arnoldi helpers (krylov.py:217-236): w -= sum_r h[r] v[r]; and
// v_out = w / nrm
__global__ void __launch_bounds__(256) k_multi_axpy(int64_t n, const double* __restrict__ V,
                                                    int64_t ld, int m,
                                                    const double* __restrict__ h,
                                                    double* __restrict__ w) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double acc = 0.0;
    for (int r = 0; r < m; ++r) acc = fma(__ldg(h + r), ldg_stream(V + r * ld + i), acc);
    w[i] -= acc;
  }
}

__global__ void k_axpy_scalar(int64_t n, double alpha, const double* __restrict__ x,
                              double* __restrict__ y) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] -= alpha * x[i];
}

__global__ void k_scale_copy(int64_t n, const double* __restrict__ x, double s,
                             double* __restrict__ y) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = x[i] / s;
}

}  // namespace gdsw
