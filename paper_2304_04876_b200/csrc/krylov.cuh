// GMRES vector kernels (krylov.py:260-361 single-reduce, 179-257 classic).
//
// * k_block_dot: the ONE fused reduction per single-reduce iteration,
//   [V[:j]; v]^T [v, z] (krylov.py:290-300). A CTA stages a 1024-element
//   tile of v and z in shared memory once; its warps then stream the basis
//   rows of that tile with 16-byte loads (each row read exactly once per
//   solve pass) against the staged tile. Few rows (norms, MGS dots): several
//   warps split each row's tile. Deterministic: fixed grid, fixed tile
//   assignment, fixed shuffle trees, and the last CTA to finish reduces the
//   per-CTA partials in a fixed order (no second launch).
// * k_sr_update: v[j], zm[j] and the speculative next candidate w in one
//   pass (krylov.py:346-351); V[:j] is read once for both a and p/delta.
#pragma once
#include "common.cuh"

namespace gdsw {

constexpr int KDOT_ROWS = 32;  // rows per block-dot launch (basis rows + self)
constexpr int KDOT_THREADS = 256;
constexpr int KDOT_TILE = 1024;
constexpr int KDOT_W2 = 2 * KDOT_ROWS;

// rows of the combined list [V[0..nv), v] restricted to [r0, r0 + nrc).
// out[2*rr + {0,1}] = row . v, row . z  (rr = local row index)
__global__ void __launch_bounds__(KDOT_THREADS, 3) k_block_dot(
    int64_t n, const double* __restrict__ V, int64_t ldv, int nv, int r0, int nrc,
    const double* __restrict__ v, const double* __restrict__ z, double* __restrict__ partial,
    double* __restrict__ out, unsigned* __restrict__ counter) {
  __shared__ double red[KDOT_THREADS / 32][4][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NW = KDOT_THREADS / 32;
  constexpr int KT = 256;      // elements per warp tile: 4 x 16-byte loads per lane
  // S warps per row when rows are few (each on its own tiles), else up to 4
  // rows per warp (all warps of the CTA on the same tile, v/z hit L1)
  const int S = nrc >= 5 ? 1 : (nrc >= 3 ? 2 : (nrc == 2 ? 4 : 8));
  const int slice = warp % S;
  const double* rows[4];
  int nq = 0;
  if (S > 1) {
    int rr = warp / S;
    if (rr < nrc) {
      int g = r0 + rr;
      rows[nq++] = g < nv ? V + (int64_t)g * ldv : v;
    }
  } else {
    for (int rr = warp; rr < nrc && nq < 4; rr += NW) {
      int g = r0 + rr;
      rows[nq++] = g < nv ? V + (int64_t)g * ldv : v;
    }
  }
  double av[4] = {0, 0, 0, 0}, az[4] = {0, 0, 0, 0};
  const int64_t ntiles = (n + KT - 1) / KT;
  const bool vec = ((ldv & 1) == 0) && ((reinterpret_cast<uintptr_t>(V) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(v) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(z) & 15) == 0);
  for (int64_t t0 = (int64_t)blockIdx.x * S; t0 < ntiles; t0 += (int64_t)gridDim.x * S) {
    const int64_t tile = t0 + slice;
    if (tile >= ntiles || nq == 0) continue;
    const int64_t base = tile * KT;
    const int cnt = (int)(n - base < KT ? n - base : KT);
    if (vec && cnt == KT) {
      double2 pv[4], pz[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int64_t e = base + 64 * t + 2 * lane;
        pv[t] = __ldg(reinterpret_cast<const double2*>(v + e));
        pz[t] = z ? __ldg(reinterpret_cast<const double2*>(z + e)) : make_double2(0.0, 0.0);
      }
      for (int q = 0; q < nq; ++q) {
        double2 x[4];
#pragma unroll
        for (int t = 0; t < 4; ++t)
          x[t] = ldg_stream(reinterpret_cast<const double2*>(rows[q] + base + 64 * t + 2 * lane));
        double a = 0.0, c = 0.0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          a = fma(x[t].x, pv[t].x, a);
          a = fma(x[t].y, pv[t].y, a);
          c = fma(x[t].x, pz[t].x, c);
          c = fma(x[t].y, pz[t].y, c);
        }
        av[q] += a;
        az[q] += c;
      }
    } else {
      for (int q = 0; q < nq; ++q) {
        double a = 0.0, c = 0.0;
        for (int e = lane; e < cnt; e += 32) {
          const double x = rows[q][base + e];
          a = fma(x, v[base + e], a);
          if (z) c = fma(x, z[base + e], c);
        }
        av[q] += a;
        az[q] += c;
      }
    }
  }
  for (int q = 0; q < 4; ++q) {
    double a = warp_sum(av[q]);
    double c = warp_sum(az[q]);
    if (lane == 0) {
      red[warp][q][0] = a;
      red[warp][q][1] = c;
    }
  }
  __syncthreads();
  for (int rr = threadIdx.x; rr < nrc; rr += KDOT_THREADS) {
    double a = 0.0, c = 0.0;
    if (S > 1) {
      for (int w = rr * S; w < rr * S + S; ++w) {
        a += red[w][0][0];
        c += red[w][0][1];
      }
    } else {
      a = red[rr % NW][rr / NW][0];
      c = red[rr % NW][rr / NW][1];
    }
    partial[(int64_t)blockIdx.x * KDOT_W2 + 2 * rr] = a;
    partial[(int64_t)blockIdx.x * KDOT_W2 + 2 * rr + 1] = c;
  }
  // the last CTA reduces all per-CTA partials in a fixed order
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int k = warp; k < 2 * nrc; k += NW) {
    double s = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) s += __ldcg(partial + (int64_t)b * KDOT_W2 + k);
    s = warp_sum(s);
    if (lane == 0) out[k] = s;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// single-reduce update (krylov.py:346-351). coef = [a(0..j), p/delta(0..j),
// delta, corr]. VW = 2: 16-byte vector path (rows of even ld, aligned).
template <int VW>
__global__ void __launch_bounds__(256) k_sr_update(int64_t n, double* __restrict__ V,
                                                   double* __restrict__ Zm, int64_t ld, int j,
                                                   const double* __restrict__ coef,
                                                   double* __restrict__ W,
                                                   const double* __restrict__ Mc,
                                                   const double* __restrict__ Zc) {
  const double delta = coef[2 * j], corr = coef[2 * j + 1];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * VW;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * VW; i < n; i += stride) {
    if (VW == 2 && i + 1 < n) {
      double2 va = {0, 0}, wp = {0, 0}, za = {0, 0};
#pragma unroll 4
      for (int r = 0; r < j; ++r) {
        const double2 vr = ldg_stream(reinterpret_cast<const double2*>(V + r * ld + i));
        const double2 zr = ldg_stream(reinterpret_cast<const double2*>(Zm + r * ld + i));
        const double a = __ldg(coef + r), pd = __ldg(coef + j + r);
        va.x = fma(a, vr.x, va.x);
        va.y = fma(a, vr.y, va.y);
        wp.x = fma(pd, vr.x, wp.x);
        wp.y = fma(pd, vr.y, wp.y);
        za.x = fma(a, zr.x, za.x);
        za.y = fma(a, zr.y, za.y);
      }
      const double2 w = *reinterpret_cast<const double2*>(W + i);
      const double2 mc = ldg_stream(reinterpret_cast<const double2*>(Mc + i));
      const double2 zc = ldg_stream(reinterpret_cast<const double2*>(Zc + i));
      double2 vj, zj, wn;
      vj.x = (w.x - va.x) / delta;
      vj.y = (w.y - va.y) / delta;
      zj.x = (mc.x - za.x) / delta;
      zj.y = (mc.y - za.y) / delta;
      wn.x = zc.x / delta - wp.x - corr * vj.x;
      wn.y = zc.y / delta - wp.y - corr * vj.y;
      __stcs(reinterpret_cast<double2*>(V + (int64_t)j * ld + i), vj);
      __stcs(reinterpret_cast<double2*>(Zm + (int64_t)j * ld + i), zj);
      *reinterpret_cast<double2*>(W + i) = wn;
    } else {
      const int64_t kend = i + VW < n ? i + VW : n;
      for (int64_t k = i; k < kend; ++k) {
        double va = 0.0, wp = 0.0, za = 0.0;
        for (int r = 0; r < j; ++r) {
          const double vr = V[r * ld + k], zr = Zm[r * ld + k];
          va = fma(coef[r], vr, va);
          wp = fma(coef[j + r], vr, wp);
          za = fma(coef[r], zr, za);
        }
        const double vj = (W[k] - va) / delta;
        V[(int64_t)j * ld + k] = vj;
        Zm[(int64_t)j * ld + k] = (Mc[k] - za) / delta;
        W[k] = Zc[k] / delta - wp - corr * vj;
      }
    }
  }
}

// device-side single-reduce scalars from the fused block (krylov.py:305-306,
// 346-350), same operation order as the host copy: lets the next update be
// enqueued before the host has read the block back.
// blk: [a(0..j), b2] .v column at even slots, [p, q] at odd slots
__global__ void k_sr_coef(int j, const double* __restrict__ blk, double* __restrict__ coef) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double aa = 0.0, ap = 0.0;
  for (int r = 0; r < j; ++r) {
    const double a = blk[2 * r], p = blk[2 * r + 1];
    aa = rn_add(aa, rn_mul(a, a));
    ap = rn_add(ap, rn_mul(a, p));
  }
  const double d2 = rn_sub(blk[2 * j], aa);
  const double delta = d2 > 0.0 ? sqrt(d2) : 0.0;
  for (int r = 0; r < j; ++r) {
    coef[r] = blk[2 * r];
    coef[j + r] = rn_div(blk[2 * r + 1], delta);
  }
  coef[2 * j] = delta;
  coef[2 * j + 1] = rn_div(rn_sub(blk[2 * j + 1], ap), rn_mul(delta, delta));
}

// x_out = x + sum_r y[r] Zm[r]   (krylov.py:340, 361)
__global__ void __launch_bounds__(256) k_x_update(int64_t n, const double* __restrict__ x,
                                                  const double* __restrict__ Zm, int64_t ld, int m,
                                                  const double* __restrict__ y,
                                                  double* __restrict__ xo) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double acc = 0.0;
#pragma unroll 4
    for (int r = 0; r < m; ++r) acc = fma(__ldg(y + r), ldg_stream(Zm + r * ld + i), acc);
    xo[i] = x[i] + acc;
  }
}

// classic Arnoldi helpers (krylov.py:217-236): w -= sum_r h[r] v[r]
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
