// GMRES vector kernels (krylov.py:260-361 single-reduce, 179-257 classic).
//
// * k_block_dot: the ONE fused reduction per single-reduce iteration,
//   [V[:j]; v]^T [v, z] (krylov.py:290-300). Each thread owns element pairs
//   (grid-stride, 16-byte loads) and keeps all 2*rows running sums in
//   registers, so every basis row is streamed exactly once with many
//   independent loads in flight. Deterministic: fixed grid, fixed element
//   assignment, fixed shuffle trees, and the last CTA to finish reduces the
//   per-CTA partials in a fixed order (no second launch).
// * k_sr_update: v[j], zm[j] and the speculative next candidate w in one
//   pass (krylov.py:346-351); V[:j] is read once for both a and p/delta.
#pragma once
#include "common.cuh"

namespace gdsw {

constexpr int KDOT_ROWS = 32;  // rows per block-dot launch (basis rows + self)
constexpr int KDOT_THREADS = 256;
constexpr int KDOT_W2 = 2 * KDOT_ROWS;

// r = b - r (residual of a host operator's product, krylov.py:164-170)
__global__ void k_b_minus(int64_t n, const double* __restrict__ b, double* __restrict__ r) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) r[i] = b[i] - r[i];
}

// device-side single-reduce scalars from the fused block (krylov.py:305-306,
// 346-350), same operation order as the host copy
__device__ __forceinline__ void sr_coef_compute(int j, const double* blk, double* coef) {
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



// the last CTA to finish reduces all per-CTA partials in CTA order
// (deterministic) and, for a single-reduce block, computes the next update's
// scalars (k_sr_coef folded in); the ticket resets itself
__device__ __forceinline__ void block_dot_finish(int nv, int nrc, int nslots, double* __restrict__ partial,
                                                 double* __restrict__ out, unsigned* __restrict__ counter,
                                                 double* __restrict__ coef) {
  constexpr int NW = KDOT_THREADS / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int k = warp; k < 2 * nrc; k += NW) {
    double s = 0.0;
    for (int b = lane; b < nslots; b += 32) s += __ldcg(partial + (int64_t)b * KDOT_W2 + k);
    s = warp_sum(s);
    if (lane == 0) out[k] = s;
  }
  if (coef) {
    __syncthreads();
    if (threadIdx.x == 0) sr_coef_compute(nv, out, coef);
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// rows of the combined list [V[0..nv), v] restricted to [r0, r0 + nrc),
// nrc <= NR. out[2*rr + {0,1}] = row . v, row . z  (rr = local row index).
// Each thread owns element pairs (grid-stride, 16-byte loads) and keeps
// 2*NR running sums in registers: every basis row is read exactly once and
// all NR row loads of a step are independent (deep memory-level
// parallelism). One shuffle tree per sum at the end, per-CTA partials in
// fixed slots, the last CTA reduces them in CTA order (deterministic).
template <int NR, int EP = 1>
__global__ void __launch_bounds__(KDOT_THREADS, NR > 8 ? 1 : 2) k_block_dot(
    int64_t n, const double* __restrict__ V, int64_t ldv, int nv, int r0, int nrc,
    const double* __restrict__ v, const double* __restrict__ z, double* __restrict__ partial,
    double* __restrict__ out, unsigned* __restrict__ counter, double* __restrict__ coef) {
  constexpr int NW = KDOT_THREADS / 32;
  __shared__ double red[NW][2 * NR];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // rows q < nb come from V[r0 + q]; row nv - r0 (if in range) is v itself
  const int nb = max(0, min(nrc, nv - r0));
  const bool self = nv - r0 >= 0 && nv - r0 < nrc;
  double av[NR], az[NR], as = 0.0, zs = 0.0;
#pragma unroll
  for (int q = 0; q < NR; ++q) av[q] = az[q] = 0.0;
  const bool vec = ((ldv & 1) == 0) && ((reinterpret_cast<uintptr_t>(V) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(v) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(z) & 15) == 0);
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const double* Vr = V ? V + (int64_t)r0 * ldv : V;
  if (vec) {
    const int64_t n2 = n >> 1;
    const int32_t ld2 = (int32_t)(ldv >> 1);
    int64_t i0 = tid;
    if (EP == 2) {
      // two element pairs per step: twice the independent loads in flight
      // for the short blocks (few rows per thread)
#pragma unroll 1
      for (; i0 + nth < n2; i0 += 2 * nth) {
        double2 pv[2], pz[2], x[2][NR];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t ie = i0 + e * nth;
          pv[e] = __ldg(reinterpret_cast<const double2*>(v) + ie);
          pz[e] = z ? __ldg(reinterpret_cast<const double2*>(z) + ie) : make_double2(0.0, 0.0);
          const double2* pb = reinterpret_cast<const double2*>(Vr) + ie;
#pragma unroll
          for (int u = 0; u < NR; ++u) {
            if (u < nb) x[e][u] = ldg_stream(pb);
            pb += ld2;
          }
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
#pragma unroll
          for (int u = 0; u < NR; ++u) {
            if (u < nb) {
              av[u] = fma(x[e][u].y, pv[e].y, fma(x[e][u].x, pv[e].x, av[u]));
              az[u] = fma(x[e][u].y, pz[e].y, fma(x[e][u].x, pz[e].x, az[u]));
            }
          }
          if (self) {
            as = fma(pv[e].y, pv[e].y, fma(pv[e].x, pv[e].x, as));
            zs = fma(pv[e].y, pz[e].y, fma(pv[e].x, pz[e].x, zs));
          }
        }
      }
    }
#pragma unroll 1
    for (int64_t i = i0; i < n2; i += nth) {
      const double2 pv = __ldg(reinterpret_cast<const double2*>(v) + i);
      const double2 pz = z ? __ldg(reinterpret_cast<const double2*>(z) + i) : make_double2(0.0, 0.0);
      const double2* pb = reinterpret_cast<const double2*>(Vr) + i;
      // rows whose loads are in flight together (one CTA per SM above 8 rows:
      // more loads per thread)
      constexpr int G = NR <= 16 ? NR : NR / 2;
#pragma unroll
      for (int q0 = 0; q0 < NR; q0 += G) {
        double2 x[G];
#pragma unroll
        for (int u = 0; u < G; ++u) {
          if (q0 + u < nb) x[u] = ldg_stream(pb);
          pb += ld2;
        }
#pragma unroll
        for (int u = 0; u < G; ++u) {
          if (q0 + u < nb) {
            av[q0 + u] = fma(x[u].y, pv.y, fma(x[u].x, pv.x, av[q0 + u]));
            az[q0 + u] = fma(x[u].y, pz.y, fma(x[u].x, pz.x, az[q0 + u]));
          }
        }
      }
      if (self) {
        as = fma(pv.y, pv.y, fma(pv.x, pv.x, as));
        zs = fma(pv.y, pz.y, fma(pv.x, pz.x, zs));
      }
    }
    if ((n & 1) && tid == 0) {
      const int64_t e = n - 1;
      const double ve = v[e], ze = z ? z[e] : 0.0;
      const double* pe = Vr + e;
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        if (q < nb) {
          av[q] = fma(*pe, ve, av[q]);
          az[q] = fma(*pe, ze, az[q]);
        }
        pe += ldv;
      }
      as = fma(ve, ve, as);
      zs = fma(ve, ze, zs);
    }
  } else {
#pragma unroll 1
    for (int64_t e = tid; e < n; e += nth) {
      const double ve = v[e], ze = z ? z[e] : 0.0;
      const double* pe = Vr + e;
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        if (q < nb) {
          const double x = *pe;
          av[q] = fma(x, ve, av[q]);
          az[q] = fma(x, ze, az[q]);
        }
        pe += ldv;
      }
      as = fma(ve, ve, as);
      zs = fma(ve, ze, zs);
    }
  }
  if (self) {  // the self row sits at slot nb
#pragma unroll
    for (int q = 0; q < NR; ++q)
      if (q == nb) {
        av[q] = as;
        az[q] = zs;
      }
  }
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    if (q < nrc) {
      const double a = warp_sum(av[q]);
      const double c = warp_sum(az[q]);
      if (lane == 0) {
        red[warp][2 * q] = a;
        red[warp][2 * q + 1] = c;
      }
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 2 * nrc; k += KDOT_THREADS) {
    double a = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) a += red[w][k];
    partial[(int64_t)blockIdx.x * KDOT_W2 + k] = a;
  }
  block_dot_finish(nv, nrc, (int)gridDim.x, partial, out, counter, coef);
}

// Row-group block dot (the 16-byte path for 5+ rows): the rows are cut into
// groups of KRG, CTA b works on group b % ng and grid-strides the element
// pairs with the other CTAs of its group, holding only 2*KRG running sums.
// That keeps four CTAs (32 warps) resident per SM; v and z are re-read once
// per group, from L2 (the groups' CTAs sweep the same pairs together). The
// grid is one full wave (KRG_CTAS_PER_SM x SMs, split evenly over the groups):
// a partial second wave costs up to 20% (tools/micro/bench_blockdot3.cu).
// Per-CTA partials sit in the CTA's slot at the group's row offset; the last
// CTA sums the slots in order (deterministic).
constexpr int KRG = 4;
constexpr int KRG_CTAS_PER_SM = 4;

// HZ: z present (a compile-time switch: a run-time one splits the load batch)
template <bool HZ>
__global__ void __launch_bounds__(KDOT_THREADS, KRG_CTAS_PER_SM) k_block_dot_rg(
    int64_t n, const double* __restrict__ V, int64_t ldv, int nv, int r0, int nrc,
    const double* __restrict__ v, const double* __restrict__ z, double* __restrict__ partial,
    double* __restrict__ out, unsigned* __restrict__ counter, double* __restrict__ coef) {
  constexpr int NW = KDOT_THREADS / 32;
  __shared__ double red[NW][2 * KRG];
  const int ng = (nrc + KRG - 1) / KRG;
  const int g = blockIdx.x % ng, cta = blockIdx.x / ng, ncta = gridDim.x / ng;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = g * KRG;
  const int nr = min(KRG, nrc - q0);                // rows of this group
  const int nb = max(0, min(nr, nv - r0 - q0));     // basis rows among them
  const bool self = nv - r0 - q0 >= 0 && nv - r0 - q0 < nr;
  constexpr bool hz = HZ;
  double av[KRG], az[KRG], as = 0.0, zs = 0.0;
#pragma unroll
  for (int q = 0; q < KRG; ++q) av[q] = az[q] = 0.0;
  if (cta < ncta) {  // gridDim.x is a multiple of ng; guard anyway
    const int64_t n2 = n >> 1, ld2 = ldv >> 1;
    const int64_t nth = (int64_t)ncta * KDOT_THREADS;
    // slots past the group's basis rows read v (cached, ignored): every
    // load of a step is then unconditional and issued back to back
    const double2* rp[KRG];
#pragma unroll
    for (int u = 0; u < KRG; ++u)
      rp[u] = u < nb ? reinterpret_cast<const double2*>(V + (int64_t)(r0 + q0 + u) * ldv)
                     : reinterpret_cast<const double2*>(v);
    (void)ld2;
#pragma unroll 1
    for (int64_t i = (int64_t)cta * KDOT_THREADS + threadIdx.x; i < n2; i += nth) {
      double2 x[KRG];
#pragma unroll
      for (int u = 0; u < KRG; ++u) x[u] = ldg_stream(rp[u] + i);
      const double2 pv = __ldg(reinterpret_cast<const double2*>(v) + i);
      const double2 pz = hz ? __ldg(reinterpret_cast<const double2*>(z) + i) : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < KRG; ++u)
        if (u < nb) {
          av[u] = fma(x[u].y, pv.y, fma(x[u].x, pv.x, av[u]));
          az[u] = fma(x[u].y, pz.y, fma(x[u].x, pz.x, az[u]));
        }
      if (self) {
        as = fma(pv.y, pv.y, fma(pv.x, pv.x, as));
        zs = fma(pv.y, pz.y, fma(pv.x, pz.x, zs));
      }
    }
    if ((n & 1) && cta == 0 && threadIdx.x == 0) {
      const int64_t e = n - 1;
      const double ve = v[e], ze = hz ? z[e] : 0.0;
      const double* pe = V + (int64_t)(r0 + q0) * ldv + e;
#pragma unroll
      for (int q = 0; q < KRG; ++q) {
        if (q < nb) {
          av[q] = fma(*pe, ve, av[q]);
          az[q] = fma(*pe, ze, az[q]);
        }
        pe += ldv;
      }
      as = fma(ve, ve, as);
      zs = fma(ve, ze, zs);
    }
  }
  if (self) {  // the self row sits at slot nb
#pragma unroll
    for (int q = 0; q < KRG; ++q)
      if (q == nb) {
        av[q] = as;
        az[q] = zs;
      }
  }
#pragma unroll
  for (int q = 0; q < KRG; ++q) {
    if (q < nr) {
      const double a = warp_sum(av[q]);
      const double c = warp_sum(az[q]);
      if (lane == 0) {
        red[warp][2 * q] = a;
        red[warp][2 * q + 1] = c;
      }
    }
  }
  __syncthreads();
  if (cta < ncta)
    for (int k = threadIdx.x; k < 2 * nr; k += KDOT_THREADS) {
      double a = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) a += red[w][k];
      partial[(int64_t)cta * KDOT_W2 + 2 * q0 + k] = a;
    }
  block_dot_finish(nv, nrc, ncta, partial, out, counter, coef);
}

// partial slots a block dot may use on `sms` SMs
inline int block_dot_slots(int sms) { return KRG_CTAS_PER_SM * sms; }

// host dispatch: the row-group kernel on the 16-byte path from 5 rows up,
// the all-rows-per-thread kernel for 1-4 rows (equal there) and for the
// unaligned path
inline void launch_block_dot(int sms, cudaStream_t s, int64_t n, const double* V, int64_t ldv,
                             int nv, int r0, int nrc, const double* v, const double* z,
                             double* partial, double* out, unsigned* counter, double* coef = nullptr) {
  const bool vec = ((ldv & 1) == 0) && ((reinterpret_cast<uintptr_t>(V) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(v) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(z) & 15) == 0);
  const unsigned grid = 2 * sms;
  if (vec && nrc > 4 && V) {
    const int ng = (nrc + KRG - 1) / KRG;
    const int per = std::max(1, KRG_CTAS_PER_SM * sms / ng);
    if (z)
      k_block_dot_rg<true><<<per * ng, KDOT_THREADS, 0, s>>>(n, V, ldv, nv, r0, nrc, v, z, partial, out, counter,
                                                            coef);
    else
      k_block_dot_rg<false><<<per * ng, KDOT_THREADS, 0, s>>>(n, V, ldv, nv, r0, nrc, v, z, partial, out, counter,
                                                             coef);
  } else if (nrc <= 4)
    k_block_dot<4, 2><<<grid, KDOT_THREADS, 0, s>>>(n, V, ldv, nv, r0, nrc, v, z, partial, out, counter, coef);
  else if (nrc <= 8)
    k_block_dot<8><<<grid, KDOT_THREADS, 0, s>>>(n, V, ldv, nv, r0, nrc, v, z, partial, out, counter, coef);
  else if (nrc <= 16)  // 32+ running sums: one CTA per SM (launch bound), half the grid
    k_block_dot<16, 2><<<(grid + 1) / 2, KDOT_THREADS, 0, s>>>(n, V, ldv, nv, r0, nrc, v, z, partial, out,
                                                          counter, coef);
  else
    k_block_dot<32><<<(grid + 1) / 2, KDOT_THREADS, 0, s>>>(n, V, ldv, nv, r0, nrc, v, z, partial, out,
                                                          counter, coef);
}

// single-reduce update (krylov.py:346-351). coef = [a(0..j), p/delta(0..j),
// delta, corr]. VW = 2: 16-byte vector path (rows of even ld, aligned).
// ZM = false: the preconditioned basis Zm is not kept (zm[j] = M v[j] by
// linearity; the cycle-end x update applies M to V y instead), so the
// update reads V[:j], W, ZC and writes v[j], w only.
template <int VW, bool ZM = true>
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
        const double a = __ldg(coef + r), pd = __ldg(coef + j + r);
        va.x = fma(a, vr.x, va.x);
        va.y = fma(a, vr.y, va.y);
        wp.x = fma(pd, vr.x, wp.x);
        wp.y = fma(pd, vr.y, wp.y);
        if (ZM) {
          const double2 zr = ldg_stream(reinterpret_cast<const double2*>(Zm + r * ld + i));
          za.x = fma(a, zr.x, za.x);
          za.y = fma(a, zr.y, za.y);
        }
      }
      const double2 w = *reinterpret_cast<const double2*>(W + i);
      const double2 zc = ldg_stream(reinterpret_cast<const double2*>(Zc + i));
      double2 vj, wn;
      vj.x = (w.x - va.x) / delta;
      vj.y = (w.y - va.y) / delta;
      wn.x = zc.x / delta - wp.x - corr * vj.x;
      wn.y = zc.y / delta - wp.y - corr * vj.y;
      __stcs(reinterpret_cast<double2*>(V + (int64_t)j * ld + i), vj);
      if (ZM) {
        const double2 mc = ldg_stream(reinterpret_cast<const double2*>(Mc + i));
        double2 zj;
        zj.x = (mc.x - za.x) / delta;
        zj.y = (mc.y - za.y) / delta;
        __stcs(reinterpret_cast<double2*>(Zm + (int64_t)j * ld + i), zj);
      }
      *reinterpret_cast<double2*>(W + i) = wn;
    } else {
      const int64_t kend = i + VW < n ? i + VW : n;
      for (int64_t k = i; k < kend; ++k) {
        double va = 0.0, wp = 0.0, za = 0.0;
        for (int r = 0; r < j; ++r) {
          const double vr = V[r * ld + k];
          va = fma(coef[r], vr, va);
          wp = fma(coef[j + r], vr, wp);
          if (ZM) za = fma(coef[r], Zm[r * ld + k], za);
        }
        const double vj = (W[k] - va) / delta;
        V[(int64_t)j * ld + k] = vj;
        if (ZM) Zm[(int64_t)j * ld + k] = (Mc[k] - za) / delta;
        W[k] = Zc[k] / delta - wp - corr * vj;
      }
    }
  }
}

// t = sum_r y[r] V[r]   (the basis combination M is applied to)
__global__ void __launch_bounds__(256) k_combine(int64_t n, const double* __restrict__ V, int64_t ld, int m,
                                                 const double* __restrict__ y, double* __restrict__ t) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double acc = 0.0;
#pragma unroll 4
    for (int r = 0; r < m; ++r) acc = fma(__ldg(y + r), ldg_stream(V + r * ld + i), acc);
    t[i] = acc;
  }
}

// xo = x + d
__global__ void k_add(int64_t n, const double* __restrict__ x, const double* __restrict__ d,
                      double* __restrict__ xo) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) xo[i] = x[i] + d[i];
}

// device-side single-reduce scalars from the fused block (krylov.py:305-306,
// 346-350), same operation order as the host copy: lets the next update be
// enqueued before the host has read the block back.
// blk: [a(0..j), b2] .v column at even slots, [p, q] at odd slots
__global__ void k_sr_coef(int j, const double* __restrict__ blk, double* __restrict__ coef) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  sr_coef_compute(j, blk, coef);
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
