// Temporally blocked FastSpTRSV (jacobi_trisolve_lower_unit / _upper,
// _kernels.py:620-656; fast_trisolve, local_solvers.py:413-427).
//
// All iters-1 sweeps of one factor in ONE launch: a CTA owns a tile of
// consecutive rows [a, b) of one block and keeps the iterates of the tile
// plus a halo in shared memory. A row only reads rows within the factor's
// reach K of it (one grid plane for natural-ordered 7-point ILU(0)), so
// sweep t is computed on the tile extended by (s - t) K halo rows (below the
// tile for L, above it for U) and the halo shrinks by K per sweep; the halo
// rows are recomputed by the neighbouring tiles' CTAs instead of exchanged.
// Only the tile's final rows are written. The factor streams from HBM once
// per apply (sweeps 2.. hit L2), the iterates never leave shared memory,
// and one launch replaces a launch per sweep.
//
// Per-row arithmetic is the sequential kernels' -- every row accumulates in
// its own column order with round-to-nearest mul/sub -- so the result is
// bit-identical to them and to the reference.
#pragma once
#include "common.cuh"
#include "sparse.cuh"

namespace gdsw {

constexpr int TB_THREADS = 1024;

struct TbTile {
  int32_t a, b;     // tile rows (concatenated)
  int32_t s0, s1;   // rows of its block
  int32_t reach;    // K of the block's factor
  int32_t pad;
};

// two rows per call, every global load of both issued before the first
// shared-memory gather (the slot loads are the latency to hide)
template <typename T, bool D16>
__device__ __forceinline__ void tb_row2(const SellDev& M, const T* __restrict__ val, int32_t i0, int32_t i1,
                                        bool ok1, T& acc0, T& acc1, const T* xs, int32_t off) {
  const int64_t b0 = sell_base(M, i0), b1 = sell_base(M, ok1 ? i1 : i0);
  const int len0 = M.row_len[i0], len1 = ok1 ? (int)M.row_len[i1] : 0;
  int32_t c0[4], c1[4];
  T v0[4], v1[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k < M.uw) {
      c0[k] = sell_col<D16>(M, i0, b0 + 32 * (int64_t)k);
      v0[k] = val[b0 + 32 * (int64_t)k];
      if (ok1) {
        c1[k] = sell_col<D16>(M, i1, b1 + 32 * (int64_t)k);
        v1[k] = val[b1 + 32 * (int64_t)k];
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k < len0) acc0 = rn_sub(acc0, rn_mul(v0[k], xs[c0[k] - off]));
    if (k < len1) acc1 = rn_sub(acc1, rn_mul(v1[k], xs[c1[k] - off]));
  }
}

// L: x^1 = b = r[gmap], x^{t+1} = b - (L - I) x^t for t = 1..s; writes
// B (the gathered right-hand side, over the tile and its halo -- neighbours
// write identical values) and F = x^{s+1}. Shared: two iterate buffers over
// [lo, b).
template <typename T, bool D16>
__global__ void __launch_bounds__(TB_THREADS, 1) k_jacobi_tb_lower(SellDev L, const T* __restrict__ lval,
                                                                  const TbTile* __restrict__ tiles, int s,
                                                                  const int32_t* __restrict__ gmap,
                                                                  const double* __restrict__ r, T* B,
                                                                  T* __restrict__ F) {
  extern __shared__ __align__(16) unsigned char tb_smem[];
  const TbTile tl = tiles[blockIdx.x];
  const int32_t lo = max(tl.s0, tl.a - s * tl.reach);
  const int32_t w = tl.b - lo;
  T* cur = reinterpret_cast<T*>(tb_smem);
  T* nxt = cur + w;
  for (int32_t i = lo + threadIdx.x; i < tl.b; i += TB_THREADS) {
    const T bi = (T)r[gmap[i]];
    B[i] = bi;
    cur[i - lo] = bi;  // x^1 = b
  }
  __syncthreads();
  for (int t = 1; t <= s; ++t) {
    const int32_t lt = max(tl.s0, tl.a - (s - t) * tl.reach);
    for (int32_t i = lt + threadIdx.x; i < tl.b; i += 2 * TB_THREADS) {
      const int32_t j = i + TB_THREADS;
      const bool okj = j < tl.b;
      T acc = B[i], accj = okj ? B[j] : T(0);
      tb_row2<T, D16>(L, lval, i, j, okj, acc, accj, cur, lo);
      if (t < s) {
        nxt[i - lo] = acc;
        if (okj) nxt[j - lo] = accj;
      } else {
        if (i >= tl.a) F[i] = acc;
        if (okj && j >= tl.a) F[j] = accj;
      }
    }
    __syncthreads();
    T* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
}

// U: y^1 = F / D (recomputed on the halo), y^{t+1} = D^-1 (F - (U - D) y^t)
// for t = 1..s; writes y^{s+1} for the tile. Shared: two iterate buffers
// over [a, hi).
template <typename T, bool D16>
__global__ void __launch_bounds__(TB_THREADS, 1) k_jacobi_tb_upper(SellDev U, const T* __restrict__ uval,
                                                                  const TbTile* __restrict__ tiles, int s,
                                                                  const T* __restrict__ diag,
                                                                  const T* __restrict__ F, T* __restrict__ y) {
  extern __shared__ __align__(16) unsigned char tb_smem[];
  const TbTile tl = tiles[blockIdx.x];
  const int32_t hi = min(tl.s1, tl.b + s * tl.reach);
  const int32_t w = hi - tl.a;
  T* cur = reinterpret_cast<T*>(tb_smem);
  T* nxt = cur + w;
  for (int32_t i = tl.a + threadIdx.x; i < hi; i += TB_THREADS) cur[i - tl.a] = rn_div(F[i], diag[i]);
  __syncthreads();
  for (int t = 1; t <= s; ++t) {
    const int32_t ht = min(tl.s1, tl.b + (s - t) * tl.reach);
    for (int32_t i = tl.a + threadIdx.x; i < ht; i += 2 * TB_THREADS) {
      const int32_t j = i + TB_THREADS;
      const bool okj = j < ht;
      T acc = F[i], accj = okj ? F[j] : T(0);
      const T di = diag[i], dj = okj ? diag[j] : T(1);
      tb_row2<T, D16>(U, uval, i, j, okj, acc, accj, cur, tl.a);
      const T yi = rn_div(acc, di), yj = rn_div(accj, dj);
      if (t < s) {
        nxt[i - tl.a] = yi;
        if (okj) nxt[j - tl.a] = yj;
      } else {
        if (i < tl.b) y[i] = yi;
        if (okj && j < tl.b) y[j] = yj;
      }
    }
    __syncthreads();
    T* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
}

}  // namespace gdsw
