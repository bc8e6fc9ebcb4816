// Factored coarse solve v = A0^-1 u for large coarse spaces: the supernodal
// partitioned inverse of the nested-dissection LU of A0 (built on the host by
// paper_2304_04876_b200/coarse_factor.py; replaces the reference's sparse LU
// + level-set solves, schwarz.py:267-272, 305, and the dense A0^-1 GEMV once
// n_c^2 values per apply stop being cheap).
//
// One persistent launch (k_cf_dataflow). A CTA takes one task = (supernode
// k, tile of rows of its stacked block), stages the block's input vector in
// shared memory and computes its rows (warp per row over row-major blocks,
// or thread per row over column-major panels for narrow supernodes):
//  forward  (leaves first): bt = u[C_k] - the children's updates on C_k
//           (fixed order), rows < s: y[C_k] = L_kk^-1 bt (strict-lower part
//           of the diagonal block + the unit diagonal), rows >= s: the
//           update cbuf[R_k] = (L_{R_k,k} L_kk^-1) bt + the children's
//           updates on R_k (multifrontal extend-add)
//  backward (root first): x[C_k] = U_kk^-1 y[C_k] - (U_kk^-1 U_{k,R_k}) x[R_k]
#pragma once
#include "common.cuh"

namespace gdsw {

// CTA shapes of the dataflow kernel (48 registers either way): local exact-LU
// solves of 32+ blocks run 128 threads x 10 resident CTAs (C3-sized
// blocks 0.245 -> 0.220 ms, C3 92.4 -> 87.8 ms), the coarse factor and few
// blocks 256 x 5 (128 threads measured slower there: n_c = 12,600, C5 2,048
// subdomains 41.6 -> 44.9 ms; C1 4.4 -> 4.56 ms). A narrow
// tile (thread per row, columns split in at least two parts) holds at most
// NT / 2 rows: the host tiler clamps to that.
constexpr int CF_NT_LOCAL = 128, CF_NT_COARSE = 256;
constexpr int cf_min_ctas(int nt) { return 1280 / nt; }  // 10 x 128, 5 x 256 (48 registers)
constexpr int CF_ROWS = 8;   // smallest tile: one row per warp

struct CoarseFactorDev {
  // dataflow schedule (k_cf_dataflow): parent of each supernode, its
  // children, and the readiness targets
  const int32_t* parent;
  const int32_t* child_ptr;
  const int32_t* child_idx;
  const int32_t* fwd_need;   // forward tiles of the children
  const int32_t* bwd_need;   // own forward tiles + the parent's backward tiles
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
  // narrow supernodes (s <= CF_CM_MAX): the forward block [L_kk^-1; M] also
  // stored column-major ((s + r) x s, column c contiguous over the rows), so
  // a thread per row streams it coalesced with no reduction; -1 otherwise
  const int64_t* f_off;
};

// widest supernode with column-major panels: coarse factors 128, local
// exact-LU blocks 512 (measured: C3-sized blocks 0.311 -> 0.298 ms with 512;
// the n_c = 12,600 coarse solve 0.287 -> 0.298 ms, so it keeps 128);
// GDSW_CF_CM_MAX overrides both
constexpr int CF_CM_MAX = 128;
constexpr int CF_CM_LOCAL = 512;

// dot of a dense row segment [j0, j1) with a shared-memory vector: lanes
// over the columns, eight independent partial sums (eight row loads in
// flight per lane: one row per warp must keep HBM busy on its own when a
// level holds few supernodes). Measured: a predicated tail (all of a short
// row's loads at once) and eight rows per warp were both slower.
template <typename T>
__device__ __forceinline__ T cf_dot(const T* __restrict__ row, const T* vec, int j0, int j1, int lane) {
  T a[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) a[u] = T(0);
  int j = j0 + lane;
  for (; j + 224 < j1; j += 256) {
    T rr[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) rr[u] = ldg_stream(row + j + 32 * u);
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = fma(rr[u], vec[j + 32 * u], a[u]);
  }
  for (; j < j1; j += 32) a[0] = fma(ldg_stream(row + j), vec[j], a[0]);
  return warp_sum(((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7])));
}

// ---------------------------------------------------------------------------
// the whole solve in ONE launch: a persistent grid takes the tasks (forward
// tiles leaves-first, then backward tiles root-first) from an atomic ticket
// in order and runs each as soon as its inputs exist: a forward tile waits
// for every forward tile of its children (their updates), a backward tile
// for its own forward tiles (y) and every backward tile of its parent (x on
// R_k; the parent waited for its own parent). Tiles signal with release
// atomics on per-supernode counters. No level barriers, so independent
// subtrees overlap. Tasks are taken in dependency order by resident CTAs,
// so every awaited tile is already running: no deadlock. The last CTA to
// leave resets the ticket and counters (graph-replay safe).
struct CfSched {
  unsigned* ticket;     // [0]: next task, [1]: CTAs done
  int32_t* fwd_ready;   // per supernode
  int32_t* bwd_ready;
  int32_t n_fwd, n_tasks, n_sn;
};

__device__ __forceinline__ int32_t ld_acquire_gpu(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// column-major forward panel of the narrow supernodes, from D (strict lower)
// and M: F[c (s + r) + i] = L_kk^-1[i][c] (i < s, zero on and above the
// diagonal), M[i - s][c] (i >= s)
template <typename T>
__global__ void k_pinv_fcm(CoarseFactorDev F, const int32_t* __restrict__ sn_list, int32_t n_list,
                           const T* __restrict__ vals, T* __restrict__ fcm) {
  const int q = sn_list[blockIdx.x];
  const int s = F.sn_s[q], r = F.sn_r[q];
  const T* D = vals + F.d_off[q];
  const T* M = vals + F.m_off[q];
  T* out = fcm + F.f_off[q];
  for (int64_t e = threadIdx.x; e < (int64_t)(s + r) * s; e += blockDim.x) {
    const int c = (int)(e / (s + r)), i = (int)(e % (s + r));
    out[e] = i < s ? (c < i ? D[(int64_t)i * s + c] : T(0)) : M[(int64_t)(i - s) * s + c];
  }
  // backward block [U_kk^-1 | -N] column-major (s rows, s + r columns):
  // B[c s + i] = U_kk^-1[i][c] (c >= i, else 0), -N[i][c - s] (c >= s)
  const T* N = vals + F.n_off[q];
  T* bo = out + (int64_t)(s + r) * s;
  for (int64_t e = threadIdx.x; e < (int64_t)(s + r) * s; e += blockDim.x) {
    const int c = (int)(e / s), i = (int)(e % s);
    bo[e] = c < s ? (c >= i ? D[(int64_t)i * s + c] : T(0)) : -N[(int64_t)i * r + (c - s)];
  }
}

// one thread's share of a column-major panel row: columns [c, c1) of the
// row at pc (column stride `ld`), CF_CMU loads in flight, four partial sums
#ifndef CF_CMU
#define CF_CMU 4
#endif
template <typename T>
__device__ __forceinline__ void cm_dot(const T* __restrict__ pc, int64_t ld, int c, int c1, const T* buf, T (&a)[4]) {
  for (; c + CF_CMU <= c1; c += CF_CMU) {
    T v[CF_CMU];
#pragma unroll
    for (int uu = 0; uu < CF_CMU; ++uu) v[uu] = ldg_stream(pc + (int64_t)(c + uu) * ld);
#pragma unroll
    for (int uu = 0; uu < CF_CMU; ++uu) a[uu & 3] = fma(v[uu], buf[c + uu], a[uu & 3]);
  }
  for (; c < c1; ++c) a[0] = fma(ldg_stream(pc + (int64_t)c * ld), buf[c], a[0]);
}

// register cap from the resident-CTA target (256 threads: 5 per SM at 48
// registers took C3-sized blocks 0.278 -> 0.245 ms; 6 and 8 spilled, slower)
template <typename T, typename TI, int CF_THREADS>
__global__ void __launch_bounds__(CF_THREADS, cf_min_ctas(CF_THREADS)) k_cf_dataflow(CoarseFactorDev F, CfSched S,
                                                            const int2* __restrict__ tasks,
                                                            const T* __restrict__ vals, const TI* __restrict__ u,
                                                            const int32_t* __restrict__ gmap, T* __restrict__ y,
                                                            T* __restrict__ cbuf, T* __restrict__ x,
                                                            const T* __restrict__ fcm) {
  extern __shared__ __align__(16) unsigned char cf_sm[];
  T* buf = reinterpret_cast<T*>(cf_sm);
  __shared__ int32_t cur;
  __shared__ T red[CF_THREADS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // thread 0 holds the next ticket while the CTA works on the current one
  // (no deadlock: the smallest unfinished ticket is always either running
  // with its inputs done, or the prefetch of a CTA whose current task is done)
  int32_t mine = 0;
  if (threadIdx.x == 0) mine = (int32_t)atomicAdd(S.ticket, 1u);
  for (;;) {
    if (threadIdx.x == 0) cur = mine;
    __syncthreads();
    const int32_t t = cur;
    if (t >= S.n_tasks) break;
    const bool fwd = t < S.n_fwd;
    const int2 tk = tasks[t];
    // tile: rows [row0, row0 + nrows) of the stacked block (sized per level
    // at install: enough tiles to fill the GPU, no more)
    const int k = tk.x, row0 = tk.y & 0xFFFF, nrows = tk.y >> 16;
    const int s = F.sn_s[k], r = F.sn_r[k];
    const int32_t* cols = F.col_ids + F.col_ptr[k];
    if (threadIdx.x == 0) {
      const int32_t* ready = fwd ? S.fwd_ready + k : S.bwd_ready + k;
      const int32_t need = fwd ? F.fwd_need[k] : F.bwd_need[k];
      while (ld_acquire_gpu(ready) < need) __nanosleep(20);
      mine = (int32_t)atomicAdd(S.ticket, 1u);
    }
    __syncthreads();
    if (fwd) {
      const int32_t cb = F.col_ptr[k];
      for (int i = threadIdx.x; i < s; i += CF_THREADS) {
        // the input chain (cols -> gmap -> u) and the first two children's
        // updates (in_ptr -> in_idx -> cbuf) issued side by side: three
        // dependent rounds instead of six; subtracted in list order
        const int32_t c = cols[i];
        const int32_t p0 = F.in_ptr[cb + i], p1 = F.in_ptr[cb + i + 1];
        const int32_t gi = gmap ? gmap[c] : c;
        const int32_t i0 = p0 < p1 ? F.in_idx[p0] : -1;
        const int32_t i1 = p0 + 1 < p1 ? F.in_idx[p0 + 1] : -1;
        T acc = (T)u[gi];
        const T c0 = i0 >= 0 ? __ldcg(cbuf + i0) : T(0);
        const T c1 = i1 >= 0 ? __ldcg(cbuf + i1) : T(0);
        if (i0 >= 0) acc -= c0;
        if (i1 >= 0) acc -= c1;
        for (int32_t p = p0 + 2; p < p1; ++p) acc -= __ldcg(cbuf + F.in_idx[p]);
        buf[i] = acc;
      }
      __syncthreads();
      if (F.f_off[k] >= 0) {
        // narrow supernode: thread per row over the column-major panel; the
        // columns split in `spl` contiguous parts (spl = 256 / rows rounded
        // down to a power of two) whose partials are combined in part order
        const T* P = fcm + F.f_off[k];
        int spl = 2;
        while (spl < 16 && nrows * spl * 2 <= CF_THREADS) spl *= 2;
        const int rows_pad = CF_THREADS / spl;
        const int half = threadIdx.x / rows_pad, q = threadIdx.x % rows_pad;
        const int row = row0 + q;
        const bool on = q < nrows;
        const int c0 = (int)((int64_t)s * half / spl), c1 = (int)((int64_t)s * (half + 1) / spl);
        T extra = T(0);
        int32_t gi = -1;
        if (on && half == 0 && row >= s) {  // extend-add terms, loaded ahead
          gi = F.row_ptr[k] + row - s;
          for (int32_t p = F.out_ptr[gi]; p < F.out_ptr[gi + 1]; ++p) extra += __ldcg(cbuf + F.out_idx[p]);
        }
        T a[4] = {T(0), T(0), T(0), T(0)};
        if (on) {
          const T* pc = P + row;
          int c = c0;
          cm_dot(pc, (int64_t)(s + r), c, c1, buf, a);
        }
        red[threadIdx.x] = (a[0] + a[1]) + (a[2] + a[3]);
        __syncthreads();
        if (on && half == 0) {
          T acc = red[threadIdx.x];
          for (int h = 1; h < spl; ++h) acc += red[threadIdx.x + h * rows_pad];
          if (row < s) y[cols[row]] = acc + buf[row];
          else cbuf[gi] = acc + extra;
        }
      } else
      for (int q = warp; q < nrows; q += CF_THREADS / 32) {
        const int row = row0 + q;
        if (row >= s + r) break;
        if (row < s) {
          const T acc = cf_dot(vals + F.d_off[k] + (int64_t)row * s, buf, 0, row, lane);
          if (lane == 0) y[cols[row]] = acc + buf[row];
        } else {
          // the children's updates on this row (extend-add) are loaded by
          // the lanes before the dot, so their latency overlaps its loads;
          // added in list order after it
          const int32_t g = F.row_ptr[k] + row - s;
          const int32_t p0 = F.out_ptr[g], np = F.out_ptr[g + 1] - p0;
          T extra = T(0);
          if (lane < np) extra = __ldcg(cbuf + F.out_idx[p0 + lane]);
          T acc = cf_dot(vals + F.m_off[k] + (int64_t)(row - s) * s, buf, 0, s, lane);
          for (int e = 0; e < min(np, 32); ++e) acc += __shfl_sync(0xffffffffu, extra, e);
          for (int32_t p = p0 + 32; p < p0 + np; ++p) acc += __ldcg(cbuf + F.out_idx[p]);
          if (lane == 0) cbuf[g] = acc;
        }
      }
    } else {
      const int32_t* rows = F.row_ids + F.row_ptr[k];
      for (int i = threadIdx.x; i < s + r; i += CF_THREADS)
        buf[i] = i < s ? __ldcg(y + cols[i]) : __ldcg(x + rows[i - s]);
      __syncthreads();
      if (F.f_off[k] >= 0) {
        // narrow supernode: thread per row over the column-major [U^-1 | -N],
        // the s + r columns split in `spl` parts combined in part order
        const T* P = fcm + F.f_off[k] + (int64_t)(s + r) * s;
        int spl = 2;
        while (spl < 16 && nrows * spl * 2 <= CF_THREADS) spl *= 2;
        const int rows_pad = CF_THREADS / spl;
        const int part = threadIdx.x / rows_pad, q = threadIdx.x % rows_pad;
        const int row = row0 + q;
        const bool on = q < nrows;
        const int w = s + r;
        const int c0 = max((int)((int64_t)w * part / spl), on ? row : 0);
        const int c1 = (int)((int64_t)w * (part + 1) / spl);
        T a[4] = {T(0), T(0), T(0), T(0)};
        if (on) {
          const T* pc = P + row;
          int c = c0;
          cm_dot(pc, (int64_t)s, c, c1, buf, a);
        }
        red[threadIdx.x] = (a[0] + a[1]) + (a[2] + a[3]);
        __syncthreads();
        if (on && part == 0) {
          T acc = red[threadIdx.x];
          for (int h = 1; h < spl; ++h) acc += red[threadIdx.x + h * rows_pad];
          x[cols[row]] = acc;
        }
      } else
      for (int q = warp; q < nrows; q += CF_THREADS / 32) {
        const int row = row0 + q;
        if (row >= s) break;
        const T a = cf_dot(vals + F.d_off[k] + (int64_t)row * s, buf, row, s, lane);
        const T b = cf_dot(vals + F.n_off[k] + (int64_t)row * r, buf + s, 0, r, lane);
        if (lane == 0) x[cols[row]] = a - b;
      }
    }
    // publish: every thread's stores, then one release increment per
    // dependent supernode
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      if (fwd) {
        atomicAdd(S.bwd_ready + k, 1);
        const int32_t p = F.parent[k];
        if (p >= 0) atomicAdd(S.fwd_ready + p, 1);
      } else {
        for (int32_t c = F.child_ptr[k]; c < F.child_ptr[k + 1]; ++c) atomicAdd(S.bwd_ready + F.child_idx[c], 1);
      }
    }
  }
  // the last CTA out resets the schedule for the next solve
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(S.ticket + 1, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    for (int32_t i = threadIdx.x; i < S.n_sn; i += CF_THREADS) {
      S.fwd_ready[i] = 0;
      S.bwd_ready[i] = 0;
    }
    if (threadIdx.x == 0) {
      S.ticket[0] = 0u;
      S.ticket[1] = 0u;
    }
  }
}

// ---------------------------------------------------------------------------
// numeric build of the local partitioned inverses ON THE DEVICE from the
// device factors (the reference's IKJ LU, k_lu_numeric): the host computes
// only the supernode structure from the symbolic patterns.
//  k_pinv_fill   : thread per (supernode, stacked row): the row's CSR
//                  entries that fall in the supernode go to its dense panels
//                  [L_CC; L_RC] ((s + r) x s) and [U_CC, U_CR] (s x (s + r))
//  k_pinv_blocks : CTA per supernode: L_CC^-1 (strict lower of D) and U_CC^-1
//                  (upper of D) by row recurrences, then M = L_RC L_CC^-1 and
//                  N = U_CC^-1 U_CR; fp64 arithmetic, stored in T
// Row recurrences: row i of L^-1 = e_i - sum_{k<i} L[i][k] row_k; row i of
// U^-1 = (e_i - sum_{k>i} U[i][k] row_k) / U[i][i] -- the host builder's.
// ---------------------------------------------------------------------------
constexpr int PB_THREADS = 256;
constexpr int PB_J = 8;  // columns per thread: supernodes up to 2,048 columns

struct PinvBuildDev {
  const int64_t* l_ptr;     // factor CSR by global block position, block-local columns
  const int32_t* l_idx;
  const int64_t* u_ptr;
  const int32_t* u_idx;
  const int32_t* pos_sn;    // [n_loc] supernode owning each position (as a column)
  const int32_t* pos_c;     // [n_loc] its index in that supernode's column list
  const int32_t* sn_base;   // [n_sn] block base of each supernode
  const int64_t* pan_off;   // [n_sn] offset of the L panel; the U panel follows it
  const int2* rows;         // fill tasks: (supernode, stacked row)
  int32_t n_rows;
};

template <typename T>
__global__ void k_pinv_fill(CoarseFactorDev F, PinvBuildDev B, const T* __restrict__ lval,
                            const T* __restrict__ uval, double* __restrict__ pan) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B.n_rows) return;
  const int2 task = B.rows[t];
  const int q = task.x, rr = task.y;
  const int s = F.sn_s[q], r = F.sn_r[q];
  const int32_t base = B.sn_base[q];
  const int32_t g = rr < s ? F.col_ids[F.col_ptr[q] + rr] : F.row_ids[F.row_ptr[q] + rr - s];
  double* lp = pan + B.pan_off[q] + (int64_t)rr * s;
  for (int64_t p = B.l_ptr[g]; p < B.l_ptr[g + 1]; ++p) {
    const int32_t j = base + B.l_idx[p];
    if (B.pos_sn[j] == q) lp[B.pos_c[j]] = (double)lval[p];
  }
  if (rr >= s) return;
  double* up = pan + B.pan_off[q] + (int64_t)(s + r) * s + (int64_t)rr * (s + r);
  const int32_t* R = F.row_ids + F.row_ptr[q];
  for (int64_t p = B.u_ptr[g]; p < B.u_ptr[g + 1]; ++p) {
    const int32_t j = base + B.u_idx[p];
    if (B.pos_sn[j] == q) {
      up[B.pos_c[j]] = (double)uval[p];
    } else {
      int lo = 0, hi = r;  // j is in R (the structure guarantees it)
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (R[mid] < j) lo = mid + 1; else hi = mid;
      }
      if (lo < r && R[lo] == j) up[s + lo] = (double)uval[p];
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(PB_THREADS) k_pinv_blocks(CoarseFactorDev F, PinvBuildDev B,
                                                            const double* __restrict__ pan,
                                                            double* __restrict__ dwork, T* __restrict__ vals,
                                                            int32_t* __restrict__ bad) {
  const int q = blockIdx.x;
  const int s = F.sn_s[q], r = F.sn_r[q];
  const double* L = pan + B.pan_off[q];              // (s + r) x s
  const double* U = L + (int64_t)(s + r) * s;        // s x (s + r)
  double* D = dwork + F.d_off[q];                    // s x s, fp64 scratch
  const int tid = threadIdx.x;
  // L_CC^-1 (strict lower of D; unit diagonal implied)
  for (int i = 0; i < s; ++i) {
    double acc[PB_J];
#pragma unroll
    for (int u = 0; u < PB_J; ++u) acc[u] = 0.0;
    for (int k = 0; k < i; ++k) {
      const double lik = L[(int64_t)i * s + k];
      if (lik == 0.0) continue;
#pragma unroll
      for (int u = 0; u < PB_J; ++u) {
        const int j = tid + PB_THREADS * u;
        if (j <= k) acc[u] += lik * (j == k ? 1.0 : D[(int64_t)k * s + j]);
      }
    }
#pragma unroll
    for (int u = 0; u < PB_J; ++u) {
      const int j = tid + PB_THREADS * u;
      if (j < i) D[(int64_t)i * s + j] = -acc[u];
    }
    __syncthreads();
  }
  // U_CC^-1 (upper of D including the diagonal)
  for (int i = s - 1; i >= 0; --i) {
    const double dii = U[(int64_t)i * (s + r) + i];
    if (dii == 0.0 || !isfinite(dii)) {
      if (tid == 0) atomicExch(bad, 1);
      return;
    }
    double acc[PB_J];
#pragma unroll
    for (int u = 0; u < PB_J; ++u) acc[u] = 0.0;
    for (int k = i + 1; k < s; ++k) {
      const double uik = U[(int64_t)i * (s + r) + k];
      if (uik == 0.0) continue;
#pragma unroll
      for (int u = 0; u < PB_J; ++u) {
        const int j = tid + PB_THREADS * u;
        if (j >= k && j < s) acc[u] += uik * D[(int64_t)k * s + j];
      }
    }
#pragma unroll
    for (int u = 0; u < PB_J; ++u) {
      const int j = tid + PB_THREADS * u;
      if (j == i) D[(int64_t)i * s + j] = 1.0 / dii;
      else if (j > i && j < s) D[(int64_t)i * s + j] = -acc[u] / dii;
    }
    __syncthreads();
  }
  // M = L_RC L_CC^-1 (r x s): M[m][j] = L_R[m][j] + sum_{k > j} L_R[m][k] Linv[k][j]
  T* M = vals + F.m_off[q];
  for (int m = 0; m < r; ++m) {
    const double* lr = L + (int64_t)(s + m) * s;
    double acc[PB_J];
#pragma unroll
    for (int u = 0; u < PB_J; ++u) {
      const int j = tid + PB_THREADS * u;
      acc[u] = j < s ? lr[j] : 0.0;
    }
    for (int k = 1; k < s; ++k) {
      const double a = lr[k];
      if (a == 0.0) continue;
#pragma unroll
      for (int u = 0; u < PB_J; ++u) {
        const int j = tid + PB_THREADS * u;
        if (j < k) acc[u] += a * D[(int64_t)k * s + j];
      }
    }
#pragma unroll
    for (int u = 0; u < PB_J; ++u) {
      const int j = tid + PB_THREADS * u;
      if (j < s) M[(int64_t)m * s + j] = (T)acc[u];
    }
  }
  // N = U_CC^-1 U_CR (s x r): N[i][m] = sum_{k >= i} Uinv[i][k] U_R[k][m]
  T* N = vals + F.n_off[q];
  for (int i = 0; i < s; ++i) {
    for (int m0 = 0; m0 < r; m0 += PB_THREADS * PB_J) {
      double acc[PB_J];
#pragma unroll
      for (int u = 0; u < PB_J; ++u) acc[u] = 0.0;
      for (int k = i; k < s; ++k) {
        const double a = D[(int64_t)i * s + k];
        if (a == 0.0) continue;
        const double* ur = U + (int64_t)k * (s + r) + s;
#pragma unroll
        for (int u = 0; u < PB_J; ++u) {
          const int m = m0 + tid + PB_THREADS * u;
          if (m < r) acc[u] += a * ur[m];
        }
      }
#pragma unroll
      for (int u = 0; u < PB_J; ++u) {
        const int m = m0 + tid + PB_THREADS * u;
        if (m < r) N[(int64_t)i * r + m] = (T)acc[u];
      }
    }
  }
  // D to the stored precision
  T* Dv = vals + F.d_off[q];
  __syncthreads();
  for (int64_t e = tid; e < (int64_t)s * s; e += PB_THREADS) Dv[e] = (T)D[e];
}

}  // namespace gdsw
