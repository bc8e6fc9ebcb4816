// libgdsw: C ABI (include/gdsw.h) over the sm_100a kernels of the rGDSW
// solve path. Host-side orchestration only; kernels live in the .cuh files.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/gdsw.h"
#include "coarse.cuh"
#include "coarse_factor.cuh"
#include "common.cuh"
#include "dist.cuh"
#include "extension.cuh"
#include "fastilu.cuh"
#include "krylov.cuh"
#include "prof.cuh"
#include "sparse.cuh"
#include "tristream.cuh"
#include "lu_numeric.cuh"

using namespace gdsw;

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return GDSW_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GDSW_E_CUDA;
  }
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline size_t esize(int dtype) { return dtype == GDSW_F32 ? 4 : 8; }

template <typename F>
void with_dtype(int dtype, F&& f) {
  if (dtype == GDSW_F64) f(double{});
  else if (dtype == GDSW_F32) f(float{});
  else throw Error(E_VALUE, "unknown dtype");
}

std::vector<int64_t> vec(const int64_t* p, size_t n) {
  require(n == 0 || p != nullptr, "missing descriptor array");
  return std::vector<int64_t>(p, p + n);
}

constexpr int TB = 256;

// process-wide generations: a captured graph is tied to the (operator,
// preconditioner) objects AND their generation, so an object freed and
// reallocated at the same address never matches a stale graph
uint64_t next_generation() {
  static std::atomic<uint64_t> g{0};
  return ++g;
}

// GDSW_L2HINT=1 enables L2 evict_last hints on the Jacobi iterates
// (measured slower on B200 at C2: off by default)
bool env_flag(const char* name) {
  const char* e = std::getenv(name);
  return e && e[0] == '1';
}

bool l2_hints_enabled() { return env_flag("GDSW_L2HINT"); }

}  // namespace

// ===========================================================================
// device CSR operator
// ===========================================================================
struct gdsw_csr {
  int64_t nrows = 0, ncols = 0, nnz = 0;
  uint64_t gen = next_generation();
  int dtype = GDSW_F64;
  SellPattern pat;
  DBuf<char> csr_val;   // values in CSR order (A.values indexing for setup gathers)
  DBuf<char> sell_val;  // values in SELL order (SpMV)
  void refresh_sell() {
    with_dtype(dtype, [&](auto tag) {
      using T = decltype(tag);
      k_csr_to_sell<T, T><<<grid_for(nrows, TB), TB>>>(
          (int32_t)nrows, pat.csr_ptr.p, pat.slice_off.p, (const T*)csr_val.p, (T*)sell_val.p, 0,
          (T*)nullptr, pat.uw);
      CK_LAUNCH();
    });
    CK(cudaDeviceSynchronize());
  }
};

namespace {
template <typename T>
void spmv_T(const gdsw_csr* a, const T* x, const T* yin, T* y, int mode, double alpha, double beta,
            cudaStream_t s) {
  if (a->nrows == 0) return;
  const int f = a->pat.fmt();
  if (f == SELL_MASK)
    k_sell_spmv<T, SELL_MASK><<<grid_for(a->nrows, TB), TB, 0, s>>>(a->pat.view(), (const T*)a->sell_val.p, x,
                                                                   yin, y, mode, (T)alpha, (T)beta);
  else if (f == SELL_D16)
    k_sell_spmv<T, SELL_D16><<<grid_for(a->nrows, TB), TB, 0, s>>>(a->pat.view(), (const T*)a->sell_val.p, x,
                                                                  yin, y, mode, (T)alpha, (T)beta);
  else
    k_sell_spmv<T, SELL_COL32><<<grid_for(a->nrows, TB), TB, 0, s>>>(a->pat.view(), (const T*)a->sell_val.p, x,
                                                                    yin, y, mode, (T)alpha, (T)beta);
  CK_LAUNCH();
}
}  // namespace

extern "C" {

const char* gdsw_last_error(void) { return g_err.c_str(); }
int gdsw_abi_version(void) { return GDSW_ABI_VERSION; }

int gdsw_csr_create(gdsw_csr** out, int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                    const int64_t* col_idx, const void* values, int dtype) {
  return guarded([&] {
    require(nrows >= 0 && ncols >= 0, "negative matrix dimension");
    require(nrows < INT32_MAX && ncols < INT32_MAX, "matrix too large for the int32 layout");
    auto a = std::make_unique<gdsw_csr>();
    a->nrows = nrows;
    a->ncols = ncols;
    a->nnz = row_ptr[nrows];
    a->dtype = dtype;
    std::vector<int64_t> zero(nrows, 0);
    a->pat.build(nrows, row_ptr, col_idx, zero.data(), 0);
    a->csr_val.alloc(a->nnz * esize(dtype));
    if (a->nnz)
      CK(cudaMemcpy(a->csr_val.p, values, a->nnz * esize(dtype), cudaMemcpyHostToDevice));
    a->sell_val.alloc(std::max<int64_t>(a->pat.padded, 1) * esize(dtype));
    CK(cudaMemset(a->sell_val.p, 0, a->sell_val.n));
    a->refresh_sell();
    *out = a.release();
  });
}

int gdsw_csr_set_values(gdsw_csr* a, const void* values) {
  return guarded([&] {
    if (a->nnz)
      CK(cudaMemcpy(a->csr_val.p, values, a->nnz * esize(a->dtype), cudaMemcpyHostToDevice));
    a->refresh_sell();
  });
}

int gdsw_csr_spmv(const gdsw_csr* a, const void* x, void* y, double alpha, double beta,
                  void* stream) {
  return guarded([&] {
    int mode = (alpha == 1.0 && beta == 0.0) ? 0 : 2;
    ProfScope ps("spmv", S(stream), (double)a->nnz * (esize(a->dtype) + a->pat.idx_bytes_per_entry()) +
                                        a->nrows * a->pat.idx_bytes_per_row() +
                                        2.0 * a->nrows * esize(a->dtype));
    with_dtype(a->dtype, [&](auto tag) {
      using T = decltype(tag);
      spmv_T<T>(a, (const T*)x, (const T*)y, (T*)y, mode, alpha, beta, S(stream));
    });
  });
}

int gdsw_csr_destroy(gdsw_csr* a) {
  delete a;
  return GDSW_OK;
}

}  // extern "C"

// ===========================================================================
// symbolic plan
// ===========================================================================
struct gdsw_plan {
  std::atomic<int> refs{1};
  int64_t n = 0, n_loc = 0, nnz_l = 0, nnz_u = 0;
  int32_t n_sub = 0;
  int method = GDSW_FAST_ILU;
  std::vector<int64_t> h_sub_ptr, h_l_ptr, h_u_ptr;
  DBuf<int32_t> sub_ptr, gmap;
  DBuf<int64_t> l_ptr, u_ptr;
  DBuf<int32_t> l_col, u_col;
  // host level schedules (block-local rows): streamed SpTRSV and numeric LU
  std::vector<int64_t> h_llev_sub, h_llev_ptr, h_llev_rows, h_ulev_sub, h_ulev_ptr, h_ulev_rows;
  // numeric LU on the GPU: permuted block pattern of A + device schedules
  bool has_ab = false;
  int32_t n_max = 0;
  DBuf<int64_t> ab_ptr, ab_src;
  DBuf<int32_t> ab_idx, l_idx32, u_idx32, lu_lev_sub, lu_lev_ptr, lu_lev_rows;
  LuDev lu_dev() const {
    return LuDev{sub_ptr.p, l_ptr.p, l_idx32.p, u_ptr.p, u_idx32.p, lu_lev_sub.p, lu_lev_ptr.p,
                 lu_lev_rows.p, ab_ptr.p, ab_idx.p, ab_src.p, n_max};
  }
  std::vector<int64_t> row_add;  // block row offset per concatenated row
  std::vector<int64_t> h_l_idx, h_u_idx;
  SellPattern l_sell, u_sell;    // Jacobi layouts (U without its diagonal)
  bool sell_ready = false;
  DBuf<int32_t> sc_ptr, sc_pos;
  std::vector<int32_t> h_sc_ptr, h_sc_pos;
  // FastILU plan
  bool fastilu = false;
  DBuf<int64_t> a_of, fi_ptr;
  DBuf<int32_t> fi_pl, fi_pu, fi_ldiag;
  int64_t n_res = 0;
  std::vector<int64_t> h_res_sub_ptr;
  DBuf<int64_t> res_sub_ptr, res_a, res_ptr;
  DBuf<int32_t> res_pl, res_pu, res_tl, res_tu;
  void ensure_sell() {
    if (sell_ready) return;
    // the sweeps take one column format for both factors: slot masks only
    // when both patterns allow them
    int32_t wl = 0, wu = 0;
    const bool mk = SellPattern::mask_feasible(n_loc, h_l_ptr.data(), h_l_idx.data(), row_add.data(), 0, &wl) &&
                    SellPattern::mask_feasible(n_loc, h_u_ptr.data(), h_u_idx.data(), row_add.data(), 1, &wu);
    l_sell.build(n_loc, h_l_ptr.data(), h_l_idx.data(), row_add.data(), 0, mk);
    u_sell.build(n_loc, h_u_ptr.data(), h_u_idx.data(), row_add.data(), 1, mk);
    require(l_sell.masked == u_sell.masked, "factor layouts disagree");
    sell_ready = true;
  }


  FastIluDev fastilu_dev() const {
    return FastIluDev{nnz_l, nnz_u, a_of.p, fi_ptr.p, fi_pl.p, fi_pu.p, fi_ldiag.p};
  }
  FastIluResDev fastilu_res_dev() const {
    return FastIluResDev{n_res, res_a.p, res_ptr.p, res_pl.p, res_pu.p, res_tl.p, res_tu.p};
  }
};

// coarse structure of one numeric preconditioner (the coarse basis pattern
// depends on the null space, so it is built in the numeric phase like the
// reference's harmonic_extension, coarse_space.py:130-179)
struct CoarsePlan {
  int64_t n = 0;
  int32_t n_sub = 0;
  int32_t n_c = 0, K = 0;
  int64_t n_gamma = 0, panel_entries = 0, n_int_total = 0;
  std::vector<double> h_pgr_val, h_pgt_val;
  DBuf<int64_t> pgr_ptr, pgt_ptr, panel_off;
  DBuf<int32_t> pgr_col, pgt_row, pi_sub, pi_row, n_int, col_ptr, col_ids, colsub, int_ptr,
      int_rows, clist_ptr, clist;
  std::vector<int64_t> h_panel_off, h_n_int, h_col_ptr;
  // extension
  int32_t n_chunks = 0;
  int64_t n_partial = 0;
  DBuf<int32_t> chunk_sub, chunk_row0, chunk_nrow, sub_chunk0;
  DBuf<int32_t> ch_g, ch_y0, ch_ny;  // per (chunk, thread): interior row, first / number of local contributions
  DBuf<int64_t> chunk_poff;
  DBuf<int64_t> aii_ptr, aii_src, aii_diag, aig_ptr, aig_src;
  DBuf<int32_t> aii_col, aig_col;
  DBuf<int64_t> pgam_ptr;
  DBuf<int32_t> pgam_col;
  DBuf<double> pgam_val;

  ProlongDev prolong() const {
    ProlongDev p{};
    p.enabled = 1;
    p.pg_ptr = pgr_ptr.p;
    p.pg_col = pgr_col.p;
    p.pi_sub = pi_sub.p;
    p.pi_row = pi_row.p;
    p.panel_off = panel_off.p;
    p.n_int = n_int.p;
    p.col_ptr = col_ptr.p;
    p.col_ids = col_ids.p;
    return p;
  }
  // chunked restriction/prolongation tables
  DBuf<int64_t> cpart_ptr, cpart_idx;
  int64_t n_cpart = 0;
  DBuf<int32_t> gamma32;
  ChunkDev chunk_dev() const {
    return ChunkDev{chunk_sub.p, chunk_row0.p, chunk_nrow.p, chunk_poff.p, int_ptr.p,  int_rows.p,
                    n_int.p,     col_ptr.p,    col_ids.p,    panel_off.p,  ch_g.p,     ch_y0.p,
                    ch_ny.p};
  }
  RestrictDev restrict_dev() const {
    return RestrictDev{n_c,       colsub.p,   col_ptr.p,    panel_off.p, n_int.p,
                       int_ptr.p, int_rows.p, pgt_ptr.p,    pgt_row.p,   clist_ptr.p,
                       clist.p};
  }
};

namespace {
void plan_release(gdsw_plan* p) {
  if (p && --p->refs == 0) delete p;
}

void build_local(gdsw_plan* P, const gdsw_local_desc* d) {
  P->n = d->n;
  P->n_sub = d->n_sub;
  P->method = d->method;
  P->n_loc = d->n_loc;
  require(d->n_sub >= 1, "plan needs at least one subdomain");
  require(d->n < INT32_MAX && d->n_loc < INT32_MAX, "problem too large for the int32 layout");
  const int32_t ns = d->n_sub;
  P->h_sub_ptr = vec(d->sub_ptr, ns + 1);
  require(P->h_sub_ptr[ns] == d->n_loc, "sub_ptr does not match n_loc");
  P->sub_ptr.upload(to_i32(P->h_sub_ptr.data(), ns + 1));
  P->gmap.upload(to_i32(d->gmap, d->n_loc));
  P->h_l_ptr = vec(d->l_ptr, d->n_loc + 1);
  P->h_u_ptr = vec(d->u_ptr, d->n_loc + 1);
  P->nnz_l = P->h_l_ptr[d->n_loc];
  P->nnz_u = P->h_u_ptr[d->n_loc];
  P->h_l_idx = vec(d->l_idx, P->nnz_l);
  P->h_u_idx = vec(d->u_idx, P->nnz_u);
  P->row_add.assign(d->n_loc, 0);
  for (int32_t s = 0; s < ns; ++s)
    for (int64_t k = P->h_sub_ptr[s]; k < P->h_sub_ptr[s + 1]; ++k) P->row_add[k] = P->h_sub_ptr[s];
  // CSR with absolute columns (level-set path, downloads)
  {
    std::vector<int32_t> lc(P->nnz_l), uc(P->nnz_u);
    for (int64_t k = 0; k < d->n_loc; ++k) {
      for (int64_t p = P->h_l_ptr[k]; p < P->h_l_ptr[k + 1]; ++p) lc[p] = (int32_t)(P->h_l_idx[p] + P->row_add[k]);
      for (int64_t p = P->h_u_ptr[k]; p < P->h_u_ptr[k + 1]; ++p) uc[p] = (int32_t)(P->h_u_idx[p] + P->row_add[k]);
    }
    P->l_ptr.upload(P->h_l_ptr);
    P->u_ptr.upload(P->h_u_ptr);
    P->l_col.upload(lc);
    P->u_col.upload(uc);
  }
  // level schedules (block-local rows)
  {
    const int64_t nl = d->llev_sub[ns], nu = d->ulev_sub[ns];
    P->h_llev_sub = vec(d->llev_sub, ns + 1);
    P->h_llev_ptr = vec(d->llev_ptr, nl + 1);
    P->h_llev_rows = vec(d->llev_rows, d->n_loc);
    P->h_ulev_sub = vec(d->ulev_sub, ns + 1);
    P->h_ulev_ptr = vec(d->ulev_ptr, nu + 1);
    P->h_ulev_rows = vec(d->ulev_rows, d->n_loc);
  }
  // owner-computes scatter: positions grouped by global row, ascending block
  {
    std::vector<int64_t> gm = vec(d->gmap, d->n_loc);
    std::vector<int32_t> cnt(d->n + 1, 0), pos(d->n_loc);
    for (int64_t k = 0; k < d->n_loc; ++k) {
      require(gm[k] >= 0 && gm[k] < d->n, "gmap entry out of range");
      cnt[gm[k] + 1]++;
    }
    for (int64_t g = 0; g < d->n; ++g) cnt[g + 1] += cnt[g];
    std::vector<int32_t> off(cnt.begin(), cnt.end() - 1);
    for (int64_t k = 0; k < d->n_loc; ++k) pos[off[gm[k]]++] = (int32_t)k;
    P->sc_ptr.upload(cnt);
    P->sc_pos.upload(pos);
    P->h_sc_ptr = std::move(cnt);
    P->h_sc_pos = std::move(pos);
  }
  if (d->method == GDSW_FAST_ILU) {
    P->fastilu = true;
    const int64_t ne = P->nnz_l + P->nnz_u;
    P->a_of.upload(vec(d->a_of, ne));
    std::vector<int64_t> fptr = vec(d->fi_ptr, ne + 1);
    P->fi_ptr.upload(fptr);
    P->fi_pl.upload(to_i32(d->fi_pl, fptr[ne]));
    P->fi_pu.upload(to_i32(d->fi_pu, fptr[ne]));
    // U position of the diagonal of column j for every L entry
    std::vector<int32_t> ldiag(P->nnz_l);
    for (int64_t k = 0; k < d->n_loc; ++k)
      for (int64_t p = P->h_l_ptr[k]; p < P->h_l_ptr[k + 1]; ++p)
        ldiag[p] = (int32_t)P->h_u_ptr[P->h_l_idx[p] + P->row_add[k]];
    P->fi_ldiag.upload(ldiag);
    P->n_res = d->n_res;
    if (d->n_res > 0) {
      P->h_res_sub_ptr = vec(d->res_sub_ptr, ns + 1);
      P->res_sub_ptr.upload(P->h_res_sub_ptr);
      P->res_a.upload(vec(d->res_a, d->n_res));
      std::vector<int64_t> rptr = vec(d->res_ptr, d->n_res + 1);
      P->res_ptr.upload(rptr);
      P->res_pl.upload(to_i32(d->res_pl, rptr[d->n_res]));
      P->res_pu.upload(to_i32(d->res_pu, rptr[d->n_res]));
      P->res_tl.upload(to_i32(d->res_tl, d->n_res));
      P->res_tu.upload(to_i32(d->res_tu, d->n_res));
    }
    P->ensure_sell();
  }
}

void build_coarse(CoarsePlan* P, const gdsw_plan* L, const gdsw_coarse_desc* c) {
  P->n = L->n;
  P->n_sub = L->n_sub;
  const int32_t ns = P->n_sub;
  P->n_c = c->n_c;
  P->n_gamma = c->n_gamma;
  std::vector<int64_t> grows = vec(c->gamma_rows, c->n_gamma);
  std::vector<int64_t> pg_ptr = vec(c->pg_ptr, c->n_gamma + 1);
  const int64_t npg = pg_ptr[c->n_gamma];
  std::vector<int64_t> pg_col = vec(c->pg_col, npg);
  std::vector<double> pg_val(c->pg_val, c->pg_val + npg);
  // prolongation rows: CSR over all vector rows (interface rows only)
  {
    std::vector<int64_t> ptr(P->n + 1, 0);
    for (int64_t t = 0; t < c->n_gamma; ++t) ptr[grows[t] + 1] = pg_ptr[t + 1] - pg_ptr[t];
    for (int64_t g = 0; g < P->n; ++g) ptr[g + 1] += ptr[g];
    std::vector<int32_t> col(npg);
    P->h_pgr_val.assign(npg, 0.0);
    for (int64_t t = 0; t < c->n_gamma; ++t)
      for (int64_t q = pg_ptr[t], o = ptr[grows[t]]; q < pg_ptr[t + 1]; ++q, ++o) {
        col[o] = (int32_t)pg_col[q];
        P->h_pgr_val[o] = pg_val[q];
      }
    P->pgr_ptr.upload(ptr);
    P->pgr_col.upload(col);
  }
  // restriction: Phi_Gamma^T, coarse-major, ascending interface row
  {
    std::vector<int64_t> ptr(c->n_c + 1, 0);
    for (int64_t q = 0; q < npg; ++q) ptr[pg_col[q] + 1]++;
    for (int32_t k = 0; k < c->n_c; ++k) ptr[k + 1] += ptr[k];
    std::vector<int64_t> off(ptr.begin(), ptr.end() - 1);
    std::vector<int32_t> row(npg);
    P->h_pgt_val.assign(npg, 0.0);
    for (int64_t t = 0; t < c->n_gamma; ++t)
      for (int64_t q = pg_ptr[t]; q < pg_ptr[t + 1]; ++q) {
        int64_t o = off[pg_col[q]]++;
        row[o] = (int32_t)grows[t];
        P->h_pgt_val[o] = pg_val[q];
      }
    P->pgt_ptr.upload(ptr);
    P->pgt_row.upload(row);
  }
  // Phi_Gamma by gamma position for the extension right-hand side
  P->pgam_ptr.upload(pg_ptr);
  P->pgam_col.upload(to_i32(pg_col.data(), npg));
  P->pgam_val.upload(pg_val);
  // interior panels
  std::vector<int64_t> iptr = vec(c->int_ptr, ns + 1);
  P->n_int_total = iptr[ns];
  std::vector<int64_t> irows = vec(c->int_rows, P->n_int_total);
  std::vector<int64_t> cptr = vec(c->col_ptr, ns + 1);
  P->K = (int32_t)cptr[ns];
  std::vector<int64_t> cids = vec(c->col_ids, P->K);
  P->h_col_ptr = cptr;
  P->h_n_int.assign(ns, 0);
  P->h_panel_off.assign(ns + 1, 0);
  std::vector<int32_t> colsub(P->K);
  for (int32_t s = 0; s < ns; ++s) {
    P->h_n_int[s] = iptr[s + 1] - iptr[s];
    require(cptr[s + 1] - cptr[s] <= EXT_MAXK, "too many coarse columns touch one subdomain");
    P->h_panel_off[s + 1] = P->h_panel_off[s] + P->h_n_int[s] * (cptr[s + 1] - cptr[s]);
    for (int64_t k = cptr[s]; k < cptr[s + 1]; ++k) colsub[k] = s;
  }
  P->panel_entries = P->h_panel_off[ns];
  P->panel_off.upload(P->h_panel_off);
  P->n_int.upload(to_i32(P->h_n_int.data(), ns));
  P->col_ptr.upload(to_i32(cptr.data(), ns + 1));
  P->col_ids.upload(to_i32(cids.data(), P->K));
  P->colsub.upload(colsub);
  P->int_ptr.upload(to_i32(iptr.data(), ns + 1));
  P->int_rows.upload(to_i32(irows.data(), irows.size()));
  {
    std::vector<int32_t> pis(P->n, -1), pir(P->n, 0);
    for (int32_t s = 0; s < ns; ++s)
      for (int64_t t = iptr[s]; t < iptr[s + 1]; ++t) {
        pis[irows[t]] = s;
        pir[irows[t]] = (int32_t)(t - iptr[s]);
      }
    P->pi_sub.upload(pis);
    P->pi_row.upload(pir);
  }
  {  // coarse column -> panel columns (ascending subdomain)
    std::vector<int32_t> cnt(c->n_c + 1, 0), lst(P->K);
    for (int32_t k = 0; k < P->K; ++k) cnt[cids[k] + 1]++;
    for (int32_t k = 0; k < c->n_c; ++k) cnt[k + 1] += cnt[k];
    std::vector<int32_t> off(cnt.begin(), cnt.end() - 1);
    for (int32_t k = 0; k < P->K; ++k) lst[off[cids[k]]++] = k;
    P->clist_ptr.upload(cnt);
    P->clist.upload(lst);
  }
  // extension chunks (<= EXT_THREADS rows, never straddling a subdomain)
  {
    std::vector<int32_t> csub, crow0, cnrow, sc0(ns + 1, 0);
    std::vector<int64_t> cpoff;
    int64_t poff = 0;
    for (int32_t s = 0; s < ns; ++s) {
      sc0[s] = (int32_t)csub.size();
      int64_t k = cptr[s + 1] - cptr[s];
      for (int64_t r0 = 0; r0 < P->h_n_int[s]; r0 += EXT_THREADS) {
        csub.push_back(s);
        crow0.push_back((int32_t)r0);
        cnrow.push_back((int32_t)std::min<int64_t>(EXT_THREADS, P->h_n_int[s] - r0));
        cpoff.push_back(poff);
        poff += k;
      }
    }
    sc0[ns] = (int32_t)csub.size();
    P->n_chunks = (int32_t)csub.size();
    P->n_partial = std::max<int64_t>(poff, 1);
    {  // flat per-thread prolongation tables: the row and its first local
       // contribution without the int_rows -> sc_ptr -> sc_pos chain
      const size_t nt = std::max<size_t>((size_t)P->n_chunks * CH_THREADS, 1);
      std::vector<int32_t> fg(nt, 0), fy(nt, -1), fn(nt, 0);
      for (int32_t ch = 0; ch < P->n_chunks; ++ch)
        for (int32_t t = 0; t < cnrow[ch]; ++t) {
          const int32_t s = csub[ch];
          const int32_t g = (int32_t)irows[iptr[s] + crow0[ch] + t];
          const size_t q = (size_t)ch * CH_THREADS + t;
          fg[q] = g;
          const int32_t a0 = L->h_sc_ptr.empty() ? 0 : L->h_sc_ptr[g];
          const int32_t a1 = L->h_sc_ptr.empty() ? 0 : L->h_sc_ptr[g + 1];
          fn[q] = a1 - a0;
          fy[q] = a1 > a0 ? L->h_sc_pos[a0] : -1;
        }
      P->ch_g.upload(fg);
      P->ch_y0.upload(fy);
      P->ch_ny.upload(fn);
    }
    P->chunk_sub.upload(csub);
    P->chunk_row0.upload(crow0);
    P->chunk_nrow.upload(cnrow);
    P->chunk_poff.upload(cpoff);
    P->sub_chunk0.upload(sc0);
    // coarse column -> the chunk partials of every panel column mapping to it
    // (ascending subdomain, then ascending chunk)
    std::vector<std::vector<int64_t>> parts(c->n_c);
    for (int32_t s = 0; s < ns; ++s)
      for (int64_t k = cptr[s]; k < cptr[s + 1]; ++k)
        for (int32_t ch = sc0[s]; ch < sc0[s + 1]; ++ch)
          parts[cids[k]].push_back(cpoff[ch] + (k - cptr[s]));
    std::vector<int64_t> pp(c->n_c + 1, 0), pidx;
    for (int32_t k = 0; k < c->n_c; ++k) {
      pidx.insert(pidx.end(), parts[k].begin(), parts[k].end());
      pp[k + 1] = (int64_t)pidx.size();
    }
    P->n_cpart = (int64_t)pidx.size();
    P->cpart_ptr.upload(pp);
    if (pidx.empty()) pidx.push_back(0);
    P->cpart_idx.upload(pidx);
    P->gamma32.upload(to_i32(grows.data(), grows.size()));
  }
  {
    std::vector<int64_t> aptr = vec(c->aii_ptr, P->n_int_total + 1);
    int64_t na = aptr[P->n_int_total];
    std::vector<int64_t> acol = vec(c->aii_col, na);
    std::vector<int64_t> diag(P->n_int_total, -1);
    for (int32_t s = 0; s < ns; ++s)
      for (int64_t t = iptr[s]; t < iptr[s + 1]; ++t)
        for (int64_t p = aptr[t]; p < aptr[t + 1]; ++p)
          if (acol[p] == t - iptr[s]) diag[t] = p;
    for (int64_t t = 0; t < P->n_int_total; ++t)
      require(diag[t] >= 0, "interior block has a structurally missing diagonal");
    P->aii_ptr.upload(aptr);
    P->aii_col.upload(to_i32(acol.data(), na));
    P->aii_src.upload(vec(c->aii_src, na));
    P->aii_diag.upload(diag);
    std::vector<int64_t> gptr = vec(c->aig_ptr, P->n_int_total + 1);
    int64_t ng = gptr[P->n_int_total];
    P->aig_ptr.upload(gptr);
    P->aig_col.upload(to_i32(c->aig_col, ng));
    P->aig_src.upload(vec(c->aig_src, ng));
  }
}
}  // namespace

extern "C" int gdsw_plan_create(gdsw_plan** out, const gdsw_local_desc* local) {
  return guarded([&] {
    auto P = std::make_unique<gdsw_plan>();
    build_local(P.get(), local);
    CK(cudaDeviceSynchronize());
    *out = P.release();
  });
}

extern "C" int gdsw_plan_destroy(gdsw_plan* p) {
  plan_release(p);
  return GDSW_OK;
}

// ===========================================================================
// numeric preconditioner
// ===========================================================================
// device copy of a supernodal partitioned inverse (coarse_factor.cuh)
struct FactorBuf {
  bool on = false;
  DBuf<int32_t> sn_s, sn_r, col_ptr, col_ids, row_ptr, row_ids, in_ptr, in_idx, out_ptr, out_idx;
  DBuf<int64_t> d_off, m_off, n_off;
  DBuf<int2> df_tasks;                    // tiles in dependency order
  DBuf<int32_t> parent, child_ptr, child_idx, fwd_need, bwd_need, ready;
  DBuf<unsigned> ticket;
  int32_t n_fwd_tasks = 0, n_df_tasks = 0, n_sn = 0, df_grid = 0;
  int nt = CF_NT_COARSE;                  // dataflow CTA size (coarse_factor.cuh)
  size_t df_smem = 0;
  DBuf<char> vals, ybuf, cbuf, fcm;
  DBuf<int64_t> f_off;
  DBuf<int32_t> cm_list;
  int32_t n_cm = 0;
  int64_t bytes = 0, n_launch = 0;
  CoarseFactorDev dev() const {
    return CoarseFactorDev{parent.p, child_ptr.p, child_idx.p, fwd_need.p, bwd_need.p,
                           sn_s.p, sn_r.p, col_ptr.p, col_ids.p, row_ptr.p, row_ids.p,
                           d_off.p, m_off.p, n_off.p, in_ptr.p, in_idx.p, out_ptr.p, out_idx.p, f_off.p};
  }
};

struct gdsw_precond {
  gdsw_plan* plan = nullptr;
  std::unique_ptr<CoarsePlan> cp;
  gdsw_dist* dist = nullptr;         // sharded layout (not owned)
  DBuf<double> part_ext, recv_ext;   // reverse-halo partial sums (ext-local)
  DBuf<double> red64;                // coarse rhs reduction scratch
  int dtype = GDSW_F64;
  size_t es = 8;
  int iters = 5;
  bool has_factors = false, jacobi_ready = false, has_phi = false, has_ainv = false;
  DBuf<char> lval, uval;           // CSR order
  DBuf<char> lsell, usell, udiag;  // Jacobi copies
  TriStream tstream;               // streamed-SpTRSV layout (exact / ILU(k))
  bool stream_built = false, stream_vals_ready = false;
  DBuf<double> panel64;
  DBuf<char> panel32;              // f32 copy when dtype == F32
  DBuf<char> pgr_val, pgt_val, ainv;
  // factored coarse solve (coarse_factor.cuh); used instead of ainv when set
  FactorBuf cf;
  // factored exact-LU local solves (same kernels, every block in one batch)
  FactorBuf lf;
  DBuf<char> xb, x1, x2, x3, pdot, cu, cv;
  // recursive: a GMRES solve holds it for its whole duration and its
  // eager passes re-enter precond_apply
  std::recursive_mutex mu;
  cudaEvent_t last = nullptr;
  // side stream for the coarse restriction + solve, overlapped with the
  // local solves (fork/join by events; single-GPU path)
  cudaStream_t side = nullptr, cap = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  struct ApplyGraph {
    const double* r;
    double* z;
    cudaStream_t s;
    cudaGraphExec_t exec;
    int64_t kernels;
  };
  std::vector<ApplyGraph> graphs;
  uint64_t gen = next_generation();  // renewed whenever graphs holding its buffers go stale
  void drop_graphs() {
    for (auto& ag : graphs)
      if (ag.exec) cudaGraphExecDestroy(ag.exec);
    graphs.clear();
    gen = next_generation();
  }
  ~gdsw_precond() {
    drop_graphs();
    if (last) cudaEventDestroy(last);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
    if (cap) cudaStreamDestroy(cap);
    plan_release(plan);
  }
  const void* panel() const { return dtype == GDSW_F32 ? (const void*)panel32.p : (const void*)panel64.p; }


  void ensure_stream_vals() {
    if (stream_vals_ready) return;
    gdsw_plan* P = plan;
    if (!stream_built) {
      TriStream::Fac L{&P->h_l_ptr, &P->h_l_idx, &P->h_llev_sub, &P->h_llev_ptr, &P->h_llev_rows, 0};
      TriStream::Fac U{&P->h_u_ptr, &P->h_u_idx, &P->h_ulev_sub, &P->h_ulev_ptr, &P->h_ulev_rows, 1};
      tstream.build(P->n_sub, P->h_sub_ptr, L, U, (int)es, P->method != GDSW_EXACT_LU);
      stream_built = true;
    }
    with_dtype(dtype, [&](auto tag) {
      using T = decltype(tag);
      if (tstream.n_place) {
        k_stream_place<T><<<grid_for(tstream.n_place, 8), dim3(32, 8)>>>(
            tstream.n_place, tstream.pl_src.p, tstream.pl_dst.p, tstream.pl_len.p, tstream.pl_stride.p,
            (const T*)lval.p, (const T*)uval.p, P->nnz_l, (T*)tstream.bytes.p);
        CK_LAUNCH();
      }
    });
    CK(cudaDeviceSynchronize());
    stream_vals_ready = true;
  }

  void ensure_jacobi() {
    if (jacobi_ready) return;
    gdsw_plan* P = plan;
    P->ensure_sell();
    lsell.alloc(std::max<int64_t>(P->l_sell.padded, 1) * es);
    usell.alloc(std::max<int64_t>(P->u_sell.padded, 1) * es);
    udiag.alloc(std::max<int64_t>(P->n_loc, 1) * es);
    CK(cudaMemset(lsell.p, 0, lsell.n));
    CK(cudaMemset(usell.p, 0, usell.n));
    with_dtype(dtype, [&](auto tag) {
      using T = decltype(tag);
      k_csr_to_sell<T, T><<<grid_for(P->n_loc, TB), TB>>>((int32_t)P->n_loc, P->l_sell.csr_ptr.p,
                                                         P->l_sell.slice_off.p, (const T*)lval.p,
                                                         (T*)lsell.p, 0, (T*)nullptr, P->l_sell.uw);
      CK_LAUNCH();
      k_csr_to_sell<T, T><<<grid_for(P->n_loc, TB), TB>>>((int32_t)P->n_loc, P->u_sell.csr_ptr.p,
                                                         P->u_sell.slice_off.p, (const T*)uval.p,
                                                         (T*)usell.p, 1, (T*)udiag.p, P->u_sell.uw);
      CK_LAUNCH();
    });
    CK(cudaDeviceSynchronize());
    jacobi_ready = true;
  }
};

namespace {

// FastSpTRSV: `iters` Jacobi iterates on L then U; returns the buffer
// holding the block solutions

template <typename T, bool HINT, int FMT, bool UNI>
T* jacobi_solve(gdsw_precond* m, const double* r, int iters, cudaStream_t s) {
  gdsw_plan* P = m->plan;
  const int32_t n = (int32_t)P->n_loc;
  T* B = (T*)m->xb.p;
  T* X1 = (T*)m->x1.p;
  T* X2 = (T*)m->x2.p;
  SellDev L = P->l_sell.view(), U = P->u_sell.view();
  const unsigned g = grid_for(n, TB);
  // alternate the sweeps' direction (GDSW_SWEEP_ALT=0: all forward)
  static const bool alt = [] {
    const char* e = std::getenv("GDSW_SWEEP_ALT");
    return !(e && e[0] == '0');
  }();
  int dir = 0;
  auto next_dir = [&] {
    const int d = dir;
    if (alt) dir ^= 1;
    return d;
  };
  const double cb = P->l_sell.idx_bytes_per_entry();  // stored column bytes per entry
  const double rb = P->l_sell.idx_bytes_per_row();    // row length / slot mask bytes
  const double lbytes = (double)P->nnz_l * (sizeof(T) + cb) + n * (rb + 3 * sizeof(T));
  const double ubytes = (double)(P->nnz_u - n) * (sizeof(T) + cb) + n * (rb + 3 * sizeof(T));
  // algorithmic bytes per launch: SELL values+columns once, row lengths,
  // b and x read once (gathers assumed cached), x_new written; the gather
  // variant reads r through gmap (4 + 8 per row, twice for the neighbours'
  // rows which are L2-resident) and writes b as well
  T* F;
  if (iters <= 1) {
    ProfScope ps("gather", s, n * (4.0 + 8.0 + sizeof(T)));
    k_gather<T><<<g, TB, 0, s>>>(n, P->gmap.p, r, B);
    CK_LAUNCH();
    F = B;
  } else {
    {
      ProfScope ps("gather_jacobi_lower", s, lbytes + n * (12.0 - sizeof(T)));
      k_gather_jacobi_lower<T, HINT, FMT, UNI><<<g, TB, 0, s>>>(L, (const T*)m->lsell.p, P->gmap.p, r, B, X1,
                                                                   next_dir());
      CK_LAUNCH();
    }
    T* cur = X1;
    T* oth = X2;
    for (int t = 2; t < iters - 1; ++t) {
      ProfScope ps("jacobi_lower", s, lbytes);
      k_jacobi_lower<T, HINT, FMT, UNI><<<g, TB, 0, s>>>(L, (const T*)m->lsell.p, B, cur, oth, next_dir());
      CK_LAUNCH();
      std::swap(cur, oth);
    }
    if (iters >= 3) {
      // last L iterate fused with U's first iterate y1 = F / diag
      T* X3 = (T*)m->x3.p;
      {
        ProfScope ps("jacobi_lower_diag", s, lbytes + n * 2.0 * sizeof(T));
        k_jacobi_lower_diag<T, HINT, FMT, UNI><<<g, TB, 0, s>>>(L, (const T*)m->lsell.p, B, cur, oth,
                                                (const T*)m->udiag.p, X3, next_dir());
        CK_LAUNCH();
      }
      F = oth;
      T* Gf = X3;
      T* Hf = cur;  // B and cur are free now
      for (int t = 1; t < iters; ++t) {
        ProfScope ps("jacobi_upper", s, ubytes + n * (double)sizeof(T));
        k_jacobi_upper<T, HINT, FMT, UNI><<<g, TB, 0, s>>>(U, (const T*)m->usell.p, (const T*)m->udiag.p, F, Gf, Hf,
                                                                next_dir());
        CK_LAUNCH();
        std::swap(Gf, Hf);
      }
      return Gf;
    }
    F = cur;
  }
  T* G = (F == B) ? X1 : B;
  T* H = (F == X2) ? X1 : X2;
  if (F == X1) { G = B; H = X2; }
  {
    ProfScope ps("diag_solve", s, n * 3.0 * sizeof(T));
    k_diag_solve<T><<<g, TB, 0, s>>>(n, (const T*)m->udiag.p, F, G);
    CK_LAUNCH();
  }
  T* cur = G;
  T* oth = H;
  for (int t = 1; t < iters; ++t) {
    ProfScope ps("jacobi_upper", s, ubytes + n * (double)sizeof(T));
    k_jacobi_upper<T, HINT, FMT, UNI><<<g, TB, 0, s>>>(U, (const T*)m->usell.p, (const T*)m->udiag.p, F, cur, oth,
                                                                next_dir());
    CK_LAUNCH();
    std::swap(cur, oth);
  }
  return cur;
}

template <typename T, typename CT, bool SMEMX, bool FWD, int NW>
void launch_stream_nw(gdsw_precond* m, const double* r, T* y, int32_t ring, size_t smem, cudaStream_t s) {
  static bool attr = [] {
    // dynamic shared memory up to the 227 KB opt-in limit minus the
    // kernel's static buffers (forwarding: 16 KB in fp64)
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, k_trisolve_stream<T, CT, SMEMX, FWD, NW>));
    const int cap = std::min<int>(220 * 1024, 227 * 1024 - (int)fa.sharedSizeBytes);
    CK(cudaFuncSetAttribute(k_trisolve_stream<T, CT, SMEMX, FWD, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            cap));
    return true;
  }();
  (void)attr;
  k_trisolve_stream<T, CT, SMEMX, FWD, NW><<<m->plan->n_sub, 32 * NW + 32, smem, s>>>(
      m->tstream.view(), ring, m->plan->sub_ptr.p, m->plan->gmap.p, r, y);
}

// consumer warps per CTA: 8 when blocks outnumber the SMs (several CTAs
// per SM), else 16 (fewer rows per warp on each level's critical path:
// C2 ILU(0) local solve 0.377 -> 0.303 ms, C3-sized blocks 1.51 -> 1.43 ms);
// GDSW_TS_WARPS=8/16/24 forces
template <typename T, typename CT, bool SMEMX, bool FWD = false>
void launch_stream(gdsw_precond* m, const double* r, T* y, int32_t ring, size_t smem, cudaStream_t s) {
  static const int nw_env = [] {
    const char* e = std::getenv("GDSW_TS_WARPS");
    return e ? std::atoi(e) : 0;
  }();
  const int nw = nw_env ? nw_env : (m->plan->n_sub > num_sms() ? 8 : 16);
  if (nw == 24) launch_stream_nw<T, CT, SMEMX, FWD, 24>(m, r, y, ring, smem, s);
  else if (nw == 16) launch_stream_nw<T, CT, SMEMX, FWD, 16>(m, r, y, ring, smem, s);
  else launch_stream_nw<T, CT, SMEMX, FWD, 8>(m, r, y, ring, smem, s);
}

template <typename T>
T* levelset_solve(gdsw_precond* m, const double* r, cudaStream_t s) {
  gdsw_plan* P = m->plan;
  m->ensure_stream_vals();
  const TriStream& ts = m->tstream;
  // algorithmic bytes: L and U entries once (value + stored column
  // width), U's diagonal, the gather (gmap + r) and the block solution
  ProfScope ps("levelset", s, (double)(P->nnz_l + P->nnz_u - P->n_loc) * (sizeof(T) + ts.csize) +
                                  P->n_loc * (12.0 + 2 * sizeof(T)));
  T* y = (T*)m->x1.p;
  // shared memory per CTA: the iterate goes to shared memory when it
  // leaves a ring of at least 4 chunks
  static const int64_t ring_env = [] {
    const char* e = std::getenv("GDSW_TS_BUDGET_KB");
    return e ? (int64_t)std::atoi(e) * 1024 : (int64_t)0;
  }();
  // measured on B200: the iterate in shared memory beats global/L1 as
  // soon as it fits next to a ring of >= 4 chunks (C1 1.20 -> 0.87 ms,
  // C3-sized blocks 2.11 -> 1.67 ms per solve); prefer a budget that keeps
  // two CTAs per SM; an iterate in global memory wants a mid-size ring
  // (L1 left for its gathers: C2 ILU(0) 0.71 -> 0.60 ms)
  static const int64_t min_chunks_env = [] {
    const char* e = std::getenv("GDSW_TS_MINCHUNKS");
    return e ? (int64_t)std::atoi(e) : (int64_t)0;
  }();
  // ring depth: at least 3 chunks
  const int64_t min_chunks = min_chunks_env ? min_chunks_env : 3;
  const int64_t xs = ts.max_rows * (int64_t)sizeof(T);
  const int64_t need = xs + min_chunks * ts.chunk_max;
  // more blocks than SMs: three CTAs per SM when the iterate and a 3-chunk
  // ring fit in 72 KB (512 C3 blocks: 3.43 -> 3.26 ms per solve)
  int64_t budget = need <= 72 * 1024 && P->n_sub > num_sms()
                       ? 72 * 1024
                       : (need <= 110 * 1024 ? 110 * 1024 : (need <= 220 * 1024 ? 220 * 1024 : 160 * 1024));
  if (ring_env) budget = ring_env;
  const bool smx = budget - xs >= min_chunks * ts.chunk_max && !env_flag("GDSW_TS_XGLOBAL");
  int64_t ring = std::max<int64_t>(2LL * ts.chunk_max, ((smx ? budget - xs : budget) & ~int64_t(15)));
  // forwarding buffers (2 x TR_FWD static values) when the iterate stays in
  // global memory
  if (!smx && ts.fwd) ring = std::min<int64_t>(ring, (220 * 1024 - 2 * TR_FWD * (int64_t)sizeof(T)) & ~int64_t(15));
  const size_t smem = (size_t)ring + (smx ? (size_t)xs : 0);
  require(smem <= 220 * 1024, "streamed SpTRSV chunk too large");
  // forwarding slots: only with the iterate in global memory; the static
  // forwarding buffers (2 x TR_FWD values) come out of the budget
  const bool fwd = ts.fwd && !smx;
  if (fwd) require(smem + 2 * TR_FWD * sizeof(T) <= 220 * 1024 && ring >= 2LL * ts.chunk_max,
                   "streamed SpTRSV chunk too large");
  if (ts.csize == 2) {
    if (smx) launch_stream<T, uint16_t, true>(m, r, y, (int32_t)ring, smem, s);
    else if (fwd) launch_stream<T, uint16_t, false, true>(m, r, y, (int32_t)ring, smem, s);
    else launch_stream<T, uint16_t, false>(m, r, y, (int32_t)ring, smem, s);
  } else {
    if (smx) launch_stream<T, int32_t, true>(m, r, y, (int32_t)ring, smem, s);
    else if (fwd) launch_stream<T, int32_t, false, true>(m, r, y, (int32_t)ring, smem, s);
    else launch_stream<T, int32_t, false>(m, r, y, (int32_t)ring, smem, s);
  }
  CK_LAUNCH();
  return y;
}

// x = A^-1 u by a supernodal partitioned inverse: one persistent dataflow launch
// (both triangles, every supernode, tiles ordered leaves-first then root-first)
template <typename T, typename TI>
void factor_solve(const FactorBuf& F, const TI* u, const int32_t* gmap, T* x, cudaStream_t s) {
  const CoarseFactorDev D = F.dev();
  // one launch: dependency-driven tiles (k_cf_dataflow)
  CfSched S{F.ticket.p, F.ready.p, F.ready.p + F.n_sn, F.n_fwd_tasks, F.n_df_tasks, F.n_sn};
  if (F.nt == CF_NT_LOCAL)
    k_cf_dataflow<T, TI, CF_NT_LOCAL><<<F.df_grid, CF_NT_LOCAL, F.df_smem, s>>>(
        D, S, F.df_tasks.p, (const T*)F.vals.p, u, gmap, (T*)F.ybuf.p, (T*)F.cbuf.p, x, (const T*)F.fcm.p);
  else
    k_cf_dataflow<T, TI, CF_NT_COARSE><<<F.df_grid, CF_NT_COARSE, F.df_smem, s>>>(
        D, S, F.df_tasks.p, (const T*)F.vals.p, u, gmap, (T*)F.ybuf.p, (T*)F.cbuf.p, x, (const T*)F.fcm.p);
  CK_LAUNCH();
}

template <typename T>
T* local_solve(gdsw_precond* m, const double* r, int jacobi_iters, cudaStream_t s) {
  gdsw_plan* P = m->plan;
  if (jacobi_iters > 0 || P->method == GDSW_FAST_ILU) {
    m->ensure_jacobi();
    const int it = jacobi_iters > 0 ? jacobi_iters : m->iters;
    const int f = P->l_sell.masked ? SELL_MASK : (P->l_sell.has16 && P->u_sell.has16) ? SELL_D16 : SELL_COL32;
    // uniform-width rows (all slots loaded at once): C2 sweeps 28.0/35.2/33.9
    // -> 25.9/30.2/27.8 us (GDSW_JACOBI_UNI=0 selects the plain loop)
    static const bool uni_off = [] {
      const char* e = std::getenv("GDSW_JACOBI_UNI");
      return e && e[0] == '0';
    }();
    const bool uni = !uni_off && P->l_sell.uw >= 1 && P->l_sell.uw <= 4 && P->u_sell.uw >= 1 &&
                     P->u_sell.uw <= 4;
    if (f == SELL_MASK)
      return uni ? jacobi_solve<T, false, SELL_MASK, true>(m, r, it, s)
                 : jacobi_solve<T, false, SELL_MASK, false>(m, r, it, s);
    if (l2_hints_enabled())
      return f == SELL_D16 ? jacobi_solve<T, true, SELL_D16, false>(m, r, it, s)
                           : jacobi_solve<T, true, SELL_COL32, false>(m, r, it, s);
    if (uni)
      return f == SELL_D16 ? jacobi_solve<T, false, SELL_D16, true>(m, r, it, s)
                           : jacobi_solve<T, false, SELL_COL32, true>(m, r, it, s);
    return f == SELL_D16 ? jacobi_solve<T, false, SELL_D16, false>(m, r, it, s)
                         : jacobi_solve<T, false, SELL_COL32, false>(m, r, it, s);
  }
  if (m->lf.on) {
    // exact LU: supernodal partitioned inverses of every block
    ProfScope ps("factor_local", s, (double)m->lf.bytes + P->n_loc * 12.0);
    T* y = (T*)m->x1.p;
    factor_solve<T, double>(m->lf, r, P->gmap.p, y, s);
    return y;
  }
  return levelset_solve<T>(m, r, s);
}

// v = A0^-1 u: dense inverse GEMV, or the factored partitioned inverse
// (one persistent dataflow launch)
template <typename T>
void coarse_solve(gdsw_precond* m, cudaStream_t cs) {
  CoarsePlan* Cp = m->cp.get();
  if (!m->cf.on) {
    ProfScope ps("coarse_solve", cs, (double)Cp->n_c * Cp->n_c * sizeof(T));
    k_coarse_gemv<T><<<grid_for(Cp->n_c, TB / 32), TB, 0, cs>>>(Cp->n_c, (const T*)m->ainv.p,
                                                                (const T*)m->cu.p, (T*)m->cv.p);
    CK_LAUNCH();
    return;
  }
  ProfScope ps("coarse_solve", cs, (double)m->cf.bytes);
  factor_solve<T, T>(m->cf, (const T*)m->cu.p, nullptr, (T*)m->cv.p, cs);
}

template <typename T>
void apply_T(gdsw_precond* m, const double* r, double* z, cudaStream_t s) {
  gdsw_plan* P = m->plan;
  CoarsePlan* Cp = m->cp.get();
  gdsw_dist* Dd = m->dist;
  if (Dd) {
    // halo rows of the (extended) input from their owners
    ProfScope ps("halo_fwd", s, 0.0);
    Dd->halo_fwd(const_cast<double*>(r), s);
  }
  // the coarse restriction, the coarse right-hand side's all-reduce (sharded
  // path) and the coarse solve only read r: they run on the side stream,
  // overlapped with the local solves, joined before the prolongation
  const bool fork = Cp && !env_flag("GDSW_NO_OVERLAP");
  cudaStream_t cs = s;
  if (fork) {
    CK(cudaEventRecord(m->ev_fork, s));
    CK(cudaStreamWaitEvent(m->side, m->ev_fork, 0));
    cs = m->side;
  }
  if (Cp) {
    ChunkDev D = Cp->chunk_dev();
    if (Cp->n_chunks > 0) {
      // panels once + r at interior rows (4 B index + 8 B value)
      ProfScope ps("restrict_panels", cs, (double)Cp->panel_entries * sizeof(T) + Cp->n_int_total * 12.0);
      k_restrict_chunks<T><<<Cp->n_chunks, RS_THREADS, 0, cs>>>(D, (const T*)m->panel(), r, (T*)m->pdot.p);
      CK_LAUNCH();
    }
    {
      ProfScope ps("restrict_columns", cs, (double)Cp->h_pgt_val.size() * (sizeof(T) + 12) +
                                               (double)Cp->n_cpart * (sizeof(T) + 8));
      k_restrict_columns<T><<<Cp->n_c, 256, 0, cs>>>(Cp->n_c, Cp->pgt_ptr.p, Cp->pgt_row.p,
                                                     (const T*)m->pgt_val.p, r, Cp->cpart_ptr.p,
                                                     Cp->cpart_idx.p, (const T*)m->pdot.p, (T*)m->cu.p);
      CK_LAUNCH();
    }
    if (Dd) {
      // coarse right-hand side: every rank's partial, summed in rank order
      // (own channel: it runs on the side stream)
      ProfScope ps("coarse_allreduce", cs, 0.0);
      k_cast_to_f64<T><<<grid_for(Cp->n_c, TB), TB, 0, cs>>>(Cp->n_c, (const T*)m->cu.p, m->red64.p);
      CK_LAUNCH();
      Dd->allreduce(m->red64.p, m->red64.p + Cp->n_c, Cp->n_c, cs, CH_CRS);
      k_cast_from_f64<T><<<grid_for(Cp->n_c, TB), TB, 0, cs>>>(Cp->n_c, m->red64.p + Cp->n_c, (T*)m->cu.p);
      CK_LAUNCH();
    }
    coarse_solve<T>(m, cs);
  }
  if (fork) CK(cudaEventRecord(m->ev_join, m->side));
  T* y = local_solve<T>(m, r, 0, s);
  RemoteAdd RA{};
  int64_t own_lo = 0, own_hi = P->n;
  if (Dd) {
    // my subdomains' contributions to rows other ranks own, sent to them;
    // theirs to my rows received, combined in subdomain order below
    ProfScope ps("halo_rev", s, 0.0);
    for (int i = 0; i < Dd->halo.nn; ++i) {
      const int64_t lo = Dd->halo.recv_lo[i], hi = Dd->halo.recv_hi[i];
      if (hi > lo) {
        k_scatter_partial<T><<<grid_for(hi - lo, TB), TB, 0, s>>>(lo, hi, P->sc_ptr.p, P->sc_pos.p, y,
                                                                  m->part_ext.p);
        CK_LAUNCH();
      }
    }
    Dd->halo_rev(m->part_ext.p, m->recv_ext.p, s);
    RA = RemoteAdd{m->recv_ext.p, Dd->pre_lo, Dd->pre_hi, Dd->post_lo, Dd->post_hi};
    own_lo = Dd->own_off;
    own_hi = Dd->own_off + Dd->n_own;
  }
  if (fork) CK(cudaStreamWaitEvent(s, m->ev_join, 0));
  if (Cp) {
    // interior rows (panel row dot, coalesced) and interface rows (CSR
    // Phi_Gamma), each + its local contributions, in one launch
    ChunkDev D = Cp->chunk_dev();
    const double ng = (double)Cp->n_gamma;
    ProfScope ps("prolong", s, (double)Cp->panel_entries * sizeof(T) +
                                   Cp->n_int_total * (4.0 + 8.0 + 8.0 + 4.0 + sizeof(T)) +
                                   (double)Cp->h_pgr_val.size() * (sizeof(T) + 4) + ng * (4.0 + 8.0 + 8.0 + 8.0) +
                                   (double)(P->n_loc - Cp->n_int_total) * (4.0 + sizeof(T)));
    const int32_t nblk = Cp->n_chunks + (int32_t)((Cp->n_gamma + CH_THREADS - 1) / CH_THREADS);
    if (nblk > 0) {
      k_prolong<T><<<nblk, CH_THREADS, 0, s>>>(Cp->n_chunks, D, (const T*)m->panel(),
                                               ProlongGamma{(int32_t)Cp->n_gamma, Cp->gamma32.p, Cp->pgam_ptr.p,
                                                            Cp->pgam_col.p},
                                               (const T*)m->pgr_val.p, (const T*)m->cv.p, P->sc_ptr.p, P->sc_pos.p,
                                               y, RA, z);
      CK_LAUNCH();
    }
  } else {
    ProfScope ps("scatter", s, P->n_loc * (4.0 + sizeof(T)) + (P->n + 1) * 4.0 + P->n * 8.0);
    k_scatter_owned<T><<<grid_for(own_hi - own_lo, TB), TB, 0, s>>>(own_lo, own_hi, P->sc_ptr.p,
                                                                    P->sc_pos.p, y, RA, z);
    CK_LAUNCH();
  }
}

// One apply's launches (about a dozen kernels plus the side-stream fork and
// join) replayed as a CUDA graph: captured on the second apply with the
// same (r, z, stream) -- the first one runs eagerly and performs every lazy
// allocation -- and dropped whenever the preconditioner's data changes.
// Not used while the per-kernel profiler records events or with
// GDSW_NO_GRAPH=1. The sharded path's collectives take their sequence
// numbers from device counters, so they replay inside graphs too.
bool apply_graph_ok(const gdsw_precond* m) {
  return !prof().on && !env_flag("GDSW_NO_GRAPH") && !env_flag("GDSW_NO_OVERLAP");
}

// the apply's launches enqueued into a stream that is being captured into a
// larger graph (the GMRES pass graph): no event handshake, no nested graph
void precond_apply_captured(gdsw_precond* m, const double* r, double* z, cudaStream_t s) {
  require(m->has_factors, "preconditioner has no numeric factors");
  std::lock_guard<std::recursive_mutex> g(m->mu);
  with_dtype(m->dtype, [&](auto tag) { apply_T<decltype(tag)>(m, r, z, s); });
}

void precond_apply(gdsw_precond* m, const double* r, double* z, cudaStream_t s) {
  require(m->has_factors, "preconditioner has no numeric factors");
  if (m->cp) require(m->has_phi && m->has_ainv, "coarse space is not set up");
  std::lock_guard<std::recursive_mutex> g(m->mu);
  CK(cudaStreamWaitEvent(s, m->last, 0));
  if (apply_graph_ok(m)) {
    for (auto& ag : m->graphs) {
      if (ag.r == r && ag.z == z) {
        if (!ag.exec) {
          // captured on a private stream (the caller's may be the legacy
          // default stream, which cannot capture); replayed on the caller's
          cudaGraph_t graph = nullptr;
          const int64_t c0 = launch_counter().load();
          CK(cudaStreamBeginCapture(m->cap, cudaStreamCaptureModeThreadLocal));
          with_dtype(m->dtype, [&](auto tag) { apply_T<decltype(tag)>(m, r, z, m->cap); });
          CK(cudaStreamEndCapture(m->cap, &graph));
          ag.kernels = launch_counter().load() - c0;
          CK(cudaGraphInstantiate(&ag.exec, graph, 0));
          CK(cudaGraphDestroy(graph));
        } else {
          launch_counter().fetch_add(ag.kernels, std::memory_order_relaxed);
        }
        CK(cudaGraphLaunch(ag.exec, s));
        CK(cudaEventRecord(m->last, s));
        return;
      }
    }
    if (m->graphs.size() < 8) m->graphs.push_back(gdsw_precond::ApplyGraph{r, z, s, nullptr, 0});
  }
  with_dtype(m->dtype, [&](auto tag) { apply_T<decltype(tag)>(m, r, z, s); });
  CK(cudaEventRecord(m->last, s));
}

template <typename T>
void upload_cast(DBuf<char>& dst, const std::vector<double>& src) {
  std::vector<T> tmp(src.begin(), src.end());
  dst.alloc(std::max<size_t>(tmp.size(), 1) * sizeof(T));
  if (!tmp.empty()) CK(cudaMemcpy(dst.p, tmp.data(), tmp.size() * sizeof(T), cudaMemcpyHostToDevice));
}

}  // namespace

extern "C" {

int gdsw_precond_create(gdsw_precond** out, gdsw_plan* plan, int dtype, int trisolve_iters) {
  return guarded([&] {
    require(dtype == GDSW_F64 || dtype == GDSW_F32, "unknown dtype");
    require(trisolve_iters >= 1, "trisolve_iters must be at least 1");
    auto m = std::make_unique<gdsw_precond>();
    m->plan = plan;
    plan->refs++;
    m->dtype = dtype;
    m->es = esize(dtype);
    m->iters = trisolve_iters;
    gdsw_plan* P = plan;
    m->lval.alloc(std::max<int64_t>(P->nnz_l, 1) * m->es);
    m->uval.alloc(std::max<int64_t>(P->nnz_u, 1) * m->es);
    const size_t nl = std::max<int64_t>(P->n_loc, 1) * m->es;
    m->xb.alloc(nl);
    m->x1.alloc(nl);
    m->x2.alloc(nl);
    m->x3.alloc(nl);
    CK(cudaEventCreateWithFlags(&m->last, cudaEventDisableTiming));
    CK(cudaStreamCreateWithFlags(&m->side, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&m->cap, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&m->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&m->ev_join, cudaEventDisableTiming));
    CK(cudaEventRecord(m->last, 0));
    *out = m.release();
  });
}

int gdsw_precond_set_coarse(gdsw_precond* m, const gdsw_coarse_desc* desc) {
  return guarded([&] {
    auto cp = std::make_unique<CoarsePlan>();
    build_coarse(cp.get(), m->plan, desc);
    with_dtype(m->dtype, [&](auto tag) {
      using T = decltype(tag);
      upload_cast<T>(m->pgr_val, cp->h_pgr_val);
      upload_cast<T>(m->pgt_val, cp->h_pgt_val);
    });
    m->pdot.alloc(std::max<int64_t>(cp->n_partial, 1) * m->es);
    m->cu.alloc(std::max<int32_t>(cp->n_c, 1) * m->es);
    m->cv.alloc(std::max<int32_t>(cp->n_c, 1) * m->es);
    m->panel64.alloc(std::max<int64_t>(cp->panel_entries, 1));
    if (m->dtype == GDSW_F32) m->panel32.alloc(std::max<int64_t>(cp->panel_entries, 1) * 4);
    m->red64.alloc(2 * (size_t)std::max(cp->n_c, 1));
    CK(cudaDeviceSynchronize());
    m->cp = std::move(cp);
    m->drop_graphs();
    m->has_phi = m->has_ainv = false;
  });
}

int gdsw_precond_set_factors(gdsw_precond* m, const void* l_vals, const void* u_vals) {
  return guarded([&] {
    gdsw_plan* P = m->plan;
    if (P->nnz_l) CK(cudaMemcpy(m->lval.p, l_vals, P->nnz_l * m->es, cudaMemcpyHostToDevice));
    if (P->nnz_u) CK(cudaMemcpy(m->uval.p, u_vals, P->nnz_u * m->es, cudaMemcpyHostToDevice));
    m->has_factors = true;
    m->drop_graphs();
    m->jacobi_ready = false;
    m->stream_vals_ready = false;
    if (P->method == GDSW_FAST_ILU) m->ensure_jacobi();
    else m->ensure_stream_vals();
  });
}

int gdsw_precond_get_factors(const gdsw_precond* m, void* l_vals, void* u_vals) {
  return guarded([&] {
    gdsw_plan* P = m->plan;
    if (P->nnz_l) CK(cudaMemcpy(l_vals, m->lval.p, P->nnz_l * m->es, cudaMemcpyDeviceToHost));
    if (P->nnz_u) CK(cudaMemcpy(u_vals, m->uval.p, P->nnz_u * m->es, cudaMemcpyDeviceToHost));
  });
}

int gdsw_plan_set_block_pattern(gdsw_plan* P, const int64_t* ab_ptr, const int64_t* ab_idx,
                                const int64_t* ab_src) {
  return guarded([&] {
    const int64_t nab = ab_ptr[P->n_loc];
    P->ab_ptr.upload(vec(ab_ptr, P->n_loc + 1));
    P->ab_idx.upload(to_i32(ab_idx, nab));
    P->ab_src.upload(vec(ab_src, nab));
    P->l_idx32.upload(to_i32(P->h_l_idx.data(), P->h_l_idx.size()));
    P->u_idx32.upload(to_i32(P->h_u_idx.data(), P->h_u_idx.size()));
    P->lu_lev_sub.upload(to_i32(P->h_llev_sub.data(), P->h_llev_sub.size()));
    P->lu_lev_ptr.upload(to_i32(P->h_llev_ptr.data(), P->h_llev_ptr.size()));
    P->lu_lev_rows.upload(to_i32(P->h_llev_rows.data(), P->h_llev_rows.size()));
    int64_t mx = 0;
    for (int32_t s = 0; s < P->n_sub; ++s) mx = std::max<int64_t>(mx, P->h_sub_ptr[s + 1] - P->h_sub_ptr[s]);
    P->n_max = (int32_t)mx;
    P->has_ab = true;
  });
}

int gdsw_precond_lu_numeric(gdsw_precond* m, const gdsw_csr* a, double diag_shift, int64_t* fail_rows) {
  return guarded([&] {
    gdsw_plan* P = m->plan;
    require(P->has_ab, "plan has no block pattern for the numeric LU");
    require(a->dtype == GDSW_F64, "the numeric LU reads the float64 operator values");
    const double* av = (const double*)a->csr_val.p;
    DBuf<double> norm(std::max(P->n_sub, 1));
    DBuf<int64_t> fail(std::max(P->n_sub, 1));
    std::vector<int64_t> none(std::max(P->n_sub, 1), INT64_MAX);
    CK(cudaMemcpy(fail.p, none.data(), none.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    with_dtype(m->dtype, [&](auto tag) {
      using T = decltype(tag);
      const size_t nscr = (size_t)P->n_sub * LU_WARPS * std::max(P->n_max, 1);
      DBuf<T> w(nscr);
      DBuf<int32_t> stamp(nscr);
      CK(cudaMemset(stamp.p, 0xff, nscr * sizeof(int32_t)));
      if (P->nnz_l) CK(cudaMemset(m->lval.p, 0, P->nnz_l * sizeof(T)));
      if (P->nnz_u) CK(cudaMemset(m->uval.p, 0, P->nnz_u * sizeof(T)));
      const LuDev D = P->lu_dev();
      k_block_norm_inf<T><<<P->n_sub, LU_THREADS>>>(D, av, norm.p);
      CK_LAUNCH();
      k_lu_numeric<T><<<P->n_sub, LU_THREADS>>>(D, av, (T)diag_shift, norm.p, (T*)m->lval.p, (T*)m->uval.p,
                                                w.p, stamp.p, fail.p);
      CK_LAUNCH();
      CK(cudaDeviceSynchronize());
    });
    std::vector<int64_t> f = fail.download();
    for (int32_t s = 0; s < P->n_sub; ++s) fail_rows[s] = f[s] == INT64_MAX ? 0 : f[s];
    m->has_factors = true;
    m->drop_graphs();
    m->jacobi_ready = false;
    m->stream_vals_ready = false;
    if (P->method == GDSW_FAST_ILU) m->ensure_jacobi();
    else m->ensure_stream_vals();
  });
}

int gdsw_precond_fastilu(gdsw_precond* m, const gdsw_csr* a, int sweeps, double* residuals) {
  return guarded([&] {
    gdsw_plan* P = m->plan;
    require(P->fastilu, "plan has no FastILU product plan");
    require(a->dtype == GDSW_F64, "FastILU reads the float64 operator values");
    require(sweeps >= 1, "factor_sweeps must be at least 1");
    const double* av = (const double*)a->csr_val.p;
    DBuf<int> flag(2);
    flag.zero();
    with_dtype(m->dtype, [&](auto tag) {
      using T = decltype(tag);
      FastIluDev F = P->fastilu_dev();
      T* lo = (T*)m->lval.p;
      T* uo = (T*)m->uval.p;
      DBuf<char> ln(std::max<int64_t>(P->nnz_l, 1) * sizeof(T)), un(std::max<int64_t>(P->nnz_u, 1) * sizeof(T));
      T* lnp = (T*)ln.p;
      T* unp = (T*)un.p;
      if (P->nnz_u) { k_fastilu_init_u<T><<<grid_for(P->nnz_u, TB), TB>>>(F, av, uo); CK_LAUNCH(); }
      if (P->nnz_l) { k_fastilu_init_l<T><<<grid_for(P->nnz_l, TB), TB>>>(F, av, uo, lo); CK_LAUNCH(); }
      DBuf<double> terms(std::max<int64_t>(P->n_res, 1)), rsum(P->n_sub);
      for (int sw = 0; sw < sweeps; ++sw) {
        const int64_t ne = P->nnz_l + P->nnz_u;
        if (ne) {
          k_fastilu_sweep<T><<<grid_for(ne, TB), TB>>>(F, av, lo, uo, lnp, unp, flag.p);
          CK_LAUNCH();
        }
        std::swap(lo, lnp);
        std::swap(uo, unp);
        if (residuals && P->n_res > 0) {
          k_fastilu_residual_terms<T><<<grid_for(P->n_res, TB), TB>>>(P->fastilu_res_dev(), av, lo, uo,
                                                                      terms.p);
          CK_LAUNCH();
          k_segment_sum<<<P->n_sub, TB>>>(P->res_sub_ptr.p, terms.p, rsum.p);
          CK_LAUNCH();
          CK(cudaMemcpy(residuals + (size_t)sw * P->n_sub, rsum.p, P->n_sub * sizeof(double),
                        cudaMemcpyDeviceToHost));
        }
      }
      // final iterate lives in lo/uo; make it the precond's arena
      if (lo != (T*)m->lval.p) {
        if (P->nnz_l) CK(cudaMemcpy(m->lval.p, lo, P->nnz_l * sizeof(T), cudaMemcpyDeviceToDevice));
        if (P->nnz_u) CK(cudaMemcpy(m->uval.p, uo, P->nnz_u * sizeof(T), cudaMemcpyDeviceToDevice));
      }
      if (P->nnz_l) { k_count_nonfinite<T><<<grid_for(P->nnz_l, TB), TB>>>(P->nnz_l, (T*)m->lval.p, flag.p + 1); CK_LAUNCH(); }
      if (P->nnz_u) { k_count_nonfinite<T><<<grid_for(P->nnz_u, TB), TB>>>(P->nnz_u, (T*)m->uval.p, flag.p + 1); CK_LAUNCH(); }
      CK(cudaDeviceSynchronize());
    });
    std::vector<int> f = flag.download();
    if (f[0] || f[1])
      throw Error(E_FLOAT,
                  "fixed-point factorization produced nonfinite entries; use a more conservative "
                  "initial guess (diagonal shift) or exact ILU");
    m->has_factors = true;
    m->drop_graphs();
    m->jacobi_ready = false;
    m->stream_vals_ready = false;
    m->ensure_jacobi();
  });
}

int gdsw_precond_extend(gdsw_precond* m, const gdsw_csr* a, double tol, int max_iters, int* iters_out,
                        double* col_resid) {
  return guarded([&] {
    require(m->cp != nullptr, "preconditioner has no coarse structure");
    CoarsePlan* P = m->cp.get();
    require(a->dtype == GDSW_F64, "the extension reads the float64 operator values");
    const int K = P->K;
    const int64_t NE = std::max<int64_t>(P->panel_entries, 1);
    const int64_t NI = P->n_int_total;
    DBuf<double> aii_val(std::max<size_t>(P->aii_src.n, 1)), aig_val(std::max<size_t>(P->aig_src.n, 1)),
        dinv(std::max<int64_t>(NI, 1));
    const double* av = (const double*)a->csr_val.p;
    // value gathers from A (setup-time, trivially parallel)
    if (P->aii_src.n) {
      k_gather_vals<<<grid_for(P->aii_src.n, TB), TB>>>((int64_t)P->aii_src.n, P->aii_src.p, av, aii_val.p);
      CK_LAUNCH();
    }
    if (P->aig_src.n) {
      k_gather_vals<<<grid_for(P->aig_src.n, TB), TB>>>((int64_t)P->aig_src.n, P->aig_src.p, av, aig_val.p);
      CK_LAUNCH();
    }
    if (NI) {
      k_make_dinv<<<grid_for(NI, TB), TB>>>(NI, P->aii_diag.p, aii_val.p, dinv.p);
      CK_LAUNCH();
    }
    ExtDev E{};
    E.n_chunks = P->n_chunks;
    E.n_sub = P->n_sub;
    E.n_int_total = NI;
    E.chunk_sub = P->chunk_sub.p;
    E.chunk_row0 = P->chunk_row0.p;
    E.chunk_nrow = P->chunk_nrow.p;
    E.chunk_poff = P->chunk_poff.p;
    E.int_ptr = P->int_ptr.p;
    E.n_int = P->n_int.p;
    E.col_ptr = P->col_ptr.p;
    E.col_ids = P->col_ids.p;
    E.panel_off = P->panel_off.p;
    E.aii_ptr = P->aii_ptr.p;
    E.aii_col = P->aii_col.p;
    E.aii_val = aii_val.p;
    E.dinv = dinv.p;
    E.aig_ptr = P->aig_ptr.p;
    E.aig_col = P->aig_col.p;
    E.aig_val = aig_val.p;
    E.pgam_ptr = P->pgam_ptr.p;
    E.pgam_col = P->pgam_col.p;
    E.pgam_val = P->pgam_val.p;
    double* X = m->panel64.p;
    DBuf<double> B(NE), R(NE), Z(NE), Pp(NE), AP(NE);
    DBuf<double> part1(P->n_partial), part2(P->n_partial);
    DBuf<double> rz(std::max(K, 1)), rzn(std::max(K, 1)), rrn(std::max(K, 1)), bb(std::max(K, 1)),
        pap(std::max(K, 1)), alpha(std::max(K, 1)), beta(std::max(K, 1));
    DBuf<int> active(std::max(K, 1)), nact(1);
    int it = 0;
    if (P->n_chunks > 0 && K > 0) {
      CK(cudaMemset(X, 0, NE * sizeof(double)));
      Pp.zero();
      AP.zero();
      k_ext_rhs<<<P->n_chunks, EXT_THREADS>>>(E, B.p);
      CK_LAUNCH();
      CK(cudaMemcpy(R.p, B.p, NE * sizeof(double), cudaMemcpyDeviceToDevice));
      const unsigned gk = grid_for(K, TB);
      k_ext_update<<<P->n_chunks, EXT_THREADS>>>(E, nullptr, X, R.p, Z.p, Pp.p, AP.p, part1.p, part2.p);
      CK_LAUNCH();
      k_ext_colsum<<<gk, TB>>>(E, P->colsub.p, P->sub_chunk0.p, part1.p, rz.p, K);
      k_ext_colsum<<<gk, TB>>>(E, P->colsub.p, P->sub_chunk0.p, part2.p, bb.p, K);
      k_init_active<<<gk, TB>>>(K, bb.p, active.p);
      CK_LAUNCH();
      CK(cudaMemset(beta.p, 0, K * sizeof(double)));
      k_ext_pupdate<<<P->n_chunks, EXT_THREADS>>>(E, beta.p, Z.p, Pp.p);
      CK_LAUNCH();
      const double tol2 = tol * tol;
      for (it = 0; it < max_iters; ++it) {
        k_ext_spmm<<<P->n_chunks, EXT_THREADS>>>(E, Pp.p, AP.p, part1.p);
        k_ext_colsum<<<gk, TB>>>(E, P->colsub.p, P->sub_chunk0.p, part1.p, pap.p, K);
        k_ext_alpha<<<gk, TB>>>(K, rz.p, pap.p, active.p, alpha.p);
        k_ext_update<<<P->n_chunks, EXT_THREADS>>>(E, alpha.p, X, R.p, Z.p, Pp.p, AP.p, part1.p, part2.p);
        k_ext_colsum<<<gk, TB>>>(E, P->colsub.p, P->sub_chunk0.p, part1.p, rzn.p, K);
        k_ext_colsum<<<gk, TB>>>(E, P->colsub.p, P->sub_chunk0.p, part2.p, rrn.p, K);
        nact.zero();
        k_ext_beta<<<gk, TB>>>(K, tol2, bb.p, rz.p, rzn.p, rrn.p, active.p, beta.p, nact.p);
        k_ext_pupdate<<<P->n_chunks, EXT_THREADS>>>(E, beta.p, Z.p, Pp.p);
        CK_LAUNCH();
        if ((it & 15) == 15) {
          int na = 0;
          CK(cudaMemcpy(&na, nact.p, sizeof(int), cudaMemcpyDeviceToHost));
          if (na == 0) { ++it; break; }
        }
      }
      k_ext_resid_max<<<P->n_chunks, EXT_THREADS>>>(E, X, B.p, part1.p);
      k_ext_colmax<<<gk, TB>>>(E, P->colsub.p, P->sub_chunk0.p, part1.p, pap.p, K);
      CK_LAUNCH();
      if (col_resid) CK(cudaMemcpy(col_resid, pap.p, K * sizeof(double), cudaMemcpyDeviceToHost));
    }
    if (m->dtype == GDSW_F32 && P->panel_entries) {
      k_cast_f64_f32<<<grid_for(P->panel_entries, TB), TB>>>(P->panel_entries, X, (float*)m->panel32.p);
      CK_LAUNCH();
    }
    CK(cudaDeviceSynchronize());
    if (iters_out) *iters_out = it;
    m->has_phi = true;
    m->drop_graphs();
  });
}

}  // extern "C"

extern "C" {

int64_t gdsw_precond_panel_entries(const gdsw_precond* m) {
  return m->cp ? m->cp->panel_entries : 0;
}

int gdsw_precond_get_panels(const gdsw_precond* m, double* panels) {
  return guarded([&] {
    require(m->has_phi, "coarse basis not computed");
    if (m->cp->panel_entries)
      CK(cudaMemcpy(panels, m->panel64.p, m->cp->panel_entries * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

// e_c as a coarse vector
__global__ void k_unit(int32_t n, int32_t c, double* __restrict__ v) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i == c ? 1.0 : 0.0;
}

// A0 = Phi^T A Phi column by column with the apply's own float64
// prolongation, SpMV and restriction kernels (the reference's coarse_matrix,
// coarse_space.py:205-207). Sharded (d != null): Phi e_c on my rows, its halo
// from the owners, A on my owned rows, my rows' share of Phi^T, then the
// partial A0 summed over ranks in rank order through the peer-memory
// all-reduce -- identical on every rank, no host round trip.
__global__ void k_abs_copy(int64_t n, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = fabs(x[i]);
}

DBuf<double> abs_copy(const double* x, size_t n) {
  DBuf<double> y(std::max<size_t>(n, 1));
  if (n) {
    k_abs_copy<<<grid_for((int64_t)n, TB), TB>>>((int64_t)n, x, y.p);
    CK_LAUNCH();
  }
  return y;
}

// pattern != null: also the structural pattern of Phi^T A Phi -- the same
// product over |Phi| and |A| (no cancellation), nonzero exactly where the
// reference's Gustavson SpGEMM creates an entry, computed zeros included
// (coarse_space.py:205-207, _kernels.py:51-94)
static void coarse_galerkin(gdsw_precond* m, const gdsw_csr* a, gdsw_dist* d, double* a0_dense,
                            uint8_t* pattern = nullptr) {
  require(m->cp != nullptr && m->has_phi, "coarse basis is not set up");
  require(a->dtype == GDSW_F64, "the Galerkin product reads the float64 operator values");
  CoarsePlan* Cp = m->cp.get();
  gdsw_plan* P = m->plan;
  const int32_t nc = Cp->n_c;
  const int64_t n = P->n;
  const int64_t off = d ? d->own_off : 0;
  if (d) require(d->ready && d->n_ext == n && a->nrows == d->n_own && a->ncols == n,
                 "layout does not match the preconditioner");
  // float64 Phi: panels (always kept in f64) + interface values
  DBuf<double> pgr(std::max<size_t>(Cp->h_pgr_val.size(), 1)), pgt(std::max<size_t>(Cp->h_pgt_val.size(), 1));
  if (!Cp->h_pgr_val.empty()) CK(cudaMemcpy(pgr.p, Cp->h_pgr_val.data(), Cp->h_pgr_val.size() * 8, cudaMemcpyHostToDevice));
  if (!Cp->h_pgt_val.empty()) CK(cudaMemcpy(pgt.p, Cp->h_pgt_val.data(), Cp->h_pgt_val.size() * 8, cudaMemcpyHostToDevice));
  DBuf<double> v(std::max(nc, 1)), z(std::max<int64_t>(n, 1)), y(std::max<int64_t>(n, 1)),
      zero_loc(std::max<int64_t>(P->n_loc, 1)), part(std::max<int64_t>(Cp->n_partial, 1)),
      a0((size_t)std::max(nc, 1) * std::max(nc, 1));
  zero_loc.zero();
  z.zero();
  const ChunkDev D = Cp->chunk_dev();
  const int32_t nblk = Cp->n_chunks + (int32_t)((Cp->n_gamma + CH_THREADS - 1) / CH_THREADS);
  // one pass: A0 (or, over absolute values, its structural pattern)
  auto product = [&](const double* panel, const double* pgr_v, const double* pgt_v, const double* aval,
                     DBuf<double>& out) {
    for (int32_t c = 0; c < nc; ++c) {
      k_unit<<<grid_for(nc, TB), TB>>>(nc, c, v.p);
      CK_LAUNCH();
      if (nblk > 0) {
        k_prolong<double><<<nblk, CH_THREADS>>>(Cp->n_chunks, D, panel,
                                               ProlongGamma{(int32_t)Cp->n_gamma, Cp->gamma32.p, Cp->pgam_ptr.p,
                                                            Cp->pgam_col.p},
                                               pgr_v, v.p, P->sc_ptr.p, P->sc_pos.p, zero_loc.p, RemoteAdd{}, z.p);
        CK_LAUNCH();
      }
      if (d) d->halo_fwd(z.p, 0);
      if (a->nrows > 0) {
        spmv_T<double>(a, z.p, nullptr, y.p + off, 0, 1.0, 0.0, 0);
        CK_LAUNCH();
      }
      if (Cp->n_chunks > 0) {
        k_restrict_chunks<double><<<Cp->n_chunks, RS_THREADS>>>(D, panel, y.p, part.p);
        CK_LAUNCH();
      }
      k_restrict_columns<double><<<nc, 256>>>(nc, Cp->pgt_ptr.p, Cp->pgt_row.p, pgt_v, y.p, Cp->cpart_ptr.p,
                                              Cp->cpart_idx.p, part.p, out.p + (size_t)c * nc);
      CK_LAUNCH();
    }
    if (d && d->nranks > 1) {
      const int64_t total = (int64_t)nc * nc, step = d->layout.red_max;
      for (int64_t o = 0; o < total; o += step)
        d->allreduce(out.p + o, out.p + o, std::min(step, total - o), 0);
    }
  };
  product(m->panel64.p, pgr.p, pgt.p, (const double*)a->sell_val.p, a0);
  CK(cudaDeviceSynchronize());
  // a0 holds columns contiguously: transpose into the row-major output
  std::vector<double> h = a0.download();
  for (int32_t c = 0; c < nc; ++c)
    for (int32_t r = 0; r < nc; ++r) a0_dense[(size_t)r * nc + c] = h[(size_t)c * nc + r];
  if (pattern) {
    DBuf<double> pan_a = abs_copy(m->panel64.p, Cp->panel_entries), pgr_a = abs_copy(pgr.p, Cp->h_pgr_val.size()),
                 pgt_a = abs_copy(pgt.p, Cp->h_pgt_val.size()),
                 a_a = abs_copy((const double*)a->sell_val.p, a->sell_val.n / sizeof(double));
    product(pan_a.p, pgr_a.p, pgt_a.p, a_a.p, a0);
    CK(cudaDeviceSynchronize());
    h = a0.download();
    for (int32_t c = 0; c < nc; ++c)
      for (int32_t r = 0; r < nc; ++r) pattern[(size_t)r * nc + c] = h[(size_t)c * nc + r] != 0.0;
  }
}

int gdsw_precond_coarse_galerkin(gdsw_precond* m, const gdsw_csr* a, double* a0_dense, uint8_t* pattern) {
  return guarded([&] { coarse_galerkin(m, a, nullptr, a0_dense, pattern); });
}

int gdsw_precond_set_coarse_inverse(gdsw_precond* m, const double* a0inv) {
  return guarded([&] {
    require(m->cp != nullptr, "preconditioner has no coarse structure");
    CoarsePlan* P = m->cp.get();
    std::vector<double> h(a0inv, a0inv + (size_t)P->n_c * P->n_c);
    with_dtype(m->dtype, [&](auto tag) { upload_cast<decltype(tag)>(m->ainv, h); });
    m->cf.on = false;
    m->has_ainv = true;
    m->drop_graphs();
  });
}

}  // extern "C"

template <typename T>
static void build_fcm(FactorBuf& F) {
  if (F.n_cm == 0) return;
  k_pinv_fcm<T><<<F.n_cm, 256>>>(F.dev(), F.cm_list.p, F.n_cm, (const T*)F.vals.p, (T*)F.fcm.p);
  CK_LAUNCH();
  CK(cudaDeviceSynchronize());
}

extern "C" {

// upload a host partitioned inverse (gdsw_coarse_factor) into F in the
// precond dtype; tasks are CF_ROWS-row tiles of each supernode's stacked
// rows (forward: s + r, backward: s)
// resident CTAs per SM of the dataflow kernel at CTA size nt
static int cf_occupancy(bool f32, int nt, size_t smem) {
  int occ = 0;
  if (nt == CF_NT_LOCAL) {
    if (f32) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cf_dataflow<float, double, CF_NT_LOCAL>, nt, smem));
    else CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cf_dataflow<double, double, CF_NT_LOCAL>, nt, smem));
  } else {
    if (f32) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cf_dataflow<float, double, CF_NT_COARSE>, nt, smem));
    else CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cf_dataflow<double, double, CF_NT_COARSE>, nt, smem));
  }
  return occ;
}

static void install_factor(FactorBuf& F, const gdsw_coarse_factor* f, int dtype, size_t es, int64_t cm_default,
                           int nt = CF_NT_COARSE) {
  F.nt = nt;
  const int nsn = f->n_sn, nl = f->n_levels;
  auto i32 = [](const int64_t* a, size_t n) { return to_i32(a, n); };
  F.sn_s.upload(i32(f->sn_s, nsn));
  F.sn_r.upload(i32(f->sn_r, nsn));
  F.col_ptr.upload(i32(f->col_ptr, nsn + 1));
  F.row_ptr.upload(i32(f->row_ptr, nsn + 1));
  F.col_ids.upload(i32(f->col_ids, f->col_ptr[nsn]));
  F.row_ids.upload(i32(f->row_ids, f->row_ptr[nsn]));
  const int64_t ncol = f->col_ptr[nsn], nrow = f->row_ptr[nsn];
  F.in_ptr.upload(i32(f->in_ptr, ncol + 1));
  F.in_idx.upload(i32(f->in_idx, f->in_ptr[ncol]));
  F.out_ptr.upload(i32(f->out_ptr, nrow + 1));
  F.out_idx.upload(i32(f->out_idx, f->out_ptr[nrow]));
  F.d_off.upload(f->d_off, nsn);
  F.m_off.upload(f->m_off, nsn);
  F.n_off.upload(f->n_off, nsn);
  {
    // narrow supernodes get a column-major copy of their forward block
    static const bool cm_off = env_flag("GDSW_CF_NOCM");
    static const int64_t cm_env = [] {
      const char* e = std::getenv("GDSW_CF_CM_MAX");
      return e ? (int64_t)std::atoi(e) : (int64_t)-1;
    }();
    const int64_t cm_max = cm_env >= 0 ? cm_env : cm_default;
    std::vector<int64_t> foff(nsn, -1);
    std::vector<int32_t> cm;
    int64_t tot = 0;
    for (int k = 0; k < nsn; ++k)
      if (!cm_off && f->sn_s[k] <= cm_max && f->sn_s[k] > 0) {
        foff[k] = tot;
        tot += 2 * (f->sn_s[k] + f->sn_r[k]) * f->sn_s[k];   // forward + backward panels
        cm.push_back(k);
      }
    F.f_off.upload(foff);
    F.cm_list.upload(cm.empty() ? std::vector<int32_t>{0} : cm);
    F.n_cm = (int32_t)cm.size();
    F.fcm.alloc((size_t)std::max<int64_t>(tot, 1) * es);
  }
  // algorithmic bytes and the largest staged vector (forward: s values,
  // backward: s + r)
  int64_t bytes = 0;
  size_t smax = 0;
  for (int k = 0; k < nsn; ++k) {
    const int64_t s = f->sn_s[k], r = f->sn_r[k];
    bytes += (s * s + 2 * r * s) * (int64_t)es;
    smax = std::max(smax, (size_t)(s + r) * es);
  }
  require(smax <= 200 * 1024, "partitioned-inverse supernode too large for shared memory");
  if (smax > 48 * 1024) {  // before the occupancy query below
    auto big = [&](auto kern) { CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax)); };
    big(k_cf_dataflow<double, double, CF_NT_LOCAL>);
    big(k_cf_dataflow<float, double, CF_NT_LOCAL>);
    big(k_cf_dataflow<float, float, CF_NT_LOCAL>);
    big(k_cf_dataflow<double, double, CF_NT_COARSE>);
    big(k_cf_dataflow<float, double, CF_NT_COARSE>);
    big(k_cf_dataflow<float, float, CF_NT_COARSE>);
  }
  // dataflow schedule: forward tiles leaves-first, backward tiles root-first;
  // parent = supernode of the first row below, readiness targets in tiles.
  // Tile rows per level and direction: about one tile per resident CTA
  // slot (GDSW_CF_TPS; measured 1 < 2 < 4 with the column-major panels: C3-
  // sized blocks 0.28 / 0.30 / 0.40 ms), clamped to 8..nt/2 rows
  {
    int occ = 0;
    occ = cf_occupancy(dtype == GDSW_F32, F.nt, smax);
    const int64_t slots = (int64_t)num_sms() * std::max(occ, 1);
    std::vector<int32_t> tile_f(nl), tile_b(nl);
    for (int l = 0; l < nl; ++l) {
      int64_t rf = 0, rb = 0;
      for (int64_t k = f->level_ptr[l]; k < f->level_ptr[l + 1]; ++k) {
        rf += f->sn_s[k] + f->sn_r[k];
        rb += f->sn_s[k];
      }
      static const int64_t tps = [] {
        const char* e = std::getenv("GDSW_CF_TPS");
        return e ? std::max<int64_t>(1, std::atoi(e)) : (int64_t)1;
      }();
      auto pick = [&](int64_t rows) {
        int64_t t = (rows + tps * slots - 1) / (tps * slots);
        t = std::min<int64_t>(F.nt / 2, std::max<int64_t>(CF_ROWS, (t + 7) / 8 * 8));
        return (int32_t)t;
      };
      tile_f[l] = pick(rf);
      tile_b[l] = pick(rb);
    }
    std::vector<int32_t> sn_of_col(f->n, -1), par(nsn, -1), nft(nsn), nbt(nsn), lev(nsn);
    for (int l = 0; l < nl; ++l)
      for (int64_t k = f->level_ptr[l]; k < f->level_ptr[l + 1]; ++k) lev[k] = l;
    for (int k = 0; k < nsn; ++k) {
      for (int64_t c = f->col_ptr[k]; c < f->col_ptr[k + 1]; ++c) sn_of_col[f->col_ids[c]] = k;
      nft[k] = (int32_t)((f->sn_s[k] + f->sn_r[k] + tile_f[lev[k]] - 1) / tile_f[lev[k]]);
      nbt[k] = (int32_t)((f->sn_s[k] + tile_b[lev[k]] - 1) / tile_b[lev[k]]);
    }
    std::vector<int32_t> cptr(nsn + 1, 0), cidx;
    for (int k = 0; k < nsn; ++k)
      if (f->sn_r[k] > 0) {
        par[k] = sn_of_col[f->row_ids[f->row_ptr[k]]];
        cptr[par[k] + 1]++;
      }
    for (int k = 0; k < nsn; ++k) cptr[k + 1] += cptr[k];
    cidx.assign(cptr[nsn], 0);
    std::vector<int32_t> fill(cptr.begin(), cptr.end() - 1), fneed(nsn, 0), bneed(nsn, 0);
    for (int k = 0; k < nsn; ++k)
      if (par[k] >= 0) {
        cidx[fill[par[k]]++] = k;
        fneed[par[k]] += nft[k];
      }
    for (int k = 0; k < nsn; ++k) bneed[k] = nft[k] + (par[k] >= 0 ? nbt[par[k]] : 0);
    std::vector<int2> df;
    auto tile = [](int64_t k, int64_t q, int64_t rows, int64_t t) {
      require(q < 65536, "partitioned-inverse supernode too tall for the tile encoding");
      return make_int2((int)k, (int)(q | (std::min<int64_t>(t, rows - q) << 16)));
    };
    for (int l = 0; l < nl; ++l)
      for (int64_t k = f->level_ptr[l]; k < f->level_ptr[l + 1]; ++k)
        for (int64_t q = 0; q < f->sn_s[k] + f->sn_r[k]; q += tile_f[l])
          df.push_back(tile(k, q, f->sn_s[k] + f->sn_r[k], tile_f[l]));
    F.n_fwd_tasks = (int32_t)df.size();
    for (int l = nl - 1; l >= 0; --l)
      for (int64_t k = f->level_ptr[l]; k < f->level_ptr[l + 1]; ++k)
        for (int64_t q = 0; q < f->sn_s[k]; q += tile_b[l]) df.push_back(tile(k, q, f->sn_s[k], tile_b[l]));
    F.n_df_tasks = (int32_t)df.size();
    F.n_sn = nsn;
    F.df_tasks.upload(df);
    F.parent.upload(par);
    F.child_ptr.upload(cptr);
    F.child_idx.upload(cidx.empty() ? std::vector<int32_t>{0} : cidx);
    F.fwd_need.upload(fneed);
    F.bwd_need.upload(bneed);
    F.ready.alloc(2 * (size_t)std::max(nsn, 1));
    F.ready.zero();
    F.ticket.alloc(2);
    F.ticket.zero();
    F.df_smem = smax;
  }
  F.bytes = bytes;
  F.n_launch = 1;
  with_dtype(dtype, [&](auto tag) {
    using T = decltype(tag);
    if (f->values) {
      std::vector<double> h(f->values, f->values + f->n_values);
      upload_cast<T>(F.vals, h);
      build_fcm<T>(F);
    } else {
      F.vals.alloc((size_t)std::max<int64_t>(f->n_values, 1) * sizeof(T));  // filled on the device
    }
    F.ybuf.alloc((size_t)f->n * sizeof(T));
    F.cbuf.alloc((size_t)std::max<int64_t>(nrow, 1) * sizeof(T));
    // persistent grid: every CTA resident
    const int occ = cf_occupancy(sizeof(T) == 4, F.nt, smax);
    F.df_grid = std::max(1, std::min(F.n_df_tasks, num_sms() * std::max(occ, 1)));
  });
  F.on = true;
}

int gdsw_precond_set_coarse_factor(gdsw_precond* m, const gdsw_coarse_factor* f) {
  return guarded([&] {
    require(m->cp != nullptr, "preconditioner has no coarse structure");
    require(f->n == m->cp->n_c, "coarse factor dimension mismatch");
    install_factor(m->cf, f, m->dtype, m->es, CF_CM_MAX);
    m->ainv.release();
    m->has_ainv = true;
    m->drop_graphs();
  });
}

}  // extern "C"

// the blocks of a structure-only partitioned inverse (values == NULL) from
// the device factors: k_pinv_fill + k_pinv_blocks (coarse_factor.cuh)
template <typename T>
static void pinv_device_build(gdsw_precond* m, FactorBuf& F, const gdsw_coarse_factor* f) {
  gdsw_plan* P = m->plan;
  require(P->has_ab && m->has_factors, "device partitioned inverse needs the device factors (GPU LU)");
  const int nsn = f->n_sn;
  std::vector<int32_t> pos_sn(P->n_loc, -1), pos_c(P->n_loc, 0), sn_base(nsn);
  std::vector<int64_t> pan_off(nsn);
  std::vector<int2> rows;
  int64_t pan = 0, smax = 0;
  for (int q = 0; q < nsn; ++q) {
    const int64_t s = f->sn_s[q], r = f->sn_r[q];
    smax = std::max(smax, s);
    for (int64_t c = 0; c < s; ++c) {
      const int64_t g = f->col_ids[f->col_ptr[q] + c];
      pos_sn[g] = q;
      pos_c[g] = (int32_t)c;
    }
    const int64_t g0 = f->col_ids[f->col_ptr[q]];
    const auto it = std::upper_bound(P->h_sub_ptr.begin(), P->h_sub_ptr.end(), g0);
    sn_base[q] = (int32_t)*(it - 1);
    pan_off[q] = pan;
    pan += 2 * (s + r) * s;
    for (int64_t t = 0; t < s + r; ++t) rows.push_back(make_int2(q, (int)t));
  }
  require(smax <= PB_THREADS * PB_J, "partitioned-inverse supernode too wide for the device build");
  DBuf<int32_t> d_pos_sn, d_pos_c, d_sn_base;
  DBuf<int64_t> d_pan_off;
  DBuf<int2> d_rows;
  d_pos_sn.upload(pos_sn);
  d_pos_c.upload(pos_c);
  d_sn_base.upload(sn_base);
  d_pan_off.upload(pan_off);
  d_rows.upload(rows);
  DBuf<double> d_pan(std::max<int64_t>(pan, 1)), dwork(std::max<int64_t>(f->n_values, 1));
  d_pan.zero();
  DBuf<int32_t> bad(1);
  bad.zero();
  const PinvBuildDev B{P->l_ptr.p, P->l_idx32.p, P->u_ptr.p, P->u_idx32.p, d_pos_sn.p, d_pos_c.p,
                       d_sn_base.p, d_pan_off.p, d_rows.p, (int32_t)rows.size()};
  const CoarseFactorDev D = F.dev();
  if (!rows.empty()) {
    k_pinv_fill<T><<<grid_for((int64_t)rows.size(), TB), TB>>>(D, B, (const T*)m->lval.p, (const T*)m->uval.p,
                                                               d_pan.p);
    CK_LAUNCH();
    k_pinv_blocks<T><<<nsn, PB_THREADS>>>(D, B, d_pan.p, dwork.p, (T*)F.vals.p, bad.p);
    CK_LAUNCH();
  }
  CK(cudaDeviceSynchronize());
  require(bad.download()[0] == 0, "matrix is singular", E_LINALG);
  build_fcm<T>(F);
}

extern "C" {

int gdsw_precond_set_local_factor(gdsw_precond* m, const gdsw_coarse_factor* f) {
  return guarded([&] {
    require(f == nullptr || f->n == m->plan->n_loc, "local factor dimension mismatch");
    if (f == nullptr) {
      m->lf = FactorBuf{};
    } else {
      // 128-thread CTAs from 32 blocks up (C3 512 blocks: 92.4 -> 87.8 ms;
      // 64 C3-sized blocks 0.245 -> 0.220 ms); few blocks keep 256 (C1, 8
      // blocks: 4.4 vs 4.56 ms)
      install_factor(m->lf, f, m->dtype, m->es, CF_CM_LOCAL,
                     m->plan->n_sub >= 32 ? CF_NT_LOCAL : CF_NT_COARSE);
      if (!f->values)
        with_dtype(m->dtype, [&](auto tag) { pinv_device_build<decltype(tag)>(m, m->lf, f); });
    }
    m->drop_graphs();
  });
}

int gdsw_precond_apply(gdsw_precond* m, const double* r, double* z, void* stream) {
  return guarded([&] { precond_apply(m, r, z, S(stream)); });
}

int gdsw_precond_local_solve(gdsw_precond* m, const double* r, void* y, int jacobi_iters, void* stream) {
  return guarded([&] {
    require(m->has_factors, "preconditioner has no numeric factors");
    std::lock_guard<std::recursive_mutex> g(m->mu);
    cudaStream_t s = S(stream);
    CK(cudaStreamWaitEvent(s, m->last, 0));
    with_dtype(m->dtype, [&](auto tag) {
      using T = decltype(tag);
      T* out = local_solve<T>(m, r, jacobi_iters, s);
      CK(cudaMemcpyAsync(y, out, m->plan->n_loc * sizeof(T), cudaMemcpyDeviceToDevice, s));
    });
    CK(cudaEventRecord(m->last, s));
  });
}

int gdsw_precond_destroy(gdsw_precond* m) {
  if (m) {
    cudaEventSynchronize(m->last);
    delete m;
  }
  return GDSW_OK;
}

}  // extern "C"

#include "gmres_driver.inc"

extern "C" {

int64_t gdsw_launch_count(void) { return launch_counter().load(); }

int gdsw_prof_enable(int on) {
  return guarded([&] {
    Prof& P = prof();
    std::lock_guard<std::mutex> g(P.mu);
    // events come from a preallocated pool so recording stays ~1 us/launch
    while (on && P.pool.size() < 16384) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      P.pool.push_back(e);
    }
    P.on = on != 0;
  });
}
int gdsw_prof_reset(void) {
  return guarded([&] {
    Prof& P = prof();
    std::lock_guard<std::mutex> g(P.mu);
    for (auto& ph : P.phases) {
      P.resolve(ph);
      ph.ms = 0.0;
      ph.launches = 0;
      ph.bytes = 0.0;
    }
  });
}
int gdsw_prof_count(void) { return (int)prof().phases.size(); }
const char* gdsw_prof_name(int k) {
  Prof& P = prof();
  return (k >= 0 && k < (int)P.phases.size()) ? P.phases[k].name.c_str() : "";
}
int gdsw_prof_read(int k, double* total_ms, int64_t* launches, double* bytes) {
  return guarded([&] {
    Prof& P = prof();
    std::lock_guard<std::mutex> g(P.mu);
    require(k >= 0 && k < (int)P.phases.size(), "no such phase");
    P.resolve(P.phases[k]);
    *total_ms = P.phases[k].ms;
    *launches = P.phases[k].launches;
    *bytes = P.phases[k].bytes;
  });
}

}  // extern "C"
