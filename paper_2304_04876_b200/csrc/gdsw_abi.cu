// libgdsw: C ABI (include/gdsw.h) over the sm_100a kernels of the rGDSW
// solve path. Host-side orchestration only; kernels live in the .cuh files.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/gdsw.h"
#include "coarse.cuh"
#include "common.cuh"
#include "extension.cuh"
#include "fastilu.cuh"
#include "krylov.cuh"
#include "prof.cuh"
#include "sparse.cuh"

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
}  // namespace

// ===========================================================================
// device CSR operator
// ===========================================================================
struct gdsw_csr {
  int64_t nrows = 0, ncols = 0, nnz = 0;
  int dtype = GDSW_F64;
  SellPattern pat;
  DBuf<char> csr_val;   // values in CSR order (A.values indexing for setup gathers)
  DBuf<char> sell_val;  // values in SELL order (SpMV)
  void refresh_sell() {
    with_dtype(dtype, [&](auto tag) {
      using T = decltype(tag);
      k_csr_to_sell<T, T><<<grid_for(nrows, TB), TB>>>(
          (int32_t)nrows, pat.csr_ptr.p, pat.slice_off.p, (const T*)csr_val.p, (T*)sell_val.p, 0,
          (T*)nullptr);
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
  k_sell_spmv<T><<<grid_for(a->nrows, TB), TB, 0, s>>>(a->pat.view(), (const T*)a->sell_val.p, x,
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
    ProfScope ps("spmv", S(stream), (double)a->nnz * (esize(a->dtype) + 4) + (a->nrows + 1) * 4.0 +
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
  DBuf<int32_t> llev_sub, llev_ptr, llev_rows, ulev_sub, ulev_ptr, ulev_rows;
  std::vector<int64_t> row_add;  // block row offset per concatenated row
  std::vector<int64_t> h_l_idx, h_u_idx;
  SellPattern l_sell, u_sell;    // Jacobi layouts (U without its diagonal)
  bool sell_ready = false;
  DBuf<int32_t> sc_ptr, sc_pos;
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
    l_sell.build(n_loc, h_l_ptr.data(), h_l_idx.data(), row_add.data(), 0);
    u_sell.build(n_loc, h_u_ptr.data(), h_u_idx.data(), row_add.data(), 1);
    sell_ready = true;
  }

  LevelSetDev levelset() const {
    return LevelSetDev{sub_ptr.p,  gmap.p,     l_ptr.p,    l_col.p,     u_ptr.p,    u_col.p,
                       llev_sub.p, llev_ptr.p, llev_rows.p, ulev_sub.p, ulev_ptr.p, ulev_rows.p};
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
  // level schedules (block-local rows -> absolute)
  auto levels = [&](const int64_t* lsub, const int64_t* lptr, const int64_t* lrows, DBuf<int32_t>& dsub,
                    DBuf<int32_t>& dptr, DBuf<int32_t>& drows) {
    std::vector<int64_t> sub = vec(lsub, ns + 1);
    int64_t nlev = sub[ns];
    std::vector<int64_t> ptr = vec(lptr, nlev + 1);
    std::vector<int64_t> rows = vec(lrows, d->n_loc);
    std::vector<int32_t> arows(d->n_loc);
    for (int32_t s = 0; s < ns; ++s)
      for (int64_t lv = sub[s]; lv < sub[s + 1]; ++lv)
        for (int64_t t = ptr[lv]; t < ptr[lv + 1]; ++t)
          arows[t] = (int32_t)(rows[t] + P->h_sub_ptr[s]);
    dsub.upload(to_i32(sub.data(), sub.size()));
    dptr.upload(to_i32(ptr.data(), ptr.size()));
    drows.upload(arows);
  };
  levels(d->llev_sub, d->llev_ptr, d->llev_rows, P->llev_sub, P->llev_ptr, P->llev_rows);
  levels(d->ulev_sub, d->ulev_ptr, d->ulev_rows, P->ulev_sub, P->ulev_ptr, P->ulev_rows);
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
    P->chunk_sub.upload(csub);
    P->chunk_row0.upload(crow0);
    P->chunk_nrow.upload(cnrow);
    P->chunk_poff.upload(cpoff);
    P->sub_chunk0.upload(sc0);
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
struct gdsw_precond {
  gdsw_plan* plan = nullptr;
  std::unique_ptr<CoarsePlan> cp;
  int dtype = GDSW_F64;
  size_t es = 8;
  int iters = 5;
  bool has_factors = false, jacobi_ready = false, has_phi = false, has_ainv = false;
  DBuf<char> lval, uval;           // CSR order
  DBuf<char> lsell, usell, udiag;  // Jacobi copies
  DBuf<double> panel64;
  DBuf<char> panel32;              // f32 copy when dtype == F32
  DBuf<char> pgr_val, pgt_val, ainv;
  DBuf<char> xb, x1, x2, pdot, cu, cv;
  std::mutex mu;
  cudaEvent_t last = nullptr;
  ~gdsw_precond() {
    if (last) cudaEventDestroy(last);
    plan_release(plan);
  }
  const void* panel() const { return dtype == GDSW_F32 ? (const void*)panel32.p : (const void*)panel64.p; }

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
                                                         (T*)lsell.p, 0, (T*)nullptr);
      CK_LAUNCH();
      k_csr_to_sell<T, T><<<grid_for(P->n_loc, TB), TB>>>((int32_t)P->n_loc, P->u_sell.csr_ptr.p,
                                                         P->u_sell.slice_off.p, (const T*)uval.p,
                                                         (T*)usell.p, 1, (T*)udiag.p);
      CK_LAUNCH();
    });
    CK(cudaDeviceSynchronize());
    jacobi_ready = true;
  }
};

namespace {

// FastSpTRSV: `iters` Jacobi iterates on L then U; returns the buffer
// holding the block solutions
template <typename T>
T* jacobi_solve(gdsw_precond* m, const double* r, int iters, cudaStream_t s) {
  gdsw_plan* P = m->plan;
  const int32_t n = (int32_t)P->n_loc;
  T* B = (T*)m->xb.p;
  T* X1 = (T*)m->x1.p;
  T* X2 = (T*)m->x2.p;
  SellDev L = P->l_sell.view(), U = P->u_sell.view();
  const unsigned g = grid_for(n, TB);
  const double lbytes = (double)P->nnz_l * (sizeof(T) + 4) + n * (2.0 + 3 * sizeof(T));
  const double ubytes = (double)(P->nnz_u - n) * (sizeof(T) + 4) + n * (2.0 + 3 * sizeof(T));
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
      k_gather_jacobi_lower<T><<<g, TB, 0, s>>>(L, (const T*)m->lsell.p, P->gmap.p, r, B, X1);
      CK_LAUNCH();
    }
    T* cur = X1;
    T* oth = X2;
    for (int t = 2; t < iters; ++t) {
      ProfScope ps("jacobi_lower", s, lbytes);
      k_jacobi_lower<T><<<g, TB, 0, s>>>(L, (const T*)m->lsell.p, B, cur, oth);
      CK_LAUNCH();
      std::swap(cur, oth);
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
    k_jacobi_upper<T><<<g, TB, 0, s>>>(U, (const T*)m->usell.p, (const T*)m->udiag.p, F, cur, oth);
    CK_LAUNCH();
    std::swap(cur, oth);
  }
  return cur;
}

template <typename T>
T* levelset_solve(gdsw_precond* m, const double* r, cudaStream_t s) {
  gdsw_plan* P = m->plan;
  ProfScope ps("levelset", s, (double)(P->nnz_l + P->nnz_u) * (sizeof(T) + 4) + P->n_loc * (8.0 + 3 * sizeof(T)));
  k_levelset<T><<<P->n_sub, 512, 0, s>>>(P->levelset(), (const T*)m->lval.p, (const T*)m->uval.p, r,
                                         (T*)m->x1.p, 0, 1);
  CK_LAUNCH();
  return (T*)m->x1.p;
}

template <typename T>
T* local_solve(gdsw_precond* m, const double* r, int jacobi_iters, cudaStream_t s) {
  gdsw_plan* P = m->plan;
  if (jacobi_iters > 0 || P->method == GDSW_FAST_ILU) {
    m->ensure_jacobi();
    return jacobi_solve<T>(m, r, jacobi_iters > 0 ? jacobi_iters : m->iters, s);
  }
  return levelset_solve<T>(m, r, s);
}

template <typename T>
void apply_T(gdsw_precond* m, const double* r, double* z, cudaStream_t s) {
  gdsw_plan* P = m->plan;
  CoarsePlan* Cp = m->cp.get();
  if (Cp) {
    RestrictDev R = Cp->restrict_dev();
    {
      ProfScope ps("coarse_restrict", s, (double)Cp->panel_entries * sizeof(T) + Cp->n_int_total * 12.0 +
                                             (double)Cp->h_pgt_val.size() * (sizeof(T) + 12));
      if (Cp->K > 0) {
        k_restrict_panels<T><<<Cp->K, TB, 0, s>>>(R, (const T*)m->panel(), r, (T*)m->pdot.p);
        CK_LAUNCH();
      }
      k_restrict_final<T><<<grid_for(Cp->n_c, TB / 32), TB, 0, s>>>(R, (const T*)m->pgt_val.p, r,
                                                                   (const T*)m->pdot.p, (T*)m->cu.p);
      CK_LAUNCH();
    }
    ProfScope ps("coarse_solve", s, (double)Cp->n_c * Cp->n_c * sizeof(T));
    k_coarse_gemv<T><<<grid_for(Cp->n_c, TB / 32), TB, 0, s>>>(Cp->n_c, (const T*)m->ainv.p,
                                                               (const T*)m->cu.p, (T*)m->cv.p);
    CK_LAUNCH();
  }
  T* y = local_solve<T>(m, r, 0, s);
  ProfScope ps("scatter_prolong", s, P->n_loc * (4.0 + sizeof(T)) + (P->n + 1) * 4.0 + P->n * 8.0 +
                                         (Cp ? (double)Cp->panel_entries * sizeof(T) : 0.0));
  ProlongDev pro{};
  if (Cp) pro = Cp->prolong();
  k_scatter_prolong<T><<<grid_for(P->n, TB), TB, 0, s>>>(
      (int32_t)P->n, P->sc_ptr.p, P->sc_pos.p, y, pro, (const T*)m->pgr_val.p,
      (const T*)m->panel(), (const T*)m->cv.p, z);
  CK_LAUNCH();
}

void precond_apply(gdsw_precond* m, const double* r, double* z, cudaStream_t s) {
  require(m->has_factors, "preconditioner has no numeric factors");
  if (m->cp) require(m->has_phi && m->has_ainv, "coarse space is not set up");
  std::lock_guard<std::mutex> g(m->mu);
  CK(cudaStreamWaitEvent(s, m->last, 0));
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
    CK(cudaEventCreateWithFlags(&m->last, cudaEventDisableTiming));
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
    m->pdot.alloc(std::max<int32_t>(cp->K, 1) * m->es);
    m->cu.alloc(std::max<int32_t>(cp->n_c, 1) * m->es);
    m->cv.alloc(std::max<int32_t>(cp->n_c, 1) * m->es);
    m->panel64.alloc(std::max<int64_t>(cp->panel_entries, 1));
    if (m->dtype == GDSW_F32) m->panel32.alloc(std::max<int64_t>(cp->panel_entries, 1) * 4);
    CK(cudaDeviceSynchronize());
    m->cp = std::move(cp);
    m->has_phi = m->has_ainv = false;
  });
}

int gdsw_precond_set_factors(gdsw_precond* m, const void* l_vals, const void* u_vals) {
  return guarded([&] {
    gdsw_plan* P = m->plan;
    if (P->nnz_l) CK(cudaMemcpy(m->lval.p, l_vals, P->nnz_l * m->es, cudaMemcpyHostToDevice));
    if (P->nnz_u) CK(cudaMemcpy(m->uval.p, u_vals, P->nnz_u * m->es, cudaMemcpyHostToDevice));
    m->has_factors = true;
    m->jacobi_ready = false;
    if (P->method == GDSW_FAST_ILU) m->ensure_jacobi();
  });
}

int gdsw_precond_get_factors(const gdsw_precond* m, void* l_vals, void* u_vals) {
  return guarded([&] {
    gdsw_plan* P = m->plan;
    if (P->nnz_l) CK(cudaMemcpy(l_vals, m->lval.p, P->nnz_l * m->es, cudaMemcpyDeviceToHost));
    if (P->nnz_u) CK(cudaMemcpy(u_vals, m->uval.p, P->nnz_u * m->es, cudaMemcpyDeviceToHost));
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
    m->jacobi_ready = false;
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

int gdsw_precond_set_coarse_inverse(gdsw_precond* m, const double* a0inv) {
  return guarded([&] {
    require(m->cp != nullptr, "preconditioner has no coarse structure");
    CoarsePlan* P = m->cp.get();
    std::vector<double> h(a0inv, a0inv + (size_t)P->n_c * P->n_c);
    with_dtype(m->dtype, [&](auto tag) { upload_cast<decltype(tag)>(m->ainv, h); });
    m->has_ainv = true;
  });
}

int gdsw_precond_apply(gdsw_precond* m, const double* r, double* z, void* stream) {
  return guarded([&] { precond_apply(m, r, z, S(stream)); });
}

int gdsw_precond_local_solve(gdsw_precond* m, const double* r, void* y, int jacobi_iters, void* stream) {
  return guarded([&] {
    require(m->has_factors, "preconditioner has no numeric factors");
    std::lock_guard<std::mutex> g(m->mu);
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

// ===========================================================================
// GMRES (krylov.py)
// ===========================================================================
struct gdsw_workspace {
  int64_t n = 0;
  int32_t R = 0;
  int nblk = 0;
  DBuf<double> V, Zm, W, MC, ZC, XC, RES, partial, dots, coef;
  DBuf<unsigned> counter;  // last-block ticket of k_block_dot (self-resetting)
  double* h_dots = nullptr;
  double* h_coef = nullptr;
  size_t n_hdots = 0, n_hcoef = 0;
  ~gdsw_workspace() {
    if (h_dots) cudaFreeHost(h_dots);
    if (h_coef) cudaFreeHost(h_coef);
  }
};

namespace {

constexpr double BREAKDOWN_REL = 1e-14;  // krylov.py:42

struct Solver {
  const gdsw_csr* a;
  gdsw_precond* m;
  const gdsw_csr* mcsr;
  const double* b;
  cudaStream_t s;
  gdsw_workspace* ws;
  int64_t n;
  int iter_red = 0, res_red = 0;

  unsigned vgrid() const { return grid_for(n, TB, (int64_t)num_sms() * 8); }

  void A(const double* x, double* y) {
    ProfScope ps("spmv", s, (double)a->nnz * 12.0 + (a->nrows + 1) * 4.0 + 2.0 * n * 8.0);
    spmv_T<double>(a, x, nullptr, y, 0, 1.0, 0.0, s);
  }
  void resid(const double* x, double* r) {
    ProfScope ps("spmv", s, (double)a->nnz * 12.0 + (a->nrows + 1) * 4.0 + 3.0 * n * 8.0);
    spmv_T<double>(a, x, b, r, 1, -1.0, 1.0, s);
  }
  void M(const double* x, double* y) {
    if (m) {
      precond_apply(m, x, y, s);
    } else if (mcsr) {
      ProfScope ps("spmv", s, (double)mcsr->nnz * 12.0 + 2.0 * n * 8.0);
      spmv_T<double>(mcsr, x, nullptr, y, 0, 1.0, 0.0, s);
    } else {
      CK(cudaMemcpyAsync(y, x, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
  }
  // rows V[0..nr) (+ v itself when self) against v (and z): host av/az of length nr+1
  void block(const double* Vb, int nr, bool self, const double* v, const double* z,
             std::vector<double>& av, std::vector<double>& az) {
    const int W2 = 2 * (KDOT_ROWS + 1);
    int nch = std::max(1, (nr + KDOT_ROWS - 1) / KDOT_ROWS);
    {
      ProfScope ps("block_dot", s, (double)(nr + (self ? 1 : 0) + (z ? 1 : 0)) * n * 8.0);
      for (int ci = 0; ci < nch; ++ci) {
        int r0 = ci * KDOT_ROWS;
        int nrc = std::min(KDOT_ROWS, nr - r0);
        if (nrc < 0) nrc = 0;
        int self_here = (self && ci == nch - 1) ? 1 : 0;
        k_block_dot<<<ws->nblk, KDOT_THREADS, 0, s>>>(n, Vb ? Vb + (int64_t)r0 * n : nullptr, n, nrc,
                                                      self_here, v, z, ws->partial.p,
                                                      ws->dots.p + (int64_t)ci * W2, ws->counter.p);
        CK_LAUNCH();
      }
    }
    CK(cudaMemcpyAsync(ws->h_dots, ws->dots.p, (size_t)nch * W2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    av.assign(nr + 1, 0.0);
    az.assign(nr + 1, 0.0);
    for (int r = 0; r < nr; ++r) {
      int ci = r / KDOT_ROWS, rr = r % KDOT_ROWS;
      av[r] = ws->h_dots[ci * W2 + 2 * rr];
      az[r] = ws->h_dots[ci * W2 + 2 * rr + 1];
    }
    if (self) {
      av[nr] = ws->h_dots[(nch - 1) * W2 + 2 * KDOT_ROWS];
      az[nr] = ws->h_dots[(nch - 1) * W2 + 2 * KDOT_ROWS + 1];
    }
  }
  double norm(const double* v) {
    std::vector<double> av, az;
    block(nullptr, 0, true, v, nullptr, av, az);
    return std::sqrt(av[0]);
  }
  void put_coef(const std::vector<double>& c) {
    std::copy(c.begin(), c.end(), ws->h_coef);
    CK(cudaMemcpyAsync(ws->coef.p, ws->h_coef, c.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  }
  void xupdate(const double* x, int mcols, const std::vector<double>& y, double* xo) {
    put_coef(y);
    ProfScope ps("x_update", s, (double)(mcols + 2) * n * 8.0);
    k_x_update<<<vgrid(), TB, 0, s>>>(n, x, ws->Zm.p, n, mcols, ws->coef.p, xo);
    CK_LAUNCH();
  }
};

double rotation_hypot(double a, double b) { return std::hypot(a, b); }

// krylov.py:118-130
double process_column(std::vector<double>& h, int R, std::vector<double>& cs, std::vector<double>& sn,
                      std::vector<double>& g, int j) {
  auto H = [&](int i, int k) -> double& { return h[(size_t)i * R + k]; };
  for (int i = 0; i < j; ++i) {
    double t = cs[i] * H(i, j) + sn[i] * H(i + 1, j);
    H(i + 1, j) = -sn[i] * H(i, j) + cs[i] * H(i + 1, j);
    H(i, j) = t;
  }
  double r = rotation_hypot(H(j, j), H(j + 1, j));
  if (r == 0.0) {
    cs[j] = 1.0;
    sn[j] = 0.0;
  } else {
    cs[j] = H(j, j) / r;
    sn[j] = H(j + 1, j) / r;
  }
  H(j, j) = cs[j] * H(j, j) + sn[j] * H(j + 1, j);
  H(j + 1, j) = 0.0;
  g[j + 1] = -sn[j] * g[j];
  g[j] = cs[j] * g[j];
  return std::fabs(g[j + 1]);
}

// krylov.py:133-138
std::vector<double> solve_y(const std::vector<double>& h, int R, const std::vector<double>& g, int m) {
  std::vector<double> y(m, 0.0);
  for (int i = m - 1; i >= 0; --i) {
    double dot = 0.0;
    for (int k = i + 1; k < m; ++k) dot += h[(size_t)i * R + k] * y[k];
    y[i] = (g[i] - dot) / h[(size_t)i * R + i];
  }
  return y;
}

struct Outcome {
  int it = 0;
  bool converged = false;
  int restarts = 0;
  std::vector<double> history{1.0};
  std::vector<std::pair<int, double>> true_res;
};

void copy_vec(double* dst, const double* src, int64_t n, cudaStream_t s) {
  if (dst != src) CK(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
}

void gmres_single_reduce(Solver& C, double* x, bool x0nz, const gdsw_krylov_cfg& cfg, Outcome& o) {
  const int R = cfg.restart;
  const int64_t n = C.n;
  double* V = C.ws->V.p;
  double* Zm = C.ws->Zm.p;
  double* W = C.ws->W.p;
  double* MC = C.ws->MC.p;
  double* ZC = C.ws->ZC.p;
  double* XC = C.ws->XC.p;
  std::vector<double> h((size_t)(R + 1) * R, 0.0), g(R + 1, 0.0), cs(R, 0.0), sn(R, 0.0);
  std::vector<double> av, az;
  bool have_denom = false;
  double denom = 0.0, bnorm = 0.0;
  auto H = [&](int i, int k) -> double& { return h[(size_t)i * R + k]; };
  while (true) {
    C.resid(x, W);
    o.restarts++;
    C.M(W, MC);
    C.A(MC, ZC);
    std::fill(g.begin(), g.end(), 0.0);
    for (int j = 0; j <= R; ++j) {
      const bool last = j == R;
      C.block(V, j, true, W, last ? nullptr : ZC, av, az);
      const double b2 = av[j], q = az[j];
      if (j == 0) C.res_red++; else C.iter_red++;
      double aa = 0.0;
      for (int r = 0; r < j; ++r) aa += av[r] * av[r];
      const double delta2 = b2 - aa;
      const double delta = delta2 > 0.0 ? std::sqrt(delta2) : 0.0;
      if (j == 0) {
        if (!have_denom) {
          have_denom = true;
          denom = delta;
          if (x0nz) {
            C.res_red++;
            bnorm = [&] {
              std::vector<double> bv, bz;
              C.block(nullptr, 0, true, C.b, nullptr, bv, bz);
              return std::sqrt(bv[0]);
            }();
          } else {
            bnorm = delta;
          }
          if (delta <= BREAKDOWN_REL * bnorm) { o.it = 0; o.converged = true; return; }
        } else {
          o.true_res.emplace_back(o.it, delta / denom);
        }
        if (delta / denom <= cfg.rel_tol) { o.converged = true; return; }
        g[0] = delta;
      } else {
        for (int r = 0; r < j; ++r) H(r, j - 1) += av[r];
        H(j, j - 1) = delta;
        o.it++;
        double est = process_column(h, R, cs, sn, g, j - 1);
        o.history.push_back(est / denom);
        const bool breakdown = delta <= BREAKDOWN_REL * bnorm;
        if (breakdown || est / denom <= cfg.rel_tol || o.it >= cfg.max_iters) {
          std::vector<double> y = solve_y(h, R, g, j);
          C.xupdate(x, j, y, XC);
          C.resid(XC, C.ws->RES.p);
          C.res_red++;
          double tr = C.norm(C.ws->RES.p);
          o.true_res.emplace_back(o.it, tr / denom);
          if (tr / denom <= cfg.rel_tol) { copy_vec(x, XC, n, C.s); o.converged = true; return; }
          if (breakdown || o.it >= cfg.max_iters) { copy_vec(x, XC, n, C.s); o.converged = false; return; }
        }
      }
      if (last) break;
      std::vector<double> coef(2 * j);
      double ap = 0.0;
      for (int r = 0; r < j; ++r) ap += av[r] * az[r];
      const double corr = (q - ap) / (delta * delta);
      for (int r = 0; r < j; ++r) {
        coef[r] = av[r];
        coef[j + r] = az[r] / delta;
        H(r, j) = az[r] / delta;
      }
      H(j, j) = corr;
      C.put_coef(coef);
      {
        ProfScope ps("sr_update", C.s, (double)(2 * j + 6) * n * 8.0);
        k_sr_update<<<C.vgrid(), TB, 0, C.s>>>(n, V, Zm, n, j, C.ws->coef.p, delta, corr, W, MC, ZC);
        CK_LAUNCH();
      }
      if (j + 1 <= R - 1) {
        C.M(W, MC);
        C.A(MC, ZC);
      }
    }
    std::vector<double> y = solve_y(h, R, g, R);
    C.xupdate(x, R, y, x);
  }
}

void gmres_classic(Solver& C, double* x, bool x0nz, const gdsw_krylov_cfg& cfg, Outcome& o) {
  const int R = cfg.restart;
  const int64_t n = C.n;
  double* V = C.ws->V.p;
  double* Zm = C.ws->Zm.p;
  double* W = C.ws->W.p;
  double* XC = C.ws->XC.p;
  double* RES = C.ws->RES.p;
  std::vector<double> h((size_t)(R + 1) * R, 0.0), g(R + 1, 0.0), cs(R, 0.0), sn(R, 0.0);
  std::vector<double> av, az;
  bool have_denom = false;
  double denom = 0.0, bnorm = 0.0;
  auto H = [&](int i, int k) -> double& { return h[(size_t)i * R + k]; };
  while (true) {
    C.resid(x, RES);
    const double beta = C.norm(RES);
    C.res_red++;
    o.restarts++;
    if (!have_denom) {
      have_denom = true;
      denom = beta;
      if (x0nz) {
        C.res_red++;
        bnorm = C.norm(C.b);
      } else {
        bnorm = beta;
      }
      if (beta <= BREAKDOWN_REL * bnorm) { o.it = 0; o.converged = true; return; }
    } else {
      o.true_res.emplace_back(o.it, beta / denom);
    }
    if (beta / denom <= cfg.rel_tol) { o.converged = true; return; }
    k_scale_copy<<<C.vgrid(), TB, 0, C.s>>>(n, RES, beta, V);
    CK_LAUNCH();
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    for (int j = 0; j < R; ++j) {
      double* vj = V + (int64_t)j * n;
      double* zj = Zm + (int64_t)j * n;
      C.M(vj, zj);
      C.A(zj, W);
      if (cfg.orthogonalization == GDSW_MGS) {
        for (int i = 0; i <= j; ++i) {
          C.block(V + (int64_t)i * n, 1, false, W, nullptr, av, az);
          C.iter_red++;
          const double hij = av[0];
          k_axpy_scalar<<<C.vgrid(), TB, 0, C.s>>>(n, hij, V + (int64_t)i * n, W);
          CK_LAUNCH();
          H(i, j) = hij;
        }
      } else {
        std::vector<double> c1, c2, t;
        C.block(V, j + 1, false, W, nullptr, c1, t);
        C.iter_red++;
        c1.resize(j + 1);
        C.put_coef(c1);
        k_multi_axpy<<<C.vgrid(), TB, 0, C.s>>>(n, V, n, j + 1, C.ws->coef.p, W);
        CK_LAUNCH();
        C.block(V, j + 1, false, W, nullptr, c2, t);
        C.iter_red++;
        c2.resize(j + 1);
        C.put_coef(c2);
        k_multi_axpy<<<C.vgrid(), TB, 0, C.s>>>(n, V, n, j + 1, C.ws->coef.p, W);
        CK_LAUNCH();
        for (int i = 0; i <= j; ++i) H(i, j) = c1[i] + c2[i];
      }
      const double nrm = C.norm(W);
      C.iter_red++;
      H(j + 1, j) = nrm;
      o.it++;
      double est = process_column(h, R, cs, sn, g, j);
      o.history.push_back(est / denom);
      const bool breakdown = nrm <= BREAKDOWN_REL * bnorm;
      if (breakdown || est / denom <= cfg.rel_tol || o.it >= cfg.max_iters) {
        std::vector<double> y = solve_y(h, R, g, j + 1);
        C.xupdate(x, j + 1, y, XC);
        C.resid(XC, RES);
        C.res_red++;
        double tr = C.norm(RES);
        o.true_res.emplace_back(o.it, tr / denom);
        if (tr / denom <= cfg.rel_tol) { copy_vec(x, XC, n, C.s); o.converged = true; return; }
        if (breakdown || o.it >= cfg.max_iters) { copy_vec(x, XC, n, C.s); o.converged = false; return; }
      }
      if (j + 1 < R) {
        k_scale_copy<<<C.vgrid(), TB, 0, C.s>>>(n, W, nrm, V + (int64_t)(j + 1) * n);
        CK_LAUNCH();
      }
    }
    std::vector<double> y = solve_y(h, R, g, R);
    C.xupdate(x, R, y, x);
  }
}

}  // namespace

extern "C" {

int gdsw_workspace_create(gdsw_workspace** out, int64_t n, int32_t restart) {
  return guarded([&] {
    require(restart >= 1, "restart must be at least 1");
    auto w = std::make_unique<gdsw_workspace>();
    w->n = n;
    w->R = restart;
    w->nblk = 2 * num_sms();
    const size_t nn = std::max<int64_t>(n, 1);
    w->V.alloc(nn * (restart + 1));
    w->Zm.alloc(nn * restart);
    w->W.alloc(nn);
    w->MC.alloc(nn);
    w->ZC.alloc(nn);
    w->XC.alloc(nn);
    w->RES.alloc(nn);
    const int W2 = 2 * (KDOT_ROWS + 1);
    const int nch = (restart + 1 + KDOT_ROWS - 1) / KDOT_ROWS + 1;
    w->partial.alloc((size_t)w->nblk * W2);
    w->dots.alloc((size_t)nch * W2);
    w->counter.alloc(1);
    w->counter.zero();
    CK(cudaDeviceSynchronize());
    w->coef.alloc(2 * (size_t)restart + 4);
    w->n_hdots = (size_t)nch * W2;
    w->n_hcoef = 2 * (size_t)restart + 4;
    CK(cudaMallocHost(&w->h_dots, w->n_hdots * sizeof(double)));
    CK(cudaMallocHost(&w->h_coef, w->n_hcoef * sizeof(double)));
    *out = w.release();
  });
}

int gdsw_workspace_destroy(gdsw_workspace* ws) {
  delete ws;
  return GDSW_OK;
}

int gdsw_gmres(const gdsw_csr* a, gdsw_precond* m, const gdsw_csr* m_csr, const double* b, double* x,
               int x0_nonzero, const gdsw_krylov_cfg* cfg, gdsw_workspace* ws, gdsw_solve_report* rep,
               double* history, int32_t* true_it, double* true_res, int32_t cap, void* stream) {
  return guarded([&] {
    require(a->dtype == GDSW_F64, "GMRES runs on a float64 operator", E_TYPE);
    require(a->nrows == a->ncols, "operator dimensions do not match the vector");
    require(ws->n == a->nrows && ws->R >= cfg->restart, "workspace does not match the solve");
    if (m) require(m->plan->n == a->nrows, "operator dimensions do not match the vector");
    if (m_csr) require(m_csr->dtype == GDSW_F64 && m_csr->nrows == a->nrows, "operator dimensions do not match the vector");
    Solver C{a, m, m_csr, b, S(stream), ws, a->nrows};
    Outcome o;
    if (cfg->variant == GDSW_SINGLE_REDUCE)
      gmres_single_reduce(C, x, x0_nonzero != 0, *cfg, o);
    else
      gmres_classic(C, x, x0_nonzero != 0, *cfg, o);
    CK(cudaStreamSynchronize(C.s));
    rep->iterations = o.it;
    rep->converged = o.converged ? 1 : 0;
    rep->iteration_reductions = C.iter_red;
    rep->residual_reductions = C.res_red;
    rep->reduction_count = C.iter_red + C.res_red;
    rep->restarts = o.restarts;
    rep->n_history = (int32_t)std::min<size_t>(o.history.size(), cap);
    rep->n_true = (int32_t)std::min<size_t>(o.true_res.size(), cap);
    for (int k = 0; k < rep->n_history; ++k) history[k] = o.history[k];
    for (int k = 0; k < rep->n_true; ++k) {
      true_it[k] = o.true_res[k].first;
      true_res[k] = o.true_res[k].second;
    }
  });
}

int gdsw_block_dot(const double* V, int64_t ldv, int32_t j, const double* v, const double* z, int64_t n,
                   double* out, void* stream) {
  return guarded([&] {
    require(ldv == n || j == 0, "block_dot expects contiguous rows (ldv == n)");
    gdsw_workspace ws;
    ws.n = n;
    ws.nblk = 2 * num_sms();
    const int W2 = 2 * (KDOT_ROWS + 1);
    const int nch = std::max(1, (j + KDOT_ROWS - 1) / KDOT_ROWS);
    ws.partial.alloc((size_t)ws.nblk * W2);
    ws.dots.alloc((size_t)nch * W2);
    ws.counter.alloc(1);
    ws.counter.zero();
    CK(cudaDeviceSynchronize());
    CK(cudaMallocHost(&ws.h_dots, (size_t)nch * W2 * sizeof(double)));
    Solver C{nullptr, nullptr, nullptr, nullptr, S(stream), &ws, n};
    std::vector<double> av, az;
    C.block(V, j, true, v, z, av, az);
    for (int r = 0; r <= j; ++r) {
      out[r] = av[r];
      out[j + 1 + r] = az[r];
    }
  });
}

// ---------------------------------------------------------------------------
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
