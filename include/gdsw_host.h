/*
 * gdsw_host.h — host-side (CPU) symbolic / setup runtime of the B200 rGDSW
 * solve path.  Everything here is pattern work or setup-time numerics that
 * the north star keeps on the host ("only ordering and symbolic analysis stay
 * on the host"); none of it runs inside the GMRES iteration.
 *
 * Each entry point restates a loop kernel of the reference package
 * (schwarzdd, /root/reference/pkg/src/schwarzdd) so that index sets, fill
 * patterns and level schedules come out bit-identical:
 *
 *   gh_node_graph          _kernels.py:152-179   node_graph
 *   gh_expand_layers       _kernels.py:182-206   expand_layers
 *   gh_nested_dissection   local_solvers.py:61-143 (_symmetrized_pattern,
 *                          _components, _peripheral_levels, _dissect)
 *   gh_symbolic_lu         local_solvers.py:205-225 + _kernels.py:233-301
 *   gh_symbolic_iluk       local_solvers.py:228-243 + _kernels.py:304-393
 *   gh_level_schedule      local_solvers.py:183-188 + _kernels.py:396-422
 *   gh_csr_gather          _kernels.py:118-149   csr_gather
 *   gh_transpose_pattern   _kernels.py:284-301   pattern_transpose
 *   gh_spgemm_{f64,f32}    _kernels.py:51-94     spgemm_count / spgemm_fill
 *   gh_lu_numeric_{f64,f32}_kernels.py:429-466   lu_numeric
 *   gh_align_pattern       _kernels.py:529-544   align_pattern
 *   gh_fastilu_plan        _kernels.py:547-617   (the merge order of
 *                          _sparse_dot_bounded, flattened into pair lists)
 *   gh_classify_interface  decomposition.py:173-250 (closure sets, classes,
 *                          connected pieces, vertex/edge/face kinds)
 *
 * Variable-length outputs come back in an opaque gh_result holding a list of
 * int64 / float64 arrays; the caller reads sizes, copies, and frees it.
 * All functions return 0 on success, nonzero on error (message via
 * gh_last_error()).
 */
#ifndef GDSW_HOST_H
#define GDSW_HOST_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct gh_result gh_result;

const char* gh_last_error(void);
int64_t gh_result_count(const gh_result* r);
int64_t gh_result_size(const gh_result* r, int64_t k);
int gh_result_kind(const gh_result* r, int64_t k);           /* 0 int64, 1 float64, 2 float32 */
int gh_result_copy(const gh_result* r, int64_t k, void* dst);
void gh_result_free(gh_result* r);

int gh_node_graph(int64_t n_nodes, int64_t dpn, const int64_t* a_ptr,
                  const int64_t* a_idx, gh_result** out);      /* {ptr, idx} */
int gh_expand_layers(int64_t n, const int64_t* g_ptr, const int64_t* g_idx,
                     uint8_t* mask, int64_t layers);
int gh_overlap_sets(int64_t n_nodes, const int64_t* g_ptr, const int64_t* g_idx,
                    const int64_t* node_owner, int64_t n_parts, int64_t n_subs,
                    const int64_t* subs, int64_t layers, gh_result** out); /* {ptr, nodes} */
int gh_nested_dissection(int64_t n, const int64_t* a_ptr, const int64_t* a_idx,
                         int64_t leaf_size, int64_t* perm_out);
int gh_symbolic_lu(int64_t n, const int64_t* a_ptr, const int64_t* a_idx,
                   const int64_t* perm, gh_result** out); /* {l_ptr,l_idx,u_ptr,u_idx} */
int gh_symbolic_iluk(int64_t n, const int64_t* a_ptr, const int64_t* a_idx,
                     const int64_t* perm, int64_t fill_level, gh_result** out);
int gh_level_schedule(int64_t n, const int64_t* ptr, const int64_t* idx,
                      int upper, int64_t* level_out, gh_result** out); /* {level_ptr, level_rows} */
int gh_csr_gather(int64_t m, const int64_t* a_ptr, const int64_t* a_idx,
                  const int64_t* rows, const int64_t* col_map,
                  gh_result** out);                          /* {ptr, idx, src} */
int gh_transpose_pattern(int64_t n_rows, int64_t n_cols, const int64_t* ptr,
                         const int64_t* idx, gh_result** out); /* {t_ptr,t_idx,t_src} */
int gh_spgemm_f64(int64_t n_rows, int64_t n_cols,
                  const int64_t* a_ptr, const int64_t* a_idx, const double* a_val,
                  const int64_t* b_ptr, const int64_t* b_idx, const double* b_val,
                  gh_result** out);                          /* {ptr, idx, val} */
int gh_spgemm_f32(int64_t n_rows, int64_t n_cols,
                  const int64_t* a_ptr, const int64_t* a_idx, const float* a_val,
                  const int64_t* b_ptr, const int64_t* b_idx, const float* b_val,
                  gh_result** out);
int64_t gh_lu_numeric_f64(int64_t n, const int64_t* l_ptr, const int64_t* l_idx,
                          const int64_t* u_ptr, const int64_t* u_idx,
                          const int64_t* a_ptr, const int64_t* a_idx,
                          const double* a_val, double* l_val, double* u_val,
                          double pivot_tol);
int64_t gh_lu_numeric_f32(int64_t n, const int64_t* l_ptr, const int64_t* l_idx,
                          const int64_t* u_ptr, const int64_t* u_idx,
                          const int64_t* a_ptr, const int64_t* a_idx,
                          const float* a_val, float* l_val, float* u_val,
                          double pivot_tol);
/* y <- alpha*A x + beta*y, rows in order (_kernels.py:23-31); host-side
 * input construction only (b = A x*), never on the GMRES path */
int gh_spmv_f64(int64_t n, const int64_t* ptr, const int64_t* idx, const double* val,
                const double* x, double* y, double alpha, double beta);
int gh_spmv_f32(int64_t n, const int64_t* ptr, const int64_t* idx, const float* val,
                const float* x, float* y, float alpha, float beta);
int gh_align_pattern(int64_t n, const int64_t* a_ptr, const int64_t* a_idx,
                     const int64_t* f_ptr, const int64_t* f_idx, int64_t* out);
int gh_fastilu_plan(int64_t n, const int64_t* l_ptr, const int64_t* l_idx,
                    const int64_t* u_ptr, const int64_t* u_idx,
                    const int64_t* a_ptr, const int64_t* a_idx,
                    gh_result** out);
/* {entry_ptr, pair_l, pair_u, res_ptr, res_pair_l, res_pair_u, res_tail_l,
 *  res_tail_u}: for every L entry then every U entry, the (L pos, U pos)
 *  products of the bounded sparse dot in merge (ascending k) order; and for
 *  every A entry the products of fastilu_residual plus its tail term. */
int gh_classify_interface(int64_t n_nodes, const int64_t* g_ptr,
                          const int64_t* g_idx, const int64_t* node_owner,
                          gh_result** out);
/* {iface_nodes, mult, piece_ptr, piece_nodes, key_ptr, keys, kind} */
/* supernodal partitioned inverses of nblk exact-LU factors in one batch
 * (the device solve of coarse_factor.cuh): block b has blk_n[b] rows, its
 * CSR L (strictly lower, unit diagonal implied) at lp + lp_off[b] /
 * li, lv + lnz_off[b] and U (diagonal first) at up + up_off[b] / ui, uv +
 * unz_off[b], in its own ND-permuted numbering; blk_base[b] = its offset in
 * the concatenated block vector. Result: {level_ptr, sn_s, sn_r, col_ptr,
 * col_ids, row_ptr, row_ids, d_off, m_off, n_off, values (f64), in_ptr,
 * in_idx, out_ptr, out_idx} -- include/gdsw.h gdsw_coarse_factor. with_values = 0:
 * the structure only (lv / uv unused, values empty; the device fills the
 * blocks from its own factors, gdsw_precond_set_local_factor). */
int gh_partitioned_inverse(int64_t nblk, const int64_t* blk_n, const int64_t* blk_base,
                           const int64_t* lp_off, const int64_t* lnz_off, const int64_t* up_off,
                           const int64_t* unz_off, const int64_t* lp, const int64_t* li,
                           const double* lv, const int64_t* up, const int64_t* ui,
                           const double* uv, int64_t relax, double zero_frac, int64_t threads,
                           int with_values, gh_result** out);

#ifdef __cplusplus
}
#endif
#endif
