/*
 * gdsw.h — C ABI of libgdsw.so, the B200 (sm_100a) solve path of the
 * two-level rGDSW Schwarz preconditioner with single-reduce GMRES.
 *
 * This is the drop-in boundary. The reference (schwarzdd, pure Python) has
 * no FFI of its own; its boundary is the Python duck-typed interface listed
 * next to each entry point below. A caller binds these with ctypes
 * (see INTEGRATION.md); paper_2304_04876_b200/device.py is that binding.
 *
 * Conventions
 *  - every entry point returns an int status (GDSW_OK = 0); on failure the
 *    message is in gdsw_last_error() (thread-local) and the status names the
 *    Python exception the reference raises for the same condition;
 *  - vectors passed to apply / spmv / gmres are caller-owned DEVICE
 *    pointers; setup descriptors carry HOST arrays (int64 like the
 *    reference's index maps, float64 values) that the library copies;
 *  - `stream` is a cudaStream_t (NULL = legacy default stream); all work of
 *    a call is enqueued on it, setup calls synchronize before returning;
 *  - dtype: GDSW_F64 or GDSW_F32 (the reference's "double"/"single"
 *    preconditioner precision, schwarz.py:57-73).
 */
#ifndef GDSW_H
#define GDSW_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define GDSW_ABI_VERSION 1

enum gdsw_status {
  GDSW_OK = 0,
  GDSW_E_VALUE = 1,  /* ValueError            (schwarz.py:297-298, 219-221, 243-245) */
  GDSW_E_LINALG = 2, /* numpy.linalg.LinAlgError (local_solvers.py:320-324)        */
  GDSW_E_FLOAT = 3,  /* FloatingPointError    (local_solvers.py:389-394)           */
  GDSW_E_ARITH = 4,  /* ArithmeticError       (coarse_space.py:198-202)            */
  GDSW_E_CUDA = 5,   /* RuntimeError: driver / launch failure                      */
  GDSW_E_TYPE = 6    /* TypeError             (krylov.py:88-100)                   */
};
enum gdsw_dtype { GDSW_F64 = 0, GDSW_F32 = 1 };
enum gdsw_method { GDSW_EXACT_LU = 0, GDSW_ILU_K = 1, GDSW_FAST_ILU = 2 };
enum gdsw_variant { GDSW_CLASSIC = 0, GDSW_SINGLE_REDUCE = 1 };
enum gdsw_orth { GDSW_MGS = 0, GDSW_CGS2 = 1 };

typedef struct gdsw_csr gdsw_csr;
typedef struct gdsw_plan gdsw_plan;
typedef struct gdsw_precond gdsw_precond;
typedef struct gdsw_workspace gdsw_workspace;

const char* gdsw_last_error(void);
int gdsw_abi_version(void);

/* ------------------------------------------------------------------------
 * Device CSR operator.
 * Replaces CsrMatrix + spmv / __matmul__ (sparse_core.py:41-82, 117-131,
 * 186-204; _kernels.py:23-31). Stored as SELL-32; y = alpha*A x + beta*y in
 * the matrix element type, rows accumulated in column order (bit-identical
 * to the reference loop).
 * ---------------------------------------------------------------------- */
int gdsw_csr_create(gdsw_csr** out, int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                    const int64_t* col_idx, const void* values, int dtype);
int gdsw_csr_set_values(gdsw_csr* a, const void* values); /* same pattern refill */
int gdsw_csr_spmv(const gdsw_csr* a, const void* x, void* y, double alpha, double beta,
                  void* stream);
int gdsw_csr_destroy(gdsw_csr* a);

/* ------------------------------------------------------------------------
 * Symbolic plan = PreconditionerSkeleton (schwarz.py:84-99, 147-203) in the
 * batched-subdomain device layout: concatenated overlap maps with the
 * orderings folded in, factor patterns, level schedules, the FastILU
 * product plan, the owner-computes scatter map and the coarse structure.
 * Pattern-only; shared by every preconditioner built on it.
 * ---------------------------------------------------------------------- */
typedef struct {
  int64_t n;          /* vector length */
  int32_t n_sub;
  int32_t method;     /* gdsw_method */
  int64_t n_loc;      /* sum of overlapped block sizes (N_Omega) */
  const int64_t* sub_ptr;   /* [n_sub+1] block row offsets                      */
  const int64_t* gmap;      /* [n_loc] global dof of block row k: dofs_i[perm_i[k]] */
  const int64_t* l_ptr;     /* [n_loc+1] concatenated strict-L rows             */
  const int64_t* l_idx;     /* block-local column                               */
  const int64_t* u_ptr;     /* [n_loc+1] concatenated U rows, diagonal first    */
  const int64_t* u_idx;
  const int64_t* llev_sub;  /* [n_sub+1] offsets into llev_ptr                  */
  const int64_t* llev_ptr;  /* [levels+1] offsets into llev_rows                */
  const int64_t* llev_rows; /* [n_loc] block-local row ids                      */
  const int64_t* ulev_sub;
  const int64_t* ulev_ptr;
  const int64_t* ulev_rows;
  /* FastILU product plan (method == GDSW_FAST_ILU), concatenated positions */
  const int64_t* a_of;      /* [nnz_l+nnz_u] A.values index of the entry, -1 = fill */
  const int64_t* fi_ptr;    /* [nnz_l+nnz_u+1]                                  */
  const int64_t* fi_pl;     /* L position of each product                       */
  const int64_t* fi_pu;     /* U position of each product                       */
  int64_t n_res;            /* residual terms = block-A entries                 */
  const int64_t* res_sub_ptr; /* [n_sub+1]                                      */
  const int64_t* res_a;     /* [n_res] A.values index                           */
  const int64_t* res_ptr;   /* [n_res+1]                                        */
  const int64_t* res_pl;
  const int64_t* res_pu;
  const int64_t* res_tl;    /* -1 when the tail term is a U entry               */
  const int64_t* res_tu;
} gdsw_local_desc;

typedef struct {
  int32_t n_c;              /* coarse dimension                                 */
  int64_t n_gamma;
  const int64_t* gamma_rows; /* [n_gamma] sorted interface dofs                 */
  const int64_t* pg_ptr;    /* [n_gamma+1] Phi rows on the interface            */
  const int64_t* pg_col;
  const double* pg_val;     /* copied bitwise from the scaled null space        */
  const int64_t* int_ptr;   /* [n_sub+1] interior rows per subdomain            */
  const int64_t* int_rows;
  const int64_t* col_ptr;   /* [n_sub+1] coarse columns touching each interior  */
  const int64_t* col_ids;
  const int64_t* aii_ptr;   /* [n_int+1] A_{I_s I_s}, local interior columns    */
  const int64_t* aii_col;
  const int64_t* aii_src;   /* A.values index                                   */
  const int64_t* aig_ptr;   /* [n_int+1] A_{I_s Gamma}, gamma positions         */
  const int64_t* aig_col;
  const int64_t* aig_src;
} gdsw_coarse_desc;

int gdsw_plan_create(gdsw_plan** out, const gdsw_local_desc* local);
/* permuted block pattern of A for the GPU numeric LU (exact_lu / ilu_k):
 * ab_ptr[n_loc+1] over the concatenated permuted block rows, ab_idx the
 * block-local column, ab_src the A.values position of each entry
 * (permute_symmetric + extract_submatrix, local_solvers.py:306-327) */
int gdsw_plan_set_block_pattern(gdsw_plan* p, const int64_t* ab_ptr, const int64_t* ab_idx,
                                const int64_t* ab_src);
int gdsw_plan_destroy(gdsw_plan* p);

/* ------------------------------------------------------------------------
 * Numeric preconditioner = TwoLevelPreconditioner (schwarz.py:130-144,
 * 213-287). Values live in one device arena per preconditioner.
 * ---------------------------------------------------------------------- */
int gdsw_precond_create(gdsw_precond** out, gdsw_plan* plan, int dtype, int trisolve_iters);
/* coarse structure of this preconditioner: the kept null-space columns per
 * interface component are value-dependent (interface_basis,
 * coarse_space.py:64-103), so the coarse pattern is bound in the numeric
 * phase, like the reference */
int gdsw_precond_set_coarse(gdsw_precond* m, const gdsw_coarse_desc* coarse);
/* host-computed exact / ILU(k) factors (build_numeric, local_solvers.py:454-460) */
int gdsw_precond_set_factors(gdsw_precond* m, const void* l_vals, const void* u_vals);
/* FastILU sweeps on the GPU (fast_ilu_numeric, local_solvers.py:343-397);
 * residuals[sweep * n_sub + s] receives the per-sweep nonlinear residuals */
int gdsw_precond_fastilu(gdsw_precond* m, const gdsw_csr* a, int sweeps, double* residuals);
int gdsw_precond_get_factors(const gdsw_precond* m, void* l_vals, void* u_vals);
/* IKJ numeric LU / ILU(k) of every block on the GPU, bit-exact with the
 * reference (lu_numeric, _kernels.py:429-466; local_solvers.py:306-340);
 * a = the f64 operator (values cast to the precond dtype); fail_rows[n_sub]
 * gets 1 + the first row whose pivot is <= 1e-14 ||A_s||_inf, or 0 */
int gdsw_precond_lu_numeric(gdsw_precond* m, const gdsw_csr* a, double diag_shift, int64_t* fail_rows);
/* harmonic extension on the GPU (harmonic_extension, coarse_space.py:130-179);
 * a = the f64 operator the coarse basis is built from; col_resid[K] gets the
 * max |A_II phi_I + A_IG phi_G| per panel column */
int gdsw_precond_extend(gdsw_precond* m, const gdsw_csr* a, double tol, int max_iters,
                        int* iters_out, double* col_resid);
int64_t gdsw_precond_panel_entries(const gdsw_precond* m);
int gdsw_precond_get_panels(const gdsw_precond* m, double* panels);
/* Galerkin product A0 = Phi^T A Phi on the GPU (coarse_matrix,
 * coarse_space.py:205-207) from the extension's float64 panels: column c =
 * restriction of A (Phi e_c); a0_dense gets n_c x n_c row-major float64.
 * pattern (optional, n_c x n_c bytes): 1 where the reference's SpGEMM creates
 * an entry (structural product over |Phi| and |A|, computed zeros kept) */
int gdsw_precond_coarse_galerkin(gdsw_precond* m, const gdsw_csr* a, double* a0_dense, uint8_t* pattern);
/* dense A0^-1 (n_c x n_c, row-major, float64; cast to the precond dtype) */
int gdsw_precond_set_coarse_inverse(gdsw_precond* m, const double* a0inv);
/* factored coarse solve (replaces the reference's sparse LU of A0 and its
 * level-set solves, schwarz.py:267-272, 305, for large n_c): supernodal
 * partitioned inverse of the nested-dissection LU, built on the host by
 * paper_2304_04876_b200/coarse_factor.py. Supernodes in processing order
 * (leaves first), grouped by tree level; all index arrays are ORIGINAL coarse
 * columns; values float64 (cast to the precond dtype); updates are passed
 * up the supernode tree by extend-add. Replaces a dense
 * inverse set before (and vice versa). */
typedef struct gdsw_coarse_factor {
  int32_t n, n_sn, n_levels;
  const int64_t* level_ptr;   /* [n_levels + 1] supernode ranges */
  const int64_t* sn_s;        /* [n_sn] columns */
  const int64_t* sn_r;        /* [n_sn] rows below the diagonal block */
  const int64_t* col_ptr;     /* [n_sn + 1] */
  const int64_t* col_ids;
  const int64_t* row_ptr;     /* [n_sn + 1] == contribution-buffer offsets */
  const int64_t* row_ids;
  const int64_t* d_off;       /* s x s: strict lower = L_kk^-1, upper = U_kk^-1 */
  const int64_t* m_off;       /* r x s: L_{R,k} L_kk^-1 */
  const int64_t* n_off;       /* s x r: U_kk^-1 U_{k,R} */
  const int64_t* in_ptr;      /* [col_ptr[n_sn] + 1] children's update slots a column subtracts */
  const int64_t* in_idx;
  const int64_t* out_ptr;     /* [row_ptr[n_sn] + 1] children's update slots an update row adds */
  const int64_t* out_idx;
  const double* values;
  int64_t n_values;
} gdsw_coarse_factor;
int gdsw_precond_set_coarse_factor(gdsw_precond* m, const gdsw_coarse_factor* f);
/* exact-LU local solves through supernodal partitioned inverses of every
 * block's factors in one batch (LocalFactorization.solve, local_solvers.py:
 * 263-278, replacing the level-set substitution, _kernels.py:473-496);
 * indices are positions in the concatenated block vector (block order, ND
 * permutation folded in). NULL removes it (level-set path again). */
int gdsw_precond_set_local_factor(gdsw_precond* m, const gdsw_coarse_factor* f);
/* z = Phi A0^-1 Phi^T r + sum_i R_i^T A_i^-1 R_i r  (apply, schwarz.py:290-327) */
int gdsw_precond_apply(gdsw_precond* m, const double* r, double* z, void* stream);
/* per-block solves only: y[k] (dtype, concatenated block rows, permuted) =
 * LocalFactorization.solve of the gathered block (local_solvers.py:263-278);
 * jacobi_iters > 0 forces FastSpTRSV with that many iterates */
int gdsw_precond_local_solve(gdsw_precond* m, const double* r, void* y, int jacobi_iters,
                             void* stream);
int gdsw_precond_destroy(gdsw_precond* m);

/* ------------------------------------------------------------------------
 * Right-preconditioned restarted GMRES (gmres, krylov.py:141-161;
 * _gmres_single_reduce 260-361; _gmres_classic 179-257). The loop runs on
 * the host in C++; vectors, operator, preconditioner and the fused
 * reductions on the device. One device->host transfer per iteration carries
 * the 2(j+1) reduced scalars for the Givens update.
 * ---------------------------------------------------------------------- */
typedef struct {
  int32_t restart;
  double rel_tol;
  int32_t max_iters;
  int32_t variant;           /* gdsw_variant */
  int32_t orthogonalization; /* gdsw_orth    */
} gdsw_krylov_cfg;

typedef struct {
  int32_t iterations;
  int32_t converged;
  int32_t reduction_count;
  int32_t iteration_reductions;
  int32_t residual_reductions;
  int32_t restarts;
  int32_t n_history;  /* entries written to history  */
  int32_t n_true;     /* entries written to true_it / true_res */
} gdsw_solve_report;

int gdsw_workspace_create(gdsw_workspace** out, int64_t n, int32_t restart);
int gdsw_workspace_destroy(gdsw_workspace* ws);
/* m: preconditioner or NULL; m_csr: CSR preconditioner or NULL (both NULL =
 * identity). x: device, in = x0, out = solution. history/true_* are host
 * arrays of capacity `cap`. */
int gdsw_gmres(const gdsw_csr* a, gdsw_precond* m, const gdsw_csr* m_csr, const double* b,
               double* x, int x0_nonzero, const gdsw_krylov_cfg* cfg, gdsw_workspace* ws,
               gdsw_solve_report* rep, double* history, int32_t* true_it, double* true_res,
               int32_t cap, void* stream);

/* Host operators: the reference's duck-typed gmres operands (callables and
 * objects with .apply, krylov.py:88-100). y = op(x) on host arrays of n
 * doubles; a nonzero return aborts the solve (GDSW_E_TYPE, the caller keeps
 * its own exception). a_fn is used when a == NULL, m_fn when m == NULL and
 * m_csr == NULL; the GMRES vectors stay on the device, each operator call
 * stages its vector through pinned host buffers (no pass graphs). */
typedef int (*gdsw_host_op)(void* ctx, const double* x, double* y, int64_t n);
int gdsw_gmres_host_ops(const gdsw_csr* a, gdsw_host_op a_fn, void* a_ctx, gdsw_precond* m,
                        const gdsw_csr* m_csr, gdsw_host_op m_fn, void* m_ctx, int64_t n,
                        const double* b, double* x, int x0_nonzero, const gdsw_krylov_cfg* cfg,
                        gdsw_workspace* ws, gdsw_solve_report* rep, double* history,
                        int32_t* true_it, double* true_res, int32_t cap, void* stream);

/* ------------------------------------------------------------------------
 * Sharded solve: one process per GPU, each rank owns a
 * contiguous row range [own_lo, own_hi) of its extended local layout of
 * n_ext rows (owned rows + halo rows owned by neighbours) and a contiguous
 * range of subdomains. Collectives are this library's own peer-memory
 * kernels: every rank maps every rank's IPC-exported mailbox (exchange the
 * 64-byte handles with any bootstrap, e.g. torch.distributed); one kernel
 * per collective, device-side release/acquire flags, no host round trip.
 * Per GMRES iteration: one halo refresh before the SpMV and one before the
 * apply, one reverse halo of overlapped partial sums, one all-reduce of the
 * coarse right-hand side and ONE all-reduce of the fused block.
 * send ranges: owned rows neighbour i needs; recv ranges: halo rows it owns
 * (both ext-local). The operator passed to gdsw_gmres_dist has n_own rows
 * and n_ext columns; the preconditioner's plan is built on n_ext rows.
 * ---------------------------------------------------------------------- */
typedef struct gdsw_dist gdsw_dist;
int gdsw_dist_create(gdsw_dist** out, int rank, int nranks, int64_t n_ext, int64_t own_lo,
                     int64_t own_hi, int n_nbr, const int32_t* nbr_rank, const int64_t* send_lo,
                     const int64_t* send_hi, const int64_t* recv_lo, const int64_t* recv_hi,
                     int64_t red_max);
int gdsw_dist_ipc_handle(gdsw_dist* d, void* handle64);
int gdsw_dist_open_peers(gdsw_dist* d, const void* handles /* nranks x 64 bytes */);
int gdsw_dist_allreduce(gdsw_dist* d, const double* in, double* out, int64_t m, void* stream);
int gdsw_dist_halo(gdsw_dist* d, double* x_ext, void* stream);
int gdsw_dist_destroy(gdsw_dist* d);
int gdsw_precond_set_dist(gdsw_precond* m, gdsw_dist* d);
/* sharded Galerkin product A0 = Phi^T A Phi (coarse_space.py:205-207): a_own
   is this rank's owned rows over its extended columns; the partial products
   are summed over ranks in rank order on the device; a0_dense: n_c x n_c
   row-major, identical on every rank */
int gdsw_dist_coarse_galerkin(gdsw_precond* m, const gdsw_csr* a_own, gdsw_dist* d, double* a0_dense,
                              uint8_t* pattern);
/* b, x: owned rows only (n_own) */
int gdsw_gmres_dist(const gdsw_csr* a, gdsw_precond* m, const gdsw_csr* m_csr, const double* b,
                    double* x, int x0_nonzero, const gdsw_krylov_cfg* cfg, gdsw_workspace* ws,
                    gdsw_dist* dist, gdsw_solve_report* rep, double* history, int32_t* true_it,
                    double* true_res, int32_t cap, void* stream);

/* fused single-reduce block reduction [V[:j]; v]^T [v, z] (krylov.py:290-300);
 * out (host) receives 2(j+1) values: [V.v..., v.v, V.z..., v.z] */
int gdsw_block_dot(const double* V, int64_t ldv, int32_t j, const double* v, const double* z,
                   int64_t n, double* out, void* stream);
/* single-reduce update (krylov.py:346-351) with the pass-j scalars in device
 * memory, coef = [a(0..j), p/delta(0..j), delta, corr]:
 *   v[j] = (w - V a)/delta;  zm[j] = (mc - Zm a)/delta (skipped when Zm is
 *   NULL);  w = zc/delta - V p/delta - corr v[j]    (rows of ld doubles) */
int gdsw_sr_update(double* V, double* Zm, int64_t ld, int64_t n, int32_t j, const double* coef, double* w,
                   const double* mc, const double* zc, void* stream);

/* ------------------------------------------------------------------------
 * Instrumentation: per-phase device time (CUDA events on the launching
 * stream) accumulated while enabled. names: see gdsw_prof_name().
 * ---------------------------------------------------------------------- */
int64_t gdsw_launch_count(void); /* kernels launched by this library so far */
int gdsw_prof_enable(int on);
int gdsw_prof_reset(void);
int gdsw_prof_count(void);
const char* gdsw_prof_name(int k);
int gdsw_prof_read(int k, double* total_ms, int64_t* launches, double* bytes);

#ifdef __cplusplus
}
#endif
#endif
