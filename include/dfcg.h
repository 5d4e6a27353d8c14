/* dfcg.h — C ABI of the B200 DFC hot path (libdfcg.so).
 *
 * Drop-in boundary for the reference's Divide-Factor-Combine hot path
 * (reference: /root/reference/proj, cited as P/):
 *   - the F-step base solvers behind `BaseSolver` (P/include/dfc/dfc.hpp:67-78):
 *       apg_mc  (P/include/dfc/solvers.hpp:241-327)  -> dfcg_apg_mc
 *       apg_rmf (P/include/dfc/solvers.hpp:332-414)  -> dfcg_apg_rmf
 *   - the C-step combiners (P/include/dfc/sketch.hpp):
 *       column_project    (:170-199) -> dfcg_column_project
 *       gen_nystrom       (:241-266) -> dfcg_gen_nystrom
 *       average_estimates (:271-298) -> dfcg_average_estimates
 *       random_project    (:204-237) -> dfcg_random_project
 *       svd_of_product    (:73-86)   -> dfcg_svd_of_product  (rank query for dfc_nys pair_deficient)
 *   - the orchestrator dfc_run (P/include/dfc/dfc.hpp:326-335) -> dfcg_dfc_run
 *
 * Conventions: plain pointers and sizes only. Dense factors are COLUMN-MAJOR (Eigen's
 * default layout, P/include/dfc/matrix_io.hpp:19). Observation triplets are sorted in
 * column-major order, as the ObservedMatrix constructor guarantees (matrix_io.hpp:38-56).
 * All arithmetic is FP64. Every function returns DFCG_OK (0) or a negative error code;
 * dfcg_last_error() returns the thread's last message. Error codes map onto the
 * reference's exceptions: DFCG_EINVAL = std::invalid_argument, DFCG_ERANGE =
 * std::out_of_range, DFCG_EBLOCK = BlockError (dfc.hpp:50-54, see dfcg_last_error_block;
 * for DFCG_EBLOCK dfcg_last_error() is the failing block's own message, without the
 * "block N: " prefix that BlockError's constructor adds).
 * Result arrays are allocated by the library (malloc) and released with dfcg_free.
 */
#ifndef DFCG_H_
#define DFCG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  DFCG_OK = 0,
  DFCG_EINVAL = -1,
  DFCG_ERANGE = -2,
  DFCG_EBLOCK = -3,
  DFCG_ECUDA = -4,
  DFCG_ENOMEM = -5,
  DFCG_ENCCL = -6,
  DFCG_EINTERNAL = -7,
  DFCG_EPARSE = -8 /* ParseError (matrix_io.hpp:22-26); dfcg_last_error_line() is its line */
};

typedef struct dfcg_ctx dfcg_ctx;

/* ApgConfig, P/include/dfc/solvers.hpp:19-26 (std::optional -> has_* flags). */
typedef struct {
  int32_t max_iters;
  double rel_tol;
  int32_t has_mu_init;
  double mu_init;
  int32_t has_mu_floor;
  double mu_floor;
  double mu_decay;
  int32_t line_search;
} dfcg_apg_cfg;

/* SolveReport, P/include/dfc/solvers.hpp:39-45. */
typedef struct {
  int32_t iterations;
  double objective;
  double residual;
  int64_t rank;
  double wall_ms;
} dfcg_solve_report;

/* ObservedMatrix, P/include/dfc/matrix_io.hpp:36-67: m x n, nnz triplets, column-major order. */
typedef struct {
  int64_t m, n, nnz;
  const int64_t* row;
  const int64_t* col;
  const double* val;
} dfcg_obs;

/* LowRankEstimate, P/include/dfc/matrix_io.hpp:71-98: L = left (m x k) * right (n x k)^T,
 * both column-major. As an input the pointers are read; as an output they are allocated. */
typedef struct {
  int64_t m, n, k;
  double* left;
  double* right;
} dfcg_lowrank;

/* OutlierEstimate, P/include/dfc/solvers.hpp:48-67 (column-major scan order). */
typedef struct {
  int64_t m, n, count;
  int64_t* row;
  int64_t* col;
  double* val;
} dfcg_sparse;

/* Per-iteration observation trace (not in the reference; parity debugging). */
typedef struct {
  int32_t it;
  int64_t rank;
  int64_t k_final;  /* k of the last partial SVD of the iteration; 0 = dense SVD path */
  int32_t svd_calls;
  double rel, mu, sigma_sum;
  double ms; /* host wall time of the iteration (each iteration ends in a device sync) */
} dfcg_iter_trace;

/* DfcConfig, P/include/dfc/dfc.hpp:36-48. variant: 0 Proj, 1 Rp, 2 Nys; task: 0 MC, 1 RMF. */
typedef struct {
  int32_t variant;
  int32_t ensemble;
  int64_t t, l, d;
  int64_t rp_p, rp_q;
  uint64_t seed;
  dfcg_apg_cfg solver;
  int32_t task;
  double lambda;
  int32_t workers;
  /* Proj-Ens anchors: 0 = every block (the reference, dfc.hpp:191-195); A > 0 = the first
   * min(A, t) plan groups (BASELINE c5's "ensemble of 4"; an extension of the reference). */
  int64_t ensemble_anchors;
} dfcg_dfc_cfg;

/* DfcReport, P/include/dfc/dfc.hpp:56-65. subproblems has n_sub entries (library-allocated). */
typedef struct {
  double divide_ms, factor_ms, combine_ms, total_ms;
  int64_t chosen_k;
  int32_t k_clamped, rank_deficient;
  int64_t n_sub;
  dfcg_solve_report* subproblems;
} dfcg_dfc_report;

int dfcg_ctx_create(int device, dfcg_ctx** out);
void dfcg_ctx_destroy(dfcg_ctx* ctx);
const char* dfcg_last_error(void);
int64_t dfcg_last_error_block(void);
int64_t dfcg_last_error_line(void); /* 1-based line of the last DFCG_EPARSE, else -1 */
void dfcg_free(void* p);
void dfcg_lowrank_free(dfcg_lowrank* e); /* frees left/right of a library-filled estimate */
void dfcg_sparse_free(dfcg_sparse* s);

/* ---- F step: base solvers (replace apg_mc / apg_rmf) -------------------------------- */
int dfcg_apg_mc(dfcg_ctx* ctx, const dfcg_obs* in, const dfcg_apg_cfg* cfg, dfcg_lowrank* out,
                dfcg_solve_report* rep, dfcg_iter_trace* trace, int64_t trace_cap, int64_t* trace_len);

int dfcg_apg_rmf(dfcg_ctx* ctx, const double* M_colmajor, int64_t m, int64_t n, double lambda,
                 const dfcg_apg_cfg* cfg, dfcg_lowrank* L, dfcg_sparse* S, dfcg_solve_report* rep,
                 dfcg_iter_trace* trace, int64_t trace_cap, int64_t* trace_len);

/* Resumable apg_mc with the observation set resident on the device: create uploads Omega
 * and computes mu_init; step advances up to n_iters APG iterations (*done = iterations run,
 * fewer if the stop test fired); finish reports and returns the current estimate without
 * ending the run. Each solver owns a CUDA stream, so solvers stepped from different host
 * threads run concurrently on the GPU. */
typedef struct dfcg_mc_solver dfcg_mc_solver;
int dfcg_mc_solver_create(dfcg_ctx* ctx, const dfcg_obs* in, const dfcg_apg_cfg* cfg, dfcg_mc_solver** out);
int dfcg_mc_solver_step(dfcg_mc_solver* sv, int64_t n_iters, int64_t* done, dfcg_iter_trace* trace,
                        int64_t trace_cap, int64_t* trace_len);
int dfcg_mc_solver_finish(dfcg_mc_solver* sv, dfcg_lowrank* out, dfcg_solve_report* rep);
void dfcg_mc_solver_destroy(dfcg_mc_solver* sv);

/* ---- C step: combiners --------------------------------------------------------------- */
/* Partition plan as CSR: group g owns group_cols[group_offsets[g] : group_offsets[g+1]]. */
int dfcg_column_project(dfcg_ctx* ctx, const dfcg_lowrank* basis, int64_t t, const dfcg_lowrank* blocks,
                        const int64_t* group_offsets, const int64_t* group_cols, int64_t n, dfcg_lowrank* out);

int dfcg_gen_nystrom(dfcg_ctx* ctx, const dfcg_lowrank* C_hat, const dfcg_lowrank* R_hat, int64_t d,
                     const int64_t* row_idx, int64_t l, const int64_t* col_idx, dfcg_lowrank* out);

/* recompress_to < 0 means std::nullopt. */
int dfcg_average_estimates(dfcg_ctx* ctx, int64_t count, const dfcg_lowrank* ests, int64_t recompress_to,
                           dfcg_lowrank* out);

int dfcg_random_project(dfcg_ctx* ctx, int64_t t, const dfcg_lowrank* blocks, const int64_t* group_offsets,
                        const int64_t* group_cols, int64_t n, int64_t k, int64_t p, int64_t q, uint64_t seed,
                        uint64_t stream, dfcg_lowrank* out);

/* Compact SVD of left * right^T (svd_of_product); out = (U, V diag(s)), s copied to s_out
 * (caller buffer of size >= min(m, n, k)) when non-null, rank in *rank. */
int dfcg_svd_of_product(dfcg_ctx* ctx, const dfcg_lowrank* in, dfcg_lowrank* out, double* s_out, int64_t* rank);
/* Diagnostics: normals [pos, pos+n) of the device-cached SVT stream SeededRng(0x737674, stream_id)
 * (stream_id 0: apg_mc, 1: apg_rmf; P/include/dfc/solvers.hpp:263,344) copied to host out[n]. */
int dfcg_normals_fetch(dfcg_ctx* ctx, int stream_id, int64_t pos, int64_t n, double* out);

/* Diagnostics: the APG-MC iteration's sparse kernels on the observed set `in` with random dense
 * operands — forward SpMM (R X, X n x b), transposed SpMM (R^T Q, Q m x b), SDDMM residual at
 * rank kY — each timed over `reps` calls with CUDA events (ms3: ms per call) and the sum of its
 * output (sum3). spmm_mode / sddmm_mode: 1 slab kernels, 0 the previous kernels, -1 default. */
int dfcg_bench_sparse(dfcg_ctx* ctx, const dfcg_obs* in, int64_t b, int64_t kY, int32_t reps, int32_t spmm_mode,
                      int32_t sddmm_mode, double* ms3, double* sum3);

/* Diagnostics: the CholeskyQR Cholesky (+ inverse) of a random SPD matrix of order n, ms per call
 * over `reps` CUDA-event-timed calls, with max |R^T R - G| / max |G| and max |R Rinv - I|. */
int dfcg_bench_cholesky(dfcg_ctx* ctx, int64_t n, int32_t reps, int32_t want_inverse, double* ms, double* relres,
                        double* invres);

/* One block of the DFC-Proj combine, for the multi-GPU split of column_project
 * (sketch.hpp:194-196): Rg = block.right (Ub^T block.left)^T, Ub m x kb column-major, Rg
 * (block.n x kb, column-major) written to a caller buffer. */
int dfcg_project_block(dfcg_ctx* ctx, const double* Ub, int64_t m, int64_t kb, const dfcg_lowrank* block,
                       double* Rg);

/* ---- multi-GPU: one process per GPU (the reference's single-process
 * parallel_for over subproblems, P/include/dfc/dfc.hpp:84-147, split over ranks) ------------- */
typedef struct dfcg_comm dfcg_comm;
/* Caller-provided collective layer on HOST buffers (e.g. torch.distributed over gloo): the
 * library stages device data through pinned memory. Each callback returns 0 on success and is
 * invoked by every participating rank in the same global order. */
typedef struct {
  void* user;
  int (*bcast)(void* user, void* buf, int64_t bytes, int32_t root);
  int (*send)(void* user, const void* buf, int64_t bytes, int32_t peer);
  int (*recv)(void* user, void* buf, int64_t bytes, int32_t peer);
} dfcg_host_transport;
/* NCCL (loaded at run time: the process's libnccl.so.2, else $DFCG_NCCL_LIB): rank 0 draws the
 * id, the caller distributes it, every rank creates its communicator on ctx's device. */
int dfcg_nccl_unique_id(unsigned char id[128]);
int dfcg_comm_init_nccl(dfcg_ctx* ctx, int32_t nranks, int32_t rank, const unsigned char id[128], dfcg_comm** out);
int dfcg_comm_init_host(int32_t nranks, int32_t rank, const dfcg_host_transport* t, dfcg_comm** out);
void dfcg_comm_destroy(dfcg_comm* comm);
/* Host-only traffic pattern through the transport (every root broadcasts, a ring of sends);
 * *errors = mismatched words seen by this rank. No CUDA for a host transport. */
int dfcg_comm_selftest(dfcg_comm* comm, int64_t* errors);
/* LPT assignment of count subproblems to nranks by observation count (descending nnz, ties to
 * the lower index; each to the least-loaded rank, ties to fewer blocks then the lower rank). */
int dfcg_assign_blocks(int64_t count, const int64_t* nnz, int32_t nranks, int32_t* owner);
/* dfc_run over the ranks of comm: every rank passes the same obs and cfg, solves its LPT share
 * of the subproblems (cfg->workers concurrent streams), and the combine moves factors only
 * (basis broadcast + row gather for Proj; R-hat for Nys; block factors for Rp). Every rank
 * returns the final estimate and the report of every subproblem; owner (optional, n_sub
 * entries up to owner_cap) receives the assignment. A failing subproblem raises DFCG_EBLOCK
 * with the lowest failing index on every rank. */
int dfcg_dfc_run_dist(dfcg_ctx* ctx, dfcg_comm* comm, const dfcg_obs* in, const dfcg_dfc_cfg* cfg, dfcg_lowrank* out,
                      dfcg_dfc_report* rep, int32_t* owner, int64_t owner_cap);

/* ---- whole D-F-C pipeline (replaces dfc_run) --------------------------------------------- */
int dfcg_dfc_run(dfcg_ctx* ctx, const dfcg_obs* in, const dfcg_dfc_cfg* cfg, dfcg_lowrank* out,
                 dfcg_dfc_report* rep);
void dfcg_dfc_report_free(dfcg_dfc_report* rep);

#ifdef __cplusplus
}
#endif

#endif /* DFCG_H_ */
