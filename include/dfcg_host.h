/* dfcg_host.h — host-side utilities exported by libdfcg.so next to the hot-path ABI.
 *
 * These restate the reference's input side so callers (bench, tests, a CLI) can build the
 * exact inputs the reference builds, without the reference:
 *   SeededRng            P/include/dfc/rng.hpp:26-74
 *   sample_without_replacement / partition_columns / extract_*   P/include/dfc/sampling.hpp:15-113
 *   gen_mc_instance / gen_rmf_instance                            P/include/dfc/simgen.hpp:30-82
 *   load_triplets / save_triplets                                 P/include/dfc/matrix_io.hpp:125-179
 * Nothing here runs on the GPU. Arrays returned through pointer-to-pointer arguments are
 * malloc'ed by the library; release them with dfcg_free (dfcg.h).
 */
#ifndef DFCG_HOST_H_
#define DFCG_HOST_H_

#include <stdint.h>

#include "dfcg.h"

#ifdef __cplusplus
extern "C" {
#endif

void dfcg_rng_u64(uint64_t seed, uint64_t stream, int64_t n, uint64_t* out);
/* The same raw stream from the bulk (vectorised) mt19937_64 the device normal cache uses. */
void dfcg_rng_u64_bulk(uint64_t seed, uint64_t stream, int64_t n, uint64_t* out);
void dfcg_rng_uniform(uint64_t seed, uint64_t stream, int64_t n, double* out);
void dfcg_rng_normal(uint64_t seed, uint64_t stream, int64_t n, double* out);
int dfcg_rng_index(uint64_t seed, uint64_t stream, int64_t count, uint64_t bound, uint64_t* out);

int dfcg_sample_without_replacement(uint64_t seed, uint64_t stream, int64_t n, int64_t l, int64_t* out);
/* cols: n entries, offsets: t + 1 entries (group g = cols[offsets[g]:offsets[g+1]], sorted). */
int dfcg_partition_columns(uint64_t seed, uint64_t stream, int64_t n, int64_t t, int64_t* cols, int64_t* offsets);

/* The D step as dfc_run runs it (sampling.hpp:83-113 extract_columns / extract_rows): ngroups
 * disjoint column groups (CSR plan) then, when nrows > 0, one row sample, extracted in one
 * parallel stable pass (DFCG_DSTEP_THREADS host threads). counts[i] (ngroups + (nrows > 0)
 * entries) and the triplets of every subproblem, concatenated in that order (column-major within
 * each, indices relabelled; library-allocated). */
int dfcg_extract_subproblems(const dfcg_obs* in, int64_t ngroups, const int64_t* group_offsets,
                             const int64_t* group_cols, int64_t nrows, const int64_t* rows, int64_t* counts,
                             int64_t** out_rows, int64_t** out_cols, double** out_vals);

/* gen_mc_instance with SeededRng(seed, stream). L0 factors column-major (library-allocated),
 * observations sorted column-major (library-allocated, s entries). */
int dfcg_gen_mc_instance(int64_t m, int64_t n, int64_t r, int64_t s, double sigma, uint64_t seed, uint64_t stream,
                         dfcg_lowrank* L0, int64_t** rows, int64_t** cols, double** vals);

/* gen_rmf_instance; outliers U[lo, hi] (the reference draws U[0,1]); M is a caller buffer of
 * m * n doubles (column-major); S0 in draw order (library-allocated). */
/* BASELINE c4 stand-in (no reference generator): recommender-shaped instance, Zipf(1) row/column
 * popularity, cells ~ row_pop * col_pop (alias sampling + dedup, ~density * m * n * subset mass),
 * values clip(round(3.6 + A B^T + N(0, noise^2)), 1, 5), A, B iid N(0, fsd^2). ncols_sub > 0
 * restricts to a column subset (returned columns are subset positions). Triplets column-major,
 * library-allocated (free with dfcg_free). */
int dfcg_gen_recsys_instance(int64_t m, int64_t n, int64_t r, double density, double fsd, double noise,
                             int64_t ncols_sub, const int64_t* cols_sub, uint64_t seed, uint64_t stream,
                             int64_t* count, int64_t** rows, int64_t** cols, double** vals);
int dfcg_gen_rmf_instance(int64_t m, int64_t n, int64_t r, int64_t s, double sigma, uint64_t seed, uint64_t stream,
                          double lo, double hi, dfcg_lowrank* L0, dfcg_sparse* S0, double* M);

/* ---- triplet text I/O (load_triplets / save_triplets, P/include/dfc/matrix_io.hpp:125-179) ----
 * "% m n" header (optional; dims inferred from the data without it), one "i j v" line per
 * observation, blank lines skipped, 0-based unless one_based. Parsed and sorted to the
 * ObservedMatrix order (column-major, matrix_io.hpp:41-43) on DFCG_IO_THREADS host threads.
 * Errors as the reference: DFCG_EPARSE (ParseError; dfcg_last_error_line() = its line, the
 * first offending line in file order), DFCG_ERANGE (index outside the declared dims),
 * DFCG_EINVAL (no header and no data; duplicate entry). Arrays are library-allocated. */
int dfcg_load_triplets_text(const char* text, int64_t len, int32_t one_based, int64_t* m, int64_t* n, int64_t* count,
                            int64_t** rows, int64_t** cols, double** vals);
int dfcg_load_triplets_file(const char* path, int32_t one_based, int64_t* m, int64_t* n, int64_t* count,
                            int64_t** rows, int64_t** cols, double** vals);
/* "% m n" then "row col %.17g" per entry in the order given (lossless: load(save(x)) == x). */
int dfcg_save_triplets_file(const char* path, const dfcg_obs* in);
int dfcg_format_triplets(const dfcg_obs* in, char** text, int64_t* len); /* text: dfcg_free */

/* ---- kernel accounting (bench / profiling; off by default) ---------------------------
 * Op classes, in order: 0 gemm (>= 2 GFLOP), 1 sddmm, 2 spmm, 3 cholesky, 4 qr_fallback,
 * 5 jacobi, 6 elementwise, 7 reduce, 8 other, 9 gemm_small (< 2 GFLOP).
 * dfcg_prof_enable clears previous records. */
#define DFCG_PROF_NUM_OPS 10
void dfcg_prof_enable(int on);
int64_t dfcg_launch_count(void);
/* Per op class: launches, summed CUDA-event ms, algorithmic FLOPs and bytes. Returns the
 * number of classes filled (DFCG_PROF_NUM_OPS) or a negative error. */
int dfcg_prof_collect(int64_t* launches, double* ms, double* flops, double* bytes);
/* Always-on cumulative work counters per op class since the library loaded (no events):
 * launches, algorithmic FLOPs and bytes. Difference two reads around a timed window. */
int dfcg_work_counters(int64_t* launches, double* flops, double* bytes);

#ifdef __cplusplus
}
#endif

#endif /* DFCG_HOST_H_ */
