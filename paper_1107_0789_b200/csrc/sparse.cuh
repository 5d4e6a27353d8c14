// Observed-set (Omega) structures and the sparse kernels of the APG-MC iteration:
//   SDDMM residual  r_e = <Yl[i,:], Yr[j,:]> - M_e     (eval_on_support, P/include/dfc/solvers.hpp:215-225,281-285)
//   SpMM            out (+)= alpha * R   X             (FactoredSparseOp::apply,         solvers.hpp:121-125)
//   SpMM^T          out (+)= alpha * R^T X             (FactoredSparseOp::apply_adjoint, solvers.hpp:126-130)
// R shares the pattern of M; its values live in CSR order (r_csr) and the CSC walk reads
// them through the csc->csr permutation, so the SDDMM writes one coalesced stream.
#pragma once

#include "common.cuh"

namespace dfcg {

// One segmented-SpMM work item: a run of entries of one row of the structure.
struct SegItem {
  int row;
  int slot;  // -1: sole segment of its row (write directly); else workspace row
  long long e0, e1;
};

struct SegPlan {
  DBuf<SegItem> items;
  DBuf<int> red_rowptr;  // rows with >1 segment: [row] -> slots range (size rows+1), or empty
  i64 n_items = 0, n_slots = 0, rows = 0;
  std::vector<int> h_multi_rows;  // rows needing a reduction
  DBuf<int> multi_rows;
};

struct DevOmega {
  i64 m = 0, n = 0, nnz = 0;
  // CSR (row-major walk): entries sorted by (row, col).
  DBuf<int> csr_rowptr, csr_row, csr_col;
  DBuf<double> m_csr;
  // CSC (column walk, the reference's entry order): entries sorted by (col, row).
  DBuf<int> csc_colptr, csc_row;
  DBuf<long long> csc2csr;  // CSC position -> CSR position
  DBuf<double> m_csc;
  SegPlan plan_csr, plan_csc;
  // Cache-blocked variants of the two walks (the chunked SpMM): items ordered by a chunk of
  // kChunkTiles 64-wide tiles of the INNER dimension, then by outer line, so the warps resident
  // at any moment gather X rows from one chunk (~kChunkTiles * 64 * b * 8 bytes, L1-sized)
  // instead of all of X (L2-bound); every (line, chunk) run is a workspace slot, summed per line
  // in chunk order. Empty (n_items == 0) when the inner dimension spans <= 2 chunks.
  static constexpr int kChunkTiles = 8;
  SegPlan plan_csr_ck, plan_csc_ck;
  bool has_empty_csr = false, has_empty_csc = false;  // structure rows / columns without entries
  std::vector<long long> h_csc2csr;  // host copy (outputs in reference order)
  // Column-tile offsets of the CSR rows for the tiled SDDMM: the entries of row r in column
  // tile q = [64q, 64q + 64) are CSR positions [tile_csr[r*(ntc+1)+q], tile_csr[r*(ntc+1)+q+1]).
  // ntc = 0 when the table would be too large (the entry-parallel kernel is used then).
  static constexpr int kTileCols = 64;
  int ntc = 0;
  DBuf<int> tile_csr;
  // The same for the CSC columns over 64-row tiles (tiled transposed SpMM): ntr = 0 when too large.
  int ntr = 0;
  DBuf<int> tile_csc;

  // rows/cols: CSC-sorted (column-major order, as ObservedMatrix guarantees).
  void build(cudaStream_t s, i64 m, i64 n, i64 nnz, const long long* rows, const long long* cols, const double* vals);
};

// r_csr[t] = <Yl[row_t,:], Yr[col_t,:]> - (sub ? m_csr[t] : 0)   (kY may be 0 -> r = -m)
void sddmm_residual(cudaStream_t s, const DevOmega& om, i64 kY, const double* Yl, i64 ldl, const double* Yr,
                    i64 ldr, const double* sub, double* r_csr);

// out[rows x b] = alpha * S X + beta * out, S given by (structure, values).
//   transpose == false: S = R (m x n) via CSR, X is n x b, out is m x b.
//   transpose == true : S = R^T (n x m) via CSC, X is m x b, out is n x b.
// vals are always in CSR order (the CSC walk indexes them through csc2csr).
// vals_csc (optional): the same values in CSC order; the transposed walk then streams them
// instead of gathering vals_csr through the permutation.
void spmm(cudaStream_t s, const DevOmega& om, bool transpose, const double* vals_csr, i64 b, double alpha,
          const double* X, i64 ldx, double beta, double* out, i64 ldo, const double* vals_csc = nullptr);

// vals_csc[p] = vals_csr[csc2csr[p]]
void csr_to_csc(cudaStream_t s, const DevOmega& om, const double* vals_csr, double* vals_csc);

// Microbenchmark override of the slab kernels (1 on, 0 off, -1 back to DFCG_SPMM_SLAB /
// DFCG_SDDMM_SLAB): process-global, for dfcg_bench_sparse only.
void set_sparse_modes(int spmm_mode, int sddmm_mode);  // spmm_mode: 0 gather (8-byte), 1 slab, 2 chunked (8-byte), 3 gather 16-byte, 4 chunked 16-byte

// D[i, j] += alpha * vals[(i,j)] for the observed pattern (row-major m x n dense D).
void scatter_add_dense(cudaStream_t s, const DevOmega& om, const double* vals_csr, double alpha, double* D, i64 ldd);

}  // namespace dfcg
