// Internal C++ API of the device solvers (below the C ABI in capi.cpp).
#pragma once

#include <chrono>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <vector>

#include "common.cuh"
#include "rng.hpp"
#include "sparse.cuh"

namespace dfcg {

// Reference ApgConfig (P/include/dfc/solvers.hpp:19-26).
struct ApgConfig {
  int max_iters = 500;
  double rel_tol = 1e-4;
  std::optional<double> mu_init, mu_floor;
  double mu_decay = 0.7;
  bool line_search = false;
};

struct SolveReport {
  int iterations = 0;
  double objective = 0.0, residual = 0.0;
  i64 rank = 0;
  double wall_ms = 0.0;
};

struct IterTrace {
  int it;
  i64 rank, k_final;
  int svd_calls;
  double rel, mu, sigma_sum;
  double ms = 0.0;
};

// Factored estimate on the device: L = left (m x k) * right (n x k)^T, both ROW-major.
struct DevLowRank {
  i64 m = 0, n = 0, k = 0;
  DBuf<double> left, right;
};

// Host-side column-major estimate (the reference's LowRankEstimate layout).
struct HostLowRank {
  i64 m = 0, n = 0, k = 0;
  std::vector<double> left, right;  // column-major m x k, n x k
};

// One per device: the cached SVT Gaussian streams and device properties.
// Streams are pooled and live as long as the context, so device buffers handed out by a
// call (freed stream-ordered on the stream that allocated them) never outlive their stream.
struct DeviceContext {
  int device = 0;
  std::unique_ptr<NormalCache> normals_mc, normals_rmf;
  std::mutex mu;
  std::vector<cudaStream_t> free_streams, all_streams;
  explicit DeviceContext(int dev);
  ~DeviceContext();
  NormalCache& normals(int stream) { return stream == 0 ? *normals_mc : *normals_rmf; }
  cudaStream_t acquire();
  void release(cudaStream_t s);
};

// RAII stream for one call: bound to the context's device, synchronised on exit.
struct CallStream {
  DeviceContext& ctx;
  cudaStream_t s = nullptr;
  explicit CallStream(DeviceContext& c);
  ~CallStream();
};

void validate_config(const ApgConfig& cfg);

// Resumable apg_mc (solvers.hpp:241-327): the ctor uploads Omega and computes mu_init,
// step() runs one APG iteration, finish() reports (and copies out the current estimate).
// Same arithmetic as running the reference loop to completion.
class McSolver {
 public:
  McSolver(DeviceContext& ctx, cudaStream_t s, i64 m, i64 n, i64 nnz, const long long* rows, const long long* cols,
           const double* vals, const ApgConfig& cfg);
  ~McSolver();
  bool step(std::vector<IterTrace>* trace = nullptr);
  void finish(DevLowRank& out, SolveReport& rep);
  int iterations() const { return iters_; }
  bool stopped() const { return stopped_ || iters_ >= cfg_.max_iters; }

 private:
  struct State;
  DeviceContext& ctx_;
  cudaStream_t s_;
  i64 m_, n_, nnz_;
  ApgConfig cfg_;
  std::unique_ptr<State> st_;
  int iters_ = 0;
  bool stopped_ = false;
  std::chrono::steady_clock::time_point start_;
};

// apg_mc on an ObservedMatrix given as CSC-sorted triplets. Result stays on the device.
void apg_mc_device(DeviceContext& ctx, cudaStream_t s, i64 m, i64 n, i64 nnz, const long long* rows,
                   const long long* cols, const double* vals, const ApgConfig& cfg, DevLowRank& out, SolveReport& rep,
                   std::vector<IterTrace>* trace);

// apg_rmf on a dense column-major m x n matrix (host pointer). Outputs: L on device, S as
// column-major-scan triplets on the host.
void apg_rmf_device(DeviceContext& ctx, cudaStream_t s, const double* M_colmajor, i64 m, i64 n, double lambda,
                    const ApgConfig& cfg, DevLowRank& out, std::vector<long long>& s_row, std::vector<long long>& s_col,
                    std::vector<double>& s_val, SolveReport& rep, std::vector<IterTrace>* trace);

// Transfers between host column-major and device row-major estimates.
void upload_lowrank(cudaStream_t s, const HostLowRank& h, DevLowRank& d);
void download_lowrank(cudaStream_t s, const DevLowRank& d, HostLowRank& h);

// ---- combiners (combine.cu), all on device row-major estimates -------------------------
struct SvdOfProduct {
  i64 r = 0;
  DevLowRank est;             // (U, V diag(s))
  DBuf<double> U, V;          // m x r, n x r row-major (orthonormal)
  std::vector<double> s;
};
SvdOfProduct svd_of_product(cudaStream_t s, i64 m, i64 n, i64 k, const double* left, const double* right,
                            double rel_cutoff = 1e-12);
void column_project(cudaStream_t s, const DevLowRank& basis, const std::vector<const DevLowRank*>& blocks,
                    const std::vector<std::vector<i64>>& groups, i64 n, DevLowRank& out);
void project_rows(cudaStream_t s, const double* Ub, i64 m, i64 kb, const DevLowRank& block, double* Rg);
void scatter_rows(cudaStream_t s, const double* src, i64 rows, i64 c, const std::vector<i64>& idx, double* dst);
void gather_rows(cudaStream_t s, const double* src, i64 c, const std::vector<i64>& idx, double* dst);
void gen_nystrom(cudaStream_t s, const DevLowRank& C, const DevLowRank& R, const std::vector<i64>& rows,
                 const std::vector<i64>& cols, DevLowRank& out);
void average_estimates(cudaStream_t s, const std::vector<const DevLowRank*>& ests, std::optional<i64> recompress_to,
                       DevLowRank& out);
void random_project(cudaStream_t s, const std::vector<const DevLowRank*>& blocks,
                    const std::vector<std::vector<i64>>& groups, i64 n, i64 k, i64 p, i64 q, SeededRng& rng,
                    DevLowRank& out);

}  // namespace dfcg
