// TEST INFRASTRUCTURE ONLY — CPU oracle for the DFC hot path.
//
// A from-scratch C++ restatement of the reference's algorithms (Eigen replaced by
// a plain column-major matrix type plus the LAPACK/BLAS that numpy bundles), used
// as the parity checker for the CUDA path and as the CPU baseline arm of bench.py.
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
// reference) may load it. The product library never links or calls it.
//
// Reference cited as P/ = /root/reference/proj/.  Parity pins: RNG golden vectors
// (P/tests/test_rng.cpp:11-48), closed-form SVT/soft-threshold, Nystrom/projection
// exact cases, and the printed acceptance values (P/test_output.txt:370-375).
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <numeric>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <utility>
#include <vector>

namespace orc {

using Index = std::int64_t;

// ---------------------------------------------------------------- RNG (P/include/dfc/rng.hpp:11-74)
inline std::uint64_t splitmix64(std::uint64_t& state) {
  state += 0x9E3779B97F4A7C15ULL;
  std::uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

class SeededRng {
 public:
  explicit SeededRng(std::uint64_t seed, std::uint64_t stream = 0) : seed_(seed), stream_(stream) {
    std::uint64_t x = seed;
    const std::uint64_t h = splitmix64(x);
    x = h ^ (0xD1B54A32D192ED03ULL * (stream + 1));
    engine_.seed(splitmix64(x));
  }
  SeededRng fork(std::uint64_t stream) const { return SeededRng(seed_, stream); }
  std::uint64_t next_u64() { return engine_(); }
  double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double uniform_pos() { return (static_cast<double>(next_u64() >> 11) + 1.0) * 0x1.0p-53; }
  std::uint64_t index(std::uint64_t n) {
    if (n == 0) throw std::invalid_argument("SeededRng::index: n must be positive");
    const std::uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    std::uint64_t x = next_u64();
    while (x >= limit) x = next_u64();
    return x % n;
  }
  double normal() {
    const double u1 = uniform_pos();
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
  }
  double normal(double mean, double sd) { return mean + sd * normal(); }

 private:
  std::uint64_t seed_, stream_;
  std::mt19937_64 engine_;
};

// ---------------------------------------------------------------- dense matrix (Eigen::MatrixXd stand-in)
struct Mat {
  Index r = 0, c = 0;
  std::vector<double> d;  // column-major
  Mat() = default;
  Mat(Index rows, Index cols) : r(rows), c(cols), d(static_cast<std::size_t>(rows * cols), 0.0) {}
  double& operator()(Index i, Index j) { return d[static_cast<std::size_t>(i + j * r)]; }
  double operator()(Index i, Index j) const { return d[static_cast<std::size_t>(i + j * r)]; }
  double* col(Index j) { return d.data() + j * r; }
  const double* col(Index j) const { return d.data() + j * r; }
  static Mat identity(Index n, Index k) {
    Mat I(n, k);
    for (Index i = 0; i < std::min(n, k); ++i) I(i, i) = 1.0;
    return I;
  }
  Mat left_cols(Index k) const {
    Mat o(r, k);
    std::copy(d.begin(), d.begin() + r * k, o.d.begin());
    return o;
  }
  Mat transpose() const {
    Mat o(c, r);
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) o(j, i) = (*this)(i, j);
    return o;
  }
  bool all_finite() const {
    for (double v : d)
      if (!std::isfinite(v)) return false;
    return true;
  }
  double sq_norm() const {
    double s = 0;
    for (double v : d) s += v * v;
    return s;
  }
};

// BLAS / LAPACK from numpy's bundled OpenBLAS (ILP64 symbols).
Mat gemm(bool ta, bool tb, double alpha, const Mat& A, const Mat& B);
void gemm_into(bool ta, bool tb, double alpha, const Mat& A, const Mat& B, double beta, Mat& C);
std::pair<Mat, Mat> thin_qr(const Mat& A);
struct Svd {
  Mat U;
  std::vector<double> s;
  Mat V;
};
Svd thin_svd(const Mat& A);  // BDCSVD(ComputeThinU|ComputeThinV) stand-in (dgesdd)

// ---------------------------------------------------------------- data model (P/include/dfc/matrix_io.hpp:36-123)
struct Observation {
  Index row, col;
  double value;
};

class ObservedMatrix {
 public:
  ObservedMatrix(Index m, Index n, std::vector<Observation> obs);
  Index rows() const { return m_; }
  Index cols() const { return n_; }
  Index count() const { return static_cast<Index>(obs_.size()); }
  bool empty() const { return obs_.empty(); }
  const std::vector<Observation>& entries() const { return obs_; }

 private:
  Index m_, n_;
  std::vector<Observation> obs_;
};

class LowRankEstimate {
 public:
  LowRankEstimate(Mat left, Mat right);
  static LowRankEstimate zero(Index m, Index n) { return LowRankEstimate(Mat(m, 0), Mat(n, 0)); }
  Index rows() const { return left_.r; }
  Index cols() const { return right_.r; }
  Index rank_bound() const { return left_.c; }
  const Mat& left() const { return left_; }
  const Mat& right() const { return right_; }

 private:
  Mat left_, right_;
};

struct SvdFactors {
  Mat U;
  std::vector<double> s;
  Mat V;
  Index rank() const { return static_cast<Index>(s.size()); }
  LowRankEstimate to_estimate() const;
};

Mat materialize(const LowRankEstimate& e);
Mat densify(const ObservedMatrix& obs);

// ---------------------------------------------------------------- sampling (P/include/dfc/sampling.hpp:15-113)
std::vector<Index> sample_without_replacement(Index n, Index l, SeededRng& rng);

class PartitionPlan {
 public:
  PartitionPlan(Index n, std::vector<std::vector<Index>> groups);
  Index total_cols() const { return n_; }
  std::size_t group_count() const { return groups_.size(); }
  const std::vector<Index>& group(std::size_t g) const { return groups_.at(g); }

 private:
  Index n_;
  std::vector<std::vector<Index>> groups_;
};

PartitionPlan partition_columns(Index n, Index t, SeededRng& rng);
ObservedMatrix extract_columns(const ObservedMatrix& obs, const std::vector<Index>& idx);
ObservedMatrix extract_rows(const ObservedMatrix& obs, const std::vector<Index>& idx);

// ---------------------------------------------------------------- simgen (P/include/dfc/simgen.hpp:30-82)
struct OutlierEstimate {
  Index m = 0, n = 0;
  std::vector<Observation> entries;
  OutlierEstimate(Index m_, Index n_, std::vector<Observation> e);
  Mat to_dense() const;
};
struct McInstance {
  LowRankEstimate L0;
  ObservedMatrix obs;
};
struct RmfInstance {
  LowRankEstimate L0;
  OutlierEstimate S0;
  Mat M;
};
LowRankEstimate gen_low_rank(Index m, Index n, Index r, SeededRng& rng);
McInstance gen_mc_instance(Index m, Index n, Index r, Index s, double sigma, SeededRng& rng);
// outlier_lo/outlier_hi: U[lo,hi] outliers; the reference draws U[0,1] (lo=0, hi=1).
RmfInstance gen_rmf_instance(Index m, Index n, Index r, Index s, double sigma, SeededRng& rng,
                             double outlier_lo = 0.0, double outlier_hi = 1.0);

// ---------------------------------------------------------------- sketch (P/include/dfc/sketch.hpp:15-298)
struct RpParams {
  Index k = 1, p = 5, q = 2;
};
struct RankTolerance {
  double rel_cutoff = 1e-12;
  double absolute(double s_max, Index m, Index n) const {
    return rel_cutoff * static_cast<double>(std::max(m, n)) * s_max;
  }
};
Index numerical_rank(const std::vector<double>& s, Index m, Index n, RankTolerance tol = {});
SvdFactors empty_svd(Index m, Index n);
SvdFactors truncated_svd(const Mat& A, Index k);
SvdFactors compact_svd(const Mat& A, RankTolerance tol = {});
SvdFactors svd_of_product(const Mat& left, const Mat& right, RankTolerance tol = {});
LowRankEstimate column_project(const LowRankEstimate& basis, const std::vector<LowRankEstimate>& blocks,
                               const PartitionPlan& plan, RankTolerance tol = {});
LowRankEstimate random_project(const std::vector<LowRankEstimate>& blocks, const PartitionPlan& plan,
                               const RpParams& params, SeededRng& rng, RankTolerance tol = {});
LowRankEstimate gen_nystrom(const LowRankEstimate& C_hat, const LowRankEstimate& R_hat,
                            const std::vector<Index>& row_idx, const std::vector<Index>& col_idx,
                            RankTolerance tol = {});
LowRankEstimate average_estimates(const std::vector<LowRankEstimate>& ests,
                                  std::optional<Index> recompress_to = std::nullopt,
                                  RankTolerance tol = {});

// ---------------------------------------------------------------- solvers (P/include/dfc/solvers.hpp:19-414)
struct ApgConfig {
  int max_iters = 500;
  double rel_tol = 1e-4;
  std::optional<double> mu_init, mu_floor;
  double mu_decay = 0.7;
  bool line_search = false;
  static ApgConfig high_accuracy() {
    ApgConfig c;
    c.rel_tol = 1e-9;
    c.mu_decay = 0.5;
    c.mu_floor = 0.0;
    c.max_iters = 400;
    return c;
  }
};
struct SolveReport {
  int iterations = 0;
  double objective = 0.0, residual = 0.0;
  Index rank = 0;
  double wall_ms = 0.0;
};
// Per-iteration trace for parity debugging (not in the reference; observation only).
struct IterTrace {
  int it;
  Index rank;      // rank of L_next
  Index k_final;   // k of the last partial SVD (0 = dense path)
  int svd_calls;   // partial/dense SVDs in this iteration (doubling retries + 1)
  double rel, mu, sigma_sum;
};

double default_rmf_lambda(Index m, Index n);
Mat soft_threshold(const Mat& A, double tau);
LowRankEstimate svt(const Mat& A, double tau);
std::pair<LowRankEstimate, SolveReport> apg_mc(const ObservedMatrix& obs, const ApgConfig& cfg = {},
                                               std::vector<IterTrace>* trace = nullptr);
std::tuple<LowRankEstimate, OutlierEstimate, SolveReport> apg_rmf(const Mat& M, double lambda,
                                                                  const ApgConfig& cfg = {},
                                                                  std::vector<IterTrace>* trace = nullptr);
double factored_inner(const LowRankEstimate& a, const LowRankEstimate& b);

namespace detail {
struct Csc;
}
// Resumable apg_mc (bench sampling of fixed iteration windows; same arithmetic as apg_mc).
struct ApgMcRun {
  ApgMcRun(const ObservedMatrix& obs, const ApgConfig& cfg);
  ~ApgMcRun();
  bool step(std::vector<IterTrace>* trace = nullptr);  // false once stopped / at max_iters
  std::pair<LowRankEstimate, SolveReport> finish() const;

  ObservedMatrix obs;
  ApgConfig cfg;
  std::unique_ptr<detail::Csc> M, R;
  std::vector<double> m_vals;
  double mu_init = 0, mu_floor = 0;
  SeededRng svd_rng;
  LowRankEstimate L_prev, L_curr;
  SvdFactors last;
  double tau_prev = 1.0, tau_curr = 1.0, mu = 0, mu_used = 0;
  Index rank_hint = 1;
  int iters = 0;
  bool stopped = false;
  std::chrono::steady_clock::time_point start;
};
double factored_diff_norm(const LowRankEstimate& a, const LowRankEstimate& b);

// ---------------------------------------------------------------- orchestrator (P/include/dfc/dfc.hpp:24-335)
enum class Task { MC = 0, RMF = 1 };
enum class DfcVariant { Proj = 0, Rp = 1, Nys = 2 };
namespace streams {
inline constexpr std::uint64_t partition = 0xDFC0000000000001ull;
inline constexpr std::uint64_t nys_rows = 0xDFC0000000000002ull;
inline constexpr std::uint64_t nys_cols = 0xDFC0000000000003ull;
inline constexpr std::uint64_t rp_draw = 0xDFC0000000000100ull;
}  // namespace streams
struct DfcConfig {
  DfcVariant variant = DfcVariant::Proj;
  bool ensemble = false;
  Index t = 4, l = 0, d = 0;
  RpParams rp;
  std::uint64_t seed = 0;
  ApgConfig solver_cfg;
  Task task = Task::MC;
  double lambda = 0.0;
  int workers = 1;
  Index ensemble_anchors = 0;  // extension (BASELINE c5 "ensemble of 4"): 0 = all t blocks
};
struct BlockError : std::runtime_error {
  BlockError(std::size_t block, const std::string& what)
      : std::runtime_error("block " + std::to_string(block) + ": " + what), block(block) {}
  std::size_t block;
};
struct DfcReport {
  std::vector<SolveReport> subproblems;
  double divide_ms = 0, factor_ms = 0, combine_ms = 0, total_ms = 0;
  Index chosen_k = 0;
  bool k_clamped = false, rank_deficient = false;
};
using BaseSolver = std::function<std::pair<LowRankEstimate, SolveReport>(const ObservedMatrix&)>;
BaseSolver make_base_solver(Task task, const ApgConfig& cfg, double lambda = 0.0);
Index median_rank(const std::vector<Index>& ranks);
std::pair<LowRankEstimate, DfcReport> dfc_proj(const ObservedMatrix& obs, const DfcConfig& cfg,
                                               const BaseSolver& solver);
std::pair<LowRankEstimate, DfcReport> dfc_rp(const ObservedMatrix& obs, const DfcConfig& cfg,
                                             const BaseSolver& solver);
std::pair<LowRankEstimate, DfcReport> dfc_nys(const ObservedMatrix& obs, const DfcConfig& cfg,
                                              const BaseSolver& solver);
std::pair<LowRankEstimate, DfcReport> dfc_run(const ObservedMatrix& obs, const DfcConfig& cfg);

}  // namespace orc
