// Compile-check stand-in for the reference's public types that integration/dfc_gpu.hpp uses
// (declarations mirror P/include/dfc/matrix_io.hpp:19-98, sampling.hpp:30-54, solvers.hpp:19-71,
// dfc.hpp:23-68 — names, members and signatures only; no algorithms). The real adapter builds
// against the reference's own headers.
#pragma once
#include <Eigen/Dense>
#include <cmath>
#include <functional>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace dfc {
using DenseMatrix = Eigen::MatrixXd;
using Index = Eigen::Index;

struct Observation {
  Index row, col;
  double value;
};
class ObservedMatrix {
 public:
  ObservedMatrix(Index m, Index n, std::vector<Observation> obs) : m_(m), n_(n), obs_(std::move(obs)) {}
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
  LowRankEstimate(DenseMatrix left, DenseMatrix right) : left_(std::move(left)), right_(std::move(right)) {}
  Index rows() const { return left_.rows(); }
  Index cols() const { return right_.rows(); }
  Index rank_bound() const { return left_.cols(); }
  const DenseMatrix& left() const { return left_; }
  const DenseMatrix& right() const { return right_; }

 private:
  DenseMatrix left_, right_;
};
inline DenseMatrix densify(const ObservedMatrix& obs) {
  DenseMatrix A = DenseMatrix::Zero(obs.rows(), obs.cols());
  for (const Observation& e : obs.entries()) A(e.row, e.col) = e.value;
  return A;
}
class PartitionPlan {
 public:
  PartitionPlan(Index n, std::vector<std::vector<Index>> groups) : n_(n), groups_(std::move(groups)) {}
  Index total_cols() const { return n_; }
  std::size_t group_count() const { return groups_.size(); }
  const std::vector<Index>& group(std::size_t g) const { return groups_.at(g); }

 private:
  Index n_;
  std::vector<std::vector<Index>> groups_;
};
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
  Index rank = 0;
  double wall_ms = 0.0;
};
inline double default_rmf_lambda(Index m, Index n) { return 1.0 / std::sqrt(static_cast<double>(std::max(m, n))); }
enum class Task { MC, RMF };
struct BlockError : std::runtime_error {
  BlockError(std::size_t block, const std::string& what)
      : std::runtime_error("block " + std::to_string(block) + ": " + what), block(block) {}
  std::size_t block;
};
using BaseSolver = std::function<std::pair<LowRankEstimate, SolveReport>(const ObservedMatrix&)>;
}  // namespace dfc
