// dfc/gpu.hpp — the adapter a reference maintainer adds to plug libdfcg.so into the reference's
// seams: BaseSolver (P/include/dfc/dfc.hpp:67-78) and the combiners
// (P/include/dfc/sketch.hpp:170-199). Compiled in this repo against integration/stub/ (a
// declarations-only stand-in for the reference headers and Eigen) by tests/test_integration_cpu.py.
#pragma once
#include <dfcg.h>  // -I<repo>/include, link -L<repo>/paper_1107_0789_b200/_lib -ldfcg

#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dfc/dfc.hpp"

namespace dfc::gpu {

// Error code -> the reference's exception types. For DFCG_EBLOCK dfcg_last_error() is the failing
// block's own message; BlockError's constructor adds the "block N: " prefix (dfc.hpp:50-54).
inline void check(int rc) {
  if (rc == DFCG_OK) return;
  const std::string msg = dfcg_last_error();
  if (rc == DFCG_EINVAL) throw std::invalid_argument(msg);
  if (rc == DFCG_ERANGE) throw std::out_of_range(msg);
  if (rc == DFCG_EBLOCK) throw BlockError(static_cast<std::size_t>(dfcg_last_error_block()), msg);
  throw std::runtime_error(msg);
}

inline dfcg_apg_cfg to_c(const ApgConfig& c) {
  return {c.max_iters, c.rel_tol, c.mu_init.has_value(), c.mu_init.value_or(0.0),
          c.mu_floor.has_value(), c.mu_floor.value_or(0.0), c.mu_decay, c.line_search};
}

inline LowRankEstimate take(dfcg_lowrank& e) {  // copy out, free the library buffers
  LowRankEstimate out(Eigen::Map<DenseMatrix>(e.left, e.m, e.k), Eigen::Map<DenseMatrix>(e.right, e.n, e.k));
  dfcg_lowrank_free(&e);
  return out;
}

inline SolveReport from_c(const dfcg_solve_report& r) {
  return SolveReport{r.iterations, r.objective, r.residual, r.rank, r.wall_ms};
}

// Drop-in for make_base_solver(task, cfg, lambda): same signature, same results (to 1e-6 relF).
inline BaseSolver make_gpu_base_solver(dfcg_ctx* ctx, Task task, const ApgConfig& cfg, double lambda = 0.0) {
  return [=](const ObservedMatrix& block) {
    if (task == Task::MC) {
      std::vector<int64_t> r, c;
      std::vector<double> v;
      for (const auto& e : block.entries()) {  // already sorted column-major (matrix_io.hpp:41-43)
        r.push_back(e.row);
        c.push_back(e.col);
        v.push_back(e.value);
      }
      dfcg_obs in{block.rows(), block.cols(), block.count(), r.data(), c.data(), v.data()};
      dfcg_apg_cfg cc = to_c(cfg);
      dfcg_lowrank out{};
      dfcg_solve_report rep{};
      check(dfcg_apg_mc(ctx, &in, &cc, &out, &rep, nullptr, 0, nullptr));
      return std::pair<LowRankEstimate, SolveReport>{take(out), from_c(rep)};
    }
    const double lam = lambda > 0 ? lambda : default_rmf_lambda(block.rows(), block.cols());
    DenseMatrix M = densify(block);
    dfcg_apg_cfg cc = to_c(cfg);
    dfcg_lowrank L{};
    dfcg_sparse S{};
    dfcg_solve_report rep{};
    check(dfcg_apg_rmf(ctx, M.data(), M.rows(), M.cols(), lam, &cc, &L, &S, &rep, nullptr, 0, nullptr));
    dfcg_sparse_free(&S);  // DFC drops S_hat, exactly like make_base_solver (dfc.hpp:75-76)
    return std::pair<LowRankEstimate, SolveReport>{take(L), from_c(rep)};
  };
}

// Drop-in for column_project(basis, blocks, plan).
inline LowRankEstimate column_project(dfcg_ctx* ctx, const LowRankEstimate& basis,
                                      const std::vector<LowRankEstimate>& blocks, const PartitionPlan& plan) {
  auto view = [](const LowRankEstimate& e) {
    return dfcg_lowrank{e.rows(), e.cols(), e.rank_bound(), const_cast<double*>(e.left().data()),
                        const_cast<double*>(e.right().data())};
  };
  std::vector<dfcg_lowrank> bl;
  std::vector<int64_t> offs{0}, cols;
  for (std::size_t g = 0; g < blocks.size(); ++g) {
    bl.push_back(view(blocks[g]));
    cols.insert(cols.end(), plan.group(g).begin(), plan.group(g).end());
    offs.push_back(static_cast<int64_t>(cols.size()));
  }
  dfcg_lowrank b = view(basis), out{};
  check(dfcg_column_project(ctx, &b, static_cast<int64_t>(bl.size()), bl.data(), offs.data(), cols.data(),
                            plan.total_cols(), &out));
  return take(out);
}

}  // namespace dfc::gpu
