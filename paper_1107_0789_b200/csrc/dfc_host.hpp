// Host-side DFC orchestrator (C++), mirroring P/include/dfc/dfc.hpp and the D-step helpers of
// P/include/dfc/sampling.hpp. The F-step BaseSolver and the C-step combiners run on the
// device; estimates stay resident in HBM between the steps.
#pragma once

#include <atomic>
#include <chrono>
#include <functional>
#include <thread>
#include <string>
#include <utility>
#include <vector>

#include "solver.hpp"

namespace dfcg {

// ObservedMatrix (matrix_io.hpp:36-67): triplets sorted column-major, validated.
struct HostObs {
  i64 m = 0, n = 0;
  std::vector<long long> row, col;
  std::vector<double> val;
  i64 count() const { return static_cast<i64>(val.size()); }
  bool empty() const { return val.empty(); }
  static HostObs make(i64 m, i64 n, std::vector<long long> row, std::vector<long long> col, std::vector<double> val);
};

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
  i64 t = 4, l = 0, d = 0;
  i64 rp_p = 5, rp_q = 2;
  std::uint64_t seed = 0;
  ApgConfig solver_cfg;
  Task task = Task::MC;
  double lambda = 0.0;
  int workers = 1;
  // Proj-Ens anchors (BASELINE c5 "ensemble of 4"; not in the reference, whose ensemble anchors
  // on every block, dfc.hpp:191-195): 0 = all t blocks, else the first min(A, t) plan groups.
  i64 ensemble_anchors = 0;
};

struct BlockError : std::runtime_error {
  BlockError(std::size_t block, const std::string& what)
      : std::runtime_error("block " + std::to_string(block) + ": " + what), block(block), inner(what) {}
  std::size_t block;
  std::string inner;  // the failing block's own message, without the "block N: " prefix
};

struct DfcReport {
  std::vector<SolveReport> subproblems;
  double divide_ms = 0, factor_ms = 0, combine_ms = 0, total_ms = 0;
  i64 chosen_k = 0;
  bool k_clamped = false, rank_deficient = false;
};

// BaseSolver (dfc.hpp:67-68), returning a device-resident estimate.
using BaseSolver = std::function<std::pair<DevLowRank, SolveReport>(const HostObs&, cudaStream_t)>;
BaseSolver make_base_solver(DeviceContext& ctx, Task task, const ApgConfig& cfg, double lambda = 0.0);

// parallel_for, dfc.hpp:84-119 — each worker thread holds its own pooled stream.
template <class Fn>
void parallel_for(DeviceContext& ctx, std::size_t count, int workers, Fn&& fn) {
  if (workers < 1) throw std::invalid_argument("parallel_for: workers must be >= 1");
  const std::size_t nthreads = std::min<std::size_t>(static_cast<std::size_t>(workers), count);
  std::vector<std::string> failures(count);
  std::vector<char> failed(count, 0);
  if (nthreads <= 1) {
    CallStream cs(ctx);
    for (std::size_t i = 0; i < count; ++i) {
      try {
        fn(i, cs.s);
      } catch (const std::exception& e) {
        throw BlockError(i, e.what());
      }
    }
    return;
  }
  std::atomic<std::size_t> next{0};
  auto worker = [&]() {
    CallStream cs(ctx);
    for (;;) {
      const std::size_t i = next.fetch_add(1);
      if (i >= count) return;
      try {
        fn(i, cs.s);
      } catch (const std::exception& e) {
        failures[i] = e.what();
        failed[i] = 1;
      }
    }
  };
  std::vector<std::thread> pool;
  for (std::size_t w = 0; w < nthreads; ++w) pool.emplace_back(worker);
  for (auto& th : pool) th.join();
  for (std::size_t i = 0; i < count; ++i)
    if (failed[i]) throw BlockError(i, failures[i]);
}

struct PhaseClock {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double lap() {
    const auto t1 = std::chrono::steady_clock::now();
    const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    t0 = t1;
    return ms;
  }
};

std::vector<i64> sample_without_replacement(i64 n, i64 l, SeededRng& rng);
std::vector<std::vector<i64>> partition_columns(i64 n, i64 t, SeededRng& rng);
HostObs extract_columns(const HostObs& obs, const std::vector<i64>& idx);
// The D step's extraction of every subproblem in one parallel pass: disjoint column groups,
// then (rows != nullptr) one row sample (extract_rows). Same outputs as the one-at-a-time calls.
std::vector<HostObs> extract_subproblems(const HostObs& obs, const std::vector<std::vector<i64>>& col_groups,
                                         const std::vector<i64>* rows);
HostObs extract_rows(const HostObs& obs, const std::vector<i64>& idx);
i64 median_rank(const std::vector<i64>& ranks);
bool nys_pair_deficient(cudaStream_t s, const DevLowRank& C, const DevLowRank& R, const std::vector<i64>& row_idx);

std::pair<DevLowRank, DfcReport> dfc_run(DeviceContext& ctx, const HostObs& obs, const DfcConfig& cfg);

// Multi-GPU dfc_run (one process per GPU, dist.hpp): every rank passes the same obs and cfg,
// solves its LPT share of the subproblems and joins the combine's exchange; every rank returns
// the final estimate. Same arithmetic as dfc_run, so the result matches it (P/tests/test_dfc.cpp:
// 322-342's scheduling invariance, extended to ranks).
class Comm;
std::pair<DevLowRank, DfcReport> dfc_run_dist(DeviceContext& ctx, Comm& comm, const HostObs& obs, const DfcConfig& cfg,
                                              std::vector<int>* owner_out = nullptr);
std::pair<DevLowRank, DfcReport> dfc_proj(DeviceContext& ctx, const HostObs& obs, const DfcConfig& cfg,
                                          const BaseSolver& solver);
std::pair<DevLowRank, DfcReport> dfc_rp(DeviceContext& ctx, const HostObs& obs, const DfcConfig& cfg,
                                        const BaseSolver& solver);
std::pair<DevLowRank, DfcReport> dfc_nys(DeviceContext& ctx, const HostObs& obs, const DfcConfig& cfg,
                                         const BaseSolver& solver);

}  // namespace dfcg
