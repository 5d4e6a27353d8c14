// Exercise integration/dfc_gpu.hpp through libdfcg.so.
//   check --cpu : error mapping through host-only entry points (no GPU needed)
//   check       : + a small MC block solved through make_gpu_base_solver, the DFC-Proj combine
//                 through column_project, and a failing dfc_run surfacing as BlockError with the
//                 reference's message ("block 0: ..." exactly once)
#include <cmath>
#include <cstdio>
#include <cstring>

#include "../include/dfcg_host.h"
#include "dfc_gpu.hpp"

using namespace dfc;

static int fails = 0;
#define EXPECT(c)                                              \
  do {                                                         \
    if (!(c)) {                                                \
      std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
      ++fails;                                                 \
    }                                                          \
  } while (0)

int main(int argc, char** argv) {
  const bool cpu_only = argc > 1 && std::strcmp(argv[1], "--cpu") == 0;
  // std::invalid_argument from DFCG_EINVAL
  try {
    gpu::check(dfcg_extract_subproblems(nullptr, 0, nullptr, nullptr, 0, nullptr, nullptr, nullptr, nullptr, nullptr));
    EXPECT(false);
  } catch (const std::invalid_argument& e) {
    EXPECT(std::strstr(e.what(), "null argument") != nullptr);
  }
  // std::out_of_range from DFCG_ERANGE: a column index outside the matrix
  {
    int64_t r[1] = {0}, c[1] = {0};
    double v[1] = {1.0};
    dfcg_obs in{2, 2, 1, r, c, v};
    int64_t offs[2] = {0, 1}, cols[1] = {5}, counts[1];
    int64_t *orr, *occ;
    double* ov;
    try {
      gpu::check(dfcg_extract_subproblems(&in, 1, offs, cols, 0, nullptr, counts, &orr, &occ, &ov));
      EXPECT(false);
    } catch (const std::out_of_range&) {
    }
  }
  if (cpu_only) {
    std::printf(fails ? "FAILED\n" : "OK cpu\n");
    return fails ? 1 : 0;
  }
  dfcg_ctx* ctx = nullptr;
  gpu::check(dfcg_ctx_create(0, &ctx));
  // MC instance from the library's restated generator, two column blocks
  const int64_t m = 60, n = 40;
  dfcg_lowrank L0{};
  int64_t *rows, *cols;
  double* vals;
  gpu::check(dfcg_gen_mc_instance(m, n, 2, 1600, 0.01, 3, 0, &L0, &rows, &cols, &vals));
  std::vector<std::vector<Observation>> parts(2);
  for (int64_t e = 0; e < 1600; ++e) parts[cols[e] < n / 2 ? 0 : 1].push_back({rows[e], cols[e] % (n / 2), vals[e]});
  auto solver = gpu::make_gpu_base_solver(ctx, Task::MC, ApgConfig{});
  std::vector<LowRankEstimate> ests;
  for (auto& p : parts) {
    auto [est, rep] = solver(ObservedMatrix(m, n / 2, p));
    EXPECT(rep.iterations > 0 && est.rank_bound() > 0 && est.rows() == m && est.cols() == n / 2);
    ests.push_back(est);
  }
  std::vector<Index> g0, g1;
  for (Index j = 0; j < n / 2; ++j) g0.push_back(j), g1.push_back(n / 2 + j);
  PartitionPlan plan(n, {g0, g1});
  LowRankEstimate out = gpu::column_project(ctx, ests[0], ests, plan);
  EXPECT(out.rows() == m && out.cols() == n && out.rank_bound() > 0);
  // DFCG_EBLOCK -> BlockError with a single "block N: " prefix
  {
    dfcg_obs in{m, n, 1600, rows, cols, vals};
    dfcg_dfc_cfg cfg{};
    cfg.t = 2;
    cfg.seed = 1;
    cfg.workers = 2;
    cfg.solver = gpu::to_c(ApgConfig{});
    cfg.solver.rel_tol = 2.0;  // invalid: every block fails validate_config
    dfcg_lowrank o{};
    try {
      gpu::check(dfcg_dfc_run(ctx, &in, &cfg, &o, nullptr));
      EXPECT(false);
    } catch (const BlockError& e) {
      EXPECT(e.block == 0);
      EXPECT(std::strncmp(e.what(), "block 0: ", 9) == 0);
      EXPECT(std::strstr(e.what() + 9, "block 0:") == nullptr);
    }
  }
  dfcg_free(rows);
  dfcg_free(cols);
  dfcg_free(vals);
  dfcg_lowrank_free(&L0);
  dfcg_ctx_destroy(ctx);
  std::printf(fails ? "FAILED\n" : "OK gpu\n");
  return fails ? 1 : 0;
}
