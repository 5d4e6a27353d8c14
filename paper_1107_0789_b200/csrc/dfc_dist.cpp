// Multi-GPU dfc_run (one process per GPU): the reference's D-F-C pipeline
// (P/include/dfc/dfc.hpp:166-335) with the subproblems sharded over ranks.
//
//   D  every rank derives the same plan (same RNG streams), counts each subproblem's
//      observations, assigns subproblems to ranks by LPT on nnz, and extracts only its own;
//   F  each rank solves its subproblems concurrently on its GPU (no exchange);
//   C  only factors move, over the Comm (NCCL on NVLink, or host callbacks):
//        Proj      basis U_b of block 0 broadcast from its owner, every rank projects its own
//                  blocks (project_rows), the w_g x k_b row slabs are gathered to the root;
//        Proj-Ens  every anchor basis U_i broadcast from its owner, each rank projects its
//                  blocks onto all of them, rows gathered to rank 0, average_estimates there;
//        Nys       R-hat's factors sent to C-hat's rank; Nys-Ens: R-hat broadcast, each rank
//                  runs gen_nystrom for its column groups, the results gathered to rank 0;
//        Rp        block factors gathered to rank 0, random_project there (every draw needs
//                  every block).
//   The final estimate is broadcast from the combining rank, so every rank returns it.
// Every device operation is the single-GPU path's own kernel on the same operands, so the
// result equals dfc_run's.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "dfc_host.hpp"
#include "dist.hpp"

namespace dfcg {

namespace {

struct SubDef {
  bool by_rows = false;  // extract_rows(idx) (Nys R-hat) or extract_columns(idx)
  std::vector<i64> idx;
};

// Observation counts of every subproblem in one pass over the triplets.
std::vector<i64> count_obs(const HostObs& obs, const std::vector<SubDef>& subs) {
  std::vector<i64> nnz(subs.size(), 0);
  std::vector<int> col_sub(static_cast<size_t>(obs.n), -1);
  int row_sub_id = -1;
  std::vector<char> in_rows;
  for (size_t i = 0; i < subs.size(); ++i) {
    if (subs[i].by_rows) {
      row_sub_id = static_cast<int>(i);
      in_rows.assign(static_cast<size_t>(obs.m), 0);
      for (i64 r : subs[i].idx) in_rows[static_cast<size_t>(r)] = 1;
    } else {
      for (i64 c : subs[i].idx) col_sub[static_cast<size_t>(c)] = static_cast<int>(i);
    }
  }
  for (i64 e = 0; e < obs.count(); ++e) {
    const int cs = col_sub[static_cast<size_t>(obs.col[e])];
    if (cs >= 0) ++nnz[static_cast<size_t>(cs)];
    if (row_sub_id >= 0 && in_rows[static_cast<size_t>(obs.row[e])]) ++nnz[static_cast<size_t>(row_sub_id)];
  }
  return nnz;
}

// Block report + estimate rank, shared from the owner (trivially copyable).
struct SubInfo {
  SolveReport rep;
  i64 k;
};

class Dist {
 public:
  Dist(DeviceContext& ctx, Comm& comm) : ctx_(ctx), comm_(comm), cs_(ctx) {}
  cudaStream_t s() const { return cs_.s; }
  int rank() const { return comm_.rank(); }

  template <class T>
  void share(T& v, int root) {
    comm_.bcast_host(&v, sizeof(T), root);
  }
  // estimate (dims m, n known everywhere) from root to every rank
  void bcast_est(DevLowRank& e, int root) {
    share(e.k, root);
    if (e.k == 0) return;
    if (rank() != root) {
      e.left.alloc(e.m * e.k, s());
      e.right.alloc(e.n * e.k, s());
    }
    comm_.bcast(e.left.get(), sizeof(double) * static_cast<size_t>(e.m * e.k), root, s());
    comm_.bcast(e.right.get(), sizeof(double) * static_cast<size_t>(e.n * e.k), root, s());
    DFCG_CUDA(cudaStreamSynchronize(s()));
  }
  // estimates ests[i] (k known everywhere) from their owners to `dst`, one batch
  void gather_ests(std::vector<DevLowRank>& ests, const std::vector<int>& owner, const std::vector<size_t>& which,
                   int dst) {
    std::vector<Comm::Xfer> ops;
    for (size_t i : which) {
      DevLowRank& e = ests[i];
      if (e.k == 0 || owner[i] == dst) continue;
      if (rank() == dst) {
        e.left.alloc(e.m * e.k, s());
        e.right.alloc(e.n * e.k, s());
      }
      ops.push_back({owner[i], dst, e.left.get(), e.left.get(), sizeof(double) * static_cast<size_t>(e.m * e.k)});
      ops.push_back({owner[i], dst, e.right.get(), e.right.get(), sizeof(double) * static_cast<size_t>(e.n * e.k)});
    }
    DFCG_CUDA(cudaStreamSynchronize(s()));  // receive buffers allocated before the transport uses them
    comm_.exchange(ops, s());
    DFCG_CUDA(cudaStreamSynchronize(s()));
  }
  Comm& comm() { return comm_; }

 private:
  DeviceContext& ctx_;
  Comm& comm_;
  CallStream cs_;
};

}  // namespace

std::pair<DevLowRank, DfcReport> dfc_run_dist(DeviceContext& ctx, Comm& comm, const HostObs& obs, const DfcConfig& cfg,
                                              std::vector<int>* owner_out) {
  const i64 m = obs.m, n = obs.n;
  if (cfg.ensemble_anchors != 0 && cfg.variant != DfcVariant::Proj)
    throw std::invalid_argument("dfc_run: ensemble_anchors applies to DFC-Proj-Ens only");
  if (cfg.ensemble_anchors < 0) throw std::invalid_argument("dfc_proj: ensemble_anchors must be >= 0");
  if (cfg.ensemble_anchors > 0 && !cfg.ensemble)
    throw std::invalid_argument("dfc_proj: ensemble_anchors needs ensemble = true");
  if (cfg.workers < 1) throw std::invalid_argument("parallel_for: workers must be >= 1");
  const BaseSolver solver = make_base_solver(ctx, cfg.task, cfg.solver_cfg, cfg.lambda);
  DfcReport report;
  PhaseClock total, phase;

  // ---- D: the reference's plan (same streams), subproblem list, LPT owners
  std::vector<std::vector<i64>> plan;
  std::vector<i64> row_idx, col_idx;
  std::vector<SubDef> subs;
  if (cfg.variant == DfcVariant::Proj || cfg.variant == DfcVariant::Rp) {
    if (cfg.t < 1 || cfg.t > n)
      throw std::invalid_argument(cfg.variant == DfcVariant::Proj ? "dfc_proj: need 1 <= t <= n"
                                                                  : "dfc_rp: need 1 <= t <= n");
    SeededRng prng(cfg.seed, streams::partition);
    plan = partition_columns(n, cfg.t, prng);
    for (const auto& g : plan) subs.push_back({false, g});
  } else {
    if (cfg.l < 1 || cfg.l > n) throw std::invalid_argument("dfc_nys: need 1 <= l <= n");
    if (cfg.d < 1 || cfg.d > m) throw std::invalid_argument("dfc_nys: need 1 <= d <= m");
    SeededRng row_rng(cfg.seed, streams::nys_rows);
    row_idx = sample_without_replacement(m, cfg.d, row_rng);
    std::sort(row_idx.begin(), row_idx.end());
    if (!cfg.ensemble) {
      SeededRng col_rng(cfg.seed, streams::nys_cols);
      col_idx = sample_without_replacement(n, cfg.l, col_rng);
      std::sort(col_idx.begin(), col_idx.end());
      subs.push_back({false, col_idx});
    } else {
      const i64 groups =
          std::clamp<i64>(static_cast<i64>(std::llround(static_cast<double>(n) / static_cast<double>(cfg.l))), 1, n);
      SeededRng prng(cfg.seed, streams::partition);
      plan = partition_columns(n, groups, prng);
      for (const auto& g : plan) subs.push_back({false, g});
    }
    subs.push_back({true, row_idx});
  }
  const std::vector<i64> nnz = count_obs(obs, subs);
  const std::vector<int> owner = assign_blocks_lpt(nnz, comm.size());
  if (owner_out) *owner_out = owner;
  std::vector<size_t> mine;
  for (size_t i = 0; i < subs.size(); ++i)
    if (owner[i] == comm.rank()) mine.push_back(i);
  // this rank's subproblems in one parallel pass (column groups first, then the row sample)
  std::vector<std::vector<i64>> own_cols;
  const std::vector<i64>* own_rows = nullptr;
  for (size_t i : mine) {
    if (subs[i].by_rows) own_rows = &subs[i].idx;
    else own_cols.push_back(subs[i].idx);
  }
  std::vector<HostObs> extracted = extract_subproblems(obs, own_cols, own_rows);
  std::vector<HostObs> blocks(mine.size());
  for (size_t j = 0, c = 0; j < mine.size(); ++j)
    blocks[j] = std::move(subs[mine[j]].by_rows ? extracted.back() : extracted[c++]);
  report.divide_ms = phase.lap();

  // ---- F: own subproblems, concurrently on this GPU
  std::vector<DevLowRank> ests(subs.size());
  for (size_t i = 0; i < subs.size(); ++i) {
    ests[i].m = subs[i].by_rows ? static_cast<i64>(subs[i].idx.size()) : m;
    ests[i].n = subs[i].by_rows ? n : static_cast<i64>(subs[i].idx.size());
  }
  std::vector<SubInfo> info(subs.size(), SubInfo{SolveReport{}, 0});
  std::string local_err;
  int local_fail = -1;
  try {
    parallel_for(ctx, mine.size(), cfg.workers, [&](std::size_t j, cudaStream_t s) {
      const size_t i = mine[j];
      if (blocks[j].empty()) return;  // zero estimate, no solver call (dfc.hpp:139-142)
      auto [est, rep] = solver(blocks[j], s);
      ests[i] = std::move(est);
      info[i] = {rep, ests[i].k};
    });
  } catch (const BlockError& e) {
    local_fail = static_cast<int>(mine[e.block]);
    local_err = e.inner;
  }
  Dist D(ctx, comm);
  // the lowest failing subproblem over all ranks wins (dfc.hpp:117-118), raised on every rank
  {
    int first = -1, first_rank = -1;
    for (int q = 0; q < comm.size(); ++q) {
      int f = q == comm.rank() ? local_fail : -1;
      D.share(f, q);
      if (f >= 0 && (first < 0 || f < first)) first = f, first_rank = q;
    }
    if (first >= 0) {
      char msg[512] = {0};
      if (comm.rank() == first_rank) std::strncpy(msg, local_err.c_str(), sizeof(msg) - 1);
      comm.bcast_host(msg, sizeof(msg), first_rank);
      throw BlockError(static_cast<std::size_t>(first), msg);
    }
  }
  for (size_t i = 0; i < subs.size(); ++i) D.share(info[i], owner[i]);
  for (size_t i = 0; i < subs.size(); ++i) {
    report.subproblems.push_back(info[i].rep);
    ests[i].k = info[i].k;
  }
  report.factor_ms = phase.lap();

  // ---- C
  const cudaStream_t s = D.s();
  DevLowRank out;
  out.m = m;
  out.n = n;
  int final_root = 0;
  auto all_ranks = [&] {
    std::vector<i64> r;
    for (const auto& e : ests) r.push_back(e.k);
    return r;
  };
  // anchor basis U_i = svd_of_product(ests[i]).U, computed on its owner, broadcast to all
  auto anchor_basis = [&](size_t i, DBuf<double>& U) {
    i64 kb = 0;
    if (comm.rank() == owner[i]) {
      SvdOfProduct bf = svd_of_product(s, m, ests[i].n, ests[i].k, ests[i].left.get(), ests[i].right.get());
      kb = bf.r;
      if (kb > 0) U = std::move(bf.U);
    }
    D.share(kb, owner[i]);
    if (kb > 0) {
      if (comm.rank() != owner[i]) U.alloc(m * kb, s);
      DFCG_CUDA(cudaStreamSynchronize(s));
      comm.bcast(U.get(), sizeof(double) * static_cast<size_t>(m * kb), owner[i], s);
    }
    return kb;
  };
  // rows of every block projected onto U (m x kb) gathered to `root`, scattered into right (n x kb)
  auto project_gather = [&](const DBuf<double>& U, i64 kb, int root, DBuf<double>& right) {
    std::vector<DBuf<double>> Rg(plan.size());
    for (size_t g = 0; g < plan.size(); ++g) {
      const i64 w = static_cast<i64>(plan[g].size());
      if (ests[g].k == 0) continue;
      if (owner[g] == comm.rank()) {
        Rg[g].alloc(w * kb, s);
        project_rows(s, U.get(), m, kb, ests[g], Rg[g].get());
      } else if (comm.rank() == root) {
        Rg[g].alloc(w * kb, s);
      }
    }
    DFCG_CUDA(cudaStreamSynchronize(s));
    std::vector<Comm::Xfer> ops;
    for (size_t g = 0; g < plan.size(); ++g)
      if (ests[g].k > 0)
        ops.push_back({owner[g], root, Rg[g].get(), Rg[g].get(),
                       sizeof(double) * static_cast<size_t>(static_cast<i64>(plan[g].size()) * kb)});
    comm.exchange(ops, s);
    if (comm.rank() == root) {
      right.alloc(n * kb, s);
      right.zero(s);
      for (size_t g = 0; g < plan.size(); ++g)
        if (ests[g].k > 0) scatter_rows(s, Rg[g].get(), static_cast<i64>(plan[g].size()), kb, plan[g], right.get());
    }
    DFCG_CUDA(cudaStreamSynchronize(s));
  };

  if (cfg.variant == DfcVariant::Proj && !cfg.ensemble) {
    // column_project(ests[0], ests, plan) (dfc.hpp:189)
    final_root = owner[0];
    DBuf<double> U;
    const i64 kb = anchor_basis(0, U);
    if (kb > 0) {
      DBuf<double> right;
      project_gather(U, kb, final_root, right);
      if (comm.rank() == final_root) {
        out.k = kb;
        out.left = std::move(U);
        out.right = std::move(right);
      }
    }
  } else if (cfg.variant == DfcVariant::Proj) {
    // every anchor's column_project, averaged and recompressed to the median block rank
    // (dfc.hpp:191-195; first ensemble_anchors groups when set)
    const size_t anchors = cfg.ensemble_anchors > 0
                               ? std::min<size_t>(static_cast<size_t>(cfg.ensemble_anchors), ests.size())
                               : ests.size();
    final_root = 0;
    std::vector<DevLowRank> projected(anchors);
    for (size_t i = 0; i < anchors; ++i) {
      DBuf<double> U;
      projected[i].m = m;
      projected[i].n = n;
      const i64 kb = anchor_basis(i, U);
      if (kb == 0) continue;
      DBuf<double> right;
      project_gather(U, kb, final_root, right);
      if (comm.rank() == final_root) {
        projected[i].k = kb;
        projected[i].left = std::move(U);
        projected[i].right = std::move(right);
      }
    }
    if (comm.rank() == final_root) {
      std::vector<const DevLowRank*> p;
      for (const auto& e : projected) p.push_back(&e);
      average_estimates(s, p, median_rank(all_ranks()), out);
    }
  } else if (cfg.variant == DfcVariant::Rp) {
    // random_project needs every block in every draw: factors gathered to rank 0 (dfc.hpp:202-248)
    final_root = 0;
    std::vector<size_t> every(ests.size());
    for (size_t i = 0; i < every.size(); ++i) every[i] = i;
    D.gather_ests(ests, owner, every, final_root);
    i64 k = median_rank(all_ranks()), p = cfg.rp_p;
    const i64 minmn = std::min(m, n);
    if (k + p > minmn) {
      report.k_clamped = true;
      p = std::min(p, minmn - 1);
      k = minmn - p;
    }
    report.chosen_k = k;
    if (comm.rank() == final_root) {
      std::vector<const DevLowRank*> bl;
      for (const auto& e : ests) bl.push_back(&e);
      if (!cfg.ensemble) {
        SeededRng rng(cfg.seed, streams::rp_draw);
        random_project(s, bl, plan, n, k, p, cfg.rp_q, rng, out);
      } else {
        std::vector<DevLowRank> draws(static_cast<size_t>(cfg.t));
        parallel_for(ctx, draws.size(), cfg.workers, [&](std::size_t i, cudaStream_t st) {
          SeededRng rng(cfg.seed, streams::rp_draw + 1 + i);
          random_project(st, bl, plan, n, k, p, cfg.rp_q, rng, draws[i]);
        });
        std::vector<const DevLowRank*> dp;
        for (const auto& e : draws) dp.push_back(&e);
        average_estimates(s, dp, k, out);
      }
    }
  } else if (!cfg.ensemble) {
    // Nys: R-hat's factors to C-hat's rank, gen_nystrom there (dfc.hpp:290-296)
    final_root = owner[0];
    D.gather_ests(ests, owner, {1}, final_root);
    int deficient = 0;
    if (comm.rank() == final_root) {
      deficient = nys_pair_deficient(s, ests[0], ests[1], row_idx) ? 1 : 0;
      gen_nystrom(s, ests[0], ests[1], row_idx, col_idx, out);
    }
    D.share(deficient, final_root);
    report.rank_deficient = deficient != 0;
  } else {
    // Nys-Ens: R-hat broadcast, gen_nystrom per column group on its owner, results averaged on
    // rank 0 (dfc.hpp:298-323)
    final_root = 0;
    const size_t nc = ests.size() - 1;
    D.bcast_est(ests[nc], owner[nc]);
    std::vector<DevLowRank> combined(nc);
    std::vector<int> deficient(nc, 0);
    std::vector<size_t> own_cols;
    for (size_t i = 0; i < nc; ++i)
      if (owner[i] == comm.rank()) own_cols.push_back(i);
    parallel_for(ctx, own_cols.size(), cfg.workers, [&](std::size_t j, cudaStream_t st) {
      const size_t i = own_cols[j];
      deficient[i] = nys_pair_deficient(st, ests[i], ests[nc], row_idx) ? 1 : 0;
      gen_nystrom(st, ests[i], ests[nc], row_idx, plan[i], combined[i]);
    });
    std::vector<size_t> all_cols(nc);
    for (size_t i = 0; i < nc; ++i) {
      all_cols[i] = i;
      combined[i].m = m;
      combined[i].n = n;
      D.share(combined[i].k, owner[i]);
      D.share(deficient[i], owner[i]);
      report.rank_deficient = report.rank_deficient || deficient[i];
    }
    std::vector<int> own_map(owner.begin(), owner.begin() + static_cast<std::ptrdiff_t>(nc));
    D.gather_ests(combined, own_map, all_cols, final_root);
    std::vector<i64> col_ranks;
    for (size_t i = 0; i < nc; ++i) col_ranks.push_back(ests[i].k);
    if (comm.rank() == final_root) {
      std::vector<const DevLowRank*> p;
      for (const auto& e : combined) p.push_back(&e);
      average_estimates(s, p, median_rank(col_ranks), out);
    }
  }
  D.bcast_est(out, final_root);
  report.combine_ms = phase.lap();
  report.total_ms = total.lap();
  return {std::move(out), std::move(report)};
}

}  // namespace dfcg
