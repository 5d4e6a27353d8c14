// Host DFC orchestrator (see dfc_host.hpp). Restates dfc_proj / dfc_rp / dfc_nys
// (P/include/dfc/dfc.hpp:166-335) and the D-step (P/include/dfc/sampling.hpp:15-113) with
// the same RNG stream ids, so partitions and samples are identical to the reference's.
// Block solves run concurrently on one device (one pooled stream per worker thread).
#include "dfc_host.hpp"

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <chrono>
#include <cmath>
#include <numeric>
#include <thread>

namespace dfcg {

HostObs HostObs::make(i64 m, i64 n, std::vector<long long> row, std::vector<long long> col, std::vector<double> val) {
  if (m < 1 || n < 1) throw std::invalid_argument("ObservedMatrix: dims must be positive");
  const size_t N = val.size();
  if (row.size() != N || col.size() != N) throw std::invalid_argument("ObservedMatrix: ragged triplets");
  std::vector<size_t> ord(N);
  std::iota(ord.begin(), ord.end(), size_t{0});
  bool sorted = true;
  for (size_t i = 1; i < N && sorted; ++i)
    sorted = col[i - 1] < col[i] || (col[i - 1] == col[i] && row[i - 1] <= row[i]);
  HostObs o;
  o.m = m;
  o.n = n;
  if (!sorted) {
    std::stable_sort(ord.begin(), ord.end(),
                     [&](size_t a, size_t b) { return col[a] != col[b] ? col[a] < col[b] : row[a] < row[b]; });
    o.row.resize(N);
    o.col.resize(N);
    o.val.resize(N);
    for (size_t i = 0; i < N; ++i) {
      o.row[i] = row[ord[i]];
      o.col[i] = col[ord[i]];
      o.val[i] = val[ord[i]];
    }
  } else {
    o.row = std::move(row);
    o.col = std::move(col);
    o.val = std::move(val);
  }
  for (size_t i = 0; i < N; ++i) {
    if (o.row[i] < 0 || o.row[i] >= m || o.col[i] < 0 || o.col[i] >= n)
      throw std::out_of_range("ObservedMatrix: entry (" + std::to_string(o.row[i]) + ", " + std::to_string(o.col[i]) +
                              ") outside " + std::to_string(m) + "x" + std::to_string(n));
    if (!std::isfinite(o.val[i])) throw std::invalid_argument("ObservedMatrix: non-finite value");
    if (i > 0 && o.row[i - 1] == o.row[i] && o.col[i - 1] == o.col[i])
      throw std::invalid_argument("ObservedMatrix: duplicate entry (" + std::to_string(o.row[i]) + ", " +
                                  std::to_string(o.col[i]) + ")");
  }
  return o;
}

// sampling.hpp:15-26. For a large population the partial Fisher-Yates runs on a hash map of
// the displaced positions (open addressing, ~32 bytes per draw) instead of an n-element
// permutation: the same RNG calls and swaps, so the same output, without the 12.8 GB index
// vector of BASELINE c5 (n = 1.6e9 cells, l = 8e7). DFCG_SWR_SPARSE=0 / 1 forces a path.
std::vector<i64> sample_without_replacement(i64 n, i64 l, SeededRng& rng) {
  if (n < 1) throw std::invalid_argument("sample_without_replacement: empty population");
  if (l < 1 || l > n) throw std::invalid_argument("sample_without_replacement: need 1 <= l <= n");
  const char* env = std::getenv("DFCG_SWR_SPARSE");
  const int mode = env ? std::atoi(env) : -1;
  const bool sparse = mode == 1 || (mode != 0 && n > (i64{1} << 27) && l < n / 4);
  if (sparse) {
    size_t cap = 16;
    while (cap < static_cast<size_t>(2 * l + 16)) cap <<= 1;
    std::vector<i64> key(cap, -1), val(cap);
    auto slot = [&](i64 x) {
      size_t h = static_cast<size_t>((static_cast<std::uint64_t>(x) * 0x9E3779B97F4A7C15ULL) >> 17) & (cap - 1);
      while (key[h] != -1 && key[h] != x) h = (h + 1) & (cap - 1);
      return h;
    };
    auto get = [&](i64 x) {
      const size_t h = slot(x);
      return key[h] == x ? val[h] : x;
    };
    std::vector<i64> out(static_cast<size_t>(l));
    for (i64 i = 0; i < l; ++i) {
      const i64 j = i + static_cast<i64>(rng.index(static_cast<std::uint64_t>(n - i)));
      const i64 vi = get(i), vj = get(j);
      out[static_cast<size_t>(i)] = vj;  // perm[i] <- perm[j]; position i is never read again
      const size_t h = slot(j);
      key[h] = j;
      val[h] = vi;  // perm[j] <- old perm[i]
    }
    return out;
  }
  std::vector<i64> perm(static_cast<size_t>(n));
  std::iota(perm.begin(), perm.end(), i64{0});
  for (i64 i = 0; i < l; ++i) {
    const i64 j = i + static_cast<i64>(rng.index(static_cast<std::uint64_t>(n - i)));
    std::swap(perm[static_cast<size_t>(i)], perm[static_cast<size_t>(j)]);
  }
  perm.resize(static_cast<size_t>(l));
  return perm;
}

// sampling.hpp:66-79
std::vector<std::vector<i64>> partition_columns(i64 n, i64 t, SeededRng& rng) {
  if (t < 1 || t > n) throw std::invalid_argument("partition_columns: need 1 <= t <= n");
  std::vector<i64> perm = sample_without_replacement(n, n, rng);
  const i64 base = n / t, rem = n % t;
  std::vector<std::vector<i64>> groups(static_cast<size_t>(t));
  size_t at = 0;
  for (i64 g = 0; g < t; ++g) {
    const i64 sz = base + (g < rem ? 1 : 0);
    auto& grp = groups[static_cast<size_t>(g)];
    grp.assign(perm.begin() + static_cast<std::ptrdiff_t>(at), perm.begin() + static_cast<std::ptrdiff_t>(at + sz));
    std::sort(grp.begin(), grp.end());
    at += static_cast<size_t>(sz);
  }
  return groups;
}

// ---- D step (sampling.hpp:83-113): parallel stable bucketing of the triplets.
// Every subproblem is a set of columns (extract_columns) or of rows (extract_rows) of the
// observed matrix. One pass tags each entry with its subproblem and new index; chunks of the
// entry array are counted in parallel, prefix-summed per (subproblem, chunk), and scattered in
// parallel — each subproblem's entries keep the input's column-major order, and the column /
// row relabelling is monotone, so every output is already a valid ObservedMatrix (sorted,
// in range, no duplicates: inherited from the validated input) without a re-sort.
// DFCG_DSTEP_THREADS bounds the host threads (default: hardware concurrency, at most 32).
namespace {

int dstep_threads(i64 work) {
  static const int env = std::getenv("DFCG_DSTEP_THREADS") ? std::atoi(std::getenv("DFCG_DSTEP_THREADS")) : 0;
  int t = env > 0 ? env : static_cast<int>(std::min(32u, std::max(1u, std::thread::hardware_concurrency())));
  return static_cast<int>(std::max<i64>(1, std::min<i64>(t, work / (1 << 16) + 1)));
}

template <class Fn>
void run_chunks(int nt, i64 total, Fn&& fn) {  // fn(chunk, begin, end)
  std::vector<std::thread> th;
  for (int c = 1; c < nt; ++c) th.emplace_back([&, c] { fn(c, total * c / nt, total * (c + 1) / nt); });
  fn(0, 0, total / nt);
  for (auto& x : th) x.join();
}

// subproblem definitions -> per-column / per-row (subproblem, new index) tables
struct SubTables {
  std::vector<int> col_sub;   // column -> column subproblem (-1: none)
  std::vector<i64> col_pos;   // column -> index inside it
  int row_sub = -1;           // the (single) row subproblem
  std::vector<i64> row_pos;   // row -> index inside it (-1: not sampled)
};

SubTables make_tables(const HostObs& obs, const std::vector<std::vector<i64>>& col_groups,
                      const std::vector<i64>* rows) {
  SubTables t;
  t.col_sub.assign(static_cast<size_t>(obs.n), -1);
  t.col_pos.assign(static_cast<size_t>(obs.n), -1);
  for (size_t g = 0; g < col_groups.size(); ++g)
    for (size_t p = 0; p < col_groups[g].size(); ++p) {
      const i64 c = col_groups[g][p];
      if (c < 0 || c >= obs.n) throw std::out_of_range("extract_columns: index out of range");
      if (t.col_sub[static_cast<size_t>(c)] >= 0) throw std::invalid_argument("extract_columns: duplicate index");
      t.col_sub[static_cast<size_t>(c)] = static_cast<int>(g);
      t.col_pos[static_cast<size_t>(c)] = static_cast<i64>(p);
    }
  if (rows) {
    t.row_sub = static_cast<int>(col_groups.size());
    t.row_pos.assign(static_cast<size_t>(obs.m), -1);
    for (size_t p = 0; p < rows->size(); ++p) {
      const i64 r = (*rows)[p];
      if (r < 0 || r >= obs.m) throw std::out_of_range("extract_rows: index out of range");
      if (t.row_pos[static_cast<size_t>(r)] >= 0) throw std::invalid_argument("extract_rows: duplicate index");
      t.row_pos[static_cast<size_t>(r)] = static_cast<i64>(p);
    }
  }
  return t;
}

}  // namespace

// Column groups (disjoint, e.g. a partition plan) and optionally one row sample, all in one
// parallel pass. Output order: the column groups, then the row subproblem.
std::vector<HostObs> extract_subproblems(const HostObs& obs, const std::vector<std::vector<i64>>& col_groups,
                                         const std::vector<i64>* rows) {
  const SubTables tb = make_tables(obs, col_groups, rows);
  const size_t G = col_groups.size() + (rows ? 1 : 0);
  const i64 N = obs.count();
  const int nt = dstep_threads(N);
  std::vector<i64> cnt(static_cast<size_t>(nt) * G, 0);  // [chunk][sub]
  run_chunks(nt, N, [&](int c, i64 b, i64 e) {
    i64* k = cnt.data() + static_cast<size_t>(c) * G;
    for (i64 i = b; i < e; ++i) {
      const int g = tb.col_sub[static_cast<size_t>(obs.col[i])];
      if (g >= 0) ++k[g];
      if (tb.row_sub >= 0 && tb.row_pos[static_cast<size_t>(obs.row[i])] >= 0) ++k[tb.row_sub];
    }
  });
  std::vector<HostObs> out(G);
  std::vector<i64> off(static_cast<size_t>(nt) * G);
  for (size_t g = 0; g < G; ++g) {
    i64 at = 0;
    for (int c = 0; c < nt; ++c) {
      off[static_cast<size_t>(c) * G + g] = at;
      at += cnt[static_cast<size_t>(c) * G + g];
    }
    HostObs& o = out[g];
    const bool is_row = tb.row_sub == static_cast<int>(g);
    o.m = is_row ? static_cast<i64>(rows->size()) : obs.m;
    o.n = is_row ? obs.n : static_cast<i64>(col_groups[g].size());
    if (o.m < 1 || o.n < 1) throw std::invalid_argument("ObservedMatrix: dims must be positive");
    o.row.resize(static_cast<size_t>(at));
    o.col.resize(static_cast<size_t>(at));
    o.val.resize(static_cast<size_t>(at));
  }
  run_chunks(nt, N, [&](int c, i64 b, i64 e) {
    i64* w = off.data() + static_cast<size_t>(c) * G;
    for (i64 i = b; i < e; ++i) {
      const size_t col = static_cast<size_t>(obs.col[i]);
      const int g = tb.col_sub[col];
      if (g >= 0) {
        HostObs& o = out[static_cast<size_t>(g)];
        const size_t p = static_cast<size_t>(w[g]++);
        o.row[p] = obs.row[i];
        o.col[p] = tb.col_pos[col];
        o.val[p] = obs.val[i];
      }
      if (tb.row_sub >= 0) {
        const i64 rp = tb.row_pos[static_cast<size_t>(obs.row[i])];
        if (rp >= 0) {
          HostObs& o = out[static_cast<size_t>(tb.row_sub)];
          const size_t p = static_cast<size_t>(w[tb.row_sub]++);
          o.row[p] = rp;
          o.col[p] = obs.col[i];
          o.val[p] = obs.val[i];
        }
      }
    }
  });
  return out;
}

// sampling.hpp:83-97
HostObs extract_columns(const HostObs& obs, const std::vector<i64>& idx) {
  return std::move(extract_subproblems(obs, {idx}, nullptr)[0]);
}

// sampling.hpp:99-113
HostObs extract_rows(const HostObs& obs, const std::vector<i64>& idx) {
  return std::move(extract_subproblems(obs, {}, &idx)[0]);
}

// make_base_solver, dfc.hpp:70-78.
BaseSolver make_base_solver(DeviceContext& ctx, Task task, const ApgConfig& cfg, double lambda) {
  if (task == Task::MC)
    return [&ctx, cfg](const HostObs& b, cudaStream_t s) {
      DevLowRank L;
      SolveReport rep;
      apg_mc_device(ctx, s, b.m, b.n, b.count(), b.row.data(), b.col.data(), b.val.data(), cfg, L, rep, nullptr);
      return std::pair<DevLowRank, SolveReport>{std::move(L), rep};
    };
  return [&ctx, cfg, lambda](const HostObs& b, cudaStream_t s) {
    const double lam = lambda > 0 ? lambda : 1.0 / std::sqrt(static_cast<double>(std::max(b.m, b.n)));
    std::vector<double> dense(static_cast<size_t>(b.m * b.n), 0.0);  // densify (matrix_io.hpp:119-123)
    for (i64 e = 0; e < b.count(); ++e) dense[static_cast<size_t>(b.col[e] * b.m + b.row[e])] = b.val[e];
    DevLowRank L;
    SolveReport rep;
    std::vector<long long> sr, sc;
    std::vector<double> sv;
    apg_rmf_device(ctx, s, dense.data(), b.m, b.n, lam, cfg, L, sr, sc, sv, rep, nullptr);
    return std::pair<DevLowRank, SolveReport>{std::move(L), rep};
  };
}

namespace {

// solve_blocks, dfc.hpp:133-147.
void solve_blocks(DeviceContext& ctx, const std::vector<HostObs>& blocks, const BaseSolver& solver, int workers,
                  std::vector<DevLowRank>& ests, std::vector<SolveReport>& reports) {
  ests.clear();
  ests.resize(blocks.size());
  reports.assign(blocks.size(), SolveReport{});
  parallel_for(ctx, blocks.size(), workers, [&](std::size_t i, cudaStream_t s) {
    if (blocks[i].empty()) {
      ests[i].m = blocks[i].m;
      ests[i].n = blocks[i].n;
      ests[i].k = 0;
      return;
    }
    auto [est, rep] = solver(blocks[i], s);
    ests[i] = std::move(est);
    reports[i] = rep;
  });
}

std::vector<i64> block_ranks(const std::vector<DevLowRank>& ests) {
  std::vector<i64> r;
  for (const auto& e : ests) r.push_back(e.k);
  return r;
}

std::vector<const DevLowRank*> ptrs(const std::vector<DevLowRank>& v) {
  std::vector<const DevLowRank*> p;
  for (const auto& e : v) p.push_back(&e);
  return p;
}

}  // namespace

// pair_deficient, dfc.hpp:272-280: rank(W) < max(rank C-hat, rank R-hat), W = C-hat's left factor
// restricted to the sampled rows (gathered on the device) times its right factor.
bool nys_pair_deficient(cudaStream_t s, const DevLowRank& C, const DevLowRank& R, const std::vector<i64>& row_idx) {
  const i64 kmax = std::max(C.k, R.k);
  if (kmax == 0 || C.k == 0) return kmax > 0;
  const i64 d = static_cast<i64>(row_idx.size());
  DBuf<double> W(d * C.k, s);
  gather_rows(s, C.left.get(), C.k, row_idx, W.get());
  SvdOfProduct f = svd_of_product(s, d, C.n, C.k, W.get(), C.right.get());
  return f.r < kmax;
}

// median_rank, dfc.hpp:159-164.
i64 median_rank(const std::vector<i64>& ranks) {
  if (ranks.empty()) throw std::invalid_argument("median_rank: empty list");
  std::vector<i64> sorted = ranks;
  std::sort(sorted.begin(), sorted.end());
  return std::max<i64>(1, sorted[(sorted.size() - 1) / 2]);
}

// dfc_proj, dfc.hpp:166-200.
std::pair<DevLowRank, DfcReport> dfc_proj(DeviceContext& ctx, const HostObs& obs, const DfcConfig& cfg,
                                          const BaseSolver& solver) {
  if (cfg.variant != DfcVariant::Proj) throw std::invalid_argument("dfc_proj: wrong variant");
  if (cfg.t < 1 || cfg.t > obs.n) throw std::invalid_argument("dfc_proj: need 1 <= t <= n");
  if (cfg.ensemble_anchors < 0) throw std::invalid_argument("dfc_proj: ensemble_anchors must be >= 0");
  if (cfg.ensemble_anchors > 0 && !cfg.ensemble)
    throw std::invalid_argument("dfc_proj: ensemble_anchors needs ensemble = true");
  DfcReport report;
  PhaseClock total, phase;
  SeededRng prng(cfg.seed, streams::partition);
  auto plan = partition_columns(obs.n, cfg.t, prng);
  std::vector<HostObs> blocks = extract_subproblems(obs, plan, nullptr);
  report.divide_ms = phase.lap();
  std::vector<DevLowRank> ests;
  solve_blocks(ctx, blocks, solver, cfg.workers, ests, report.subproblems);
  report.factor_ms = phase.lap();
  DevLowRank out;
  out.m = obs.m;
  out.n = obs.n;
  const auto bl = ptrs(ests);
  if (!cfg.ensemble) {
    CallStream cs(ctx);
    column_project(cs.s, ests[0], bl, plan, obs.n, out);
  } else {
    // every block projected onto each anchor's column space (all t blocks in the reference;
    // the first ensemble_anchors plan groups when that knob is set)
    const std::size_t anchors = cfg.ensemble_anchors > 0
                                    ? std::min<std::size_t>(static_cast<std::size_t>(cfg.ensemble_anchors), ests.size())
                                    : ests.size();
    std::vector<DevLowRank> projected(anchors);
    parallel_for(ctx, anchors, cfg.workers,
                 [&](std::size_t i, cudaStream_t s) { column_project(s, ests[i], bl, plan, obs.n, projected[i]); });
    CallStream cs(ctx);
    average_estimates(cs.s, ptrs(projected), median_rank(block_ranks(ests)), out);
  }
  report.combine_ms = phase.lap();
  report.total_ms = total.lap();
  return {std::move(out), std::move(report)};
}

// dfc_rp, dfc.hpp:202-248.
std::pair<DevLowRank, DfcReport> dfc_rp(DeviceContext& ctx, const HostObs& obs, const DfcConfig& cfg,
                                        const BaseSolver& solver) {
  if (cfg.variant != DfcVariant::Rp) throw std::invalid_argument("dfc_rp: wrong variant");
  if (cfg.t < 1 || cfg.t > obs.n) throw std::invalid_argument("dfc_rp: need 1 <= t <= n");
  DfcReport report;
  PhaseClock total, phase;
  SeededRng prng(cfg.seed, streams::partition);
  auto plan = partition_columns(obs.n, cfg.t, prng);
  std::vector<HostObs> blocks = extract_subproblems(obs, plan, nullptr);
  report.divide_ms = phase.lap();
  std::vector<DevLowRank> ests;
  solve_blocks(ctx, blocks, solver, cfg.workers, ests, report.subproblems);
  report.factor_ms = phase.lap();
  i64 k = median_rank(block_ranks(ests)), p = cfg.rp_p;
  const i64 minmn = std::min(obs.m, obs.n);
  if (k + p > minmn) {
    report.k_clamped = true;
    p = std::min(p, minmn - 1);
    k = minmn - p;
  }
  report.chosen_k = k;
  DevLowRank out;
  const auto bl = ptrs(ests);
  if (!cfg.ensemble) {
    SeededRng rng(cfg.seed, streams::rp_draw);
    CallStream cs(ctx);
    random_project(cs.s, bl, plan, obs.n, k, p, cfg.rp_q, rng, out);
  } else {
    std::vector<DevLowRank> draws(static_cast<size_t>(cfg.t));
    parallel_for(ctx, draws.size(), cfg.workers, [&](std::size_t i, cudaStream_t s) {
      SeededRng rng(cfg.seed, streams::rp_draw + 1 + i);
      random_project(s, bl, plan, obs.n, k, p, cfg.rp_q, rng, draws[i]);
    });
    CallStream cs(ctx);
    average_estimates(cs.s, ptrs(draws), k, out);
  }
  report.combine_ms = phase.lap();
  report.total_ms = total.lap();
  return {std::move(out), std::move(report)};
}

// dfc_nys, dfc.hpp:250-324.
std::pair<DevLowRank, DfcReport> dfc_nys(DeviceContext& ctx, const HostObs& obs, const DfcConfig& cfg,
                                         const BaseSolver& solver) {
  if (cfg.variant != DfcVariant::Nys) throw std::invalid_argument("dfc_nys: wrong variant");
  const i64 m = obs.m, n = obs.n;
  if (cfg.l < 1 || cfg.l > n) throw std::invalid_argument("dfc_nys: need 1 <= l <= n");
  if (cfg.d < 1 || cfg.d > m) throw std::invalid_argument("dfc_nys: need 1 <= d <= m");
  DfcReport report;
  PhaseClock total, phase;
  SeededRng row_rng(cfg.seed, streams::nys_rows);
  std::vector<i64> row_idx = sample_without_replacement(m, cfg.d, row_rng);
  std::sort(row_idx.begin(), row_idx.end());
  auto pair_deficient = [&](cudaStream_t s, const DevLowRank& C, const DevLowRank& R) {
    return nys_pair_deficient(s, C, R, row_idx);
  };
  if (!cfg.ensemble) {
    SeededRng col_rng(cfg.seed, streams::nys_cols);
    std::vector<i64> col_idx = sample_without_replacement(n, cfg.l, col_rng);
    std::sort(col_idx.begin(), col_idx.end());
    std::vector<HostObs> blocks = extract_subproblems(obs, {col_idx}, &row_idx);
    report.divide_ms = phase.lap();
    std::vector<DevLowRank> ests;
    solve_blocks(ctx, blocks, solver, cfg.workers, ests, report.subproblems);
    report.factor_ms = phase.lap();
    DevLowRank out;
    {
      CallStream cs(ctx);
      report.rank_deficient = pair_deficient(cs.s, ests[0], ests[1]);
      gen_nystrom(cs.s, ests[0], ests[1], row_idx, col_idx, out);
    }
    report.combine_ms = phase.lap();
    report.total_ms = total.lap();
    return {std::move(out), std::move(report)};
  }
  const i64 groups =
      std::clamp<i64>(static_cast<i64>(std::llround(static_cast<double>(n) / static_cast<double>(cfg.l))), 1, n);
  SeededRng prng(cfg.seed, streams::partition);
  auto plan = partition_columns(n, groups, prng);
  std::vector<HostObs> blocks = extract_subproblems(obs, plan, &row_idx);
  report.divide_ms = phase.lap();
  std::vector<DevLowRank> ests;
  solve_blocks(ctx, blocks, solver, cfg.workers, ests, report.subproblems);
  report.factor_ms = phase.lap();
  const DevLowRank& R_hat = ests.back();
  const size_t nc = ests.size() - 1;
  std::vector<DevLowRank> combined(nc);
  std::vector<char> deficient(nc, 0);
  parallel_for(ctx, nc, cfg.workers, [&](std::size_t i, cudaStream_t s) {
    deficient[i] = pair_deficient(s, ests[i], R_hat) ? 1 : 0;
    gen_nystrom(s, ests[i], R_hat, row_idx, plan[i], combined[i]);
  });
  for (char f : deficient) report.rank_deficient = report.rank_deficient || f;
  std::vector<i64> col_ranks;
  for (size_t i = 0; i < nc; ++i) col_ranks.push_back(ests[i].k);
  DevLowRank out;
  {
    CallStream cs(ctx);
    average_estimates(cs.s, ptrs(combined), median_rank(col_ranks), out);
  }
  report.combine_ms = phase.lap();
  report.total_ms = total.lap();
  return {std::move(out), std::move(report)};
}

// dfc_run, dfc.hpp:326-335.
std::pair<DevLowRank, DfcReport> dfc_run(DeviceContext& ctx, const HostObs& obs, const DfcConfig& cfg) {
  if (cfg.ensemble_anchors != 0 && cfg.variant != DfcVariant::Proj)
    throw std::invalid_argument("dfc_run: ensemble_anchors applies to DFC-Proj-Ens only");
  const BaseSolver solver = make_base_solver(ctx, cfg.task, cfg.solver_cfg, cfg.lambda);
  switch (cfg.variant) {
    case DfcVariant::Proj: return dfc_proj(ctx, obs, cfg, solver);
    case DfcVariant::Rp: return dfc_rp(ctx, obs, cfg, solver);
    case DfcVariant::Nys: return dfc_nys(ctx, obs, cfg, solver);
  }
  throw std::logic_error("dfc_run: unknown variant");
}

}  // namespace dfcg
