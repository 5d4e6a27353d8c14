// TEST INFRASTRUCTURE ONLY — C ABI of the CPU oracle, loaded by tests/ and bench.py
// (cpu_baseline and --impl reference) through oracle/__init__.py.
#include <cstring>
#include <string>

#include "dfc_oracle.hpp"

using orc::Index;

namespace {
thread_local std::string g_err;
thread_local long long g_err_block = -1;

enum : int { kOk = 0, kInvalid = -1, kRange = -2, kBlock = -3, kRuntime = -4 };

template <class F>
int guard(F&& f) {
  try {
    f();
    return kOk;
  } catch (const orc::BlockError& e) {
    g_err = e.what();
    g_err_block = static_cast<long long>(e.block);
    return kBlock;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return kInvalid;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return kRange;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kRuntime;
  }
}

orc::Mat from_colmajor(Index r, Index c, const double* p) {
  orc::Mat M(r, c);
  if (r > 0 && c > 0) std::memcpy(M.d.data(), p, sizeof(double) * static_cast<std::size_t>(r * c));
  return M;
}
}  // namespace

struct OrcObs {
  orc::ObservedMatrix obs;
};
struct OrcEst {
  orc::LowRankEstimate est;
};
struct OrcTrip {
  std::vector<orc::Observation> e;
};

extern "C" {

struct OrcApgCfg {
  int max_iters;
  double rel_tol;
  int has_mu_init;
  double mu_init;
  int has_mu_floor;
  double mu_floor;
  double mu_decay;
  int line_search;
};
struct OrcReport {
  int iterations;
  double objective, residual;
  long long rank;
  double wall_ms;
};
struct OrcTrace {
  int it;
  long long rank, k_final;
  int svd_calls;
  double rel, mu, sigma_sum;
};
struct OrcDfcCfg {
  int variant, ensemble;
  long long t, l, d, rp_k, rp_p, rp_q;
  unsigned long long seed;
  OrcApgCfg solver;
  int task;
  double lambda;
  int workers;
  long long ensemble_anchors;
};
struct OrcDfcReport {
  double divide_ms, factor_ms, combine_ms, total_ms;
  long long chosen_k;
  int k_clamped, rank_deficient;
  long long nsub;
};

const char* orc_last_error() { return g_err.c_str(); }
long long orc_last_error_block() { return g_err_block; }

// ---------------------------------------------------------------- RNG / sampling
void orc_rng_u64(unsigned long long seed, unsigned long long stream, long long n, unsigned long long* out) {
  orc::SeededRng r(seed, stream);
  for (long long i = 0; i < n; ++i) out[i] = r.next_u64();
}
void orc_rng_uniform(unsigned long long seed, unsigned long long stream, long long n, double* out) {
  orc::SeededRng r(seed, stream);
  for (long long i = 0; i < n; ++i) out[i] = r.uniform();
}
void orc_rng_uniform_pos(unsigned long long seed, unsigned long long stream, long long n, double* out) {
  orc::SeededRng r(seed, stream);
  for (long long i = 0; i < n; ++i) out[i] = r.uniform_pos();
}
void orc_rng_normal(unsigned long long seed, unsigned long long stream, long long n, double* out) {
  orc::SeededRng r(seed, stream);
  for (long long i = 0; i < n; ++i) out[i] = r.normal();
}
int orc_rng_index(unsigned long long seed, unsigned long long stream, long long count, unsigned long long bound,
                  unsigned long long* out) {
  return guard([&] {
    orc::SeededRng r(seed, stream);
    for (long long i = 0; i < count; ++i) out[i] = r.index(bound);
  });
}
int orc_sample_without_replacement(unsigned long long seed, unsigned long long stream, long long n, long long l,
                                   long long* out) {
  return guard([&] {
    orc::SeededRng r(seed, stream);
    auto v = orc::sample_without_replacement(n, l, r);
    for (std::size_t i = 0; i < v.size(); ++i) out[i] = v[i];
  });
}
int orc_partition_columns(unsigned long long seed, unsigned long long stream, long long n, long long t,
                          long long* cols, long long* offsets) {
  return guard([&] {
    orc::SeededRng r(seed, stream);
    orc::PartitionPlan plan = orc::partition_columns(n, t, r);
    long long at = 0;
    offsets[0] = 0;
    for (std::size_t g = 0; g < plan.group_count(); ++g) {
      for (Index c : plan.group(g)) cols[at++] = c;
      offsets[g + 1] = at;
    }
  });
}

// ---------------------------------------------------------------- handles
int orc_obs_new(long long m, long long n, long long nnz, const long long* rows, const long long* cols,
                const double* vals, OrcObs** out) {
  return guard([&] {
    std::vector<orc::Observation> v(static_cast<std::size_t>(nnz));
    for (long long i = 0; i < nnz; ++i) v[static_cast<std::size_t>(i)] = {rows[i], cols[i], vals[i]};
    *out = new OrcObs{orc::ObservedMatrix(m, n, std::move(v))};
  });
}
void orc_obs_free(OrcObs* o) { delete o; }
void orc_obs_dims(const OrcObs* o, long long* m, long long* n, long long* nnz) {
  *m = o->obs.rows();
  *n = o->obs.cols();
  *nnz = o->obs.count();
}
void orc_obs_get(const OrcObs* o, long long* rows, long long* cols, double* vals) {
  std::size_t i = 0;
  for (const auto& e : o->obs.entries()) {
    rows[i] = e.row;
    cols[i] = e.col;
    vals[i] = e.value;
    ++i;
  }
}
int orc_extract_columns(const OrcObs* o, long long count, const long long* idx, OrcObs** out) {
  return guard([&] { *out = new OrcObs{orc::extract_columns(o->obs, std::vector<Index>(idx, idx + count))}; });
}
int orc_extract_rows(const OrcObs* o, long long count, const long long* idx, OrcObs** out) {
  return guard([&] { *out = new OrcObs{orc::extract_rows(o->obs, std::vector<Index>(idx, idx + count))}; });
}

int orc_est_new(long long m, long long n, long long k, const double* left, const double* right, OrcEst** out) {
  return guard([&] { *out = new OrcEst{orc::LowRankEstimate(from_colmajor(m, k, left), from_colmajor(n, k, right))}; });
}
void orc_est_free(OrcEst* e) { delete e; }
void orc_est_dims(const OrcEst* e, long long* m, long long* n, long long* k) {
  *m = e->est.rows();
  *n = e->est.cols();
  *k = e->est.rank_bound();
}
void orc_est_get(const OrcEst* e, double* left, double* right) {
  std::memcpy(left, e->est.left().d.data(), sizeof(double) * e->est.left().d.size());
  std::memcpy(right, e->est.right().d.data(), sizeof(double) * e->est.right().d.size());
}

void orc_trip_free(OrcTrip* t) { delete t; }
long long orc_trip_count(const OrcTrip* t) { return static_cast<long long>(t->e.size()); }
void orc_trip_get(const OrcTrip* t, long long* rows, long long* cols, double* vals) {
  for (std::size_t i = 0; i < t->e.size(); ++i) {
    rows[i] = t->e[i].row;
    cols[i] = t->e[i].col;
    vals[i] = t->e[i].value;
  }
}

// ---------------------------------------------------------------- generators
int orc_gen_low_rank(long long m, long long n, long long r, unsigned long long seed, unsigned long long stream,
                     OrcEst** L0) {
  return guard([&] {
    orc::SeededRng rng(seed, stream);
    *L0 = new OrcEst{orc::gen_low_rank(m, n, r, rng)};
  });
}
int orc_gen_mc(long long m, long long n, long long r, long long s, double sigma, unsigned long long seed,
               unsigned long long stream, OrcEst** L0, OrcObs** obs) {
  return guard([&] {
    orc::SeededRng rng(seed, stream);
    orc::McInstance inst = orc::gen_mc_instance(m, n, r, s, sigma, rng);
    *L0 = new OrcEst{std::move(inst.L0)};
    *obs = new OrcObs{std::move(inst.obs)};
  });
}
int orc_gen_rmf(long long m, long long n, long long r, long long s, double sigma, unsigned long long seed,
                unsigned long long stream, double lo, double hi, OrcEst** L0, OrcTrip** S0, double* M) {
  return guard([&] {
    orc::SeededRng rng(seed, stream);
    orc::RmfInstance inst = orc::gen_rmf_instance(m, n, r, s, sigma, rng, lo, hi);
    *L0 = new OrcEst{std::move(inst.L0)};
    *S0 = new OrcTrip{std::move(inst.S0.entries)};
    std::memcpy(M, inst.M.d.data(), sizeof(double) * inst.M.d.size());
  });
}

// ---------------------------------------------------------------- solvers
static orc::ApgConfig to_cfg(const OrcApgCfg* c) {
  orc::ApgConfig cfg;
  if (!c) return cfg;
  cfg.max_iters = c->max_iters;
  cfg.rel_tol = c->rel_tol;
  if (c->has_mu_init) cfg.mu_init = c->mu_init;
  if (c->has_mu_floor) cfg.mu_floor = c->mu_floor;
  cfg.mu_decay = c->mu_decay;
  cfg.line_search = c->line_search != 0;
  return cfg;
}
static void to_report(const orc::SolveReport& r, OrcReport* o) {
  if (!o) return;
  o->iterations = r.iterations;
  o->objective = r.objective;
  o->residual = r.residual;
  o->rank = r.rank;
  o->wall_ms = r.wall_ms;
}
static void to_trace(const std::vector<orc::IterTrace>& tr, OrcTrace* out, long long cap, long long* len) {
  if (len) *len = static_cast<long long>(tr.size());
  if (!out) return;
  for (std::size_t i = 0; i < tr.size() && static_cast<long long>(i) < cap; ++i)
    out[i] = {tr[i].it, tr[i].rank, tr[i].k_final, tr[i].svd_calls, tr[i].rel, tr[i].mu, tr[i].sigma_sum};
}

int orc_apg_mc(const OrcObs* obs, const OrcApgCfg* c, OrcEst** out, OrcReport* rep, OrcTrace* trace, long long cap,
               long long* len) {
  return guard([&] {
    std::vector<orc::IterTrace> tr;
    auto [L, r] = orc::apg_mc(obs->obs, to_cfg(c), &tr);
    *out = new OrcEst{std::move(L)};
    to_report(r, rep);
    to_trace(tr, trace, cap, len);
  });
}

// Resumable APG-MC run (bench windows): create, step n iterations, finish, free.
int orc_mc_run_new(const OrcObs* obs, const OrcApgCfg* c, orc::ApgMcRun** out) {
  return guard([&] { *out = new orc::ApgMcRun(obs->obs, to_cfg(c)); });
}
int orc_mc_run_step(orc::ApgMcRun* r, long long n, long long* done) {
  return guard([&] {
    long long k = 0;
    while (k < n && r->step()) ++k;
    *done = k;
  });
}
// Same, with the per-iteration trace of the stepped iterations (fixture generation).
int orc_mc_run_step_trace(orc::ApgMcRun* r, long long n, long long* done, OrcTrace* trace, long long cap,
                          long long* len) {
  return guard([&] {
    std::vector<orc::IterTrace> tr;
    long long k = 0;
    while (k < n && r->step(&tr)) ++k;
    *done = k;
    to_trace(tr, trace, cap, len);
  });
}
int orc_mc_run_finish(orc::ApgMcRun* r, OrcEst** out, OrcReport* rep) {
  return guard([&] {
    auto [L, rp] = r->finish();
    *out = new OrcEst{std::move(L)};
    to_report(rp, rep);
  });
}
void orc_mc_run_free(orc::ApgMcRun* r) { delete r; }

int orc_apg_rmf(long long m, long long n, const double* M, double lambda, const OrcApgCfg* c, OrcEst** L, OrcTrip** S,
                OrcReport* rep, OrcTrace* trace, long long cap, long long* len) {
  return guard([&] {
    std::vector<orc::IterTrace> tr;
    auto [Lh, Sh, r] = orc::apg_rmf(from_colmajor(m, n, M), lambda, to_cfg(c), &tr);
    *L = new OrcEst{std::move(Lh)};
    *S = new OrcTrip{std::move(Sh.entries)};
    to_report(r, rep);
    to_trace(tr, trace, cap, len);
  });
}

int orc_svt(long long m, long long n, const double* A, double tau, OrcEst** out) {
  return guard([&] { *out = new OrcEst{orc::svt(from_colmajor(m, n, A), tau)}; });
}
int orc_soft_threshold(long long m, long long n, const double* A, double tau, double* out) {
  return guard([&] {
    orc::Mat r = orc::soft_threshold(from_colmajor(m, n, A), tau);
    std::memcpy(out, r.d.data(), sizeof(double) * r.d.size());
  });
}
int orc_compact_svd(long long m, long long n, const double* A, OrcEst** out) {
  return guard([&] { *out = new OrcEst{orc::compact_svd(from_colmajor(m, n, A)).to_estimate()}; });
}
double orc_factored_diff_norm(const OrcEst* a, const OrcEst* b) { return orc::factored_diff_norm(a->est, b->est); }
double orc_default_rmf_lambda(long long m, long long n) { return orc::default_rmf_lambda(m, n); }

// ---------------------------------------------------------------- combiners
static orc::PartitionPlan make_plan(long long t, const long long* offsets, const long long* cols, long long n) {
  std::vector<std::vector<Index>> g(static_cast<std::size_t>(t));
  for (long long i = 0; i < t; ++i) g[static_cast<std::size_t>(i)].assign(cols + offsets[i], cols + offsets[i + 1]);
  return orc::PartitionPlan(n, std::move(g));
}
static std::vector<orc::LowRankEstimate> gather(long long t, const OrcEst* const* ests) {
  std::vector<orc::LowRankEstimate> v;
  for (long long i = 0; i < t; ++i) v.push_back(ests[i]->est);
  return v;
}

int orc_column_project(const OrcEst* basis, long long t, const OrcEst* const* blocks, const long long* offsets,
                       const long long* cols, long long n, OrcEst** out) {
  return guard([&] {
    orc::PartitionPlan plan = make_plan(t, offsets, cols, n);
    *out = new OrcEst{orc::column_project(basis->est, gather(t, blocks), plan)};
  });
}
int orc_random_project(long long t, const OrcEst* const* blocks, const long long* offsets, const long long* cols,
                       long long n, long long k, long long p, long long q, unsigned long long seed,
                       unsigned long long stream, OrcEst** out) {
  return guard([&] {
    orc::PartitionPlan plan = make_plan(t, offsets, cols, n);
    orc::SeededRng rng(seed, stream);
    *out = new OrcEst{orc::random_project(gather(t, blocks), plan, orc::RpParams{k, p, q}, rng)};
  });
}
int orc_gen_nystrom(const OrcEst* C, const OrcEst* R, long long d, const long long* rows, long long l,
                    const long long* cols, OrcEst** out) {
  return guard([&] {
    *out = new OrcEst{orc::gen_nystrom(C->est, R->est, std::vector<Index>(rows, rows + d),
                                       std::vector<Index>(cols, cols + l))};
  });
}
int orc_average_estimates(long long count, const OrcEst* const* ests, long long recompress_to, OrcEst** out) {
  return guard([&] {
    std::optional<Index> rc;
    if (recompress_to >= 0) rc = recompress_to;
    *out = new OrcEst{orc::average_estimates(gather(count, ests), rc)};
  });
}

// ---------------------------------------------------------------- orchestrator
int orc_dfc_run(const OrcObs* obs, const OrcDfcCfg* c, OrcEst** out, OrcDfcReport* rep, OrcReport* subs,
                long long sub_cap) {
  return guard([&] {
    orc::DfcConfig cfg;
    cfg.variant = static_cast<orc::DfcVariant>(c->variant);
    cfg.ensemble = c->ensemble != 0;
    cfg.t = c->t;
    cfg.l = c->l;
    cfg.d = c->d;
    cfg.rp = orc::RpParams{c->rp_k, c->rp_p, c->rp_q};
    cfg.seed = c->seed;
    cfg.solver_cfg = to_cfg(&c->solver);
    cfg.task = static_cast<orc::Task>(c->task);
    cfg.lambda = c->lambda;
    cfg.workers = c->workers;
    cfg.ensemble_anchors = c->ensemble_anchors;
    if (cfg.ensemble_anchors != 0 && cfg.variant != orc::DfcVariant::Proj)
      throw std::invalid_argument("dfc_run: ensemble_anchors applies to DFC-Proj-Ens only");
    auto [L, r] = orc::dfc_run(obs->obs, cfg);
    *out = new OrcEst{std::move(L)};
    rep->divide_ms = r.divide_ms;
    rep->factor_ms = r.factor_ms;
    rep->combine_ms = r.combine_ms;
    rep->total_ms = r.total_ms;
    rep->chosen_k = r.chosen_k;
    rep->k_clamped = r.k_clamped;
    rep->rank_deficient = r.rank_deficient;
    rep->nsub = static_cast<long long>(r.subproblems.size());
    for (std::size_t i = 0; i < r.subproblems.size() && static_cast<long long>(i) < sub_cap; ++i)
      to_report(r.subproblems[i], subs + i);
  });
}

}  // extern "C"

extern "C" void scipy_openblas_set_num_threads64_(int);
extern "C" void orc_set_blas_threads(int n) { scipy_openblas_set_num_threads64_(n); }
