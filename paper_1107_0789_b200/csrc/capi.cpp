// C ABI (include/dfcg.h): argument validation, host<->device layout conversion, exception ->
// error-code mapping. Everything below this file is C++/CUDA; nothing here computes.
#include "../../include/dfcg.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <new>
#include <string>

#include "dfc_host.hpp"
#include "triplet_io.hpp"
#include "dist.hpp"

using namespace dfcg;

struct dfcg_ctx {
  DeviceContext* dev;
};

struct dfcg_comm {
  std::unique_ptr<Comm> comm;
};

struct dfcg_mc_solver {
  DeviceContext* dev;
  cudaStream_t s;
  std::unique_ptr<McSolver> solver;
};

namespace {

thread_local std::string g_err;
thread_local int64_t g_err_block = -1;
thread_local int64_t g_err_line = -1;

template <class F>
int guard(F&& f) {
  g_err.clear();
  g_err_block = -1;
  g_err_line = -1;
  try {
    f();
    return DFCG_OK;
  } catch (const ParseError& e) {
    g_err = e.what();
    g_err_line = static_cast<int64_t>(e.line);
    return DFCG_EPARSE;
  } catch (const BlockError& e) {
    // the inner message: a caller rethrowing BlockError(dfcg_last_error_block(), msg) adds the
    // "block N: " prefix itself (P/include/dfc/dfc.hpp:50-54), exactly once
    g_err = e.inner;
    g_err_block = static_cast<int64_t>(e.block);
    return DFCG_EBLOCK;
  } catch (const CudaError& e) {
    g_err = e.what();
    return DFCG_ECUDA;
  } catch (const NcclError& e) {
    g_err = e.what();
    return DFCG_ENCCL;
  } catch (const std::bad_alloc& e) {
    g_err = "out of host memory";
    return DFCG_ENOMEM;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return DFCG_EINVAL;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return DFCG_ERANGE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DFCG_EINTERNAL;
  }
}

ApgConfig to_cfg(const dfcg_apg_cfg* c) {
  ApgConfig cfg;
  if (!c) return cfg;
  cfg.max_iters = c->max_iters;
  cfg.rel_tol = c->rel_tol;
  if (c->has_mu_init) cfg.mu_init = c->mu_init;
  if (c->has_mu_floor) cfg.mu_floor = c->mu_floor;
  cfg.mu_decay = c->mu_decay;
  cfg.line_search = c->line_search != 0;
  return cfg;
}

void to_report(const SolveReport& r, dfcg_solve_report* o) {
  if (!o) return;
  o->iterations = r.iterations;
  o->objective = r.objective;
  o->residual = r.residual;
  o->rank = r.rank;
  o->wall_ms = r.wall_ms;
}

void to_trace(const std::vector<IterTrace>& tr, dfcg_iter_trace* out, int64_t cap, int64_t* len) {
  if (len) *len = static_cast<int64_t>(tr.size());
  if (!out) return;
  for (size_t i = 0; i < tr.size() && static_cast<int64_t>(i) < cap; ++i)
    out[i] = {tr[i].it, tr[i].rank, tr[i].k_final, tr[i].svd_calls, tr[i].rel, tr[i].mu, tr[i].sigma_sum, tr[i].ms};
}

double* dup_array(const std::vector<double>& v) {
  double* p = static_cast<double*>(std::malloc(sizeof(double) * std::max<size_t>(1, v.size())));
  if (!p) throw std::bad_alloc();
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(double) * v.size());
  return p;
}

// Device estimate -> caller-owned (malloc) column-major factors: transposed on the device,
// copied straight into the output arrays (no intermediate host copies).
void to_c(cudaStream_t s, const DevLowRank& d, dfcg_lowrank* out) {
  out->m = d.m;
  out->n = d.n;
  out->k = d.k;
  const size_t nl = static_cast<size_t>(d.m * d.k), nr = static_cast<size_t>(d.n * d.k);
  out->left = static_cast<double*>(std::malloc(sizeof(double) * std::max<size_t>(1, nl)));
  out->right = static_cast<double*>(std::malloc(sizeof(double) * std::max<size_t>(1, nr)));
  if (!out->left || !out->right) {
    std::free(out->left);
    std::free(out->right);
    out->left = out->right = nullptr;
    throw std::bad_alloc();
  }
  if (d.k == 0) return;
  DBuf<double> tl(d.m * d.k, s), tr(d.n * d.k, s);
  transpose(s, d.m, d.k, d.left.get(), d.k, tl.get(), d.m);
  transpose(s, d.n, d.k, d.right.get(), d.k, tr.get(), d.n);
  DFCG_CUDA(cudaMemcpyAsync(out->left, tl.get(), sizeof(double) * nl, cudaMemcpyDeviceToHost, s));
  DFCG_CUDA(cudaMemcpyAsync(out->right, tr.get(), sizeof(double) * nr, cudaMemcpyDeviceToHost, s));
  DFCG_CUDA(cudaStreamSynchronize(s));
}

// Caller's column-major estimate -> device (row-major): validated in place (LowRankEstimate
// ctor, matrix_io.hpp:73-84), uploaded straight from the caller's arrays.
DevLowRank to_dev(cudaStream_t s, const dfcg_lowrank* e) {
  if (!e) throw std::invalid_argument("LowRankEstimate: null estimate");
  if (e->m < 1 || e->n < 1) throw std::invalid_argument("LowRankEstimate: dims must be positive");
  if (e->k < 0 || e->k > std::min(e->m, e->n)) throw std::invalid_argument("LowRankEstimate: k exceeds min(m, n)");
  const i64 nl = e->m * e->k, nr = e->n * e->k;
  for (i64 i = 0; i < nl; ++i)
    if (!std::isfinite(e->left[i])) throw std::invalid_argument("LowRankEstimate: non-finite factor entry");
  for (i64 i = 0; i < nr; ++i)
    if (!std::isfinite(e->right[i])) throw std::invalid_argument("LowRankEstimate: non-finite factor entry");
  DevLowRank d;
  d.m = e->m;
  d.n = e->n;
  d.k = e->k;
  if (e->k == 0) return d;
  DBuf<double> tl(nl, s), tr(nr, s);
  d.left.alloc(nl, s);
  d.right.alloc(nr, s);
  DFCG_CUDA(cudaMemcpyAsync(tl.get(), e->left, sizeof(double) * nl, cudaMemcpyHostToDevice, s));
  DFCG_CUDA(cudaMemcpyAsync(tr.get(), e->right, sizeof(double) * nr, cudaMemcpyHostToDevice, s));
  transpose(s, e->k, e->m, tl.get(), e->m, d.left.get(), e->k);  // column-major m x k == row-major k x m
  transpose(s, e->k, e->n, tr.get(), e->n, d.right.get(), e->k);
  DFCG_CUDA(cudaStreamSynchronize(s));
  return d;
}

std::vector<std::vector<i64>> groups_from(int64_t t, const int64_t* offsets, const int64_t* cols, int64_t n) {
  if (t < 0) throw std::invalid_argument("partition: negative group count");
  std::vector<std::vector<i64>> g(static_cast<size_t>(t));
  std::vector<char> seen(static_cast<size_t>(std::max<int64_t>(n, 0)), 0);
  size_t total = 0, min_sz = static_cast<size_t>(std::max<int64_t>(n, 0)), max_sz = 0;
  for (int64_t i = 0; i < t; ++i) {
    g[static_cast<size_t>(i)].assign(cols + offsets[i], cols + offsets[i + 1]);
    const auto& grp = g[static_cast<size_t>(i)];
    min_sz = std::min(min_sz, grp.size());
    max_sz = std::max(max_sz, grp.size());
    for (size_t p = 0; p < grp.size(); ++p) {  // PartitionPlan ctor checks (sampling.hpp:32-51)
      const i64 c = grp[p];
      if (c < 0 || c >= n) throw std::out_of_range("PartitionPlan: column out of range");
      if (seen[static_cast<size_t>(c)]++) throw std::invalid_argument("PartitionPlan: overlapping groups");
      if (p > 0 && grp[p - 1] >= c) throw std::invalid_argument("PartitionPlan: group not sorted");
      ++total;
    }
  }
  if (total != static_cast<size_t>(n)) throw std::invalid_argument("PartitionPlan: groups do not cover all columns");
  if (t > 0 && max_sz > min_sz + 1) throw std::invalid_argument("PartitionPlan: group sizes differ by more than 1");
  return g;
}

}  // namespace

// Shared error channel for the host utilities in hostgen.cpp.
int dfcg_guard_call(const std::function<void()>& f) { return guard(f); }

extern "C" {

int dfcg_ctx_create(int device, dfcg_ctx** out) {
  return guard([&] {
    int n = 0;
    DFCG_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw std::invalid_argument("dfcg_ctx_create: no such CUDA device");
    auto* c = new dfcg_ctx{new DeviceContext(device)};
    *out = c;
  });
}

int dfcg_normals_fetch(dfcg_ctx* ctx, int stream_id, int64_t pos, int64_t n, double* out) {
  return guard([&] {
    if (!ctx || !out || pos < 0 || n < 0 || (stream_id != 0 && stream_id != 1))
      throw std::invalid_argument("dfcg_normals_fetch: bad argument");
    CallStream cs(*ctx->dev);
    DBuf<double> d(n, cs.s);
    ctx->dev->normals(stream_id).fetch(pos, n, d.get(), cs.s);
    DFCG_CUDA(cudaMemcpyAsync(out, d.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, cs.s));
    DFCG_CUDA(cudaStreamSynchronize(cs.s));
  });
}

// Diagnostics: the per-iteration sparse kernels on one observed set, CUDA-event timed.
int dfcg_bench_sparse(dfcg_ctx* ctx, const dfcg_obs* in, int64_t b, int64_t kY, int32_t reps, int32_t spmm_mode,
                      int32_t sddmm_mode, double* ms3, double* sum3) {
  return guard([&] {
    if (!ctx || !in || !ms3 || !sum3 || b < 1 || kY < 1 || reps < 1)
      throw std::invalid_argument("dfcg_bench_sparse: bad argument");
    HostObs obs = HostObs::make(in->m, in->n, std::vector<long long>(in->row, in->row + in->nnz),
                                std::vector<long long>(in->col, in->col + in->nnz),
                                std::vector<double>(in->val, in->val + in->nnz));
    CallStream cs(*ctx->dev);
    const cudaStream_t s = cs.s;
    DevOmega om;
    om.build(s, obs.m, obs.n, obs.count(), obs.row.data(), obs.col.data(), obs.val.data());
    auto fill = [&](i64 count, std::uint64_t seed) {
      std::vector<double> h(static_cast<size_t>(count));
      std::uint64_t x = seed;
      for (auto& v : h) {
        x = x * 6364136223846793005ULL + 1442695040888963407ULL;
        v = static_cast<double>(x >> 11) * (1.0 / 9007199254740992.0) - 0.5;
      }
      DBuf<double> d(count, s);
      DFCG_CUDA(cudaMemcpyAsync(d.get(), h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, s));
      DFCG_CUDA(cudaStreamSynchronize(s));
      return d;
    };
    // DFCG_BENCH_LDX: leading dimension of the gathered sketches (default b: packed rows)
    const i64 ldx = std::getenv("DFCG_BENCH_LDX") ? std::max<i64>(b, std::atoll(std::getenv("DFCG_BENCH_LDX"))) : b;
    DBuf<double> X = fill(obs.n * ldx, 1), Q = fill(obs.m * ldx, 2), Yl = fill(obs.m * kY, 3), Yr = fill(obs.n * kY, 4);
    DBuf<double> outm(obs.m * b, s), outn(obs.n * b, s), r(std::max<i64>(1, obs.count()), s);
    set_sparse_modes(spmm_mode, sddmm_mode);
    cudaEvent_t e0, e1;
    DFCG_CUDA(cudaEventCreate(&e0));
    DFCG_CUDA(cudaEventCreate(&e1));
    auto timed = [&](auto&& fn) {
      fn();  // warm-up (and the one-time attribute opt-ins)
      DFCG_CUDA(cudaEventRecord(e0, s));
      for (int i = 0; i < reps; ++i) fn();
      DFCG_CUDA(cudaEventRecord(e1, s));
      DFCG_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      DFCG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      return static_cast<double>(ms) / reps;
    };
    auto total = [&](const DBuf<double>& d, i64 count) {
      std::vector<double> h(static_cast<size_t>(count));
      DFCG_CUDA(cudaMemcpyAsync(h.data(), d.get(), sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s));
      DFCG_CUDA(cudaStreamSynchronize(s));
      double t = 0;
      for (double v : h) t += v;
      return t;
    };
    try {
      ms3[0] = timed([&] { spmm(s, om, false, om.m_csr.get(), b, 1.0, X.get(), ldx, 0.0, outm.get(), b); });
      sum3[0] = total(outm, obs.m * b);
      ms3[1] = timed([&] {
        spmm(s, om, true, om.m_csr.get(), b, 1.0, Q.get(), ldx, 0.0, outn.get(), b, om.m_csc.get());
      });
      sum3[1] = total(outn, obs.n * b);
      ms3[2] = timed([&] { sddmm_residual(s, om, kY, Yl.get(), kY, Yr.get(), kY, om.m_csr.get(), r.get()); });
      sum3[2] = total(r, obs.count());
    } catch (...) {
      set_sparse_modes(-1, -1);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      throw;
    }
    set_sparse_modes(-1, -1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

// Diagnostics: cholesky_inverse (the Cholesky + inverse of CholeskyQR) of a random SPD Gram
// (G = X^T X + n I, X 2n x n) of order n, CUDA-event timed over `reps` calls; relres = max
// |R^T R - G| / max |G| and max |R Rinv - I| of the last call.
extern "C++" {
namespace dfcg {
void cholesky_inverse_public(cudaStream_t s, i64 n, double* G, i64 ldg, double* Rinv, i64 ldr, double rel_tol,
                             int* fail, bool want_inverse, bool scale);
}
}
int dfcg_bench_cholesky(dfcg_ctx* ctx, int64_t n, int32_t reps, int32_t want_inverse, double* ms, double* relres,
                        double* invres) {
  return guard([&] {
    if (!ctx || !ms || n < 1 || reps < 1) throw std::invalid_argument("dfcg_bench_cholesky: bad argument");
    CallStream cs(*ctx->dev);
    const cudaStream_t s = cs.s;
    std::vector<double> X(static_cast<size_t>(2 * n * n)), G(static_cast<size_t>(n * n), 0.0);
    std::uint64_t x = 12345;
    for (auto& v : X) {
      x = x * 6364136223846793005ULL + 1442695040888963407ULL;
      v = static_cast<double>(x >> 11) * (1.0 / 9007199254740992.0) - 0.5;
    }
    for (i64 i = 0; i < n; ++i)
      for (i64 j = 0; j < n; ++j) {
        double a = 0;
        for (i64 r = 0; r < 2 * n; ++r) a += X[r * n + i] * X[r * n + j];
        G[i * n + j] = a + (i == j ? n : 0.0);
      }
    DBuf<double> G0(n * n, s), Gw(n * n, s), Ri(n * n, s);
    DBuf<int> fail(1, s);
    DFCG_CUDA(cudaMemcpyAsync(G0.get(), G.data(), sizeof(double) * G.size(), cudaMemcpyHostToDevice, s));
    cudaEvent_t e0, e1;
    DFCG_CUDA(cudaEventCreate(&e0));
    DFCG_CUDA(cudaEventCreate(&e1));
    float total = 0;
    for (int it = 0; it <= reps; ++it) {
      DFCG_CUDA(cudaMemcpyAsync(Gw.get(), G0.get(), sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s));
      fail.zero(s);
      DFCG_CUDA(cudaEventRecord(e0, s));
      cholesky_inverse_public(s, n, Gw.get(), n, Ri.get(), n, 1e-11, fail.get(), want_inverse != 0, true);
      DFCG_CUDA(cudaEventRecord(e1, s));
      DFCG_CUDA(cudaEventSynchronize(e1));
      float t = 0;
      DFCG_CUDA(cudaEventElapsedTime(&t, e0, e1));
      if (it > 0) total += t;  // the first call is a warm-up
    }
    *ms = total / reps;
    std::vector<double> R(static_cast<size_t>(n * n)), Rinv(static_cast<size_t>(n * n));
    DFCG_CUDA(cudaMemcpyAsync(R.data(), Gw.get(), sizeof(double) * n * n, cudaMemcpyDeviceToHost, s));
    DFCG_CUDA(cudaMemcpyAsync(Rinv.data(), Ri.get(), sizeof(double) * n * n, cudaMemcpyDeviceToHost, s));
    DFCG_CUDA(cudaStreamSynchronize(s));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    double gmax = 0, rmax = 0, imax = 0;
    for (i64 i = 0; i < n; ++i)
      for (i64 j = 0; j < n; ++j) {
        double a = 0, b = 0;
        for (i64 l = 0; l <= std::min(i, j); ++l) a += R[l * n + i] * R[l * n + j];
        for (i64 l = i; l <= j; ++l) b += R[i * n + l] * Rinv[l * n + j];
        gmax = std::max(gmax, std::fabs(G[i * n + j]));
        rmax = std::max(rmax, std::fabs(a - G[i * n + j]));
        if (want_inverse) imax = std::max(imax, std::fabs(b - (i == j ? 1.0 : 0.0)));
      }
    if (relres) *relres = rmax / gmax;
    if (invres) *invres = imax;
  });
}

void dfcg_ctx_destroy(dfcg_ctx* ctx) {
  if (!ctx) return;
  delete ctx->dev;
  delete ctx;
}

const char* dfcg_last_error(void) { return g_err.c_str(); }
int64_t dfcg_last_error_block(void) { return g_err_block; }
int64_t dfcg_last_error_line(void) { return g_err_line; }
void dfcg_free(void* p) { std::free(p); }

void dfcg_lowrank_free(dfcg_lowrank* e) {
  if (!e) return;
  std::free(e->left);
  std::free(e->right);
  e->left = e->right = nullptr;
}

void dfcg_sparse_free(dfcg_sparse* s) {
  if (!s) return;
  std::free(s->row);
  std::free(s->col);
  std::free(s->val);
  s->row = s->col = nullptr;
  s->val = nullptr;
}

int dfcg_apg_mc(dfcg_ctx* ctx, const dfcg_obs* in, const dfcg_apg_cfg* cfg, dfcg_lowrank* out,
                dfcg_solve_report* rep, dfcg_iter_trace* trace, int64_t trace_cap, int64_t* trace_len) {
  return guard([&] {
    if (!ctx || !in || !out) throw std::invalid_argument("dfcg_apg_mc: null argument");
    HostObs obs = HostObs::make(in->m, in->n, std::vector<long long>(in->row, in->row + in->nnz),
                                std::vector<long long>(in->col, in->col + in->nnz),
                                std::vector<double>(in->val, in->val + in->nnz));
    CallStream cs(*ctx->dev);
    DevLowRank L;
    SolveReport r;
    std::vector<IterTrace> tr;
    apg_mc_device(*ctx->dev, cs.s, obs.m, obs.n, obs.count(), obs.row.data(), obs.col.data(), obs.val.data(),
                  to_cfg(cfg), L, r, &tr);
    to_c(cs.s, L, out);
    to_report(r, rep);
    to_trace(tr, trace, trace_cap, trace_len);
  });
}

int dfcg_mc_solver_create(dfcg_ctx* ctx, const dfcg_obs* in, const dfcg_apg_cfg* cfg, dfcg_mc_solver** out) {
  return guard([&] {
    if (!ctx || !in || !out) throw std::invalid_argument("dfcg_mc_solver_create: null argument");
    HostObs obs = HostObs::make(in->m, in->n, std::vector<long long>(in->row, in->row + in->nnz),
                                std::vector<long long>(in->col, in->col + in->nnz),
                                std::vector<double>(in->val, in->val + in->nnz));
    DFCG_CUDA(cudaSetDevice(ctx->dev->device));
    auto* h = new dfcg_mc_solver{ctx->dev, ctx->dev->acquire(), nullptr};
    try {
      h->solver = std::make_unique<McSolver>(*ctx->dev, h->s, obs.m, obs.n, obs.count(), obs.row.data(),
                                             obs.col.data(), obs.val.data(), to_cfg(cfg));
      DFCG_CUDA(cudaStreamSynchronize(h->s));
    } catch (...) {
      ctx->dev->release(h->s);
      delete h;
      throw;
    }
    *out = h;
  });
}

int dfcg_mc_solver_step(dfcg_mc_solver* sv, int64_t n_iters, int64_t* done, dfcg_iter_trace* trace,
                        int64_t trace_cap, int64_t* trace_len) {
  return guard([&] {
    if (!sv) throw std::invalid_argument("dfcg_mc_solver_step: null solver");
    DFCG_CUDA(cudaSetDevice(sv->dev->device));
    std::vector<IterTrace> tr;
    int64_t k = 0;
    while (k < n_iters && sv->solver->step(&tr)) ++k;
    DFCG_CUDA(cudaStreamSynchronize(sv->s));
    if (done) *done = k;
    to_trace(tr, trace, trace_cap, trace_len);
  });
}

int dfcg_mc_solver_finish(dfcg_mc_solver* sv, dfcg_lowrank* out, dfcg_solve_report* rep) {
  return guard([&] {
    if (!sv || !out) throw std::invalid_argument("dfcg_mc_solver_finish: null argument");
    DFCG_CUDA(cudaSetDevice(sv->dev->device));
    DevLowRank L;
    SolveReport r;
    sv->solver->finish(L, r);
    to_c(sv->s, L, out);
    to_report(r, rep);
  });
}

void dfcg_mc_solver_destroy(dfcg_mc_solver* sv) {
  if (!sv) return;
  cudaSetDevice(sv->dev->device);
  sv->solver.reset();
  cudaStreamSynchronize(sv->s);
  sv->dev->release(sv->s);
  delete sv;
}

int dfcg_apg_rmf(dfcg_ctx* ctx, const double* M_colmajor, int64_t m, int64_t n, double lambda,
                 const dfcg_apg_cfg* cfg, dfcg_lowrank* L, dfcg_sparse* S, dfcg_solve_report* rep,
                 dfcg_iter_trace* trace, int64_t trace_cap, int64_t* trace_len) {
  return guard([&] {
    if (!ctx || !M_colmajor || !L) throw std::invalid_argument("dfcg_apg_rmf: null argument");
    if (m < 1 || n < 1) throw std::invalid_argument("apg_rmf: dims must be positive");
    CallStream cs(*ctx->dev);
    DevLowRank Ld;
    SolveReport r;
    std::vector<IterTrace> tr;
    std::vector<long long> sr, sc;
    std::vector<double> sv;
    apg_rmf_device(*ctx->dev, cs.s, M_colmajor, m, n, lambda, to_cfg(cfg), Ld, sr, sc, sv, r, &tr);
    to_c(cs.s, Ld, L);
    if (S) {
      S->m = m;
      S->n = n;
      S->count = static_cast<int64_t>(sv.size());
      S->row = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * std::max<size_t>(1, sr.size())));
      S->col = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * std::max<size_t>(1, sc.size())));
      S->val = dup_array(sv);
      if (!sr.empty()) {
        std::memcpy(S->row, sr.data(), sizeof(int64_t) * sr.size());
        std::memcpy(S->col, sc.data(), sizeof(int64_t) * sc.size());
      }
    }
    to_report(r, rep);
    to_trace(tr, trace, trace_cap, trace_len);
  });
}

int dfcg_column_project(dfcg_ctx* ctx, const dfcg_lowrank* basis, int64_t t, const dfcg_lowrank* blocks,
                        const int64_t* group_offsets, const int64_t* group_cols, int64_t n, dfcg_lowrank* out) {
  return guard([&] {
    if (!ctx || !basis || !out) throw std::invalid_argument("dfcg_column_project: null argument");
    if (t == 0) throw std::invalid_argument("column_project: no blocks");
    auto groups = groups_from(t, group_offsets, group_cols, n);
    CallStream cs(*ctx->dev);
    DevLowRank b = to_dev(cs.s, basis);
    std::vector<DevLowRank> bl(static_cast<size_t>(t));
    std::vector<const DevLowRank*> p;
    for (int64_t i = 0; i < t; ++i) {
      bl[static_cast<size_t>(i)] = to_dev(cs.s, &blocks[i]);
      p.push_back(&bl[static_cast<size_t>(i)]);
    }
    DevLowRank o;
    column_project(cs.s, b, p, groups, n, o);
    to_c(cs.s, o, out);
  });
}

int dfcg_gen_nystrom(dfcg_ctx* ctx, const dfcg_lowrank* C_hat, const dfcg_lowrank* R_hat, int64_t d,
                     const int64_t* row_idx, int64_t l, const int64_t* col_idx, dfcg_lowrank* out) {
  return guard([&] {
    if (!ctx || !C_hat || !R_hat || !out) throw std::invalid_argument("dfcg_gen_nystrom: null argument");
    CallStream cs(*ctx->dev);
    DevLowRank C = to_dev(cs.s, C_hat), R = to_dev(cs.s, R_hat), o;
    gen_nystrom(cs.s, C, R, std::vector<i64>(row_idx, row_idx + d), std::vector<i64>(col_idx, col_idx + l), o);
    to_c(cs.s, o, out);
  });
}

int dfcg_average_estimates(dfcg_ctx* ctx, int64_t count, const dfcg_lowrank* ests, int64_t recompress_to,
                           dfcg_lowrank* out) {
  return guard([&] {
    if (!ctx || !out) throw std::invalid_argument("dfcg_average_estimates: null argument");
    if (count <= 0) throw std::invalid_argument("average_estimates: empty list");
    CallStream cs(*ctx->dev);
    std::vector<DevLowRank> d(static_cast<size_t>(count));
    std::vector<const DevLowRank*> p;
    for (int64_t i = 0; i < count; ++i) {
      d[static_cast<size_t>(i)] = to_dev(cs.s, &ests[i]);
      p.push_back(&d[static_cast<size_t>(i)]);
    }
    DevLowRank o;
    std::optional<i64> rc;
    if (recompress_to >= 0) rc = recompress_to;
    average_estimates(cs.s, p, rc, o);
    to_c(cs.s, o, out);
  });
}

int dfcg_random_project(dfcg_ctx* ctx, int64_t t, const dfcg_lowrank* blocks, const int64_t* group_offsets,
                        const int64_t* group_cols, int64_t n, int64_t k, int64_t p, int64_t q, uint64_t seed,
                        uint64_t stream, dfcg_lowrank* out) {
  return guard([&] {
    if (!ctx || !out) throw std::invalid_argument("dfcg_random_project: null argument");
    if (t == 0) throw std::invalid_argument("random_project: no blocks");
    auto groups = groups_from(t, group_offsets, group_cols, n);
    CallStream cs(*ctx->dev);
    std::vector<DevLowRank> d(static_cast<size_t>(t));
    std::vector<const DevLowRank*> ptr;
    for (int64_t i = 0; i < t; ++i) {
      d[static_cast<size_t>(i)] = to_dev(cs.s, &blocks[i]);
      ptr.push_back(&d[static_cast<size_t>(i)]);
    }
    SeededRng rng(seed, stream);
    DevLowRank o;
    random_project(cs.s, ptr, groups, n, k, p, q, rng, o);
    to_c(cs.s, o, out);
  });
}

int dfcg_svd_of_product(dfcg_ctx* ctx, const dfcg_lowrank* in, dfcg_lowrank* out, double* s_out, int64_t* rank) {
  return guard([&] {
    if (!ctx || !in || !out) throw std::invalid_argument("dfcg_svd_of_product: null argument");
    CallStream cs(*ctx->dev);
    // raw factor pair (k may exceed min(m, n) here, as in svd_of_product's callers)
    HostLowRank h;
    h.m = in->m;
    h.n = in->n;
    h.k = in->k;
    h.left.assign(in->left, in->left + h.m * h.k);
    h.right.assign(in->right, in->right + h.n * h.k);
    DBuf<double> l(std::max<i64>(1, h.m * h.k), cs.s), r(std::max<i64>(1, h.n * h.k), cs.s),
        tl(std::max<i64>(1, h.m * h.k), cs.s), tr(std::max<i64>(1, h.n * h.k), cs.s);
    if (h.k > 0) {
      DFCG_CUDA(cudaMemcpyAsync(tl.get(), h.left.data(), sizeof(double) * h.m * h.k, cudaMemcpyHostToDevice, cs.s));
      DFCG_CUDA(cudaMemcpyAsync(tr.get(), h.right.data(), sizeof(double) * h.n * h.k, cudaMemcpyHostToDevice, cs.s));
      transpose(cs.s, h.k, h.m, tl.get(), h.m, l.get(), h.k);
      transpose(cs.s, h.k, h.n, tr.get(), h.n, r.get(), h.k);
    }
    SvdOfProduct f = svd_of_product(cs.s, h.m, h.n, h.k, l.get(), r.get());
    to_c(cs.s, f.est, out);
    if (s_out)
      for (size_t i = 0; i < f.s.size(); ++i) s_out[i] = f.s[i];
    if (rank) *rank = f.r;
  });
}

int dfcg_project_block(dfcg_ctx* ctx, const double* Ub, int64_t m, int64_t kb, const dfcg_lowrank* block,
                       double* Rg) {
  return guard([&] {
    if (!ctx || !Ub || !block || !Rg) throw std::invalid_argument("dfcg_project_block: null argument");
    if (block->m != m) throw std::invalid_argument("column_project: row count mismatch");
    CallStream cs(*ctx->dev);
    const i64 w = block->n;
    if (kb == 0) return;
    if (block->k == 0) {
      std::fill(Rg, Rg + w * kb, 0.0);
      return;
    }
    DevLowRank B = to_dev(cs.s, block);
    // Ub col-major m x kb == row-major kb x m -> transpose to row-major m x kb
    DBuf<double> ut(m * kb, cs.s), U(m * kb, cs.s), proj(kb * B.k, cs.s), R(w * kb, cs.s), Rt(w * kb, cs.s);
    DFCG_CUDA(cudaMemcpyAsync(ut.get(), Ub, sizeof(double) * m * kb, cudaMemcpyHostToDevice, cs.s));
    transpose(cs.s, kb, m, ut.get(), m, U.get(), kb);
    gemm(cs.s, true, false, kb, B.k, m, 1.0, U.get(), kb, B.left.get(), B.k, 0.0, proj.get(), B.k);
    gemm(cs.s, false, true, w, kb, B.k, 1.0, B.right.get(), B.k, proj.get(), B.k, 0.0, R.get(), kb);
    transpose(cs.s, w, kb, R.get(), kb, Rt.get(), w);
    DFCG_CUDA(cudaMemcpyAsync(Rg, Rt.get(), sizeof(double) * w * kb, cudaMemcpyDeviceToHost, cs.s));
    DFCG_CUDA(cudaStreamSynchronize(cs.s));
  });
}

namespace {

HostObs obs_from_c(const dfcg_obs* in) {
  return HostObs::make(in->m, in->n, std::vector<long long>(in->row, in->row + in->nnz),
                       std::vector<long long>(in->col, in->col + in->nnz),
                       std::vector<double>(in->val, in->val + in->nnz));
}

DfcConfig dfc_cfg_from_c(const dfcg_dfc_cfg* c) {
  DfcConfig cfg;
  if (c->variant < 0 || c->variant > 2) throw std::invalid_argument("dfc_run: unknown variant");
  cfg.variant = static_cast<DfcVariant>(c->variant);
  cfg.ensemble = c->ensemble != 0;
  cfg.t = c->t;
  cfg.l = c->l;
  cfg.d = c->d;
  cfg.rp_p = c->rp_p;
  cfg.rp_q = c->rp_q;
  cfg.seed = c->seed;
  cfg.solver_cfg = to_cfg(&c->solver);
  cfg.task = c->task == 1 ? Task::RMF : Task::MC;
  cfg.lambda = c->lambda;
  cfg.workers = c->workers;
  cfg.ensemble_anchors = c->ensemble_anchors;
  return cfg;
}

void dfc_report_to_c(const DfcReport& r, dfcg_dfc_report* rep) {
  if (!rep) return;
  rep->divide_ms = r.divide_ms;
  rep->factor_ms = r.factor_ms;
  rep->combine_ms = r.combine_ms;
  rep->total_ms = r.total_ms;
  rep->chosen_k = r.chosen_k;
  rep->k_clamped = r.k_clamped;
  rep->rank_deficient = r.rank_deficient;
  rep->n_sub = static_cast<int64_t>(r.subproblems.size());
  rep->subproblems = static_cast<dfcg_solve_report*>(
      std::malloc(sizeof(dfcg_solve_report) * std::max<size_t>(1, r.subproblems.size())));
  if (!rep->subproblems) throw std::bad_alloc();
  for (size_t i = 0; i < r.subproblems.size(); ++i) to_report(r.subproblems[i], &rep->subproblems[i]);
}

}  // namespace

int dfcg_dfc_run(dfcg_ctx* ctx, const dfcg_obs* in, const dfcg_dfc_cfg* c, dfcg_lowrank* out, dfcg_dfc_report* rep) {
  return guard([&] {
    if (!ctx || !in || !c || !out) throw std::invalid_argument("dfcg_dfc_run: null argument");
    HostObs obs = obs_from_c(in);
    auto [est, r] = dfc_run(*ctx->dev, obs, dfc_cfg_from_c(c));
    {
      CallStream cs(*ctx->dev);
      to_c(cs.s, est, out);
    }
    dfc_report_to_c(r, rep);
  });
}

// ---- multi-GPU
int dfcg_nccl_unique_id(unsigned char id[128]) {
  return guard([&] {
    if (!id) throw std::invalid_argument("dfcg_nccl_unique_id: null argument");
    nccl_unique_id(id);
  });
}

int dfcg_comm_init_nccl(dfcg_ctx* ctx, int32_t nranks, int32_t rank, const unsigned char id[128], dfcg_comm** out) {
  return guard([&] {
    if (!ctx || !id || !out) throw std::invalid_argument("dfcg_comm_init_nccl: null argument");
    auto c = std::make_unique<dfcg_comm>();
    c->comm = make_nccl_comm(nranks, rank, id, ctx->dev->device);
    *out = c.release();
  });
}

int dfcg_comm_init_host(int32_t nranks, int32_t rank, const dfcg_host_transport* t, dfcg_comm** out) {
  return guard([&] {
    if (!t || !out) throw std::invalid_argument("dfcg_comm_init_host: null argument");
    auto c = std::make_unique<dfcg_comm>();
    c->comm = make_host_comm(nranks, rank, *t);
    *out = c.release();
  });
}

void dfcg_comm_destroy(dfcg_comm* comm) { delete comm; }

int dfcg_comm_selftest(dfcg_comm* comm, int64_t* errors) {
  return guard([&] {
    if (!comm || !errors) throw std::invalid_argument("dfcg_comm_selftest: null argument");
    *errors = comm->comm->selftest();
  });
}

int dfcg_assign_blocks(int64_t count, const int64_t* nnz, int32_t nranks, int32_t* owner) {
  return guard([&] {
    if (count < 0 || (count > 0 && (!nnz || !owner))) throw std::invalid_argument("dfcg_assign_blocks: null argument");
    const std::vector<int> o = assign_blocks_lpt(std::vector<i64>(nnz, nnz + count), nranks);
    for (int64_t i = 0; i < count; ++i) owner[i] = o[static_cast<size_t>(i)];
  });
}

int dfcg_dfc_run_dist(dfcg_ctx* ctx, dfcg_comm* comm, const dfcg_obs* in, const dfcg_dfc_cfg* c, dfcg_lowrank* out,
                      dfcg_dfc_report* rep, int32_t* owner, int64_t owner_cap) {
  return guard([&] {
    if (!ctx || !comm || !in || !c || !out) throw std::invalid_argument("dfcg_dfc_run_dist: null argument");
    HostObs obs = obs_from_c(in);
    std::vector<int> own;
    auto [est, r] = dfc_run_dist(*ctx->dev, *comm->comm, obs, dfc_cfg_from_c(c), &own);
    {
      CallStream cs(*ctx->dev);
      to_c(cs.s, est, out);
    }
    dfc_report_to_c(r, rep);
    if (owner)
      for (size_t i = 0; i < own.size() && static_cast<int64_t>(i) < owner_cap; ++i) owner[i] = own[i];
  });
}

void dfcg_dfc_report_free(dfcg_dfc_report* rep) {
  if (!rep) return;
  std::free(rep->subproblems);
  rep->subproblems = nullptr;
}

}  // extern "C"
