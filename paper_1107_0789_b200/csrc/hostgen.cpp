// Host utilities (include/dfcg_host.h): the reference's RNG, sampling and instance
// generators (P/include/dfc/rng.hpp, sampling.hpp, simgen.hpp), restated so the bench can
// synthesise the reference's exact inputs on the GPU box.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>

#include "../../include/dfcg_host.h"
#include "dfc_host.hpp"
#include "triplet_io.hpp"

using namespace dfcg;

namespace {

template <class T>
T* dup(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * std::max<size_t>(1, v.size())));
  if (!p) throw std::bad_alloc();
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}

// gen_low_rank, simgen.hpp:30-40 (factor std (1/r)^(1/4), A then B, column-major fill).
void gen_low_rank(i64 m, i64 n, i64 r, SeededRng& rng, std::vector<double>& A, std::vector<double>& B) {
  if (r < 1 || r > std::min(m, n)) throw std::invalid_argument("gen_low_rank: need 1 <= r <= min(m,n)");
  const double sd = std::pow(1.0 / static_cast<double>(r), 0.25);
  A.assign(static_cast<size_t>(m * r), 0.0);
  B.assign(static_cast<size_t>(n * r), 0.0);
  for (i64 j = 0; j < r; ++j)
    for (i64 i = 0; i < m; ++i) A[static_cast<size_t>(j * m + i)] = rng.normal(0.0, sd);
  for (i64 j = 0; j < r; ++j)
    for (i64 i = 0; i < n; ++i) B[static_cast<size_t>(j * n + i)] = rng.normal(0.0, sd);
}

double row_dot(const std::vector<double>& A, i64 m, i64 i, const std::vector<double>& B, i64 n, i64 j, i64 r) {
  double acc = 0.0;
  for (i64 k = 0; k < r; ++k) acc += A[static_cast<size_t>(k * m + i)] * B[static_cast<size_t>(k * n + j)];
  return acc;
}

}  // namespace


namespace dfcg {

void Mt64::seed(std::uint64_t s) {
  mt[0] = s;
  for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + static_cast<std::uint64_t>(i);
  idx = 312;
}

namespace {
constexpr std::uint64_t kUM = 0xFFFFFFFF80000000ULL, kLM = 0x7FFFFFFFULL, kMA = 0xB5026F5AA96619E9ULL;

// One MT19937-64 twist: new[i] for i < 156 reads old words only; i in [156, 311) reads new[i - 156]
// and old[i], old[i + 1]; i = 311 reads new[0] and new[155] — three loops without carried
// dependences (the in-place reference loop is the same recurrence).
__attribute__((optimize("O3"), target_clones("avx512f", "avx2", "default"))) void mt64_twist(std::uint64_t* __restrict__ mt, std::uint64_t* __restrict__ nw) {
  for (int i = 0; i < 156; ++i) {
    const std::uint64_t x = (mt[i] & kUM) | (mt[i + 1] & kLM);
    nw[i] = mt[i + 156] ^ (x >> 1) ^ ((0 - (x & 1ULL)) & kMA);
  }
  for (int i = 156; i < 311; ++i) {
    const std::uint64_t x = (mt[i] & kUM) | (mt[i + 1] & kLM);
    nw[i] = nw[i - 156] ^ (x >> 1) ^ ((0 - (x & 1ULL)) & kMA);
  }
  const std::uint64_t x = (mt[311] & kUM) | (nw[0] & kLM);
  nw[311] = nw[155] ^ (x >> 1) ^ ((0 - (x & 1ULL)) & kMA);
}

__attribute__((optimize("O3"), target_clones("avx512f", "avx2", "default"))) void mt64_temper(const std::uint64_t* __restrict__ mt, std::uint64_t* __restrict__ out,
                                                 int n) {
  for (int i = 0; i < n; ++i) {
    std::uint64_t y = mt[i];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    out[i] = y;
  }
}
}  // namespace

void mt64_fill(Mt64& g, std::uint64_t* out, std::int64_t n) {
  std::uint64_t nw[312];
  while (n > 0) {
    if (g.idx == 312) {
      mt64_twist(g.mt, nw);
      std::memcpy(g.mt, nw, sizeof(nw));
      g.idx = 0;
    }
    const int take = static_cast<int>(std::min<std::int64_t>(n, 312 - g.idx));
    mt64_temper(g.mt + g.idx, out, take);
    g.idx += take;
    out += take;
    n -= take;
  }
}

}  // namespace dfcg

extern "C" {

void dfcg_rng_u64_bulk(uint64_t seed, uint64_t stream, int64_t n, uint64_t* out) {
  Mt64 g;
  g.seed(SeededRng::engine_seed(seed, stream));
  mt64_fill(g, out, n);
}

void dfcg_rng_u64(uint64_t seed, uint64_t stream, int64_t n, uint64_t* out) {
  SeededRng r(seed, stream);
  for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
void dfcg_rng_uniform(uint64_t seed, uint64_t stream, int64_t n, double* out) {
  SeededRng r(seed, stream);
  for (int64_t i = 0; i < n; ++i) out[i] = r.uniform();
}
void dfcg_rng_normal(uint64_t seed, uint64_t stream, int64_t n, double* out) {
  SeededRng r(seed, stream);
  for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
}

}  // extern "C"

// The remaining entry points report errors through capi.cpp's thread-local channel.
extern int dfcg_guard_call(const std::function<void()>& f);

extern "C" {

int dfcg_rng_index(uint64_t seed, uint64_t stream, int64_t count, uint64_t bound, uint64_t* out) {
  return dfcg_guard_call([&] {
    SeededRng r(seed, stream);
    for (int64_t i = 0; i < count; ++i) out[i] = r.index(bound);
  });
}

int dfcg_sample_without_replacement(uint64_t seed, uint64_t stream, int64_t n, int64_t l, int64_t* out) {
  return dfcg_guard_call([&] {
    SeededRng r(seed, stream);
    auto v = sample_without_replacement(n, l, r);
    std::memcpy(out, v.data(), sizeof(int64_t) * v.size());
  });
}

int dfcg_partition_columns(uint64_t seed, uint64_t stream, int64_t n, int64_t t, int64_t* cols, int64_t* offsets) {
  return dfcg_guard_call([&] {
    SeededRng r(seed, stream);
    auto plan = partition_columns(n, t, r);
    int64_t at = 0;
    offsets[0] = 0;
    for (size_t g = 0; g < plan.size(); ++g) {
      for (i64 c : plan[g]) cols[at++] = c;
      offsets[g + 1] = at;
    }
  });
}

int dfcg_extract_subproblems(const dfcg_obs* in, int64_t ngroups, const int64_t* group_offsets,
                             const int64_t* group_cols, int64_t nrows, const int64_t* rows, int64_t* counts,
                             int64_t** out_rows, int64_t** out_cols, double** out_vals) {
  return dfcg_guard_call([&] {
    if (!in || !counts || !out_rows || !out_cols || !out_vals || (ngroups > 0 && (!group_offsets || !group_cols)) ||
        (nrows > 0 && !rows))
      throw std::invalid_argument("dfcg_extract_subproblems: null argument");
    HostObs obs = HostObs::make(in->m, in->n, std::vector<long long>(in->row, in->row + in->nnz),
                                std::vector<long long>(in->col, in->col + in->nnz),
                                std::vector<double>(in->val, in->val + in->nnz));
    std::vector<std::vector<i64>> groups(static_cast<size_t>(ngroups));
    for (int64_t g = 0; g < ngroups; ++g) groups[g].assign(group_cols + group_offsets[g], group_cols + group_offsets[g + 1]);
    std::vector<i64> r(rows, rows + std::max<int64_t>(nrows, 0));
    std::vector<HostObs> subs = extract_subproblems(obs, groups, nrows > 0 ? &r : nullptr);
    size_t total = 0;
    for (const auto& o : subs) total += o.val.size();
    *out_rows = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * std::max<size_t>(1, total)));
    *out_cols = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * std::max<size_t>(1, total)));
    *out_vals = static_cast<double*>(std::malloc(sizeof(double) * std::max<size_t>(1, total)));
    if (!*out_rows || !*out_cols || !*out_vals) throw std::bad_alloc();
    size_t at = 0;
    for (size_t i = 0; i < subs.size(); ++i) {
      counts[i] = static_cast<int64_t>(subs[i].val.size());
      std::memcpy(*out_rows + at, subs[i].row.data(), sizeof(int64_t) * subs[i].val.size());
      std::memcpy(*out_cols + at, subs[i].col.data(), sizeof(int64_t) * subs[i].val.size());
      std::memcpy(*out_vals + at, subs[i].val.data(), sizeof(double) * subs[i].val.size());
      at += subs[i].val.size();
    }
  });
}

// BASELINE configs[3] (c4) stand-in — recommender-shaped matrix completion, which the
// reference's generators cannot produce: m x n with Zipf(s = 1) row and column
// popularity (the Zipf ranks assigned by random permutations), cells drawn with probability
// proportional to row_pop * col_pop (Walker alias tables) and deduplicated, values
// clip(round(3.6 + A B^T + N(0, noise^2)), 1, 5) with A, B iid N(0, fsd^2). Restricted to a column
// subset (a D-step block), the cells are drawn conditional on the column lying in the subset and
// the target count scales with the subset's popularity mass, so each block is the block of the
// full instance in distribution. Everything on SeededRng(seed, stream); parity of this generator
// is unpinned (no reference), the solves on its output are checked against the oracle.
namespace {
struct Alias {
  std::vector<double> prob;
  std::vector<int> alias;
  explicit Alias(const std::vector<double>& w) : prob(w.size()), alias(w.size()) {
    const i64 k = static_cast<i64>(w.size());
    double tot = 0.0;
    for (double x : w) tot += x;
    std::vector<double> q(w.size());
    std::vector<int> small, large;
    for (i64 i = 0; i < k; ++i) {
      q[i] = w[i] * k / tot;
      (q[i] < 1.0 ? small : large).push_back(static_cast<int>(i));
    }
    while (!small.empty() && !large.empty()) {
      const int a = small.back(), b = large.back();
      small.pop_back();
      prob[a] = q[a];
      alias[a] = b;
      q[b] -= 1.0 - q[a];
      if (q[b] < 1.0) {
        large.pop_back();
        small.push_back(b);
      }
    }
    for (int i : large) prob[i] = 1.0, alias[i] = i;
    for (int i : small) prob[i] = 1.0, alias[i] = i;
  }
  int sample(SeededRng& r) const {
    const i64 i = static_cast<i64>(r.index(prob.size()));
    return r.uniform() < prob[i] ? static_cast<int>(i) : alias[i];
  }
};
std::vector<double> zipf_popularity(i64 k, SeededRng& r) {  // 1 / rank, ranks a random permutation
  std::vector<i64> perm(k);
  for (i64 i = 0; i < k; ++i) perm[i] = i;
  for (i64 i = k - 1; i > 0; --i) std::swap(perm[i], perm[static_cast<i64>(r.index(i + 1))]);
  std::vector<double> w(k);
  for (i64 i = 0; i < k; ++i) w[i] = 1.0 / static_cast<double>(perm[i] + 1);
  return w;
}
}  // namespace

int dfcg_gen_recsys_instance(int64_t m, int64_t n, int64_t r, double density, double fsd, double noise,
                             int64_t ncols_sub, const int64_t* cols_sub, uint64_t seed, uint64_t stream,
                             int64_t* count, int64_t** rows, int64_t** cols, double** vals) {
  return dfcg_guard_call([&] {
    if (m < 1 || n < 1 || r < 1 || !(density > 0 && density <= 1))
      throw std::invalid_argument("gen_recsys_instance: bad shape or density");
    SeededRng rng(seed, stream);
    std::vector<double> A(static_cast<size_t>(m * r)), B(static_cast<size_t>(n * r));
    for (double& x : A) x = rng.normal(0.0, fsd);
    for (double& x : B) x = rng.normal(0.0, fsd);
    const std::vector<double> rp = zipf_popularity(m, rng), cp = zipf_popularity(n, rng);
    std::vector<i64> sub;
    if (ncols_sub > 0) {
      sub.assign(cols_sub, cols_sub + ncols_sub);
      for (i64 c : sub)
        if (c < 0 || c >= n) throw std::out_of_range("gen_recsys_instance: column subset out of range");
    } else {
      sub.resize(static_cast<size_t>(n));
      for (i64 j = 0; j < n; ++j) sub[static_cast<size_t>(j)] = j;
    }
    const i64 w = static_cast<i64>(sub.size());
    std::vector<double> wq(static_cast<size_t>(w));
    double mass = 0.0, tot = 0.0;
    for (double x : cp) tot += x;
    for (i64 j = 0; j < w; ++j) mass += (wq[static_cast<size_t>(j)] = cp[static_cast<size_t>(sub[static_cast<size_t>(j)])]);
    const i64 target = std::max<i64>(1, std::llround(density * static_cast<double>(m) * static_cast<double>(n) * mass / tot));
    const Alias ar(rp), ac(wq);
    std::vector<std::uint64_t> keys;  // local column * m + row: column-major order
    for (int round = 0; round < 8 && static_cast<i64>(keys.size()) < target - target / 100; ++round) {
      const i64 want = target - static_cast<i64>(keys.size());
      for (i64 d = 0; d < want; ++d) {
        const std::uint64_t row = static_cast<std::uint64_t>(ar.sample(rng));
        const std::uint64_t col = static_cast<std::uint64_t>(ac.sample(rng));
        keys.push_back(col * static_cast<std::uint64_t>(m) + row);
      }
      std::sort(keys.begin(), keys.end());
      keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    }
    const i64 cnt = static_cast<i64>(keys.size());
    int64_t* ro = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * std::max<i64>(cnt, 1)));
    int64_t* co = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * std::max<i64>(cnt, 1)));
    double* va = static_cast<double*>(std::malloc(sizeof(double) * std::max<i64>(cnt, 1)));
    if (!ro || !co || !va) throw std::bad_alloc();
    for (i64 e = 0; e < cnt; ++e) {
      const i64 i = static_cast<i64>(keys[static_cast<size_t>(e)] % static_cast<std::uint64_t>(m));
      const i64 jl = static_cast<i64>(keys[static_cast<size_t>(e)] / static_cast<std::uint64_t>(m));
      const i64 j = sub[static_cast<size_t>(jl)];
      double dot = 0.0;
      for (i64 k = 0; k < r; ++k) dot += A[static_cast<size_t>(k * m + i)] * B[static_cast<size_t>(k * n + j)];
      const double v = std::round(3.6 + dot + rng.normal(0.0, noise));
      ro[e] = i;
      co[e] = jl;
      va[e] = std::min(5.0, std::max(1.0, v));
    }
    *count = cnt;
    *rows = ro;
    *cols = co;
    *vals = va;
  });
}

// gen_mc_instance, simgen.hpp:45-59.
int dfcg_gen_mc_instance(int64_t m, int64_t n, int64_t r, int64_t s, double sigma, uint64_t seed, uint64_t stream,
                         dfcg_lowrank* L0, int64_t** rows, int64_t** cols, double** vals) {
  return dfcg_guard_call([&] {
    if (s < 1 || s > m * n) throw std::invalid_argument("gen_mc_instance: need 1 <= s <= m*n");
    if (sigma < 0) throw std::invalid_argument("gen_mc_instance: sigma must be nonnegative");
    SeededRng rng(seed, stream);
    std::vector<double> A, B;
    gen_low_rank(m, n, r, rng, A, B);
    std::vector<i64> cells = sample_without_replacement(m * n, s, rng);
    std::vector<long long> ri(static_cast<size_t>(s)), ci(static_cast<size_t>(s));
    std::vector<double> v(static_cast<size_t>(s));
    for (i64 e = 0; e < s; ++e) {
      const i64 c = cells[static_cast<size_t>(e)];
      const i64 i = c % m, j = c / m;
      const double noise = sigma > 0 ? rng.normal(0.0, sigma) : 0.0;
      ri[static_cast<size_t>(e)] = i;
      ci[static_cast<size_t>(e)] = j;
      v[static_cast<size_t>(e)] = row_dot(A, m, i, B, n, j, r) + noise;
    }
    std::vector<i64>().swap(cells);
    HostObs obs = HostObs::make(m, n, std::move(ri), std::move(ci), std::move(v));  // sorts column-major
    L0->m = m;
    L0->n = n;
    L0->k = r;
    L0->left = dup(A);
    L0->right = dup(B);
    *rows = dup(std::vector<int64_t>(obs.row.begin(), obs.row.end()));
    *cols = dup(std::vector<int64_t>(obs.col.begin(), obs.col.end()));
    *vals = dup(obs.val);
  });
}

// load_triplets / save_triplets, matrix_io.hpp:125-179 (parallel; triplet_io.cpp).
namespace {
void triplets_out(TripletFile& f, int64_t* m, int64_t* n, int64_t* count, int64_t** rows, int64_t** cols,
                  double** vals) {
  *m = f.m;
  *n = f.n;
  *count = static_cast<int64_t>(f.val.size());
  *rows = dup(std::vector<int64_t>(f.row.begin(), f.row.end()));
  std::vector<long long>().swap(f.row);
  *cols = dup(std::vector<int64_t>(f.col.begin(), f.col.end()));
  std::vector<long long>().swap(f.col);
  *vals = dup(f.val);
}
}  // namespace

int dfcg_load_triplets_text(const char* text, int64_t len, int32_t one_based, int64_t* m, int64_t* n, int64_t* count,
                            int64_t** rows, int64_t** cols, double** vals) {
  return dfcg_guard_call([&] {
    if ((!text && len > 0) || len < 0 || !m || !n || !count || !rows || !cols || !vals)
      throw std::invalid_argument("dfcg_load_triplets_text: bad argument");
    TripletFile f = load_triplets_text(text ? text : "", static_cast<size_t>(len), one_based != 0);
    triplets_out(f, m, n, count, rows, cols, vals);
  });
}

int dfcg_load_triplets_file(const char* path, int32_t one_based, int64_t* m, int64_t* n, int64_t* count,
                            int64_t** rows, int64_t** cols, double** vals) {
  return dfcg_guard_call([&] {
    if (!path || !m || !n || !count || !rows || !cols || !vals)
      throw std::invalid_argument("dfcg_load_triplets_file: bad argument");
    TripletFile f = load_triplets_file(path, one_based != 0);
    triplets_out(f, m, n, count, rows, cols, vals);
  });
}

int dfcg_save_triplets_file(const char* path, const dfcg_obs* in) {
  return dfcg_guard_call([&] {
    if (!path || !in || in->nnz < 0 || (in->nnz > 0 && (!in->row || !in->col || !in->val)))
      throw std::invalid_argument("dfcg_save_triplets_file: bad argument");
    static_assert(sizeof(long long) == sizeof(int64_t), "index width");
    save_triplets_file(path, in->m, in->n, static_cast<size_t>(in->nnz), reinterpret_cast<const long long*>(in->row),
                       reinterpret_cast<const long long*>(in->col), in->val);
  });
}

int dfcg_format_triplets(const dfcg_obs* in, char** text, int64_t* len) {
  return dfcg_guard_call([&] {
    if (!in || !text || !len || in->nnz < 0 || (in->nnz > 0 && (!in->row || !in->col || !in->val)))
      throw std::invalid_argument("dfcg_format_triplets: bad argument");
    const std::string s = format_triplets(in->m, in->n, static_cast<size_t>(in->nnz),
                                          reinterpret_cast<const long long*>(in->row),
                                          reinterpret_cast<const long long*>(in->col), in->val);
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    if (!p) throw std::bad_alloc();
    std::memcpy(p, s.data(), s.size());
    p[s.size()] = 0;
    *text = p;
    *len = static_cast<int64_t>(s.size());
  });
}

// gen_rmf_instance, simgen.hpp:64-82 (outlier range parameterised).
int dfcg_gen_rmf_instance(int64_t m, int64_t n, int64_t r, int64_t s, double sigma, uint64_t seed, uint64_t stream,
                          double lo, double hi, dfcg_lowrank* L0, dfcg_sparse* S0, double* M) {
  return dfcg_guard_call([&] {
    if (s < 0 || s > m * n) throw std::invalid_argument("gen_rmf_instance: need 0 <= s <= m*n");
    if (sigma < 0) throw std::invalid_argument("gen_rmf_instance: sigma must be nonnegative");
    SeededRng rng(seed, stream);
    std::vector<double> A, B;
    gen_low_rank(m, n, r, rng, A, B);
    std::vector<long long> sr, sc;
    std::vector<double> sv;
    if (s > 0) {
      std::vector<i64> cells = sample_without_replacement(m * n, s, rng);
      for (i64 c : cells) {
        const double u = rng.uniform();
        sr.push_back(c % m);
        sc.push_back(c / m);
        sv.push_back((lo == 0.0 && hi == 1.0) ? u : lo + (hi - lo) * u);
      }
    }
    // M = materialize(L0) + S0 (+ noise, column-major fill)
    for (i64 j = 0; j < n; ++j)
      for (i64 i = 0; i < m; ++i) M[j * m + i] = row_dot(A, m, i, B, n, j, r);
    for (size_t e = 0; e < sv.size(); ++e) M[sc[e] * m + sr[e]] += sv[e];
    if (sigma > 0)
      for (i64 j = 0; j < n; ++j)
        for (i64 i = 0; i < m; ++i) M[j * m + i] += rng.normal(0.0, sigma);
    L0->m = m;
    L0->n = n;
    L0->k = r;
    L0->left = dup(A);
    L0->right = dup(B);
    S0->m = m;
    S0->n = n;
    S0->count = static_cast<int64_t>(sv.size());
    S0->row = dup(std::vector<int64_t>(sr.begin(), sr.end()));
    S0->col = dup(std::vector<int64_t>(sc.begin(), sc.end()));
    S0->val = dup(sv);
  });
}

}  // extern "C"
