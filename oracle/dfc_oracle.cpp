// TEST INFRASTRUCTURE ONLY — CPU oracle for the DFC hot path (see dfc_oracle.hpp).
// Each function cites the reference lines it restates (P/ = /root/reference/proj/).
#include "dfc_oracle.hpp"

#include <cstring>

// numpy's bundled OpenBLAS, ILP64 ("64_" suffix).
extern "C" {
void scipy_cblas_dgemm64_(int order, int ta, int tb, std::int64_t m, std::int64_t n, std::int64_t k,
                          double alpha, const double* a, std::int64_t lda, const double* b,
                          std::int64_t ldb, double beta, double* c, std::int64_t ldc);
std::int64_t scipy_LAPACKE_dgeqrf64_(int layout, std::int64_t m, std::int64_t n, double* a,
                                     std::int64_t lda, double* tau);
std::int64_t scipy_LAPACKE_dorgqr64_(int layout, std::int64_t m, std::int64_t n, std::int64_t k,
                                     double* a, std::int64_t lda, const double* tau);
std::int64_t scipy_LAPACKE_dgesdd64_(int layout, char jobz, std::int64_t m, std::int64_t n, double* a,
                                     std::int64_t lda, double* s, double* u, std::int64_t ldu,
                                     double* vt, std::int64_t ldvt);
std::int64_t scipy_LAPACKE_dgesvd64_(int layout, char jobu, char jobvt, std::int64_t m, std::int64_t n,
                                     double* a, std::int64_t lda, double* s, double* u,
                                     std::int64_t ldu, double* vt, std::int64_t ldvt, double* superb);
}

namespace orc {

namespace {
constexpr int kColMajor = 102, kNoTrans = 111, kTrans = 112;
}

// ================================================================ dense kernels (Eigen stand-ins)
void gemm_into(bool ta, bool tb, double alpha, const Mat& A, const Mat& B, double beta, Mat& C) {
  const Index m = ta ? A.c : A.r, k = ta ? A.r : A.c;
  const Index n = tb ? B.r : B.c;
  const Index kb = tb ? B.c : B.r;
  if (k != kb) throw std::invalid_argument("gemm: inner dimension mismatch");
  if (C.r != m || C.c != n) throw std::invalid_argument("gemm: output shape mismatch");
  if (m == 0 || n == 0) return;
  if (k == 0) {
    for (double& v : C.d) v *= beta;
    return;
  }
  scipy_cblas_dgemm64_(kColMajor, ta ? kTrans : kNoTrans, tb ? kTrans : kNoTrans, m, n, k, alpha,
                       A.d.data(), std::max<Index>(1, A.r), B.d.data(), std::max<Index>(1, B.r), beta,
                       C.d.data(), std::max<Index>(1, C.r));
}

Mat gemm(bool ta, bool tb, double alpha, const Mat& A, const Mat& B) {
  Mat C(ta ? A.c : A.r, tb ? B.r : B.c);
  gemm_into(ta, tb, alpha, A, B, 0.0, C);
  return C;
}

// thin_qr, P/include/dfc/sketch.hpp:41-47 (Eigen HouseholderQR; Q = H * I[:, :r], R = triu(top r rows)).
std::pair<Mat, Mat> thin_qr(const Mat& A) {
  const Index m = A.r, n = A.c, r = std::min(m, n);
  if (r == 0) return {Mat(m, 0), Mat(0, n)};
  Mat F = A;
  std::vector<double> tau(static_cast<std::size_t>(r));
  if (scipy_LAPACKE_dgeqrf64_(kColMajor, m, n, F.d.data(), m, tau.data()) != 0)
    throw std::runtime_error("thin_qr: dgeqrf failed");
  Mat R(r, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i <= std::min(j, r - 1); ++i) R(i, j) = F(i, j);
  Mat Q(m, r);
  std::copy(F.d.begin(), F.d.begin() + m * r, Q.d.begin());
  if (scipy_LAPACKE_dorgqr64_(kColMajor, m, r, r, Q.d.data(), m, tau.data()) != 0)
    throw std::runtime_error("thin_qr: dorgqr failed");
  return {std::move(Q), std::move(R)};
}

// Eigen::BDCSVD(A, ComputeThinU | ComputeThinV) stand-in: divide-and-conquer dgesdd,
// dgesvd if it fails to converge. Singular values nonincreasing.
Svd thin_svd(const Mat& A) {
  const Index m = A.r, n = A.c, p = std::min(m, n);
  Svd out{Mat(m, p), std::vector<double>(static_cast<std::size_t>(p)), Mat(n, p)};
  if (p == 0) return out;
  Mat W = A;
  Mat VT(p, n);
  std::int64_t info = scipy_LAPACKE_dgesdd64_(kColMajor, 'S', m, n, W.d.data(), m, out.s.data(),
                                              out.U.d.data(), m, VT.d.data(), p);
  if (info != 0) {
    W = A;
    std::vector<double> superb(static_cast<std::size_t>(std::max<Index>(1, p)));
    info = scipy_LAPACKE_dgesvd64_(kColMajor, 'S', 'S', m, n, W.d.data(), m, out.s.data(),
                                   out.U.d.data(), m, VT.d.data(), p, superb.data());
    if (info != 0) throw std::runtime_error("thin_svd: LAPACK SVD failed to converge");
  }
  out.V = VT.transpose();
  return out;
}

// ================================================================ data model (P/include/dfc/matrix_io.hpp)
// ObservedMatrix ctor, matrix_io.hpp:38-56: sort column-major, validate range/finite/duplicates.
ObservedMatrix::ObservedMatrix(Index m, Index n, std::vector<Observation> obs) : m_(m), n_(n), obs_(std::move(obs)) {
  if (m < 1 || n < 1) throw std::invalid_argument("ObservedMatrix: dims must be positive");
  std::sort(obs_.begin(), obs_.end(), [](const Observation& a, const Observation& b) {
    return a.col != b.col ? a.col < b.col : a.row < b.row;
  });
  for (std::size_t i = 0; i < obs_.size(); ++i) {
    const Observation& e = obs_[i];
    if (e.row < 0 || e.row >= m_ || e.col < 0 || e.col >= n_)
      throw std::out_of_range("ObservedMatrix: entry (" + std::to_string(e.row) + ", " + std::to_string(e.col) +
                              ") outside " + std::to_string(m_) + "x" + std::to_string(n_));
    if (!std::isfinite(e.value)) throw std::invalid_argument("ObservedMatrix: non-finite value");
    if (i > 0 && obs_[i - 1].row == e.row && obs_[i - 1].col == e.col)
      throw std::invalid_argument("ObservedMatrix: duplicate entry (" + std::to_string(e.row) + ", " +
                                  std::to_string(e.col) + ")");
  }
}

// LowRankEstimate ctor, matrix_io.hpp:73-84.
LowRankEstimate::LowRankEstimate(Mat left, Mat right) : left_(std::move(left)), right_(std::move(right)) {
  if (left_.c != right_.c) throw std::invalid_argument("LowRankEstimate: factor rank mismatch");
  if (left_.r < 1 || right_.r < 1) throw std::invalid_argument("LowRankEstimate: dims must be positive");
  if (left_.c > std::min(left_.r, right_.r)) throw std::invalid_argument("LowRankEstimate: k exceeds min(m, n)");
  if (!left_.all_finite() || !right_.all_finite())
    throw std::invalid_argument("LowRankEstimate: non-finite factor entry");
}

// SvdFactors::to_estimate, matrix_io.hpp:108-111: left = U, right = V diag(s).
LowRankEstimate SvdFactors::to_estimate() const {
  if (s.empty()) return LowRankEstimate::zero(U.r, V.r);
  Mat right = V;
  for (Index j = 0; j < right.c; ++j)
    for (Index i = 0; i < right.r; ++i) right(i, j) *= s[static_cast<std::size_t>(j)];
  return LowRankEstimate(U, std::move(right));
}

Mat materialize(const LowRankEstimate& e) {
  if (e.rank_bound() == 0) return Mat(e.rows(), e.cols());
  return gemm(false, true, 1.0, e.left(), e.right());
}

Mat densify(const ObservedMatrix& obs) {
  Mat A(obs.rows(), obs.cols());
  for (const auto& e : obs.entries()) A(e.row, e.col) = e.value;
  return A;
}

// ================================================================ sampling (P/include/dfc/sampling.hpp)
// sampling.hpp:15-26, partial Fisher-Yates in draw order.
std::vector<Index> sample_without_replacement(Index n, Index l, SeededRng& rng) {
  if (n < 1) throw std::invalid_argument("sample_without_replacement: empty population");
  if (l < 1 || l > n) throw std::invalid_argument("sample_without_replacement: need 1 <= l <= n");
  std::vector<Index> perm(static_cast<std::size_t>(n));
  std::iota(perm.begin(), perm.end(), Index{0});
  for (Index i = 0; i < l; ++i) {
    const Index j = i + static_cast<Index>(rng.index(static_cast<std::uint64_t>(n - i)));
    std::swap(perm[static_cast<std::size_t>(i)], perm[static_cast<std::size_t>(j)]);
  }
  perm.resize(static_cast<std::size_t>(l));
  return perm;
}

// PartitionPlan, sampling.hpp:32-51.
PartitionPlan::PartitionPlan(Index n, std::vector<std::vector<Index>> groups) : n_(n), groups_(std::move(groups)) {
  std::vector<char> seen(static_cast<std::size_t>(n), 0);
  std::size_t total = 0, min_sz = static_cast<std::size_t>(n), max_sz = 0;
  for (const auto& g : groups_) {
    min_sz = std::min(min_sz, g.size());
    max_sz = std::max(max_sz, g.size());
    for (std::size_t p = 0; p < g.size(); ++p) {
      const Index c = g[p];
      if (c < 0 || c >= n) throw std::out_of_range("PartitionPlan: column out of range");
      if (seen[static_cast<std::size_t>(c)]++) throw std::invalid_argument("PartitionPlan: overlapping groups");
      if (p > 0 && g[p - 1] >= c) throw std::invalid_argument("PartitionPlan: group not sorted");
      ++total;
    }
  }
  if (total != static_cast<std::size_t>(n)) throw std::invalid_argument("PartitionPlan: groups do not cover all columns");
  if (max_sz > min_sz + 1) throw std::invalid_argument("PartitionPlan: group sizes differ by more than 1");
}

// partition_columns, sampling.hpp:66-79.
PartitionPlan partition_columns(Index n, Index t, SeededRng& rng) {
  if (t < 1 || t > n) throw std::invalid_argument("partition_columns: need 1 <= t <= n");
  std::vector<Index> perm = sample_without_replacement(n, n, rng);
  const Index base = n / t, rem = n % t;
  std::vector<std::vector<Index>> groups(static_cast<std::size_t>(t));
  std::size_t at = 0;
  for (Index g = 0; g < t; ++g) {
    const Index sz = base + (g < rem ? 1 : 0);
    auto& grp = groups[static_cast<std::size_t>(g)];
    grp.assign(perm.begin() + static_cast<std::ptrdiff_t>(at), perm.begin() + static_cast<std::ptrdiff_t>(at + sz));
    std::sort(grp.begin(), grp.end());
    at += static_cast<std::size_t>(sz);
  }
  return PartitionPlan(n, std::move(groups));
}

// extract_columns / extract_rows, sampling.hpp:83-113.
ObservedMatrix extract_columns(const ObservedMatrix& obs, const std::vector<Index>& idx) {
  std::vector<Index> pos(static_cast<std::size_t>(obs.cols()), Index{-1});
  for (std::size_t p = 0; p < idx.size(); ++p) {
    const Index c = idx[p];
    if (c < 0 || c >= obs.cols()) throw std::out_of_range("extract_columns: index out of range");
    if (pos[static_cast<std::size_t>(c)] >= 0) throw std::invalid_argument("extract_columns: duplicate index");
    pos[static_cast<std::size_t>(c)] = static_cast<Index>(p);
  }
  std::vector<Observation> sub;
  for (const auto& e : obs.entries()) {
    const Index p = pos[static_cast<std::size_t>(e.col)];
    if (p >= 0) sub.push_back({e.row, p, e.value});
  }
  return ObservedMatrix(obs.rows(), static_cast<Index>(idx.size()), std::move(sub));
}

ObservedMatrix extract_rows(const ObservedMatrix& obs, const std::vector<Index>& idx) {
  std::vector<Index> pos(static_cast<std::size_t>(obs.rows()), Index{-1});
  for (std::size_t p = 0; p < idx.size(); ++p) {
    const Index r = idx[p];
    if (r < 0 || r >= obs.rows()) throw std::out_of_range("extract_rows: index out of range");
    if (pos[static_cast<std::size_t>(r)] >= 0) throw std::invalid_argument("extract_rows: duplicate index");
    pos[static_cast<std::size_t>(r)] = static_cast<Index>(p);
  }
  std::vector<Observation> sub;
  for (const auto& e : obs.entries()) {
    const Index p = pos[static_cast<std::size_t>(e.row)];
    if (p >= 0) sub.push_back({p, e.col, e.value});
  }
  return ObservedMatrix(static_cast<Index>(idx.size()), obs.cols(), std::move(sub));
}

// ================================================================ simgen (P/include/dfc/simgen.hpp)
OutlierEstimate::OutlierEstimate(Index m_, Index n_, std::vector<Observation> e) : m(m_), n(n_), entries(std::move(e)) {
  if (m < 1 || n < 1) throw std::invalid_argument("OutlierEstimate: dims must be positive");
  for (const auto& o : entries) {
    if (o.row < 0 || o.row >= m || o.col < 0 || o.col >= n)
      throw std::out_of_range("OutlierEstimate: entry out of range");
    if (!std::isfinite(o.value)) throw std::invalid_argument("OutlierEstimate: non-finite value");
  }
}

Mat OutlierEstimate::to_dense() const {
  Mat S(m, n);
  for (const auto& o : entries) S(o.row, o.col) = o.value;
  return S;
}

static double row_dot(const Mat& A, Index i, const Mat& B, Index j) {
  double acc = 0.0;
  for (Index k = 0; k < A.c; ++k) acc += A(i, k) * B(j, k);
  return acc;
}

// gen_low_rank, simgen.hpp:30-40: factor std (1/r)^(1/4), A then B, column-major fill.
LowRankEstimate gen_low_rank(Index m, Index n, Index r, SeededRng& rng) {
  if (r < 1 || r > std::min(m, n)) throw std::invalid_argument("gen_low_rank: need 1 <= r <= min(m,n)");
  const double sd = std::pow(1.0 / static_cast<double>(r), 0.25);
  Mat A(m, r), B(n, r);
  for (Index j = 0; j < r; ++j)
    for (Index i = 0; i < m; ++i) A(i, j) = rng.normal(0.0, sd);
  for (Index j = 0; j < r; ++j)
    for (Index i = 0; i < n; ++i) B(i, j) = rng.normal(0.0, sd);
  return LowRankEstimate(std::move(A), std::move(B));
}

// gen_mc_instance, simgen.hpp:45-59.
McInstance gen_mc_instance(Index m, Index n, Index r, Index s, double sigma, SeededRng& rng) {
  if (s < 1 || s > m * n) throw std::invalid_argument("gen_mc_instance: need 1 <= s <= m*n");
  if (sigma < 0) throw std::invalid_argument("gen_mc_instance: sigma must be nonnegative");
  LowRankEstimate L0 = gen_low_rank(m, n, r, rng);
  std::vector<Index> cells = sample_without_replacement(m * n, s, rng);
  std::vector<Observation> obs;
  obs.reserve(static_cast<std::size_t>(s));
  for (Index c : cells) {
    const Index i = c % m, j = c / m;
    const double noise = sigma > 0 ? rng.normal(0.0, sigma) : 0.0;
    obs.push_back({i, j, row_dot(L0.left(), i, L0.right(), j) + noise});
  }
  return McInstance{std::move(L0), ObservedMatrix(m, n, std::move(obs))};
}

// gen_rmf_instance, simgen.hpp:64-82 (outlier range parameterised; reference = U[0,1]).
RmfInstance gen_rmf_instance(Index m, Index n, Index r, Index s, double sigma, SeededRng& rng, double lo, double hi) {
  if (s < 0 || s > m * n) throw std::invalid_argument("gen_rmf_instance: need 0 <= s <= m*n");
  if (sigma < 0) throw std::invalid_argument("gen_rmf_instance: sigma must be nonnegative");
  LowRankEstimate L0 = gen_low_rank(m, n, r, rng);
  std::vector<Observation> outliers;
  if (s > 0) {
    std::vector<Index> cells = sample_without_replacement(m * n, s, rng);
    outliers.reserve(static_cast<std::size_t>(s));
    for (Index c : cells) {
      const double u = rng.uniform();
      outliers.push_back({c % m, c / m, (lo == 0.0 && hi == 1.0) ? u : lo + (hi - lo) * u});
    }
  }
  OutlierEstimate S0(m, n, std::move(outliers));
  // M = materialize(L0) + S0: entries as plain row dots (Eigen's GEMM summation order is not
  // reproducible anyway); the product's generator uses the same loop, so both agree bitwise.
  Mat M(m, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < m; ++i) M(i, j) = row_dot(L0.left(), i, L0.right(), j);
  for (const auto& o : S0.entries) M(o.row, o.col) += o.value;
  if (sigma > 0)
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < m; ++i) M(i, j) += rng.normal(0.0, sigma);
  return RmfInstance{std::move(L0), std::move(S0), std::move(M)};
}

// ================================================================ sketch (P/include/dfc/sketch.hpp)
// numerical_rank, sketch.hpp:31-38.
Index numerical_rank(const std::vector<double>& s, Index m, Index n, RankTolerance tol) {
  if (s.empty()) return 0;
  const double cut = tol.absolute(s[0], m, n);
  Index r = 0;
  while (r < static_cast<Index>(s.size()) && s[static_cast<std::size_t>(r)] > cut) ++r;
  return r;
}

SvdFactors empty_svd(Index m, Index n) { return SvdFactors{Mat(m, 0), {}, Mat(n, 0)}; }

static SvdFactors head(const Svd& f, Index k) {
  return SvdFactors{f.U.left_cols(k), std::vector<double>(f.s.begin(), f.s.begin() + k), f.V.left_cols(k)};
}

// truncated_svd, sketch.hpp:54-60.
SvdFactors truncated_svd(const Mat& A, Index k) {
  if (k < 1 || k > std::min(A.r, A.c)) throw std::invalid_argument("truncated_svd: need 1 <= k <= min(m,n)");
  return head(thin_svd(A), k);
}

// compact_svd, sketch.hpp:63-69.
SvdFactors compact_svd(const Mat& A, RankTolerance tol) {
  Svd f = thin_svd(A);
  const Index r = numerical_rank(f.s, A.r, A.c, tol);
  if (r == 0) return empty_svd(A.r, A.c);
  return head(f, r);
}

// svd_of_product, sketch.hpp:73-86: QR both factors, SVD of Rl Rr^T.
SvdFactors svd_of_product(const Mat& left, const Mat& right, RankTolerance tol) {
  const Index m = left.r, n = right.r;
  if (left.c != right.c) throw std::invalid_argument("svd_of_product: rank mismatch");
  if (left.c == 0) return empty_svd(m, n);
  auto [Ql, Rl] = thin_qr(left);
  auto [Qr, Rr] = thin_qr(right);
  Mat core = gemm(false, true, 1.0, Rl, Rr);
  Svd svd = thin_svd(core);
  const Index r = numerical_rank(svd.s, m, n, tol);
  if (r == 0) return empty_svd(m, n);
  return SvdFactors{gemm(false, false, 1.0, Ql, svd.U.left_cols(r)),
                    std::vector<double>(svd.s.begin(), svd.s.begin() + r),
                    gemm(false, false, 1.0, Qr, svd.V.left_cols(r))};
}

namespace detail {

// gaussian_matrix, sketch.hpp:133-138: column-major normals.
Mat gaussian_matrix(Index rows, Index cols, SeededRng& rng) {
  Mat G(rows, cols);
  for (Index j = 0; j < cols; ++j)
    for (Index i = 0; i < rows; ++i) G(i, j) = rng.normal();
  return G;
}

// BlocksOp, sketch.hpp:99-131.
struct BlocksOp {
  const std::vector<LowRankEstimate>& blocks;
  const PartitionPlan& plan;
  Index m;
  Index rows() const { return m; }
  Index cols() const { return plan.total_cols(); }
  Mat apply(const Mat& X) const {
    Mat Y(m, X.c);
    for (std::size_t g = 0; g < blocks.size(); ++g) {
      const auto& idx = plan.group(g);
      if (blocks[g].rank_bound() == 0) continue;
      Mat Xg(static_cast<Index>(idx.size()), X.c);
      for (Index c = 0; c < X.c; ++c)
        for (std::size_t p = 0; p < idx.size(); ++p) Xg(static_cast<Index>(p), c) = X(idx[p], c);
      Mat T = gemm(true, false, 1.0, blocks[g].right(), Xg);
      gemm_into(false, false, 1.0, blocks[g].left(), T, 1.0, Y);
    }
    return Y;
  }
  Mat apply_adjoint(const Mat& X) const {
    Mat Y(plan.total_cols(), X.c);
    for (std::size_t g = 0; g < blocks.size(); ++g) {
      const auto& idx = plan.group(g);
      if (blocks[g].rank_bound() == 0) continue;
      Mat T = gemm(true, false, 1.0, blocks[g].left(), X);
      Mat Yg = gemm(false, false, 1.0, blocks[g].right(), T);
      for (Index c = 0; c < X.c; ++c)
        for (std::size_t p = 0; p < idx.size(); ++p) Y(idx[p], c) = Yg(static_cast<Index>(p), c);
    }
    return Y;
  }
};

}  // namespace detail

// randomized_range / partial_svd, sketch.hpp:144-166.
template <class Op>
Mat randomized_range(const Op& op, Index b, Index q, SeededRng& rng) {
  Mat G = detail::gaussian_matrix(op.cols(), b, rng);
  Mat Q = thin_qr(op.apply(G)).first;
  for (Index it = 0; it < q; ++it) {
    Mat Z = thin_qr(op.apply_adjoint(Q)).first;
    Q = thin_qr(op.apply(Z)).first;
  }
  return Q;
}

template <class Op>
SvdFactors partial_svd(const Op& op, Index k, Index p, Index q, SeededRng& rng) {
  const Index b = std::min(k + p, std::min(op.rows(), op.cols()));
  if (b == 0 || k < 1) return empty_svd(op.rows(), op.cols());
  Mat Q = randomized_range(op, b, q, rng);
  Mat Z = op.apply_adjoint(Q);
  Svd svd = thin_svd(Z);
  const Index kk = std::min<Index>(k, static_cast<Index>(svd.s.size()));
  return SvdFactors{gemm(false, false, 1.0, Q, svd.V.left_cols(kk)),
                    std::vector<double>(svd.s.begin(), svd.s.begin() + kk), svd.U.left_cols(kk)};
}

// column_project, sketch.hpp:170-199.
LowRankEstimate column_project(const LowRankEstimate& basis, const std::vector<LowRankEstimate>& blocks,
                               const PartitionPlan& plan, RankTolerance tol) {
  if (blocks.empty()) throw std::invalid_argument("column_project: no blocks");
  if (blocks.size() != plan.group_count()) throw std::invalid_argument("column_project: block count does not match plan");
  const Index m = basis.rows(), n = plan.total_cols();
  for (std::size_t g = 0; g < blocks.size(); ++g) {
    if (blocks[g].rows() != m) throw std::invalid_argument("column_project: row count mismatch");
    if (blocks[g].cols() != static_cast<Index>(plan.group(g).size()))
      throw std::invalid_argument("column_project: block width does not match plan group");
  }
  SvdFactors bf = svd_of_product(basis.left(), basis.right(), tol);
  if (bf.rank() == 0) return LowRankEstimate::zero(m, n);
  const Mat& Ub = bf.U;
  Mat right(n, Ub.c);
  for (std::size_t g = 0; g < blocks.size(); ++g) {
    const auto& idx = plan.group(g);
    if (blocks[g].rank_bound() == 0) continue;  // rows stay zero
    Mat proj = gemm(true, false, 1.0, Ub, blocks[g].left());     // kb x kg
    Mat Rg = gemm(false, true, 1.0, blocks[g].right(), proj);   // w x kb
    for (Index c = 0; c < Rg.c; ++c)
      for (std::size_t p = 0; p < idx.size(); ++p) right(idx[p], c) = Rg(static_cast<Index>(p), c);
  }
  return LowRankEstimate(Ub, std::move(right));
}

// random_project, sketch.hpp:204-237.
LowRankEstimate random_project(const std::vector<LowRankEstimate>& blocks, const PartitionPlan& plan,
                               const RpParams& params, SeededRng& rng, RankTolerance tol) {
  if (blocks.empty()) throw std::invalid_argument("random_project: no blocks");
  if (blocks.size() != plan.group_count()) throw std::invalid_argument("random_project: block count does not match plan");
  if (params.k < 1 || params.p < 0 || params.q < 0) throw std::invalid_argument("random_project: bad RpParams");
  const Index m = blocks[0].rows(), n = plan.total_cols();
  for (std::size_t g = 0; g < blocks.size(); ++g) {
    if (blocks[g].rows() != m) throw std::invalid_argument("random_project: row count mismatch");
    if (blocks[g].cols() != static_cast<Index>(plan.group(g).size()))
      throw std::invalid_argument("random_project: block width does not match plan group");
  }
  if (params.k + params.p > std::min(m, n)) throw std::invalid_argument("random_project: k + p exceeds min(m, n)");
  detail::BlocksOp op{blocks, plan, m};
  const Index b = params.k + params.p;
  Mat G = detail::gaussian_matrix(n, b, rng);
  Mat Y = op.apply(G);
  for (Index it = 0; it < params.q; ++it) {
    Mat Q = thin_qr(Y).first;
    Mat Z = thin_qr(op.apply_adjoint(Q)).first;
    Y = op.apply(Z);
  }
  Svd svd = thin_svd(Y);
  const Index kk = std::min(params.k, numerical_rank(svd.s, m, n, tol));
  if (kk == 0) return LowRankEstimate::zero(m, n);
  Mat Q = svd.U.left_cols(kk);
  Mat right = op.apply_adjoint(Q);
  return LowRankEstimate(std::move(Q), std::move(right));
}

// gen_nystrom, sketch.hpp:241-266.
LowRankEstimate gen_nystrom(const LowRankEstimate& C_hat, const LowRankEstimate& R_hat,
                            const std::vector<Index>& row_idx, const std::vector<Index>& col_idx, RankTolerance tol) {
  const Index m = C_hat.rows(), n = R_hat.cols();
  const Index d = static_cast<Index>(row_idx.size()), l = static_cast<Index>(col_idx.size());
  if (R_hat.rows() != d) throw std::invalid_argument("gen_nystrom: R_hat rows != |row_idx|");
  if (C_hat.cols() != l) throw std::invalid_argument("gen_nystrom: C_hat cols != |col_idx|");
  for (Index i : row_idx)
    if (i < 0 || i >= m) throw std::out_of_range("gen_nystrom: row index out of range");
  for (Index j : col_idx)
    if (j < 0 || j >= n) throw std::out_of_range("gen_nystrom: col index out of range");
  if (C_hat.rank_bound() == 0 || R_hat.rank_bound() == 0) return LowRankEstimate::zero(m, n);
  Mat Wleft(d, C_hat.rank_bound());
  for (Index c = 0; c < Wleft.c; ++c)
    for (Index i = 0; i < d; ++i) Wleft(i, c) = C_hat.left()(row_idx[static_cast<std::size_t>(i)], c);
  SvdFactors wf = svd_of_product(Wleft, C_hat.right(), tol);
  if (wf.rank() == 0) return LowRankEstimate::zero(m, n);
  Mat T = gemm(true, false, 1.0, C_hat.right(), wf.V);  // kC x rW
  for (Index c = 0; c < T.c; ++c)
    for (Index i = 0; i < T.r; ++i) T(i, c) /= wf.s[static_cast<std::size_t>(c)];
  Mat left = gemm(false, false, 1.0, C_hat.left(), T);
  Mat T2 = gemm(true, false, 1.0, R_hat.left(), wf.U);   // kR x rW
  Mat right = gemm(false, false, 1.0, R_hat.right(), T2);
  return LowRankEstimate(std::move(left), std::move(right));
}

// average_estimates, sketch.hpp:271-298.
LowRankEstimate average_estimates(const std::vector<LowRankEstimate>& ests, std::optional<Index> recompress_to,
                                  RankTolerance tol) {
  if (ests.empty()) throw std::invalid_argument("average_estimates: empty list");
  const Index m = ests[0].rows(), n = ests[0].cols();
  Index total_k = 0;
  for (const auto& e : ests) {
    if (e.rows() != m || e.cols() != n) throw std::invalid_argument("average_estimates: dimension mismatch");
    total_k += e.rank_bound();
  }
  if (total_k == 0) return LowRankEstimate::zero(m, n);
  Mat left(m, total_k), right(n, total_k);
  const double scale = 1.0 / static_cast<double>(ests.size());
  Index at = 0;
  for (const auto& e : ests) {
    const Index k = e.rank_bound();
    for (Index c = 0; c < k; ++c) {
      for (Index i = 0; i < m; ++i) left(i, at + c) = e.left()(i, c);
      for (Index i = 0; i < n; ++i) right(i, at + c) = e.right()(i, c) * scale;
    }
    at += k;
  }
  if (!recompress_to && total_k <= std::min(m, n)) return LowRankEstimate(std::move(left), std::move(right));
  SvdFactors f = svd_of_product(left, right, tol);
  Index keep = f.rank();
  if (recompress_to) keep = std::min(keep, std::max<Index>(*recompress_to, 0));
  if (keep == 0) return LowRankEstimate::zero(m, n);
  return SvdFactors{f.U.left_cols(keep), std::vector<double>(f.s.begin(), f.s.begin() + keep), f.V.left_cols(keep)}
      .to_estimate();
}

// ================================================================ solvers (P/include/dfc/solvers.hpp)
double default_rmf_lambda(Index m, Index n) { return 1.0 / std::sqrt(static_cast<double>(std::max(m, n))); }

// soft_threshold, solvers.hpp:73-79.
Mat soft_threshold(const Mat& A, double tau) {
  if (tau < 0) throw std::invalid_argument("soft_threshold: tau must be nonnegative");
  Mat out(A.r, A.c);
  for (std::size_t i = 0; i < A.d.size(); ++i) {
    const double a = A.d[i];
    const double mag = std::abs(a) - tau;
    out.d[i] = mag > 0 ? (a > 0 ? mag : -mag) : 0.0;
  }
  return out;
}

namespace detail {

// CSC sparse matrix with the observation pattern (Eigen::SparseMatrix<double> stand-in).
struct Csc {
  Index m = 0, n = 0;
  std::vector<Index> colptr, row;
  std::vector<double> val;
  Mat times(const Mat& X) const {  // S * X
    Mat Y(m, X.c);
    for (Index c = 0; c < X.c; ++c) {
      double* y = Y.col(c);
      const double* x = X.col(c);
      for (Index j = 0; j < n; ++j) {
        const double xj = x[j];
        for (Index e = colptr[static_cast<std::size_t>(j)]; e < colptr[static_cast<std::size_t>(j + 1)]; ++e)
          y[row[static_cast<std::size_t>(e)]] += val[static_cast<std::size_t>(e)] * xj;
      }
    }
    return Y;
  }
  Mat adjoint_times(const Mat& X) const {  // S^T * X
    Mat Y(n, X.c);
    for (Index c = 0; c < X.c; ++c) {
      double* y = Y.col(c);
      const double* x = X.col(c);
      for (Index j = 0; j < n; ++j) {
        double acc = 0.0;
        for (Index e = colptr[static_cast<std::size_t>(j)]; e < colptr[static_cast<std::size_t>(j + 1)]; ++e)
          acc += val[static_cast<std::size_t>(e)] * x[row[static_cast<std::size_t>(e)]];
        y[j] = acc;
      }
    }
    return Y;
  }
  std::vector<double> times_vec(const std::vector<double>& v) const {
    std::vector<double> y(static_cast<std::size_t>(m), 0.0);
    for (Index j = 0; j < n; ++j)
      for (Index e = colptr[static_cast<std::size_t>(j)]; e < colptr[static_cast<std::size_t>(j + 1)]; ++e)
        y[static_cast<std::size_t>(row[static_cast<std::size_t>(e)])] += val[static_cast<std::size_t>(e)] * v[static_cast<std::size_t>(j)];
    return y;
  }
  std::vector<double> adjoint_times_vec(const std::vector<double>& v) const {
    std::vector<double> y(static_cast<std::size_t>(n), 0.0);
    for (Index j = 0; j < n; ++j) {
      double acc = 0.0;
      for (Index e = colptr[static_cast<std::size_t>(j)]; e < colptr[static_cast<std::size_t>(j + 1)]; ++e)
        acc += val[static_cast<std::size_t>(e)] * v[static_cast<std::size_t>(row[static_cast<std::size_t>(e)])];
      y[static_cast<std::size_t>(j)] = acc;
    }
    return y;
  }
};

static double vnorm(const std::vector<double>& v) {
  double s = 0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}

// spectral_norm, solvers.hpp:147-165: alternating power iteration from v = 1/sqrt(n).
template <class MV, class MTV>
double spectral_norm_impl(Index ncols, MV mv, MTV mtv, int max_iters = 200, double tol = 1e-10) {
  std::vector<double> v(static_cast<std::size_t>(ncols), 1.0);
  {
    const double nv = vnorm(v);
    for (double& x : v) x /= nv;
  }
  double s = 0.0, prev = 0.0;
  for (int it = 0; it < max_iters; ++it) {
    std::vector<double> w = mv(v);
    const double nw = vnorm(w);
    if (nw == 0.0) return 0.0;
    for (double& x : w) x /= nw;
    std::vector<double> z = mtv(w);
    s = vnorm(z);
    if (s == 0.0) return 0.0;
    for (std::size_t i = 0; i < z.size(); ++i) v[i] = z[i] / s;
    if (std::abs(s - prev) <= tol * s) break;
    prev = s;
  }
  return s;
}

double spectral_norm(const Csc& S) {
  return spectral_norm_impl(S.n, [&](const std::vector<double>& v) { return S.times_vec(v); },
                            [&](const std::vector<double>& v) { return S.adjoint_times_vec(v); });
}

double spectral_norm(const Mat& A) {
  auto mv = [&](const std::vector<double>& v) {
    std::vector<double> y(static_cast<std::size_t>(A.r), 0.0);
    for (Index j = 0; j < A.c; ++j)
      for (Index i = 0; i < A.r; ++i) y[static_cast<std::size_t>(i)] += A(i, j) * v[static_cast<std::size_t>(j)];
    return y;
  };
  auto mtv = [&](const std::vector<double>& v) {
    std::vector<double> y(static_cast<std::size_t>(A.c), 0.0);
    for (Index j = 0; j < A.c; ++j) {
      double acc = 0;
      for (Index i = 0; i < A.r; ++i) acc += A(i, j) * v[static_cast<std::size_t>(i)];
      y[static_cast<std::size_t>(j)] = acc;
    }
    return y;
  };
  return spectral_norm_impl(A.c, mv, mtv);
}

// shrink_factors, solvers.hpp:83-88.
SvdFactors shrink_factors(const SvdFactors& f, double tau) {
  Index r = 0;
  while (r < f.rank() && f.s[static_cast<std::size_t>(r)] > tau) ++r;
  if (r == 0) return empty_svd(f.U.r, f.V.r);
  std::vector<double> s(f.s.begin(), f.s.begin() + r);
  for (double& x : s) x -= tau;
  return SvdFactors{f.U.left_cols(r), std::move(s), f.V.left_cols(r)};
}

// svt_factors_dense, solvers.hpp:90-93.
SvdFactors svt_factors_dense(const Mat& A, double tau) {
  Svd f = thin_svd(A);
  return shrink_factors(SvdFactors{f.U, f.s, f.V}, tau);
}

struct SvtStats {
  Index k_final = 0;
  int calls = 0;
};

// svt_operator, solvers.hpp:98-109.
template <class Op>
SvdFactors svt_operator(const Op& op, double tau, Index rank_hint, SeededRng& rng, SvtStats* st) {
  const Index minmn = std::min(op.rows(), op.cols());
  st->calls = 0;
  st->k_final = 0;
  if (minmn <= 64) {
    st->calls = 1;
    return svt_factors_dense(op.to_dense(), tau);
  }
  Index k = std::clamp<Index>(rank_hint + 5, 1, minmn);
  for (;;) {
    ++st->calls;
    if (k >= minmn) {
      st->k_final = 0;
      return svt_factors_dense(op.to_dense(), tau);
    }
    st->k_final = k;
    SvdFactors f = partial_svd(op, k, 10, 2, rng);
    if (f.rank() < k || f.s[static_cast<std::size_t>(f.rank() - 1)] <= tau) return shrink_factors(f, tau);
    k = std::min<Index>(2 * k, minmn);
  }
}

// FactoredSparseOp, solvers.hpp:112-136: G = left right^T + s_coeff S.
struct FactoredSparseOp {
  const Mat& left;
  const Mat& right;
  const Csc& S;
  double s_coeff;
  Index rows() const { return left.r; }
  Index cols() const { return right.r; }
  Mat apply(const Mat& X) const {
    Mat Y = S.times(X);
    for (double& v : Y.d) v *= s_coeff;
    if (left.c > 0) {
      Mat T = gemm(true, false, 1.0, right, X);
      gemm_into(false, false, 1.0, left, T, 1.0, Y);
    }
    return Y;
  }
  Mat apply_adjoint(const Mat& X) const {
    Mat Y = S.adjoint_times(X);
    for (double& v : Y.d) v *= s_coeff;
    if (left.c > 0) {
      Mat T = gemm(true, false, 1.0, left, X);
      gemm_into(false, false, 1.0, right, T, 1.0, Y);
    }
    return Y;
  }
  Mat to_dense() const {
    Mat Y(S.m, S.n);
    for (Index j = 0; j < S.n; ++j)
      for (Index e = S.colptr[static_cast<std::size_t>(j)]; e < S.colptr[static_cast<std::size_t>(j + 1)]; ++e)
        Y(S.row[static_cast<std::size_t>(e)], j) = s_coeff * S.val[static_cast<std::size_t>(e)];
    if (left.c > 0) gemm_into(false, true, 1.0, left, right, 1.0, Y);
    return Y;
  }
};

// DenseOp, solvers.hpp:138-145.
struct DenseOp {
  const Mat& A;
  Index rows() const { return A.r; }
  Index cols() const { return A.c; }
  Mat apply(const Mat& X) const { return gemm(false, false, 1.0, A, X); }
  Mat apply_adjoint(const Mat& X) const { return gemm(true, false, 1.0, A, X); }
  Mat to_dense() const { return A; }
};

// validate_config, solvers.hpp:167-177.
void validate_config(const ApgConfig& cfg) {
  if (cfg.max_iters < 1) throw std::invalid_argument("ApgConfig: max_iters must be >= 1");
  if (!(cfg.rel_tol > 0 && cfg.rel_tol < 1)) throw std::invalid_argument("ApgConfig: rel_tol must be in (0,1)");
  if (!(cfg.mu_decay > 0 && cfg.mu_decay < 1)) throw std::invalid_argument("ApgConfig: mu_decay must be in (0,1)");
  if (cfg.mu_init && *cfg.mu_init < 0) throw std::invalid_argument("ApgConfig: mu_init < 0");
  if (cfg.mu_floor && *cfg.mu_floor < 0) throw std::invalid_argument("ApgConfig: mu_floor < 0");
  if (cfg.mu_init && cfg.mu_floor && *cfg.mu_floor > *cfg.mu_init)
    throw std::invalid_argument("ApgConfig: mu_floor exceeds mu_init");
}

// extrapolate, solvers.hpp:196-212.
LowRankEstimate extrapolate(const LowRankEstimate& curr, const LowRankEstimate& prev, double beta) {
  if (beta == 0.0 || prev.rank_bound() == 0) {
    if (curr.rank_bound() == 0) return curr;
    Mat r = curr.right();
    for (double& v : r.d) v *= (1.0 + beta);
    return LowRankEstimate(curr.left(), std::move(r));
  }
  const Index m = curr.rows(), n = curr.cols();
  const Index kc = curr.rank_bound(), kp = prev.rank_bound();
  Mat left(m, kc + kp), right(n, kc + kp);
  std::copy(curr.left().d.begin(), curr.left().d.end(), left.d.begin());
  std::copy(prev.left().d.begin(), prev.left().d.end(), left.d.begin() + m * kc);
  for (std::size_t i = 0; i < curr.right().d.size(); ++i) right.d[i] = (1.0 + beta) * curr.right().d[i];
  for (std::size_t i = 0; i < prev.right().d.size(); ++i)
    right.d[static_cast<std::size_t>(n * kc) + i] = -beta * prev.right().d[i];
  if (kc + kp > std::min(m, n)) return svd_of_product(left, right).to_estimate();
  return LowRankEstimate(std::move(left), std::move(right));
}

// eval_on_support, solvers.hpp:215-225.
std::vector<double> eval_on_support(const LowRankEstimate& est, const std::vector<Observation>& entries) {
  std::vector<double> v(entries.size(), 0.0);
  if (est.rank_bound() == 0) return v;
  for (std::size_t i = 0; i < entries.size(); ++i) v[i] = row_dot(est.left(), entries[i].row, est.right(), entries[i].col);
  return v;
}

double factored_norm(const LowRankEstimate& a) { return std::sqrt(std::max(0.0, factored_inner(a, a))); }

}  // namespace detail

// factored_inner / factored_diff_norm, solvers.hpp:179-193.
double factored_inner(const LowRankEstimate& a, const LowRankEstimate& b) {
  if (a.rank_bound() == 0 || b.rank_bound() == 0) return 0.0;
  Mat L = gemm(true, false, 1.0, a.left(), b.left());
  Mat R = gemm(true, false, 1.0, a.right(), b.right());
  double s = 0.0;
  for (std::size_t i = 0; i < L.d.size(); ++i) s += L.d[i] * R.d[i];
  return s;
}

double factored_diff_norm(const LowRankEstimate& a, const LowRankEstimate& b) {
  const double d2 = factored_inner(a, a) - 2.0 * factored_inner(a, b) + factored_inner(b, b);
  return std::sqrt(std::max(0.0, d2));
}

// svt, solvers.hpp:230-233.
LowRankEstimate svt(const Mat& A, double tau) {
  if (tau < 0) throw std::invalid_argument("svt: tau must be nonnegative");
  return detail::svt_factors_dense(A, tau).to_estimate();
}

static double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

static double sum_of(const std::vector<double>& v) {
  double s = 0;
  for (double x : v) s += x;
  return s;
}

// apg_mc, solvers.hpp:241-327, as a resumable run (setup in the ctor, one APG iteration per
// step(), report in finish()); apg_mc() drives it to completion exactly like the reference loop.
ApgMcRun::ApgMcRun(const ObservedMatrix& obs_, const ApgConfig& cfg_)
    : obs(obs_), cfg(cfg_), svd_rng(0x737674u, 0), L_prev(LowRankEstimate::zero(1, 1)),
      L_curr(LowRankEstimate::zero(1, 1)) {
  start = std::chrono::steady_clock::now();
  if (obs.empty()) throw std::invalid_argument("apg_mc: empty observation set");
  detail::validate_config(cfg);
  const Index m = obs.rows(), n = obs.cols(), N = obs.count();
  M = std::make_unique<detail::Csc>();
  M->m = m;
  M->n = n;
  M->colptr.assign(static_cast<std::size_t>(n + 1), 0);
  M->row.resize(static_cast<std::size_t>(N));
  M->val.resize(static_cast<std::size_t>(N));
  for (Index e = 0; e < N; ++e) {
    const auto& o = obs.entries()[static_cast<std::size_t>(e)];
    M->colptr[static_cast<std::size_t>(o.col + 1)]++;
    M->row[static_cast<std::size_t>(e)] = o.row;
    M->val[static_cast<std::size_t>(e)] = o.value;
  }
  for (Index j = 0; j < n; ++j) M->colptr[static_cast<std::size_t>(j + 1)] += M->colptr[static_cast<std::size_t>(j)];
  m_vals = M->val;
  mu_init = cfg.mu_init.value_or(0.99 * detail::spectral_norm(*M));
  mu_floor = cfg.mu_floor.value_or(1e-4 * mu_init);
  if (mu_floor > mu_init) throw std::invalid_argument("apg_mc: mu_floor exceeds mu_init");
  R = std::make_unique<detail::Csc>(*M);
  L_prev = LowRankEstimate::zero(m, n);
  L_curr = L_prev;
  last = empty_svd(m, n);
  mu = mu_used = mu_init;
}

ApgMcRun::~ApgMcRun() = default;

bool ApgMcRun::step(std::vector<IterTrace>* trace) {
  if (stopped || iters >= cfg.max_iters) return false;
  const Index m = obs.rows(), n = obs.cols(), N = obs.count();
  const int it = ++iters;
  const double beta = (tau_prev - 1.0) / tau_curr;
  LowRankEstimate Y = detail::extrapolate(L_curr, L_prev, beta);
  std::vector<double> y_vals = detail::eval_on_support(Y, obs.entries());
  for (Index i = 0; i < N; ++i)
    R->val[static_cast<std::size_t>(i)] = y_vals[static_cast<std::size_t>(i)] - m_vals[static_cast<std::size_t>(i)];

  double step = 1.0;
  SvdFactors f;
  LowRankEstimate L_next = LowRankEstimate::zero(m, n);
  detail::SvtStats st;
  for (;;) {
    detail::FactoredSparseOp G{Y.left(), Y.right(), *R, -step};
    f = detail::svt_operator(G, step * mu, rank_hint, svd_rng, &st);
    L_next = f.to_estimate();
    if (!cfg.line_search || step <= 0.125) break;
    std::vector<double> nv = detail::eval_on_support(L_next, obs.entries());
    double f_next = 0, f_y = 0, lin = 0;
    for (Index i = 0; i < N; ++i) {
      const std::size_t u = static_cast<std::size_t>(i);
      f_next += (nv[u] - m_vals[u]) * (nv[u] - m_vals[u]);
      f_y += (y_vals[u] - m_vals[u]) * (y_vals[u] - m_vals[u]);
      lin += (y_vals[u] - m_vals[u]) * (nv[u] - y_vals[u]);
    }
    f_next *= 0.5;
    f_y *= 0.5;
    const double dist2 = factored_diff_norm(L_next, Y);
    if (f_next <= f_y + lin + dist2 * dist2 / (2.0 * step) + 1e-12) break;
    step *= 0.5;
  }
  const double rel = factored_diff_norm(L_next, L_curr) / std::max(1.0, detail::factored_norm(L_curr));
  const double tau_next = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * tau_curr * tau_curr));
  L_prev = std::move(L_curr);
  L_curr = std::move(L_next);
  last = std::move(f);
  tau_prev = tau_curr;
  tau_curr = tau_next;
  rank_hint = std::max<Index>(1, L_curr.rank_bound());
  mu_used = mu;
  if (trace) trace->push_back({it, L_curr.rank_bound(), st.k_final, st.calls, rel, mu, sum_of(last.s)});
  mu = std::max(cfg.mu_decay * mu, mu_floor);
  if (rel < cfg.rel_tol) stopped = true;
  return true;
}

std::pair<LowRankEstimate, SolveReport> ApgMcRun::finish() const {
  const Index N = obs.count();
  SolveReport rep;
  rep.iterations = iters;
  rep.rank = L_curr.rank_bound();
  std::vector<double> fv = detail::eval_on_support(L_curr, obs.entries());
  double res2 = 0;
  for (Index i = 0; i < N; ++i) {
    const double d = fv[static_cast<std::size_t>(i)] - m_vals[static_cast<std::size_t>(i)];
    res2 += d * d;
  }
  rep.residual = std::sqrt(res2);
  rep.objective = mu_used * sum_of(last.s) + 0.5 * rep.residual * rep.residual;
  rep.wall_ms = ms_since(start);
  return {L_curr, rep};
}

std::pair<LowRankEstimate, SolveReport> apg_mc(const ObservedMatrix& obs, const ApgConfig& cfg,
                                               std::vector<IterTrace>* trace) {
  ApgMcRun run(obs, cfg);
  while (run.step(trace)) {
  }
  return run.finish();
}

// apg_rmf, solvers.hpp:332-414.
std::tuple<LowRankEstimate, OutlierEstimate, SolveReport> apg_rmf(const Mat& Mfull, double lambda, const ApgConfig& cfg,
                                                                  std::vector<IterTrace>* trace) {
  const auto start = std::chrono::steady_clock::now();
  if (!(lambda > 0)) throw std::invalid_argument("apg_rmf: lambda must be positive");
  if (!Mfull.all_finite()) throw std::invalid_argument("apg_rmf: non-finite input");
  detail::validate_config(cfg);
  const Index m = Mfull.r, n = Mfull.c;
  const std::size_t mn = Mfull.d.size();

  const double mu_init = cfg.mu_init.value_or(0.99 * detail::spectral_norm(Mfull));
  const double mu_floor = cfg.mu_floor.value_or(1e-4 * mu_init);
  if (mu_floor > mu_init) throw std::invalid_argument("apg_rmf: mu_floor exceeds mu_init");

  SeededRng svd_rng(0x737674u, 1);
  SvdFactors last = empty_svd(m, n);
  Mat Ld_prev(m, n), Ld_curr(m, n), S_prev(m, n), S_curr(m, n);
  double tau_prev = 1.0, tau_curr = 1.0, mu = mu_init, mu_used = mu_init;
  Index rank_hint = 1;
  int iters = 0;

  for (int it = 1; it <= cfg.max_iters; ++it) {
    iters = it;
    const double beta = (tau_prev - 1.0) / tau_curr;
    Mat YL(m, n), YS(m, n), g(m, n);
    for (std::size_t i = 0; i < mn; ++i) {
      YL.d[i] = Ld_curr.d[i] + beta * (Ld_curr.d[i] - Ld_prev.d[i]);
      YS.d[i] = S_curr.d[i] + beta * (S_curr.d[i] - S_prev.d[i]);
      g.d[i] = YL.d[i] + YS.d[i] - Mfull.d[i];
    }
    double step = 0.5;
    SvdFactors f;
    Mat Ld_next, S_next;
    detail::SvtStats st;
    for (;;) {
      Mat GL(m, n), YSg(m, n);
      for (std::size_t i = 0; i < mn; ++i) {
        GL.d[i] = YL.d[i] - step * g.d[i];
        YSg.d[i] = YS.d[i] - step * g.d[i];
      }
      f = detail::svt_operator(detail::DenseOp{GL}, step * mu, rank_hint, svd_rng, &st);
      if (f.rank() == 0) {
        Ld_next = Mat(m, n);
      } else {
        Mat Us = f.U;
        for (Index c = 0; c < Us.c; ++c)
          for (Index i = 0; i < m; ++i) Us(i, c) *= f.s[static_cast<std::size_t>(c)];
        Ld_next = gemm(false, true, 1.0, Us, f.V);
      }
      S_next = soft_threshold(YSg, step * lambda * mu);
      if (!cfg.line_search || step <= 0.0625) break;
      double f_next = 0, f_y = 0, lin = 0, dist2 = 0;
      for (std::size_t i = 0; i < mn; ++i) {
        const double r = Mfull.d[i] - Ld_next.d[i] - S_next.d[i];
        f_next += r * r;
        f_y += g.d[i] * g.d[i];
        lin += g.d[i] * (Ld_next.d[i] - YL.d[i] + S_next.d[i] - YS.d[i]);
        dist2 += (Ld_next.d[i] - YL.d[i]) * (Ld_next.d[i] - YL.d[i]) + (S_next.d[i] - YS.d[i]) * (S_next.d[i] - YS.d[i]);
      }
      if (0.5 * f_next <= 0.5 * f_y + lin + dist2 / (2.0 * step) + 1e-12) break;
      step *= 0.5;
    }
    double dL = 0, dS = 0, nL = 0, nS = 0;
    for (std::size_t i = 0; i < mn; ++i) {
      dL += (Ld_next.d[i] - Ld_curr.d[i]) * (Ld_next.d[i] - Ld_curr.d[i]);
      dS += (S_next.d[i] - S_curr.d[i]) * (S_next.d[i] - S_curr.d[i]);
      nL += Ld_curr.d[i] * Ld_curr.d[i];
      nS += S_curr.d[i] * S_curr.d[i];
    }
    const double denom = std::max(1.0, std::sqrt(nL + nS));
    const double rel = std::sqrt(dL + dS) / denom;
    const double tau_next = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * tau_curr * tau_curr));
    Ld_prev = std::move(Ld_curr);
    Ld_curr = std::move(Ld_next);
    S_prev = std::move(S_curr);
    S_curr = std::move(S_next);
    last = std::move(f);
    tau_prev = tau_curr;
    tau_curr = tau_next;
    rank_hint = std::max<Index>(1, last.rank());
    mu_used = mu;
    if (trace) trace->push_back({it, last.rank(), st.k_final, st.calls, rel, mu, sum_of(last.s)});
    mu = std::max(cfg.mu_decay * mu, mu_floor);
    if (rel < cfg.rel_tol) break;
  }

  LowRankEstimate L = last.to_estimate();
  std::vector<Observation> s_entries;
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < m; ++i)
      if (S_curr(i, j) != 0.0) s_entries.push_back({i, j, S_curr(i, j)});
  OutlierEstimate S(m, n, std::move(s_entries));

  SolveReport rep;
  rep.iterations = iters;
  rep.rank = L.rank_bound();
  double res2 = 0, l1 = 0;
  for (std::size_t i = 0; i < mn; ++i) {
    const double r = Mfull.d[i] - Ld_curr.d[i] - S_curr.d[i];
    res2 += r * r;
    l1 += std::abs(S_curr.d[i]);
  }
  rep.residual = std::sqrt(res2);
  rep.objective = sum_of(last.s) + lambda * l1 + (mu_used > 0 ? rep.residual * rep.residual / (2.0 * mu_used) : 0.0);
  rep.wall_ms = ms_since(start);
  return {std::move(L), std::move(S), rep};
}

// ================================================================ orchestrator (P/include/dfc/dfc.hpp)
// make_base_solver, dfc.hpp:70-78.
BaseSolver make_base_solver(Task task, const ApgConfig& cfg, double lambda) {
  if (task == Task::MC) return [cfg](const ObservedMatrix& block) { return apg_mc(block, cfg); };
  return [cfg, lambda](const ObservedMatrix& block) {
    const double lam = lambda > 0 ? lambda : default_rmf_lambda(block.rows(), block.cols());
    auto [L, S, rep] = apg_rmf(densify(block), lam, cfg);
    return std::pair<LowRankEstimate, SolveReport>{std::move(L), rep};
  };
}

namespace detail {

// parallel_for, dfc.hpp:84-119: lowest-index failure wins.
template <class Fn>
void parallel_for(std::size_t count, int workers, Fn&& fn) {
  if (workers < 1) throw std::invalid_argument("parallel_for: workers must be >= 1");
  const std::size_t nthreads = std::min<std::size_t>(static_cast<std::size_t>(workers), count);
  std::vector<std::string> failures(count);
  std::vector<char> failed(count, 0);
  if (nthreads <= 1) {
    for (std::size_t i = 0; i < count; ++i) {
      try {
        fn(i);
      } catch (const std::exception& e) {
        throw BlockError(i, e.what());
      }
    }
    return;
  }
  std::atomic<std::size_t> next{0};
  auto worker = [&]() {
    for (;;) {
      const std::size_t i = next.fetch_add(1);
      if (i >= count) return;
      try {
        fn(i);
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

// solve_blocks, dfc.hpp:133-147: empty blocks get a zero estimate and no solver call.
void solve_blocks(const std::vector<ObservedMatrix>& blocks, const BaseSolver& solver, int workers,
                  std::vector<LowRankEstimate>& ests, std::vector<SolveReport>& reports) {
  ests.assign(blocks.size(), LowRankEstimate::zero(1, 1));
  reports.assign(blocks.size(), SolveReport{});
  parallel_for(blocks.size(), workers, [&](std::size_t i) {
    if (blocks[i].empty()) {
      ests[i] = LowRankEstimate::zero(blocks[i].rows(), blocks[i].cols());
      return;
    }
    auto [est, rep] = solver(blocks[i]);
    ests[i] = std::move(est);
    reports[i] = rep;
  });
}

std::vector<Index> block_ranks(const std::vector<LowRankEstimate>& ests) {
  std::vector<Index> r;
  for (const auto& e : ests) r.push_back(e.rank_bound());
  return r;
}

}  // namespace detail

// median_rank, dfc.hpp:159-164.
Index median_rank(const std::vector<Index>& ranks) {
  if (ranks.empty()) throw std::invalid_argument("median_rank: empty list");
  std::vector<Index> sorted = ranks;
  std::sort(sorted.begin(), sorted.end());
  return std::max<Index>(1, sorted[(sorted.size() - 1) / 2]);
}

// dfc_proj, dfc.hpp:166-200.
std::pair<LowRankEstimate, DfcReport> dfc_proj(const ObservedMatrix& obs, const DfcConfig& cfg, const BaseSolver& solver) {
  if (cfg.variant != DfcVariant::Proj) throw std::invalid_argument("dfc_proj: wrong variant");
  if (cfg.t < 1 || cfg.t > obs.cols()) throw std::invalid_argument("dfc_proj: need 1 <= t <= n");
  if (cfg.ensemble_anchors < 0) throw std::invalid_argument("dfc_proj: ensemble_anchors must be >= 0");
  if (cfg.ensemble_anchors > 0 && !cfg.ensemble)
    throw std::invalid_argument("dfc_proj: ensemble_anchors needs ensemble = true");
  DfcReport report;
  detail::PhaseClock total, phase;
  SeededRng prng(cfg.seed, streams::partition);
  PartitionPlan plan = partition_columns(obs.cols(), cfg.t, prng);
  std::vector<ObservedMatrix> blocks;
  for (std::size_t g = 0; g < plan.group_count(); ++g) blocks.push_back(extract_columns(obs, plan.group(g)));
  report.divide_ms = phase.lap();
  std::vector<LowRankEstimate> ests;
  detail::solve_blocks(blocks, solver, cfg.workers, ests, report.subproblems);
  report.factor_ms = phase.lap();
  LowRankEstimate out = LowRankEstimate::zero(obs.rows(), obs.cols());
  if (!cfg.ensemble) {
    out = column_project(ests[0], ests, plan);
  } else {
    // extension: the first `ensemble_anchors` plan groups anchor the ensemble (0 = all t, the
    // reference's dfc.hpp:191-195); the recompression target stays the median of ALL block ranks
    const std::size_t anchors = cfg.ensemble_anchors > 0
                                    ? std::min<std::size_t>(static_cast<std::size_t>(cfg.ensemble_anchors), ests.size())
                                    : ests.size();
    std::vector<LowRankEstimate> projected(anchors, LowRankEstimate::zero(1, 1));
    detail::parallel_for(anchors, cfg.workers, [&](std::size_t i) { projected[i] = column_project(ests[i], ests, plan); });
    out = average_estimates(projected, median_rank(detail::block_ranks(ests)));
  }
  report.combine_ms = phase.lap();
  report.total_ms = total.lap();
  return {std::move(out), std::move(report)};
}

// dfc_rp, dfc.hpp:202-248.
std::pair<LowRankEstimate, DfcReport> dfc_rp(const ObservedMatrix& obs, const DfcConfig& cfg, const BaseSolver& solver) {
  if (cfg.variant != DfcVariant::Rp) throw std::invalid_argument("dfc_rp: wrong variant");
  if (cfg.t < 1 || cfg.t > obs.cols()) throw std::invalid_argument("dfc_rp: need 1 <= t <= n");
  DfcReport report;
  detail::PhaseClock total, phase;
  SeededRng prng(cfg.seed, streams::partition);
  PartitionPlan plan = partition_columns(obs.cols(), cfg.t, prng);
  std::vector<ObservedMatrix> blocks;
  for (std::size_t g = 0; g < plan.group_count(); ++g) blocks.push_back(extract_columns(obs, plan.group(g)));
  report.divide_ms = phase.lap();
  std::vector<LowRankEstimate> ests;
  detail::solve_blocks(blocks, solver, cfg.workers, ests, report.subproblems);
  report.factor_ms = phase.lap();
  RpParams params = cfg.rp;
  params.k = median_rank(detail::block_ranks(ests));
  const Index minmn = std::min(obs.rows(), obs.cols());
  if (params.k + params.p > minmn) {
    report.k_clamped = true;
    params.p = std::min(params.p, minmn - 1);
    params.k = minmn - params.p;
  }
  report.chosen_k = params.k;
  LowRankEstimate out = LowRankEstimate::zero(obs.rows(), obs.cols());
  if (!cfg.ensemble) {
    SeededRng rng(cfg.seed, streams::rp_draw);
    out = random_project(ests, plan, params, rng);
  } else {
    std::vector<LowRankEstimate> draws(static_cast<std::size_t>(cfg.t), LowRankEstimate::zero(1, 1));
    detail::parallel_for(draws.size(), cfg.workers, [&](std::size_t i) {
      SeededRng rng(cfg.seed, streams::rp_draw + 1 + i);
      draws[i] = random_project(ests, plan, params, rng);
    });
    out = average_estimates(draws, params.k);
  }
  report.combine_ms = phase.lap();
  report.total_ms = total.lap();
  return {std::move(out), std::move(report)};
}

// dfc_nys, dfc.hpp:250-324.
std::pair<LowRankEstimate, DfcReport> dfc_nys(const ObservedMatrix& obs, const DfcConfig& cfg, const BaseSolver& solver) {
  if (cfg.variant != DfcVariant::Nys) throw std::invalid_argument("dfc_nys: wrong variant");
  const Index m = obs.rows(), n = obs.cols();
  if (cfg.l < 1 || cfg.l > n) throw std::invalid_argument("dfc_nys: need 1 <= l <= n");
  if (cfg.d < 1 || cfg.d > m) throw std::invalid_argument("dfc_nys: need 1 <= d <= m");
  DfcReport report;
  detail::PhaseClock total, phase;
  SeededRng row_rng(cfg.seed, streams::nys_rows);
  std::vector<Index> row_idx = sample_without_replacement(m, cfg.d, row_rng);
  std::sort(row_idx.begin(), row_idx.end());
  auto finish = [&](LowRankEstimate out) {
    report.combine_ms = phase.lap();
    report.total_ms = total.lap();
    return std::pair<LowRankEstimate, DfcReport>{std::move(out), std::move(report)};
  };
  auto pair_deficient = [&](const LowRankEstimate& C_hat, const LowRankEstimate& R_hat) {
    const Index kmax = std::max(C_hat.rank_bound(), R_hat.rank_bound());
    if (kmax == 0 || C_hat.rank_bound() == 0) return kmax > 0;
    Mat Wleft(static_cast<Index>(row_idx.size()), C_hat.rank_bound());
    for (Index c = 0; c < Wleft.c; ++c)
      for (std::size_t i = 0; i < row_idx.size(); ++i) Wleft(static_cast<Index>(i), c) = C_hat.left()(row_idx[i], c);
    return svd_of_product(Wleft, C_hat.right()).rank() < kmax;
  };
  if (!cfg.ensemble) {
    SeededRng col_rng(cfg.seed, streams::nys_cols);
    std::vector<Index> col_idx = sample_without_replacement(n, cfg.l, col_rng);
    std::sort(col_idx.begin(), col_idx.end());
    std::vector<ObservedMatrix> blocks{extract_columns(obs, col_idx), extract_rows(obs, row_idx)};
    report.divide_ms = phase.lap();
    std::vector<LowRankEstimate> ests;
    detail::solve_blocks(blocks, solver, cfg.workers, ests, report.subproblems);
    report.factor_ms = phase.lap();
    report.rank_deficient = pair_deficient(ests[0], ests[1]);
    return finish(gen_nystrom(ests[0], ests[1], row_idx, col_idx));
  }
  const Index groups =
      std::clamp<Index>(static_cast<Index>(std::llround(static_cast<double>(n) / static_cast<double>(cfg.l))), 1, n);
  SeededRng prng(cfg.seed, streams::partition);
  PartitionPlan plan = partition_columns(n, groups, prng);
  std::vector<ObservedMatrix> blocks;
  for (std::size_t g = 0; g < plan.group_count(); ++g) blocks.push_back(extract_columns(obs, plan.group(g)));
  blocks.push_back(extract_rows(obs, row_idx));
  report.divide_ms = phase.lap();
  std::vector<LowRankEstimate> ests;
  detail::solve_blocks(blocks, solver, cfg.workers, ests, report.subproblems);
  report.factor_ms = phase.lap();
  const LowRankEstimate& R_hat = ests.back();
  std::vector<LowRankEstimate> col_ests(ests.begin(), ests.end() - 1);
  std::vector<LowRankEstimate> combined(col_ests.size(), LowRankEstimate::zero(1, 1));
  std::vector<char> deficient(col_ests.size(), 0);
  detail::parallel_for(col_ests.size(), cfg.workers, [&](std::size_t i) {
    deficient[i] = pair_deficient(col_ests[i], R_hat) ? 1 : 0;
    combined[i] = gen_nystrom(col_ests[i], R_hat, row_idx, plan.group(i));
  });
  for (char f : deficient) report.rank_deficient = report.rank_deficient || f;
  return finish(average_estimates(combined, median_rank(detail::block_ranks(col_ests))));
}

// dfc_run, dfc.hpp:326-335.
std::pair<LowRankEstimate, DfcReport> dfc_run(const ObservedMatrix& obs, const DfcConfig& cfg) {
  const BaseSolver solver = make_base_solver(cfg.task, cfg.solver_cfg, cfg.lambda);
  switch (cfg.variant) {
    case DfcVariant::Proj: return dfc_proj(obs, cfg, solver);
    case DfcVariant::Rp: return dfc_rp(obs, cfg, solver);
    case DfcVariant::Nys: return dfc_nys(obs, cfg, solver);
  }
  throw std::logic_error("dfc_run: unknown variant");
}

}  // namespace orc
