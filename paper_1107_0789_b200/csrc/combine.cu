// C-step combiners on the device (P/include/dfc/sketch.hpp):
//   svd_of_product (:73-86), column_project (:170-199, DFC-Proj), gen_nystrom (:241-266,
//   DFC-Nys), average_estimates (:271-298, ensembles), random_project + BlocksOp
//   (:99-131, 204-237, DFC-RP). All contractions are FP64 DMMA GEMMs (dense.cu); the
//   factorizations are thin_qr / thin_svd (factor.cu).
#include <algorithm>
#include <cmath>

#include "solver.hpp"

namespace dfcg {

namespace {

int grid_for(i64 total, int threads = 256) {
  return static_cast<int>(std::max<i64>(1, std::min<i64>((total + threads - 1) / threads, 4096)));
}

// dst[p, :] = src[idx[p], :]  (l rows of width c)
__global__ void gather_rows_kernel(i64 l, i64 c, const double* __restrict__ src, i64 lds,
                                   const long long* __restrict__ idx, double* __restrict__ dst, i64 ldd) {
  const i64 total = l * c;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 p = e / c, j = e % c;
    dst[p * ldd + j] = src[idx[p] * lds + j];
  }
}

// dst[idx[p], :] = src[p, :]
__global__ void scatter_rows_kernel(i64 l, i64 c, const double* __restrict__ src, i64 lds,
                                    const long long* __restrict__ idx, double* __restrict__ dst, i64 ldd) {
  const i64 total = l * c;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 p = e / c, j = e % c;
    dst[idx[p] * ldd + j] = src[p * lds + j];
  }
}

__global__ void scale_cols_kernel(i64 rows, i64 cols, double* A, i64 lda, const double* __restrict__ scale,
                                  int invert) {
  const i64 total = rows * cols;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 r = e / cols, c = e % cols;
    A[r * lda + c] = invert ? A[r * lda + c] / scale[c] : A[r * lda + c] * scale[c];
  }
}

DBuf<long long> upload_idx(cudaStream_t s, const std::vector<i64>& v) {
  DBuf<long long> d(std::max<size_t>(1, v.size()), s);
  if (!v.empty())
    DFCG_CUDA(cudaMemcpyAsync(d.get(), v.data(), sizeof(long long) * v.size(), cudaMemcpyHostToDevice, s));
  DFCG_CUDA(cudaStreamSynchronize(s));
  return d;
}

DBuf<double> upload_vec(cudaStream_t s, const std::vector<double>& v) {
  DBuf<double> d(std::max<size_t>(1, v.size()), s);
  if (!v.empty())
    DFCG_CUDA(cudaMemcpyAsync(d.get(), v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice, s));
  DFCG_CUDA(cudaStreamSynchronize(s));
  return d;
}

i64 numerical_rank(const std::vector<double>& s, i64 m, i64 n, double rel_cutoff) {
  if (s.empty()) return 0;
  const double cut = rel_cutoff * static_cast<double>(std::max(m, n)) * s[0];
  i64 r = 0;
  while (r < static_cast<i64>(s.size()) && s[static_cast<size_t>(r)] > cut) ++r;
  return r;
}

// Thin QR that also accepts wide inputs: for rows <= cols the orthonormal factor is the
// identity of R^rows and R = A (Eigen's thin_qr returns Q rows x rows, R rows x cols; only
// span(Q) and Q R = A are used by svd_of_product).
struct QrOut {
  i64 r = 0;          // number of Q columns
  bool identity = false;
  DBuf<double> Q, R;  // rows x r, r x cols (row-major)
};
QrOut general_qr(cudaStream_t s, i64 rows, i64 cols, const double* A) {
  QrOut o;
  if (rows <= cols) {
    o.r = rows;
    o.identity = true;
    o.R.alloc(rows * cols, s);
    copy2d(s, rows, cols, A, cols, o.R.get(), cols);
    return o;
  }
  o.r = cols;
  o.Q.alloc(rows * cols, s);
  o.R.alloc(cols * cols, s);
  copy2d(s, rows, cols, A, cols, o.Q.get(), cols);
  thin_qr(s, rows, cols, o.Q.get(), cols, o.R.get(), cols);
  return o;
}

// Thin SVD of a general (possibly wide) matrix; U rows x p, V cols x p, p = min(rows, cols).
void general_svd(cudaStream_t s, i64 rows, i64 cols, const double* A, DBuf<double>& U, DBuf<double>& V,
                 std::vector<double>& sv) {
  const i64 p = std::min(rows, cols);
  U.alloc(rows * p, s);
  V.alloc(cols * p, s);
  if (rows >= cols) {
    DBuf<double> W(rows * cols, s);
    copy2d(s, rows, cols, A, cols, W.get(), cols);
    thin_svd(s, rows, cols, W.get(), cols, U.get(), p, V.get(), p, sv);
  } else {
    DBuf<double> W(cols * rows, s);
    transpose(s, rows, cols, A, cols, W.get(), rows);
    thin_svd(s, cols, rows, W.get(), rows, V.get(), p, U.get(), p, sv);
  }
}

// BlocksOp (sketch.hpp:99-131): the column-blocked factored matrix [C_1 ... C_t].
struct BlocksOp {
  const std::vector<const DevLowRank*>& blocks;
  const std::vector<DBuf<long long>>& idx;
  const std::vector<std::vector<i64>>& groups;
  i64 m, n;
  void apply(cudaStream_t s, const double* X, i64 b, double* Y) const {  // X n x b -> Y m x b
    DFCG_CUDA(cudaMemsetAsync(Y, 0, sizeof(double) * m * b, s));
    for (size_t g = 0; g < blocks.size(); ++g) {
      const DevLowRank& B = *blocks[g];
      if (B.k == 0) continue;
      const i64 w = static_cast<i64>(groups[g].size());
      DBuf<double> Xg(w * b, s), T(B.k * b, s);
      gather_rows_kernel<<<grid_for(w * b), 256, 0, s>>>(w, b, X, b, idx[g].get(), Xg.get(), b);
      DFCG_LAUNCH_CHECK();
      gemm(s, true, false, B.k, b, w, 1.0, B.right.get(), B.k, Xg.get(), b, 0.0, T.get(), b);
      gemm(s, false, false, m, b, B.k, 1.0, B.left.get(), B.k, T.get(), b, 1.0, Y, b);
    }
  }
  void apply_adjoint(cudaStream_t s, const double* X, i64 b, double* Y) const {  // X m x b -> Y n x b
    DFCG_CUDA(cudaMemsetAsync(Y, 0, sizeof(double) * n * b, s));
    for (size_t g = 0; g < blocks.size(); ++g) {
      const DevLowRank& B = *blocks[g];
      if (B.k == 0) continue;
      const i64 w = static_cast<i64>(groups[g].size());
      DBuf<double> T(B.k * b, s), Yg(w * b, s);
      gemm(s, true, false, B.k, b, m, 1.0, B.left.get(), B.k, X, b, 0.0, T.get(), b);
      gemm(s, false, false, w, b, B.k, 1.0, B.right.get(), B.k, T.get(), b, 0.0, Yg.get(), b);
      scatter_rows_kernel<<<grid_for(w * b), 256, 0, s>>>(w, b, Yg.get(), b, idx[g].get(), Y, b);
      DFCG_LAUNCH_CHECK();
    }
  }
};

}  // namespace

// svd_of_product (sketch.hpp:73-86): QR both factors, SVD of Rl Rr^T, truncate at the
// numerical rank 1e-12 * max(m, n) * s_max.
SvdOfProduct svd_of_product(cudaStream_t s, i64 m, i64 n, i64 k, const double* left, const double* right,
                            double rel_cutoff) {
  SvdOfProduct out;
  out.est.m = m;
  out.est.n = n;
  if (k == 0) return out;
  QrOut ql = general_qr(s, m, k, left);
  QrOut qr = general_qr(s, n, k, right);
  DBuf<double> core(ql.r * qr.r, s);
  gemm(s, false, true, ql.r, qr.r, k, 1.0, ql.R.get(), k, qr.R.get(), k, 0.0, core.get(), qr.r);
  DBuf<double> Uc, Vc;
  std::vector<double> sv;
  general_svd(s, ql.r, qr.r, core.get(), Uc, Vc, sv);
  const i64 p = std::min(ql.r, qr.r);
  const i64 r = numerical_rank(sv, m, n, rel_cutoff);
  out.r = r;
  out.s.assign(sv.begin(), sv.begin() + r);
  if (r == 0) return out;
  out.U.alloc(m * r, s);
  out.V.alloc(n * r, s);
  if (ql.identity) copy2d(s, m, r, Uc.get(), p, out.U.get(), r);
  else gemm(s, false, false, m, r, ql.r, 1.0, ql.Q.get(), ql.r, Uc.get(), p, 0.0, out.U.get(), r);
  if (qr.identity) copy2d(s, n, r, Vc.get(), p, out.V.get(), r);
  else gemm(s, false, false, n, r, qr.r, 1.0, qr.Q.get(), qr.r, Vc.get(), p, 0.0, out.V.get(), r);
  // est = to_estimate(): (U, V diag(s))
  out.est.k = r;
  out.est.left.alloc(m * r, s);
  out.est.right.alloc(n * r, s);
  copy2d(s, m, r, out.U.get(), r, out.est.left.get(), r);
  copy2d(s, n, r, out.V.get(), r, out.est.right.get(), r);
  DBuf<double> ds = upload_vec(s, out.s);
  scale_cols_kernel<<<grid_for(n * r), 256, 0, s>>>(n, r, out.est.right.get(), r, ds.get(), 0);
  DFCG_LAUNCH_CHECK();
  DFCG_CUDA(cudaStreamSynchronize(s));
  return out;
}

// column_project (sketch.hpp:170-199): U_b U_b^T [C_1 ... C_t], original column order.
void column_project(cudaStream_t s, const DevLowRank& basis, const std::vector<const DevLowRank*>& blocks,
                    const std::vector<std::vector<i64>>& groups, i64 n, DevLowRank& out) {
  if (blocks.empty()) throw std::invalid_argument("column_project: no blocks");
  if (blocks.size() != groups.size()) throw std::invalid_argument("column_project: block count does not match plan");
  const i64 m = basis.m;
  for (size_t g = 0; g < blocks.size(); ++g) {
    if (blocks[g]->m != m) throw std::invalid_argument("column_project: row count mismatch");
    if (blocks[g]->n != static_cast<i64>(groups[g].size()))
      throw std::invalid_argument("column_project: block width does not match plan group");
  }
  out = DevLowRank{};
  out.m = m;
  out.n = n;
  SvdOfProduct bf = svd_of_product(s, m, basis.n, basis.k, basis.left.get(), basis.right.get());
  if (bf.r == 0) return;
  const i64 kb = bf.r;
  out.k = kb;
  out.left = std::move(bf.U);
  out.right.alloc(n * kb, s);
  out.right.zero(s);
  for (size_t g = 0; g < blocks.size(); ++g) {
    const DevLowRank& B = *blocks[g];
    if (B.k == 0) continue;
    const i64 w = static_cast<i64>(groups[g].size());
    DBuf<double> Rg(w * kb, s);
    project_rows(s, out.left.get(), m, kb, B, Rg.get());
    scatter_rows(s, Rg.get(), w, kb, groups[g], out.right.get());
  }
  DFCG_CUDA(cudaStreamSynchronize(s));
}

// One block of column_project (sketch.hpp:194-196): Rg = right_g (Ub^T left_g)^T, w_g x kb.
// The multi-GPU combine runs it on the block's own rank; the arithmetic is the same GEMM pair.
void project_rows(cudaStream_t s, const double* Ub, i64 m, i64 kb, const DevLowRank& B, double* Rg) {
  if (B.m != m) throw std::invalid_argument("column_project: row count mismatch");
  const i64 w = B.n;
  if (B.k == 0) {
    DFCG_CUDA(cudaMemsetAsync(Rg, 0, sizeof(double) * static_cast<size_t>(w * kb), s));
    return;
  }
  DBuf<double> proj(kb * B.k, s);
  gemm(s, true, false, kb, B.k, m, 1.0, Ub, kb, B.left.get(), B.k, 0.0, proj.get(), B.k);  // Ub^T left_g
  gemm(s, false, true, w, kb, B.k, 1.0, B.right.get(), B.k, proj.get(), B.k, 0.0, Rg, kb);  // right_g proj^T
}

// dst[idx[p], :] = src[p, :] for the rows of one plan group (width c, row-major, ld c)
void scatter_rows(cudaStream_t s, const double* src, i64 rows, i64 c, const std::vector<i64>& idx, double* dst) {
  if (rows == 0 || c == 0) return;
  DBuf<long long> d = upload_idx(s, idx);
  scatter_rows_kernel<<<grid_for(rows * c), 256, 0, s>>>(rows, c, src, c, d.get(), dst, c);
  DFCG_LAUNCH_CHECK();
}

// dst[p, :] = src[idx[p], :] (width c, row-major, ld c)
void gather_rows(cudaStream_t s, const double* src, i64 c, const std::vector<i64>& idx, double* dst) {
  const i64 l = static_cast<i64>(idx.size());
  if (l == 0 || c == 0) return;
  DBuf<long long> d = upload_idx(s, idx);
  gather_rows_kernel<<<grid_for(l * c), 256, 0, s>>>(l, c, src, c, d.get(), dst, c);
  DFCG_LAUNCH_CHECK();
}

// gen_nystrom (sketch.hpp:241-266): C W^+ R with W = C_hat restricted to the sampled rows.
void gen_nystrom(cudaStream_t s, const DevLowRank& C, const DevLowRank& R, const std::vector<i64>& rows,
                 const std::vector<i64>& cols, DevLowRank& out) {
  const i64 m = C.m, n = R.n;
  const i64 d = static_cast<i64>(rows.size()), l = static_cast<i64>(cols.size());
  if (R.m != d) throw std::invalid_argument("gen_nystrom: R_hat rows != |row_idx|");
  if (C.n != l) throw std::invalid_argument("gen_nystrom: C_hat cols != |col_idx|");
  for (i64 i : rows)
    if (i < 0 || i >= m) throw std::out_of_range("gen_nystrom: row index out of range");
  for (i64 j : cols)
    if (j < 0 || j >= n) throw std::out_of_range("gen_nystrom: col index out of range");
  out = DevLowRank{};
  out.m = m;
  out.n = n;
  if (C.k == 0 || R.k == 0) return;
  DBuf<double> Wleft(d * C.k, s);
  DBuf<long long> ridx = upload_idx(s, rows);
  gather_rows_kernel<<<grid_for(d * C.k), 256, 0, s>>>(d, C.k, C.left.get(), C.k, ridx.get(), Wleft.get(), C.k);
  DFCG_LAUNCH_CHECK();
  SvdOfProduct wf = svd_of_product(s, d, l, C.k, Wleft.get(), C.right.get());
  if (wf.r == 0) return;
  const i64 r = wf.r;
  DBuf<double> T(C.k * r, s), T2(R.k * r, s);
  gemm(s, true, false, C.k, r, l, 1.0, C.right.get(), C.k, wf.V.get(), r, 0.0, T.get(), r);  // C.right^T V_W
  DBuf<double> ds = upload_vec(s, wf.s);
  scale_cols_kernel<<<grid_for(C.k * r), 256, 0, s>>>(C.k, r, T.get(), r, ds.get(), 1);      // * s^-1
  DFCG_LAUNCH_CHECK();
  out.k = r;
  out.left.alloc(m * r, s);
  out.right.alloc(n * r, s);
  gemm(s, false, false, m, r, C.k, 1.0, C.left.get(), C.k, T.get(), r, 0.0, out.left.get(), r);
  gemm(s, true, false, R.k, r, d, 1.0, R.left.get(), R.k, wf.U.get(), r, 0.0, T2.get(), r);  // R.left^T U_W
  gemm(s, false, false, n, r, R.k, 1.0, R.right.get(), R.k, T2.get(), r, 0.0, out.right.get(), r);
  DFCG_CUDA(cudaStreamSynchronize(s));
}

// average_estimates (sketch.hpp:271-298).
void average_estimates(cudaStream_t s, const std::vector<const DevLowRank*>& ests, std::optional<i64> recompress_to,
                       DevLowRank& out) {
  if (ests.empty()) throw std::invalid_argument("average_estimates: empty list");
  const i64 m = ests[0]->m, n = ests[0]->n;
  i64 K = 0;
  for (const DevLowRank* e : ests) {
    if (e->m != m || e->n != n) throw std::invalid_argument("average_estimates: dimension mismatch");
    K += e->k;
  }
  out = DevLowRank{};
  out.m = m;
  out.n = n;
  if (K == 0) return;
  DBuf<double> left(m * K, s), right(n * K, s);
  const double scale = 1.0 / static_cast<double>(ests.size());
  i64 at = 0;
  for (const DevLowRank* e : ests) {
    if (e->k == 0) continue;
    copy2d(s, m, e->k, e->left.get(), e->k, left.get() + at, K);
    copy2d(s, n, e->k, e->right.get(), e->k, right.get() + at, K, scale);
    at += e->k;
  }
  if (!recompress_to && K <= std::min(m, n)) {
    out.k = K;
    out.left = std::move(left);
    out.right = std::move(right);
    DFCG_CUDA(cudaStreamSynchronize(s));
    return;
  }
  SvdOfProduct f = svd_of_product(s, m, n, K, left.get(), right.get());
  i64 keep = f.r;
  if (recompress_to) keep = std::min(keep, std::max<i64>(*recompress_to, 0));
  if (keep == 0) return;
  out.k = keep;
  out.left.alloc(m * keep, s);
  out.right.alloc(n * keep, s);
  copy2d(s, m, keep, f.est.left.get(), f.r, out.left.get(), keep);
  copy2d(s, n, keep, f.est.right.get(), f.r, out.right.get(), keep);
  DFCG_CUDA(cudaStreamSynchronize(s));
}

// random_project (sketch.hpp:204-237).
void random_project(cudaStream_t s, const std::vector<const DevLowRank*>& blocks,
                    const std::vector<std::vector<i64>>& groups, i64 n, i64 k, i64 p, i64 q, SeededRng& rng,
                    DevLowRank& out) {
  if (blocks.empty()) throw std::invalid_argument("random_project: no blocks");
  if (blocks.size() != groups.size()) throw std::invalid_argument("random_project: block count does not match plan");
  if (k < 1 || p < 0 || q < 0) throw std::invalid_argument("random_project: bad RpParams");
  const i64 m = blocks[0]->m;
  for (size_t g = 0; g < blocks.size(); ++g) {
    if (blocks[g]->m != m) throw std::invalid_argument("random_project: row count mismatch");
    if (blocks[g]->n != static_cast<i64>(groups[g].size()))
      throw std::invalid_argument("random_project: block width does not match plan group");
  }
  if (k + p > std::min(m, n)) throw std::invalid_argument("random_project: k + p exceeds min(m, n)");
  std::vector<DBuf<long long>> idx;
  for (const auto& g : groups) idx.push_back(upload_idx(s, g));
  BlocksOp op{blocks, idx, groups, m, n};
  const i64 b = k + p;
  // gaussian_matrix(n, b): column-major draws
  std::vector<double> hg(static_cast<size_t>(n * b));
  for (i64 j = 0; j < b; ++j)
    for (i64 i = 0; i < n; ++i) hg[static_cast<size_t>(i * b + j)] = rng.normal();
  DBuf<double> G = upload_vec(s, hg), Y(m * b, s), Z(n * b, s);
  op.apply(s, G.get(), b, Y.get());
  for (i64 it = 0; it < q; ++it) {
    thin_qr(s, m, b, Y.get(), b, nullptr, 0);  // Q overwrites Y
    op.apply_adjoint(s, Y.get(), b, Z.get());
    thin_qr(s, n, b, Z.get(), b, nullptr, 0);
    op.apply(s, Z.get(), b, Y.get());
  }
  DBuf<double> U, V;
  std::vector<double> sv;
  general_svd(s, m, b, Y.get(), U, V, sv);
  const i64 kk = std::min(k, numerical_rank(sv, m, n, 1e-12));
  out = DevLowRank{};
  out.m = m;
  out.n = n;
  if (kk == 0) return;
  const i64 pcols = std::min(m, b);
  out.k = kk;
  out.left.alloc(m * kk, s);
  out.right.alloc(n * kk, s);
  copy2d(s, m, kk, U.get(), pcols, out.left.get(), kk);
  op.apply_adjoint(s, out.left.get(), kk, out.right.get());
  DFCG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace dfcg
