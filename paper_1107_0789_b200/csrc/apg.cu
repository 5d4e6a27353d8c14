// APG base solvers on the device: apg_mc (P/include/dfc/solvers.hpp:241-327) and apg_rmf
// (:332-414), with the rank-adaptive randomized SVT (svt_operator :98-109, partial_svd /
// randomized_range P/include/dfc/sketch.hpp:144-166) running entirely on the GPU.
//
// Control flow (iteration count, k doubling, shrink count, continuation, stop test) is the
// reference's, decided on the host from a handful of device scalars per iteration. The
// Gaussian test matrices come from the same SeededRng(0x737674, 0|1) stream, consumed in
// the same order. One deliberate difference: extrapolate (:196-212) compacts Y with an
// exact svd_of_product when kc + kp > min(m, n); the device keeps the concatenated factors
// instead — the same matrix Y (the compaction only drops singular values <= 1e-12 *
// max(m,n) * s_max), consumed only through Y*X, Y^T*X and P_Omega(Y).
// High-rank iterations apply the same operator materialised (dense_operator: Y off Omega, M on
// it) and, when cheaper, compressed by a CholeskyQR2 factor (OpTri for m >= n, OpWideQR for
// m < n): the randomized SVT then runs in the R factor's coordinates — same spans, same draws.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <cuda_profiler_api.h>

#include "solver.hpp"

namespace dfcg {

namespace {

int grid_for(i64 total, int threads = 256) {
  return static_cast<int>(std::max<i64>(1, std::min<i64>((total + threads - 1) / threads, 4096)));
}

// dst[r, c] = src[r, c] * scale[c]   (rows x cols)
__global__ void scale_cols_kernel(i64 rows, i64 cols, const double* __restrict__ src, i64 lds,
                                  const double* __restrict__ scale, double* __restrict__ dst, i64 ldd) {
  const i64 total = rows * cols;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 r = e / cols, c = e % cols;
    dst[r * ldd + c] = src[r * lds + c] * scale[c];
  }
}

// r = a pc + b pp - m (a term is skipped, not multiplied, when its coefficient is 0: the
// buffer may hold stale values then)
__global__ void residual_combine_kernel(i64 n, double a, const double* __restrict__ pc, double b,
                                        const double* __restrict__ pp, const double* __restrict__ mv,
                                        double* __restrict__ r) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    double v = 0.0;
    if (a != 0.0) v = a * pc[i];
    if (b != 0.0) v = fma(b, pp[i], v);
    r[i] = v - mv[i];
  }
}

void residual_combine(cudaStream_t s, i64 n, double a, const double* pc, double b, const double* pp,
                      const double* mv, double* r) {
  if (n <= 0) return;
  prof::Scope scope(prof::kElementwise, s, 3.0 * n, 8.0 * n * ((a != 0.0) + (b != 0.0) + 2.0));
  residual_combine_kernel<<<grid_for(n), 256, 0, s>>>(n, a, pc, b, pp, mv, r);
  DFCG_LAUNCH_CHECK();
}

// Dense APG-MC operator, row-major m x w: with step 1 the operator G = Y - (P_Omega(Y) -
// P_Omega(M)) of FactoredSparseOp (solvers.hpp:112-136) is Y off the observed set and M on it.
// Pass 1: A = a Dc + b Dp (a term with coefficient 0 is skipped, its buffer may be stale).
__global__ void dense_extrap_kernel(i64 n, double a, const double* __restrict__ dc, double b,
                                    const double* __restrict__ dp, double* __restrict__ A) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    double v = 0.0;
    if (a != 0.0) v = a * dc[i];
    if (b != 0.0) v = fma(b, dp[i], v);
    A[i] = v;
  }
}

// Pass 2 (one CTA per row, CSR walk: columns ascend, so the stores of a row coalesce):
// A[i, j] = M_e for every observed (i, j).
__global__ void dense_observe_kernel(i64 w, const int* __restrict__ rowptr, const int* __restrict__ ccol,
                                     const double* __restrict__ m_csr, double* __restrict__ A) {
  const i64 i = blockIdx.x;
  double* row = A + i * w;
  for (int e = rowptr[i] + threadIdx.x; e < rowptr[i + 1]; e += blockDim.x) row[ccol[e]] = m_csr[e];
}

// P_Omega of a dense row-major iterate in CSR order: out[e] = D[row_e, col_e].
__global__ void dense_gather_kernel(i64 w, const int* __restrict__ rowptr, const int* __restrict__ ccol,
                                    const double* __restrict__ D, double* __restrict__ out) {
  const i64 i = blockIdx.x;
  const double* row = D + i * w;
  for (int e = rowptr[i] + threadIdx.x; e < rowptr[i + 1]; e += blockDim.x) out[e] = row[ccol[e]];
}

__global__ void fill_kernel(i64 n, double v, double* x) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    x[i] = v;
}

__global__ void scale_by_inv_kernel(i64 n, const double* __restrict__ x, const double* __restrict__ nrm,
                                    double* __restrict__ y) {
  const double d = *nrm;
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    y[i] = x[i] / d;
}

__global__ void sqrt_kernel(double* x) { *x = sqrt(*x); }

// RMF fused extrapolation + gradient + soft-threshold (solvers.hpp:358-360,366,370):
//   yl = Ld + b (Ld - Ldp); ys = S + b (S - Sp); g = yl + ys - M
//   GL = yl - step g ; S_next = soft(ys - step g, thr)
__global__ void rmf_fused_kernel(i64 n, double beta, double step, double thr, const double* __restrict__ Ld,
                                 const double* __restrict__ Ldp, const double* __restrict__ S,
                                 const double* __restrict__ Sp, const double* __restrict__ M, double* __restrict__ GL,
                                 double* __restrict__ Snext) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const double ld = Ld[i], s = S[i];
    const double yl = ld + beta * (ld - Ldp[i]);
    const double ys = s + beta * (s - Sp[i]);
    const double g = yl + ys - M[i];
    GL[i] = yl - step * g;
    const double a = ys - step * g;
    const double mag = fabs(a) - thr;
    Snext[i] = mag > 0 ? (a > 0 ? mag : -mag) : 0.0;
  }
}

// Line-search variant inputs: YL, YS, g materialised.
__global__ void rmf_extrap_kernel(i64 n, double beta, const double* __restrict__ Ld, const double* __restrict__ Ldp,
                                  const double* __restrict__ S, const double* __restrict__ Sp,
                                  const double* __restrict__ M, double* __restrict__ YL, double* __restrict__ YS,
                                  double* __restrict__ G) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const double ld = Ld[i], s = S[i];
    const double yl = ld + beta * (ld - Ldp[i]);
    const double ys = s + beta * (s - Sp[i]);
    YL[i] = yl;
    YS[i] = ys;
    G[i] = yl + ys - M[i];
  }
}

__global__ void rmf_step_kernel(i64 n, double step, double thr, const double* __restrict__ YL,
                                const double* __restrict__ YS, const double* __restrict__ G, double* __restrict__ GL,
                                double* __restrict__ Snext) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const double g = G[i];
    GL[i] = YL[i] - step * g;
    const double a = YS[i] - step * g;
    const double mag = fabs(a) - thr;
    Snext[i] = mag > 0 ? (a > 0 ? mag : -mag) : 0.0;
  }
}

// Deterministic multi-output reductions over n elements: fixed grid, per-block partials,
// single-block final sum. K quantities per element.
constexpr int RB = 1024, RT = 256;  // 1024 blocks: a 256-block grid streamed a 200 MB pair at 3.3 TB/s (ncu)

template <int K, class F>
__global__ void multi_sum_partial(i64 n, F f, double* part) {
  double acc[K];
#pragma unroll
  for (int q = 0; q < K; ++q) acc[q] = 0.0;
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    f(i, acc);
  __shared__ double sh[K][RT / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < K; ++q) {
    double v = acc[q];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sh[q][w] = v;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double v = 0.0;
    for (int j = 0; j < RT / 32; ++j) v += sh[threadIdx.x][j];
    part[threadIdx.x * gridDim.x + blockIdx.x] = v;
  }
}

__global__ void multi_sum_final(int K, int nb, const double* part, double* out) {
  __shared__ double sh[RT];
  for (int q = 0; q < K; ++q) {
    double v = 0.0;
    for (int j = threadIdx.x; j < nb; j += blockDim.x) v += part[q * nb + j];
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[q] = sh[0];
    __syncthreads();
  }
}

template <int K, class F>
std::vector<double> multi_sum(cudaStream_t s, i64 n, F f) {
  prof::Scope scope(prof::kReduce, s, 3.0 * K * n, 8.0 * 4 * n);
  DBuf<double> part(K * RB, s), out(K, s);
  multi_sum_partial<K><<<RB, RT, 0, s>>>(n, f, part.get());
  DFCG_LAUNCH_CHECK();
  multi_sum_final<<<1, RT, 0, s>>>(K, RB, part.get(), out.get());
  DFCG_LAUNCH_CHECK();
  std::vector<double> h(K);
  DFCG_CUDA(cudaMemcpyAsync(h.data(), out.get(), sizeof(double) * K, cudaMemcpyDeviceToHost, s));
  DFCG_CUDA(cudaStreamSynchronize(s));
  return h;
}

double host_scalar(cudaStream_t s, const double* d) {
  double h = 0.0;
  DFCG_CUDA(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, s));
  DFCG_CUDA(cudaStreamSynchronize(s));
  return h;
}

double dev_dot(cudaStream_t s, i64 n, const double* a, const double* b) {
  if (n <= 0) return 0.0;
  DBuf<double> out(1, s);
  dot_sum(s, n, a, b, out.get());
  return host_scalar(s, out.get());
}

// ---------------------------------------------------------------- operators
// Sketch buffers use an even leading dimension (b rounded up) so the DMMA GEMMs take their
// 16-byte operand loads; the padding column is never read (K / N extents stay b).
inline i64 even_ld(i64 b) { return b + (b & 1); }

// FactoredSparseOp (solvers.hpp:112-136): G = left right^T + coeff * R.
struct OpMC {
  const DevOmega* om;
  const double* r_csr;
  const double* r_csc;  // the same residual in CSC order (transposed products)
  double coeff;
  i64 m, w, kY;
  const double* left;   // m x kY row-major (ld ldy)
  const double* right;  // w x kY row-major (ld ldy)
  i64 kc;               // the first kc columns of `left` are L_curr's left factor
  i64 ldy;
  i64 rows() const { return m; }
  i64 cols() const { return w; }
  i64 zrows() const { return w; }  // rows of the n-side range-finder vectors
  void apply_g0(cudaStream_t s, const double* X, i64 ldx, i64 b, double* out, i64 ldo) const {
    apply(s, X, ldx, b, out, ldo);
  }
  void apply(cudaStream_t s, const double* X, i64 ldx, i64 b, double* out, i64 ldo) const {  // w x b -> m x b
    if (kY > 0) {
      const i64 ldt = even_ld(b);
      DBuf<double> T(kY * ldt, s);
      gemm(s, true, false, kY, b, w, 1.0, right, ldy, X, ldx, 0.0, T.get(), ldt);
      gemm(s, false, false, m, b, kY, 1.0, left, ldy, T.get(), ldt, 0.0, out, ldo);
      spmm(s, *om, false, r_csr, b, coeff, X, ldx, 1.0, out, ldo);
    } else {
      spmm(s, *om, false, r_csr, b, coeff, X, ldx, 0.0, out, ldo);
    }
  }
  // keep (optional): receives T = left^T X (kY x b, ld even_ld(b)), whose first kc rows are
  // L_curr.left^T X.
  void apply_adjoint(cudaStream_t s, const double* X, i64 ldx, i64 b, double* out, i64 ldo,
                     DBuf<double>* keep = nullptr) const {
    if (kY > 0) {
      const i64 ldt = even_ld(b);
      DBuf<double> T(kY * ldt, s);
      gemm(s, true, false, kY, b, m, 1.0, left, ldy, X, ldx, 0.0, T.get(), ldt);
      gemm(s, false, false, w, b, kY, 1.0, right, ldy, T.get(), ldt, 0.0, out, ldo);
      spmm(s, *om, true, r_csr, b, coeff, X, ldx, 1.0, out, ldo, r_csc);
      if (keep) *keep = std::move(T);
    } else {
      spmm(s, *om, true, r_csr, b, coeff, X, ldx, 0.0, out, ldo, r_csc);
    }
  }
  i64 keep_rows() const { return kc; }
  void to_dense(cudaStream_t s, double* D) const {  // m x w row-major
    if (kY > 0) gemm(s, false, true, m, w, kY, 1.0, left, ldy, right, ldy, 0.0, D, w);
    else DFCG_CUDA(cudaMemsetAsync(D, 0, sizeof(double) * m * w, s));
    scatter_add_dense(s, *om, r_csr, coeff, D, w);
  }
};

// The dense APG-MC operator (row-major m x w), see dense_operator().
struct OpDenseRM {
  const double* A;
  i64 m, w;
  i64 rows() const { return m; }
  i64 cols() const { return w; }
  i64 zrows() const { return w; }
  void apply_g0(cudaStream_t s, const double* X, i64 ldx, i64 b, double* out, i64 ldo) const {
    apply(s, X, ldx, b, out, ldo);
  }
  void apply(cudaStream_t s, const double* X, i64 ldx, i64 b, double* out, i64 ldo) const {
    gemm(s, false, false, m, b, w, 1.0, A, w, X, ldx, 0.0, out, ldo);
  }
  void apply_adjoint(cudaStream_t s, const double* X, i64 ldx, i64 b, double* out, i64 ldo,
                     DBuf<double>* = nullptr) const {
    gemm(s, true, false, w, b, m, 1.0, A, w, X, ldx, 0.0, out, ldo);
  }
  i64 keep_rows() const { return -1; }
  void to_dense(cudaStream_t s, double* D) const { copy2d(s, m, w, A, w, D, w); }
};

// The same operator compressed by a CholeskyQR2 factor A = Q_A R_A (m >= w, Q_A orthonormal,
// never formed): every range-finder quantity of partial_svd is basis-invariant, so the SVT of A
// runs on the w x w triangle R_A in Q_A's coordinates (orth(A Z) = Q_A orth(R_A Z), A^T Q_A Q~
// = R_A^T Q~) and only the left factor maps back, U = Q_A U~ = A R_A^-1 U~. R_A is backward
// stable (A = Q_A R_A + O(eps ||A||)), like the products with A it replaces.
struct OpTri {
  const double* R;  // w x w row-major, upper (lower part zero)
  i64 w;
  i64 rows() const { return w; }
  i64 cols() const { return w; }
  i64 zrows() const { return w; }
  void apply_g0(cudaStream_t s, const double* X, i64 ldx, i64 b, double* out, i64 ldo) const {
    apply(s, X, ldx, b, out, ldo);
  }
  void apply(cudaStream_t s, const double* X, i64 ldx, i64 b, double* out, i64 ldo) const {
    gemm_tri_a(s, false, w, b, 1.0, R, w, X, ldx, 0.0, out, ldo);
  }
  void apply_adjoint(cudaStream_t s, const double* X, i64 ldx, i64 b, double* out, i64 ldo,
                     DBuf<double>* = nullptr) const {
    gemm_tri_a(s, true, w, b, 1.0, R, w, X, ldx, 0.0, out, ldo);
  }
  i64 keep_rows() const { return -1; }
  void to_dense(cudaStream_t s, double* D) const { copy2d(s, w, w, R, w, D, w); }
};

// Wide dense operator (m < n) compressed by CholeskyQR2 of its transpose: A^T = Q_B R, i.e.
// A = R^T Q_B^T (R m x m upper). The first range-finder product is A G0 itself; every later
// n-side vector lies in span(Q_B) and is kept in its coordinates (Z = Q_B Z~): A Z = R^T Z~,
// A^T Q = Q_B (R Q). The right factor maps back as V = Q_B V~ = A^T R^-1 V~ (deferred).
struct OpWideQR {
  const double* A;  // m x n row-major
  const double* R;  // m x m row-major, upper (lower part zero)
  i64 m, n;
  i64 rows() const { return m; }
  i64 cols() const { return n; }
  i64 zrows() const { return m; }
  void apply_g0(cudaStream_t s, const double* X, i64 ldx, i64 b, double* out, i64 ldo) const {
    gemm(s, false, false, m, b, n, 1.0, A, n, X, ldx, 0.0, out, ldo);
  }
  void apply(cudaStream_t s, const double* X, i64 ldx, i64 b, double* out, i64 ldo) const {
    gemm_tri_a(s, true, m, b, 1.0, R, m, X, ldx, 0.0, out, ldo);
  }
  void apply_adjoint(cudaStream_t s, const double* X, i64 ldx, i64 b, double* out, i64 ldo,
                     DBuf<double>* = nullptr) const {
    gemm_tri_a(s, false, m, b, 1.0, R, m, X, ldx, 0.0, out, ldo);
  }
  i64 keep_rows() const { return -1; }
  void to_dense(cudaStream_t s, double* D) const { transpose(s, m, m, R, m, D, m); }  // R^T
};

// DenseOp (solvers.hpp:138-145) over a column-major m x w matrix A (== row-major w x m "At").
struct OpDense {
  const double* At;
  i64 m, w;
  i64 rows() const { return m; }
  i64 cols() const { return w; }
  i64 zrows() const { return w; }
  void apply_g0(cudaStream_t s, const double* X, i64 ldx, i64 b, double* out, i64 ldo) const {
    apply(s, X, ldx, b, out, ldo);
  }
  void apply(cudaStream_t s, const double* X, i64 ldx, i64 b, double* out, i64 ldo) const {
    gemm(s, true, false, m, b, w, 1.0, At, m, X, ldx, 0.0, out, ldo);
  }
  void apply_adjoint(cudaStream_t s, const double* X, i64 ldx, i64 b, double* out, i64 ldo,
                     DBuf<double>* = nullptr) const {
    gemm(s, false, false, w, b, m, 1.0, At, m, X, ldx, 0.0, out, ldo);
  }
  i64 keep_rows() const { return -1; }  // no factor Grams for a dense operator
  void to_dense(cudaStream_t s, double* D) const { transpose(s, w, m, At, m, D, w); }
};

// Result of the SVT: L_next = (U, V diag(s)), s = shrunk singular values (host copy).
struct SvtResult {
  i64 r = 0;
  DBuf<double> left, right;  // m x r, w x r row-major
  std::vector<double> s;
  i64 k_final = 0;
  int calls = 0;
  // Left-factor Grams from the randomized path (left = Q Vz with Q^T Q = I): ll = left^T left
  // = Vz^T Vz (r x r) and lc = Lc.left^T left (kc x r) read off the last adjoint product, so
  // the factored inner products of the stop test need no m-side GEMM.
  bool grams = false;
  DBuf<double> ll, lc;
};

// shrink_factors (solvers.hpp:83-88) applied to device factors U (m x ncand, ldu) and
// V (w x ncand, ldv) with singular values sv (descending, host).
void shrink_into(cudaStream_t s, i64 m, i64 w, const double* U, i64 ldu, const double* V, i64 ldv,
                 const std::vector<double>& sv, double tau, SvtResult& res) {
  i64 r = 0;
  while (r < static_cast<i64>(sv.size()) && sv[static_cast<size_t>(r)] > tau) ++r;
  res.r = r;
  res.s.assign(sv.begin(), sv.begin() + r);
  for (double& x : res.s) x -= tau;
  if (r == 0) return;
  res.left.alloc(m * r, s);
  res.right.alloc(w * r, s);
  copy2d(s, m, r, U, ldu, res.left.get(), r);
  DBuf<double> sc(r, s);
  DFCG_CUDA(cudaMemcpyAsync(sc.get(), res.s.data(), sizeof(double) * r, cudaMemcpyHostToDevice, s));
  scale_cols_kernel<<<grid_for(w * r), 256, 0, s>>>(w, r, V, ldv, sc.get(), res.right.get(), r);
  DFCG_LAUNCH_CHECK();
  DFCG_CUDA(cudaStreamSynchronize(s));  // res.s host buffer used by the async copy
}

// svt_factors_dense (solvers.hpp:90-93) on the materialised operator.
template <class Op>
void svt_dense(cudaStream_t s, const Op& op, double tau, SvtResult& res) {
  const i64 m = op.rows(), w = op.zrows();  // (compressed operators: w = the coordinate count)
  DBuf<double> D(m * w, s);
  op.to_dense(s, D.get());
  std::vector<double> sv;
  if (m >= w) {
    DBuf<double> U(m * w, s), V(w * w, s);
    thin_svd(s, m, w, D.get(), w, U.get(), w, V.get(), w, sv, tau);
    shrink_into(s, m, w, U.get(), w, V.get(), w, sv, tau, res);
  } else {
    DBuf<double> Dt(w * m, s), U(w * m, s), V(m * m, s);
    transpose(s, m, w, D.get(), w, Dt.get(), m);
    thin_svd(s, w, m, Dt.get(), m, U.get(), m, V.get(), m, sv, tau);  // D^T = U S V^T -> D = V S U^T
    shrink_into(s, m, w, V.get(), m, U.get(), m, sv, tau, res);
  }
}

struct NormalCursor {
  NormalCache* cache;
  i64 pos = 0;
};

// partial_svd (sketch.hpp:156-166) + randomized_range (:144-153) with p, q; then the SVT
// acceptance test and shrink of svt_operator (solvers.hpp:105-106).  Returns true if the
// result was accepted (f.rank() < k or s[k-1] <= tau), filling res.
template <class Op>
bool partial_svt(cudaStream_t s, const Op& op, i64 k, i64 p, i64 q, NormalCursor& cur, double tau, SvtResult& res) {
  const i64 m = op.rows(), w = op.cols(), wz = op.zrows();  // wz: rows of the n-side vectors
  const i64 b = std::min(k + p, std::min(m, w));
  const i64 bl = even_ld(b);  // leading dimension of every sketch-width buffer
  // gaussian_matrix(w, b): column-major draws == row-major b x w; transpose to w x b.
  DBuf<double> Gt(b * w, s), G(w * bl, s), X(m * bl, s), Z(wz * bl, s);
  cur.cache->fetch(cur.pos, w * b, Gt.get(), s);
  cur.pos += w * b;
  transpose(s, b, w, Gt.get(), w, G.get(), bl);
  op.apply_g0(s, G.get(), bl, b, X.get(), bl);
  G.release();
  Gt.release();
  // m-side bases are kept lazily: the orthonormal basis is Q = X M (M = R^-1 of a CholQR
  // factor of X), and M is applied on the n side after the next product, A^T Q = (A^T X) M,
  // so the m x b x b triangular products of the intermediate bases (and of the second
  // CholQR pass of the final one) are never formed. Intermediate bases need one CholQR pass
  // (same span, well conditioned); the final projector gets two. Any Cholesky breakdown
  // falls back to the explicit thin_qr (Householder), with M = I.
  DBuf<double> M(b * bl, s), Xt;
  bool lazy = false;
  auto orth_m = [&](bool final_basis) {
    lazy = false;
    if (!cholqr_factor(s, m, b, X.get(), bl, M.get(), bl)) {
      thin_qr(s, m, b, X.get(), bl, nullptr, 0, final_basis ? 2 : 1);
      return;
    }
    if (!final_basis) {
      lazy = true;
      return;
    }
    Xt.alloc(m * bl, s);  // pass 1 explicit: X <- X R1^-1; pass 2 lazy
    gemm_upper_b(s, m, b, 1.0, X.get(), bl, M.get(), bl, 0.0, Xt.get(), bl);
    std::swap(X, Xt);
    if (cholqr_factor(s, m, b, X.get(), bl, M.get(), bl)) lazy = true;
    else thin_qr(s, m, b, X.get(), bl, nullptr, 0, 1);
  };
  auto adjoint = [&](DBuf<double>* keep) {  // Z = A^T Q
    op.apply_adjoint(s, X.get(), bl, b, Z.get(), bl, keep);
    if (lazy) {
      DBuf<double> Zm(wz * bl, s);
      gemm_upper_b(s, wz, b, 1.0, Z.get(), bl, M.get(), bl, 0.0, Zm.get(), bl);
      std::swap(Z, Zm);
    }
  };
  orth_m(q == 0);
  for (i64 it = 0; it < q; ++it) {
    adjoint(nullptr);
    thin_qr(s, wz, b, Z.get(), bl, nullptr, 0, 1);
    op.apply(s, Z.get(), bl, b, X.get(), bl);
    orth_m(it + 1 == q);
  }
  DBuf<double> T;
  adjoint(&T);  // Z = A^T Q (w x b); T = Yl^T X (before M, ld bl) for the factor Grams
  DBuf<double> Uz(wz * bl, s), Vz(b * bl, s);
  std::vector<double> sv;
  thin_svd(s, wz, b, Z.get(), bl, Uz.get(), bl, Vz.get(), bl, sv, tau);
  const i64 kk = std::min<i64>(k, static_cast<i64>(sv.size()));
  sv.resize(static_cast<size_t>(kk));
  if (!(kk < k || sv[static_cast<size_t>(kk - 1)] <= tau)) return false;
  // accepted: U = Q Vz[:, :kk] = X (M Vz[:, :kk]), V = Uz[:, :kk]; shrink keeps the first r <= kk
  i64 r = 0;
  while (r < kk && sv[static_cast<size_t>(r)] > tau) ++r;
  res.r = r;
  res.s.assign(sv.begin(), sv.begin() + r);
  for (double& x : res.s) x -= tau;
  if (r == 0) return true;
  res.left.alloc(m * r, s);
  res.right.alloc(wz * r, s);
  DBuf<double> MV;
  const double* coef = Vz.get();  // b x r block mapping X to the left factor
  i64 ldcoef = bl;
  if (lazy) {
    ldcoef = even_ld(r);
    MV.alloc(b * ldcoef, s);
    gemm(s, false, false, b, r, b, 1.0, M.get(), bl, Vz.get(), bl, 0.0, MV.get(), ldcoef);
    coef = MV.get();
  }
  gemm(s, false, false, m, r, b, 1.0, X.get(), bl, coef, ldcoef, 0.0, res.left.get(), r);
  const i64 kc = op.keep_rows();
  if (kc >= 0 && T.size() >= kc * bl) {  // left = Q Vz_r: left^T left = Vz_r^T Vz_r, Lc.left^T left = T[:kc] coef
    res.grams = true;
    res.ll.alloc(r * r, s);
    gemm(s, true, false, r, r, b, 1.0, Vz.get(), bl, Vz.get(), bl, 0.0, res.ll.get(), r);
    if (kc > 0) {
      res.lc.alloc(kc * r, s);
      gemm(s, false, false, kc, r, b, 1.0, T.get(), bl, coef, ldcoef, 0.0, res.lc.get(), r);
    }
  }
  DBuf<double> sc(r, s);
  DFCG_CUDA(cudaMemcpyAsync(sc.get(), res.s.data(), sizeof(double) * r, cudaMemcpyHostToDevice, s));
  scale_cols_kernel<<<grid_for(wz * r), 256, 0, s>>>(wz, r, Uz.get(), bl, sc.get(), res.right.get(), r);
  DFCG_LAUNCH_CHECK();
  DFCG_CUDA(cudaStreamSynchronize(s));
  return true;
}

// svt_operator (solvers.hpp:98-109).
template <class Op>
void svt_operator(cudaStream_t s, const Op& op, double tau, i64 rank_hint, NormalCursor& cur, SvtResult& res) {
  const i64 minmn = std::min(op.rows(), op.cols());
  res.calls = 0;
  res.k_final = 0;
  if (minmn <= 64) {
    res.calls = 1;
    svt_dense(s, op, tau, res);
    return;
  }
  i64 k = std::clamp<i64>(rank_hint + 5, 1, minmn);
  for (;;) {
    ++res.calls;
    if (k >= minmn) {
      res.k_final = 0;
      svt_dense(s, op, tau, res);
      return;
    }
    res.k_final = k;
    if (partial_svt(s, op, k, 10, 2, cur, tau, res)) return;
    k = std::min<i64>(2 * k, minmn);
  }
}

// factored_inner (solvers.hpp:179-184): sum((a.l^T b.l) .* (a.r^T b.r)).
// lda / ldb: leading dimensions of a's / b's factors (0: the rank)
double factored_inner(cudaStream_t s, i64 m, i64 n, i64 ka, const double* al, const double* ar, i64 kb,
                      const double* bl, const double* br, i64 lda = 0, i64 ldb = 0) {
  if (ka == 0 || kb == 0) return 0.0;
  if (lda == 0) lda = ka;
  if (ldb == 0) ldb = kb;
  DBuf<double> L(ka * kb, s), R(ka * kb, s);
  gemm(s, true, false, ka, kb, m, 1.0, al, lda, bl, ldb, 0.0, L.get(), kb);
  gemm(s, true, false, ka, kb, n, 1.0, ar, lda, br, ldb, 0.0, R.get(), kb);
  return dev_dot(s, ka * kb, L.get(), R.get());
}

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

double sum_of(const std::vector<double>& v) {
  double a = 0.0;
  for (double x : v) a += x;
  return a;
}

}  // namespace

// ---------------------------------------------------------------- normal stream
__global__ void box_muller_kernel(const std::uint64_t* __restrict__ raw, double* __restrict__ out, i64 n) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const double u1 = (static_cast<double>(raw[2 * i] >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = static_cast<double>(raw[2 * i + 1] >> 11) * 0x1.0p-53;
    out[i] = sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
  }
}

void box_muller_device(cudaStream_t s, const std::uint64_t* raw, double* out, i64 n) {
  box_muller_kernel<<<grid_for(n), 256, 0, s>>>(raw, out, n);
  DFCG_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- context / streams
DeviceContext::DeviceContext(int dev) : device(dev) {
  DFCG_CUDA(cudaSetDevice(dev));
  cudaMemPool_t pool;
  DFCG_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  std::uint64_t threshold = UINT64_MAX;
  DFCG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
  // Solves share the device pool from concurrent streams: memory freed on one solve's stream
  // must not be handed to another with an inserted wait on the first stream's pending work
  // (that couples independent blocks); reuse is only stream-local, opportunistic (the free has
  // already completed) or along existing event dependencies.
  int no = 0;
  DFCG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no));
  // Reserve the pool up front (DFCG_POOL_RESERVE_GB, default 16; 0 disables): growing it maps new
  // memory under a context-wide driver lock, a stall every concurrent solve then shares.
  const char* res_env = std::getenv("DFCG_POOL_RESERVE_GB");
  const double reserve_gb = res_env ? std::atof(res_env) : 16.0;
  size_t free_b = 0, total_b = 0;
  DFCG_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const size_t reserve = static_cast<size_t>(std::min(reserve_gb * 1e9, 0.5 * static_cast<double>(free_b)));
  if (reserve > 0) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, reserve, nullptr) == cudaSuccess) {
      DFCG_CUDA(cudaFreeAsync(p, nullptr));
      DFCG_CUDA(cudaStreamSynchronize(nullptr));
    } else {
      cudaGetLastError();
    }
  }
  normals_mc = std::make_unique<NormalCache>(dev, 0x737674u, 0);
  normals_rmf = std::make_unique<NormalCache>(dev, 0x737674u, 1);
}

DeviceContext::~DeviceContext() {
  cudaSetDevice(device);
  for (cudaStream_t st : all_streams) {
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  }
}

namespace {
std::atomic<int> g_active_streams[64];
// Counts a solve as active on its device while it is stepping (RAII).
struct ActiveSolve {
  int dev;
  explicit ActiveSolve(int d) : dev(d) {
    if (dev >= 0 && dev < 64) g_active_streams[dev]++;
  }
  ~ActiveSolve() {
    if (dev >= 0 && dev < 64) g_active_streams[dev]--;
  }
};
}  // namespace
int active_streams(int dev) { return dev >= 0 && dev < 64 ? g_active_streams[dev].load() : 1; }

cudaStream_t DeviceContext::acquire() {
  std::lock_guard<std::mutex> lock(mu);
  if (!free_streams.empty()) {
    cudaStream_t st = free_streams.back();
    free_streams.pop_back();
    return st;
  }
  cudaStream_t st;
  DFCG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  all_streams.push_back(st);
  return st;
}

void DeviceContext::release(cudaStream_t st) {
  std::lock_guard<std::mutex> lock(mu);
  free_streams.push_back(st);
}

CallStream::CallStream(DeviceContext& c) : ctx(c) {
  DFCG_CUDA(cudaSetDevice(c.device));
  s = c.acquire();
}
CallStream::~CallStream() {
  cudaStreamSynchronize(s);
  ctx.release(s);
}

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

// ---------------------------------------------------------------- apg_mc
// spectral_norm (solvers.hpp:147-165) of P_Omega(M): alternating power iteration.
static double spectral_norm_omega(cudaStream_t s, const DevOmega& om) {
  const i64 m = om.m, n = om.n;
  DBuf<double> v(n, s), wv(m, s), z(n, s), nrm(1, s);
  fill_kernel<<<grid_for(n), 256, 0, s>>>(n, 1.0, v.get());
  DFCG_LAUNCH_CHECK();
  dot_sum(s, n, v.get(), v.get(), nrm.get());
  sqrt_kernel<<<1, 1, 0, s>>>(nrm.get());
  scale_by_inv_kernel<<<grid_for(n), 256, 0, s>>>(n, v.get(), nrm.get(), v.get());
  DFCG_LAUNCH_CHECK();
  double sv = 0.0, prev = 0.0;
  for (int it = 0; it < 200; ++it) {
    spmm(s, om, false, om.m_csr.get(), 1, 1.0, v.get(), 1, 0.0, wv.get(), 1);
    dot_sum(s, m, wv.get(), wv.get(), nrm.get());
    sqrt_kernel<<<1, 1, 0, s>>>(nrm.get());
    const double nw = host_scalar(s, nrm.get());
    if (nw == 0.0) return 0.0;
    scale_by_inv_kernel<<<grid_for(m), 256, 0, s>>>(m, wv.get(), nrm.get(), wv.get());
    spmm(s, om, true, om.m_csr.get(), 1, 1.0, wv.get(), 1, 0.0, z.get(), 1);
    dot_sum(s, n, z.get(), z.get(), nrm.get());
    sqrt_kernel<<<1, 1, 0, s>>>(nrm.get());
    sv = host_scalar(s, nrm.get());
    if (sv == 0.0) return 0.0;
    scale_by_inv_kernel<<<grid_for(n), 256, 0, s>>>(n, z.get(), nrm.get(), v.get());
    DFCG_LAUNCH_CHECK();
    if (std::abs(sv - prev) <= 1e-10 * sv) break;
    prev = sv;
  }
  return sv;
}

struct McSolver::State {
  DevOmega om;
  NormalCursor cur;
  DBuf<double> r_csr, r_csc;
  // P_Omega of the current / previous iterate (CSR order): by linearity P_Omega(Y) =
  // (1+beta) P_Omega(L_curr) - beta P_Omega(L_prev), so each iteration runs one SDDMM at rank
  // r (the new iterate) instead of one at the concatenated rank of Y.
  DBuf<double> pc, pp;
  DevLowRank Lp, Lc;
  double icc = 0.0;  // factored_inner(L_curr, L_curr)
  std::vector<double> last_s;
  double mu_init = 0, mu_floor = 0, tau_prev = 1.0, tau_curr = 1.0, mu = 0, mu_used = 0;
  i64 rank_hint = 1;
  // Dense-operator mode (high-rank iterations, see dense_operator()): the current / previous
  // iterates as dense column-major m x n matrices (dc_ok / dp_ok: in sync with Lc / Lp) and
  // the materialised operator.
  DBuf<double> Dc, Dp, Ad[2];
  bool dc_ok = false, dp_ok = false;
  // Compressed dense iterations: R_A, R_A^-1 of the current operator; an estimate whose left
  // factor was not formed keeps (lazy_* = index of the operator buffer Ad[] it came from, cl_*
  // = R_A^-1 U~, w x k): left = A cl.
  DBuf<double> RA, RAinv, cl_c, cl_p;
  // RA / RAinv factor the previous iteration's operator (same side): the next CholeskyQR may
  // start from them (cholqr2_r warm); ra_warm counts warm factorisations since the last cold one.
  bool ra_ok = false;
  int ra_warm = 0;
  // a refused warm pass (the operator moved too far: its Gram's smallest pivot fell below the
  // threshold) costs m w^2 FLOPs for nothing: no warm attempt for ra_skip iterations after one,
  // twice as long after each further refusal (ra_backoff)
  int ra_skip = 0, ra_backoff = 2;
  int lazy_c = -1, lazy_p = -1;
  bool wide = false;  // the deferred factor: the left one (tall, m >= n) or the right one (m < n)
  int ad_next = 0;  // Ad[] buffer the next dense iteration writes
};

// The deferred factor of an estimate produced by a compressed dense iteration: left = A cl
// (m x k, tall operator) or right = A^T cl (n x k, wide operator), A = Ad[src] row-major m x n.
static void materialize(cudaStream_t s, i64 m, i64 n, bool wide, const DBuf<double>& A, const DBuf<double>& cl,
                        DevLowRank& L) {
  if (!wide) {
    L.left.alloc(m * L.k, s);
    gemm(s, false, false, m, L.k, n, 1.0, A.get(), n, cl.get(), L.k, 0.0, L.left.get(), L.k);
  } else {
    L.right.alloc(n * L.k, s);
    gemm(s, true, false, n, L.k, m, 1.0, A.get(), n, cl.get(), L.k, 0.0, L.right.get(), L.k);
  }
}

// Whether a dense iteration compresses the operator (cost model in FLOPs, written for m >= n;
// a wide block, m < n, is compressed on its rows — OpWideQR — with m and n exchanged):
// uncompressed ~ m n (12 b + 2 r) + 5 m b^2 + 2 m b r (six products with A, the m-side
// CholQR, the left factor, the densified iterate); compressed ~ 5 m n^2 (CholeskyQR2 of A:
// two Grams and a triangular product, and the iterate as A (R_A^-1 P)). DFCG_DENSE_OP=1 / 2
// forces uncompressed / compressed (when admissible).
// Warm CholeskyQR factorisations (preconditioned by the previous iteration's R_A^-1) between two
// cold ones: P R_A - I picks up one rounding per product, a cold CholeskyQR2 resets it. Over a
// whole c2 block solve (496 iterations, profiles/r02_warmqr_full_solve.txt): runs of 8 leave
// max |R_A R_A^-1 - I| = 4.9e-11, runs of 16 6.3e-11 (no warm pass refused, smallest pivot 4.9e-3).
static const int kCholqrWarmRun =
    std::getenv("DFCG_CHOLQR_WARM_RUN") ? std::max(0, std::atoi(std::getenv("DFCG_CHOLQR_WARM_RUN"))) : 16;

static bool compress_operator(i64 m, i64 n, i64 rank_hint, bool warm = false) {
  const char* env = std::getenv("DFCG_DENSE_OP");
  const int mode = env ? std::atoi(env) : -1;
  if (mode == 1) return false;
  if (mode == 2) return true;
  const i64 lo = std::min(m, n);  // the compressed side (n for a tall block, m for a wide one)
  if (lo < 128) return false;
  const double b = static_cast<double>(std::min<i64>(rank_hint + 15, lo)), r = static_cast<double>(rank_hint);
  const double nn = static_cast<double>(lo);
  // warm: the factorisation is expected to start from the previous iteration's factor (one
  // triangular product and one Gram instead of two Grams and a triangular product)
  return 12.0 * b + 2.0 * r + 5.0 * b * b / nn + 2.0 * b * r / nn > (warm ? 4.0 : 5.0) * nn;
}

// Whether an iteration applies the SVT operator materialised (dense m x n, step 1:
// Y off Omega, M on it) instead of factored (left right^T - R with SpMM). Six applications
// per partial SVD cost 2 m n b FLOPs each dense, against 2 (m+n) kY b in the low-rank GEMMs
// plus an SpMM over N entries (gather-bound: ~8x its FLOP count at GEMM rate); the dense
// form adds one m x n x r GEMM per iteration (the new iterate) and two HBM passes. At a c2
// block at default ApgConfig (m=1e4, n=1250, N=1.25e6, kY~1440) the dense form does ~20%
// fewer FLOPs and no sparse gathers (and its compressed variant, compress_operator(), ~45%
// fewer); in the low-rank regime (kY ~ 2r ~ 60) the factored form wins. DFCG_DENSE_OP=0
// forces the factored form, 1 / 2 the dense one (tests). Not used with line search (step < 1).
static bool dense_operator(i64 m, i64 n, i64 nnz, i64 kY, bool line_search) {
  const char* env = std::getenv("DFCG_DENSE_OP");  // read per call: tests switch it in-process
  const int mode = env ? std::atoi(env) : -1;
  if (line_search || mode == 0) return false;
  const double mn = static_cast<double>(m) * static_cast<double>(n);
  if (3.0 * 8.0 * mn > 16e9) return false;  // three dense m x n buffers per solve
  if (mode >= 1) return true;
  return static_cast<double>(m + n) * static_cast<double>(kY) + 8.0 * static_cast<double>(nnz) >= mn;
}

// D (row-major m x n) = L.left L.right^T, or 0 for a zero estimate.
static void densify(cudaStream_t s, const DevLowRank& L, i64 m, i64 n, DBuf<double>& D) {
  D.ensure(m * n, s);
  if (L.k == 0) {
    D.zero(s);
    return;
  }
  gemm(s, false, true, m, n, L.k, 1.0, L.left.get(), L.k, L.right.get(), L.k, 0.0, D.get(), n);
}

McSolver::McSolver(DeviceContext& ctx, cudaStream_t s, i64 m, i64 n, i64 nnz, const long long* rows,
                   const long long* cols, const double* vals, const ApgConfig& cfg)
    : ctx_(ctx), s_(s), m_(m), n_(n), nnz_(nnz), cfg_(cfg), st_(std::make_unique<State>()) {
  start_ = std::chrono::steady_clock::now();
  if (nnz == 0) throw std::invalid_argument("apg_mc: empty observation set");
  validate_config(cfg);
  State& st = *st_;
  st.om.build(s, m, n, nnz, rows, cols, vals);
  st.mu_init = cfg.mu_init ? *cfg.mu_init : 0.99 * spectral_norm_omega(s, st.om);
  st.mu_floor = cfg.mu_floor ? *cfg.mu_floor : 1e-4 * st.mu_init;
  if (st.mu_floor > st.mu_init) throw std::invalid_argument("apg_mc: mu_floor exceeds mu_init");
  st.cur = NormalCursor{&ctx.normals(0), 0};
  st.r_csr.alloc(nnz, s);
  st.r_csc.alloc(nnz, s);
  st.pc.alloc(nnz, s);
  st.pp.alloc(nnz, s);
  st.Lp.m = st.Lc.m = m;
  st.Lp.n = st.Lc.n = n;
  st.mu = st.mu_used = st.mu_init;
}

McSolver::~McSolver() = default;

// One iteration of the apg_mc loop (solvers.hpp:275-317).
bool McSolver::step(std::vector<IterTrace>* trace) {
  if (stopped_ || iters_ >= cfg_.max_iters) return false;
  ActiveSolve busy(ctx_.device);
  prof::NvtxRange nvtx_iteration("apg_mc iteration");
  // ncu --profile-from-start off: DFCG_PROFILE_ITER=k brackets iteration k of every solve.
  static const int profile_iter = std::getenv("DFCG_PROFILE_ITER") ? std::atoi(std::getenv("DFCG_PROFILE_ITER")) : -1;
  struct ProfRange {
    bool on;
    explicit ProfRange(bool o) : on(o) {
      if (on) cudaProfilerStart();
    }
    ~ProfRange() {
      if (on) cudaProfilerStop();
    }
  } prof_range(iters_ + 1 == profile_iter);
  const auto it_start = std::chrono::steady_clock::now();
  State& st = *st_;
  cudaStream_t s = s_;
  const i64 m = m_, n = n_, nnz = nnz_;
  const int it = ++iters_;
  const double beta = (st.tau_prev - 1.0) / st.tau_curr;
  // Y = extrapolate(L_curr, L_prev, beta) as concatenated factors (no compaction).
  DevLowRank& Lc = st.Lc;
  DevLowRank& Lp = st.Lp;
  const bool concat = !(beta == 0.0 || Lp.k == 0);
  const i64 kY = concat ? Lc.k + Lp.k : Lc.k;
  const bool dense = dense_operator(m, n, nnz, kY, cfg_.line_search);
  if (!dense) {  // the factored operator needs the left factors compressed iterations deferred
    if (st.lazy_c >= 0) materialize(s, m, n, st.wide, st.Ad[st.lazy_c], st.cl_c, Lc);
    if (concat && st.lazy_p >= 0) materialize(s, m, n, st.wide, st.Ad[st.lazy_p], st.cl_p, Lp);
    if (st.lazy_c >= 0) st.lazy_c = -1;
    if (concat && st.lazy_p >= 0) st.lazy_p = -1;
  }
  bool compressed = false;
  int ai = -1;  // Ad[] buffer holding this iteration's dense operator
  if (dense) {
    // A = (1+beta) Dc - beta Dp off Omega, M on Omega (row-major m x n)
    if (!st.dc_ok) densify(s, Lc, m, n, st.Dc);
    st.dc_ok = true;
    if (concat && !st.dp_ok) {
      densify(s, Lp, m, n, st.Dp);
      st.dp_ok = true;
    }
    ai = st.ad_next;
    st.ad_next ^= 1;
    // Ad[ai] may be the source of a deferred left factor: L_curr's is formed first (it becomes
    // L_prev, which a following factored iteration needs); L_prev's is dropped with L_prev.
    if (st.lazy_c == ai) {
      materialize(s, m, n, st.wide, st.Ad[ai], st.cl_c, Lc);
      st.lazy_c = -1;
    }
    if (st.lazy_p == ai) st.lazy_p = -2;  // lost: L_prev is not used in factored form again
    st.Ad[ai].ensure(m * n, s);
    {
      prof::Scope scope(prof::kElementwise, s, 3.0 * m * n, 8.0 * m * n * (1.0 + (Lc.k > 0) + concat) + 20.0 * nnz);
      dense_extrap_kernel<<<grid_for(m * n), 256, 0, s>>>(m * n, Lc.k > 0 ? 1.0 + beta : 0.0, st.Dc.get(),
                                                          concat ? -beta : 0.0, st.Dp.get(), st.Ad[ai].get());
      DFCG_LAUNCH_CHECK();
      dense_observe_kernel<<<static_cast<int>(m), 256, 0, s>>>(n, st.om.csr_rowptr.get(), st.om.csr_col.get(),
                                                               st.om.m_csr.get(), st.Ad[ai].get());
      DFCG_LAUNCH_CHECK();
    }
    if (compress_operator(m, n, st.rank_hint, st.ra_ok && st.ra_skip == 0)) {
      const i64 lo = std::min(m, n);
      st.RA.ensure(lo * lo, s);
      st.RAinv.ensure(lo * lo, s);
      st.wide = m < n;
      const bool warm = st.ra_ok && st.ra_warm < kCholqrWarmRun && st.ra_skip == 0;
      if (st.ra_skip > 0) --st.ra_skip;
      bool used_warm = false;
      compressed = st.wide ? cholqr2_r(s, n, m, st.Ad[ai].get(), n, st.RA.get(), st.RAinv.get(), 1e-13, true, warm,
                                       &used_warm)
                           : cholqr2_r(s, m, n, st.Ad[ai].get(), n, st.RA.get(), st.RAinv.get(), 1e-13, false, warm,
                                       &used_warm);
      st.ra_warm = used_warm ? st.ra_warm + 1 : 0;
      if (warm && !used_warm) {
        st.ra_skip = st.ra_backoff;
        st.ra_backoff = std::min(2 * st.ra_backoff, 64);
      } else if (used_warm) {
        st.ra_backoff = 2;
      }
    }
  }
  st.ra_ok = compressed;  // a factor to start the next iteration's CholeskyQR from
  DBuf<double> Yl, Yr;
  const i64 ldy = std::max<i64>(1, even_ld(kY));  // even: 16-byte GEMM operand loads
  if (kY > 0 && !dense) {
    Yl.alloc(m * ldy, s);
    Yr.alloc(n * ldy, s);
    if (Lc.k > 0) {
      copy2d(s, m, Lc.k, Lc.left.get(), Lc.k, Yl.get(), ldy);
      copy2d(s, n, Lc.k, Lc.right.get(), Lc.k, Yr.get(), ldy, 1.0 + beta);
    }
    if (concat) {
      copy2d(s, m, Lp.k, Lp.left.get(), Lp.k, Yl.get() + Lc.k, ldy);
      copy2d(s, n, Lp.k, Lp.right.get(), Lp.k, Yr.get() + Lc.k, ldy, -beta);
    }
  }
  // R = P_Omega(Y) - P_Omega(M) = (1+beta) P_Omega(L_curr) - beta P_Omega(L_prev) - P_Omega(M)
  if (!dense) {
    residual_combine(s, nnz, Lc.k > 0 ? 1.0 + beta : 0.0, st.pc.get(), concat ? -beta : 0.0, st.pp.get(),
                     st.om.m_csr.get(), st.r_csr.get());
    csr_to_csc(s, st.om, st.r_csr.get(), st.r_csc.get());
  }

  double step = 1.0;
  SvtResult f;
  if (compressed && st.wide) {
    OpWideQR G{st.Ad[ai].get(), st.RA.get(), m, n};
    svt_operator(s, G, st.mu, st.rank_hint, st.cur, f);
  } else if (compressed) {
    OpTri G{st.RA.get(), n};
    svt_operator(s, G, st.mu, st.rank_hint, st.cur, f);
  } else if (dense) {
    OpDenseRM G{st.Ad[ai].get(), m, n};
    svt_operator(s, G, st.mu, st.rank_hint, st.cur, f);
  }
  for (; !dense;) {
    OpMC G{&st.om, st.r_csr.get(), st.r_csc.get(), -step, m, n, kY, Yl.get(), Yr.get(), Lc.k, ldy};
    f = SvtResult{};
    svt_operator(s, G, step * st.mu, st.rank_hint, st.cur, f);
    if (!cfg_.line_search || step <= 0.125) break;
    // backtracking majorization test (solvers.hpp:294-302)
    DBuf<double> nd(nnz, s);
    sddmm_residual(s, st.om, f.r, f.left.get(), f.r, f.right.get(), f.r, st.om.m_csr.get(), nd.get());  // next - m
    const double f_next = 0.5 * dev_dot(s, nnz, nd.get(), nd.get());
    const double rr = dev_dot(s, nnz, st.r_csr.get(), st.r_csr.get());
    const double f_y = 0.5 * rr;
    const double lin = dev_dot(s, nnz, st.r_csr.get(), nd.get()) - rr;  // sum (y-m)(next-y)
    const double d2 = factored_inner(s, m, n, f.r, f.left.get(), f.right.get(), f.r, f.left.get(), f.right.get()) -
                      2.0 * factored_inner(s, m, n, f.r, f.left.get(), f.right.get(), kY, Yl.get(), Yr.get(), 0, ldy) +
                      factored_inner(s, m, n, kY, Yl.get(), Yr.get(), kY, Yl.get(), Yr.get(), ldy, ldy);
    const double dist2 = std::sqrt(std::max(0.0, d2));
    if (f_next <= f_y + lin + dist2 * dist2 / (2.0 * step) + 1e-12) break;
    step *= 0.5;
  }
  // rel = ||L_next - L_curr|| / max(1, ||L_curr||) via factored inner products (:305-306)
  double inn, inc;
  if (dense) {
    // L_next densified (the next iteration's Dc); the factored inner products of the stop
    // test (solvers.hpp:179-193) as Frobenius inner products of the dense iterates — the
    // same quantities and the same cancellation formula below.
    std::swap(st.Dc, st.Dp);
    st.dp_ok = st.dc_ok;
    if (compressed && st.wide) {
      // f.right = V~ S (Q_B coordinates): cl = R^-1 V~ S, L_next = (left cl^T) A; the n x r
      // right factor itself is deferred (materialize) until a factored iteration or finish().
      st.Dc.ensure(m * n, s);
      DBuf<double> cl;
      if (f.r > 0) {
        cl.alloc(m * f.r, s);
        gemm_tri_a(s, false, m, f.r, 1.0, st.RAinv.get(), m, f.right.get(), f.r, 0.0, cl.get(), f.r);
        DBuf<double> T2(m * m, s);
        gemm(s, false, true, m, m, f.r, 1.0, f.left.get(), f.r, cl.get(), f.r, 0.0, T2.get(), m);
        gemm(s, false, false, m, n, m, 1.0, T2.get(), m, st.Ad[ai].get(), n, 0.0, st.Dc.get(), n);
      } else {
        st.Dc.zero(s);
      }
      f.right = DBuf<double>{};
      st.lazy_p = st.lazy_c;
      std::swap(st.cl_p, st.cl_c);
      st.cl_c = std::move(cl);
      st.lazy_c = f.r > 0 ? ai : -1;
    } else if (compressed) {
      // f.left = U~ (Q_A coordinates): cl = R_A^-1 U~, L_next = A (cl right^T); the m x r left
      // factor itself is deferred (materialize) until a factored iteration or finish().
      st.Dc.ensure(m * n, s);
      DBuf<double> cl;
      if (f.r > 0) {
        cl.alloc(n * f.r, s);
        gemm_tri_a(s, false, n, f.r, 1.0, st.RAinv.get(), n, f.left.get(), f.r, 0.0, cl.get(), f.r);
        DBuf<double> T2(n * n, s);
        gemm(s, false, true, n, n, f.r, 1.0, cl.get(), f.r, f.right.get(), f.r, 0.0, T2.get(), n);
        gemm(s, false, false, m, n, n, 1.0, st.Ad[ai].get(), n, T2.get(), n, 0.0, st.Dc.get(), n);
      } else {
        st.Dc.zero(s);
      }
      f.left = DBuf<double>{};
      st.lazy_p = st.lazy_c;
      std::swap(st.cl_p, st.cl_c);
      st.cl_c = std::move(cl);
      st.lazy_c = f.r > 0 ? ai : -1;
    } else {
      DevLowRank nx;
      nx.k = f.r;
      nx.left = std::move(f.left);
      nx.right = std::move(f.right);
      densify(s, nx, m, n, st.Dc);
      f.left = std::move(nx.left);
      f.right = std::move(nx.right);
      st.lazy_p = st.lazy_c;
      std::swap(st.cl_p, st.cl_c);
      st.lazy_c = -1;
    }
    st.dc_ok = true;
    const double* pn = st.Dc.get();
    const double* pcur = st.Dp.get();
    const bool have_c = Lc.k > 0;
    auto sums = multi_sum<2>(s, m * n, [=] __device__(i64 i, double* acc) {
      const double v = pn[i];
      acc[0] += v * v;
      if (have_c) acc[1] += v * pcur[i];
    });
    inn = f.r > 0 ? sums[0] : 0.0;
    inc = (f.r > 0 && have_c) ? sums[1] : 0.0;
  } else if (f.grams && f.r > 0) {  // m-side Grams come with the SVT result; only the n-side GEMMs remain
    DBuf<double> rr(f.r * f.r, s);
    gemm(s, true, false, f.r, f.r, n, 1.0, f.right.get(), f.r, f.right.get(), f.r, 0.0, rr.get(), f.r);
    inn = dev_dot(s, f.r * f.r, f.ll.get(), rr.get());
    inc = 0.0;
    if (Lc.k > 0) {
      DBuf<double> rc(Lc.k * f.r, s);
      gemm(s, true, false, Lc.k, f.r, n, 1.0, Lc.right.get(), Lc.k, f.right.get(), f.r, 0.0, rc.get(), f.r);
      inc = dev_dot(s, Lc.k * f.r, f.lc.get(), rc.get());
    }
  } else {
    inn = factored_inner(s, m, n, f.r, f.left.get(), f.right.get(), f.r, f.left.get(), f.right.get());
    inc = factored_inner(s, m, n, f.r, f.left.get(), f.right.get(), Lc.k, Lc.left.get(), Lc.right.get());
  }
  // P_Omega(L_next) for the next residual (pp <- pc <- new)
  std::swap(st.pc, st.pp);
  if (dense) {
    dense_gather_kernel<<<static_cast<int>(m), 256, 0, s>>>(n, st.om.csr_rowptr.get(), st.om.csr_col.get(),
                                                            st.Dc.get(), st.pc.get());
    DFCG_LAUNCH_CHECK();
  } else {
    if (f.r > 0) sddmm_residual(s, st.om, f.r, f.left.get(), f.r, f.right.get(), f.r, nullptr, st.pc.get());
    // the dense copies (if any) shift with the iterates: old Dc is the new Dp
    std::swap(st.Dc, st.Dp);
    st.dp_ok = st.dc_ok;
    st.dc_ok = false;
    st.lazy_p = st.lazy_c;
    std::swap(st.cl_p, st.cl_c);
    st.lazy_c = -1;
  }
  const double d2 = inn - 2.0 * inc + st.icc;
  const double rel = std::sqrt(std::max(0.0, d2)) / std::max(1.0, std::sqrt(std::max(0.0, st.icc)));
  const double tau_next = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * st.tau_curr * st.tau_curr));
  Lp = std::move(Lc);
  Lc = DevLowRank{};
  Lc.m = m;
  Lc.n = n;
  Lc.k = f.r;
  Lc.left = std::move(f.left);
  Lc.right = std::move(f.right);
  st.icc = inn;
  st.last_s = f.s;
  st.tau_prev = st.tau_curr;
  st.tau_curr = tau_next;
  st.rank_hint = std::max<i64>(1, Lc.k);
  st.mu_used = st.mu;
  if (trace) trace->push_back({it, Lc.k, f.k_final, f.calls, rel, st.mu, sum_of(st.last_s), ms_since(it_start)});
  st.mu = std::max(cfg_.mu_decay * st.mu, st.mu_floor);
  if (rel < cfg_.rel_tol) stopped_ = true;
  return true;
}

// Report (solvers.hpp:319-326); the estimate is copied so the solver can keep stepping.
void McSolver::finish(DevLowRank& out, SolveReport& rep) {
  State& st = *st_;
  cudaStream_t s = s_;
  if (st.lazy_c >= 0) {
    materialize(s, m_, n_, st.wide, st.Ad[st.lazy_c], st.cl_c, st.Lc);
    st.lazy_c = -1;
  }
  const DevLowRank& Lc = st.Lc;
  rep.iterations = iters_;
  rep.rank = Lc.k;
  DBuf<double> fin(nnz_, s);
  residual_combine(s, nnz_, Lc.k > 0 ? 1.0 : 0.0, st.pc.get(), 0.0, st.pp.get(), st.om.m_csr.get(), fin.get());
  rep.residual = std::sqrt(dev_dot(s, nnz_, fin.get(), fin.get()));
  rep.objective = st.mu_used * sum_of(st.last_s) + 0.5 * rep.residual * rep.residual;
  out = DevLowRank{};
  out.m = m_;
  out.n = n_;
  out.k = Lc.k;
  if (Lc.k > 0) {
    out.left.alloc(m_ * Lc.k, s);
    out.right.alloc(n_ * Lc.k, s);
    copy2d(s, m_, Lc.k, Lc.left.get(), Lc.k, out.left.get(), Lc.k);
    copy2d(s, n_, Lc.k, Lc.right.get(), Lc.k, out.right.get(), Lc.k);
  }
  DFCG_CUDA(cudaStreamSynchronize(s));
  rep.wall_ms = ms_since(start_);
}

void apg_mc_device(DeviceContext& ctx, cudaStream_t s, i64 m, i64 n, i64 nnz, const long long* rows,
                   const long long* cols, const double* vals, const ApgConfig& cfg, DevLowRank& out, SolveReport& rep,
                   std::vector<IterTrace>* trace) {
  McSolver solver(ctx, s, m, n, nnz, rows, cols, vals, cfg);
  while (solver.step(trace)) {
  }
  solver.finish(out, rep);
}

// ---------------------------------------------------------------- apg_rmf
void apg_rmf_device(DeviceContext& ctx, cudaStream_t s, const double* M_colmajor, i64 m, i64 n, double lambda,
                    const ApgConfig& cfg, DevLowRank& out, std::vector<long long>& s_row, std::vector<long long>& s_col,
                    std::vector<double>& s_val, SolveReport& rep, std::vector<IterTrace>* trace) {
  const auto start = std::chrono::steady_clock::now();
  ActiveSolve busy(ctx.device);
  if (!(lambda > 0)) throw std::invalid_argument("apg_rmf: lambda must be positive");
  const i64 mn = m * n;
  for (i64 i = 0; i < mn; ++i)
    if (!std::isfinite(M_colmajor[i])) throw std::invalid_argument("apg_rmf: non-finite input");
  validate_config(cfg);
  // Dense m x n matrices are kept column-major (== row-major n x m), like the input.
  DBuf<double> M(mn, s), Ld(mn, s), Ldp(mn, s), Sc(mn, s), Sp(mn, s), GL(mn, s), Sn(mn, s), Ldn(mn, s);
  DFCG_CUDA(cudaMemcpyAsync(M.get(), M_colmajor, sizeof(double) * mn, cudaMemcpyHostToDevice, s));
  Ld.zero(s);
  Ldp.zero(s);
  Sc.zero(s);
  Sp.zero(s);

  auto spectral = [&]() {  // dense power iteration on M (m x n)
    DBuf<double> v(n, s), wv(m, s), z(n, s), nrm(1, s);
    fill_kernel<<<grid_for(n), 256, 0, s>>>(n, 1.0, v.get());
    DFCG_LAUNCH_CHECK();
    dot_sum(s, n, v.get(), v.get(), nrm.get());
    sqrt_kernel<<<1, 1, 0, s>>>(nrm.get());
    scale_by_inv_kernel<<<grid_for(n), 256, 0, s>>>(n, v.get(), nrm.get(), v.get());
    double sv = 0.0, prev = 0.0;
    for (int it = 0; it < 200; ++it) {
      gemm(s, true, false, m, 1, n, 1.0, M.get(), m, v.get(), 1, 0.0, wv.get(), 1);  // M v
      dot_sum(s, m, wv.get(), wv.get(), nrm.get());
      sqrt_kernel<<<1, 1, 0, s>>>(nrm.get());
      const double nw = host_scalar(s, nrm.get());
      if (nw == 0.0) return 0.0;
      scale_by_inv_kernel<<<grid_for(m), 256, 0, s>>>(m, wv.get(), nrm.get(), wv.get());
      gemm(s, false, false, n, 1, m, 1.0, M.get(), m, wv.get(), 1, 0.0, z.get(), 1);  // M^T w
      dot_sum(s, n, z.get(), z.get(), nrm.get());
      sqrt_kernel<<<1, 1, 0, s>>>(nrm.get());
      sv = host_scalar(s, nrm.get());
      if (sv == 0.0) return 0.0;
      scale_by_inv_kernel<<<grid_for(n), 256, 0, s>>>(n, z.get(), nrm.get(), v.get());
      DFCG_LAUNCH_CHECK();
      if (std::abs(sv - prev) <= 1e-10 * sv) break;
      prev = sv;
    }
    return sv;
  };
  const double mu_init = cfg.mu_init ? *cfg.mu_init : 0.99 * spectral();
  const double mu_floor = cfg.mu_floor ? *cfg.mu_floor : 1e-4 * mu_init;
  if (mu_floor > mu_init) throw std::invalid_argument("apg_rmf: mu_floor exceeds mu_init");

  NormalCursor cur{&ctx.normals(1), 0};
  SvtResult last;
  DBuf<double> RA, RAinv, cl_last;  // compressed iterations (see below)
  bool ra_ok = false;               // RA / RAinv factor the previous iteration's operator
  int ra_warm = 0, ra_skip = 0, ra_backoff = 2;  // as in McSolver::State
  bool left_deferred = false;
  double tau_prev = 1.0, tau_curr = 1.0, mu = mu_init, mu_used = mu_init;
  i64 rank_hint = 1;
  int iters = 0;
  const int gb = grid_for(mn);
  DBuf<double> YL, YS, Gd;
  if (cfg.line_search) {
    YL.alloc(mn, s);
    YS.alloc(mn, s);
    Gd.alloc(mn, s);
  }
  auto it_start = std::chrono::steady_clock::now();
  for (int it = 1; it <= cfg.max_iters; ++it) {
    iters = it;
    const double beta = (tau_prev - 1.0) / tau_curr;
    double step = 0.5;
    SvtResult f;
    if (cfg.line_search) {
      rmf_extrap_kernel<<<gb, 256, 0, s>>>(mn, beta, Ld.get(), Ldp.get(), Sc.get(), Sp.get(), M.get(), YL.get(),
                                           YS.get(), Gd.get());
      DFCG_LAUNCH_CHECK();
    }
    for (;;) {
      {
        prof::Scope scope(prof::kElementwise, s, 10.0 * mn, (cfg.line_search ? 5.0 : 7.0) * 8.0 * mn);
        if (cfg.line_search) {
          rmf_step_kernel<<<gb, 256, 0, s>>>(mn, step, step * lambda * mu, YL.get(), YS.get(), Gd.get(), GL.get(),
                                             Sn.get());
        } else {
          rmf_fused_kernel<<<gb, 256, 0, s>>>(mn, beta, step, step * lambda * mu, Ld.get(), Ldp.get(), Sc.get(),
                                              Sp.get(), M.get(), GL.get(), Sn.get());
        }
        DFCG_LAUNCH_CHECK();
      }
      f = SvtResult{};
      // The dense operator GL (column-major m x n) compressed by CholeskyQR2 when tall and the
      // cost model says so (OpTri, as in apg_mc): the SVT runs on R_A, the next L_d is
      // GL (R_A^-1 U~ S V^T) and the left factor is deferred (only the last one is output).
      bool compressed = false;
      if (!cfg.line_search && m >= n && compress_operator(m, n, rank_hint, ra_ok && ra_skip == 0)) {
        RA.ensure(n * n, s);
        RAinv.ensure(n * n, s);
        bool used_warm = false;
        const bool warm = ra_ok && ra_warm < kCholqrWarmRun && ra_skip == 0;
        if (ra_skip > 0) --ra_skip;
        compressed = cholqr2_r(s, m, n, GL.get(), m, RA.get(), RAinv.get(), 1e-13, true, warm, &used_warm);
        ra_warm = used_warm ? ra_warm + 1 : 0;
        if (warm && !used_warm) {
          ra_skip = ra_backoff;
          ra_backoff = std::min(2 * ra_backoff, 64);
        } else if (used_warm) {
          ra_backoff = 2;
        }
      }
      ra_ok = compressed;
      if (compressed) {
        OpTri op{RA.get(), n};
        svt_operator(s, op, step * mu, rank_hint, cur, f);
        cl_last = DBuf<double>{};
        if (f.r > 0) {
          cl_last.alloc(n * f.r, s);
          gemm_tri_a(s, false, n, f.r, 1.0, RAinv.get(), n, f.left.get(), f.r, 0.0, cl_last.get(), f.r);
          DBuf<double> T2(n * n, s);
          gemm(s, false, true, n, n, f.r, 1.0, cl_last.get(), f.r, f.right.get(), f.r, 0.0, T2.get(), n);
          // L_d (column-major == row-major n x m) = T2^T GL^T
          gemm(s, true, false, n, m, n, 1.0, T2.get(), n, GL.get(), m, 0.0, Ldn.get(), m);
        } else {
          Ldn.zero(s);
        }
        f.left = DBuf<double>{};
        left_deferred = f.r > 0;
      } else {
        OpDense op{GL.get(), m, n};
        svt_operator(s, op, step * mu, rank_hint, cur, f);
        left_deferred = false;
        // Ld_next = U diag(s) V^T  (column-major m x n == row-major n x m: V diag(s) U^T)
        if (f.r == 0) {
          Ldn.zero(s);
        } else {
          gemm(s, false, true, n, m, f.r, 1.0, f.right.get(), f.r, f.left.get(), f.r, 0.0, Ldn.get(), m);
        }
      }
      if (!cfg.line_search || step <= 0.0625) break;
      const double* pM = M.get();
      const double* pLn = Ldn.get();
      const double* pSn = Sn.get();
      const double* pYL = YL.get();
      const double* pYS = YS.get();
      const double* pG = Gd.get();
      auto sums = multi_sum<4>(s, mn, [=] __device__(i64 i, double* acc) {
        const double r = pM[i] - pLn[i] - pSn[i];
        const double g = pG[i];
        const double dl = pLn[i] - pYL[i], ds = pSn[i] - pYS[i];
        acc[0] += r * r;
        acc[1] += g * g;
        acc[2] += g * (dl + ds);
        acc[3] += dl * dl + ds * ds;
      });
      if (0.5 * sums[0] <= 0.5 * sums[1] + sums[2] + sums[3] / (2.0 * step) + 1e-12) break;
      step *= 0.5;
    }
    const double* pLd = Ld.get();
    const double* pLn = Ldn.get();
    const double* pSc = Sc.get();
    const double* pSn = Sn.get();
    auto sums = multi_sum<4>(s, mn, [=] __device__(i64 i, double* acc) {
      const double dl = pLn[i] - pLd[i], ds = pSn[i] - pSc[i];
      acc[0] += dl * dl;
      acc[1] += ds * ds;
      acc[2] += pLd[i] * pLd[i];
      acc[3] += pSc[i] * pSc[i];
    });
    const double denom = std::max(1.0, std::sqrt(sums[2] + sums[3]));
    const double rel = std::sqrt(sums[0] + sums[1]) / denom;
    const double tau_next = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * tau_curr * tau_curr));
    std::swap(Ldp, Ld);
    std::swap(Ld, Ldn);  // Ld <- next, Ldn <- old prev (scratch)
    std::swap(Sp, Sc);
    std::swap(Sc, Sn);
    last = std::move(f);
    tau_prev = tau_curr;
    tau_curr = tau_next;
    rank_hint = std::max<i64>(1, last.r);
    mu_used = mu;
    if (trace) trace->push_back({it, last.r, last.k_final, last.calls, rel, mu, sum_of(last.s), ms_since(it_start)});
    it_start = std::chrono::steady_clock::now();
    mu = std::max(cfg.mu_decay * mu, mu_floor);
    if (rel < cfg.rel_tol) break;
  }
  // outputs (solvers.hpp:398-413)
  const double* pM = M.get();
  const double* pLd = Ld.get();
  const double* pSc = Sc.get();
  auto sums = multi_sum<2>(s, mn, [=] __device__(i64 i, double* acc) {
    const double r = pM[i] - pLd[i] - pSc[i];
    acc[0] += r * r;
    acc[1] += fabs(pSc[i]);
  });
  rep.iterations = iters;
  rep.rank = last.r;
  rep.residual = std::sqrt(sums[0]);
  rep.objective =
      sum_of(last.s) + lambda * sums[1] + (mu_used > 0 ? rep.residual * rep.residual / (2.0 * mu_used) : 0.0);
  std::vector<double> hS(mn);
  DFCG_CUDA(cudaMemcpyAsync(hS.data(), Sc.get(), sizeof(double) * mn, cudaMemcpyDeviceToHost, s));
  DFCG_CUDA(cudaStreamSynchronize(s));
  s_row.clear();
  s_col.clear();
  s_val.clear();
  for (i64 j = 0; j < n; ++j)
    for (i64 i = 0; i < m; ++i) {
      const double v = hS[j * m + i];
      if (v != 0.0) {
        s_row.push_back(i);
        s_col.push_back(j);
        s_val.push_back(v);
      }
    }
  out = DevLowRank{};
  out.m = m;
  out.n = n;
  out.k = last.r;
  if (left_deferred) {  // the last iteration's left factor: GL R_A^-1 U~ (GL is that iteration's)
    last.left.alloc(m * last.r, s);
    gemm(s, true, false, m, last.r, n, 1.0, GL.get(), m, cl_last.get(), last.r, 0.0, last.left.get(), last.r);
  }
  out.left = std::move(last.left);
  out.right = std::move(last.right);
  rep.wall_ms = ms_since(start);
}

// ---------------------------------------------------------------- transfers
void upload_lowrank(cudaStream_t s, const HostLowRank& h, DevLowRank& d) {
  d = DevLowRank{};
  d.m = h.m;
  d.n = h.n;
  d.k = h.k;
  if (h.k == 0) return;
  DBuf<double> tl(h.m * h.k, s), tr(h.n * h.k, s);
  d.left.alloc(h.m * h.k, s);
  d.right.alloc(h.n * h.k, s);
  DFCG_CUDA(cudaMemcpyAsync(tl.get(), h.left.data(), sizeof(double) * h.m * h.k, cudaMemcpyHostToDevice, s));
  DFCG_CUDA(cudaMemcpyAsync(tr.get(), h.right.data(), sizeof(double) * h.n * h.k, cudaMemcpyHostToDevice, s));
  // column-major m x k == row-major k x m
  transpose(s, h.k, h.m, tl.get(), h.m, d.left.get(), h.k);
  transpose(s, h.k, h.n, tr.get(), h.n, d.right.get(), h.k);
  DFCG_CUDA(cudaStreamSynchronize(s));
}

void download_lowrank(cudaStream_t s, const DevLowRank& d, HostLowRank& h) {
  h.m = d.m;
  h.n = d.n;
  h.k = d.k;
  h.left.assign(static_cast<size_t>(d.m * d.k), 0.0);
  h.right.assign(static_cast<size_t>(d.n * d.k), 0.0);
  if (d.k == 0) return;
  DBuf<double> tl(d.m * d.k, s), tr(d.n * d.k, s);
  transpose(s, d.m, d.k, d.left.get(), d.k, tl.get(), d.m);
  transpose(s, d.n, d.k, d.right.get(), d.k, tr.get(), d.n);
  DFCG_CUDA(cudaMemcpyAsync(h.left.data(), tl.get(), sizeof(double) * d.m * d.k, cudaMemcpyDeviceToHost, s));
  DFCG_CUDA(cudaMemcpyAsync(h.right.data(), tr.get(), sizeof(double) * d.n * d.k, cudaMemcpyDeviceToHost, s));
  DFCG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace dfcg
