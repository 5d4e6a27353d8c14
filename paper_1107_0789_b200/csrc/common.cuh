// Shared device utilities for the DFC B200 library (FP64 throughout).
//
// Conventions: every dense matrix on the device is ROW-MAJOR ("C order") with an
// explicit leading dimension, so factor rows are contiguous for the SDDMM gathers
// and sketch rows are contiguous for the SpMM gathers. The C ABI converts from the
// reference's column-major Eigen layout (P/include/dfc/matrix_io.hpp:19) at the edge.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "prof.hpp"

namespace dfcg {

using i64 = std::int64_t;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define DFCG_CUDA(call)                                                                          \
  do {                                                                                           \
    cudaError_t e_ = (call);                                                                     \
    if (e_ != cudaSuccess)                                                                       \
      throw ::dfcg::CudaError(std::string(#call) + " failed: " + cudaGetErrorString(e_) + " at " + \
                              __FILE__ + ":" + std::to_string(__LINE__));                        \
  } while (0)

#define DFCG_LAUNCH_CHECK()             \
  do {                                  \
    ::dfcg::prof::count_launch();       \
    DFCG_CUDA(cudaGetLastError());      \
  } while (0)

inline int cdiv(i64 a, i64 b) { return static_cast<int>((a + b - 1) / b); }

// Bit of `dev` in a per-device flag word (one-time kernel attribute opt-ins). The flag words
// are std::atomic<std::uint64_t>: concurrent first callers may both run the (idempotent)
// setup, then set the bit; ordinals >= 64 are rejected instead of shifting out of range.
inline std::uint64_t dev_bit(int dev) {
  if (dev < 0 || dev >= 64) throw std::runtime_error("device ordinal outside [0, 64)");
  return std::uint64_t{1} << dev;
}

// Stream-ordered device buffer (cudaMallocAsync from the device's default pool,
// whose release threshold is raised at context creation so reuse is cheap).
template <class T>
class DBuf {
 public:
  DBuf() = default;
  DBuf(i64 n, cudaStream_t s) { alloc(n, s); }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { *this = std::move(o); }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      s_ = o.s_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  void alloc(i64 n, cudaStream_t s) {
    release();
    s_ = s;
    n_ = n;
    if (n > 0) DFCG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), sizeof(T) * static_cast<size_t>(n), s));
  }
  // Grow-only reallocation (contents not preserved).
  void ensure(i64 n, cudaStream_t s) {
    if (n > n_ || p_ == nullptr) alloc(std::max<i64>(n, 1), s);
  }
  void release() {
    if (p_) cudaFreeAsync(p_, s_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  i64 size() const { return n_; }
  void zero(cudaStream_t s) const {
    if (n_ > 0) DFCG_CUDA(cudaMemsetAsync(p_, 0, sizeof(T) * static_cast<size_t>(n_), s));
  }

 private:
  T* p_ = nullptr;
  i64 n_ = 0;
  cudaStream_t s_ = nullptr;
};

// ---------------------------------------------------------------- dense kernels (dense.cu)
// C[MxN] = alpha * op(A)[MxK] * op(B)[KxN] + beta * C, all row-major.
//   !ta: A(i,k) = A[i*lda + k]      ta: A(i,k) = A[k*lda + i]
//   !tb: B(k,j) = B[k*ldb + j]      tb: B(k,j) = B[j*ldb + k]
// FP64 DMMA (mma.sync m8n8k4), cp.async multi-stage pipeline, deterministic split-K.
void gemm(cudaStream_t s, bool ta, bool tb, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda,
          const double* B, i64 ldb, double beta, double* C, i64 ldc);

// Upper triangle (tiles on or above the diagonal) of G = X^T X, X rows x cols row-major; the
// strictly-lower tiles of G are not written (SYRK: half the Gram FLOPs).
// C = alpha A B + beta C with B (N x N) upper triangular, its lower part stored as zeros (the
// diagonal tiles read it): the K loop of each column tile stops at the diagonal — half the
// FLOPs of gemm.
void gemm_upper_b(cudaStream_t s, i64 M, i64 N, double alpha, const double* A, i64 lda, const double* B, i64 ldb,
                  double beta, double* C, i64 ldc);
void gram_upper(cudaStream_t s, i64 rows, i64 cols, const double* X, i64 ldx, double* G, i64 ldg);
// C (M x N) = alpha op(A) B + beta C for an upper-triangular M x M matrix A (lower part stored
// as zeros): op(A) = A (ta = false) or A^T (ta = true); the K loop of each row tile skips the
// zero half (half the FLOPs).
void gemm_tri_a(cudaStream_t s, bool ta, i64 M, i64 N, double alpha, const double* A, i64 lda, const double* B,
                i64 ldb, double beta, double* C, i64 ldc);
// Upper triangle of G = A A^T (rows x rows), A row-major rows x k.
void gram_upper_nt(cudaStream_t s, i64 rows, i64 k, const double* A, i64 lda, double* G, i64 ldg);
// C (M x N) = alpha A^T B + beta C with A stored row-major N x M (A^T(i,k) = A[k*lda + i]) and
// B (N x N) upper triangular (lower part stored as zeros): the TRMM of a transposed operand.
void gemm_ta_upper_b(cudaStream_t s, i64 M, i64 N, double alpha, const double* A, i64 lda, const double* B, i64 ldb,
                     double beta, double* C, i64 ldc);

// dst (rows x cols, ldd) = alpha * src (rows x cols, lds)  [alpha may be 1]
void copy2d(cudaStream_t s, i64 rows, i64 cols, const double* src, i64 lds, double* dst, i64 ldd, double alpha = 1.0);
// dst (cols x rows, ldd) = src^T  (src rows x cols, lds)
void transpose(cudaStream_t s, i64 rows, i64 cols, const double* src, i64 lds, double* dst, i64 ldd);
// Set a rows x cols block to the identity pattern (ones on the diagonal).
void set_identity(cudaStream_t s, i64 rows, i64 cols, double* dst, i64 ldd);
// out = sum(a .* b) over n elements, deterministic (fixed-shape tree).  out is a device scalar.
void dot_sum(cudaStream_t s, i64 n, const double* a, const double* b, double* out);
// Columns gather+scale: dst[:, c] = src[:, idx[c]] * (scale ? scale[c] : 1), rows x ncols, row-major.
void gather_cols(cudaStream_t s, i64 rows, i64 ncols, const double* src, i64 lds, const int* idx,
                 const double* scale, double* dst, i64 ldd);
// Column norms of a row-major rows x cols matrix: out[c] = ||src[:, c]||_2 (deterministic).
void col_norms(cudaStream_t s, i64 rows, i64 cols, const double* src, i64 lds, double* out);

// ---------------------------------------------------------------- cp.async helpers (device)
// 8-byte copies go through L1 (.ca), 16-byte ones bypass it (.cg); pred == false zero-fills.
#ifdef __CUDACC__
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem), "r"(pred ? 8 : 0));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem), "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
#endif

// out[i] = sqrt(-2 log(u1)) cos(2 pi u2), u1 = ((raw[2i] >> 11) + 1) 2^-53, u2 = (raw[2i+1] >> 11)
// 2^-53: SeededRng::normal (P/include/dfc/rng.hpp:62-66) on raw mt19937_64 words, on the device.
void box_muller_device(cudaStream_t s, const std::uint64_t* raw, double* out, i64 n);

// Programmatic dependent launch (PDL): a kernel launched with pdl_launch may begin while its
// stream predecessor is still running; it must call pdl_wait() before it touches any global
// memory the predecessor reads or writes (the wait returns once the predecessor grid has
// completed and its writes are visible), and may call pdl_trigger() to let its own successor
// launch early. Hides the launch gap of the latency-bound chains (blocked Cholesky, small GEMMs,
// Jacobi rounds) of a solve that has the GPU to itself (see pdl_enabled(), dense.cu).
bool pdl_enabled();
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::); }
template <typename... KArgs, typename... Args>
void pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  DFCG_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}
#endif

// APG solves currently stepping on device `dev`: kernels with a latency / occupancy trade-off
// (the Jacobi cluster size) consult it.
int active_streams(int dev);

// ---------------------------------------------------------------- factorizations (factor.cu)
struct Workspace;  // forward

// Thin QR of a row-major rows x cols matrix X (rows >= cols): X = Q R, Q overwrites X,
// R (cols x cols, row-major, upper) written when R != nullptr. CholeskyQR2 fast path
// with a blocked Householder fallback when the Gram factor is too ill-conditioned.
// Returns true when the Householder fallback ran.
// passes = 1 gives a well-conditioned basis of span(X) (orthogonality ~ eps cond(X)^2),
// enough for the intermediate bases of the range finder; passes = 2 is CholeskyQR2.
bool thin_qr(cudaStream_t s, i64 rows, i64 cols, double* X, i64 ldx, double* R, i64 ldr, int passes = 2);
// One CholQR factor without forming Q: Rinv = R^-1 (upper, lower part zero) with
// R^T R = X^T X, so X Rinv has orthonormal columns to ~eps cond(X)^2. Returns false (Rinv
// unusable) when a Cholesky pivot signals cond(X) >~ 3e5.
bool cholqr_factor(cudaStream_t s, i64 rows, i64 cols, const double* X, i64 ldx, double* Rinv, i64 ldr);
// CholeskyQR2 R factor of a tall row-major rows x cols matrix A (A = Q R, Q orthonormal and
// never formed beyond the first pass): R (cols x cols, upper, lower part zero) and Rinv = R^-1.
// rel_tol1: breakdown threshold of the first pass's (Jacobi-scaled) Cholesky pivots. Returns
// false on breakdown (cond(A) too large for CholeskyQR2); R / Rinv are then unusable.
// trans: the tall matrix is A^T, A stored row-major cols x rows (lda).
// warm: R / Rinv hold the factor of the previous (nearby) operator on entry; it preconditions a
// single pass (see the definition). *used_warm reports whether that pass was accepted.
bool cholqr2_r(cudaStream_t s, i64 rows, i64 cols, const double* A, i64 lda, double* R, double* Rinv,
               double rel_tol1, bool trans = false, bool warm = false, bool* used_warm = nullptr);
// Householder QR only (tests / fallback).
void householder_qr(cudaStream_t s, i64 rows, i64 cols, double* X, i64 ldx, double* R, i64 ldr);

// Thin SVD of a row-major rows x cols matrix A (rows >= cols; A is left intact).
//   U (rows x cols, ldu), V (cols x cols, ldv), singular values sorted nonincreasing (host
//   copy returned in s_host).
// Method: columns sorted by norm, thin QR (CholQR2 / Householder fallback), one-sided block
// Jacobi on R^T (QR-preconditioned Jacobi; few sweeps since R^T is graded).
// u_tau > 0 promises that only the triplets with sigma > u_tau are used: U may then be
// recovered as A V Sigma^-1 instead of accumulating the rotations (columns with sigma <= u_tau
// are not accurate in that mode).
void thin_svd(cudaStream_t s, i64 rows, i64 cols, double* A, i64 lda, double* U, i64 ldu, double* V, i64 ldv,
              std::vector<double>& s_host, double u_tau = 0.0);

}  // namespace dfcg
