// Dense FP64 factorizations on the device: thin QR and thin SVD.
//
// thin_qr  (stands in for Eigen HouseholderQR in thin_qr, P/include/dfc/sketch.hpp:41-47):
//   CholeskyQR2 — Gram by DMMA GEMM, blocked Cholesky (64x64 diagonal blocks in shared
//   memory, TRSM/SYRK as GEMMs), explicit triangular inverse, Q = X R^-1 as one GEMM —
//   repeated twice. When a Cholesky pivot signals cond(X) > ~3e5 (or rank deficiency), the
//   call falls back to blocked Householder QR (panel kernel + compact-WY GEMM updates),
//   which is what the reference computes. Only span(Q) matters downstream: every consumer
//   (randomized range finder, svd_of_product) is invariant to the choice of basis.
// thin_svd (stands in for Eigen BDCSVD, sketch.hpp:57-86, solvers.hpp:90-93):
//   optional QR preconditioning, then one-sided block Jacobi (16-column blocks, round-robin
//   pair ordering, Gram/update by DMMA, inner 32x32 symmetric Jacobi in shared memory).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <numeric>

#include <mutex>
#include <unordered_map>

#include "common.cuh"

#include <cooperative_groups.h>
#include <map>
#include <tuple>
namespace cg = cooperative_groups;

namespace dfcg {

namespace {

int grid_for(i64 total, int threads = 256) {
  return static_cast<int>(std::max<i64>(1, std::min<i64>((total + threads - 1) / threads, 4096)));
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Reciprocal square root from the MUFU seed plus two Newton steps (seed ~2^-22 relative -> full
// double precision): ~half the dependent instructions of the IEEE-rounded sequence.
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  double e = fma(-h * y, y, 0.5);  // y <- y (1.5 - x y^2 / 2)
  y = fma(y, e, y);
  e = fma(-h * y, y, 0.5);
  return fma(y, e, y);
}

// ================================================================ Cholesky (upper, G = R^T R)
constexpr int CNB = 64;

__global__ void diag_max_kernel(i64 n, const double* G, i64 ldg, double* out) {
  __shared__ double sh[256];
  double m = 0.0;
  for (i64 i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, G[i * ldg + i]);
  sh[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// Factor the kb x kb (kb <= CNB = 64) diagonal block at (k0,k0) in place (upper R, lower part
// zeroed) and write R^-1 into Rinv. One CTA of 8 warps, the block resident in shared memory,
// processed in 8-column micro-panels:
//   factor  warp 0 factors the 8x8 diagonal micro-block warp-synchronously (lane j owns
//           column j in registers, pivots and row k of R broadcast by shuffles, no barriers);
//   trsm    one thread per column right of the micro-panel solves R_D^T x = a (8 steps);
//   update  4x4 register tiles apply the rank-8 update to the trailing upper triangle.
// The inverse: warp w inverts diagonal micro-block w, then recursive doubling over block
// pairs, X12 = -X11 (R12 X22), with all pairs of a level in parallel (6 barriers at kb = 64).
// Pivots below rel_tol * maxdiag set *fail (the caller falls back to Householder QR).
constexpr int PB = 8;  // micro-panel width
constexpr int PLD = CNB + 1;
constexpr size_t kPotrfSmem = sizeof(double) * (2 * CNB * PLD + (CNB / 2) * PLD + CNB);

#ifdef DFCG_POTRF_TRACE  // phase timestamps for tools/potrf_bench.cu
__device__ long long g_potrf_trace[64];
#define POTRF_STAMP(i)                \
  if (threadIdx.x == 0) {             \
    const long long now_ = clock64(); \
    g_potrf_trace[i] += now_ - tp_;   \
    tp_ = now_;                       \
  }
#else
#define POTRF_STAMP(i)
#endif
// The 64x64 diagonal-block factorisation as a device function (256 threads, kPotrfSmem of
// shared memory at psm): used by potrf_diag_kernel and by the fused cooperative Cholesky.
// G is read through L2 (__ldcg): in the fused kernel other CTAs wrote it since the last grid sync.
__device__ void potrf_tile(int kb, double* G, i64 ldg, double* Rinv, i64 ldr, const double* maxdiag, double rel_tol,
                           int* fail, int want_inv, double* psm) {
#ifdef DFCG_POTRF_TRACE
  long long tp_ = clock64();
#endif
  double(*A)[PLD] = reinterpret_cast<double(*)[PLD]>(psm);                // R (upper)
  double(*X)[PLD] = reinterpret_cast<double(*)[PLD]>(psm + CNB * PLD);    // R^-1 (upper)
  double(*S)[PLD] = reinterpret_cast<double(*)[PLD]>(psm + 2 * CNB * PLD);  // doubling scratch (CNB/2 rows)
  double* dinv = psm + 2 * CNB * PLD + (CNB / 2) * PLD;                    // 1 / r_kk
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int kbp = (kb + PB - 1) / PB * PB;  // micro-panels that hold real columns
  {  // all loads first (unconditional, address clamped), then the stores: every load in flight
    double v[CNB * CNB / 256];
#pragma unroll
    for (int it = 0; it < CNB * CNB / 256; ++it) {
      const int e = t + 256 * it, r = e / CNB, c = e % CNB;
      const bool ok = r < kb && c < kb && r <= c;
      v[it] = __ldcg(G + (ok ? r * ldg + c : 0));
    }
#pragma unroll
    for (int it = 0; it < CNB * CNB / 256; ++it) {
      const int e = t + 256 * it, r = e / CNB, c = e % CNB;
      const bool ok = r < kb && c < kb && r <= c;
      A[r][c] = ok ? v[it] : (r == c && r >= kb ? 1.0 : 0.0);
      X[r][c] = 0.0;
    }
  }
  const double thr = rel_tol * __ldcg(maxdiag);
  __syncthreads();
  POTRF_STAMP(1)
  for (int c0 = 0; c0 < kbp; c0 += PB) {
    if (warp == 0) {  // ---- factor the 8x8 diagonal micro-block
      // every lane factors the whole upper triangle in registers (no shuffles on the pivot
      // chain); lane j < 8 then stores column j
      double a[PB][PB], ipv[PB];
#pragma unroll
      for (int i = 0; i < PB; ++i)
#pragma unroll
        for (int j = i; j < PB; ++j) a[i][j] = A[c0 + i][c0 + j];
#pragma unroll
      for (int k = 0; k < PB; ++k) {
        const double piv = a[k][k];
        const bool bad = c0 + k < kb && (!(piv > thr) || !isfinite(piv));
        const double pv = bad ? 1.0 : piv;
        const double ip = rsqrt_nr(pv);
        if (bad) *fail = 1;  // warp-uniform (every lane holds the same block)
        a[k][k] = pv * ip;
        ipv[k] = ip;
#pragma unroll
        for (int j = k + 1; j < PB; ++j) a[k][j] *= ip;
#pragma unroll
        for (int i = k + 1; i < PB; ++i)
#pragma unroll
          for (int j = i; j < PB; ++j) a[i][j] = fma(-a[k][i], a[k][j], a[i][j]);
      }
      if (lane == 0) {  // one writer: stores are cheap next to divergent per-lane column writes
#pragma unroll
        for (int i = 0; i < PB; ++i) dinv[c0 + i] = ipv[i];
#pragma unroll
        for (int i = 0; i < PB; ++i) {
#pragma unroll
          for (int j = i; j < PB; ++j) A[c0 + i][c0 + j] = a[i][j];
        }
      }
    }
    __syncthreads();
    POTRF_STAMP(6)
    const int c1 = c0 + PB, n2 = kbp - c1;
    if (n2 == 0) break;
    if (t < n2) {  // ---- panel: R[c0:c1, c] = R_D^-T A[c0:c1, c]
      const int c = c1 + t;
      double x[PB];
#pragma unroll
      for (int i = 0; i < PB; ++i) {
        double acc = A[c0 + i][c];
#pragma unroll
        for (int l = 0; l < i; ++l) acc = fma(-A[c0 + l][c0 + i], x[l], acc);
        x[i] = acc * dinv[c0 + i];
        A[c0 + i][c] = x[i];
      }
    }
    __syncthreads();
    POTRF_STAMP(7)
    {  // ---- trailing update of the upper triangle (4x4 tiles, tile row <= tile column)
      const int nt = n2 / 4;
      for (int e = t; e < nt * nt; e += 256) {
        const int ti = e / nt, tj = e % nt;
        if (ti > tj) continue;
        const int r = c1 + 4 * ti, c = c1 + 4 * tj;
        double acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = A[r + a][c + b];
#pragma unroll
        for (int l = 0; l < PB; ++l) {
          double ri[4], cj[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) ri[a] = A[c0 + l][r + a];
#pragma unroll
          for (int b = 0; b < 4; ++b) cj[b] = A[c0 + l][c + b];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = fma(-ri[a], cj[b], acc[a][b]);
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) A[r + a][c + b] = acc[a][b];
      }
    }
    __syncthreads();
    POTRF_STAMP(8)
  }
  POTRF_STAMP(2)
  if (!want_inv) {  // the blocked Cholesky's critical path: R only (inverses batched later)
    for (int e = t; e < kb * kb; e += 256) {
      const int r = e / kb, c = e % kb;
      G[r * ldg + c] = r <= c ? A[r][c] : 0.0;
    }
    return;
  }
  // ---- inverse: diagonal micro-blocks (warp w -> block w; lane j -> column j)
  if (PB * warp < kbp) {
    const int w0 = PB * warp, j = lane & (PB - 1);
    double x[PB];
#pragma unroll
    for (int i = PB - 1; i >= 0; --i) {
      double v = 0.0;
      if (i == j) {
        v = dinv[w0 + i];
      } else if (i < j) {
        double s = 0.0;
#pragma unroll
        for (int l = i + 1; l < PB; ++l)
          if (l <= j) s = fma(A[w0 + i][w0 + l], x[l], s);
        v = -dinv[w0 + i] * s;
      }
      x[i] = v;
    }
    if (lane < PB) {
#pragma unroll
      for (int i = 0; i < PB; ++i) X[w0 + i][w0 + j] = x[i];
    }
  }
  __syncthreads();
  POTRF_STAMP(3)
  // ---- recursive doubling: for each pair of adjacent s-blocks, X12 = -X11 (R12 X22)
  // (two triangular products, all pairs of a level in parallel): 2 log2(kb/8) barriers
  // instead of a sequential block back-substitution.
  for (int s = PB; s < kbp; s *= 2) {
    const int npairs = (kbp + 2 * s - 1) / (2 * s);
    for (int e = t; e < npairs * s * s; e += 256) {  // T = R12 X22 (X22's lower part is zero)
      const int q = e / (s * s), i = (e / s) % s, j = e % s;
      const int a0 = 2 * q * s, b0 = a0 + s, s2 = min(s, kbp - b0);  // s2: multiple of 8
      if (j >= s2) continue;
      double s0 = 0.0, s1 = 0.0, s2a = 0.0, s3 = 0.0;
      for (int k = 0; k < s2; k += PB) {
#pragma unroll
        for (int u = 0; u < PB; u += 4) {
          s0 = fma(A[a0 + i][b0 + k + u], X[b0 + k + u][b0 + j], s0);
          s1 = fma(A[a0 + i][b0 + k + u + 1], X[b0 + k + u + 1][b0 + j], s1);
          s2a = fma(A[a0 + i][b0 + k + u + 2], X[b0 + k + u + 2][b0 + j], s2a);
          s3 = fma(A[a0 + i][b0 + k + u + 3], X[b0 + k + u + 3][b0 + j], s3);
        }
      }
      S[q * s + i][j] = (s0 + s1) + (s2a + s3);
    }
    __syncthreads();
    for (int e = t; e < npairs * s * s; e += 256) {  // X12 = -X11 T (X11's lower part is zero)
      const int q = e / (s * s), i = (e / s) % s, j = e % s;
      const int a0 = 2 * q * s, b0 = a0 + s, s2 = min(s, kbp - b0);
      if (j >= s2) continue;
      double s0 = 0.0, s1 = 0.0, s2a = 0.0, s3 = 0.0;
      for (int k = 0; k < s; k += PB) {
#pragma unroll
        for (int u = 0; u < PB; u += 4) {
          s0 = fma(X[a0 + i][a0 + k + u], S[q * s + k + u][j], s0);
          s1 = fma(X[a0 + i][a0 + k + u + 1], S[q * s + k + u + 1][j], s1);
          s2a = fma(X[a0 + i][a0 + k + u + 2], S[q * s + k + u + 2][j], s2a);
          s3 = fma(X[a0 + i][a0 + k + u + 3], S[q * s + k + u + 3][j], s3);
        }
      }
      X[a0 + i][b0 + j] = -((s0 + s1) + (s2a + s3));
    }
    __syncthreads();
  }
  POTRF_STAMP(4)
  for (int e = t; e < kb * kb; e += 256) {
    const int r = e / kb, c = e % kb;
    G[r * ldg + c] = r <= c ? A[r][c] : 0.0;
    Rinv[r * ldr + c] = r <= c ? X[r][c] : 0.0;
  }
  __syncthreads();
  POTRF_STAMP(5)
}

__global__ void __launch_bounds__(256) potrf_diag_kernel(int kb, double* G, i64 ldg, double* Rinv, i64 ldr,
                                                         const double* maxdiag, double rel_tol, int* fail,
                                                         int want_inv) {
  extern __shared__ double psm[];
  pdl_wait();
  pdl_trigger();
  potrf_tile(kb, G, ldg, Rinv, ldr, maxdiag, rel_tol, fail, want_inv, psm);
}

// Panel TRSM of the blocked Cholesky without an explicit inverse: X = R_kk^-T P for the kb x rem
// panel P (in place). One warp per panel column, lane l holding rows l and l + 32: per pivot i
// the owner scales x_i, a shuffle broadcasts it and every lane updates its later rows — a
// 64-step chain of (shuffle, FMA) per column, all columns in parallel; R_kk in shared memory.
constexpr int TRSM_T = 256;
__global__ void __launch_bounds__(TRSM_T) trsm_panel_kernel(int kb, i64 rem, const double* __restrict__ Rkk, i64 ldg,
                                                            double* __restrict__ P) {
  __shared__ double R[CNB][CNB + 1];
  __shared__ double rd[CNB];
  pdl_wait();
  pdl_trigger();
  const int t = threadIdx.x, lane = t & 31;
  for (int e = t; e < kb * kb; e += TRSM_T) {
    const int r = e / kb, c = e % kb;
    R[r][c] = r <= c ? Rkk[r * ldg + c] : 0.0;
  }
  __syncthreads();
  if (t < kb) rd[t] = 1.0 / R[t][t];
  __syncthreads();
  const i64 c = static_cast<i64>(blockIdx.x) * (TRSM_T / 32) + (t >> 5);
  if (c >= rem) return;
  double x0 = lane < kb ? P[lane * ldg + c] : 0.0;
  double x1 = lane + 32 < kb ? P[(lane + 32) * ldg + c] : 0.0;
  for (int i = 0; i < kb; ++i) {
    double xi;
    if (i < 32) {
      if (lane == i) x0 *= rd[i];
      xi = __shfl_sync(0xffffffffu, x0, i);
    } else {
      if (lane == i - 32) x1 *= rd[i];
      xi = __shfl_sync(0xffffffffu, x1, i - 32);
    }
    if (lane > i && lane < kb) x0 = fma(-R[i][lane], xi, x0);
    if (lane + 32 > i && lane + 32 < kb) x1 = fma(-R[i][lane + 32], xi, x1);
  }
  if (lane < kb) P[lane * ldg + c] = x0;
  if (lane + 32 < kb) P[(lane + 32) * ldg + c] = x1;
}

// Inverses of every CNB x CNB diagonal block of an upper-triangular R (one CTA per block, all at
// once after the factorisation — off the blocked Cholesky's critical path), by the same micro-
// block inversion + recursive doubling as potrf_diag_kernel.
__global__ void __launch_bounds__(256) trinv_diag_kernel(i64 n, const double* __restrict__ G, i64 ldg,
                                                         double* __restrict__ Rinv, i64 ldr) {
  extern __shared__ double psm[];
  pdl_wait();
  pdl_trigger();
  double(*A)[PLD] = reinterpret_cast<double(*)[PLD]>(psm);
  double(*X)[PLD] = reinterpret_cast<double(*)[PLD]>(psm + CNB * PLD);
  double(*S)[PLD] = reinterpret_cast<double(*)[PLD]>(psm + 2 * CNB * PLD);
  double* dinv = psm + 2 * CNB * PLD + (CNB / 2) * PLD;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const i64 k0 = static_cast<i64>(blockIdx.x) * CNB;
  const int kb = static_cast<int>(min(static_cast<i64>(CNB), n - k0));
  const int kbp = (kb + PB - 1) / PB * PB;
  for (int e = t; e < CNB * CNB; e += 256) {
    const int r = e / CNB, c = e % CNB;
    const bool ok = r < kb && c < kb && r <= c;
    A[r][c] = ok ? G[(k0 + r) * ldg + k0 + c] : (r == c && r >= kb ? 1.0 : 0.0);
    X[r][c] = 0.0;
  }
  __syncthreads();
  if (t < CNB) dinv[t] = 1.0 / A[t][t];
  __syncthreads();
  if (PB * warp < kbp) {  // diagonal micro-blocks (warp w -> block w; lane j -> column j)
    const int w0 = PB * warp, j = lane & (PB - 1);
    double x[PB];
#pragma unroll
    for (int i = PB - 1; i >= 0; --i) {
      double v = 0.0;
      if (i == j) {
        v = dinv[w0 + i];
      } else if (i < j) {
        double sacc = 0.0;
#pragma unroll
        for (int l = i + 1; l < PB; ++l)
          if (l <= j) sacc = fma(A[w0 + i][w0 + l], x[l], sacc);
        v = -dinv[w0 + i] * sacc;
      }
      x[i] = v;
    }
    if (lane < PB) {
#pragma unroll
      for (int i = 0; i < PB; ++i) X[w0 + i][w0 + j] = x[i];
    }
  }
  __syncthreads();
  for (int sz = PB; sz < kbp; sz *= 2) {  // recursive doubling: X12 = -X11 (R12 X22)
    const int npairs = (kbp + 2 * sz - 1) / (2 * sz);
    for (int e = t; e < npairs * sz * sz; e += 256) {
      const int q = e / (sz * sz), i = (e / sz) % sz, j = e % sz;
      const int a0 = 2 * q * sz, b0 = a0 + sz, s2 = min(sz, kbp - b0);
      if (j >= s2) continue;
      double acc = 0.0;
      for (int k = 0; k < s2; ++k) acc = fma(A[a0 + i][b0 + k], X[b0 + k][b0 + j], acc);
      S[q * sz + i][j] = acc;
    }
    __syncthreads();
    for (int e = t; e < npairs * sz * sz; e += 256) {
      const int q = e / (sz * sz), i = (e / sz) % sz, j = e % sz;
      const int a0 = 2 * q * sz, b0 = a0 + sz, s2 = min(sz, kbp - b0);
      if (j >= s2) continue;
      double acc = 0.0;
      for (int k = 0; k < sz; ++k) acc = fma(X[a0 + i][a0 + k], S[q * sz + k][j], acc);
      X[a0 + i][b0 + j] = -acc;
    }
    __syncthreads();
  }
  for (int e = t; e < kb * kb; e += 256) {
    const int r = e / kb, c = e % kb;
    Rinv[(k0 + r) * ldr + k0 + c] = r <= c ? X[r][c] : 0.0;
  }
}

// ---------------------------------------------------------------- fused tile Cholesky
// The whole blocked Cholesky (and the inverse) of an n x n Gram in ONE cooperative launch of P
// persistent CTAs, on 64 x 64 tiles, instead of ~4 launches per 64-column panel (potrf, panel
// TRSM, look-ahead update, trailing update) plus 2 GEMMs per panel for the inverse. Step k:
//   phase A  TRSM of row k as a product with the diagonal inverse: R_kj = X_kk^T G_kj (j > k), and
//            (inverse) the l = k-1 term of every running sum T_ij = sum_{l=i}^{j-1} X_il R_lj
//            (i <= k-1 < j), one tile product per task;
//   phase B  trailing update G_ij -= R_ki^T R_kj (k < i <= j; CTA 0 updates tile (k+1, k+1) and
//            factors it right away — the look-ahead — while the other CTAs update the rest), and
//            (inverse) X_ik = -T_ik X_kk (X R = I column by column);
// one grid-wide barrier after each phase (2 per tile step). Every tile task is a sum of 64 x 64 x
// 64 FP64 DMMA products (8 warps, 16 x 32 each), operands staged through shared memory with
// L2-only cp.async (the tiles were written by other SMs since the last barrier).
// Same arithmetic as the launch-per-panel path up to summation order within a tile product.
constexpr int CF_LD = CNB + 4;  // padded shared-tile row (conflict-free DMMA fragments)
constexpr size_t kCholFusedSmem = std::max(kPotrfSmem, sizeof(double) * 2 * CNB * CF_LD);

#ifdef DFCG_CHOL_TRACE  // phase timestamps (globaltimer ns) of CTA 0 and CTA 1: tools/chol_trace.cu
__device__ unsigned long long g_chol_trace[64][2][6];
__device__ __forceinline__ void chol_stamp(int k, int who, int slot) {
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == 1) && k < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_chol_trace[k][blockIdx.x][slot] = t;
  }
}
#define CHOL_STAMP(k, slot) chol_stamp(k, 0, slot)
#else
#define CHOL_STAMP(k, slot)
#endif

struct CholFusedArgs {
  int n, nt, want_inv;
  double* G;
  i64 ldg;
  double* Rinv;
  i64 ldr;
  double* T;  // n x n scratch (ld ldt): the inverse's running sums T_ij, i < j
  i64 ldt;
  const double* maxdiag;
  double rel_tol;
  int* fail;
};

// acc += op(A) B for 64 x 64 tiles (rows / cols beyond ra / cb and k beyond kk are zero-filled):
// op(A) = A^T (ta) or A; A at a (ld lda), B at b (ld ldb). 256 threads.
__device__ __forceinline__ void cf_tile_product(double (&acc)[2][4][2], bool ta, const double* a, i64 lda,
                                                const double* b, i64 ldb, int ra, int kk, int cb, double* sm) {
  double* sA = sm;                 // [r][k] (ta: stored [k][r])
  double* sB = sm + CNB * CF_LD;   // [k][c]
  const int t = threadIdx.x;
  // 16-byte L2-only copies (cp.async.cg: tiles written by other SMs since the last grid barrier
  // must not come from a stale L1 line — the T scratch is rewritten every step), all in flight
  // at once; pairs straddling the tile's valid extent copy 8 bytes and zero-fill the rest.
  // Requires even leading dimensions and 16-byte aligned tiles (the host pads otherwise).
  auto cp16n = [](double* dst, const double* src, int bytes) {
    const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(src), "r"(bytes));
  };
#pragma unroll
  for (int it = 0; it < (CNB * CNB / 2) / 256; ++it) {
    const int e = t + it * 256, r = e / (CNB / 2), c = 2 * (e % (CNB / 2));
    // A: stored row r (= k for ta, = output row otherwise), stored cols c, c+1
    const int arows = ta ? kk : ra, acols = ta ? ra : kk;
    const int na = r < arows ? min(2, max(0, acols - c)) : 0;
    cp16n(sA + r * CF_LD + c, na ? a + r * lda + c : a, 8 * na);
    const int nb = r < kk ? min(2, max(0, cb - c)) : 0;
    cp16n(sB + r * CF_LD + c, nb ? b + r * ldb + c : b, 8 * nb);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int lane = t & 31, warp = t >> 5;
  const int wm = (warp >> 1) * 16, wn = (warp & 1) * 32;
  const int fr = lane >> 2, fk = lane & 3;
#pragma unroll 4
  for (int k0 = 0; k0 < CNB; k0 += 4) {
    double af[2], bf[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int r = wm + i * 8 + fr, k = k0 + fk;
      af[i] = ta ? sA[k * CF_LD + r] : sA[r * CF_LD + k];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) bf[j] = sB[(k0 + fk) * CF_LD + wn + j * 8 + fr];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
  }
  __syncthreads();  // the tiles are restaged by the next product
}

// c[r, col] = alpha acc + (beta ? c : 0) over the valid rows / cols
__device__ __forceinline__ void cf_store(const double (&acc)[2][4][2], double* c, i64 ldc, int rows, int cols,
                                         double alpha, bool accumulate) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp >> 1) * 16, wn = (warp & 1) * 32;
  const int er = lane >> 2, ec = (lane & 3) * 2;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = wm + i * 8 + er, col = wn + j * 8 + ec + h;
        if (r < rows && col < cols) {
          double* p = c + r * ldc + col;
          *p = accumulate ? __ldcg(p) + alpha * acc[i][j][h] : alpha * acc[i][j][h];
        }
      }
}

__device__ __forceinline__ void cf_zero(double (&acc)[2][4][2]) {
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

__global__ void __launch_bounds__(256, 2) chol_fused_kernel(CholFusedArgs p) {
  extern __shared__ double csm[];
  cg::grid_group grid = cg::this_grid();
  const int P = gridDim.x, c = blockIdx.x, nt = p.nt;
  auto tsz = [&](int i) { return min(CNB, p.n - i * CNB); };
  auto gt = [&](int i, int j) { return p.G + static_cast<i64>(i) * CNB * p.ldg + static_cast<i64>(j) * CNB; };
  auto xt = [&](int i, int j) { return p.Rinv + static_cast<i64>(i) * CNB * p.ldr + static_cast<i64>(j) * CNB; };
  auto tt = [&](int i, int j) { return p.T + static_cast<i64>(i) * CNB * p.ldt + static_cast<i64>(j) * CNB; };
  double acc[2][4][2];
  if (c == 0) {
    potrf_tile(tsz(0), gt(0, 0), p.ldg, xt(0, 0), p.ldr, p.maxdiag, p.rel_tol, p.fail, 1, csm);
    __syncthreads();
  }
  grid.sync();
  for (int k = 0; k < nt; ++k) {
    const int kb = tsz(k);
    CHOL_STAMP(k, 0);
    // ---- phase A: R_kj = X_kk^T G_kj (j > k); and the inverse's running sums
    //      T_ij += X_{i,k-1} R_{k-1,j} for i <= k-1 < j (the l = k-1 term of
    //      T_ij = sum_{l=i}^{j-1} X_il R_lj: every product is its own task, no serial chain)
    {
      const int ntr = nt - k - 1, nacc = p.want_inv && k > 0 ? k * (nt - k) : 0;
      for (int task = c; task < ntr + nacc; task += P) {
        cf_zero(acc);
        if (task < ntr) {
          const int j = k + 1 + task;
          cf_tile_product(acc, true, xt(k, k), p.ldr, gt(k, j), p.ldg, kb, kb, tsz(j), csm);
          cf_store(acc, gt(k, j), p.ldg, kb, tsz(j), 1.0, false);
        } else {
          const int q = task - ntr, i = q / (nt - k), j = k + q % (nt - k), l = k - 1;
          cf_tile_product(acc, false, xt(i, l), p.ldr, gt(l, j), p.ldg, tsz(i), tsz(l), tsz(j), csm);
          cf_store(acc, tt(i, j), p.ldt, tsz(i), tsz(j), 1.0, i != l);  // the l = i term starts the sum
        }
      }
    }
    CHOL_STAMP(k, 1);
    grid.sync();
    CHOL_STAMP(k, 2);
    // ---- phase B: trailing update (+ look-ahead factorisation of tile k+1), X_ik = -T_i X_kk
    {
      const int m = nt - k - 1;  // trailing tiles per side
      const int nup = m * (m + 1) / 2, nxi = p.want_inv ? k : 0;
      if (c == 0 && m > 0) {
        cf_zero(acc);
        cf_tile_product(acc, true, gt(k, k + 1), p.ldg, gt(k, k + 1), p.ldg, tsz(k + 1), kb, tsz(k + 1), csm);
        cf_store(acc, gt(k + 1, k + 1), p.ldg, tsz(k + 1), tsz(k + 1), -1.0, true);
        __threadfence_block();
        __syncthreads();
        CHOL_STAMP(k, 3);
        potrf_tile(tsz(k + 1), gt(k + 1, k + 1), p.ldg, xt(k + 1, k + 1), p.ldr, p.maxdiag, p.rel_tol, p.fail, 1,
                   csm);
        __syncthreads();
        CHOL_STAMP(k, 4);
      }
      // the other update tiles and the X column, over CTAs 1..P-1 (CTA 0 too when P == 1)
      const int workers = P > 1 ? P - 1 : 1, w = P > 1 ? c - 1 : 0;
      if (P == 1 || c > 0) {
        for (int task = w; task < (nup - (m > 0 ? 1 : 0)) + nxi; task += workers) {
          cf_zero(acc);
          const int nu = nup - (m > 0 ? 1 : 0);
          if (task < nu) {
            // tile index over the upper triangle of the trailing block, skipping (k+1, k+1)
            int idx = task + 1, i = 0;
            while (idx >= m - i) idx -= m - i, ++i;
            const int ti = k + 1 + i, tj = ti + idx;
            cf_tile_product(acc, true, gt(k, ti), p.ldg, gt(k, tj), p.ldg, tsz(ti), kb, tsz(tj), csm);
            cf_store(acc, gt(ti, tj), p.ldg, tsz(ti), tsz(tj), -1.0, true);
          } else {  // X_ik = -T_ik X_kk (T_ik complete: its last term was added in phase A)
            const int i = task - nu;
            cf_tile_product(acc, false, tt(i, k), p.ldt, xt(k, k), p.ldr, tsz(i), kb, kb, csm);
            cf_store(acc, xt(i, k), p.ldr, tsz(i), kb, -1.0, false);
          }
        }
      }
    }
    CHOL_STAMP(k, 5);
    grid.sync();
  }
  // strictly-lower tiles of R are zero (the diagonal tiles were written by potrf_tile)
  for (int task = c; task < nt * nt; task += P) {
    const int i = task / nt, j = task % nt;
    if (i <= j) continue;
    double* g = gt(i, j);
    for (int e = threadIdx.x; e < tsz(i) * tsz(j); e += 256) g[(e / tsz(j)) * p.ldg + e % tsz(j)] = 0.0;
  }
}

__global__ void zero_lower_kernel(i64 n, double* A, i64 lda) {
  const i64 total = n * n;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = e / n, j = e % n;
    if (i > j) A[i * lda + j] = 0.0;
  }
}

// In-place blocked Cholesky of G (n x n) -> upper R (lower part zeroed); Rinv = R^-1.
// want_inverse == false: only R is produced and Rinv's contents are unspecified (scratch).
// The look-ahead helper stream and its two events belong to the calling stream: one helper per
// main stream, created on first use and kept for the process (main streams are pooled by the
// DeviceContext and the solvers, so the helper count is bounded by theirs, whichever host threads
// come and go). A helper shared between solves would queue one solve's potrf behind another's.
struct AuxStream {
  cudaStream_t s = nullptr;
  cudaEvent_t updated = nullptr, factored = nullptr;
};
AuxStream& aux_for(cudaStream_t main) {
  static std::mutex mu;
  static std::unordered_map<cudaStream_t, AuxStream> helpers;  // node-based: references stay valid
  std::lock_guard<std::mutex> lock(mu);
  AuxStream& a = helpers[main];
  if (!a.s) {
    DFCG_CUDA(cudaStreamCreateWithFlags(&a.s, cudaStreamNonBlocking));
    DFCG_CUDA(cudaEventCreateWithFlags(&a.updated, cudaEventDisableTiming));
    DFCG_CUDA(cudaEventCreateWithFlags(&a.factored, cudaEventDisableTiming));
  }
  return a;
}

void cholesky_inverse_raw(cudaStream_t s, i64 n, double* G, i64 ldg, double* Rinv, i64 ldr, double rel_tol,
                          int* fail, bool want_inverse) {
  static std::atomic<std::uint64_t> configured{0};  // one bit per device: opt in to > 48 KB dynamic shared memory
  int dev = 0;
  DFCG_CUDA(cudaGetDevice(&dev));
  if (!(configured.load() & dev_bit(dev))) {
    DFCG_CUDA(cudaFuncSetAttribute(potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(kPotrfSmem)));
    DFCG_CUDA(cudaFuncSetAttribute(trinv_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(kPotrfSmem)));
    configured.fetch_or(dev_bit(dev));
  }
  // DFCG_CHOL_INV_LATE=0: the diagonal inverses inside potrf and the panel TRSM as a GEMM with
  // them (the previous critical path); default: potrf without the inverse, substitution TRSM,
  // all diagonal inverses in one launch after the factorisation.
  static const bool late = !(std::getenv("DFCG_CHOL_INV_LATE") && std::atoi(std::getenv("DFCG_CHOL_INV_LATE")) == 0);
  DBuf<double> maxdiag(1, s);
  diag_max_kernel<<<1, 256, 0, s>>>(n, G, ldg, maxdiag.get());
  DFCG_LAUNCH_CHECK();
  DFCG_CUDA(cudaMemset2DAsync(Rinv, sizeof(double) * ldr, 0, sizeof(double) * n, n, s));
  // One cooperative launch for the whole factorisation (chol_fused_kernel) instead of the
  // launch-per-panel path below: the packed c2 step drops from 11263 to 6048 launches (136.0 ->
  // 142.0 block-it/s) and a lone c2 iteration from 20.7 to 19.7 ms (profiles/r02_lone_fused*_v3,
  // r02_bench_c2_cholfused*_v3). DFCG_CHOL_FUSED=0 keeps the per-panel path, 3 fuses only while
  // three or more solves share the GPU.
  static const int fused_mode = std::getenv("DFCG_CHOL_FUSED") ? std::atoi(std::getenv("DFCG_CHOL_FUSED")) : 1;
  // Large factorisations keep the per-panel path: their trailing updates are full-GPU GEMMs
  // (the base APG on the whole 10^4 x 10^4 matrix factors n ~ 3600: 35 ms fused on 64 CTAs
  // against the per-panel path, profiles/r02_bench_cholesky_large.txt). DFCG_CHOL_FUSED_MAXN.
  static const i64 fused_maxn =
      std::getenv("DFCG_CHOL_FUSED_MAXN") ? std::atoll(std::getenv("DFCG_CHOL_FUSED_MAXN")) : 2048;
  if (n > CNB && n <= fused_maxn && (fused_mode == 1 || (fused_mode == 3 && active_streams(dev) >= 3))) {
    static std::atomic<std::uint64_t> fused_cfg{0};
    static int occ = 0, nsm = 0;
    if (!(fused_cfg.load() & dev_bit(dev))) {
      DFCG_CUDA(cudaFuncSetAttribute(chol_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kCholFusedSmem)));
      DFCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chol_fused_kernel, 256, kCholFusedSmem));
      DFCG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
      fused_cfg.fetch_or(dev_bit(dev));
    }
    const int nt = static_cast<int>((n + CNB - 1) / CNB);
    const int share = std::max(1, active_streams(dev));
    // the tile copies are 16-byte cp.async: work on even-ld, aligned copies when the caller's
    // layout is not (one 2-D copy in, one out)
    auto aligned = [](const double* p, i64 ld) { return ld % 2 == 0 && reinterpret_cast<std::uintptr_t>(p) % 16 == 0; };
    const bool in_place = aligned(G, ldg) && aligned(Rinv, ldr);
    const i64 np = (n + 1) & ~i64{1};
    DBuf<double> Gp, Rp;
    double* Gf = G;
    double* Rf = Rinv;
    i64 ldgf = ldg, ldrf = ldr;
    if (!in_place) {
      Gp.alloc(n * np, s);
      Rp.alloc(n * np, s);
      copy2d(s, n, n, G, ldg, Gp.get(), np);
      Rp.zero(s);
      Gf = Gp.get();
      Rf = Rp.get();
      ldgf = ldrf = np;
    }
    // CTAs: the widest phase's task count, at most this solve's share of the co-resident slots
    const int widest = std::max(nt * (nt - 1) / 2 + (want_inverse ? nt : 0), want_inverse ? (nt / 2) * (nt - nt / 2) + nt : nt);
    // at most 64 CTAs (the 1250-column factorisation gains nothing past it,
    // profiles/r02_bench_cholesky.txt); 128 registers, two CTAs per SM, so a CTA waiting at a
    // grid barrier holds half an SM, not all of it, while other solves' kernels run (packed F step)
    int P = std::max(2, std::min({widest, 64, std::max(2, occ * nsm / share)}));
    if (const char* pe = std::getenv("DFCG_CHOL_P")) P = std::max(2, std::min(std::atoi(pe), occ * nsm));  // tuning
    DBuf<double> T(want_inverse ? n * np : 1, s);
    CholFusedArgs a{static_cast<int>(n), nt, want_inverse ? 1 : 0, Gf, ldgf, Rf, ldrf, T.get(), np, maxdiag.get(),
                    rel_tol, fail};
    void* kargs[] = {&a};
    prof::Scope scope(prof::kCholesky, s, n * n * n / 3.0 + (want_inverse ? n * n * n / 3.0 : 0.0),
                      16.0 * n * n);
    DFCG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(chol_fused_kernel), dim3(P), dim3(256), kargs,
                                          kCholFusedSmem, s));
    DFCG_LAUNCH_CHECK();
    if (!in_place) {
      copy2d(s, n, n, Gp.get(), np, G, ldg);
      copy2d(s, n, n, Rp.get(), np, Rinv, ldr);
    }
    return;
  }
  // Look-ahead: after the panel TRSM of block k, the next diagonal block is updated first and
  // factored on a helper stream while the rest of the trailing update runs on s, so the
  // latency-bound 64x64 potrf overlaps the trailing GEMM instead of following it.
  AuxStream& aux = aux_for(s);
  auto potrf = [&](cudaStream_t st, i64 k0, int kb) {
    prof::Scope scope(prof::kCholesky, st, kb * kb * kb / 3.0 + kb * kb * kb / 3.0, 16.0 * kb * kb);
    pdl_launch(potrf_diag_kernel, dim3(1), dim3(256), kPotrfSmem, st, kb, G + k0 * ldg + k0, ldg,
               Rinv + k0 * ldr + k0, ldr, static_cast<const double*>(maxdiag.get()), rel_tol, fail, late ? 0 : 1);
    DFCG_LAUNCH_CHECK();
  };
  potrf(s, 0, static_cast<int>(std::min<i64>(CNB, n)));
  for (i64 k0 = 0; k0 < n; k0 += CNB) {
    const int kb = static_cast<int>(std::min<i64>(CNB, n - k0));
    if (k0 > 0) DFCG_CUDA(cudaStreamWaitEvent(s, aux.factored, 0));  // potrf(k) ran on the helper
    const i64 rem = n - k0 - kb;
    if (rem <= 0) break;
    double* panel = G + k0 * ldg + k0 + kb;  // kb x rem
    // R[k, J] = Rkk^-T G[k, J]
    if (late) {
      prof::Scope scope(prof::kCholesky, s, 1.0 * kb * kb * rem, 16.0 * kb * rem);
      pdl_launch(trsm_panel_kernel, dim3(static_cast<unsigned>((rem + TRSM_T / 32 - 1) / (TRSM_T / 32))), dim3(TRSM_T), 0, s, kb,
                 rem, static_cast<const double*>(G + k0 * ldg + k0), ldg, panel);
      DFCG_LAUNCH_CHECK();
    } else {
      gemm(s, true, false, kb, rem, kb, 1.0, Rinv + k0 * ldr + k0, ldr, panel, ldg, 0.0, panel, ldg);
    }
    // next diagonal block: G[k1, k1] -= R[k, k1]^T R[k, k1], then factored on the helper stream
    const i64 k1 = k0 + kb;
    const int kb1 = static_cast<int>(std::min<i64>(CNB, rem));
    gemm(s, true, false, kb1, kb1, kb, -1.0, panel, ldg, panel, ldg, 1.0, G + k1 * ldg + k1, ldg);
    DFCG_CUDA(cudaEventRecord(aux.updated, s));
    DFCG_CUDA(cudaStreamWaitEvent(aux.s, aux.updated, 0));
    potrf(aux.s, k1, kb1);
    DFCG_CUDA(cudaEventRecord(aux.factored, aux.s));
    // the rest of the trailing update (rows k1.., columns past the next diagonal block)
    if (rem > kb1)
      gemm(s, true, false, rem, rem - kb1, kb, -1.0, panel, ldg, panel + kb1, ldg, 1.0, G + k1 * ldg + k1 + kb1, ldg);
  }
  zero_lower_kernel<<<grid_for(n * n), 256, 0, s>>>(n, G, ldg);
  DFCG_LAUNCH_CHECK();
  if (late && want_inverse) {
    prof::Scope scope(prof::kCholesky, s, n * CNB * CNB / 3.0, 16.0 * n * CNB);
    pdl_launch(trinv_diag_kernel, dim3(static_cast<unsigned>((n + CNB - 1) / CNB)), dim3(256), kPotrfSmem, s, n,
               static_cast<const double*>(G), ldg, Rinv, ldr);
    DFCG_LAUNCH_CHECK();
  }
  // Off-diagonal blocks of the inverse: Rinv[0:J, J] = -Rinv[0:J,0:J] R[0:J, J] Rinv[J,J].
  if (want_inverse && n > CNB) {
    DBuf<double> T(n * CNB, s);
    for (i64 j0 = CNB; j0 < n; j0 += CNB) {
      const i64 jb = std::min<i64>(CNB, n - j0);
      gemm(s, false, false, j0, jb, j0, 1.0, Rinv, ldr, G + j0, ldg, 0.0, T.get(), jb);
      gemm(s, false, false, j0, jb, jb, -1.0, T.get(), jb, Rinv + j0 * ldr + j0, ldr, 0.0, Rinv + j0, ldr);
    }
  }
}

// Diagonal scaling for the Cholesky of a Gram: d = sqrt(diag G) (zero pivots keep d = 1), then
// G <- D^-1 G D^-1 on the upper part (two kernels: the diagonal is read before it is rescaled)
__global__ void gram_diag_kernel(i64 n, const double* G, i64 ldg, double* d) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const double g = G[i * ldg + i];
    d[i] = g > 0.0 ? sqrt(g) : 1.0;
  }
}
__global__ void gram_scale_kernel(i64 n, double* G, i64 ldg, const double* d) {
  const i64 total = n * n;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = e / n, j = e % n;
    if (i <= j) G[i * ldg + j] = G[i * ldg + j] / (d[i] * d[j]);
  }
}
// R' -> R' D (columns, upper part), Rinv' -> D^-1 Rinv' (rows)
__global__ void chol_unscale_kernel(i64 n, double* R, i64 ldg, double* Rinv, i64 ldr, const double* d, int inv) {
  const i64 total = n * n;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = e / n, j = e % n;
    if (i > j) continue;
    R[i * ldg + j] *= d[j];
    if (inv) Rinv[i * ldr + j] /= d[i];
  }
}

// Cholesky of a Gram matrix, R^T R = G, with the inverse: the Gram is first scaled to unit
// diagonal (Jacobi preconditioning, G' = D^-1 G D^-1, R = R' D, R^-1 = D^-1 R'^-1), so the
// breakdown test (pivot < rel_tol * max pivot) fires on ill-conditioning of the column
// directions only, not on column scaling — an SVT factor V diag(s), whose singular values span
// many decades, stays on the CholQR path instead of the Householder fallback.
// scale == false keeps the raw breakdown test (pivot < rel_tol * max diag G): it then also
// certifies cond(X) < ~3e5, which the Gram-based R of thin_svd relies on for accuracy.
void cholesky_inverse(cudaStream_t s, i64 n, double* G, i64 ldg, double* Rinv, i64 ldr, double rel_tol, int* fail,
                      bool want_inverse = true, bool scale = true) {
  if (n <= 0) return;
  static const int scale_mode = std::getenv("DFCG_CHOL_SCALE") ? std::atoi(std::getenv("DFCG_CHOL_SCALE")) : 1;
  if (!scale || scale_mode == 0) {
    cholesky_inverse_raw(s, n, G, ldg, Rinv, ldr, rel_tol, fail, want_inverse);
    return;
  }
  DBuf<double> d(n, s);
  gram_diag_kernel<<<grid_for(n), 256, 0, s>>>(n, G, ldg, d.get());
  DFCG_LAUNCH_CHECK();
  gram_scale_kernel<<<grid_for(n * n), 256, 0, s>>>(n, G, ldg, d.get());
  DFCG_LAUNCH_CHECK();
  cholesky_inverse_raw(s, n, G, ldg, Rinv, ldr, rel_tol, fail, want_inverse);
  chol_unscale_kernel<<<grid_for(n * n), 256, 0, s>>>(n, G, ldg, Rinv, ldr, d.get(), want_inverse ? 1 : 0);
  DFCG_LAUNCH_CHECK();
}

// ================================================================ Householder QR (fallback)
constexpr int HNB = 32, HTHREADS = 512;

// LAPACK dgeqr2 on the panel X[p0:, p0:p0+nb] (row-major, ld). Reflector j stored below the
// diagonal (implicit unit head), beta on the diagonal, tau[j].
__global__ void __launch_bounds__(HTHREADS) hh_panel_kernel(i64 rows, int nb, double* X, i64 ld, double* tau) {
  __shared__ double red[HTHREADS / 32][HNB + 1];
  __shared__ double colsum[HNB + 1];
  __shared__ double s_beta, s_tau, s_scale;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int j = 0; j < nb; ++j) {
    // norm^2 of X[j+1:, j]
    double acc = 0.0;
    for (i64 r = j + 1 + t; r < rows; r += HTHREADS) {
      const double v = X[r * ld + j];
      acc += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[warp][0] = acc;
    __syncthreads();
    if (t == 0) {
      double nrm2 = 0.0;
      for (int w = 0; w < HTHREADS / 32; ++w) nrm2 += red[w][0];
      const double alpha = X[static_cast<i64>(j) * ld + j];
      if (nrm2 == 0.0) {
        s_tau = 0.0;
        s_beta = alpha;
        s_scale = 0.0;
      } else {
        const double beta = -copysign(sqrt(alpha * alpha + nrm2), alpha);
        s_tau = (beta - alpha) / beta;
        s_scale = 1.0 / (alpha - beta);
        s_beta = beta;
      }
      tau[j] = s_tau;
      X[static_cast<i64>(j) * ld + j] = s_beta;
    }
    __syncthreads();
    const double sc = s_scale, tj = s_tau;
    for (i64 r = j + 1 + t; r < rows; r += HTHREADS) X[r * ld + j] *= sc;
    __syncthreads();
    if (tj == 0.0) continue;
    // w_c = x_c[j] + sum_r v_r x_c[r] for remaining panel columns c
    const int nc = nb - j - 1;
    if (nc <= 0) continue;
    double part[HNB];
#pragma unroll
    for (int c = 0; c < HNB; ++c) part[c] = 0.0;
    for (i64 r = j + 1 + t; r < rows; r += HTHREADS) {
      const double v = X[r * ld + j];
#pragma unroll
      for (int c = 0; c < HNB; ++c)
        if (c < nc) part[c] += v * X[r * ld + j + 1 + c];
    }
#pragma unroll
    for (int c = 0; c < HNB; ++c) {
      double v = part[c];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[warp][c] = v;
    }
    __syncthreads();
    if (t < nc) {
      double s = X[static_cast<i64>(j) * ld + j + 1 + t];
      for (int w = 0; w < HTHREADS / 32; ++w) s += red[w][t];
      colsum[t] = tj * s;
    }
    __syncthreads();
    for (int c = t; c < nc; c += HTHREADS) X[static_cast<i64>(j) * ld + j + 1 + c] -= colsum[c];
    for (i64 r = j + 1 + t; r < rows; r += HTHREADS) {
      const double v = X[r * ld + j];
      for (int c = 0; c < nc; ++c) X[r * ld + j + 1 + c] -= colsum[c] * v;
    }
    __syncthreads();
  }
}

// Explicit panel V (rows x nb, unit diagonal, zeros above) from the factored panel.
__global__ void hh_extract_v(i64 rows, int nb, const double* X, i64 ld, double* V) {
  const i64 total = rows * nb;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 r = e / nb;
    const int c = static_cast<int>(e % nb);
    V[e] = r < c ? 0.0 : (r == c ? 1.0 : X[r * ld + c]);
  }
}

// dlarft (forward, columnwise): T upper nb x nb from S = V^T V and tau.
__global__ void hh_build_t(int nb, const double* S, const double* tau, double* T) {
  __shared__ double t[HNB][HNB + 1];
  const int i = threadIdx.x;
  for (int e = i; e < HNB * (HNB + 1); e += blockDim.x) (&t[0][0])[e] = 0.0;
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    // T[0:j, j] = -tau_j * T[0:j, 0:j] * S[0:j, j]
    double v = 0.0;
    if (i < j)
      for (int l = i; l < j; ++l) v += t[i][l] * S[l * nb + j];
    __syncthreads();
    if (i < j) t[i][j] = -tau[j] * v;
    if (i == j) t[j][j] = tau[j];
    __syncthreads();
  }
  for (int e = i; e < nb * nb; e += blockDim.x) T[e] = t[e / nb][e % nb];
}

__global__ void extract_upper(i64 n, const double* X, i64 ldx, double* R, i64 ldr) {
  const i64 total = n * n;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = e / n, j = e % n;
    R[i * ldr + j] = i <= j ? X[i * ldx + j] : 0.0;
  }
}

// ================================================================ one-sided block Jacobi SVD
constexpr int JCHUNK = 64;

// Round-robin schedule: pairs[(round * npairs + p) * 2 + {0,1}] = block ids.
std::vector<int> round_robin(int p) {
  std::vector<int> out;
  std::vector<int> ring(p);
  std::iota(ring.begin(), ring.end(), 0);
  for (int r = 0; r < p - 1; ++r) {
    for (int k = 0; k < p / 2; ++k) {
      out.push_back(ring[k]);
      out.push_back(ring[p - 1 - k]);
    }
    const int last = ring[p - 1];  // rotate all but the first
    for (int k = p - 1; k > 1; --k) ring[k] = ring[k - 1];
    ring[1] = last;
  }
  return out;
}

// One Jacobi round: each CTA orthogonalises the JW = 2*NB columns of one block pair of W
// (rows x n) and applies the same rotation to the pair's columns of V (nv x n).
//   Gram by DMMA over 64-row chunks -> inner cyclic Jacobi EVD of the JW x JW Gram in shared
//   memory (parallel ordering, JW/2 rotations per step) -> [W_I W_J] <- [W_I W_J] R, same for V.
// Pairs whose columns are already orthogonal to `tol` are left untouched.
template <int NB>
__global__ void __launch_bounds__(16 * NB) jacobi_round_kernel(i64 rows, i64 nv, double* W, i64 ldw, double* V,
                                                               i64 ldv, const int* pairs, double tol,
                                                               unsigned long long* offmax, int inner_sweeps) {
  constexpr int JW = 2 * NB, T = 16 * NB, NT = JW / 8;  // NT = 8x8 tiles per side
  __shared__ double chunk[JCHUNK][JW + 1];
  __shared__ double g[JW][JW + 1];
  __shared__ double rot[JW][JW + 1];
  __shared__ double cs[JW / 2][2];
  __shared__ int pp[JW / 2][2];
  __shared__ double s_off;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int bi = pairs[2 * blockIdx.x], bj = pairs[2 * blockIdx.x + 1];
  auto gcol = [&](int c) -> i64 { return c < NB ? static_cast<i64>(bi) * NB + c : static_cast<i64>(bj) * NB + c - NB; };

  // ---- Gram G = P^T P over the rows; warp w owns tiles w*TPW .. w*TPW+TPW-1 of the NT x NT grid
  constexpr int TPW = (NT * NT) / (T / 32);
  double acc[TPW][2];
#pragma unroll
  for (int q = 0; q < TPW; ++q) acc[q][0] = acc[q][1] = 0.0;
  for (i64 r0 = 0; r0 < rows; r0 += JCHUNK) {
    __syncthreads();
    for (int e = t; e < JCHUNK * JW; e += T) {
      const int r = e / JW, c = e % JW;
      const i64 gr = r0 + r;
      chunk[r][c] = gr < rows ? W[gr * ldw + gcol(c)] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < JCHUNK; k += 4) {
#pragma unroll
      for (int q = 0; q < TPW; ++q) {
        const int tile = warp * TPW + q, ti = tile / NT, tj = tile % NT;
        const double a = chunk[k + (lane & 3)][ti * 8 + (lane >> 2)];  // A = P^T
        const double b = chunk[k + (lane & 3)][tj * 8 + (lane >> 2)];  // B = P
        dmma(acc[q], a, b);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < TPW; ++q) {
    const int tile = warp * TPW + q, ti = tile / NT, tj = tile % NT;
    const int r = ti * 8 + (lane >> 2), c = tj * 8 + (lane & 3) * 2;
    g[r][c] = acc[q][0];
    g[r][c + 1] = acc[q][1];
  }
  for (int e = t; e < JW * JW; e += T) rot[e / JW][e % JW] = (e / JW == e % JW) ? 1.0 : 0.0;
  __syncthreads();

  auto off_measure = [&]() {  // max |g_ab| / sqrt(g_aa g_bb), a < b
    double mx = 0.0;
    for (int e = t; e < JW * JW; e += T) {
      const int a = e / JW, b = e % JW;
      if (a >= b) continue;
      const double d = sqrt(g[a][a]) * sqrt(g[b][b]);
      if (d > 0.0) mx = fmax(mx, fabs(g[a][b]) / d);
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __syncthreads();
    if (t == 0) s_off = 0.0;
    __syncthreads();
    if (lane == 0)
      atomicMax(reinterpret_cast<unsigned long long*>(&s_off), static_cast<unsigned long long>(__double_as_longlong(mx)));
    __syncthreads();
    return s_off;
  };
  const double off0 = off_measure();
  if (t == 0) atomicMax(offmax, static_cast<unsigned long long>(__double_as_longlong(off0)));
  if (off0 <= tol) return;

  // ---- inner cyclic Jacobi EVD of g (JW x JW)
  for (int sweep = 0; sweep < inner_sweeps; ++sweep) {
    if (sweep > 0 && off_measure() <= 0.1 * tol) break;
    for (int step = 0; step < JW - 1; ++step) {
      if (t < JW / 2) {
        int a, b;  // round-robin on JW items: 0 fixed, ring of JW-1
        if (t == 0) {
          a = 0;
          b = 1 + (step % (JW - 1));
        } else {
          a = 1 + ((step + t) % (JW - 1));
          b = 1 + ((step + (JW - 1) - t) % (JW - 1));
        }
        if (a > b) {
          const int tmp = a;
          a = b;
          b = tmp;
        }
        pp[t][0] = a;
        pp[t][1] = b;
        const double gpq = g[a][b], gpp = g[a][a], gqq = g[b][b];
        double c = 1.0, sn = 0.0;
        if (fabs(gpq) > 1e-300 && fabs(gpq) > 1e-17 * sqrt(gpp * gqq)) {
          const double theta = (gqq - gpp) / (2.0 * gpq);
          const double tt = copysign(1.0, theta) / (fabs(theta) + sqrt(1.0 + theta * theta));
          c = 1.0 / sqrt(1.0 + tt * tt);
          sn = tt * c;
        }
        cs[t][0] = c;
        cs[t][1] = sn;
      }
      __syncthreads();
      for (int e = t; e < (JW / 2) * JW; e += T) {  // columns: g <- g J ; rot <- rot J
        const int k = e / JW, r = e % JW;
        const int a = pp[k][0], b = pp[k][1];
        const double c = cs[k][0], sn = cs[k][1];
        const double ga = g[r][a], gb = g[r][b];
        g[r][a] = c * ga - sn * gb;
        g[r][b] = sn * ga + c * gb;
        const double ra = rot[r][a], rb = rot[r][b];
        rot[r][a] = c * ra - sn * rb;
        rot[r][b] = sn * ra + c * rb;
      }
      __syncthreads();
      for (int e = t; e < (JW / 2) * JW; e += T) {  // rows: g <- J^T g
        const int k = e / JW, r = e % JW;
        const int a = pp[k][0], b = pp[k][1];
        const double c = cs[k][0], sn = cs[k][1];
        const double ga = g[a][r], gb = g[b][r];
        g[a][r] = c * ga - sn * gb;
        g[b][r] = sn * ga + c * gb;
      }
      __syncthreads();
    }
  }

  // ---- P <- P rot on W (rows) and V (nv rows); 64-row chunks, 8 x NT tiles, 4 per warp
  auto apply = [&](double* M, i64 ld, i64 nrows) {
    for (i64 r0 = 0; r0 < nrows; r0 += JCHUNK) {
      __syncthreads();
      for (int e = t; e < JCHUNK * JW; e += T) {
        const int r = e / JW, c = e % JW;
        const i64 gr = r0 + r;
        chunk[r][c] = gr < nrows ? M[gr * ld + gcol(c)] : 0.0;
      }
      __syncthreads();
      double o[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
#pragma unroll
      for (int k = 0; k < JW; k += 4) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int tile = warp * 4 + q, rt = tile / NT, ct = tile % NT;
          dmma(o[q], chunk[rt * 8 + (lane >> 2)][k + (lane & 3)], rot[k + (lane & 3)][ct * 8 + (lane >> 2)]);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int tile = warp * 4 + q, rt = tile / NT, ct = tile % NT;
        const i64 gr = r0 + rt * 8 + (lane >> 2);
        if (gr < nrows) {
          const int c = ct * 8 + (lane & 3) * 2;
          M[gr * ld + gcol(c)] = o[q][0];
          M[gr * ld + gcol(c + 1)] = o[q][1];
        }
      }
    }
  };
  apply(W, ldw, rows);
  apply(V, ldv, nv);
}

// Shared-memory-resident variant of the round. One CTA (or a cluster of CS CTAs, each with a
// slab of the rows) per block pair; NB = 8 or 16 columns per block:
//   stage   the pair's 2NB columns of W (and of V when both fit) with 16-byte cp.async into a
//           swizzled row layout (chunk q of row r at q ^ 2(r & 3): conflict-free for both DMMA
//           fragment patterns below, no padding, 16-byte aligned);
//   Gram    by DMMA over the 8 warps, fixed-order reduction through 4 shared slots;
//   EVD     the 2NB x 2NB Gram, one barrier per step: each thread owns a 2x2 block (P, Q) of the
//           pairing and applies J_P^T G J_Q into the other buffer of a double-buffered Gram,
//           the rest rotate the accumulated rotation; every thread recomputes the rotations it
//           needs from the pre-step Gram;
//   apply   W_pair <- W_pair rot by DMMA with the rotation fragments held in registers,
//           16-byte stores; then the same for the V pair.
// The host sizes the slab from the shared memory left by the static arrays (thin_svd).

// swizzled position of column c (0..2NB-1) in row r of a staged pair
__device__ __forceinline__ int jswz(int r, int c) { return ((((c >> 1) ^ ((r & 3) << 1))) << 1) | (c & 1); }

// pair k of step `step` of the JW-column round-robin ordering (column 0 fixed), a < b
template <int JW>
__device__ __forceinline__ void jpair(int step, int k, int& a, int& b) {
  constexpr int M = JW - 1;
  if (k == 0) {
    a = 0;
    b = 1 + step;
  } else {
    int x = step + k, y = step + M - k;
    x = x >= M ? x - M : x;
    y = y >= M ? y - M : y;
    a = 1 + x;
    b = 1 + y;
    if (a > b) {
      const int tmp = a;
      a = b;
      b = tmp;
    }
  }
}

// Symmetric 2x2 Schur rotation of (a, b): t = 2 g_ab sign(d) / (|d| + sqrt(d^2 + 4 g_ab^2)),
// d = g_bb - g_aa; identity when g_ab is negligible. The angle is evaluated in single precision
// on (d, 2 g_ab) scaled by a power of two, then (c, s) is renormalised in double so that
// c^2 + s^2 = 1 to double rounding: the rotation stays exactly orthogonal and only its angle
// carries a ~1e-7 relative error, which leaves g_ab at ~1e-7 of its value per visit — still
// ahead of the quadratic rate. Half the dependent FP64 latency of the all-double formula,
// which bounded every inner step.
__device__ __forceinline__ void rot_from_gram(double gpp, double gqq, double gpq, double& c, double& sn) {
  c = 1.0;
  sn = 0.0;
  if (fabs(gpq) > 1e-300 && gpq * gpq > 1e-34 * (gpp * gqq)) {
    const double dd = gqq - gpp, two = 2.0 * gpq;
    const double m = fmax(fabs(dd), fabs(two));
    const int ex = (__double2hiint(m) >> 20) & 0x7ff;         // biased exponent of m
    const double sc = __hiloint2double((2046 - ex) << 20, 0);  // 2^-(ex - 1023): m * sc in [1, 2)
    const float x = static_cast<float>(dd * sc), y = static_cast<float>(two * sc);
    const float hh = fmaf(x, x, y * y);
    const float tf = __fdividef(x >= 0.0f ? y : -y, fabsf(x) + hh * rsqrtf(hh));
    const float cf = rsqrtf(fmaf(tf, tf, 1.0f));
    const double cd = cf, sd = tf * cf;
    const double del = fma(cd, cd, sd * sd) - 1.0;        // |del| ~ 1e-7
    const double nrm = fma(del, fma(del, 0.375, -0.5), 1.0);  // (1 + del)^-1/2 to O(del^3)
    c = cd * nrm;
    sn = sd * nrm;
  }
}
template <int LD>
__device__ __forceinline__ void jrot(const double (*g)[LD], int a, int b, double& c, double& sn) {
  rot_from_gram(g[a][a], g[b][b], g[a][b], c, sn);
}

// Single-CTA one-sided Jacobi for small problems (rows, n <= 64): W (and the rotation
// accumulator V when nv > 0) resident in shared memory, cyclic round-robin sweeps over single
// column pairs (a warp per pair, lanes over rows, warp-reduced Gram entries), the convergence
// test on the device. One launch per SVD instead of (p - 1) round launches plus a host
// synchronisation per sweep — the low-rank regime's SVDs are a few dozen columns.
constexpr int kSmallN = 64;
__global__ void __launch_bounds__(256) jacobi_small_kernel(int rows, int n, int nv, double* W, i64 ldw, double* V,
                                                           i64 ldv, double tol, double stop_tol, int max_sweeps,
                                                           unsigned long long* offmax, int* sweeps_out) {
  extern __shared__ double jsm[];  // W, then V when nv > 0
  double(*Ws)[kSmallN + 1] = reinterpret_cast<double(*)[kSmallN + 1]>(jsm);
  double(*Vs)[kSmallN + 1] = reinterpret_cast<double(*)[kSmallN + 1]>(jsm + kSmallN * (kSmallN + 1));
  __shared__ unsigned long long s_off;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int e = t; e < kSmallN * kSmallN; e += 256) {
    const int r = e / kSmallN, c = e % kSmallN;
    Ws[r][c] = (r < rows && c < n) ? W[r * ldw + c] : 0.0;
    if (nv > 0) Vs[r][c] = (r < nv && c < n) ? V[r * ldv + c] : 0.0;
  }
  const int n2 = n + (n & 1);  // round-robin over an even count (a dummy column when n is odd)
  // pairing table: step s, slot k -> (a, b), a < b (round robin with column 0 fixed)
  __shared__ unsigned char pa[kSmallN - 1][kSmallN / 2], pb[kSmallN - 1][kSmallN / 2];
  for (int e = t; e < (n2 - 1) * (n2 / 2); e += 256) {
    const int st = e / (n2 / 2), k = e % (n2 / 2);
    auto ring = [&](int i) {
      if (i == 0) return 0;
      int x = i - 1 - st;
      if (x < 0) x += n2 - 1;
      return 1 + x;
    };
    const int a = ring(k), b = ring(n2 - 1 - k);
    pa[st][k] = static_cast<unsigned char>(a < b ? a : b);
    pb[st][k] = static_cast<unsigned char>(a < b ? b : a);
  }
  __syncthreads();
  // a half-warp per column pair (16 lanes x 4 rows), 16 pairs in flight per step
  const int h = lane >> 4, l16 = lane & 15;
  const unsigned hmask = h ? 0xffff0000u : 0x0000ffffu;
  int sweep = 0;
  double off2 = 0.0;  // 1 when some pair started the sweep above stop_tol
  while (sweep < max_sweeps) {
    if (t == 0) s_off = 0;
    double wmax = 0.0;
    for (int step = 0; step < n2 - 1; ++step) {
      for (int k = 2 * warp + h; k < n2 / 2; k += 16) {
        const int a = pa[step][k], b = pb[step][k];
        if (b >= n) continue;  // the dummy column (uniform over the half-warp)
        double xa[4], xb[4];
        double aa = 0.0, bb = 0.0, ab = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          xa[j] = Ws[l16 + 16 * j][a];
          xb[j] = Ws[l16 + 16 * j][b];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          aa = fma(xa[j], xa[j], aa);
          bb = fma(xb[j], xb[j], bb);
          ab = fma(xa[j], xb[j], ab);
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
          aa += __shfl_xor_sync(hmask, aa, o);
          bb += __shfl_xor_sync(hmask, bb, o);
          ab += __shfl_xor_sync(hmask, ab, o);
        }
        // cosine tests without a division: ab^2 > c^2 aa bb
        const double d = aa * bb, ab2 = ab * ab;
        if (ab2 > stop_tol * stop_tol * d) wmax = 1.0;  // this sweep does not meet the stop test
        if (ab2 > tol * tol * d && d > 0.0) {  // uniform over the half-warp
          double c, sn;
          rot_from_gram(aa, bb, ab, c, sn);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            Ws[l16 + 16 * j][a] = c * xa[j] - sn * xb[j];
            Ws[l16 + 16 * j][b] = sn * xa[j] + c * xb[j];
          }
          if (nv > 0) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const double va = Vs[l16 + 16 * j][a], vb = Vs[l16 + 16 * j][b];
              Vs[l16 + 16 * j][a] = c * va - sn * vb;
              Vs[l16 + 16 * j][b] = sn * va + c * vb;
            }
          }
        }
      }
      __syncthreads();
    }
    for (int o = 16; o > 0; o >>= 1) wmax = fmax(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
    if (lane == 0) atomicMax(&s_off, static_cast<unsigned long long>(__double_as_longlong(wmax)));
    __syncthreads();
    off2 = __longlong_as_double(static_cast<long long>(s_off));
    ++sweep;
    __syncthreads();
    if (off2 == 0.0) break;  // every pair started the sweep with cosine <= stop_tol
  }
  const double off = off2 == 0.0 ? stop_tol : 1.0;  // (the small kernel reports pass / fail only)
  for (int e = t; e < kSmallN * kSmallN; e += 256) {
    const int r = e / kSmallN, c = e % kSmallN;
    if (r < rows && c < n) W[r * ldw + c] = Ws[r][c];
    if (nv > 0 && r < nv && c < n) V[r * ldv + c] = Vs[r][c];
  }
  if (t == 0) {
    *sweeps_out = sweep;
    *offmax = static_cast<unsigned long long>(__double_as_longlong(off));
  }
}

// CS > 1: a thread-block cluster of CS CTAs shares one block pair, each CTA staging, reducing
// and rotating a contiguous slab of the rows; the 16x16 partial Grams are summed over the
// cluster through distributed shared memory in rank order (every CTA gets the identical Gram
// and runs the identical inner EVD). Used when few solves share the GPU (single-block latency).
// Per-SVD arguments of the round kernel, read from device memory so the p - 1 launches of a
// sweep are identical across SVDs of one shape class and their CUDA graph is reused (the
// round index and the inner-sweep count stay kernel parameters, fixed per graph node).
struct JacobiArgs {
  i64 rows, nv, ldw, ldv;
  double* W;
  double* V;
  unsigned long long* offmax;
  double tol;
  int p, prefetch_v;
};

// The round body, shared by the launch-per-round kernel (PDL: griddepcontrol between rounds) and
// the persistent sweep kernel (grid barriers between rounds). offmax: where this round's largest
// pair cosine goes.
template <int NB, int CS, bool PDL>
__device__ __forceinline__ void jacobi_round_body(const JacobiArgs* __restrict__ ja, unsigned long long* offmax,
                                                  int round, int inner_sweeps) {
  static_assert(NB == 8 || NB == 16, "8- or 16-column blocks (16 or 32 columns per pair)");
  const i64 rows_ = ja->rows, nv_ = ja->nv, ldw = ja->ldw, ldv = ja->ldv;
  double* W = ja->W;
  double* V = ja->V;
  const double tol = ja->tol;
  const int p = ja->p, prefetch_v = ja->prefetch_v;
  constexpr int JW = 2 * NB, T = 256, NT = JW / 8, CH = JW / 2, KS = JW / 4;
  extern __shared__ __align__(16) double dyn[];
  const int crank = static_cast<int>(blockIdx.x % CS), pk = static_cast<int>(blockIdx.x / CS);
  int rows, nv, rows4, nv4;
  {  // this CTA's slab of the W rows and of the V rows (multiples of 4)
    const int R = static_cast<int>(rows_), R4 = (R + 3) & ~3, NV = static_cast<int>(nv_), NV4 = (NV + 3) & ~3;
    const int cw = ((R4 / 4 + CS - 1) / CS) * 4, cv = ((NV4 / 4 + CS - 1) / CS) * 4;
    const int rw = crank * cw, rv = crank * cv;
    rows4 = max(0, min(cw, R4 - rw));
    rows = max(0, min(cw, R - rw));
    nv4 = max(0, min(cv, NV4 - rv));
    nv = max(0, min(cv, NV - rv));
    W += static_cast<i64>(rw) * ldw;
    V += static_cast<i64>(rv) * ldv;
  }
  const int cap = rows4 > nv4 ? rows4 : nv4;
  double* Wp = dyn;
  double* Vp = prefetch_v ? Wp + cap * JW : Wp;
  double* red = Wp + (prefetch_v ? 2 : 1) * cap * JW;  // one JW x JW partial Gram (the other three
                                                        // reduction slots reuse g and rot)
  __shared__ double g[2][JW][JW + 1];
  __shared__ double rot[JW][JW + 1];
  __shared__ double s_off;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  // round-robin pairing (round_robin() on the host): ring[0] = 0, ring[i] = 1 + (i - 1 - round)
  // mod (p - 1); CTA k takes (ring[k], ring[p - 1 - k]). No global load before the staging.
  auto ring = [&](int i) { return i == 0 ? 0 : 1 + ((i - 1 - round) % (p - 1) + (p - 1)) % (p - 1); };
  const int bi = ring(pk), bj = ring(p - 1 - pk);
  auto gcol = [&](int c) -> i64 { return c < NB ? static_cast<i64>(bi) * NB + c : static_cast<i64>(bj) * NB + c - NB; };

  // staging: thread t moves 16-byte chunk q = t % CH (pair columns 2q, 2q+1) of rows t/CH, t/CH + T/CH, ...
  const int q = t % CH, r0 = t / CH;
  const i64 gq = gcol(2 * q);
  const int soff = (q ^ ((r0 & 3) << 1)) << 1;  // swizzled chunk: r & 3 is fixed per thread
  auto stage = [&](double* dst, const double* src, i64 ld, int n, int n4) {
    const double* sp = src + r0 * ld + gq;
    double* dp = dst + r0 * JW + soff;
    for (int r = r0; r < n4; r += T / CH, sp += (T / CH) * ld, dp += (T / CH) * JW) cp_async16(dp, r < n ? sp : src, r < n);
  };
  // Programmatic dependent launch (when the host enables it): everything above only reads the
  // argument block; the previous round's writes to W are visible after griddepcontrol.wait, and
  // the next round may start launching once every CTA of this one has issued its loads.
  if constexpr (PDL) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  stage(Wp, W, ldw, rows, rows4);
  asm volatile("cp.async.commit_group;\n" ::);
  if constexpr (PDL) asm volatile("griddepcontrol.launch_dependents;\n" ::);
  if (prefetch_v) {  // second group: the V pair, consumed only after the rotation is known
    stage(Vp, V, ldv, nv, nv4);
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 1;\n" ::);
  } else {
    asm volatile("cp.async.wait_group 0;\n" ::);
  }
  __syncthreads();

  // ---- Gram (DMMA): rows split over the warps; lane reads column ti*8 + lane/4 of row k + lane%4
  {
    int oc[NT];
#pragma unroll
    for (int ti = 0; ti < NT; ++ti) oc[ti] = jswz(lane & 3, ti * 8 + (lane >> 2));
    double acc[NT * NT][2];
#pragma unroll
    for (int e = 0; e < NT * NT; ++e) acc[e][0] = acc[e][1] = 0.0;
    for (int k = 4 * warp; k < rows4; k += 32) {
      const double* row = Wp + (k + (lane & 3)) * JW;
      double x[NT];
#pragma unroll
      for (int ti = 0; ti < NT; ++ti) x[ti] = row[oc[ti]];
#pragma unroll
      for (int ti = 0; ti < NT; ++ti)
#pragma unroll
        for (int tj = 0; tj < NT; ++tj) dmma(acc[ti * NT + tj], x[ti], x[tj]);
    }
    // fixed-order reduction of the 8 warp partials through 4 slots (red, g[1], rot, g[0]):
    // warps 4..7 publish, warps 0..3 fold them in (w + (w + 4)), publish, then sum slots 0..3
    const int sl = warp & 3;  // this warp's slot (warps w and w + 4 share slot w)
    double* const sp = sl == 0 ? red : (sl == 1 ? &g[1][0][0] : (sl == 2 ? &rot[0][0] : &g[0][0][0]));
    const int sld = sl == 0 ? JW : JW + 1;
    auto publish = [&]() {
#pragma unroll
      for (int e = 0; e < NT * NT; ++e) {
        const int r = (e / NT) * 8 + (lane >> 2), c = (e % NT) * 8 + (lane & 3) * 2;
        sp[r * sld + c] = acc[e][0];
        sp[r * sld + c + 1] = acc[e][1];
      }
    };
    if (warp >= 4) publish();
    __syncthreads();
    if (warp < 4) {
#pragma unroll
      for (int e = 0; e < NT * NT; ++e) {
        const int r = (e / NT) * 8 + (lane >> 2), c = (e % NT) * 8 + (lane & 3) * 2;
        acc[e][0] += sp[r * sld + c];
        acc[e][1] += sp[r * sld + c + 1];
      }
    }
    __syncthreads();
    if (warp < 4) publish();
    __syncthreads();
    for (int e = t; e < JW * JW; e += T) {  // thread e reads slot 3 == g[0] at e before writing it
      const int r = e / JW, c = e % JW;
      g[0][r][c] = (red[r * JW + c] + g[1][r][c]) + (rot[r][c] + g[0][r][c]);
    }
    __syncthreads();
    for (int e = t; e < JW * JW; e += T) rot[e / JW][e % JW] = (e / JW == e % JW) ? 1.0 : 0.0;
  }
  if constexpr (CS > 1) {  // sum the cluster's partial Grams in rank order
    __shared__ double gpart[JW * JW];
    for (int e = t; e < JW * JW; e += T) gpart[e] = g[0][e / JW][e % JW];
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();
    for (int e = t; e < JW * JW; e += T) {
      double v = 0.0;
#pragma unroll
      for (int r = 0; r < CS; ++r) v += cluster.map_shared_rank(gpart, r)[e];
      g[0][e / JW][e % JW] = v;
    }
    cluster.sync();  // every remote read done before any CTA of the cluster may exit
  }
  __syncthreads();

  // ---- off-diagonal measure (all pairs of the JW columns)
  {
    double mx = 0.0;
    for (int e = t; e < JW * JW; e += T) {
      const int a = e / JW, b = e % JW;
      if (a < b) {
        const double d = sqrt(g[0][a][a]) * sqrt(g[0][b][b]);
        if (d > 0.0) mx = fmax(mx, fabs(g[0][a][b]) / d);
      }
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (t == 0) s_off = 0.0;
    __syncthreads();
    if (lane == 0)
      atomicMax(reinterpret_cast<unsigned long long*>(&s_off), static_cast<unsigned long long>(__double_as_longlong(mx)));
    __syncthreads();
  }
  const double off0 = s_off;
  if (t == 0 && crank == 0) atomicMax(offmax, static_cast<unsigned long long>(__double_as_longlong(off0)));
  if (off0 <= tol) {
    asm volatile("cp.async.wait_group 0;\n" ::);  // no copy may land after the CTA retires
    return;
  }

  // ---- inner Jacobi on the Gram, one barrier per step. inner_sweeps > 0: that many cyclic
  // sweeps over all column pairs (JW - 1 steps); inner_sweeps == 0: the NB^2 cross pairs only
  // (NB steps, column i of block I with column (i + step) % NB of block J). The host uses the
  // full sweep in the first round of every outer sweep (each block appears once there, so its
  // internal pairs are rotated once per sweep) and cross steps elsewhere: every column pair is
  // then rotated exactly once per outer sweep, a cyclic Jacobi ordering.
  int cur = 0;
  const bool cross = inner_sweeps == 0;
  const int nsteps = cross ? NB : (JW - 1) * inner_sweeps;
  if constexpr (NB == 8) {
    // Warp-synchronous EVD (16 x 16): warp 0 runs every step with __syncwarp between steps
    // instead of a CTA barrier. Lane l computes rotation k = l % 8 (four copies), owns the Gram
    // 2x2 blocks (P = l / 4, Q = 2 (l % 4) + {0, 1}) with the other rotations taken by shuffles,
    // and rotates rows l / 8 + 4 j (j < 4) of the accumulator for its own pair k.
    if (warp == 0) {
      for (int it = 0; it < nsteps; ++it) {
        const int step = cross ? it : it % (JW - 1);
        auto pair_of = [&](int k, int& a, int& b) {
          if (cross) {
            a = k;
            b = NB + ((k + step) & (NB - 1));
          } else {
            jpair<JW>(step, k, a, b);
          }
        };
        const int k = lane & 7, P = lane >> 2;
        int a, b, aP, bP;
        pair_of(k, a, b);
        pair_of(P, aP, bP);
        double c, sn;
        jrot(g[cur], a, b, c, sn);
        const double cP = __shfl_sync(0xffffffffu, c, P), sP = __shfl_sync(0xffffffffu, sn, P);
        const int nx = cur ^ 1;
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          const int Q = 2 * (lane & 3) + qq;
          int aQ, bQ;
          pair_of(Q, aQ, bQ);
          const double cQ = __shfl_sync(0xffffffffu, c, Q), sQ = __shfl_sync(0xffffffffu, sn, Q);
          const double x00 = g[cur][aP][aQ], x01 = g[cur][aP][bQ], x10 = g[cur][bP][aQ], x11 = g[cur][bP][bQ];
          const double y00 = cQ * x00 - sQ * x01, y01 = sQ * x00 + cQ * x01;  // columns: G J_Q
          const double y10 = cQ * x10 - sQ * x11, y11 = sQ * x10 + cQ * x11;
          g[nx][aP][aQ] = cP * y00 - sP * y10;  // rows: J_P^T (G J_Q)
          g[nx][bP][aQ] = sP * y00 + cP * y10;
          g[nx][aP][bQ] = cP * y01 - sP * y11;
          g[nx][bP][bQ] = sP * y01 + cP * y11;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = (lane >> 3) + 4 * j;
          const double ra = rot[r][a], rb = rot[r][b];
          rot[r][a] = c * ra - sn * rb;
          rot[r][b] = sn * ra + c * rb;
        }
        __syncwarp();
        cur = nx;
      }
    }
    __syncthreads();
  }
  for (int it = 0; NB != 8 && it < nsteps; ++it) {
    const int step = cross ? it : it % (JW - 1);
    auto pair_of = [&](int k, int& a, int& b) {
      if (cross) {
        a = k;
        b = NB + ((k + step) & (NB - 1));
      } else {
        jpair<JW>(step, k, a, b);
      }
    };
    // 2x2 blocks (P, Q) of the pairing: NB^2 of them, one per thread (NB = 16) or the first 64
    if (t < NB * NB) {
      const int P = t / NB, Q = t % NB;
      int aP, bP, aQ, bQ;
      pair_of(P, aP, bP);
      pair_of(Q, aQ, bQ);
      double cP, sP, cQ, sQ;
      jrot(g[cur], aP, bP, cP, sP);
      jrot(g[cur], aQ, bQ, cQ, sQ);
      const double x00 = g[cur][aP][aQ], x01 = g[cur][aP][bQ], x10 = g[cur][bP][aQ], x11 = g[cur][bP][bQ];
      const double y00 = cQ * x00 - sQ * x01, y01 = sQ * x00 + cQ * x01;  // columns: G J_Q
      const double y10 = cQ * x10 - sQ * x11, y11 = sQ * x10 + cQ * x11;
      const int nx = cur ^ 1;  // rows: J_P^T (G J_Q)
      g[nx][aP][aQ] = cP * y00 - sP * y10;
      g[nx][bP][aQ] = sP * y00 + cP * y10;
      g[nx][aP][bQ] = cP * y01 - sP * y11;
      g[nx][bP][bQ] = sP * y01 + cP * y11;
    }
    // accumulated rotation: JW rows x NB pairs; NB = 8 uses the threads left over above
    constexpr int RU = JW * NB;
    for (int u = (NB == 8 ? t - 64 : t); u >= 0 && u < RU; u += (NB == 8 ? RU : T)) {
      const int k = u / JW, r = u % JW;
      int a, b;
      pair_of(k, a, b);
      double c, sn;
      jrot(g[cur], a, b, c, sn);
      const double ra = rot[r][a], rb = rot[r][b];
      rot[r][a] = c * ra - sn * rb;
      rot[r][b] = sn * ra + c * rb;
    }
    __syncthreads();
    cur ^= 1;
  }

  // ---- apply: M_pair <- M_pair rot from the staged copy; B fragments (rot) live in registers
  double bf[KS][NT];
#pragma unroll
  for (int kk = 0; kk < KS; ++kk)
#pragma unroll
    for (int ct = 0; ct < NT; ++ct) bf[kk][ct] = rot[kk * 4 + (lane & 3)][ct * 8 + (lane >> 2)];
  int ao[KS];  // swizzled A-fragment offsets: row rt*8 + lane/4 (r & 3 == (lane/4) & 3), column kk*4 + lane%4
#pragma unroll
  for (int kk = 0; kk < KS; ++kk) ao[kk] = jswz((lane >> 2) & 3, kk * 4 + (lane & 3));
  i64 cc[NT];
#pragma unroll
  for (int ct = 0; ct < NT; ++ct) cc[ct] = gcol(ct * 8 + (lane & 3) * 2);
  // two row tiles per iteration: independent DMMA chains hide the DMMA latency
  auto apply = [&](const double* Sp, double* M, i64 ld, int n, int n4) {
    const int tiles = (n + 7) >> 3;
    for (int rt = warp; rt < tiles; rt += 2 * (T / 32)) {
      const bool two_tiles = rt + T / 32 < tiles;  // warp-uniform
      const int r = rt * 8 + (lane >> 2), r2 = r + 8 * (T / 32);
      double o[NT][2], pz[NT][2];
#pragma unroll
      for (int ct = 0; ct < NT; ++ct) o[ct][0] = o[ct][1] = pz[ct][0] = pz[ct][1] = 0.0;
      double a[KS], b[KS];
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {  // rows past the staged block read as 0 (no divergence)
        a[kk] = r < n4 ? Sp[r * JW + ao[kk]] : 0.0;
        b[kk] = two_tiles && r2 < n4 ? Sp[r2 * JW + ao[kk]] : 0.0;
      }
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
#pragma unroll
        for (int ct = 0; ct < NT; ++ct) dmma(o[ct], a[kk], bf[kk][ct]);
        if (two_tiles) {
#pragma unroll
          for (int ct = 0; ct < NT; ++ct) dmma(pz[ct], b[kk], bf[kk][ct]);
        }
      }
      if (r < n) {
#pragma unroll
        for (int ct = 0; ct < NT; ++ct) *reinterpret_cast<double2*>(M + r * ld + cc[ct]) = make_double2(o[ct][0], o[ct][1]);
      }
      if (two_tiles && r2 < n) {
#pragma unroll
        for (int ct = 0; ct < NT; ++ct)
          *reinterpret_cast<double2*>(M + r2 * ld + cc[ct]) = make_double2(pz[ct][0], pz[ct][1]);
      }
    }
  };
  apply(Wp, W, ldw, rows, rows4);
  if (nv == 0) return;
  // V pair: prefetched into Vp, or staged now into the (free) Wp buffer
  __syncthreads();
  if (!prefetch_v) {
    stage(Vp, V, ldv, nv, nv4);
    asm volatile("cp.async.commit_group;\n" ::);
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  apply(Vp, V, ldv, nv, nv4);
}

template <int NB, int CS>
__global__ void __launch_bounds__(256, NB == 8 ? 2 : 1)
    jacobi_round_resident_kernel(const JacobiArgs* __restrict__ ja, int round, int inner_sweeps) {
  jacobi_round_body<NB, CS, true>(ja, ja->offmax, round, inner_sweeps);
}

// Persistent Jacobi: every sweep of one SVD in ONE cooperative launch (the p - 1 rounds of a
// sweep separated by grid barriers, the stop test on the device) instead of p - 1 launches per
// sweep and a host round trip after each sweep. Same rounds, same pairing, same arithmetic: the
// result is bitwise that of the launch-per-round path. Sweep s takes its largest cosine in
// slot s % 3 of ja->offmax (three slots: CTA 0 clears slot (s + 1) % 3 at the start of sweep s,
// whose last readers finished before the first barrier of sweep s - 1). sweeps_out: the sweeps
// executed.
template <int NB, int CS>
__global__ void __launch_bounds__(256, NB == 8 ? 2 : 1)
    jacobi_sweeps_kernel(const JacobiArgs* __restrict__ ja, double stop_tol, int max_sweeps, int* sweeps_out,
                         unsigned* __restrict__ ver) {
  cg::grid_group grid = cg::this_grid();
  const int p = ja->p;
  int sweep = 0;
  // ver != nullptr: point-to-point ordering between rounds instead of a grid barrier. ver[b]
  // counts the CTAs that have finished a round on column block b (CS per round): the CTA that
  // takes (bi, bj) in a round waits until both blocks carry every earlier round, and publishes
  // them when its own writes are out. A block is touched by one cluster per round, so this is
  // the only ordering the rounds need; the grid barrier stays at the end of each sweep (the
  // sweep's largest cosine must be complete before the stop test).
  unsigned gen = 0;  // rounds finished so far
  const int pk = static_cast<int>(blockIdx.x / CS);
  while (sweep < max_sweeps) {
    unsigned long long* slot = ja->offmax + sweep % 3;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(ja->offmax + (sweep + 1) % 3, 0ull);
    for (int r = 0; r < p - 1; ++r) {
      if (ver) {
        auto ring = [&](int i) { return i == 0 ? 0 : 1 + ((i - 1 - r) % (p - 1) + (p - 1)) % (p - 1); };
        const int bi = ring(pk), bj = ring(p - 1 - pk);
        if (threadIdx.x == 0) {
          const unsigned need = static_cast<unsigned>(CS) * gen;
          unsigned v;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ver + bi) : "memory");
          } while (v < need);
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ver + bj) : "memory");
          } while (v < need);
        }
        __syncthreads();
        jacobi_round_body<NB, CS, false>(ja, slot, r, r == 0 ? 1 : 0);
        __syncthreads();  // every thread's stores of this round are issued
        if (threadIdx.x == 0) {
          __threadfence();
          atomicAdd(ver + bi, 1u);
          atomicAdd(ver + bj, 1u);
        }
        ++gen;
      } else {
        jacobi_round_body<NB, CS, false>(ja, slot, r, r == 0 ? 1 : 0);
        grid.sync();
      }
    }
    if (ver) grid.sync();
    ++sweep;
    const double off = __longlong_as_double(static_cast<long long>(__ldcg(slot)));
    if (off <= stop_tol) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps_out = sweep;
}

// A[:, c] /= s[c] (columns with s[c] == 0 are zeroed)
__global__ void div_cols_kernel(i64 rows, i64 cols, double* A, i64 lda, const double* s) {
  const i64 total = rows * cols;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 r = e / cols, c = e % cols;
    const double sv = s[c];
    A[r * lda + c] = sv > 0.0 ? A[r * lda + c] / sv : 0.0;
  }
}

// dst[idx[p], :] = src[p, :]
__global__ void scatter_rows_int_kernel(i64 l, i64 c, const double* __restrict__ src, i64 lds,
                                        const int* __restrict__ idx, double* __restrict__ dst, i64 ldd) {
  const i64 total = l * c;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 p = e / c, j = e % c;
    dst[static_cast<i64>(idx[p]) * ldd + j] = src[p * lds + j];
  }
}

__global__ void scale_cols_kernel(i64 rows, i64 cols, double* A, i64 lda, const double* s, i64 ldo, double* out,
                                  const int* perm) {
  const i64 total = rows * cols;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 r = e / cols, c = e % cols;
    const int src = perm[c];
    const double sv = s[c];
    out[r * ldo + c] = sv > 0.0 ? A[r * lda + src] / sv : 0.0;
  }
}

}  // namespace

// ---------------------------------------------------------------- Householder QR
void householder_qr(cudaStream_t s, i64 rows, i64 cols, double* X, i64 ldx, double* R, i64 ldr) {
  if (rows < cols) throw std::invalid_argument("householder_qr: rows < cols");
  const i64 np = (cols + HNB - 1) / HNB;
  DBuf<double> tau(cols, s), Tall(np * HNB * HNB, s), V(rows * HNB, s), S(HNB * HNB, s),
      W1(HNB * std::max<i64>(cols, 1), s), W2(HNB * std::max<i64>(cols, 1), s);
  for (i64 p = 0; p < np; ++p) {
    const i64 p0 = p * HNB;
    const int nb = static_cast<int>(std::min<i64>(HNB, cols - p0));
    const i64 pr = rows - p0;
    double* panel = X + p0 * ldx + p0;
    prof::Scope scope(prof::kQrFallback, s, 4.0 * pr * nb * nb, 16.0 * pr * nb);
    hh_panel_kernel<<<1, HTHREADS, 0, s>>>(pr, nb, panel, ldx, tau.get() + p0);
    DFCG_LAUNCH_CHECK();
    hh_extract_v<<<grid_for(pr * nb), 256, 0, s>>>(pr, nb, panel, ldx, V.get());
    DFCG_LAUNCH_CHECK();
    gemm(s, true, false, nb, nb, pr, 1.0, V.get(), nb, V.get(), nb, 0.0, S.get(), nb);
    double* T = Tall.get() + p * HNB * HNB;
    hh_build_t<<<1, HNB, 0, s>>>(nb, S.get(), tau.get() + p0, T);
    DFCG_LAUNCH_CHECK();
    const i64 rem = cols - p0 - nb;
    if (rem > 0) {
      double* A2 = X + p0 * ldx + p0 + nb;
      gemm(s, true, false, nb, rem, pr, 1.0, V.get(), nb, A2, ldx, 0.0, W1.get(), rem);        // V^T A2
      gemm(s, true, false, nb, rem, nb, 1.0, T, nb, W1.get(), rem, 0.0, W2.get(), rem);         // T^T W1
      gemm(s, false, false, pr, rem, nb, -1.0, V.get(), nb, W2.get(), rem, 1.0, A2, ldx);       // A2 -= V W2
    }
  }
  if (R) {
    extract_upper<<<grid_for(cols * cols), 256, 0, s>>>(cols, X, ldx, R, ldr);
    DFCG_LAUNCH_CHECK();
  }
  // Q = H_1 ... H_np [I; 0], accumulated backwards into a fresh buffer then copied over X.
  DBuf<double> Q(rows * cols, s);
  set_identity(s, rows, cols, Q.get(), cols);
  for (i64 p = np - 1; p >= 0; --p) {
    const i64 p0 = p * HNB;
    const int nb = static_cast<int>(std::min<i64>(HNB, cols - p0));
    const i64 pr = rows - p0;
    hh_extract_v<<<grid_for(pr * nb), 256, 0, s>>>(pr, nb, X + p0 * ldx + p0, ldx, V.get());
    DFCG_LAUNCH_CHECK();
    const double* T = Tall.get() + p * HNB * HNB;
    const i64 qc = cols - p0;
    double* Qs = Q.get() + p0 * cols + p0;
    gemm(s, true, false, nb, qc, pr, 1.0, V.get(), nb, Qs, cols, 0.0, W1.get(), qc);   // V^T Q
    gemm(s, false, false, nb, qc, nb, 1.0, T, nb, W1.get(), qc, 0.0, W2.get(), qc);    // T W1
    gemm(s, false, false, pr, qc, nb, -1.0, V.get(), nb, W2.get(), qc, 1.0, Qs, cols); // Q -= V W2
  }
  copy2d(s, rows, cols, Q.get(), cols, X, ldx);
}

// ---------------------------------------------------------------- CholeskyQR2 + fallback
bool cholqr_factor(cudaStream_t s, i64 rows, i64 cols, const double* X, i64 ldx, double* Rinv, i64 ldr) {
  if (cols <= 0) return true;
  DBuf<int> fail(1, s);
  fail.zero(s);
  DBuf<double> G(cols * cols, s);
  gram_upper(s, rows, cols, X, ldx, G.get(), cols);
  cholesky_inverse(s, cols, G.get(), cols, Rinv, ldr, 1e-11, fail.get());
  int h_fail = 0;
  DFCG_CUDA(cudaMemcpyAsync(&h_fail, fail.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  DFCG_CUDA(cudaStreamSynchronize(s));
  return h_fail == 0;
}

// dg[i] = G[i, i]
__global__ void diag_copy_kernel(i64 n, const double* __restrict__ G, i64 ldg, double* __restrict__ dg) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    dg[i] = G[i * ldg + i];
}

// out = min_i R[i, i]^2 / dg[i]: the smallest pivot of the Cholesky of the unit-diagonal Gram
// D^-1 G D^-1 (dg = diag G before the factorisation, R its factor) = min_i sin^2 of the angle
// between column i and the span of the columns before it. One CTA.
__global__ void min_scaled_pivot_kernel(i64 n, const double* __restrict__ R, i64 ldr, const double* __restrict__ dg,
                                        double* __restrict__ out) {
  __shared__ double sm[256];
  double v = 1.0;
  for (i64 i = threadIdx.x; i < n; i += 256) {
    const double r = R[i * ldr + i], d = dg[i];
    if (d > 0.0) v = fmin(v, r * r / d);
  }
  sm[threadIdx.x] = v;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (static_cast<int>(threadIdx.x) < o) sm[threadIdx.x] = fmin(sm[threadIdx.x], sm[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}

bool cholqr2_r(cudaStream_t s, i64 rows, i64 cols, const double* A, i64 lda, double* R, double* Rinv,
               double rel_tol1, bool trans, bool warm, bool* used_warm) {
  if (used_warm) *used_warm = false;
  if (cols <= 0) return true;
  DBuf<int> fail(1, s);
  fail.zero(s);
  DBuf<double> G(cols * cols, s), R1inv(cols * cols, s);
  DBuf<double> dg(cols + 1, s);  // diag of the Gram, then the smallest scaled pivot
  static const bool trace_qr = std::getenv("DFCG_TRACE_CHOLQR") != nullptr;
  // Warm start: the caller's R / Rinv hold the factor of the PREVIOUS operator A' (A changes
  // slowly from one APG iteration to the next). P = R'^-1 preconditions A: Q1 = A P is close to
  // orthonormal, so ONE CholQR pass on Q1 has CholeskyQR2's accuracy (orthogonality ~ eps
  // cond(A P)^2), and the pass that only served to build the preconditioner — the Gram of A and
  // its Cholesky, m w^2 FLOPs and a w x w factorisation per iteration — is skipped:
  //   Q1 = A P,  R1^T R1 = Q1^T Q1,  R = R1 R',  Rinv = P R1^-1.
  // Accepted only when the smallest pivot of the (unit-diagonal) Gram of Q1 is >= 1e-4
  // (DFCG_CHOLQR_WARM_PIVOT), i.e. cond(A P)^2 <~ 1e4-1e5 and the loss of orthogonality <~ 1e-11;
  // otherwise the cold CholeskyQR2 below runs. The caller refreshes with a cold factorisation
  // every few iterations (R' P - I accumulates rounding). DFCG_CHOLQR_WARM=0 disables.
  static const int warm_env = std::getenv("DFCG_CHOLQR_WARM") ? std::atoi(std::getenv("DFCG_CHOLQR_WARM")) : 1;
  static const double warm_piv =
      std::getenv("DFCG_CHOLQR_WARM_PIVOT") ? std::atof(std::getenv("DFCG_CHOLQR_WARM_PIVOT")) : 1e-4;
  if (warm && warm_env != 0) {
    DBuf<double> Q1(rows * cols, s), R1winv(cols * cols, s);
    if (trans) gemm_ta_upper_b(s, rows, cols, 1.0, A, lda, Rinv, cols, 0.0, Q1.get(), cols);
    else gemm_upper_b(s, rows, cols, 1.0, A, lda, Rinv, cols, 0.0, Q1.get(), cols);
    gram_upper(s, rows, cols, Q1.get(), cols, G.get(), cols);
    diag_copy_kernel<<<grid_for(cols), 256, 0, s>>>(cols, G.get(), cols, dg.get());
    DFCG_LAUNCH_CHECK();
    cholesky_inverse(s, cols, G.get(), cols, R1winv.get(), cols, 1e-11, fail.get());
    min_scaled_pivot_kernel<<<1, 256, 0, s>>>(cols, G.get(), cols, dg.get(), dg.get() + cols);
    DFCG_LAUNCH_CHECK();
    int w_fail = 0;
    double w_piv = 0.0;
    DFCG_CUDA(cudaMemcpyAsync(&w_fail, fail.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    DFCG_CUDA(cudaMemcpyAsync(&w_piv, dg.get() + cols, sizeof(double), cudaMemcpyDeviceToHost, s));
    DFCG_CUDA(cudaStreamSynchronize(s));
    if (trace_qr)
      std::fprintf(stderr, "[cholqr2_r] %lld x %lld warm pass: smallest scaled pivot %.3e%s\n", (long long)rows,
                   (long long)cols, w_piv, w_fail ? " (breakdown)" : "");
    if (!w_fail && w_piv >= warm_piv) {
      // R = R1 R' and Rinv = P R1^-1 (upper triangles, lower parts stored as zeros); Q1 is scratch
      gemm_upper_b(s, cols, cols, 1.0, G.get(), cols, R, cols, 0.0, Q1.get(), cols);
      copy2d(s, cols, cols, Q1.get(), cols, R, cols);
      gemm_upper_b(s, cols, cols, 1.0, Rinv, cols, R1winv.get(), cols, 0.0, Q1.get(), cols);
      copy2d(s, cols, cols, Q1.get(), cols, Rinv, cols);
      if (used_warm) *used_warm = true;
      if (trace_qr) {  // consistency of the accumulated pair: max |R Rinv - I|
        gemm_upper_b(s, cols, cols, 1.0, R, cols, Rinv, cols, 0.0, Q1.get(), cols);
        std::vector<double> h(static_cast<size_t>(cols * cols));
        DFCG_CUDA(cudaMemcpyAsync(h.data(), Q1.get(), sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s));
        DFCG_CUDA(cudaStreamSynchronize(s));
        double mx = 0.0;
        for (i64 i = 0; i < cols; ++i)
          for (i64 j = 0; j < cols; ++j)
            mx = std::max(mx, std::fabs(h[static_cast<size_t>(i * cols + j)] - (i == j ? 1.0 : 0.0)));
        std::fprintf(stderr, "[cholqr2_r] warm pair: max |R Rinv - I| = %.3e\n", mx);
      }
      return true;
    }
    fail.zero(s);
  }
  // pass 1: R1^T R1 = A^T A, Q1 = A R1^-1 (orthogonal to ~eps cond(A)^2)
  if (trans) gram_upper_nt(s, cols, rows, A, lda, G.get(), cols);
  else gram_upper(s, rows, cols, A, lda, G.get(), cols);
  diag_copy_kernel<<<grid_for(cols), 256, 0, s>>>(cols, G.get(), cols, dg.get());
  DFCG_LAUNCH_CHECK();
  cholesky_inverse(s, cols, G.get(), cols, R1inv.get(), cols, rel_tol1, fail.get());
  min_scaled_pivot_kernel<<<1, 256, 0, s>>>(cols, G.get(), cols, dg.get(), dg.get() + cols);
  DFCG_LAUNCH_CHECK();
  int h_fail = 0;
  double h_piv = 0.0;
  DFCG_CUDA(cudaMemcpyAsync(&h_fail, fail.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  DFCG_CUDA(cudaMemcpyAsync(&h_piv, dg.get() + cols, sizeof(double), cudaMemcpyDeviceToHost, s));
  DFCG_CUDA(cudaStreamSynchronize(s));
  if (h_fail) return false;
  // One pass is enough when A is well conditioned. Q_A = A R1^-1 is never formed: the iteration
  // works on R_A alone and only needs A = Q_A R_A with Q_A^T Q_A = I + E; one pass leaves
  // |E| ~ eps cond(A D^-1)^2, which perturbs the SVT input by |E| |A| (the SVT is
  // nonexpansive). The smallest scaled pivot bounds cond(A D^-1)^2 from below by its inverse
  // and tracks it within a small factor on the APG operators (dense, noisy blocks): at
  // pivot >= DFCG_CHOLQR_SINGLE_PIVOT (default 1e-4, the warm pass's threshold) |E| <~ 1e-11. The
  // second pass (2 m w^2 of the iteration's FLOPs: the explicit Q1 and its Gram) runs only below
  // that — always at a c2 block, whose operator's smallest pivot is ~1e-8 (the warm start above is
  // what saves the pass there). DFCG_CHOLQR_SINGLE=0: always two passes.
  static const int single_env = std::getenv("DFCG_CHOLQR_SINGLE") ? std::atoi(std::getenv("DFCG_CHOLQR_SINGLE")) : 1;
  static const double single_piv =
      std::getenv("DFCG_CHOLQR_SINGLE_PIVOT") ? std::atof(std::getenv("DFCG_CHOLQR_SINGLE_PIVOT")) : 1e-4;
  if (trace_qr)
    std::fprintf(stderr, "[cholqr2_r] %lld x %lld smallest scaled pivot %.3e\n", (long long)rows, (long long)cols, h_piv);
  if (single_env != 0 && h_piv >= single_piv) {
    copy2d(s, cols, cols, G.get(), cols, R, cols);
    copy2d(s, cols, cols, R1inv.get(), cols, Rinv, cols);
    return true;
  }
  DBuf<double> Q1(rows * cols, s), R2inv(cols * cols, s);
  if (trans) gemm_ta_upper_b(s, rows, cols, 1.0, A, lda, R1inv.get(), cols, 0.0, Q1.get(), cols);
  else gemm_upper_b(s, rows, cols, 1.0, A, lda, R1inv.get(), cols, 0.0, Q1.get(), cols);
  // pass 2 on the explicit Q1: R2^T R2 = Q1^T Q1; A = (Q1 R2^-1) (R2 R1)
  gram_upper(s, rows, cols, Q1.get(), cols, R, cols);
  cholesky_inverse(s, cols, R, cols, R2inv.get(), cols, 1e-11, fail.get());
  DFCG_CUDA(cudaMemcpyAsync(&h_fail, fail.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  DFCG_CUDA(cudaStreamSynchronize(s));
  if (h_fail) return false;
  // R = R2 R1 (G still holds R1), Rinv = R1^-1 R2^-1: products of upper triangles whose lower
  // parts are stored as zeros (Q1 is free scratch now)
  gemm_upper_b(s, cols, cols, 1.0, R, cols, G.get(), cols, 0.0, Q1.get(), cols);
  copy2d(s, cols, cols, Q1.get(), cols, R, cols);
  gemm_upper_b(s, cols, cols, 1.0, R1inv.get(), cols, R2inv.get(), cols, 0.0, Rinv, cols);
  return true;
}

bool thin_qr(cudaStream_t s, i64 rows, i64 cols, double* X, i64 ldx, double* R, i64 ldr, int passes) {
  if (cols <= 0) return false;
  if (rows < cols) throw std::invalid_argument("thin_qr: rows < cols");
  if (R) passes = 2;
  DBuf<int> fail(1, s);
  fail.zero(s);
  DBuf<double> G(cols * cols, s), Rinv(cols * cols, s), Q1(rows * cols, s), Q2, R1;
  const double rel_tol = 1e-11;
  // pass 1 (the Cholesky reads only the upper triangle of the Gram)
  gram_upper(s, rows, cols, X, ldx, G.get(), cols);
  cholesky_inverse(s, cols, G.get(), cols, Rinv.get(), cols, rel_tol, fail.get());
  gemm_upper_b(s, rows, cols, 1.0, X, ldx, Rinv.get(), cols, 0.0, Q1.get(), cols);
  if (R) {
    R1.alloc(cols * cols, s);
    DFCG_CUDA(cudaMemcpyAsync(R1.get(), G.get(), sizeof(double) * cols * cols, cudaMemcpyDeviceToDevice, s));
  }
  const double* Qfinal = Q1.get();
  if (passes >= 2) {
    Q2.alloc(rows * cols, s);
    gram_upper(s, rows, cols, Q1.get(), cols, G.get(), cols);
    cholesky_inverse(s, cols, G.get(), cols, Rinv.get(), cols, rel_tol, fail.get());
    gemm_upper_b(s, rows, cols, 1.0, Q1.get(), cols, Rinv.get(), cols, 0.0, Q2.get(), cols);
    Qfinal = Q2.get();
  }
  int h_fail = 0;
  DFCG_CUDA(cudaMemcpyAsync(&h_fail, fail.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  DFCG_CUDA(cudaStreamSynchronize(s));
  if (h_fail) {
    householder_qr(s, rows, cols, X, ldx, R, ldr);
    return true;
  }
  copy2d(s, rows, cols, Qfinal, cols, X, ldx);
  if (R) gemm(s, false, false, cols, cols, cols, 1.0, G.get(), cols, R1.get(), cols, 0.0, R, ldr);  // R2 R1
  return false;
}

// ---------------------------------------------------------------- thin SVD
void thin_svd(cudaStream_t s, i64 rows, i64 cols, double* A, i64 lda, double* U, i64 ldu, double* V, i64 ldv,
              std::vector<double>& s_host, double u_tau) {
  s_host.assign(static_cast<size_t>(std::max<i64>(cols, 0)), 0.0);
  if (cols <= 0) return;
  if (rows < cols) throw std::invalid_argument("thin_svd: rows < cols");
  // Preconditioning (Drmac-Veselic style): columns sorted by norm, thin QR  A P = Q R, then
  // one-sided Jacobi on R^T (graded, near-orthogonal columns -> few sweeps):
  //   R^T J = W (orthogonal columns, norms sigma)  =>  A = (Q J) Sigma (P W Sigma^-1)^T.
  DBuf<double> nrm(cols, s);
  col_norms(s, rows, cols, A, lda, nrm.get());
  std::vector<double> h_nrm(cols);
  DFCG_CUDA(cudaMemcpyAsync(h_nrm.data(), nrm.get(), sizeof(double) * cols, cudaMemcpyDeviceToHost, s));
  DFCG_CUDA(cudaStreamSynchronize(s));
  std::vector<int> cperm(cols);
  std::iota(cperm.begin(), cperm.end(), 0);
  std::stable_sort(cperm.begin(), cperm.end(), [&](int a, int b) { return h_nrm[a] > h_nrm[b]; });
  // Callers that keep only the triplets with sigma > u_tau may skip accumulating the rotations:
  // U is then recovered as A V Sigma^-1. Column c carries an error ~ eps (||A|| / sigma_c)^2 +
  // off * ||A|| / sigma_c, so its contribution sigma_c u_c v_c^T is off by < 1e-9 ||A|| when
  // ||A||_F <= 1e7 u_tau. This halves the data every Jacobi round moves (the W pair only).
  double frob2 = 0.0;
  for (double x : h_nrm) frob2 += x * x;
  const bool derive_u = u_tau > 0.0 && std::sqrt(frob2) <= 1e7 * u_tau;
  DBuf<int> dcperm(cols, s);
  DFCG_CUDA(cudaMemcpyAsync(dcperm.get(), cperm.data(), sizeof(int) * cols, cudaMemcpyHostToDevice, s));
  DBuf<double> Qx(rows * cols, s), R(cols * cols, s);
  gather_cols(s, rows, cols, A, lda, dcperm.get(), nullptr, Qx.get(), cols);
  // With U derived from V only R is needed, and one Cholesky of the Gram gives it: no Q, no
  // second CholQR pass. The Cholesky succeeds only for kappa(A) < ~3e5, which bounds the
  // Gram's effect on a kept singular value by eps ||A||^2 / sigma_c < 1e-10 ||A||; otherwise
  // (or when every triplet is needed) the backward-stable CholQR2 / Householder R is used.
  bool have_r = false;
  if (derive_u) {
    DBuf<int> fail(1, s);
    DBuf<double> Rinv(cols * cols, s);
    fail.zero(s);
    gram_upper(s, rows, cols, Qx.get(), cols, R.get(), cols);
    cholesky_inverse(s, cols, R.get(), cols, Rinv.get(), cols, 1e-11, fail.get(), false, false);
    int h_fail = 0;
    DFCG_CUDA(cudaMemcpyAsync(&h_fail, fail.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    DFCG_CUDA(cudaStreamSynchronize(s));
    have_r = h_fail == 0;
  }
  if (!have_r) thin_qr(s, rows, cols, Qx.get(), cols, R.get(), cols);

  // Block width: 8-column blocks (16-column pairs). 16-column blocks halve the rounds per sweep
  // but measured slower on B200 at b ~ 720 (single block: 576 vs 477 ms per 40 iterations; the
  // ~200 KB slab also takes a whole SM, which cost 2x in the concurrent F step), so they are
  // only reachable through DFCG_JACOBI_NB=16 for experiments.
  static const int nb_env = std::getenv("DFCG_JACOBI_NB") ? std::atoi(std::getenv("DFCG_JACOBI_NB")) : 0;
  const int NB = nb_env == 16 ? 16 : 8;
  const int p0 = static_cast<int>((cols + NB - 1) / NB);
  const int p = std::max(2, p0 + (p0 & 1));
  const i64 np = static_cast<i64>(p) * NB;  // padded column count
  const i64 wrows = cols;
  const i64 nj = derive_u ? 0 : np;  // rows of the accumulated rotation J (0: not accumulated)
  DBuf<double> W(wrows * np, s), J(std::max<i64>(nj, 1) * np, s);
  W.zero(s);
  transpose(s, cols, cols, R.get(), cols, W.get(), np);  // W = R^T
  if (nj) set_identity(s, np, np, J.get(), np);
  const std::vector<int> sched = round_robin(p);
  DBuf<int> pairs(static_cast<i64>(sched.size()), s);
  DFCG_CUDA(cudaMemcpyAsync(pairs.get(), sched.data(), sizeof(int) * sched.size(), cudaMemcpyHostToDevice, s));
  DBuf<unsigned long long> off(1, s);
  // Pairs whose cosine exceeds tol = 1e-11 are rotated; the sweeps stop once a whole sweep
  // started with every cosine <= stop_tol = 1e-5. Cyclic Jacobi converges quadratically there
  // (measured on the c2 shapes: a sweep starting at c leaves ~1.3-5 c^2), so that last sweep
  // leaves the columns orthogonal to ~5e-10 (or the rounding floor, ~1e-11 — too close to tol
  // to serve as the stopping test too). 1e-6 cost a ninth sweep in ~40% of the c2 SVDs (the
  // eighth starting at 1-3e-6) for no measurable change in the results.
  const double tol = 1e-11, stop_tol = 1e-5;
  const int npairs = p / 2;
  const int JW = 2 * NB;
  const i64 cap_rows = std::max((wrows + 3) / 4 * 4, (nj + 3) / 4 * 4);
  int dev = 0;
  DFCG_CUDA(cudaGetDevice(&dev));
  // Shared memory per CTA: the slab (cw rows of JW doubles, twice with the V prefetch) plus one
  // JW x JW reduction slot, under the opt-in limit left by the static arrays (the Gram pair and
  // rotation; the cluster variants add the shared partial Gram).
  const size_t static_b = sizeof(double) * (3 * JW * (JW + 1) + 8) + (NB == 8 ? 1024 : 0);
  auto dyn_cap = [&](int cs) {
    return 232448 - static_b - (cs > 1 ? sizeof(double) * JW * JW : 0) - 1024;
  };
  auto dyn_for = [&](i64 cw, int pre) { return sizeof(double) * ((pre ? 2 : 1) * cw * JW + JW * JW); };
  // Cluster size: split each pair's rows over CS CTAs when few solves share the GPU, so a lone
  // block's rounds use more SMs (the concurrent F step keeps CS = 1: same work, fewer CTAs), or
  // when one CTA's shared memory cannot hold a slab.
  static const int cs_env = std::getenv("DFCG_JACOBI_CLUSTER") ? std::atoi(std::getenv("DFCG_JACOBI_CLUSTER")) : 0;
  auto slab = [&](int cs) { return ((cap_rows / 4 + cs - 1) / cs) * 4; };
  int CS = 0;  // 0: streaming (non-resident) round kernel
  for (int c : {1, 2, 4})
    if (dyn_for(slab(c), 0) <= dyn_cap(c)) {
      CS = c;
      break;
    }
  const bool resident = CS > 0;
  if (resident) {
    int nsm = 0;
    DFCG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const i64 slots = 2 * static_cast<i64>(nsm);
    const i64 k = std::max(1, active_streams(dev));
    // 2-CTA clusters when they fit (a lone c2 block: 8.1 ms of Jacobi per iteration against 8.5
    // with 4 and 9.2 with 1, with programmatic dependent launch of the rounds); 4 only when the
    // slab already needed it (the loop above)
    if (CS == 1 && k * npairs * 2 <= slots && wrows >= 128 && dyn_for(slab(2), 0) <= dyn_cap(2)) CS = 2;
    if (cs_env == 1 || cs_env == 2 || cs_env == 4)
      if (dyn_for(slab(cs_env), 0) <= dyn_cap(cs_env)) CS = cs_env;
  }
  if (!resident && NB != 8) throw std::runtime_error("thin_svd: no resident Jacobi configuration");
  const i64 cw = resident ? slab(CS) : cap_rows;  // rows per CTA (slab)
  const int prefetch_v = resident && nj > 0 && dyn_for(cw, 1) <= dyn_cap(CS) ? 1 : 0;  // W and V slabs both fit
  const size_t smem = dyn_for(cw, prefetch_v);
  if (resident) {
    static std::atomic<std::uint64_t> configured{0};
    if (!(configured.load() & dev_bit(dev))) {
      auto opt_in = [&](const void* fn, size_t b) {
        DFCG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(b)));
      };
      const size_t s8 = 232448 - sizeof(double) * (3 * 16 * 17 + 8) - 1024 - 1024;
      const size_t s16 = 232448 - sizeof(double) * (3 * 32 * 33 + 8) - 1024;
      opt_in(reinterpret_cast<const void*>(jacobi_round_resident_kernel<8, 1>), s8);
      opt_in(reinterpret_cast<const void*>(jacobi_round_resident_kernel<8, 2>), s8 - 2048);
      opt_in(reinterpret_cast<const void*>(jacobi_round_resident_kernel<8, 4>), s8 - 2048);
      opt_in(reinterpret_cast<const void*>(jacobi_round_resident_kernel<16, 1>), s16);
      opt_in(reinterpret_cast<const void*>(jacobi_round_resident_kernel<16, 2>), s16 - 8192);
      opt_in(reinterpret_cast<const void*>(jacobi_round_resident_kernel<16, 4>), s16 - 8192);
      configured.fetch_or(dev_bit(dev));
    }
  }
  // Optional (DFCG_JACOBI_GRAPH=1): the p - 1 round launches of a sweep, identical from sweep
  // to sweep, captured once into a CUDA graph and replayed per sweep — measured 9.7 -> 8.4 ms of
  // Jacobi per c2 iteration for a lone block, but slower whenever several solves share the GPU
  // (92 vs 109 block-it/s with eight; 65 when selected per call by the number of active solves,
  // the instantiations of the per-thread graphs landing in the timed window), so the rounds are
  // launched directly by default.
  // Graph cache (per host thread): one captured sweep per shape class (device, block width,
  // cluster size, pair count, V prefetch, shared-memory bucket), with its own argument block
  // and off-diagonal accumulator at fixed addresses. The shared memory is bucketed to 64-row
  // slabs so consecutive SVDs of slowly varying width share a graph.
  static const int graph_env = std::getenv("DFCG_JACOBI_GRAPH") ? std::atoi(std::getenv("DFCG_JACOBI_GRAPH")) : -1;
  const bool use_graph = graph_env == 1;
  struct SweepGraph {
    int dev, nb, cs, npairs, pre;
    size_t smem;
    cudaGraphExec_t exec;
    JacobiArgs* d_args;
    unsigned long long* d_off;
  };
  thread_local std::vector<SweepGraph> graphs;
  const bool small_svd = cols <= kSmallN && wrows <= kSmallN && nj <= kSmallN;
  size_t smem_launch = smem;
  SweepGraph* sg = nullptr;
  bool capture = false;
  if (resident && !small_svd && use_graph) {
    const i64 cw_b = (cw + 63) / 64 * 64;
    if (dyn_for(cw_b, prefetch_v) <= dyn_cap(CS)) smem_launch = dyn_for(cw_b, prefetch_v);
    for (SweepGraph& g : graphs)
      if (g.dev == dev && g.nb == NB && g.cs == CS && g.npairs == npairs && g.pre == prefetch_v && g.smem == smem_launch)
        sg = &g;
    if (!sg && graphs.size() < 64) {
      graphs.push_back(SweepGraph{dev, NB, CS, npairs, prefetch_v, smem_launch, nullptr, nullptr, nullptr});
      sg = &graphs.back();
      DFCG_CUDA(cudaMalloc(reinterpret_cast<void**>(&sg->d_args), sizeof(JacobiArgs)));
      DFCG_CUDA(cudaMalloc(reinterpret_cast<void**>(&sg->d_off), sizeof(unsigned long long)));
      capture = true;
    }
  }
  // this SVD's argument block: the cached graph's, or a stream-ordered one
  DBuf<JacobiArgs> own_args;
  JacobiArgs* d_args = sg ? sg->d_args : nullptr;
  unsigned long long* d_off = sg ? sg->d_off : off.get();
  if (!sg) {
    own_args.alloc(1, s);
    d_args = own_args.get();
  }
  const JacobiArgs h_args{wrows, nj, np, np, W.get(), J.get(), d_off, tol, p, prefetch_v};
  DFCG_CUDA(cudaMemcpyAsync(d_args, &h_args, sizeof(JacobiArgs), cudaMemcpyHostToDevice, s));
  static const int pdl_env = std::getenv("DFCG_JACOBI_PDL") ? std::atoi(std::getenv("DFCG_JACOBI_PDL")) : 1;
  const bool use_pdl = pdl_env == 1;
  auto launch_round = [&](int r) {
    const int inner = r == 0 ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(npairs * CS));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem_launch;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (CS > 1) {
      attr[na].id = cudaLaunchAttributeClusterDimension;
      attr[na].val.clusterDim.x = static_cast<unsigned>(CS);
      attr[na].val.clusterDim.y = 1;
      attr[na].val.clusterDim.z = 1;
      ++na;
    }
    if (use_pdl && r > 0) {  // round r overlaps its launch with round r - 1 (griddepcontrol in the kernel)
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    const JacobiArgs* ap = d_args;
#define DFCG_JROUND(nb, cs) DFCG_CUDA(cudaLaunchKernelEx(&cfg, jacobi_round_resident_kernel<nb, cs>, ap, r, inner))
    if (NB == 8) {
      if (CS == 1) DFCG_JROUND(8, 1);
      else if (CS == 2) DFCG_JROUND(8, 2);
      else DFCG_JROUND(8, 4);
    } else {
      if (CS == 1) DFCG_JROUND(16, 1);
      else if (CS == 2) DFCG_JROUND(16, 2);
      else DFCG_JROUND(16, 4);
    }
#undef DFCG_JROUND
  };
  static const bool trace_svd = std::getenv("DFCG_TRACE_SVD") != nullptr;
  const bool small = cols <= kSmallN && wrows <= kSmallN && nj <= kSmallN;
  if (small) {  // one launch, convergence on the device
    DBuf<int> nsw(1, s);
    {
      prof::Scope scope(prof::kJacobi, s, 8.0 * 6.0 * cols * cols * (wrows + nj), 8.0 * 16.0 * cols * (wrows + nj));
      constexpr size_t kOne = sizeof(double) * kSmallN * (kSmallN + 1);
      static std::atomic<std::uint64_t> configured{0};
      int dev = 0;
      DFCG_CUDA(cudaGetDevice(&dev));
      if (!(configured.load() & dev_bit(dev))) {
        DFCG_CUDA(cudaFuncSetAttribute(jacobi_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(2 * kOne)));
        configured.fetch_or(dev_bit(dev));
      }
      jacobi_small_kernel<<<1, 256, (nj > 0 ? 2 : 1) * kOne, s>>>(static_cast<int>(wrows), static_cast<int>(cols),
                                                                  static_cast<int>(nj), W.get(), np, J.get(), np, tol,
                                                                  stop_tol, 60, off.get(), nsw.get());
      DFCG_LAUNCH_CHECK();
    }
    if (trace_svd) {
      int h = 0;
      unsigned long long ho = 0;
      DFCG_CUDA(cudaMemcpyAsync(&h, nsw.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
      DFCG_CUDA(cudaMemcpyAsync(&ho, off.get(), sizeof(ho), cudaMemcpyDeviceToHost, s));
      DFCG_CUDA(cudaStreamSynchronize(s));
      double ov;
      std::memcpy(&ov, &ho, sizeof(double));
      std::fprintf(stderr, "[svd] %lldx%lld small kernel: %d sweeps, converged flag %.0e\n", (long long)rows,
                   (long long)cols, h, ov);
    }
  }
  if (capture) {
    DFCG_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    DFCG_CUDA(cudaMemsetAsync(sg->d_off, 0, sizeof(unsigned long long), s));
    for (int r = 0; r < p - 1; ++r) launch_round(r);
    cudaGraph_t graph = nullptr;
    DFCG_CUDA(cudaStreamEndCapture(s, &graph));
    DFCG_CUDA(cudaGraphInstantiate(&sg->exec, graph, 0));
    DFCG_CUDA(cudaGraphDestroy(graph));
  }
  cudaGraphExec_t sweep_exec = sg ? sg->exec : nullptr;
  // Persistent sweeps (jacobi_sweeps_kernel): one cooperative launch per SVD, stop test on the
  // device. DFCG_JACOBI_PERSIST=0 keeps the launch-per-round path, 1 always persists, 2 (default)
  // persists while at most two solves share the GPU (the latency-bound lone-block regime).
  static const int persist_env =
      std::getenv("DFCG_JACOBI_PERSIST") ? std::atoi(std::getenv("DFCG_JACOBI_PERSIST")) : 2;
  bool persist = resident && !small && !sweep_exec &&
                 (persist_env == 1 || (persist_env == 2 && active_streams(dev) <= 2));
  if (persist) {
    auto fn = [&]() -> const void* {
      if (NB == 8) {
        if (CS == 1) return reinterpret_cast<const void*>(jacobi_sweeps_kernel<8, 1>);
        if (CS == 2) return reinterpret_cast<const void*>(jacobi_sweeps_kernel<8, 2>);
        return reinterpret_cast<const void*>(jacobi_sweeps_kernel<8, 4>);
      }
      if (CS == 1) return reinterpret_cast<const void*>(jacobi_sweeps_kernel<16, 1>);
      if (CS == 2) return reinterpret_cast<const void*>(jacobi_sweeps_kernel<16, 2>);
      return reinterpret_cast<const void*>(jacobi_sweeps_kernel<16, 4>);
    }();
    static std::mutex mu;
    // (kernel, device, dynamic shared memory) -> CTAs that can be co-resident on the whole GPU.
    // With clusters the bound is cudaOccupancyMaxActiveClusters x CS (cluster placement within
    // GPCs leaves it below SMs x CTAs per SM: the full-matrix base APG's 187-pair SVD passed
    // the per-SM bound at CS = 2 and the cooperative launch was refused).
    static std::map<std::tuple<const void*, int, size_t>, i64> occ_cache;
    i64 co_resident = 0;
    {
      std::lock_guard<std::mutex> lock(mu);
      const auto key = std::make_tuple(fn, dev, smem);
      auto it = occ_cache.find(key);
      if (it == occ_cache.end()) {
        const size_t cap = dyn_cap(CS);
        DFCG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cap)));
        int occ = 0, nsm = 0;
        DFCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, smem));
        DFCG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        co_resident = static_cast<i64>(occ) * nsm;
        if (CS > 1) {
          cudaLaunchConfig_t qc = {};
          qc.gridDim = dim3(static_cast<unsigned>(CS) * 1024u);
          qc.blockDim = dim3(256);
          qc.dynamicSmemBytes = smem;
          cudaLaunchAttribute qa[1];
          qa[0].id = cudaLaunchAttributeClusterDimension;
          qa[0].val.clusterDim.x = static_cast<unsigned>(CS);
          qa[0].val.clusterDim.y = 1;
          qa[0].val.clusterDim.z = 1;
          qc.attrs = qa;
          qc.numAttrs = 1;
          int ncl = 0;
          DFCG_CUDA(cudaOccupancyMaxActiveClusters(&ncl, fn, &qc));
          co_resident = std::min<i64>(co_resident, static_cast<i64>(ncl) * CS);
        }
        occ_cache[key] = co_resident;
      } else {
        co_resident = it->second;
      }
    }
    persist = static_cast<i64>(npairs) * CS <= co_resident;
    if (persist) {
      DBuf<unsigned long long> offs(3, s);
      DBuf<int> nsw(1, s);
      offs.zero(s);
      // DFCG_JACOBI_P2P=1: point-to-point round ordering (block version counters) instead of a
      // grid barrier per round. Measured level with the barriers (8.47 vs 8.43 ms of Jacobi per
      // lone c2 iteration, profiles/r02_lone_jacobi_p2p.txt): the round's own serial chain, not
      // the barrier, is what a sweep waits for. Opt-in.
      static const int p2p_env = std::getenv("DFCG_JACOBI_P2P") ? std::atoi(std::getenv("DFCG_JACOBI_P2P")) : 0;
      DBuf<unsigned> vers;
      if (p2p_env != 0) {
        vers.alloc(p, s);
        vers.zero(s);
      }
      unsigned* verp = p2p_env != 0 ? vers.get() : nullptr;
      const JacobiArgs pa{wrows, nj, np, np, W.get(), J.get(), offs.get(), tol, p, prefetch_v};
      DFCG_CUDA(cudaMemcpyAsync(d_args, &pa, sizeof(JacobiArgs), cudaMemcpyHostToDevice, s));
      const double per_sweep_flops = (p - 1.0) * npairs * (2.0 * wrows + 2.0 * (wrows + nj)) * JW * JW;
      const double per_sweep_bytes = (p - 1.0) * npairs * 16.0 * (wrows + nj) * JW;
      int h_sweeps = 0;
      {
        prof::Scope scope(prof::kJacobi, s, 0.0, 0.0, 0);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(npairs * CS));
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[2];
        int na = 0;
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na].val.cooperative = 1;
        ++na;
        if (CS > 1) {
          attr[na].id = cudaLaunchAttributeClusterDimension;
          attr[na].val.clusterDim.x = static_cast<unsigned>(CS);
          attr[na].val.clusterDim.y = 1;
          attr[na].val.clusterDim.z = 1;
          ++na;
        }
        cfg.attrs = attr;
        cfg.numAttrs = na;
        const JacobiArgs* ap = d_args;
        const double stol = stop_tol;
        const int maxsw = 60;
        int* so = nsw.get();
        cudaError_t lerr = cudaSuccess;
#define DFCG_JSWEEPS(nb, cs) lerr = cudaLaunchKernelEx(&cfg, jacobi_sweeps_kernel<nb, cs>, ap, stol, maxsw, so, verp)
        if (NB == 8) {
          if (CS == 1) DFCG_JSWEEPS(8, 1);
          else if (CS == 2) DFCG_JSWEEPS(8, 2);
          else DFCG_JSWEEPS(8, 4);
        } else {
          if (CS == 1) DFCG_JSWEEPS(16, 1);
          else if (CS == 2) DFCG_JSWEEPS(16, 2);
          else DFCG_JSWEEPS(16, 4);
        }
#undef DFCG_JSWEEPS
        if (lerr == cudaErrorCooperativeLaunchTooLarge) {
          // the occupancy query overestimated (e.g. another context's carve-out): nothing was
          // launched; fall back to one launch per round below
          (void)cudaGetLastError();
          persist = false;
        } else {
          DFCG_CUDA(lerr);
          DFCG_LAUNCH_CHECK();
          DFCG_CUDA(cudaMemcpyAsync(&h_sweeps, so, sizeof(int), cudaMemcpyDeviceToHost, s));
          DFCG_CUDA(cudaStreamSynchronize(s));
          scope.add_work(h_sweeps * per_sweep_flops, h_sweeps * per_sweep_bytes, 1);
        }
      }
      if (trace_svd && persist)
        std::fprintf(stderr, "[svd] %lldx%lld persistent: %d sweeps (CS %d)\n", (long long)rows, (long long)cols,
                     h_sweeps, CS);
    }
  }
  for (int sweep = 0; sweep < 60 && !small && !persist; ++sweep) {
    if (sweep_exec) {
      prof::Scope scope(prof::kJacobi, s, (p - 1.0) * npairs * (2.0 * wrows + 2.0 * (wrows + nj)) * JW * JW,
                        (p - 1.0) * npairs * 16.0 * (wrows + nj) * JW, p - 1);
      DFCG_CUDA(cudaGraphLaunch(sweep_exec, s));
      prof::count_launch(p - 1);
    } else {
      off.zero(s);
      // one event pair per sweep, counted as p - 1 round launches (algorithmic per round: Gram +
      // rotation of each pair's columns, every W / V element read and written once)
      prof::Scope scope(prof::kJacobi, s, (p - 1.0) * npairs * (2.0 * wrows + 2.0 * (wrows + nj)) * JW * JW,
                        (p - 1.0) * npairs * 16.0 * (wrows + nj) * JW, p - 1);
      for (int r = 0; r < p - 1; ++r) {
        const int* pr = pairs.get() + 2 * static_cast<i64>(r) * npairs;
        if (resident)
          launch_round(r);
        else
          jacobi_round_kernel<8><<<npairs, 16 * 8, 0, s>>>(wrows, nj, W.get(), np, J.get(), np, pr, tol, off.get(), 2);
        DFCG_LAUNCH_CHECK();
      }
    }
    unsigned long long h_off = 0;
    DFCG_CUDA(cudaMemcpyAsync(&h_off, d_off, sizeof(h_off), cudaMemcpyDeviceToHost, s));
    DFCG_CUDA(cudaStreamSynchronize(s));
    double offv;
    std::memcpy(&offv, &h_off, sizeof(double));
    if (trace_svd)
      std::fprintf(stderr, "[svd] %lldx%lld sweep %d off %.3e\n", (long long)rows, (long long)cols, sweep, offv);
    if (offv <= stop_tol) break;
  }
  // singular values = column norms of W; sort descending (stable by index)
  DBuf<double> sig(np, s);
  col_norms(s, wrows, np, W.get(), np, sig.get());
  std::vector<double> h_sig(np);
  DFCG_CUDA(cudaMemcpyAsync(h_sig.data(), sig.get(), sizeof(double) * np, cudaMemcpyDeviceToHost, s));
  DFCG_CUDA(cudaStreamSynchronize(s));
  std::vector<int> all(np);
  std::iota(all.begin(), all.end(), 0);
  std::stable_sort(all.begin(), all.end(), [&](int a, int b) { return h_sig[a] > h_sig[b]; });
  std::vector<int> perm(cols);
  for (i64 c = 0; c < cols; ++c) {
    perm[c] = all[c];
    s_host[c] = h_sig[all[c]];
  }
  DBuf<int> dperm(cols, s);
  DBuf<double> dsig(cols, s);
  DFCG_CUDA(cudaMemcpyAsync(dperm.get(), perm.data(), sizeof(int) * cols, cudaMemcpyHostToDevice, s));
  DFCG_CUDA(cudaMemcpyAsync(dsig.get(), s_host.data(), sizeof(double) * cols, cudaMemcpyHostToDevice, s));
  if (!derive_u) {  // U = Q J[:, perm]
    DBuf<double> Js(cols * cols, s);
    gather_cols(s, cols, cols, J.get(), np, dperm.get(), nullptr, Js.get(), cols);
    gemm(s, false, false, rows, cols, cols, 1.0, Qx.get(), cols, Js.get(), cols, 0.0, U, ldu);
  }
  // V = P (W[:, perm] / sigma): row j of the normalised W goes to row cperm[j]
  DBuf<double> Wn(cols * cols, s);
  scale_cols_kernel<<<grid_for(cols * cols), 256, 0, s>>>(cols, cols, W.get(), np, dsig.get(), cols, Wn.get(),
                                                          dperm.get());
  DFCG_LAUNCH_CHECK();
  scatter_rows_int_kernel<<<grid_for(cols * cols), 256, 0, s>>>(cols, cols, Wn.get(), cols, dcperm.get(), V, ldv);
  DFCG_LAUNCH_CHECK();
  if (derive_u) {  // U = A V Sigma^-1 (A is intact: the QR ran on a permuted copy)
    gemm(s, false, false, rows, cols, cols, 1.0, A, lda, V, ldv, 0.0, U, ldu);
    div_cols_kernel<<<grid_for(rows * cols), 256, 0, s>>>(rows, cols, U, ldu, dsig.get());
    DFCG_LAUNCH_CHECK();
  }
  DFCG_CUDA(cudaStreamSynchronize(s));  // host vectors (perm, s_host, cperm) used by async copies
}

// Exported for the dfcg_bench_cholesky diagnostic (the internal entry lives in the anonymous
// namespace above).
void cholesky_inverse_public(cudaStream_t s, i64 n, double* G, i64 ldg, double* Rinv, i64 ldr, double rel_tol,
                             int* fail, bool want_inverse, bool scale) {
  cholesky_inverse(s, n, G, ldg, Rinv, ldr, rel_tol, fail, want_inverse, scale);
}

}  // namespace dfcg
