// Dense FP64 building blocks: DMMA GEMM (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4; FP64 has
// no tcgen05 kind on sm_100a), copies/transposes, deterministic reductions.
//
// GEMM tiling: CTA 64x64, BK=16, 4 warps (2x2) of 32x32, 3-stage cp.async pipeline (see the
// tile policy above launch_gemm).
// Shared-memory tiles are stored in the global layout's contiguous order and padded so
// every DMMA fragment load is a 2-wavefront (conflict-free for 8-byte lanes) access.
#include "common.cuh"

#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

namespace dfcg {

namespace {

constexpr int BK = 16, STAGES = 3;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Shared-memory operand tile of ROWS (M or N index) x BK (k).
//   KMajor == false: [rows][k] with k contiguous, row stride BK + 4
//   KMajor == true : [k][rows] with rows contiguous, k stride ROWS + 4
// Both paddings make every DMMA fragment load a 2-wavefront (conflict-free) access and keep
// even positions 16-byte aligned. (An unpadded XOR-swizzled layout measured 4-20% slower.)
// VEC: 16-byte cp.async (even leading dimension, 16-byte aligned base; a pair straddling the
// matrix edge copies 8 bytes and zero-fills the rest), else 8-byte cp.async.
template <bool KMajor, int ROWS>
struct Tile {
  static constexpr int PAD_K = BK + 4, PAD_R = ROWS + 4;
  static constexpr int elems = KMajor ? BK * PAD_R : ROWS * PAD_K;
  __device__ __forceinline__ static int pos(int r, int k) { return KMajor ? k * PAD_R + r : r * PAD_K + k; }
  template <int THREADS, bool VEC>
  __device__ __forceinline__ static void load(double* sm, const double* g, i64 ld, i64 r0, i64 k0, i64 R, i64 Kend,
                                              int tid) {
    if (VEC) {
#pragma unroll
      for (int it = 0; it < (ROWS * BK) / (2 * THREADS); ++it) {
        const int e = tid + it * THREADS;
        int r, k;
        i64 rem;
        const double* src;
        if (!KMajor) {
          r = e / (BK / 2);
          k = 2 * (e % (BK / 2));
          const i64 gr = r0 + r, gk = k0 + k;
          rem = gr < R ? Kend - gk : 0;
          src = rem > 0 ? g + gr * ld + gk : g;
        } else {
          k = e / (ROWS / 2);
          r = 2 * (e % (ROWS / 2));
          const i64 gr = r0 + r, gk = k0 + k;
          rem = gk < Kend ? R - gr : 0;
          src = rem > 0 ? g + gk * ld + gr : g;
        }
        const int bytes = rem >= 2 ? 16 : (rem == 1 ? 8 : 0);
        const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(sm + pos(r, k)));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(src), "r"(bytes));
      }
    } else {
#pragma unroll
      for (int it = 0; it < (ROWS * BK) / THREADS; ++it) {
        const int e = tid + it * THREADS;
        if (!KMajor) {
          const int r = e / BK, k = e % BK;
          const i64 gr = r0 + r, gk = k0 + k;
          const bool ok = gr < R && gk < Kend;
          cp_async8(sm + pos(r, k), ok ? g + gr * ld + gk : g, ok);
        } else {
          const int k = e / ROWS, r = e % ROWS;
          const i64 gr = r0 + r, gk = k0 + k;
          const bool ok = gr < R && gk < Kend;
          cp_async8(sm + pos(r, k), ok ? g + gk * ld + gr : g, ok);
        }
      }
    }
  }
  __device__ __forceinline__ static double frag(const double* sm, int r, int k) { return sm[pos(r, k)]; }
};

// C tile BM x BN per CTA; warps in a (BM/WM) x (BN/WN) grid, each computing WM x WN with
// (WM/8) x (WN/8) DMMA 8x8 accumulators.
// A tile: !TA -> A(i,k) at A[i*lda+k] -> [rows][k]; TA -> A(i,k) at A[k*lda+i] -> [k][rows].
// B tile: !TB -> B(k,j) at B[k*ldb+j] -> [k][rows]; TB -> B(k,j) at B[j*ldb+k] -> [rows][k].
template <bool TA, bool TB, int BM, int BN, int WM, int WN, bool VEC>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32)
    gemm_kernel(i64 M, i64 N, i64 K, i64 kchunk, double alpha, const double* __restrict__ A, i64 lda,
                const double* __restrict__ B, i64 ldb, double beta, double* __restrict__ C, i64 ldc,
                double* __restrict__ ws, int upper_only) {
  constexpr int THREADS = (BM / WM) * (BN / WN) * 32, FM = WM / 8, FN = WN / 8;
  using TileA = Tile<TA, BM>;
  using TileB = Tile<!TB, BN>;
  extern __shared__ double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * TileA::elems;

  pdl_wait();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp / (BN / WN)) * WM, wn = (warp % (BN / WN)) * WN;
  const i64 m0 = static_cast<i64>(blockIdx.y) * BM, n0 = static_cast<i64>(blockIdx.x) * BN;
  // flags & 1 (SYRK-style): tiles strictly below the diagonal are skipped (C left as is).
  // flags & 2 (B upper triangular, TRMM-style): B(k, j) = 0 for k > j, so the K loop of this
  // column tile stops at n0 + BN.
  // flags & 4 (op(A) upper triangular): op(A)(i, k) = 0 for k < i, the K loop of this row tile
  // starts at m0; flags & 8 (op(A) lower triangular): it stops at m0 + BM.
  if ((upper_only & 1) && m0 >= n0 + BN) return;
  i64 kbeg = static_cast<i64>(blockIdx.z) * kchunk;
  i64 kend = min(K, kbeg + kchunk);
  if (upper_only & 2) kend = min(kend, n0 + BN);
  if (upper_only & 4) kbeg = max(kbeg, m0);
  if (upper_only & 8) kend = min(kend, m0 + BM);
  const int ntiles = kend > kbeg ? static_cast<int>((kend - kbeg + BK - 1) / BK) : 0;

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < ntiles) {
      TileA::template load<THREADS, VEC>(sA + st * TileA::elems, A, lda, m0, kbeg + st * BK, M, kend, tid);
      TileB::template load<THREADS, VEC>(sB + st * TileB::elems, B, ldb, n0, kbeg + st * BK, N, kend, tid);
    }
    cp_async_commit();
  }
  pdl_trigger();

  const int fr = lane >> 2, fk = lane & 3;
  for (int t = 0; t < ntiles; ++t) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nt = t + STAGES - 1;
      if (nt < ntiles) {
        const int st = nt % STAGES;
        TileA::template load<THREADS, VEC>(sA + st * TileA::elems, A, lda, m0, kbeg + static_cast<i64>(nt) * BK, M,
                                      kend, tid);
        TileB::template load<THREADS, VEC>(sB + st * TileB::elems, B, ldb, n0, kbeg + static_cast<i64>(nt) * BK, N,
                                      kend, tid);
      }
      cp_async_commit();
    }
    const double* a = sA + (t % STAGES) * TileA::elems;
    const double* b = sB + (t % STAGES) * TileB::elems;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[FM], bf[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = TileA::frag(a, wm + i * 8 + fr, kk + fk);
#pragma unroll
      for (int j = 0; j < FN; ++j) bf[j] = TileB::frag(b, wn + j * 8 + fr, kk + fk);
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // Epilogue: lane holds C(row = lane/4, col = 2*(lane%4) + {0,1}) of each 8x8 tile.
  const int er = lane >> 2, ec = (lane & 3) * 2;
#pragma unroll
  for (int i = 0; i < FM; ++i) {
#pragma unroll
    for (int j = 0; j < FN; ++j) {
      const i64 row = m0 + wm + i * 8 + er;
      if (row >= M) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const i64 col = n0 + wn + j * 8 + ec + h;
        if (col >= N) continue;
        if (ws) {
          ws[(static_cast<i64>(blockIdx.z) * M + row) * N + col] = acc[i][j][h];
        } else {
          double v = alpha * acc[i][j][h];
          if (beta != 0.0) v += beta * C[row * ldc + col];
          C[row * ldc + col] = v;
        }
      }
    }
  }
}

__global__ void splitk_reduce(i64 M, i64 N, int splits, const double* __restrict__ ws, double alpha, double beta,
                              double* __restrict__ C, i64 ldc) {
  pdl_wait();
  pdl_trigger();
  const i64 total = M * N;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += ws[z * total + e];
    const i64 row = e / N, col = e % N;
    double v = alpha * s;
    if (beta != 0.0) v += beta * C[row * ldc + col];
    C[row * ldc + col] = v;
  }
}

__global__ void scale_kernel(i64 M, i64 N, double beta, double* C, i64 ldc) {
  const i64 total = M * N;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 row = e / N, col = e % N;
    C[row * ldc + col] = beta == 0.0 ? 0.0 : beta * C[row * ldc + col];
  }
}

int g_num_sms = 0;

}  // namespace

// On when at most two solves share the device (latency mode: a lone block per GPU, the two
// DFC-Nys subproblems): measured 24.3 -> 23.2 ms per lone c2 iteration, but 128.6 -> 120.2
// block-it/s with eight concurrent solves (dependent CTAs waiting at griddepcontrol.wait hold SM
// slots other streams would use). DFCG_PDL=0 / 2 forces off / on.
bool pdl_enabled() {
  static const int env = std::getenv("DFCG_PDL") ? std::atoi(std::getenv("DFCG_PDL")) : 1;
  if (env == 0) return false;
  if (env == 2) return true;
  int dev = 0;
  cudaGetDevice(&dev);
  return active_streams(dev) <= 2;
}

namespace {

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

// CTAs of one GEMM configuration resident per SM (configures the shared-memory opt-in of both
// load variants once).
template <bool TA, bool TB, int BM, int BN, int WM, int WN>
int gemm_resident() {
  constexpr int THREADS = (BM / WM) * (BN / WN) * 32;
  const size_t smem = sizeof(double) * STAGES * (Tile<TA, BM>::elems + Tile<!TB, BN>::elems);
  static std::atomic<std::uint64_t> configured{0};  // one bit per device
  static int resident = 0;
  int dev = 0;
  DFCG_CUDA(cudaGetDevice(&dev));
  if (!(configured.load() & dev_bit(dev))) {
    DFCG_CUDA(cudaFuncSetAttribute(gemm_kernel<TA, TB, BM, BN, WM, WN, false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    DFCG_CUDA(cudaFuncSetAttribute(gemm_kernel<TA, TB, BM, BN, WM, WN, true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int r0 = 0, r1 = 0;
    DFCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r0, gemm_kernel<TA, TB, BM, BN, WM, WN, false>, THREADS,
                                                            smem));
    DFCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r1, gemm_kernel<TA, TB, BM, BN, WM, WN, true>, THREADS,
                                                            smem));
    resident = std::max(1, std::min(r0, r1));
    configured.fetch_or(dev_bit(dev));
  }
  return resident;
}

template <bool TA, bool TB, int BM, int BN, int WM, int WN>
void launch_gemm_cfg(cudaStream_t s, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda, const double* B,
                     i64 ldb, double beta, double* C, i64 ldc, int upper_only) {
  constexpr int THREADS = (BM / WM) * (BN / WN) * 32;
  const size_t smem = sizeof(double) * STAGES * (Tile<TA, BM>::elems + Tile<!TB, BN>::elems);
  const int resident = gemm_resident<TA, TB, BM, BN, WM, WN>();
  const int gx = cdiv(N, BN), gy = cdiv(M, BM);
  const i64 tiles = (upper_only & 1) ? static_cast<i64>(gx) * (gx + 1) / 2 : static_cast<i64>(gx) * gy;
  // Split K when the tiles alone do not fill the resident slots: among the admissible split
  // counts, take the one whose CTA count best fills whole waves (ties and a 1%
  // per-split workspace cost favour fewer splits).
  const i64 slots = static_cast<i64>(resident) * num_sms();
  int splits = 1;
  if (tiles < slots && K > 4 * BK) {
    // >= 128 k per CTA, <= 128 splits, workspace <= 16 Mi doubles
    const int smax = static_cast<int>(std::max<i64>(1, std::min<i64>({128, K / 128, (i64{1} << 24) / (M * N)})));
    double best = -1.0;
    for (int sp = 1; sp <= smax; ++sp) {
      const double w = static_cast<double>(tiles) * sp / slots;
      const double fill = w >= 1.0 ? w / std::ceil(w) : w;
      const double sc = fill * (1.0 - 0.01 * (sp - 1));
      if (sc > best + 1e-9) {
        best = sc;
        splits = sp;
      }
    }
  }
  i64 kchunk = (K + splits - 1) / splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  splits = static_cast<int>((K + kchunk - 1) / kchunk);
  // 16-byte operand loads when both operands allow them
  const bool vec = lda % 2 == 0 && ldb % 2 == 0 && reinterpret_cast<std::uintptr_t>(A) % 16 == 0 &&
                   reinterpret_cast<std::uintptr_t>(B) % 16 == 0;
  auto run = [&](dim3 grid, i64 kc, double* ws) {
    if (vec)
      pdl_launch(gemm_kernel<TA, TB, BM, BN, WM, WN, true>, grid, dim3(THREADS), smem, s, M, N, K, kc, alpha, A, lda, B,
                 ldb, beta, C, ldc, ws, upper_only);
    else
      pdl_launch(gemm_kernel<TA, TB, BM, BN, WM, WN, false>, grid, dim3(THREADS), smem, s, M, N, K, kc, alpha, A, lda,
                 B, ldb, beta, C, ldc, ws, upper_only);
    DFCG_LAUNCH_CHECK();
  };
  if (splits <= 1) {
    run(dim3(gx, gy, 1), std::max<i64>(K, 1), nullptr);
    return;
  }
  DBuf<double> ws(static_cast<i64>(splits) * M * N, s);
  if (upper_only & 1) ws.zero(s);  // skipped tiles leave their partials unwritten
  run(dim3(gx, gy, splits), kchunk, ws.get());
  const int rb = static_cast<int>(std::min<i64>((M * N + 255) / 256, 4L * num_sms()));
  pdl_launch(splitk_reduce, dim3(rb), dim3(256), 0, s, M, N, splits, ws.get(), alpha, beta, C, ldc);
  DFCG_LAUNCH_CHECK();
}

// Tile policy (measured on B200 with tools/gemm_bench against cuBLAS, profiles/r01_gemm_*):
// DMMA throughput needs many resident warps more than large warp tiles — 64x64 CTAs of four
// 32x32 warps (127 registers, 4 CTAs / 16 warps per SM) beat 128x128 CTAs of 64x32 warps
// (225 registers, one CTA per SM) by ~25% on the APG shapes (profiles/r01_gemm_variants_*);
// tile width and split-K count are
// chosen to fill whole waves of resident CTAs. DFCG_GEMM_VARIANT=4|7 forces 64x64|64x48.
template <bool TA, bool TB>
void launch_gemm(cudaStream_t s, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda, const double* B,
                 i64 ldb, double beta, double* C, i64 ldc, int upper_only) {
  static const int variant = std::getenv("DFCG_GEMM_VARIANT") ? std::atoi(std::getenv("DFCG_GEMM_VARIANT")) : 0;
#define DFCG_GEMM_CFG(bm, bn, wm, wn) \
  launch_gemm_cfg<TA, TB, bm, bn, wm, wn>(s, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, upper_only)
  switch (variant) {
    case 4: DFCG_GEMM_CFG(64, 64, 32, 32); return;
    case 7: DFCG_GEMM_CFG(64, 48, 32, 24); return;
    default: break;
  }
  // 64x64 or 64x48 tiles, whichever wastes less of the last wave and of the ragged last tile
  // column (N = 720 = 15 x 48: 64-wide tiles leave the 12th column 75% empty).
  auto score = [&](int bm, int bn, int resident) {
    const double tm = cdiv(M, bm), tn = cdiv(N, bn);
    const double area = static_cast<double>(M) * N / (tm * bm * tn * bn);
    const double tiles = (upper_only & 1) ? tn * (tn + 1) / 2 : tm * tn;
    const double slots = static_cast<double>(resident) * num_sms();
    const double waves = tiles / slots;
    return area * (waves >= 1.0 ? waves / std::ceil(waves) : 1.0);
  };
  const double s64 = score(64, 64, gemm_resident<TA, TB, 64, 64, 32, 32>());
  const double s48 = score(64, 48, gemm_resident<TA, TB, 64, 48, 32, 24>());
  if (!(upper_only & 1) && s48 > 1.02 * s64) DFCG_GEMM_CFG(64, 48, 32, 24);
  else DFCG_GEMM_CFG(64, 64, 32, 32);
#undef DFCG_GEMM_CFG
}

// ---------------------------------------------------------------- small kernels
__global__ void copy2d_kernel(i64 rows, i64 cols, const double* __restrict__ src, i64 lds, double* __restrict__ dst,
                              i64 ldd, double alpha) {
  const i64 total = rows * cols;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 r = e / cols, c = e % cols;
    dst[r * ldd + c] = alpha == 1.0 ? src[r * lds + c] : alpha * src[r * lds + c];
  }
}

__global__ void transpose_kernel(i64 rows, i64 cols, const double* __restrict__ src, i64 lds,
                                 double* __restrict__ dst, i64 ldd) {
  __shared__ double tile[32][33];
  const i64 r0 = static_cast<i64>(blockIdx.y) * 32, c0 = static_cast<i64>(blockIdx.x) * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const i64 r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = src[r * lds + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const i64 c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[c * ldd + r] = tile[threadIdx.x][i];
  }
}

__global__ void identity_kernel(i64 rows, i64 cols, double* dst, i64 ldd) {
  const i64 total = rows * cols;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 r = e / cols, c = e % cols;
    dst[r * ldd + c] = r == c ? 1.0 : 0.0;
  }
}

// Deterministic two-level reduction: fixed grid of 256 blocks writing partials, then
// one block summing them in index order.
constexpr int RED_BLOCKS = 256, RED_THREADS = 256;

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  v = (threadIdx.x < nw) ? sh[threadIdx.x] : 0.0;
  if (w == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;  // valid in thread 0
}

__global__ void dot_partial(i64 n, const double* __restrict__ a, const double* __restrict__ b, double* part) {
  double acc = 0.0;
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    acc += a[i] * b[i];
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void sum_final(int n, const double* part, double* out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += part[i];
  acc = block_sum(acc);
  if (threadIdx.x == 0) *out = acc;
}

__global__ void gather_cols_kernel(i64 rows, i64 ncols, const double* __restrict__ src, i64 lds,
                                   const int* __restrict__ idx, const double* __restrict__ scale,
                                   double* __restrict__ dst, i64 ldd) {
  const i64 total = rows * ncols;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 r = e / ncols;
    const int c = static_cast<int>(e % ncols);
    const double v = src[r * lds + idx[c]];
    dst[r * ldd + c] = scale ? v * scale[c] : v;
  }
}

// One block per 32-column strip; 32 row groups with four independent accumulators each (the
// loads of one thread stay in flight together); fixed-order combination.
__global__ void __launch_bounds__(1024) col_norms_kernel(i64 rows, i64 cols, const double* __restrict__ src, i64 lds,
                                                         double* out) {
  __shared__ double part[32][33];
  const int c = threadIdx.x & 31, rgrp = threadIdx.x >> 5;  // 32 row groups
  const i64 col = static_cast<i64>(blockIdx.x) * 32 + c;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (col < cols) {
    i64 r = rgrp;
    for (; r + 96 < rows; r += 128) {
      const double v0 = src[r * lds + col], v1 = src[(r + 32) * lds + col], v2 = src[(r + 64) * lds + col],
                   v3 = src[(r + 96) * lds + col];
      a0 = fma(v0, v0, a0);
      a1 = fma(v1, v1, a1);
      a2 = fma(v2, v2, a2);
      a3 = fma(v3, v3, a3);
    }
    for (; r < rows; r += 32) {
      const double v = src[r * lds + col];
      a0 = fma(v, v, a0);
    }
  }
  part[rgrp][c] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (rgrp == 0 && col < cols) {
    double s = 0.0;
    for (int g = 0; g < 32; ++g) s += part[g][c];
    out[col] = sqrt(s);
  }
}

int grid_for(i64 total, int threads = 256) {
  return static_cast<int>(std::max<i64>(1, std::min<i64>((total + threads - 1) / threads, 8L * num_sms())));
}

}  // namespace

// DFCG_TRACE_GEMM=1 (diagnostics, while kernel accounting is enabled): time every call alone
struct GemmTrace {
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  cudaStream_t s;
  const char* tag;
  i64 M, N, K;
  double flops;
  GemmTrace(cudaStream_t s_, const char* tag_, i64 M_, i64 N_, i64 K_, double flops_)
      : s(s_), tag(tag_), M(M_), N(N_), K(K_), flops(flops_) {
    static const bool on = std::getenv("DFCG_TRACE_GEMM") != nullptr;
    if (!on || !prof::g_enabled.load()) return;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    cudaEventRecord(t0, s);
  }
  ~GemmTrace() {
    if (!t0) return;
    cudaEventRecord(t1, s);
    cudaEventSynchronize(t1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t0, t1);
    std::fprintf(stderr, "[gemm] %s M=%lld N=%lld K=%lld  %.1f us  %.2f TF/s\n", tag, (long long)M, (long long)N,
                 (long long)K, ms * 1e3, flops / (ms * 1e-3) / 1e12);
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
  }
};

void gemm(cudaStream_t s, bool ta, bool tb, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda,
          const double* B, i64 ldb, double beta, double* C, i64 ldc) {
  if (M <= 0 || N <= 0) return;
  prof::Scope scope(2.0 * M * N * K >= 2e9 ? prof::kGemm : prof::kGemmSmall, s, 2.0 * M * N * K,
                    8.0 * (M * K + K * N + M * N * (beta != 0.0 ? 2.0 : 1.0)));
  if (K <= 0 || alpha == 0.0) {
    scale_kernel<<<grid_for(M * N), 256, 0, s>>>(M, N, beta, C, ldc);
    DFCG_LAUNCH_CHECK();
    return;
  }
  static const char* tags[4] = {"NN", "TN", "NT", "TT"};
  GemmTrace tr(s, tags[(ta ? 1 : 0) + (tb ? 2 : 0)], M, N, K, 2.0 * M * N * K);
  if (!ta && !tb) launch_gemm<false, false>(s, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, 0);
  else if (ta && !tb) launch_gemm<true, false>(s, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, 0);
  else if (!ta && tb) launch_gemm<false, true>(s, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, 0);
  else launch_gemm<true, true>(s, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, 0);
}

void gemm_tri_a(cudaStream_t s, bool ta, i64 M, i64 N, double alpha, const double* A, i64 lda, const double* B,
                i64 ldb, double beta, double* C, i64 ldc) {
  if (M <= 0 || N <= 0) return;
  prof::Scope scope(1.0 * M * M * N >= 2e9 ? prof::kGemm : prof::kGemmSmall, s, 1.0 * M * (M + 1) * N,
                    8.0 * (M * M / 2 + M * N + M * N * (beta != 0.0 ? 2.0 : 1.0)));
  GemmTrace tr(s, ta ? "TRLT" : "TRUP", M, N, M, 1.0 * M * (M + 1) * N);
  if (ta) launch_gemm<true, false>(s, M, N, M, alpha, A, lda, B, ldb, beta, C, ldc, 8);
  else launch_gemm<false, false>(s, M, N, M, alpha, A, lda, B, ldb, beta, C, ldc, 4);
}

void gemm_upper_b(cudaStream_t s, i64 M, i64 N, double alpha, const double* A, i64 lda, const double* B, i64 ldb,
                  double beta, double* C, i64 ldc) {
  if (M <= 0 || N <= 0) return;
  prof::Scope scope(1.0 * M * N * (N + 1) >= 2e9 ? prof::kGemm : prof::kGemmSmall, s, 1.0 * M * N * (N + 1),
                    8.0 * (M * N + N * N / 2 + M * N * (beta != 0.0 ? 2.0 : 1.0)));
  GemmTrace tr(s, "TRMM", M, N, N, 1.0 * M * N * (N + 1));
  launch_gemm<false, false>(s, M, N, N, alpha, A, lda, B, ldb, beta, C, ldc, 2);
}

void gram_upper_nt(cudaStream_t s, i64 rows, i64 k, const double* A, i64 lda, double* G, i64 ldg) {
  if (rows <= 0 || k <= 0) return;
  prof::Scope scope(1.0 * rows * (rows + 1) * k >= 2e9 ? prof::kGemm : prof::kGemmSmall, s,
                    1.0 * rows * (rows + 1) * k, 8.0 * (rows * k + rows * rows));
  launch_gemm<false, true>(s, rows, rows, k, 1.0, A, lda, A, lda, 0.0, G, ldg, 1);
}

void gemm_ta_upper_b(cudaStream_t s, i64 M, i64 N, double alpha, const double* A, i64 lda, const double* B, i64 ldb,
                     double beta, double* C, i64 ldc) {
  if (M <= 0 || N <= 0) return;
  prof::Scope scope(1.0 * M * N * (N + 1) >= 2e9 ? prof::kGemm : prof::kGemmSmall, s, 1.0 * M * N * (N + 1),
                    8.0 * (M * N + N * N / 2 + M * N * (beta != 0.0 ? 2.0 : 1.0)));
  launch_gemm<true, false>(s, M, N, N, alpha, A, lda, B, ldb, beta, C, ldc, 2);
}

void gram_upper(cudaStream_t s, i64 rows, i64 cols, const double* X, i64 ldx, double* G, i64 ldg) {
  if (rows <= 0 || cols <= 0) return;
  prof::Scope scope(1.0 * cols * (cols + 1) * rows >= 2e9 ? prof::kGemm : prof::kGemmSmall, s,
                    1.0 * cols * (cols + 1) * rows, 8.0 * (rows * cols + cols * cols));
  GemmTrace tr(s, "SYRK", cols, cols, rows, 1.0 * cols * (cols + 1) * rows);
  launch_gemm<true, false>(s, cols, cols, rows, 1.0, X, ldx, X, ldx, 0.0, G, ldg, 1);
}

void copy2d(cudaStream_t s, i64 rows, i64 cols, const double* src, i64 lds, double* dst, i64 ldd, double alpha) {
  if (rows <= 0 || cols <= 0) return;
  if (alpha == 1.0) {
    DFCG_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * ldd, src, sizeof(double) * lds, sizeof(double) * cols, rows,
                                cudaMemcpyDeviceToDevice, s));
    return;
  }
  prof::Scope scope(prof::kElementwise, s, 0.0, 16.0 * rows * cols);
  copy2d_kernel<<<grid_for(rows * cols), 256, 0, s>>>(rows, cols, src, lds, dst, ldd, alpha);
  DFCG_LAUNCH_CHECK();
}

void transpose(cudaStream_t s, i64 rows, i64 cols, const double* src, i64 lds, double* dst, i64 ldd) {
  if (rows <= 0 || cols <= 0) return;
  prof::Scope scope(prof::kElementwise, s, 0.0, 16.0 * rows * cols);
  dim3 grid(cdiv(cols, 32), cdiv(rows, 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(rows, cols, src, lds, dst, ldd);
  DFCG_LAUNCH_CHECK();
}

void set_identity(cudaStream_t s, i64 rows, i64 cols, double* dst, i64 ldd) {
  if (rows <= 0 || cols <= 0) return;
  identity_kernel<<<grid_for(rows * cols), 256, 0, s>>>(rows, cols, dst, ldd);
  DFCG_LAUNCH_CHECK();
}

void dot_sum(cudaStream_t s, i64 n, const double* a, const double* b, double* out) {
  prof::Scope scope(prof::kReduce, s, 2.0 * n, 16.0 * n);
  DBuf<double> part(RED_BLOCKS, s);
  dot_partial<<<RED_BLOCKS, RED_THREADS, 0, s>>>(n, a, b, part.get());
  DFCG_LAUNCH_CHECK();
  sum_final<<<1, RED_THREADS, 0, s>>>(RED_BLOCKS, part.get(), out);
  DFCG_LAUNCH_CHECK();
}

void gather_cols(cudaStream_t s, i64 rows, i64 ncols, const double* src, i64 lds, const int* idx,
                 const double* scale, double* dst, i64 ldd) {
  if (rows <= 0 || ncols <= 0) return;
  prof::Scope scope(prof::kElementwise, s, 0.0, 16.0 * rows * ncols);
  gather_cols_kernel<<<grid_for(rows * ncols), 256, 0, s>>>(rows, ncols, src, lds, idx, scale, dst, ldd);
  DFCG_LAUNCH_CHECK();
}

void col_norms(cudaStream_t s, i64 rows, i64 cols, const double* src, i64 lds, double* out) {
  if (cols <= 0) return;
  prof::Scope scope(prof::kReduce, s, 2.0 * rows * cols, 8.0 * rows * cols);
  col_norms_kernel<<<cdiv(cols, 32), 1024, 0, s>>>(rows, cols, src, lds, out);
  DFCG_LAUNCH_CHECK();
}

}  // namespace dfcg
