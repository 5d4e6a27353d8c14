// Sparse kernels for the observed set Omega (see sparse.cuh).
//
// SDDMM: entry-parallel over the CSR stream, G lanes per entry (G ~ kY/4, power of two),
// factor rows gathered contiguously (row-major factors), group reduction by xor-shuffles.
// SpMM: segmented work list (<= 64 or 128 entries per item) so long CSC columns split across
// warps; multi-segment rows reduce their partials in a fixed order (deterministic).
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "sparse.cuh"

namespace dfcg {

namespace {

constexpr int kSpmmCpl = 4;
constexpr int SLAB_WARPS = 16;  // warps per CTA of the slab SpMM / SDDMM kernels

// kernel-choice overrides for the microbenchmark entry (dfcg_bench_sparse); -1: environment
std::atomic<int> g_spmm_mode{-1}, g_sddmm_mode{-1};

int pow2_at_least(i64 v) {
  int g = 1;
  while (g < v && g < 32) g <<= 1;
  return g;
}

template <int G>
__global__ void sddmm_kernel(i64 N, i64 kY, const int* __restrict__ row, const int* __restrict__ col,
                             const double* __restrict__ Yl, i64 ldl, const double* __restrict__ Yr, i64 ldr,
                             const double* __restrict__ sub, double* __restrict__ out) {
  constexpr int PER_WARP = 32 / G;
  const int lane = threadIdx.x & 31, lig = lane % G;
  const i64 warp = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
  for (i64 base = warp * PER_WARP; base < N; base += nwarps * PER_WARP) {
    const i64 e = base + lane / G;
    double acc = 0.0;
    if (e < N && kY > 0) {
      const double* yl = Yl + static_cast<i64>(row[e]) * ldl;
      const double* yr = Yr + static_cast<i64>(col[e]) * ldr;
      for (i64 k = lig; k < kY; k += G) acc = fma(yl[k], yr[k], acc);
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (e < N && lig == 0) out[e] = sub ? acc - sub[e] : acc;
  }
}

// Segmented SpMM. transpose=false: items walk CSR rows, structure idx = csr_col, value t.
// transpose=true: items walk CSC columns, idx = csc_row, value csc2csr[e].
template <int G, bool T, int CPL = kSpmmCpl>
__global__ void spmm_kernel(i64 n_items, const SegItem* __restrict__ items, const int* __restrict__ idx,
                            const long long* __restrict__ perm, const double* __restrict__ vals, i64 b, double alpha,
                            const double* __restrict__ X, i64 ldx, double beta, double* __restrict__ out, i64 ldo,
                            double* __restrict__ ws) {
  constexpr int PER_WARP = 32 / G;
  const int lane = threadIdx.x & 31, lig = lane % G;
  const i64 gid = ((static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * PER_WARP + lane / G;
  if (gid >= n_items) return;
  const SegItem it = items[gid];
  // CPL columns per lane per pass: one walk of the segment covers CPL G columns
  for (i64 c0 = 0; c0 < b; c0 += CPL * G) {
    double acc[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) acc[q] = 0.0;
    // entries in batches of 4: all index/value loads issued before the dependent X gathers
    long long e = it.e0;
    for (; e + 4 <= it.e1; e += 4) {
      int ix[4];
      double vv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ix[u] = idx[e + u];
        vv[u] = perm ? vals[perm[e + u]] : vals[e + u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double* x = X + static_cast<i64>(ix[u]) * ldx + c0 + lig;
#pragma unroll
        for (int q = 0; q < CPL; ++q)
          if (c0 + lig + q * G < b) acc[q] = fma(vv[u], x[q * G], acc[q]);
      }
    }
    for (; e < it.e1; ++e) {
      const double v = perm ? vals[perm[e]] : vals[e];
      const double* x = X + static_cast<i64>(idx[e]) * ldx + c0 + lig;
#pragma unroll
      for (int q = 0; q < CPL; ++q)
        if (c0 + lig + q * G < b) acc[q] = fma(v, x[q * G], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const i64 c = c0 + lig + q * G;
      if (c >= b) continue;
      if (it.slot < 0) {
        double* o = out + static_cast<i64>(it.row) * ldo + c;
        *o = beta == 0.0 ? alpha * acc[q] : alpha * acc[q] + beta * *o;
      } else {
        ws[static_cast<i64>(it.slot) * b + c] = acc[q];
      }
    }
  }
}

// Segmented SpMM, 16-byte variant (opt-in, DFCG_SPMM16=1; needs 16-byte aligned sketch rows: even
// ldx, aligned base — every sketch buffer of the range finder is). Same items, same per-column FMA
// order as spmm_kernel (bitwise the same output); two changes, both aimed at the kernel's
// limiter, the L1 data pipe (ncu: l1tex__data_pipe_lsu_wavefronts at 87% of peak, L2 at 43%,
// DRAM at 9%, profiles/r02_ncu_spmm_c5.txt — ~6.4 wavefronts per entry against 2.2 for the
// 280-byte row alone):
//   * X rows are read as double2 (G lanes x 16 bytes per row segment, 2 chunks per lane per pass);
//   * index and value are loaded once per entry by ONE lane of the group (coalesced, G entries
//     per load) and handed to the group by shuffles, instead of every lane of the group loading
//     the same two words (a 16-lane broadcast load writes back 16 x 12 bytes per entry).
// A group whose segment is shorter leaves its loop early: every shuffle names only the group's
// own lanes in its mask. The last chunk of an odd b reads one padding double (ldx >= b + 1).
template <int G, bool T>
__global__ void spmm16_kernel(i64 n_items, const SegItem* __restrict__ items, const int* __restrict__ idx,
                              const double* __restrict__ vals, i64 b, double alpha, const double* __restrict__ X,
                              i64 ldx, double beta, double* __restrict__ out, i64 ldo, double* __restrict__ ws) {
  constexpr int PER_WARP = 32 / G;
  const int lane = threadIdx.x & 31, lig = lane % G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (lane - lig));
  const i64 gid = ((static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * PER_WARP + lane / G;
  if (gid >= n_items) return;  // whole groups leave together
  const SegItem it = items[gid];
  const i64 nch = (b + 1) >> 1;  // double2 chunks per row
  const i64 ld2 = ldx >> 1;
  const double2* __restrict__ X2 = reinterpret_cast<const double2*>(X);
  for (i64 c0 = 0; c0 < nch; c0 += 2 * G) {
    const bool on0 = c0 + lig < nch, on1 = c0 + lig + G < nch;
    double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
    for (long long e = it.e0; e < it.e1; e += G) {
      const long long mine = e + lig;
      const int my_ix = mine < it.e1 ? idx[mine] : 0;
      const double my_v = mine < it.e1 ? vals[mine] : 0.0;
      const int cnt = static_cast<int>(it.e1 - e < G ? it.e1 - e : G);
      int u = 0;
      for (; u + 4 <= cnt; u += 4) {
        int ix[4];
        double vv[4];
        double2 x0[4], x1[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          ix[q] = __shfl_sync(gmask, my_ix, u + q, G);
          vv[q] = __shfl_sync(gmask, my_v, u + q, G);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2* x = X2 + static_cast<i64>(ix[q]) * ld2 + c0 + lig;
          x0[q] = on0 ? __ldg(x) : make_double2(0.0, 0.0);
          x1[q] = on1 ? __ldg(x + G) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          a0.x = fma(vv[q], x0[q].x, a0.x);
          a0.y = fma(vv[q], x0[q].y, a0.y);
          a1.x = fma(vv[q], x1[q].x, a1.x);
          a1.y = fma(vv[q], x1[q].y, a1.y);
        }
      }
      for (; u < cnt; ++u) {
        const int ix = __shfl_sync(gmask, my_ix, u, G);
        const double v = __shfl_sync(gmask, my_v, u, G);
        const double2* x = X2 + static_cast<i64>(ix) * ld2 + c0 + lig;
        if (on0) {
          const double2 t = __ldg(x);
          a0.x = fma(v, t.x, a0.x);
          a0.y = fma(v, t.y, a0.y);
        }
        if (on1) {
          const double2 t = __ldg(x + G);
          a1.x = fma(v, t.x, a1.x);
          a1.y = fma(v, t.y, a1.y);
        }
      }
    }
    auto put = [&](i64 c, double acc) {
      if (c >= b) return;
      if (it.slot < 0) {
        double* o = out + static_cast<i64>(it.row) * ldo + c;
        *o = beta == 0.0 ? alpha * acc : alpha * acc + beta * *o;
      } else {
        ws[static_cast<i64>(it.slot) * b + c] = acc;
      }
    };
    if (on0) {
      put(2 * (c0 + lig), a0.x);
      put(2 * (c0 + lig) + 1, a0.y);
    }
    if (on1) {
      put(2 * (c0 + lig + G), a1.x);
      put(2 * (c0 + lig + G) + 1, a1.y);
    }
  }
}

// Slab SpMM for sketches of b <= 64 columns: out[o, :] (+)= alpha sum_e v_e X[idx_e, :] over the
// entries e of outer line o (a CSR row for R X, a CSC column for R^T X).
//
// Why: the segmented kernel gathers a b-wide row of X from L2 for every entry (N b 8 bytes of L2
// reads, ~20x the algorithmic HBM bytes at b ~ 35; L2 throughput is only ~2x HBM on B200), so it
// is L2-bound. Here X streams through shared memory in slabs of SB inner rows (double-buffered
// cp.async), once per CTA of RB = 16 R outer lines, and every entry's X row is read from shared
// memory: the X traffic from L2 drops by RB x density, the per-entry operand traffic moves to
// shared memory (128 B/clk/SM), which bounds the kernel.
//
// Mapping: each warp owns R consecutive outer lines; its 32 lanes form gpw = 32 / G groups of
// G = ceil(b / 4) lanes, lane (g, j) holding columns 4j .. 4j+3 (two 16-byte shared loads per
// entry, conflict-free within a group). The entries of one line in the slab are loaded 32 at a
// time, coalesced, and dealt round-robin to the groups by shuffles: group g accumulates entries
// g, g + gpw, ... of every line (balanced to one entry; warp-uniform control flow). After the last
// slab the groups' partial sums are added in group order (shuffles) and group 0 writes.
// Deterministic: fixed slab order, fixed entry-to-group deal, fixed group reduction order.
// Inner dimension split into gridDim.y chunks (whole slabs) when the outer lines alone do not
// fill the GPU: partial results go to ws and spmm_chunk_reduce adds them in chunk order.
template <int R>
__global__ void __launch_bounds__(SLAB_WARPS * 32, 1)
    spmm_slab_kernel(i64 n_outer, i64 n_inner, int nt, const int* __restrict__ tptr, const int* __restrict__ idx,
                     const double* __restrict__ vals, int b, int G, int SB, double alpha,
                     const double* __restrict__ X, i64 ldx, double beta, double* __restrict__ out, i64 ldo,
                     int chunk_tiles, double* __restrict__ ws) {
  extern __shared__ __align__(16) double xs[];  // [2][SB][BP]
  const int BP = 4 * G;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int gpw = 32 / G, g = lane / G, j = lane - g * G;
  const bool active = g < gpw;  // lanes past the last whole group idle in the FMA loop
  const i64 o0 = (static_cast<i64>(blockIdx.x) * SLAB_WARPS + warp) * R;
  const int q_begin = blockIdx.y * chunk_tiles, q_end = min(nt, q_begin + chunk_tiles);
  const int TPS = SB / DevOmega::kTileCols;
  const int nslab = (q_end - q_begin + TPS - 1) / TPS;
  // lane j of a group owns columns {2j, 2j+1} and {2G+2j, 2G+2j+1}: each 16-byte shared load of a
  // group covers one contiguous 16G-byte run of its X row (conflict-free within the group)
  double acc[R][4];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;

  auto stage = [&](int sl, int buf) {  // slab sl -> buffer buf (8-byte copies: any ldx)
    const int q0 = q_begin + sl * TPS;
    const i64 in0 = static_cast<i64>(q0) * DevOmega::kTileCols;
    const int rows_in = static_cast<int>(min(static_cast<i64>(SB), n_inner - in0));
    double* dst = xs + static_cast<size_t>(buf) * SB * BP;
    for (int e = t; e < rows_in * b; e += SLAB_WARPS * 32) {
      const int r = e / b, c = e - r * b;
      cp_async8(dst + r * BP + c, X + (in0 + r) * ldx + c, true);
    }
    cp_async_commit();
  };
  if (nslab > 0) stage(0, 0);
  for (int sl = 0; sl < nslab; ++sl) {
    const int q0 = q_begin + sl * TPS, q1 = min(q_end, q0 + TPS);
    const i64 in0 = static_cast<i64>(q0) * DevOmega::kTileCols;
    // the slab's entries of the warp's R lines, first 32 of each, loaded before the wait on the
    // slab copy: R independent coalesced loads in flight at once
    int tv = 0;
    if (lane < 2 * R) {
      const i64 o = o0 + (lane % R);
      tv = o < n_outer ? tptr[o * (nt + 1) + (lane < R ? q0 : q1)] : 0;
    }
    int e0[R], e1[R], ix[R];
    double v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      e0[r] = __shfl_sync(0xffffffffu, tv, r);
      e1[r] = __shfl_sync(0xffffffffu, tv, R + r);
      ix[r] = 0;
      v[r] = 0.0;
      if (lane < e1[r] - e0[r]) {
        ix[r] = idx[e0[r] + lane] - static_cast<int>(in0);
        v[r] = vals[e0[r] + lane];
      }
    }
    if (sl + 1 < nslab) {
      stage(sl + 1, (sl + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* xb = xs + static_cast<size_t>(sl & 1) * SB * BP + 2 * j;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      for (int base = e0[r]; base < e1[r]; base += 32) {
        const int n_here = min(32, e1[r] - base);
        int ixc = ix[r];
        double vc = v[r];
        if (base > e0[r]) {  // lines with more than 32 entries in this slab
          ixc = 0;
          vc = 0.0;
          if (lane < n_here) {
            ixc = idx[base + lane] - static_cast<int>(in0);
            vc = vals[base + lane];
          }
        }
        for (int jj = 0; jj < n_here; jj += gpw) {
          const int src = jj + g;
          const int ixs = __shfl_sync(0xffffffffu, ixc, src & 31);
          const double vs = __shfl_sync(0xffffffffu, vc, src & 31);
          if (active && src < n_here) {
            const double* xr = xb + ixs * BP;
            const double2 a = *reinterpret_cast<const double2*>(xr);
            const double2 c2 = *reinterpret_cast<const double2*>(xr + 2 * G);
            acc[r][0] = fma(vs, a.x, acc[r][0]);
            acc[r][1] = fma(vs, a.y, acc[r][1]);
            acc[r][2] = fma(vs, c2.x, acc[r][2]);
            acc[r][3] = fma(vs, c2.y, acc[r][3]);
          }
        }
      }
    }
    __syncthreads();  // buffer (sl & 1) is refilled by the next iteration's stage
  }
  // groups' partials in group order into group 0
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double sum = acc[r][c];
      for (int k = 1; k < gpw; ++k) sum += __shfl_sync(0xffffffffu, acc[r][c], (lane + k * G) & 31);
      acc[r][c] = sum;
    }
  if (g != 0) return;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const i64 o = o0 + r;
    if (o >= n_outer) break;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int col = (c < 2 ? 2 * j : 2 * G + 2 * j) + (c & 1);
      if (col >= b) continue;
      if (ws) {
        ws[(static_cast<i64>(blockIdx.y) * n_outer + o) * b + col] = acc[r][c];
      } else {
        double* p = out + o * ldo + col;
        *p = beta == 0.0 ? alpha * acc[r][c] : fma(beta, *p, alpha * acc[r][c]);
      }
    }
  }
}

__global__ void spmm_chunk_reduce(i64 n_outer, int b, int chunks, const double* __restrict__ ws, double alpha,
                                  double beta, double* __restrict__ out, i64 ldo) {
  const i64 total = n_outer * b;
  for (i64 t = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<i64>(gridDim.x) * blockDim.x) {
    double sacc = 0.0;
    for (int y = 0; y < chunks; ++y) sacc += ws[y * total + t];
    const i64 o = t / b, c = t - o * b;
    double* p = out + o * ldo + c;
    *p = beta == 0.0 ? alpha * sacc : fma(beta, *p, alpha * sacc);
  }
}

// Rows split into several segments: out[row] = alpha * sum(slots in order) + beta * out[row].
__global__ void seg_reduce_kernel(i64 nrows, const int* __restrict__ rows, const int* __restrict__ slot_ptr, i64 b,
                                  const double* __restrict__ ws, double alpha, double beta, double* __restrict__ out,
                                  i64 ldo) {
  const i64 total = nrows * b;
  for (i64 t = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 r = t / b, c = t % b;
    double s = 0.0;
    for (int k = slot_ptr[r]; k < slot_ptr[r + 1]; ++k) s += ws[static_cast<i64>(k) * b + c];
    double* o = out + static_cast<i64>(rows[r]) * ldo + c;
    *o = beta == 0.0 ? alpha * s : alpha * s + beta * *o;
  }
}

// Rows with no entries at all still need out = beta * out.
__global__ void empty_rows_kernel(i64 nrows, const int* __restrict__ ptr, i64 b, double beta, double* out, i64 ldo) {
  const i64 total = nrows * b;
  for (i64 t = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 r = t / b, c = t % b;
    if (ptr[r] == ptr[r + 1]) out[r * ldo + c] = beta == 0.0 ? 0.0 : beta * out[r * ldo + c];
  }
}

__global__ void scatter_dense_kernel(i64 N, const int* __restrict__ row, const int* __restrict__ col,
                                     const double* __restrict__ vals, double alpha, double* __restrict__ D, i64 ldd) {
  for (i64 t = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; t < N;
       t += static_cast<i64>(gridDim.x) * blockDim.x)
    D[static_cast<i64>(row[t]) * ldd + col[t]] += alpha * vals[t];
}

// Tiled SDDMM: one CTA per 64 x 64 tile of the observed matrix. The tile's factor rows
// Yl[i0:i0+64, :] and Yr[j0:j0+64, :] stream through shared memory in 32-wide k chunks (double
// buffered, cp.async) and every thread accumulates the dot products of up to SEPT of the tile's
// entries from there: each factor row is read from L2 once per tile instead of once per entry
// (~6x less L2 traffic at 10% density). Each lane walks a chunk starting at k = lane, so the
// 16 lanes of a shared-memory phase hit 16 distinct banks whatever rows they read.
// Tile widths: TW column tiles of the CSR table per CTA (TW = 1: 64 x 64 tiles, the high-rank
// c2 setting; TW = 4 with 16-wide k chunks at kY <= 32: 64 x 256 tiles, four times the entries
// per CTA to amortise the per-tile setup at low rank and low density).
constexpr int STR = 64, SDD_T = 256, SEPT = 4;
template <int TW, int SKC>
constexpr size_t sddmm_smem() { return sizeof(double) * 2 * (STR + TW * DevOmega::kTileCols) * SKC; }

template <int TW, int SKC>
__global__ void __launch_bounds__(SDD_T) sddmm_tile_kernel(i64 m, i64 n, i64 kY, int ntc, const int* __restrict__ tptr,
                                                           const int* __restrict__ col, const double* __restrict__ Yl,
                                                           i64 ldl, const double* __restrict__ Yr, i64 ldr,
                                                           const double* __restrict__ sub, double* __restrict__ out) {
  constexpr int STC = TW * DevOmega::kTileCols;
  extern __shared__ double sm[];  // [2][STR][SKC] then [2][STC][SKC]
  double* sl = sm;
  double* sr = sm + 2 * STR * SKC;
  __shared__ int pre[STR + 1];
  __shared__ int base_pos[STR];
  const int t = threadIdx.x, lane = t & 31;
  const i64 i0 = static_cast<i64>(blockIdx.y) * STR, j0 = static_cast<i64>(blockIdx.x) * STC;
  const int q0 = blockIdx.x * TW, q1 = min(ntc, q0 + TW);
  if (t < STR) {  // the tile's row counts, prefix-summed by warp scans (two warps)
    const i64 i = i0 + t;
    int b0 = 0, c = 0;
    if (i < m) {
      b0 = tptr[i * (ntc + 1) + q0];
      c = tptr[i * (ntc + 1) + q1] - b0;
    }
    base_pos[t] = b0;
    int v = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    pre[t + 1] = v;  // inclusive within the warp
  }
  __syncthreads();
  if (t >= 32 && t < STR) pre[t + 1] += pre[32];  // second warp: add the first warp's total
  if (t == 0) pre[0] = 0;
  __syncthreads();
  const int total = pre[STR];
  if (total == 0) return;
  const i64 rows_in = min(static_cast<i64>(STR), m - i0), cols_in = min(static_cast<i64>(STC), n - j0);
  // staging (16-byte cp.async; ldl, ldr even and the bases 16-byte aligned, see the host side):
  // thread t copies the column pair 2 (t % 16) of rows t / 16, t / 16 + 16, ... of both tiles.
  // kY is rounded up to even by the host (the padding column holds zeros), so a pair is either
  // entirely inside k < kY or entirely outside.
  constexpr int PR = SKC / 2, RS = SDD_T / PR;  // pairs per row, rows per pass
  const int skk = 2 * (t % PR), sr0 = t / PR;
  auto stage = [&](int buf, i64 k0) {
    double* dl = sl + buf * STR * SKC + sr0 * SKC + skk;
    double* dr = sr + buf * STC * SKC + sr0 * SKC + skk;
    const bool kin = k0 + skk < kY;
    const double* gl = Yl + (i0 + sr0) * ldl + k0 + skk;
    const double* gr = Yr + (j0 + sr0) * ldr + k0 + skk;
#pragma unroll
    for (int q = 0; q < STR / RS; ++q) {
      const bool ok = kin && sr0 + q * RS < rows_in;
      cp_async16(dl + q * RS * SKC, ok ? gl + q * RS * ldl : Yl, ok);
    }
#pragma unroll
    for (int q = 0; q < STC / RS; ++q) {
      const bool ok = kin && sr0 + q * RS < cols_in;
      cp_async16(dr + q * RS * SKC, ok ? gr + q * RS * ldr : Yr, ok);
    }
    cp_async_commit();
  };
  for (int first = 0; first < total; first += SDD_T * SEPT) {
    __syncthreads();  // previous pass done with the staging buffers
    int li[SEPT], lj[SEPT], pos[SEPT];
    double acc[SEPT];
#pragma unroll
    for (int q = 0; q < SEPT; ++q) {
      const int e = first + t + q * SDD_T;
      acc[q] = 0.0;
      li[q] = -1;
      if (e < total) {
        int lo = 0, hi = STR;  // largest r with pre[r] <= e
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (pre[mid] <= e) lo = mid;
          else hi = mid;
        }
        li[q] = lo;
        pos[q] = base_pos[lo] + (e - pre[lo]);
        lj[q] = static_cast<int>(col[pos[q]] - j0);
      }
    }
    const int nk = static_cast<int>((kY + SKC - 1) / SKC);
    if (nk > 0) stage(0, 0);
    for (int kc = 0; kc < nk; ++kc) {
      if (kc + 1 < nk) {
        stage((kc + 1) & 1, static_cast<i64>(kc + 1) * SKC);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const double* dl = sl + (kc & 1) * STR * SKC;
      const double* dr = sr + (kc & 1) * STC * SKC;
#pragma unroll
      for (int q = 0; q < SEPT; ++q) {
        if (!__any_sync(0xffffffffu, li[q] >= 0)) break;  // later slots are empty for the whole warp
        if (li[q] < 0) continue;
        // 16-byte loads, the pair index rotated by lane: 8 lanes of a phase hit 8 distinct slots
        const double2* a = reinterpret_cast<const double2*>(dl + li[q] * SKC);
        const double2* b = reinterpret_cast<const double2*>(dr + lj[q] * SKC);
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < SKC / 2; ++kk) {
          const int k = (kk + lane) & (SKC / 2 - 1);
          const double2 x = a[k], y = b[k];
          s0 = fma(x.x, y.x, s0);
          s1 = fma(x.y, y.y, s1);
        }
        acc[q] += s0 + s1;
      }
      __syncthreads();  // the buffer just read is refilled by the next iteration's stage
    }
#pragma unroll
    for (int q = 0; q < SEPT; ++q)
      if (li[q] >= 0) out[pos[q]] = sub ? acc[q] - sub[pos[q]] : acc[q];
  }
}

// Slab SDDMM for kY <= 64: r_e = <Yl[i, :], Yr[j, :]> - sub_e over the CSR entries.
// Each warp owns R consecutive rows; their Yl rows sit in registers for the whole kernel (group
// lane j holds Yl[i][4j .. 4j+3]); Yr streams through shared memory in slabs of SB rows (double
// buffered cp.async, each slab read from L2 once per CTA of 16 R rows). The entries of a row
// inside the slab are loaded 32 at a time (coalesced) and dealt round-robin to the warp's 32 / G
// groups (G = power of two >= kY / 4): a group forms its entry's dot product from two 16-byte
// shared loads per lane and a log2(G)-step xor-shuffle reduction; the group leader writes r_e.
// Per entry: 8 kY bytes of shared-memory operand traffic (the bound) instead of the entry-
// parallel kernel's 16 kY bytes of L2 gathers.
template <int R, int G>
__global__ void __launch_bounds__(SLAB_WARPS * 32, 1)
    sddmm_slab_kernel(i64 m, i64 n, int kY, int ntc, int SB, const int* __restrict__ tptr,
                      const int* __restrict__ col, const double* __restrict__ Yl, i64 ldl,
                      const double* __restrict__ Yr, i64 ldr, const double* __restrict__ sub,
                      double* __restrict__ out) {
  extern __shared__ __align__(16) double ys[];  // [2][SB][BP]
  constexpr int BP = 4 * G, GPW = 32 / G;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int g = lane / G, j = lane % G;
  const bool kact = 4 * j < kY;  // lanes past the k extent load nothing
  const i64 r0 = (static_cast<i64>(blockIdx.x) * SLAB_WARPS + warp) * R;
  double yl[R][4];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int k = 4 * j + c;
      yl[r][c] = (r0 + r < m && k < kY) ? Yl[(r0 + r) * ldl + k] : 0.0;
    }
  const int TPS = SB / DevOmega::kTileCols;
  const int nslab = (ntc + TPS - 1) / TPS;
  auto stage = [&](int sl, int buf) {
    const i64 c0 = static_cast<i64>(sl) * SB;
    const int rows_in = static_cast<int>(min(static_cast<i64>(SB), n - c0));
    double* dst = ys + static_cast<size_t>(buf) * SB * BP;
    for (int e = t; e < rows_in * BP; e += SLAB_WARPS * 32) {
      const int rr = e / BP, k = e - rr * BP;
      if (k < kY) cp_async8(dst + e, Yr + (c0 + rr) * ldr + k, true);
      else dst[e] = 0.0;
    }
    cp_async_commit();
  };
  if (nslab > 0) stage(0, 0);
  for (int sl = 0; sl < nslab; ++sl) {
    if (sl + 1 < nslab) {
      stage(sl + 1, (sl + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int q0 = sl * TPS, q1 = min(ntc, q0 + TPS);
    const int c0 = sl * SB;
    const double* yb = ys + static_cast<size_t>(sl & 1) * SB * BP + 4 * j;
    int tv = 0;
    if (lane < 2 * R) {
      const i64 i = r0 + (lane % R);
      tv = i < m ? tptr[i * (ntc + 1) + (lane < R ? q0 : q1)] : 0;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int e0 = __shfl_sync(0xffffffffu, tv, r), e1 = __shfl_sync(0xffffffffu, tv, R + r);
      for (int base = e0; base < e1; base += 32) {
        const int n_here = min(32, e1 - base);
        int cj = 0;
        if (lane < n_here) cj = col[base + lane] - c0;
        for (int jj = 0; jj < n_here; jj += GPW) {
          const int src = jj + g;
          const int cs = __shfl_sync(0xffffffffu, cj, src & 31);
          double p = 0.0;
          if (kact && src < n_here) {
            const double2* yr = reinterpret_cast<const double2*>(yb + cs * BP);
            const double2 a = yr[0], b2 = yr[1];
            p = fma(yl[r][0], a.x, fma(yl[r][1], a.y, fma(yl[r][2], b2.x, yl[r][3] * b2.y)));
          }
#pragma unroll
          for (int o = G / 2; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
          if (j == 0 && src < n_here) {
            const int e = base + src;
            out[e] = sub ? p - sub[e] : p;
          }
        }
      }
    }
    __syncthreads();
  }
}

int grid_for(i64 total, int threads = 256) {
  return static_cast<int>(std::max<i64>(1, std::min<i64>((total + threads - 1) / threads, 4096)));
}

void build_plan(cudaStream_t s, SegPlan& p, i64 rows, const std::vector<int>& ptr, int seg_len) {
  const int SEG = seg_len;
  std::vector<SegItem> items;
  std::vector<int> multi_rows, slot_ptr{0};
  int slot = 0;
  for (i64 r = 0; r < rows; ++r) {
    const long long a = ptr[r], bnd = ptr[r + 1];
    const long long nseg = (bnd - a + SEG - 1) / SEG;
    if (nseg == 1) {
      items.push_back({static_cast<int>(r), -1, a, bnd});
    } else if (nseg > 1) {
      multi_rows.push_back(static_cast<int>(r));
      for (long long sgm = 0; sgm < nseg; ++sgm)
        items.push_back({static_cast<int>(r), slot++, a + sgm * SEG, std::min(bnd, a + (sgm + 1) * SEG)});
      slot_ptr.push_back(slot);
    }
  }
  p.rows = rows;
  p.n_items = static_cast<i64>(items.size());
  p.n_slots = slot;
  p.h_multi_rows = multi_rows;
  p.items.alloc(std::max<i64>(1, p.n_items), s);
  if (p.n_items)
    DFCG_CUDA(cudaMemcpyAsync(p.items.get(), items.data(), sizeof(SegItem) * items.size(), cudaMemcpyHostToDevice, s));
  p.multi_rows.alloc(std::max<size_t>(1, multi_rows.size()), s);
  p.red_rowptr.alloc(static_cast<i64>(slot_ptr.size()), s);
  if (!multi_rows.empty())
    DFCG_CUDA(cudaMemcpyAsync(p.multi_rows.get(), multi_rows.data(), sizeof(int) * multi_rows.size(),
                              cudaMemcpyHostToDevice, s));
  DFCG_CUDA(cudaMemcpyAsync(p.red_rowptr.get(), slot_ptr.data(), sizeof(int) * slot_ptr.size(), cudaMemcpyHostToDevice,
                            s));
  // host vectors must outlive the async copies
  DFCG_CUDA(cudaStreamSynchronize(s));
}

// Chunked plan (see DevOmega::plan_csr_ck): tab is the walk's per-line 64-tile offset table
// (lines x (nt + 1)); items in (chunk, line) order, segments <= seg_len entries, slots grouped per
// line in chunk order (seg_reduce_kernel's layout); a line with a single run writes directly.
void build_chunked_plan(cudaStream_t s, SegPlan& p, i64 rows, const std::vector<int>& tab, int nt, int seg_len) {
  const int ct = DevOmega::kChunkTiles;
  const int nchunks = (nt + ct - 1) / ct;
  auto run = [&](i64 r, int c, long long& a, long long& b) {
    a = tab[static_cast<size_t>(r * (nt + 1) + c * ct)];
    b = tab[static_cast<size_t>(r * (nt + 1) + std::min(nt, (c + 1) * ct))];
  };
  std::vector<int> nseg(static_cast<size_t>(rows), 0);
  for (int c = 0; c < nchunks; ++c)
    for (i64 r = 0; r < rows; ++r) {
      long long a, b;
      run(r, c, a, b);
      if (b > a) nseg[static_cast<size_t>(r)] += static_cast<int>((b - a + seg_len - 1) / seg_len);
    }
  std::vector<int> base(static_cast<size_t>(rows) + 1, 0), multi_rows, slot_ptr{0};
  int slot = 0;
  for (i64 r = 0; r < rows; ++r) {
    base[static_cast<size_t>(r)] = slot;
    if (nseg[static_cast<size_t>(r)] > 1) {
      multi_rows.push_back(static_cast<int>(r));
      slot += nseg[static_cast<size_t>(r)];
      slot_ptr.push_back(slot);
    }
  }
  std::vector<int> next(base.begin(), base.end() - 1);
  std::vector<SegItem> items;
  for (int c = 0; c < nchunks; ++c)
    for (i64 r = 0; r < rows; ++r) {
      long long a, b;
      run(r, c, a, b);
      for (long long e = a; e < b; e += seg_len) {
        const int sl = nseg[static_cast<size_t>(r)] > 1 ? next[static_cast<size_t>(r)]++ : -1;
        items.push_back({static_cast<int>(r), sl, e, std::min(b, e + seg_len)});
      }
    }
  p.rows = rows;
  p.n_items = static_cast<i64>(items.size());
  p.n_slots = slot;
  p.h_multi_rows = multi_rows;
  p.items.alloc(std::max<i64>(1, p.n_items), s);
  if (p.n_items)
    DFCG_CUDA(cudaMemcpyAsync(p.items.get(), items.data(), sizeof(SegItem) * items.size(), cudaMemcpyHostToDevice, s));
  p.multi_rows.alloc(std::max<size_t>(1, multi_rows.size()), s);
  p.red_rowptr.alloc(static_cast<i64>(slot_ptr.size()), s);
  if (!multi_rows.empty())
    DFCG_CUDA(cudaMemcpyAsync(p.multi_rows.get(), multi_rows.data(), sizeof(int) * multi_rows.size(),
                              cudaMemcpyHostToDevice, s));
  DFCG_CUDA(cudaMemcpyAsync(p.red_rowptr.get(), slot_ptr.data(), sizeof(int) * slot_ptr.size(), cudaMemcpyHostToDevice,
                            s));
  DFCG_CUDA(cudaStreamSynchronize(s));  // host vectors must outlive the async copies
}

template <class T>
void upload(cudaStream_t s, DBuf<T>& d, const std::vector<T>& h) {
  d.alloc(std::max<size_t>(1, h.size()), s);
  if (!h.empty()) DFCG_CUDA(cudaMemcpyAsync(d.get(), h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, s));
}

}  // namespace

void set_sparse_modes(int spmm_mode, int sddmm_mode) {
  g_spmm_mode.store(spmm_mode);
  g_sddmm_mode.store(sddmm_mode);
}

void DevOmega::build(cudaStream_t s, i64 m_, i64 n_, i64 nnz_, const long long* rows, const long long* cols,
                     const double* vals) {
  m = m_;
  n = n_;
  nnz = nnz_;
  if (m > INT32_MAX || n > INT32_MAX || nnz > (1LL << 40)) throw std::invalid_argument("Omega: dimensions too large");
  std::vector<int> colptr(n + 1, 0), crow(nnz), rowptr(m + 1, 0), rcol(nnz), rrow(nnz);
  std::vector<double> mc(vals, vals + nnz), mr(nnz);
  std::vector<long long> c2r(nnz);
  for (i64 e = 0; e < nnz; ++e) {
    colptr[cols[e] + 1]++;
    rowptr[rows[e] + 1]++;
    crow[e] = static_cast<int>(rows[e]);
  }
  for (i64 j = 0; j < n; ++j) colptr[j + 1] += colptr[j];
  for (i64 i = 0; i < m; ++i) rowptr[i + 1] += rowptr[i];
  std::vector<int> fill(rowptr.begin(), rowptr.end() - 1);
  for (i64 e = 0; e < nnz; ++e) {  // CSC order is column-major, so each CSR row fills in column order
    const int r = static_cast<int>(rows[e]);
    const int t = fill[r]++;
    rcol[t] = static_cast<int>(cols[e]);
    rrow[t] = r;
    mr[t] = vals[e];
    c2r[e] = t;
  }
  upload(s, csc_colptr, colptr);
  upload(s, csc_row, crow);
  upload(s, csr_rowptr, rowptr);
  upload(s, csr_col, rcol);
  upload(s, csr_row, rrow);
  upload(s, m_csc, mc);
  upload(s, m_csr, mr);
  upload(s, csc2csr, c2r);
  // Segment length: long enough that a typical structure row is one segment (no partial-sum
  // reduction pass), short enough that the longest rows still spread over several warps.
  auto seg_for = [](i64 rows, i64 nnz) {
    const i64 avg = rows > 0 ? (nnz + rows - 1) / rows : 1;
    return avg <= 128 ? 128 : 64;
  };
  build_plan(s, plan_csr, m, rowptr, seg_for(m, nnz));
  build_plan(s, plan_csc, n, colptr, seg_for(n, nnz));
  has_empty_csr = has_empty_csc = false;
  for (i64 r = 0; r < m; ++r) has_empty_csr |= rowptr[r + 1] == rowptr[r];
  for (i64 c = 0; c < n; ++c) has_empty_csc |= colptr[c + 1] == colptr[c];
  // column-tile offsets of every CSR row (tiled SDDMM), when the table stays small
  const i64 tiles = (n + kTileCols - 1) / kTileCols;
  if (m * (tiles + 1) <= (i64{1} << 26)) {
    ntc = static_cast<int>(tiles);
    std::vector<int> h(static_cast<size_t>(m * (tiles + 1)));
    for (i64 r = 0; r < m; ++r) {
      int e = rowptr[r];
      for (i64 q = 0; q <= tiles; ++q) {
        const long long lim = q * kTileCols;
        while (e < rowptr[r + 1] && rcol[e] < lim) ++e;
        h[static_cast<size_t>(r * (tiles + 1) + q)] = q == tiles ? rowptr[r + 1] : e;
      }
    }
    upload(s, tile_csr, h);
    DFCG_CUDA(cudaStreamSynchronize(s));
    if (ntc > 2 * kChunkTiles) build_chunked_plan(s, plan_csr_ck, m, h, ntc, seg_for(m, nnz));
  }
  // row-tile offsets of every CSC column (rows ascend within a column)
  const i64 rtiles = (m + kTileCols - 1) / kTileCols;
  if (n * (rtiles + 1) <= (i64{1} << 26)) {
    ntr = static_cast<int>(rtiles);
    std::vector<int> h(static_cast<size_t>(n * (rtiles + 1)));
    for (i64 c = 0; c < n; ++c) {
      int e = colptr[c];
      for (i64 q = 0; q <= rtiles; ++q) {
        const long long lim = q * kTileCols;
        while (e < colptr[c + 1] && crow[e] < lim) ++e;
        h[static_cast<size_t>(c * (rtiles + 1) + q)] = q == rtiles ? colptr[c + 1] : e;
      }
    }
    upload(s, tile_csc, h);
    DFCG_CUDA(cudaStreamSynchronize(s));
    if (ntr > 2 * kChunkTiles) build_chunked_plan(s, plan_csc_ck, n, h, ntr, seg_for(n, nnz));
  }
  h_csc2csr = std::move(c2r);
}

void sddmm_residual(cudaStream_t s, const DevOmega& om, i64 kY, const double* Yl, i64 ldl, const double* Yr, i64 ldr,
                    const double* sub, double* r_csr) {
  if (om.nnz == 0) return;
  // algorithmic bytes: row+col index, M_e, r_e per entry + both factors once
  prof::Scope scope(prof::kSddmm, s, 2.0 * kY * om.nnz, 24.0 * om.nnz + 8.0 * (om.m + om.n) * kY);
  const char* tile_env = std::getenv("DFCG_SDDMM_TILE");  // 0 / 1 force the entry-parallel / tiled kernel
  const int tile_mode = tile_env ? std::atoi(tile_env) : -1;
  // slab SDDMM: measured slower than the tiled kernel (tools/bench_sparse.py, profiles/
  // r02_bench_sparse.txt: 1038 vs 439 us at the c5 block), so opt-in (DFCG_SDDMM_SLAB=1)
  static const int slab_env0 = std::getenv("DFCG_SDDMM_SLAB") ? std::atoi(std::getenv("DFCG_SDDMM_SLAB")) : 0;
  const int slab_env = g_sddmm_mode.load() >= 0 ? g_sddmm_mode.load() : slab_env0;
  if (om.ntc > 0 && tile_mode == -1 && slab_env != 0 && kY >= 1 && kY <= 64) {
    int G = 1;
    while (4 * G < kY) G *= 2;
    const int BP = 4 * G;
    const int SB = std::max(64, std::min(1024, static_cast<int>((150 * 1024 / (2 * 8 * BP)) / 64 * 64)));
    int dev = 0, nsm = 148;
    DFCG_CUDA(cudaGetDevice(&dev));
    DFCG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int R = (om.m + 16 * 8 - 1) / (16 * 8) >= nsm ? 8 : 4;
    const unsigned grid = static_cast<unsigned>((om.m + SLAB_WARPS * R - 1) / (SLAB_WARPS * R));
    const size_t smem = sizeof(double) * 2 * SB * BP;
    static std::atomic<std::uint64_t> configured{0};
    if (!(configured.load() & dev_bit(dev))) {
#define SDS_ATTR(r, g) \
  DFCG_CUDA(cudaFuncSetAttribute(sddmm_slab_kernel<r, g>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
      SDS_ATTR(4, 1) SDS_ATTR(4, 2) SDS_ATTR(4, 4) SDS_ATTR(4, 8) SDS_ATTR(4, 16)
      SDS_ATTR(8, 1) SDS_ATTR(8, 2) SDS_ATTR(8, 4) SDS_ATTR(8, 8) SDS_ATTR(8, 16)
#undef SDS_ATTR
      configured.fetch_or(dev_bit(dev));
    }
#define SDS_CASE(r, g)                                                                                       \
  if (R == r && G == g)                                                                                      \
    sddmm_slab_kernel<r, g><<<grid, SLAB_WARPS * 32, smem, s>>>(om.m, om.n, static_cast<int>(kY), om.ntc, SB, \
                                                                om.tile_csr.get(), om.csr_col.get(), Yl, ldl, Yr,  \
                                                                ldr, sub, r_csr);
    SDS_CASE(4, 1) SDS_CASE(4, 2) SDS_CASE(4, 4) SDS_CASE(4, 8) SDS_CASE(4, 16)
    SDS_CASE(8, 1) SDS_CASE(8, 2) SDS_CASE(8, 4) SDS_CASE(8, 8) SDS_CASE(8, 16)
#undef SDS_CASE
    DFCG_LAUNCH_CHECK();
    return;
  }
  if (om.ntc > 0 && tile_mode != 0) {
    static std::atomic<std::uint64_t> configured{0};  // one bit per device
    int dev = 0;
    DFCG_CUDA(cudaGetDevice(&dev));
    if (!(configured.load() & dev_bit(dev))) {
      DFCG_CUDA(cudaFuncSetAttribute(sddmm_tile_kernel<1, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(sddmm_smem<1, 32>())));
      DFCG_CUDA(cudaFuncSetAttribute(sddmm_tile_kernel<4, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(sddmm_smem<4, 16>())));
      configured.fetch_or(dev_bit(dev));
    }
    // 16-byte staging needs even leading dimensions and an even k extent: repack the factors
    // (a few tens of microseconds) unless they already qualify; the padding column is zero.
    const i64 k2 = (kY + 1) & ~i64{1};
    DBuf<double> pl, pr;
    const bool aligned = (ldl % 2 == 0) && (ldr % 2 == 0) && k2 == kY &&
                         (reinterpret_cast<std::uintptr_t>(Yl) % 16 == 0) &&
                         (reinterpret_cast<std::uintptr_t>(Yr) % 16 == 0);
    if (!aligned) {
      pl.alloc(om.m * k2, s);
      pr.alloc(om.n * k2, s);
      if (k2 != kY) {
        pl.zero(s);
        pr.zero(s);
      }
      copy2d(s, om.m, kY, Yl, ldl, pl.get(), k2);
      copy2d(s, om.n, kY, Yr, ldr, pr.get(), k2);
      Yl = pl.get();
      Yr = pr.get();
      ldl = ldr = k2;
    }
    static const int tw_env = std::getenv("DFCG_SDDMM_TW") ? std::atoi(std::getenv("DFCG_SDDMM_TW")) : 0;
    const bool wide = tw_env == 4;
    const unsigned gy = static_cast<unsigned>((om.m + STR - 1) / STR);
    // Tile width at kY <= 32 (16-wide k chunks): 64 x 128 tiles (49 KB of shared memory, four CTAs
    // per SM) — the tiled kernel is latency-bound (ncu: no pipe above 45 %, occupancy 24 % with
    // the 82 KB 64 x 256 tiles, profiles/r02_ncu_sddmm_c5.txt), and the narrower tile measured
    // 336 vs 435 us at the c5 block and 26.8 vs 34.9 us at the c2 block; 64 x 64 tiles (434 /
    // 28.8 us), 64 x 192 (461 / 35.6 us) and single-buffered 32-wide chunks (406-502 us) are
    // slower (profiles/r02_bench_sddmm_tiles.txt). DFCG_SDDMM_TW=4 keeps 64 x 256, 1 forces
    // the 64 x 64 / 32-wide kernel of kY > 32.
    if (tw_env ? tw_env == 2 : k2 <= 32) {
      static std::atomic<std::uint64_t> cfg2{0};
      if (!(cfg2.load() & dev_bit(dev))) {
        DFCG_CUDA(cudaFuncSetAttribute(sddmm_tile_kernel<2, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(sddmm_smem<2, 16>())));
        cfg2.fetch_or(dev_bit(dev));
      }
      sddmm_tile_kernel<2, 16><<<dim3((om.ntc + 1) / 2, gy), SDD_T, sddmm_smem<2, 16>(), s>>>(
          om.m, om.n, k2, om.ntc, om.tile_csr.get(), om.csr_col.get(), Yl, ldl, Yr, ldr, sub, r_csr);
    } else if (wide)
      sddmm_tile_kernel<4, 16><<<dim3((om.ntc + 3) / 4, gy), SDD_T, sddmm_smem<4, 16>(), s>>>(
          om.m, om.n, k2, om.ntc, om.tile_csr.get(), om.csr_col.get(), Yl, ldl, Yr, ldr, sub, r_csr);
    else
      sddmm_tile_kernel<1, 32><<<dim3(om.ntc, gy), SDD_T, sddmm_smem<1, 32>(), s>>>(
          om.m, om.n, k2, om.ntc, om.tile_csr.get(), om.csr_col.get(), Yl, ldl, Yr, ldr, sub, r_csr);
    DFCG_LAUNCH_CHECK();
    return;
  }
  const int G = pow2_at_least((kY + 3) / 4);
  const i64 warps = (om.nnz + (32 / G) - 1) / (32 / G);
  const int blocks = static_cast<int>(std::min<i64>((warps + 7) / 8, 65535L * 4));
#define SDDMM_CASE(g)                                                                                        \
  case g:                                                                                                    \
    sddmm_kernel<g><<<blocks, 256, 0, s>>>(om.nnz, kY, om.csr_row.get(), om.csr_col.get(), Yl, ldl, Yr, ldr, \
                                           sub, r_csr);                                                      \
    break;
  switch (G) {
    SDDMM_CASE(1)
    SDDMM_CASE(2)
    SDDMM_CASE(4)
    SDDMM_CASE(8)
    SDDMM_CASE(16)
    SDDMM_CASE(32)
  }
#undef SDDMM_CASE
  DFCG_LAUNCH_CHECK();
}

void spmm(cudaStream_t s, const DevOmega& om, bool transpose, const double* vals_csr, i64 b, double alpha,
          const double* X, i64 ldx, double beta, double* out, i64 ldo, const double* vals_csc) {
  const SegPlan& p = transpose ? om.plan_csc : om.plan_csr;
  const i64 out_rows = transpose ? om.n : om.m;
  if (b <= 0 || out_rows <= 0) return;
  const int* ptr = transpose ? om.csc_colptr.get() : om.csr_rowptr.get();
  // algorithmic bytes: idx + value (+ permutation) per entry, X read once, out written (read if beta)
  const i64 in_rows = transpose ? om.m : om.n;
  prof::Scope scope(prof::kSpmm, s, 2.0 * om.nnz * b,
                    (transpose ? 20.0 : 12.0) * om.nnz + 8.0 * b * (in_rows + out_rows * (beta != 0.0 ? 2 : 1)));
  {  // slab kernel: b <= 64, the tile table of the walk, CSC values streamed (transpose)
    // slab SpMM: measured slower than the segmented gather kernel (tools/bench_sparse.py,
    // profiles/r02_bench_sparse.txt: 568 vs 280 us at the c5 block — 16 warps per SM with a
    // dependent entry load per line and slab hide too little latency), so opt-in (DFCG_SPMM_SLAB=1)
    static const int slab_env0 = std::getenv("DFCG_SPMM_SLAB") ? std::atoi(std::getenv("DFCG_SPMM_SLAB")) : 0;
    const int slab_env = g_spmm_mode.load() >= 0 ? (g_spmm_mode.load() == 1 ? 1 : 0) : slab_env0;
    const int nt = transpose ? om.ntr : om.ntc;
    const double* tv = transpose ? vals_csc : vals_csr;
    if (slab_env != 0 && b >= 1 && b <= 64 && nt > 0 && tv) {
      const int* tptr = transpose ? om.tile_csc.get() : om.tile_csr.get();
      const int* tidx = transpose ? om.csc_row.get() : om.csr_col.get();
      const int G = static_cast<int>((b + 3) / 4), BP = 4 * G;
      // slab rows: two buffers within ~150 KB of shared memory, a multiple of the 64-row tiles
      const int SB = std::max(64, std::min(512, static_cast<int>((150 * 1024 / (2 * 8 * BP)) / 64 * 64)));
      int nsm = 148;
      {
        int dev = 0;
        DFCG_CUDA(cudaGetDevice(&dev));
        DFCG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
      }
      // 4 lines per warp (64 per CTA, one CTA per SM); the inner dimension is split into chunks
      // of whole slabs so the grid fills whole waves (>= 85% of the last) or reaches >= 4 waves
      const int R = 4;
      const i64 outer_blocks = (out_rows + SLAB_WARPS * R - 1) / (SLAB_WARPS * R);
      const int TPS = SB / DevOmega::kTileCols;
      const int max_chunks = std::max(1, (nt + TPS - 1) / TPS);
      int chunks = 1;
      {
        double best = -1.0;
        for (int c = 1; c <= std::min(max_chunks, 64); ++c) {
          const i64 tot = outer_blocks * c;
          const i64 waves = (tot + nsm - 1) / nsm;
          const double eff = static_cast<double>(tot) / static_cast<double>(waves * nsm);
          const double score = eff - (waves > 8 ? 0.01 * (waves - 8) : 0.0);
          if (score > best + 1e-9) best = score, chunks = c;
          if (waves >= 4 && eff >= 0.85) break;
        }
      }
      const int chunk_tiles = ((nt + chunks - 1) / chunks + TPS - 1) / TPS * TPS;
      chunks = (nt + chunk_tiles - 1) / chunk_tiles;
      const size_t smem = sizeof(double) * 2 * SB * BP;
      static std::atomic<std::uint64_t> configured{0};
      int dev = 0;
      DFCG_CUDA(cudaGetDevice(&dev));
      if (!(configured.load() & dev_bit(dev))) {
        DFCG_CUDA(cudaFuncSetAttribute(spmm_slab_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        configured.fetch_or(dev_bit(dev));
      }
      DBuf<double> ws;
      if (chunks > 1) ws.alloc(static_cast<i64>(chunks) * out_rows * b, s);
      const dim3 grid(static_cast<unsigned>(outer_blocks), static_cast<unsigned>(chunks));
      spmm_slab_kernel<4><<<grid, SLAB_WARPS * 32, smem, s>>>(out_rows, in_rows, nt, tptr, tidx, tv,
                                                                 static_cast<int>(b), G, SB, alpha, X, ldx, beta, out,
                                                                 ldo, chunk_tiles, chunks > 1 ? ws.get() : nullptr);
      DFCG_LAUNCH_CHECK();
      if (chunks > 1) {
        spmm_chunk_reduce<<<grid_for(out_rows * b), 256, 0, s>>>(out_rows, static_cast<int>(b), chunks, ws.get(),
                                                                 alpha, beta, out, ldo);
        DFCG_LAUNCH_CHECK();
      }
      return;
    }
  }
  if (transpose ? om.has_empty_csc : om.has_empty_csr) {  // rows with no entries: out = beta out
    empty_rows_kernel<<<grid_for(out_rows * b), 256, 0, s>>>(out_rows, ptr, b, beta, out, ldo);
    DFCG_LAUNCH_CHECK();
  }
  if (p.n_items == 0) return;
  // chunked (cache-blocked) plan of the same walk when it exists: opt-in (DFCG_SPMM_CHUNK=1), it
  // measured slower than the plain walk (c5 block: 305 vs 281 us forward, 334 vs 260 us
  // transposed; profiles/r02_bench_sparse2.txt): the gather kernel is bound by L1 wavefronts per
  // entry, not by L2 misses, so keeping the X chunk L1-resident does not help
  static const int chunk_env = std::getenv("DFCG_SPMM_CHUNK") ? std::atoi(std::getenv("DFCG_SPMM_CHUNK")) : 0;
  const int mode = g_spmm_mode.load();
  const SegPlan& pc = transpose ? om.plan_csc_ck : om.plan_csr_ck;
  const bool chunked = pc.n_items > 0 && (mode >= 0 ? mode == 2 || mode == 4 : chunk_env != 0);
  const SegPlan& pp = chunked ? pc : p;
  DBuf<double> ws;
  if (pp.n_slots) ws.alloc(pp.n_slots * b, s);
  // 16-byte variant (spmm16_kernel): CSC-ordered values streamed (no permutation gather), even
  // ldx >= b + (b & 1), 16-byte aligned X. Opt-in (DFCG_SPMM16=1; bench modes 3 / 4): measured
  // slower at the c5 block (355 vs 275 us forward, 306 vs 253 us transposed — the shuffles go
  // through the same data pipe as the loads they replace) and level at the c2 block (38.8 vs
  // 39.0 us, 39.1 vs 45.5 us transposed); profiles/r02_bench_sparse16.txt.
  static const int v16_env = std::getenv("DFCG_SPMM16") ? std::atoi(std::getenv("DFCG_SPMM16")) : 0;
  const bool use16 = (mode >= 0 ? mode == 3 || mode == 4 : v16_env != 0) &&
                     !(transpose && !vals_csc) && ldx % 2 == 0 && ldx >= b + (b & 1) &&
                     reinterpret_cast<std::uintptr_t>(X) % 16 == 0;
  if (use16) {
    const int G16 = pow2_at_least((((b + 1) >> 1) + 1) / 2);  // 2 double2 chunks per lane per pass
    const i64 warps16 = (pp.n_items + (32 / G16) - 1) / (32 / G16);
    const int blocks16 = static_cast<int>((warps16 + 7) / 8);
    const int* idx16 = transpose ? om.csc_row.get() : om.csr_col.get();
    const double* vals16 = transpose ? vals_csc : vals_csr;
#define SPMM16_CASE(g)                                                                                              \
  case g:                                                                                                           \
    if (transpose)                                                                                                  \
      spmm16_kernel<g, true><<<blocks16, 256, 0, s>>>(pp.n_items, pp.items.get(), idx16, vals16, b, alpha, X, ldx,  \
                                                       beta, out, ldo, ws.get());                                   \
    else                                                                                                            \
      spmm16_kernel<g, false><<<blocks16, 256, 0, s>>>(pp.n_items, pp.items.get(), idx16, vals16, b, alpha, X, ldx, \
                                                        beta, out, ldo, ws.get());                                  \
    break;
    switch (G16) {
      SPMM16_CASE(1)
      SPMM16_CASE(2)
      SPMM16_CASE(4)
      SPMM16_CASE(8)
      SPMM16_CASE(16)
      SPMM16_CASE(32)
    }
#undef SPMM16_CASE
    DFCG_LAUNCH_CHECK();
    if (!pp.h_multi_rows.empty()) {
      const i64 nr = static_cast<i64>(pp.h_multi_rows.size());
      seg_reduce_kernel<<<grid_for(nr * b), 256, 0, s>>>(nr, pp.multi_rows.get(), pp.red_rowptr.get(), b, ws.get(),
                                                         alpha, beta, out, ldo);
      DFCG_LAUNCH_CHECK();
    }
    return;
  }
  // Wide variant (bench mode 5 / DFCG_SPMM_WIDE=1): 2 columns per lane, so b = 35 takes one item per
  // warp (32 contiguous lanes on the row's first 256 bytes) instead of two half-warp items.
  static const int wide_env = std::getenv("DFCG_SPMM_WIDE") ? std::atoi(std::getenv("DFCG_SPMM_WIDE")) : 0;
  if (mode >= 0 ? mode == 5 : wide_env != 0) {
    const int GW = pow2_at_least((b + 1) / 2);
    const i64 warpsw = (pp.n_items + (32 / GW) - 1) / (32 / GW);
    const int blocksw = static_cast<int>((warpsw + 7) / 8);
    const int* idxw = transpose ? om.csc_row.get() : om.csr_col.get();
    const double* valsw = transpose && vals_csc ? vals_csc : vals_csr;
    const long long* permw = transpose && !vals_csc ? om.csc2csr.get() : nullptr;
#define SPMMW_CASE(g)                                                                                              \
  case g:                                                                                                          \
    if (transpose)                                                                                                 \
      spmm_kernel<g, true, 2><<<blocksw, 256, 0, s>>>(pp.n_items, pp.items.get(), idxw, permw, valsw, b, alpha, X,  \
                                                       ldx, beta, out, ldo, ws.get());                             \
    else                                                                                                           \
      spmm_kernel<g, false, 2><<<blocksw, 256, 0, s>>>(pp.n_items, pp.items.get(), idxw, permw, valsw, b, alpha, X, \
                                                        ldx, beta, out, ldo, ws.get());                            \
    break;
    switch (GW) {
      SPMMW_CASE(1)
      SPMMW_CASE(2)
      SPMMW_CASE(4)
      SPMMW_CASE(8)
      SPMMW_CASE(16)
      SPMMW_CASE(32)
    }
#undef SPMMW_CASE
    DFCG_LAUNCH_CHECK();
    if (!pp.h_multi_rows.empty()) {
      const i64 nr = static_cast<i64>(pp.h_multi_rows.size());
      seg_reduce_kernel<<<grid_for(nr * b), 256, 0, s>>>(nr, pp.multi_rows.get(), pp.red_rowptr.get(), b, ws.get(),
                                                         alpha, beta, out, ldo);
      DFCG_LAUNCH_CHECK();
    }
    return;
  }
  // lanes per item: enough for one pass over the b columns at kSpmmCpl columns per lane
  const int G = pow2_at_least((b + kSpmmCpl - 1) / kSpmmCpl);
  const i64 warps = (pp.n_items + (32 / G) - 1) / (32 / G);
  const int blocks = static_cast<int>((warps + 7) / 8);
  const int* idx = transpose ? om.csc_row.get() : om.csr_col.get();
  // the transposed walk streams CSC-ordered values when the caller has them, else it gathers
  // the CSR values through the permutation (random 8-byte reads)
  const double* vals = transpose && vals_csc ? vals_csc : vals_csr;
  const long long* perm = transpose && !vals_csc ? om.csc2csr.get() : nullptr;
#define SPMM_CASE(g)                                                                                               \
  case g:                                                                                                          \
    if (transpose)                                                                                                 \
      spmm_kernel<g, true><<<blocks, 256, 0, s>>>(pp.n_items, pp.items.get(), idx, perm, vals, b, alpha, X, ldx,     \
                                                   beta, out, ldo, ws.get());                                      \
    else                                                                                                           \
      spmm_kernel<g, false><<<blocks, 256, 0, s>>>(pp.n_items, pp.items.get(), idx, perm, vals, b, alpha, X,         \
                                                    ldx, beta, out, ldo, ws.get());                                \
    break;
  switch (G) {
    SPMM_CASE(1)
    SPMM_CASE(2)
    SPMM_CASE(4)
    SPMM_CASE(8)
    SPMM_CASE(16)
    SPMM_CASE(32)
  }
#undef SPMM_CASE
  DFCG_LAUNCH_CHECK();
  if (!pp.h_multi_rows.empty()) {
    const i64 nr = static_cast<i64>(pp.h_multi_rows.size());
    seg_reduce_kernel<<<grid_for(nr * b), 256, 0, s>>>(nr, pp.multi_rows.get(), pp.red_rowptr.get(), b, ws.get(), alpha,
                                                       beta, out, ldo);
    DFCG_LAUNCH_CHECK();
  }
}

__global__ void csr_to_csc_kernel(i64 N, const long long* __restrict__ csc2csr, const double* __restrict__ src,
                                  double* __restrict__ dst) {
  for (i64 t = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; t < N;
       t += static_cast<i64>(gridDim.x) * blockDim.x)
    dst[t] = src[csc2csr[t]];
}

void csr_to_csc(cudaStream_t s, const DevOmega& om, const double* vals_csr, double* vals_csc) {
  if (om.nnz == 0) return;
  prof::Scope scope(prof::kElementwise, s, 0.0, 24.0 * om.nnz);
  csr_to_csc_kernel<<<grid_for(om.nnz), 256, 0, s>>>(om.nnz, om.csc2csr.get(), vals_csr, vals_csc);
  DFCG_LAUNCH_CHECK();
}

void scatter_add_dense(cudaStream_t s, const DevOmega& om, const double* vals_csr, double alpha, double* D, i64 ldd) {
  if (om.nnz == 0) return;
  scatter_dense_kernel<<<grid_for(om.nnz), 256, 0, s>>>(om.nnz, om.csr_row.get(), om.csr_col.get(), vals_csr, alpha,
                                                         D, ldd);
  DFCG_LAUNCH_CHECK();
}

}  // namespace dfcg
