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
template <int G, bool T>
__global__ void spmm_kernel(i64 n_items, const SegItem* __restrict__ items, const int* __restrict__ idx,
                            const long long* __restrict__ perm, const double* __restrict__ vals, i64 b, double alpha,
                            const double* __restrict__ X, i64 ldx, double beta, double* __restrict__ out, i64 ldo,
                            double* __restrict__ ws) {
  constexpr int PER_WARP = 32 / G;
  const int lane = threadIdx.x & 31, lig = lane % G;
  const i64 gid = ((static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * PER_WARP + lane / G;
  if (gid >= n_items) return;
  const SegItem it = items[gid];
  constexpr int CPL = kSpmmCpl;  // columns per lane per pass: one walk of the segment covers CPL G columns
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

// Tiled SpMM (experimental, see spmm()) for sketches up to 64 columns: out[o, :] (+)= alpha sum_e v_e X[idx_e, :] over the
// entries e of outer line o (a CSR row for R X, a CSC column for R^T X). One CTA per 128 outer
// lines (16 warps x 8 lines, accumulators in registers: lane l holds columns l and l + 32) and
// one chunk of the inner dimension; the chunk's X rows stream through shared memory 256 at a
// time, so X is read from L2 once per 128 lines instead of once per entry (the segmented kernel
// gathers a b-wide X row per entry: L2-bound, ~10% of the HBM roofline at the c5 block). Each
// line's entries of a 256-row X slab are one contiguous range of the per-line 64-tile table.
// Deterministic: a line's entries are summed in storage order; chunk partials (ws, when the
// inner dimension is split for parallelism) are combined in chunk order by spmm_chunk_reduce.
constexpr int TSP_LINES = 8, TSP_WARPS = 16, TSP_OB = TSP_LINES * TSP_WARPS, TSP_SLAB = 256;

__global__ void __launch_bounds__(TSP_WARPS * 32)
    spmm_tile_kernel(i64 n_outer, i64 n_inner, int nt, const int* __restrict__ tptr, const int* __restrict__ idx,
                     const double* __restrict__ vals, int b, double alpha, const double* __restrict__ X, i64 ldx,
                     double beta, double* __restrict__ out, i64 ldo, int chunk_tiles, double* __restrict__ ws) {
  extern __shared__ double xs[];  // [TSP_SLAB][b]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const i64 o0 = static_cast<i64>(blockIdx.x) * TSP_OB + warp * TSP_LINES;
  const int q_begin = blockIdx.y * chunk_tiles, q_end = min(nt, q_begin + chunk_tiles);
  constexpr int TPS = TSP_SLAB / DevOmega::kTileCols;  // 64-tiles per slab
  double acc[TSP_LINES][2];
#pragma unroll
  for (int r = 0; r < TSP_LINES; ++r) acc[r][0] = acc[r][1] = 0.0;
  const bool c1 = lane + 32 < b;
  for (int q0 = q_begin; q0 < q_end; q0 += TPS) {
    const int q1 = min(q_end, q0 + TPS);
    const i64 in0 = static_cast<i64>(q0) * DevOmega::kTileCols;
    const int rows_in = static_cast<int>(min(static_cast<i64>(q1 - q0) * DevOmega::kTileCols, n_inner - in0));
    __syncthreads();  // the previous slab is consumed
    // asynchronous 8-byte copies: no register round trip, every load in flight at once
    for (int e = t; e < rows_in * b; e += blockDim.x) {
      const int r = e / b, c = e - r * b;
      cp_async8(xs + e, X + (in0 + r) * ldx + c, true);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    // the warp's 8 lines: slab ranges [e0, e1) via two table loads per line (lanes 0-15), and
    // each line's first 32 entries loaded up front, one per lane (coalesced); the FMAs then take
    // (index, value) by shuffle — no dependent global load inside the entry loop
    int tv = 0;
    if (lane < 2 * TSP_LINES) {
      const i64 o = o0 + (lane & (TSP_LINES - 1));
      tv = o < n_outer ? tptr[o * (nt + 1) + (lane < TSP_LINES ? q0 : q1)] : 0;
    }
    int e0[TSP_LINES], e1[TSP_LINES], ix0[TSP_LINES];
    double v0[TSP_LINES];
#pragma unroll
    for (int r = 0; r < TSP_LINES; ++r) {
      e0[r] = __shfl_sync(0xffffffffu, tv, r);
      e1[r] = __shfl_sync(0xffffffffu, tv, TSP_LINES + r);
      const int e = e0[r] + lane;
      ix0[r] = 0;
      v0[r] = 0.0;
      if (e < e1[r]) {
        ix0[r] = static_cast<int>(idx[e] - in0);
        v0[r] = vals[e];
      }
    }
#pragma unroll
    for (int r = 0; r < TSP_LINES; ++r) {
      const int cnt_all = e1[r] - e0[r];
      for (int base = 0; base < cnt_all; base += 32) {
        int ixc = ix0[r];
        double vc = v0[r];
        if (base > 0) {  // lines with more than 32 entries in this slab
          const int e = e0[r] + base + lane;
          ixc = 0;
          vc = 0.0;
          if (e < e1[r]) {
            ixc = static_cast<int>(idx[e] - in0);
            vc = vals[e];
          }
        }
        const int cnt = min(32, cnt_all - base);
        for (int jj = 0; jj < cnt; ++jj) {
          const double* xr = xs + __shfl_sync(0xffffffffu, ixc, jj) * b;
          const double v = __shfl_sync(0xffffffffu, vc, jj);
          acc[r][0] = fma(v, lane < b ? xr[lane] : 0.0, acc[r][0]);
          if (c1) acc[r][1] = fma(v, xr[lane + 32], acc[r][1]);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < TSP_LINES; ++r) {
    const i64 o = o0 + r;
    if (o >= n_outer) break;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      if (c >= b) continue;
      if (ws) {
        ws[(static_cast<i64>(blockIdx.y) * n_outer + o) * b + c] = acc[r][h];
      } else {
        double* p = out + o * ldo + c;
        *p = beta == 0.0 ? alpha * acc[r][h] : fma(beta, *p, alpha * acc[r][h]);
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

template <class T>
void upload(cudaStream_t s, DBuf<T>& d, const std::vector<T>& h) {
  d.alloc(std::max<size_t>(1, h.size()), s);
  if (!h.empty()) DFCG_CUDA(cudaMemcpyAsync(d.get(), h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, s));
}

}  // namespace

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
    const bool wide = tw_env ? tw_env == 4 : k2 <= 32;
    const unsigned gy = static_cast<unsigned>((om.m + STR - 1) / STR);
    if (wide)
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
  {  // tiled kernel: 2 <= b <= 64, the tile table of the walk, CSC values streamed (transpose)
    // Experimental (DFCG_SPMM_TILE=1): measured slower than the segmented kernel at the c5 block
    // (567 vs 273 us per call at b = 35, N = 1e7: one CTA per SM at 126 registers, slab staging
    // and the per-slab barriers are not overlapped with the entry loop), so off by default.
    static const bool tiled_env = std::getenv("DFCG_SPMM_TILE") && std::atoi(std::getenv("DFCG_SPMM_TILE")) == 1;
    const int nt = transpose ? om.ntr : om.ntc;
    const double* tv = transpose ? vals_csc : vals_csr;
    if (tiled_env && b >= 2 && b <= 64 && nt > 0 && tv) {
      const int* tptr = transpose ? om.tile_csc.get() : om.tile_csr.get();
      const int* tidx = transpose ? om.csc_row.get() : om.csr_col.get();
      const i64 outer_blocks = (out_rows + TSP_OB - 1) / TSP_OB;
      // split the inner dimension until the grid covers ~2 CTAs per SM (chunks of >= one slab)
      const int max_chunks = std::max(1, (nt + 3) / 4);
      int chunks = static_cast<int>(std::min<i64>(max_chunks, std::max<i64>(1, (2 * 148 + outer_blocks - 1) / outer_blocks)));
      const int chunk_tiles = (nt + chunks - 1) / chunks;
      chunks = (nt + chunk_tiles - 1) / chunk_tiles;
      const size_t smem = sizeof(double) * TSP_SLAB * b;
      static std::atomic<std::uint64_t> configured{0};
      int dev = 0;
      DFCG_CUDA(cudaGetDevice(&dev));
      if (!(configured.load() & dev_bit(dev))) {
        DFCG_CUDA(cudaFuncSetAttribute(spmm_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(sizeof(double) * TSP_SLAB * 64)));
        configured.fetch_or(dev_bit(dev));
      }
      DBuf<double> ws;
      if (chunks > 1) ws.alloc(static_cast<i64>(chunks) * out_rows * b, s);
      spmm_tile_kernel<<<dim3(static_cast<unsigned>(outer_blocks), static_cast<unsigned>(chunks)), TSP_WARPS * 32,
                         smem, s>>>(out_rows, in_rows, nt, tptr, tidx, tv, static_cast<int>(b), alpha, X, ldx, beta,
                                    out, ldo, chunk_tiles, chunks > 1 ? ws.get() : nullptr);
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
  DBuf<double> ws;
  if (p.n_slots) ws.alloc(p.n_slots * b, s);
  // lanes per item: enough for one pass over the b columns at kSpmmCpl columns per lane
  const int G = pow2_at_least((b + kSpmmCpl - 1) / kSpmmCpl);
  const i64 warps = (p.n_items + (32 / G) - 1) / (32 / G);
  const int blocks = static_cast<int>((warps + 7) / 8);
  const int* idx = transpose ? om.csc_row.get() : om.csr_col.get();
  // the transposed walk streams CSC-ordered values when the caller has them, else it gathers
  // the CSR values through the permutation (random 8-byte reads)
  const double* vals = transpose && vals_csc ? vals_csc : vals_csr;
  const long long* perm = transpose && !vals_csc ? om.csc2csr.get() : nullptr;
#define SPMM_CASE(g)                                                                                               \
  case g:                                                                                                          \
    if (transpose)                                                                                                 \
      spmm_kernel<g, true><<<blocks, 256, 0, s>>>(p.n_items, p.items.get(), idx, perm, vals, b, alpha, X, ldx,     \
                                                   beta, out, ldo, ws.get());                                      \
    else                                                                                                           \
      spmm_kernel<g, false><<<blocks, 256, 0, s>>>(p.n_items, p.items.get(), idx, perm, vals, b, alpha, X,         \
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
  if (!p.h_multi_rows.empty()) {
    const i64 nr = static_cast<i64>(p.h_multi_rows.size());
    seg_reduce_kernel<<<grid_for(nr * b), 256, 0, s>>>(nr, p.multi_rows.get(), p.red_rowptr.get(), b, ws.get(), alpha,
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
