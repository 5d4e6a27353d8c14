// Sparse kernels for the observed set Omega (see sparse.cuh).
//
// SDDMM: entry-parallel over the CSR stream, G lanes per entry (G ~ kY/4, power of two),
// factor rows gathered contiguously (row-major factors), group reduction by xor-shuffles.
// SpMM: segmented work list (<= SEG entries per item) so long CSC columns split across
// warps; multi-segment rows reduce their partials in a fixed order (deterministic).
#include <algorithm>

#include "sparse.cuh"

namespace dfcg {

namespace {

constexpr int SEG = 64;
// The chunked path re-walks every nonzero once per 16-column chunk; measured 2x slower than
// the segmented kernel at b ~ 700 (ncu: instruction-bound), so it is disabled for now.
constexpr i64 kSlabMinB = i64{1} << 40;

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
  constexpr int CPL = 4;  // columns per lane per pass: one walk of the segment covers 4 G columns
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
        vv[u] = T ? vals[perm[e + u]] : vals[e + u];
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
      const double v = T ? vals[perm[e]] : vals[e];
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

// Shared-memory-chunked SpMM for wide sketches: CTA (chunk c, slab q, row split) stages
// X[q*H : (q+1)*H, 16c : 16c+16] in shared memory once and streams its structure rows'
// entries against it (half-warp per output row, lane = column), so each X element is read
// from L2 once per CTA instead of once per nonzero. Partial sums per slab when ns > 1.
constexpr int CW = 16, SLAB_THREADS = 512;
template <bool T>
__global__ void __launch_bounds__(SLAB_THREADS) spmm_slab_kernel(i64 rows, int ns, int rsplit,
                                                                 const int* __restrict__ slab,
                                                                 const int* __restrict__ idx,
                                                                 const long long* __restrict__ perm,
                                                                 const double* __restrict__ vals, i64 in_rows, i64 b,
                                                                 double alpha, const double* __restrict__ X, i64 ldx,
                                                                 double beta, double* __restrict__ out, i64 ldo,
                                                                 double* __restrict__ ws) {
  extern __shared__ double xs[];  // H x CW
  constexpr int H = DevOmega::kSlabRows, NW = SLAB_THREADS / 32;
  const int c = blockIdx.x, q = blockIdx.y, split = blockIdx.z;
  const i64 c0 = static_cast<i64>(c) * CW, s0 = static_cast<i64>(q) * H;
  const i64 h = min(static_cast<i64>(H), in_rows - s0);
  const int w = static_cast<int>(min(static_cast<i64>(CW), b - c0));
  for (i64 e = threadIdx.x; e < h * CW; e += blockDim.x) {
    const i64 r = e / CW;
    const int cc = static_cast<int>(e % CW);
    xs[e] = cc < w ? X[(s0 + r) * ldx + c0 + cc] : 0.0;
  }
  __syncthreads();
  // warp per structure row: the row's entries are fetched 32 at a time (coalesced, one per
  // lane) and broadcast by shuffles; half-warp hh takes entries j + 16 hh of each batch, lane
  // column = lane & 15; the two halves are combined at the end (fixed order).
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, col = lane & 15, hh = lane >> 4;
  const i64 per = (rows + rsplit - 1) / rsplit;
  const i64 rb = static_cast<i64>(split) * per, re = min(rows, rb + per);
  for (i64 r = rb + warp; r < re; r += NW) {
    const int e0 = slab[r * (ns + 1) + q], e1 = slab[r * (ns + 1) + q + 1];
    double acc = 0.0;
    for (int base = e0; base < e1; base += 32) {
      const int e = base + lane;
      int myidx = static_cast<int>(s0);
      double myv = 0.0;
      if (e < e1) {
        myidx = idx[e];
        myv = T ? vals[perm[e]] : vals[e];
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int src = j + 16 * hh;
        const int ii = __shfl_sync(0xffffffffu, myidx, src);
        const double v = __shfl_sync(0xffffffffu, myv, src);
        acc = fma(v, xs[static_cast<i64>(ii - s0) * CW + col], acc);
      }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 16);
    if (hh == 0 && col < w) {
      if (ns == 1) {
        double* o = out + r * ldo + c0 + col;
        *o = beta == 0.0 ? alpha * acc : alpha * acc + beta * *o;
      } else {
        ws[(static_cast<i64>(q) * rows + r) * b + c0 + col] = acc;
      }
    }
  }
}

__global__ void slab_reduce_kernel(i64 rows, int ns, i64 b, const double* __restrict__ ws, double alpha,
                                   double beta, double* __restrict__ out, i64 ldo) {
  const i64 total = rows * b;
  for (i64 t = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 r = t / b, c = t % b;
    double s = 0.0;
    for (int q = 0; q < ns; ++q) s += ws[(static_cast<i64>(q) * rows + r) * b + c];
    double* o = out + r * ldo + c;
    *o = beta == 0.0 ? alpha * s : alpha * s + beta * *o;
  }
}

int grid_for(i64 total, int threads = 256) {
  return static_cast<int>(std::max<i64>(1, std::min<i64>((total + threads - 1) / threads, 4096)));
}

void build_plan(cudaStream_t s, SegPlan& p, i64 rows, const std::vector<int>& ptr) {
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
  build_plan(s, plan_csr, m, rowptr);
  build_plan(s, plan_csc, n, colptr);
  // slab offsets (input index = column for CSR rows, row for CSC columns; both sorted)
  auto slabs = [&](i64 rows, const std::vector<int>& ptr, const std::vector<int>& idx, i64 in_rows, int& ns,
                   DBuf<int>& out) {
    ns = static_cast<int>((in_rows + kSlabRows - 1) / kSlabRows);
    std::vector<int> h(static_cast<size_t>(rows * (ns + 1)));
    for (i64 r = 0; r < rows; ++r) {
      int e = ptr[r];
      for (int q = 0; q <= ns; ++q) {
        const long long lim = static_cast<long long>(q) * kSlabRows;
        while (e < ptr[r + 1] && idx[e] < lim) ++e;
        h[static_cast<size_t>(r * (ns + 1) + q)] = q == ns ? ptr[r + 1] : e;
      }
    }
    upload(s, out, h);
    DFCG_CUDA(cudaStreamSynchronize(s));
  };
  slabs(m, rowptr, rcol, n, nslab_csr, slab_csr);
  slabs(n, colptr, crow, m, nslab_csc, slab_csc);
  h_csc2csr = std::move(c2r);
}

void sddmm_residual(cudaStream_t s, const DevOmega& om, i64 kY, const double* Yl, i64 ldl, const double* Yr, i64 ldr,
                    const double* sub, double* r_csr) {
  if (om.nnz == 0) return;
  // algorithmic bytes: row+col index, M_e, r_e per entry + both factors once
  prof::Scope scope(prof::kSddmm, s, 2.0 * kY * om.nnz, 24.0 * om.nnz + 8.0 * (om.m + om.n) * kY);
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
          const double* X, i64 ldx, double beta, double* out, i64 ldo) {
  const SegPlan& p = transpose ? om.plan_csc : om.plan_csr;
  const i64 out_rows = transpose ? om.n : om.m;
  if (b <= 0 || out_rows <= 0) return;
  const int* ptr = transpose ? om.csc_colptr.get() : om.csr_rowptr.get();
  if (b >= kSlabMinB) {  // wide sketch: shared-memory-chunked path (off: slower than the segmented kernel)
    const i64 in_rows = transpose ? om.m : om.n;
    prof::Scope scope(prof::kSpmm, s, 2.0 * om.nnz * b,
                      (transpose ? 20.0 : 12.0) * om.nnz + 8.0 * b * (in_rows + out_rows * (beta != 0.0 ? 2 : 1)));
    const int ns = transpose ? om.nslab_csc : om.nslab_csr;
    const int chunks = cdiv(b, CW);
    const int rsplit = std::max(1, std::min<int>(static_cast<int>((out_rows + 15) / 16),
                                                 (148 + chunks * ns - 1) / (chunks * ns)));
    const size_t smem = sizeof(double) * DevOmega::kSlabRows * CW;
    static unsigned configured = 0;
    int dev = 0;
    DFCG_CUDA(cudaGetDevice(&dev));
    if (!(configured & (1u << dev))) {
      DFCG_CUDA(cudaFuncSetAttribute(spmm_slab_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
      DFCG_CUDA(cudaFuncSetAttribute(spmm_slab_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
      configured |= 1u << dev;
    }
    DBuf<double> ws;
    if (ns > 1) ws.alloc(static_cast<i64>(ns) * out_rows * b, s);
    const dim3 grid(chunks, ns, rsplit);
    if (transpose)
      spmm_slab_kernel<true><<<grid, SLAB_THREADS, smem, s>>>(out_rows, ns, rsplit, om.slab_csc.get(), om.csc_row.get(),
                                                     om.csc2csr.get(), vals_csr, in_rows, b, alpha, X, ldx, beta, out,
                                                     ldo, ws.get());
    else
      spmm_slab_kernel<false><<<grid, SLAB_THREADS, smem, s>>>(out_rows, ns, rsplit, om.slab_csr.get(), om.csr_col.get(),
                                                      om.csc2csr.get(), vals_csr, in_rows, b, alpha, X, ldx, beta,
                                                      out, ldo, ws.get());
    DFCG_LAUNCH_CHECK();
    if (ns > 1) {
      slab_reduce_kernel<<<grid_for(out_rows * b), 256, 0, s>>>(out_rows, ns, b, ws.get(), alpha, beta, out, ldo);
      DFCG_LAUNCH_CHECK();
    }
    return;
  }
  // algorithmic bytes: idx + value (+ permutation) per entry, X read once, out written (read if beta)
  const i64 in_rows = transpose ? om.m : om.n;
  prof::Scope scope(prof::kSpmm, s, 2.0 * om.nnz * b,
                    (transpose ? 20.0 : 12.0) * om.nnz + 8.0 * b * (in_rows + out_rows * (beta != 0.0 ? 2 : 1)));
  empty_rows_kernel<<<grid_for(out_rows * b), 256, 0, s>>>(out_rows, ptr, b, beta, out, ldo);
  DFCG_LAUNCH_CHECK();
  if (p.n_items == 0) return;
  DBuf<double> ws;
  if (p.n_slots) ws.alloc(p.n_slots * b, s);
  const int G = pow2_at_least(b);
  const i64 warps = (p.n_items + (32 / G) - 1) / (32 / G);
  const int blocks = static_cast<int>((warps + 7) / 8);
  const int* idx = transpose ? om.csc_row.get() : om.csr_col.get();
  const long long* perm = om.csc2csr.get();
#define SPMM_CASE(g)                                                                                               \
  case g:                                                                                                          \
    if (transpose)                                                                                                 \
      spmm_kernel<g, true><<<blocks, 256, 0, s>>>(p.n_items, p.items.get(), idx, perm, vals_csr, b, alpha, X, ldx, \
                                                   beta, out, ldo, ws.get());                                      \
    else                                                                                                           \
      spmm_kernel<g, false><<<blocks, 256, 0, s>>>(p.n_items, p.items.get(), idx, perm, vals_csr, b, alpha, X,     \
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

void scatter_add_dense(cudaStream_t s, const DevOmega& om, const double* vals_csr, double alpha, double* D, i64 ldd) {
  if (om.nnz == 0) return;
  scatter_dense_kernel<<<grid_for(om.nnz), 256, 0, s>>>(om.nnz, om.csr_row.get(), om.csr_col.get(), vals_csr, alpha,
                                                         D, ldd);
  DFCG_LAUNCH_CHECK();
}

}  // namespace dfcg
