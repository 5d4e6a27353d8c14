// Phase timing of the blocked potrf kernel (factor.cu compiled in with DFCG_POTRF_TRACE).
#define DFCG_POTRF_TRACE
#include "../paper_1107_0789_b200/csrc/factor.cu"

#include <cstdio>
#include <vector>

int main() {
  using namespace dfcg;
  const int n = 64, reps = 50;
  std::vector<double> h(n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) h[i * n + j] = (i == j ? n : 0.0) + 1.0 / (1.0 + i + j);
  double *G, *R, *md;
  int* fail;
  cudaMalloc(&G, sizeof(double) * n * n);
  cudaMalloc(&R, sizeof(double) * n * n);
  cudaMalloc(&md, sizeof(double));
  cudaMalloc(&fail, sizeof(int));
  const double mdv = n + 1.0;
  cudaMemcpy(md, &mdv, sizeof(double), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kPotrfSmem));
  long long zero[64] = {0};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int kb : {64, 25}) {
    cudaMemcpyToSymbol(g_potrf_trace, zero, sizeof(zero));
    float ms = 0;
    for (int r = 0; r < reps; ++r) {
      cudaMemcpy(G, h.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
      cudaEventRecord(e0);
      potrf_diag_kernel<<<1, 256, kPotrfSmem>>>(kb, G, n, R, n, md, 1e-11, fail, 1);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float t = 0;
      cudaEventElapsedTime(&t, e0, e1);
      ms += t;
    }
    long long tr[64];
    cudaMemcpyFromSymbol(tr, g_potrf_trace, sizeof(tr));
    std::printf("kb=%d: %.2f us per launch (events); cycles per launch: load %lld factor %lld trsm %lld update %lld "
                "inv-diag %lld back-sub %lld store %lld\n",
                kb, 1e3 * ms / reps, tr[1] / reps, tr[6] / reps, tr[7] / reps, tr[8] / reps, tr[3] / reps, tr[4] / reps,
                tr[5] / reps);
  }
  return 0;
}
