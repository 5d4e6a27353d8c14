// GEMM microbenchmark: dfcg::gemm (and gemm_upper_b / gram_upper) against cuBLAS DGEMM on the
// shapes of the c2 APG iteration. Build: make -C tools gemm_bench; run on the GPU box.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_1107_0789_b200/csrc/common.cuh"

using dfcg::i64;

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      std::printf("cuda %s at %d\n", cudaGetErrorString(e_), __LINE__);    \
      return 1;                                                            \
    }                                                                      \
  } while (0)

struct Shape {
  const char* name;
  bool ta, tb;
  i64 M, N, K;
  int mode;  // 0 gemm, 1 gemm_upper_b (B triangular, K == N), 2 gram_upper (A^T A, M == N)
  double flops() const { return mode == 1 ? 1.0 * M * N * (N + 1) : mode == 2 ? 1.0 * M * (M + 1) * K : 2.0 * M * N * K; }
};

int main() {
  const Shape shapes[] = {
      {"dense apply TN 10000x720x1250", true, false, 10000, 720, 1250, 0},
      {"dense adj   NN 1250x720x10000", false, false, 1250, 720, 10000, 0},
      {"densify     NT 1250x10000x700", false, true, 1250, 10000, 700, 0},
      {"left X*coef NN 10000x700x720", false, false, 10000, 700, 720, 0},
      {"Yl*T        NN 10000x720x1437", false, false, 10000, 720, 1437, 0},
      {"Yl*T even   NN 10000x720x1438", false, false, 10000, 720, 1438, 0},
      {"Yl^T*X even TN 1438x720x10000", true, false, 1438, 720, 10000, 0},
      {"Yl^T*X      TN 1437x720x10000", true, false, 1437, 720, 10000, 0},
      {"X*Rinv      NN 10000x720x720", false, false, 10000, 720, 720, 0},
      {"X*Rinv tri  NN 10000x720x720", false, false, 10000, 720, 720, 1},
      {"gram upper  TN 720x720x10000", true, false, 720, 720, 10000, 2},
      {"gram full   TN 720x720x10000", true, false, 720, 720, 10000, 0},
      {"Yr^T*X      TN 1437x720x1250", true, false, 1437, 720, 1250, 0},
      {"Yr*T        NN 1250x720x1437", false, false, 1250, 720, 1437, 0},
      {"square      NN 4096^3", false, false, 4096, 4096, 4096, 0},
      {"chol trsm   TN 64x656x64", true, false, 64, 656, 64, 0},
      {"chol syrk   TN 656x656x64", true, false, 656, 656, 64, 0},
  };
  {  // keep freed pool memory cached, as the library's DeviceContext does (split-K workspaces)
    cudaMemPool_t pool;
    cudaDeviceGetDefaultMemPool(&pool, 0);
    unsigned long long thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cublasHandle_t h;
  cublasCreate(&h);
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cublasSetStream(h, s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (const Shape& sh : shapes) {
    const i64 M = sh.M, N = sh.N, K = sh.K;
    const i64 lda = sh.ta ? M : K, ldb = sh.tb ? K : N, ldc = N;
    const i64 asz = M * K, bsz = K * N, csz = M * N;
    double *A, *B, *C;
    CK(cudaMalloc(&A, sizeof(double) * asz));
    CK(cudaMalloc(&B, sizeof(double) * bsz));
    CK(cudaMalloc(&C, sizeof(double) * csz));
    std::vector<double> hv(std::max(asz, bsz));
    for (i64 i = 0; i < (i64)hv.size(); ++i) hv[i] = ((i * 2654435761u) % 1000) / 1000.0 - 0.5;
    CK(cudaMemcpy(A, hv.data(), sizeof(double) * asz, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(B, hv.data(), sizeof(double) * bsz, cudaMemcpyHostToDevice));
    auto ours = [&]() {
      if (sh.mode == 1) dfcg::gemm_upper_b(s, M, N, 1.0, A, lda, B, ldb, 0.0, C, ldc);
      else if (sh.mode == 2) dfcg::gram_upper(s, K, M, A, M, C, ldc);
      else dfcg::gemm(s, sh.ta, sh.tb, M, N, K, 1.0, A, lda, B, ldb, 0.0, C, ldc);
    };
    const double one = 1.0, zero = 0.0;
    auto theirs = [&]() {
      cublasDgemm(h, sh.tb ? CUBLAS_OP_T : CUBLAS_OP_N, sh.ta ? CUBLAS_OP_T : CUBLAS_OP_N, (int)N, (int)M, (int)K, &one,
                  B, (int)ldb, A, (int)lda, &zero, C, (int)ldc);
    };
    double t_ours = 0, t_cub = 0;
    for (int which = 0; which < 2; ++which) {
      for (int w = 0; w < 3; ++w) which ? theirs() : ours();
      CK(cudaStreamSynchronize(s));
      const int reps = 10;
      cudaEventRecord(e0, s);
      for (int r = 0; r < reps; ++r) which ? theirs() : ours();
      cudaEventRecord(e1, s);
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      (which ? t_cub : t_ours) = ms / reps;
    }
    const double cub_flops = 2.0 * M * N * K;
    std::printf("%-32s ours %8.1f us %6.2f TF/s | cublas %8.1f us %6.2f TF/s\n", sh.name, t_ours * 1e3,
                sh.flops() / (t_ours * 1e-3) / 1e12, t_cub * 1e3, cub_flops / (t_cub * 1e-3) / 1e12);
    cudaFree(A);
    cudaFree(B);
    cudaFree(C);
  }
  return 0;
}
