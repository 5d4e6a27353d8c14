// Phase timing of the fused cooperative Cholesky (factor.cu compiled in with DFCG_CHOL_TRACE):
// per 64-column step, CTA 0 (diagonal factor owner) and CTA 1 (a worker): phase A work, the
// barrier after it, CTA 0's look-ahead update and potrf, phase B work, the barrier after it.
#define DFCG_CHOL_TRACE
#include "../paper_1107_0789_b200/csrc/factor.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

int main(int argc, char** argv) {
  using namespace dfcg;
  const int n = argc > 1 ? std::atoi(argv[1]) : 720;
  std::vector<double> X(2 * n * n), G(n * n);
  unsigned long long x = 7;
  for (auto& v : X) {
    x = x * 6364136223846793005ULL + 1442695040888963407ULL;
    v = static_cast<double>(x >> 11) / 9007199254740992.0 - 0.5;
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double a = 0;
      for (int r = 0; r < 2 * n; ++r) a += X[r * n + i] * X[r * n + j];
      G[i * n + j] = a + (i == j ? n : 0.0);
    }
  cudaStream_t s;
  cudaStreamCreate(&s);
  double *dG, *dR;
  int* fail;
  cudaMalloc(&dG, sizeof(double) * n * n);
  cudaMalloc(&dR, sizeof(double) * n * n);
  cudaMalloc(&fail, sizeof(int));
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(dG, G.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
    cudaMemset(fail, 0, sizeof(int));
    cholesky_inverse(s, n, dG, n, dR, n, 1e-11, fail, true, true);
    cudaStreamSynchronize(s);
  }
  unsigned long long tr[64][2][6];
  cudaMemcpyFromSymbol(tr, g_chol_trace, sizeof(tr));
  const int nt = (n + 63) / 64;
  std::printf("n = %d, %d steps; microseconds per step (CTA 0 | CTA 1)\n", n, nt);
  std::printf("step  A-work0  syncA0  upd0  potrf0  B-rest0  syncB0 | A-work1 syncA1 B-work1 syncB1\n");
  double sum[10] = {0};
  for (int k = 0; k < nt; ++k) {
    auto d = [&](int c, int a, int b) { return (tr[k][c][b] - tr[k][c][a]) / 1e3; };
    const double nxt0 = k + 1 < nt ? (tr[k + 1][0][0] - tr[k][0][5]) / 1e3 : 0.0;
    const double nxt1 = k + 1 < nt ? (tr[k + 1][1][0] - tr[k][1][5]) / 1e3 : 0.0;
    const double v[10] = {d(0, 0, 1), d(0, 1, 2), d(0, 2, 3), d(0, 3, 4), d(0, 4, 5), nxt0,
                          d(1, 0, 1), d(1, 1, 2), d(1, 2, 5), nxt1};
    std::printf("%4d  %7.1f %7.1f %5.1f %7.1f %8.1f %7.1f | %7.1f %6.1f %7.1f %6.1f\n", k, v[0], v[1], v[2], v[3], v[4],
                v[5], v[6], v[7], v[8], v[9]);
    for (int i = 0; i < 10; ++i) sum[i] += v[i];
  }
  std::printf("sum   %7.1f %7.1f %5.1f %7.1f %8.1f %7.1f | %7.1f %6.1f %7.1f %6.1f  total %.1f us\n", sum[0], sum[1],
              sum[2], sum[3], sum[4], sum[5], sum[6], sum[7], sum[8], sum[9],
              (tr[nt - 1][0][5] - tr[0][0][0]) / 1e3);
  return 0;
}
