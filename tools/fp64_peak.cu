// Microbenchmark: FP64 peak on B200 via DMMA (mma.sync m8n8k4 f64) and via DFMA.
// Used once to fix the FP64 roofline denominator (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[16];
  for (int i = 0; i < 16; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void copy_kernel(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int grid = sms * bps;
      dmma_loop<<<grid, threads>>>(out, 100);
      cudaEventRecord(e0);
      dmma_loop<<<grid, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = (double)grid * (threads / 32) * iters * 8 * 512.0;
      printf("DMMA m8n8k4 grid=%d threads=%d: %.2f TFLOP/s\n", grid, threads, flops / ms / 1e9);
      dfma_loop<<<grid, threads>>>(out, 100);
      cudaEventRecord(e0);
      dfma_loop<<<grid, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = (double)grid * threads * iters * 16 * 2.0;
      printf("DFMA      grid=%d threads=%d: %.2f TFLOP/s\n", grid, threads, flops / ms / 1e9);
    }
  }
  size_t n = (size_t)1 << 27;  // 4 GiB each in double4? 2^27 * 32 B = 4 GiB
  double4 *a, *b;
  cudaMalloc(&a, n * sizeof(double4));
  cudaMalloc(&b, n * sizeof(double4));
  cudaMemset(a, 0, n * sizeof(double4));
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    copy_kernel<<<sms * 8, 256>>>(a, b, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy: %.1f GB/s\n", 2.0 * n * sizeof(double4) / ms / 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
