// Dependent-latency microbenchmark (one warp, clock64): FP64 FMA, FP32 FMA, shuffles, shared
// loads, MUFU seeds and the Newton rsqrt, IEEE sqrt / division. Calibrates the latency-bound
// kernels (Jacobi inner steps, potrf pivot chains).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  double e = fma(-h * y, y, 0.5);
  y = fma(y, e, y);
  e = fma(-h * y, y, 0.5);
  return fma(y, e, y);
}

template <int OP>
__global__ void chain(double* out, long long* cyc, double seed) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = seed + lane;
  sm[lane + 32] = 0.5;
  __syncwarp();
  double x = seed + lane * 1e-3;
  float xf = static_cast<float>(x);
  int idx = lane;
  constexpr int N = 256;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    if (OP == 0) x = fma(x, 0.999999, 1e-7);
    if (OP == 1) xf = fmaf(xf, 0.999999f, 1e-7f);
    if (OP == 2) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
    if (OP == 3) { x = sm[idx & 63] + 1.0; idx = static_cast<int>(x) & 31; }
    if (OP == 4) x = rsqrt_nr(x + 1.0);
    if (OP == 5) x = sqrt(x + 1.0);
    if (OP == 6) x = 1.0 / (x + 1.0);
    if (OP == 7) { double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x + 1.0)); x = y; }
    if (OP == 8) x = x * 1.0000001;
  }
  long long t1 = clock64();
  out[lane] = x + xf;
  if (lane == 0) cyc[OP] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 64 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  chain<0><<<1, 32>>>(out, cyc, 1.0);
  chain<1><<<1, 32>>>(out, cyc, 1.0);
  chain<2><<<1, 32>>>(out, cyc, 1.0);
  chain<3><<<1, 32>>>(out, cyc, 1.0);
  chain<4><<<1, 32>>>(out, cyc, 1.0);
  chain<5><<<1, 32>>>(out, cyc, 1.0);
  chain<6><<<1, 32>>>(out, cyc, 1.0);
  chain<7><<<1, 32>>>(out, cyc, 1.0);
  chain<8><<<1, 32>>>(out, cyc, 1.0);
  cudaDeviceSynchronize();
  const char* names[] = {"DFMA", "FFMA", "SHFL(f64)", "LDS.64+DADD+cvt", "rsqrt_nr (MUFU+2 Newton)", "IEEE sqrt f64",
                         "IEEE div f64", "MUFU.RSQ64H", "DMUL"};
  for (int i = 0; i < 9; ++i) std::printf("%-26s %6.1f cycles per dependent op\n", names[i], cyc[i] / 256.0);
  return 0;
}
