// Opt-in kernel accounting: CUDA-event timing per op class on the launching stream, plus the
// algorithmic FLOPs / bytes of each launch, so bench.py can report achieved GB/s or TFLOP/s of
// the dominant kernel measured live (roofline). Off by default; when off a scope costs one
// relaxed atomic load. A global launch counter backs bench.py's gpu_launches claim.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

namespace dfcg {
namespace prof {

enum Op : int {
  kGemm = 0,
  kSddmm,
  kSpmm,
  kCholesky,
  kQrFallback,
  kJacobi,
  kElementwise,
  kReduce,
  kOther,
  kGemmSmall,  // GEMMs below 2 GFLOP (factorisation internals, small products): latency-bound
  kNumOps
};

extern std::atomic<bool> g_enabled;
extern std::atomic<long long> g_launches;
// Always-on work counters per op class (algorithmic FLOPs / bytes / launches of every scope,
// no events): bench.py reads them around its timed window for the packed-step roofline.
extern std::atomic<long long> g_work_flops[kNumOps], g_work_bytes[kNumOps], g_work_launches[kNumOps];

// NVTX ranges on the calling host thread when DFCG_NVTX=1 (no-ops otherwise)
void nvtx_push(const char* name);
void nvtx_pop();
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtx_push(name); }
  ~NvtxRange() { nvtx_pop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

inline void count_launch(long long n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// RAII scope: records start/stop events on `s` when profiling is enabled.
class Scope {
 public:
  // launches: kernel launches the scope spans (e.g. the rounds of a Jacobi sweep), so per-launch
  // rates stay per kernel without an event pair around every launch.
  Scope(Op op, cudaStream_t s, double flops, double bytes, int launches = 1);
  ~Scope();
  // work known only after the launch (e.g. the sweeps a persistent Jacobi kernel executed)
  void add_work(double flops, double bytes, int launches);
  Scope(const Scope&) = delete;
  Scope& operator=(const Scope&) = delete;

 private:
  bool on_ = false;
  Op op_;
  cudaStream_t s_;
  double flops_, bytes_;
  int launches_ = 1;
  cudaEvent_t e0_ = nullptr, e1_ = nullptr;
};

}  // namespace prof
}  // namespace dfcg
