// Kernel accounting (see prof.hpp) and its C ABI (dfcg_prof_*, declared in include/dfcg_host.h).
#include "prof.hpp"

#include <nvtx3/nvToolsExt.h>

#include <cstdlib>
#include <mutex>
#include <vector>

#include "../../include/dfcg_host.h"

namespace dfcg {
namespace prof {

std::atomic<bool> g_enabled{false};
std::atomic<long long> g_launches{0};
std::atomic<long long> g_work_flops[kNumOps], g_work_bytes[kNumOps], g_work_launches[kNumOps];

namespace {
struct Rec {
  Op op;
  double flops, bytes;
  int launches;
  cudaEvent_t e0, e1;
};
std::mutex g_mu;
std::vector<Rec> g_recs;
}  // namespace

// DFCG_NVTX=1: every scope is also an NVTX range named after its op class (and every APG
// iteration one, see nvtx_push / nvtx_pop), so an nsys / ncu timeline shows the phases of each
// solve on its host thread. Header-only NVTX v3: a no-op unless a tool injects itself.
static const bool g_nvtx = std::getenv("DFCG_NVTX") && std::atoi(std::getenv("DFCG_NVTX")) != 0;
static const char* const kOpNames[kNumOps] = {"gemm",   "sddmm",       "spmm",   "cholesky", "qr_fallback",
                                              "jacobi", "elementwise", "reduce", "other",    "gemm_small"};

void nvtx_push(const char* name) {
  if (g_nvtx) nvtxRangePushA(name);
}
void nvtx_pop() {
  if (g_nvtx) nvtxRangePop();
}

Scope::Scope(Op op, cudaStream_t s, double flops, double bytes, int launches)
    : op_(op), s_(s), flops_(flops), bytes_(bytes), launches_(launches) {
  if (g_nvtx) nvtxRangePushA(kOpNames[op]);
  g_work_flops[op].fetch_add(static_cast<long long>(flops), std::memory_order_relaxed);
  g_work_bytes[op].fetch_add(static_cast<long long>(bytes), std::memory_order_relaxed);
  g_work_launches[op].fetch_add(launches, std::memory_order_relaxed);
  if (!g_enabled.load(std::memory_order_relaxed)) return;
  on_ = true;
  cudaEventCreate(&e0_);
  cudaEventCreate(&e1_);
  cudaEventRecord(e0_, s_);
}

void Scope::add_work(double flops, double bytes, int launches) {
  g_work_flops[op_].fetch_add(static_cast<long long>(flops), std::memory_order_relaxed);
  g_work_bytes[op_].fetch_add(static_cast<long long>(bytes), std::memory_order_relaxed);
  g_work_launches[op_].fetch_add(launches, std::memory_order_relaxed);
  flops_ += flops;
  bytes_ += bytes;
  launches_ += launches;
}

Scope::~Scope() {
  if (g_nvtx) nvtxRangePop();
  if (!on_) return;
  cudaEventRecord(e1_, s_);
  std::lock_guard<std::mutex> lock(g_mu);
  g_recs.push_back({op_, flops_, bytes_, launches_, e0_, e1_});
}

}  // namespace prof
}  // namespace dfcg

using namespace dfcg::prof;

extern "C" {

void dfcg_prof_enable(int on) {
  std::lock_guard<std::mutex> lock(g_mu);
  for (auto& r : g_recs) {
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  g_recs.clear();
  g_enabled.store(on != 0);
}

int64_t dfcg_launch_count(void) { return g_launches.load(); }

int dfcg_work_counters(int64_t* launches, double* flops, double* bytes) {
  for (int i = 0; i < kNumOps; ++i) {
    launches[i] = g_work_launches[i].load();
    flops[i] = static_cast<double>(g_work_flops[i].load());
    bytes[i] = static_cast<double>(g_work_bytes[i].load());
  }
  return kNumOps;
}

int dfcg_prof_collect(int64_t* launches, double* ms, double* flops, double* bytes) {
  std::lock_guard<std::mutex> lock(g_mu);
  for (int i = 0; i < kNumOps; ++i) {
    launches[i] = 0;
    ms[i] = flops[i] = bytes[i] = 0.0;
  }
  for (auto& r : g_recs) {
    if (cudaEventSynchronize(r.e1) != cudaSuccess) return -4;
    float t = 0.f;
    cudaEventElapsedTime(&t, r.e0, r.e1);
    launches[r.op] += r.launches;
    ms[r.op] += t;
    flops[r.op] += r.flops;
    bytes[r.op] += r.bytes;
  }
  return kNumOps;
}

}  // extern "C"
