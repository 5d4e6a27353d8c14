// Host RNG for the product path: the reference's SeededRng (P/include/dfc/rng.hpp:11-74),
// restated so the device SVT consumes the bit-identical Gaussian stream, plus a per-device
// cache of that stream (the SVT draws from the constant seed 0x737674 in every solve,
// P/include/dfc/solvers.hpp:263,344, so one cached prefix serves every block on a GPU).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace dfcg {

inline std::uint64_t splitmix64(std::uint64_t& state) {
  state += 0x9E3779B97F4A7C15ULL;
  std::uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// mt19937_64 with bulk output (bit-identical to std::mt19937_64: same parameters, seeding and
// tempering), its twist written as three dependence-free loops over a second state array so
// the compiler vectorises it — the sequential part of the normal stream (hostgen.cpp).
struct Mt64 {
  std::uint64_t mt[312];
  int idx = 312;
  void seed(std::uint64_t s);
};
// out[0:n) = the engine's next n outputs.
void mt64_fill(Mt64& g, std::uint64_t* out, std::int64_t n);

class SeededRng {
 public:
  // The mt19937_64 seed SeededRng(seed, stream) uses (P/include/dfc/rng.hpp:19-26 restated).
  static std::uint64_t engine_seed(std::uint64_t seed, std::uint64_t stream) {
    std::uint64_t x = seed;
    const std::uint64_t h = splitmix64(x);
    x = h ^ (0xD1B54A32D192ED03ULL * (stream + 1));
    return splitmix64(x);
  }
  explicit SeededRng(std::uint64_t seed, std::uint64_t stream = 0) : seed_(seed), stream_(stream) {
    engine_.seed(engine_seed(seed, stream));
  }
  std::uint64_t next_u64() { return engine_(); }
  double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double uniform_pos() { return (static_cast<double>(next_u64() >> 11) + 1.0) * 0x1.0p-53; }
  std::uint64_t index(std::uint64_t n) {
    if (n == 0) throw std::invalid_argument("SeededRng::index: n must be positive");
    const std::uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    std::uint64_t x = next_u64();
    while (x >= limit) x = next_u64();
    return x % n;
  }
  double normal() {
    const double u1 = uniform_pos();
    const double u2 = uniform();
    return box_muller(u1, u2);
  }
  double normal(double mean, double sd) { return mean + sd * normal(); }
  static double box_muller(double u1, double u2) {
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
  }
  std::uint64_t seed() const { return seed_; }
  std::uint64_t stream() const { return stream_; }

 private:
  std::uint64_t seed_, stream_;
  std::mt19937_64 engine_;
};

// Device-resident window of the normal stream of SeededRng(seed, stream), in fixed chunks that
// are immutable while resident (a fetch pins the chunks it copies from). Background threads draw
// the chunks each fetch will need next (kAhead past its window), so the sequential mt19937_64
// draws never sit on a solve's critical path in steady state; least-recently-fetched chunks
// are evicted beyond a device budget and redrawn from their engine snapshot if a later solve
// (every solve restarts at position 0) asks again. Uploads run on the cache's own
// non-blocking stream (no legacy-stream synchronisation with the solves' streams).
class NormalCache {
 public:
  static constexpr i64 kChunk = i64{1} << 22;  // 4 Mi normals = 32 MiB per chunk
  static constexpr i64 kAhead = 4;

  NormalCache(int device, std::uint64_t seed, std::uint64_t stream) : device_(device) {
    mt_.seed(SeededRng::engine_seed(seed, stream));
    const char* env = std::getenv("DFCG_NORMALS_MAX_CHUNKS");
    max_resident_ = env ? std::max<i64>(2 * kAhead + 2, std::atoll(env)) : 64;
  }
  ~NormalCache() {
    {
      std::lock_guard<std::mutex> lock(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    if (worker_.joinable()) worker_.join();
    if (transformer_.joinable()) transformer_.join();
    for (double* p : chunks_)
      if (p) cudaFree(p);
    for (auto& evs : use_ev_)
      for (cudaEvent_t e : evs) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_free_) cudaEventDestroy(e);
    for (std::uint64_t* p : raw_buf_)
      if (p) cudaFreeHost(p);
    if (stream_) cudaStreamDestroy(stream_);
  }

  // dst[0:count) <- normals[pos : pos+count) on stream s.
  void fetch(i64 pos, i64 count, double* dst, cudaStream_t s) {
    if (count <= 0) return;
    const i64 c0 = pos / kChunk, c1 = (pos + count + kChunk - 1) / kChunk;  // chunks [c0, c1)
    static const i64 ahead = std::getenv("DFCG_NORMALS_AHEAD") ? std::atoll(std::getenv("DFCG_NORMALS_AHEAD")) : kAhead;
    std::vector<double*> src(static_cast<size_t>(c1 - c0));
    {
      std::unique_lock<std::mutex> lock(mu_);
      if (error_) throw std::runtime_error(err_msg_);
      grow(c1 + ahead);
      bool more = false;
      for (i64 c = c0; c < c1 + ahead; ++c)
        if (!chunks_[c] && !inflight_[c] && want_.insert(c).second) more = true;
      if (more) {
        if (!worker_.joinable()) {
          worker_ = std::thread([this] { run_raw(); });
          transformer_ = std::thread([this] { run_transform(); });
        }
        cv_.notify_all();
      }
      for (;;) {  // (a needed chunk evicted before this fetch pinned it is requested again)
        if (error_) throw std::runtime_error(err_msg_);
        bool ready = true, ask = false;
        for (i64 c = c0; c < c1; ++c)
          if (!chunks_[c]) {
            ready = false;
            if (!inflight_[c] && want_.insert(c).second) ask = true;
          }
        if (ready) break;
        if (ask) cv_.notify_all();
        cv_.wait(lock);
      }
      for (i64 c = c0; c < c1; ++c) {
        src[static_cast<size_t>(c - c0)] = chunks_[c];
        ++pins_[c];  // not evicted until this fetch's copies are ordered before its free
        last_use_[c] = ++clock_;
      }
    }
    i64 done = 0;
    while (done < count) {
      const i64 p = pos + done;
      const i64 c = p / kChunk, off = p % kChunk;
      const i64 n = std::min(count - done, kChunk - off);
      DFCG_CUDA(cudaMemcpyAsync(dst + done, src[static_cast<size_t>(c - c0)] + off, sizeof(double) * n,
                                cudaMemcpyDeviceToDevice, s));
      done += n;
    }
    // One event per fetch and chunk: fetches on different streams each keep their own record,
    // and eviction orders the free after ALL of them (completed ones are recycled here).
    std::lock_guard<std::mutex> lock(mu_);
    for (i64 c = c0; c < c1; ++c) {
      auto& evs = use_ev_[c];
      for (size_t i = 0; i < evs.size();) {
        if (cudaEventQuery(evs[i]) == cudaSuccess) {
          ev_free_.push_back(evs[i]);
          evs[i] = evs.back();
          evs.pop_back();
        } else {
          ++i;
        }
      }
      cudaEvent_t ev = nullptr;
      if (!ev_free_.empty()) {
        ev = ev_free_.back();
        ev_free_.pop_back();
      } else {
        DFCG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      }
      DFCG_CUDA(cudaEventRecord(ev, s));
      evs.push_back(ev);
      --pins_[c];
    }
  }

 private:
  // Chunk bookkeeping (under mu_): device chunk or nullptr (not resident), the engine state at
  // the start of every chunk drawn so far (an evicted chunk is redrawn from it), pin counts of
  // in-progress fetches, and LRU stamps. At most max_resident_ chunks stay on the device
  // (DFCG_NORMALS_MAX_CHUNKS, default 64 = 2 GiB): a solve draws w * b normals per partial SVD,
  // so an unbounded prefix reached 29 GB for a 500-iteration DFC-Nys row block and growing the
  // device pool for it stalled every concurrent solve.
  void grow(i64 n) {
    if (static_cast<i64>(chunks_.size()) >= n) return;
    chunks_.resize(static_cast<size_t>(n), nullptr);
    inflight_.resize(static_cast<size_t>(n), 0);
    pins_.resize(static_cast<size_t>(n), 0);
    last_use_.resize(static_cast<size_t>(n), 0);
    use_ev_.resize(static_cast<size_t>(n));
  }

  // Two-stage pipeline: this thread draws the raw 64-bit words of a chunk (sequential
  // mt19937_64, the stream's only serial part; an evicted chunk restarts from its snapshot)
  // while run_transform() uploads the previous one and turns it into normals on the device.
  void run_raw() {
    try {
      DFCG_CUDA(cudaSetDevice(device_));
      // three pinned raw buffers cycle between the two stages (no allocation or first-touch
      // page faults per chunk, DMA-speed uploads)
      for (int i = 0; i < kRawBufs; ++i) {
        DFCG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&raw_buf_[i]), sizeof(std::uint64_t) * 2 * kChunk));
        std::lock_guard<std::mutex> lock(mu_);
        raw_free_.push_back(i);
      }
      for (;;) {
        int b = -1;
        i64 c = -1;
        Mt64 g;
        bool sequential = false;
        {
          std::unique_lock<std::mutex> lock(mu_);
          cv_.wait(lock, [&] { return stop_ || (!want_.empty() && !raw_free_.empty()); });
          if (stop_) return;
          c = *want_.begin();
          const i64 next = static_cast<i64>(snap_.size());
          if (c >= next) {  // draw forward: the next chunk in sequence (a prerequisite of c)
            if (c == next) want_.erase(want_.begin());
            c = next;
            snap_.push_back(mt_);
            sequential = true;
            grow(c + 1);
          } else {  // redraw an evicted chunk from its snapshot
            want_.erase(want_.begin());
            if (chunks_[c] || inflight_[c]) continue;
            g = snap_[static_cast<size_t>(c)];
          }
          inflight_[c] = 1;
          b = raw_free_.back();
          raw_free_.pop_back();
        }
        if (sequential) mt64_fill(mt_, raw_buf_[b], 2 * kChunk);
        else mt64_fill(g, raw_buf_[b], 2 * kChunk);
        {
          std::lock_guard<std::mutex> lock(mu_);
          raw_q_.push_back({c, b});
        }
        cv_.notify_all();
      }
    } catch (const std::exception& e) {
      fail(e.what());
    }
  }

  void run_transform() {
    try {
      DFCG_CUDA(cudaSetDevice(device_));
      DFCG_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
      std::uint64_t* raw_dev = nullptr;
      DFCG_CUDA(cudaMalloc(reinterpret_cast<void**>(&raw_dev), sizeof(std::uint64_t) * 2 * kChunk));
      for (;;) {
        i64 c = -1;
        int b = -1;
        std::vector<std::pair<double*, std::vector<cudaEvent_t>>> victims;
        {
          std::unique_lock<std::mutex> lock(mu_);
          cv_.wait(lock, [&] { return stop_ || !raw_q_.empty(); });
          if (stop_) break;
          c = raw_q_.front().first;
          b = raw_q_.front().second;
          raw_q_.erase(raw_q_.begin());
          // evict least-recently fetched, unpinned chunks down to the budget (this one included)
          i64 resident = 1;
          for (double* p : chunks_) resident += p != nullptr;
          while (resident > max_resident_) {
            i64 v = -1;
            for (i64 k = 0; k < static_cast<i64>(chunks_.size()); ++k)
              if (chunks_[k] && pins_[k] == 0 && (v < 0 || last_use_[k] < last_use_[v])) v = k;
            if (v < 0) break;
            victims.push_back({chunks_[v], std::move(use_ev_[v])});
            use_ev_[v].clear();
            chunks_[v] = nullptr;
            --resident;
          }
        }
        for (auto& [p, evs] : victims) {  // freed on this stream after every fetch's copies
          for (cudaEvent_t ev : evs) DFCG_CUDA(cudaStreamWaitEvent(stream_, ev, 0));
          DFCG_CUDA(cudaFreeAsync(p, stream_));
        }
        if (!victims.empty()) {  // the waits captured the records; the events can be reused
          std::lock_guard<std::mutex> lock(mu_);
          for (auto& [p, evs] : victims) ev_free_.insert(ev_free_.end(), evs.begin(), evs.end());
        }
        // Box-Muller on the device (CUDA's log / cos, <= 1 ulp from the host libm the oracle
        // uses; the raw words are bit-identical): the host keeps only the serial draws.
        double* d = nullptr;
        DFCG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(double) * kChunk, stream_));
        DFCG_CUDA(cudaMemcpyAsync(raw_dev, raw_buf_[b], sizeof(std::uint64_t) * 2 * kChunk, cudaMemcpyHostToDevice,
                                  stream_));
        box_muller_device(stream_, raw_dev, d, kChunk);
        DFCG_CUDA(cudaStreamSynchronize(stream_));
        {
          std::lock_guard<std::mutex> lock(mu_);
          raw_free_.push_back(b);
          chunks_[c] = d;
          inflight_[c] = 0;
          last_use_[c] = ++clock_;
        }
        cv_.notify_all();
      }
      cudaFree(raw_dev);
    } catch (const std::exception& e) {
      fail(e.what());
    }
  }

  void fail(const char* what) {
    std::lock_guard<std::mutex> lock(mu_);
    error_ = true;
    err_msg_ = std::string("NormalCache: ") + what;
    cv_.notify_all();
  }

  int device_;
  Mt64 mt_;  // the engine after the last chunk drawn in sequence
  std::mutex mu_;
  std::condition_variable cv_;
  std::thread worker_, transformer_;
  bool stop_ = false, error_ = false;
  std::string err_msg_;
  i64 max_resident_ = 64;
  std::uint64_t clock_ = 0;
  std::set<i64> want_;
  std::vector<Mt64> snap_;
  std::vector<double*> chunks_;
  std::vector<char> inflight_;
  std::vector<int> pins_;
  std::vector<std::uint64_t> last_use_;
  std::vector<std::vector<cudaEvent_t>> use_ev_;  // per chunk: one event per fetch not known done
  std::vector<cudaEvent_t> ev_free_;
  static constexpr int kRawBufs = 3;
  std::uint64_t* raw_buf_[kRawBufs] = {nullptr, nullptr, nullptr};
  std::vector<std::pair<i64, int>> raw_q_;
  std::vector<int> raw_free_;
  cudaStream_t stream_ = nullptr;
};

}  // namespace dfcg
