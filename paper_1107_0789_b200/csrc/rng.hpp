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

// Device-resident prefix of the normal stream of SeededRng(seed, stream), in fixed chunks that
// are immutable once published (concurrent solves read them without locking). A background
// thread generates ahead of the furthest position any solve has asked for (kAhead chunks), so
// the sequential mt19937_64 draws and the host Box-Muller never sit on a solve's critical
// path in steady state; the upload goes through pinned memory on the cache's own non-blocking
// stream (no legacy-stream synchronisation with the solves' streams).
class NormalCache {
 public:
  static constexpr i64 kChunk = i64{1} << 22;  // 4 Mi normals = 32 MiB per chunk
  static constexpr i64 kAhead = 4;

  NormalCache(int device, std::uint64_t seed, std::uint64_t stream) : device_(device) {
    mt_.seed(SeededRng::engine_seed(seed, stream));
  }
  ~NormalCache() {
    {
      std::lock_guard<std::mutex> lock(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    if (worker_.joinable()) worker_.join();
    if (transformer_.joinable()) transformer_.join();
    for (double* p : chunks_) cudaFree(p);
    for (std::uint64_t* p : raw_buf_)
      if (p) cudaFreeHost(p);
    if (stream_) cudaStreamDestroy(stream_);
  }

  // dst[0:count) <- normals[pos : pos+count) on stream s.
  void fetch(i64 pos, i64 count, double* dst, cudaStream_t s) {
    if (count <= 0) return;
    const i64 need = (pos + count + kChunk - 1) / kChunk;
    std::vector<double*> src;
    {
      std::unique_lock<std::mutex> lock(mu_);
      if (error_) throw std::runtime_error(err_msg_);
      static const i64 ahead = std::getenv("DFCG_NORMALS_AHEAD") ? std::atoll(std::getenv("DFCG_NORMALS_AHEAD")) : kAhead;
      if (need + ahead > wanted_) {
        wanted_ = need + ahead;
        if (!worker_.joinable()) {
          worker_ = std::thread([this] { run_raw(); });
          transformer_ = std::thread([this] { run_transform(); });
        }
        cv_.notify_all();
      }
      cv_.wait(lock, [&] { return static_cast<i64>(chunks_.size()) >= need || error_; });
      if (error_) throw std::runtime_error(err_msg_);
      src = chunks_;
    }
    i64 done = 0;
    while (done < count) {
      const i64 p = pos + done;
      const i64 c = p / kChunk, off = p % kChunk;
      const i64 n = std::min(count - done, kChunk - off);
      DFCG_CUDA(cudaMemcpyAsync(dst + done, src[static_cast<size_t>(c)] + off, sizeof(double) * n,
                                cudaMemcpyDeviceToDevice, s));
      done += n;
    }
  }

 private:
  // Two-stage pipeline: this thread draws the raw 64-bit words of chunk k + 1 (sequential
  // mt19937_64, the stream's only serial part) while run_transform() uploads chunk k and turns
  // it into normals on the device — a chunk every max(draw, transform) instead of their sum. Wide
  // blocks consume w * b normals per partial SVD (7.2 M for a 1250 x 10000 DFC-Nys row block),
  // so the generator's rate bounds them otherwise.
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
        {
          std::unique_lock<std::mutex> lock(mu_);
          cv_.wait(lock, [&] { return stop_ || (raw_made_ < wanted_ && !raw_free_.empty()); });
          if (stop_) return;
          b = raw_free_.back();
          raw_free_.pop_back();
        }
        mt64_fill(mt_, raw_buf_[b], 2 * kChunk);
        {
          std::lock_guard<std::mutex> lock(mu_);
          raw_q_.push_back(b);
          ++raw_made_;
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
        int b = -1;
        {
          std::unique_lock<std::mutex> lock(mu_);
          cv_.wait(lock, [&] { return stop_ || !raw_q_.empty(); });
          if (stop_) break;
          b = raw_q_.front();
          raw_q_.erase(raw_q_.begin());
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
          chunks_.push_back(d);
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
  Mt64 mt_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::thread worker_, transformer_;
  bool stop_ = false, error_ = false;
  std::string err_msg_;
  i64 wanted_ = 0, raw_made_ = 0;
  static constexpr int kRawBufs = 3;
  std::uint64_t* raw_buf_[kRawBufs] = {nullptr, nullptr, nullptr};
  std::vector<int> raw_q_, raw_free_;
  std::vector<double*> chunks_;
  cudaStream_t stream_ = nullptr;
};

}  // namespace dfcg
