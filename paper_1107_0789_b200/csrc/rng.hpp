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

class SeededRng {
 public:
  explicit SeededRng(std::uint64_t seed, std::uint64_t stream = 0) : seed_(seed), stream_(stream) {
    std::uint64_t x = seed;
    const std::uint64_t h = splitmix64(x);
    x = h ^ (0xD1B54A32D192ED03ULL * (stream + 1));
    engine_.seed(splitmix64(x));
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

  NormalCache(int device, std::uint64_t seed, std::uint64_t stream) : device_(device), rng_(seed, stream) {}
  ~NormalCache() {
    {
      std::lock_guard<std::mutex> lock(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    if (worker_.joinable()) worker_.join();
    for (double* p : chunks_) cudaFree(p);
    if (pinned_) cudaFreeHost(pinned_);
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
        if (!worker_.joinable()) worker_ = std::thread([this] { run(); });
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
  void run() {
    try {
      DFCG_CUDA(cudaSetDevice(device_));
      DFCG_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
      DFCG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&pinned_), sizeof(double) * kChunk));
      std::vector<std::uint64_t> raw(2 * kChunk);
      for (;;) {
        {
          std::unique_lock<std::mutex> lock(mu_);
          cv_.wait(lock, [&] { return stop_ || static_cast<i64>(chunks_.size()) < wanted_; });
          if (stop_) return;
        }
        // Raw 64-bit draws are sequential (mt19937_64); the Box-Muller transform runs on host
        // threads so the stream stays bit-identical to the reference's std::log/std::cos.
        for (auto& r : raw) r = rng_.next_u64();
        // A few transform threads only: the generator runs beside the solves' host threads, and a
        // burst that takes every core delays their kernel launches (the GPU then idles).
        const unsigned nt = std::max(1u, std::min(4u, std::thread::hardware_concurrency() / 4));
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < nt; ++t)
          pool.emplace_back([&, t] {
            for (i64 i = t; i < kChunk; i += nt) {
              const double u1 = (static_cast<double>(raw[2 * i] >> 11) + 1.0) * 0x1.0p-53;
              const double u2 = static_cast<double>(raw[2 * i + 1] >> 11) * 0x1.0p-53;
              pinned_[i] = SeededRng::box_muller(u1, u2);
            }
          });
        for (auto& th : pool) th.join();
        double* d = nullptr;
        DFCG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(double) * kChunk, stream_));
        DFCG_CUDA(cudaMemcpyAsync(d, pinned_, sizeof(double) * kChunk, cudaMemcpyHostToDevice, stream_));
        DFCG_CUDA(cudaStreamSynchronize(stream_));
        {
          std::lock_guard<std::mutex> lock(mu_);
          chunks_.push_back(d);
        }
        cv_.notify_all();
      }
    } catch (const std::exception& e) {
      std::lock_guard<std::mutex> lock(mu_);
      error_ = true;
      err_msg_ = std::string("NormalCache: ") + e.what();
      cv_.notify_all();
    }
  }

  int device_;
  SeededRng rng_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::thread worker_;
  bool stop_ = false, error_ = false;
  std::string err_msg_;
  i64 wanted_ = 0;
  std::vector<double*> chunks_;
  double* pinned_ = nullptr;
  cudaStream_t stream_ = nullptr;
};

}  // namespace dfcg
