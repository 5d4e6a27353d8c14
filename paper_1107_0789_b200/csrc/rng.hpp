// Host RNG for the product path: the reference's SeededRng (P/include/dfc/rng.hpp:11-74),
// restated so the device SVT consumes the bit-identical Gaussian stream, plus a per-device
// cache of that stream (the SVT draws from the constant seed 0x737674 in every solve,
// P/include/dfc/solvers.hpp:263,344, so one cached prefix serves every block on a GPU).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <mutex>
#include <random>
#include <stdexcept>
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

// Device-resident prefix of the normal stream of SeededRng(seed, stream), grown on demand in
// fixed chunks (immutable once written, so concurrent solves read them without locking).
class NormalCache {
 public:
  static constexpr i64 kChunk = i64{1} << 22;  // 4 Mi normals = 32 MiB per chunk

  NormalCache(int device, std::uint64_t seed, std::uint64_t stream) : device_(device), rng_(seed, stream) {}
  ~NormalCache() {
    for (double* p : chunks_) cudaFree(p);
  }

  // dst[0:count) <- normals[pos : pos+count) on stream s.
  void fetch(i64 pos, i64 count, double* dst, cudaStream_t s) {
    if (count <= 0) return;
    ensure(pos + count);
    i64 done = 0;
    while (done < count) {
      const i64 p = pos + done;
      const i64 c = p / kChunk, off = p % kChunk;
      const i64 n = std::min(count - done, kChunk - off);
      DFCG_CUDA(cudaMemcpyAsync(dst + done, chunks_[static_cast<size_t>(c)] + off, sizeof(double) * n,
                                cudaMemcpyDeviceToDevice, s));
      done += n;
    }
  }

 private:
  void ensure(i64 upto) {
    std::lock_guard<std::mutex> lock(mu_);
    while (static_cast<i64>(chunks_.size()) * kChunk < upto) grow();
  }

  // Raw 64-bit draws are sequential (mt19937_64); the Box-Muller transform runs on host
  // threads so the stream stays bit-identical to the reference's std::log/std::cos.
  void grow() {
    std::vector<std::uint64_t> raw(2 * kChunk);
    for (auto& r : raw) r = rng_.next_u64();
    std::vector<double> out(kChunk);
    const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nt; ++t)
      pool.emplace_back([&, t] {
        for (i64 i = t; i < kChunk; i += nt) {
          const double u1 = (static_cast<double>(raw[2 * i] >> 11) + 1.0) * 0x1.0p-53;
          const double u2 = static_cast<double>(raw[2 * i + 1] >> 11) * 0x1.0p-53;
          out[i] = SeededRng::box_muller(u1, u2);
        }
      });
    for (auto& th : pool) th.join();
    int prev = 0;
    DFCG_CUDA(cudaGetDevice(&prev));
    DFCG_CUDA(cudaSetDevice(device_));
    double* d = nullptr;
    DFCG_CUDA(cudaMalloc(&d, sizeof(double) * kChunk));
    DFCG_CUDA(cudaMemcpy(d, out.data(), sizeof(double) * kChunk, cudaMemcpyHostToDevice));
    DFCG_CUDA(cudaSetDevice(prev));
    chunks_.push_back(d);
  }

  int device_;
  SeededRng rng_;
  std::mutex mu_;
  std::vector<double*> chunks_;
};

}  // namespace dfcg
