// Transports of the multi-GPU combine (see dist.hpp).
#include "dist.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>

namespace dfcg {

namespace {

// ---------------------------------------------------------------- NCCL, loaded at run time
// libdfcg.so does not link NCCL: the process's already-loaded libnccl.so.2 (torch's, when the
// caller initialised torch.distributed) is reused, else DFCG_NCCL_LIB, else the loader path.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h && std::getenv("DFCG_NCCL_LIB")) h = dlopen(std::getenv("DFCG_NCCL_LIB"), RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p && err.empty()) err = std::string("libnccl.so.2 lacks ") + name;
      return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!err.empty()) throw NcclError(err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw NcclError(std::string(what) + " failed: " + nccl().GetErrorString(r));
}

class NcclComm final : public Comm {
 public:
  NcclComm(int nranks, int rank, const unsigned char id[128], int device) : Comm(nranks, rank), device_(device) {
    const NcclApi& api = nccl();
    ncclUniqueId uid;
    static_assert(sizeof(uid) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(&uid, id, sizeof(uid));
    DFCG_CUDA(cudaSetDevice(device));
    nccl_check(api.CommInitRank(&comm_, nranks, uid, rank), "ncclCommInitRank");
    DFCG_CUDA(cudaMalloc(&scratch_, kScratch));
  }
  ~NcclComm() override {
    if (comm_) nccl().CommDestroy(comm_);
    if (scratch_) cudaFree(scratch_);
  }
  void bcast(void* buf, size_t bytes, int root, cudaStream_t s) override {
    if (size() == 1 || bytes == 0) return;
    nccl_check(nccl().Broadcast(buf, buf, bytes, ncclUint8, root, comm_, s), "ncclBroadcast");
  }
  void exchange(const std::vector<Xfer>& ops, cudaStream_t s) override {
    const NcclApi& api = nccl();
    bool grouped = false;
    for (const Xfer& x : ops) {
      if (x.bytes == 0) continue;
      if (x.src == x.dst) {
        if (x.src == rank() && x.recv_buf != x.send_buf)
          DFCG_CUDA(cudaMemcpyAsync(x.recv_buf, x.send_buf, x.bytes, cudaMemcpyDeviceToDevice, s));
        continue;
      }
      if (x.src != rank() && x.dst != rank()) continue;
      if (!grouped) {
        nccl_check(api.GroupStart(), "ncclGroupStart");
        grouped = true;
      }
      if (x.src == rank()) nccl_check(api.Send(x.send_buf, x.bytes, ncclUint8, x.dst, comm_, s), "ncclSend");
      else nccl_check(api.Recv(x.recv_buf, x.bytes, ncclUint8, x.src, comm_, s), "ncclRecv");
    }
    if (grouped) nccl_check(api.GroupEnd(), "ncclGroupEnd");
  }
  void bcast_host(void* buf, size_t bytes, int root) override {
    if (size() == 1 || bytes == 0) return;
    cudaStream_t s = nullptr;
    DFCG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    for (size_t off = 0; off < bytes; off += kScratch) {
      const size_t n = std::min(kScratch, bytes - off);
      char* hb = static_cast<char*>(buf) + off;
      if (rank() == root) DFCG_CUDA(cudaMemcpyAsync(scratch_, hb, n, cudaMemcpyHostToDevice, s));
      nccl_check(nccl().Broadcast(scratch_, scratch_, n, ncclUint8, root, comm_, s), "ncclBroadcast");
      DFCG_CUDA(cudaMemcpyAsync(hb, scratch_, n, cudaMemcpyDeviceToHost, s));
      DFCG_CUDA(cudaStreamSynchronize(s));
    }
    cudaStreamDestroy(s);
  }
  void p2p_host(void* buf, size_t bytes, int src, int dst) override {
    if (src == dst || bytes == 0) return;
    cudaStream_t s = nullptr;
    DFCG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    for (size_t off = 0; off < bytes; off += kScratch) {
      const size_t n = std::min(kScratch, bytes - off);
      char* hb = static_cast<char*>(buf) + off;
      if (rank() == src) {
        DFCG_CUDA(cudaMemcpyAsync(scratch_, hb, n, cudaMemcpyHostToDevice, s));
        nccl_check(nccl().Send(scratch_, n, ncclUint8, dst, comm_, s), "ncclSend");
      } else {
        nccl_check(nccl().Recv(scratch_, n, ncclUint8, src, comm_, s), "ncclRecv");
        DFCG_CUDA(cudaMemcpyAsync(hb, scratch_, n, cudaMemcpyDeviceToHost, s));
      }
      DFCG_CUDA(cudaStreamSynchronize(s));
    }
    cudaStreamDestroy(s);
  }

 private:
  static constexpr size_t kScratch = size_t{1} << 20;
  int device_;
  ncclComm_t comm_ = nullptr;
  void* scratch_ = nullptr;
};

// ---------------------------------------------------------------- host callbacks
class HostComm final : public Comm {
 public:
  HostComm(int nranks, int rank, const dfcg_host_transport& t) : Comm(nranks, rank), t_(t) {
    if (!t.bcast || !t.send || !t.recv) throw std::invalid_argument("dfcg_host_transport: null callback");
  }
  ~HostComm() override {
    if (pinned_) cudaFreeHost(pinned_);
  }
  void bcast(void* buf, size_t bytes, int root, cudaStream_t s) override {
    if (size() == 1 || bytes == 0) return;
    char* h = stage(bytes);
    if (rank() == root) {
      DFCG_CUDA(cudaMemcpyAsync(h, buf, bytes, cudaMemcpyDeviceToHost, s));
      DFCG_CUDA(cudaStreamSynchronize(s));
    }
    bcast_host(h, bytes, root);
    if (rank() != root) {
      DFCG_CUDA(cudaMemcpyAsync(buf, h, bytes, cudaMemcpyHostToDevice, s));
      DFCG_CUDA(cudaStreamSynchronize(s));
    }
  }
  void exchange(const std::vector<Xfer>& ops, cudaStream_t s) override {
    for (const Xfer& x : ops) {
      if (x.bytes == 0 || (x.src != rank() && x.dst != rank())) continue;
      if (x.src == x.dst) {
        if (x.recv_buf != x.send_buf)
          DFCG_CUDA(cudaMemcpyAsync(x.recv_buf, x.send_buf, x.bytes, cudaMemcpyDeviceToDevice, s));
        continue;
      }
      char* h = stage(x.bytes);
      if (x.src == rank()) {
        DFCG_CUDA(cudaMemcpyAsync(h, x.send_buf, x.bytes, cudaMemcpyDeviceToHost, s));
        DFCG_CUDA(cudaStreamSynchronize(s));
        call(t_.send(t_.user, h, static_cast<int64_t>(x.bytes), x.dst), "send");
      } else {
        call(t_.recv(t_.user, h, static_cast<int64_t>(x.bytes), x.src), "recv");
        DFCG_CUDA(cudaMemcpyAsync(x.recv_buf, h, x.bytes, cudaMemcpyHostToDevice, s));
        DFCG_CUDA(cudaStreamSynchronize(s));
      }
    }
  }
  void bcast_host(void* buf, size_t bytes, int root) override {
    if (size() == 1 || bytes == 0) return;
    call(t_.bcast(t_.user, buf, static_cast<int64_t>(bytes), root), "bcast");
  }
  void p2p_host(void* buf, size_t bytes, int src, int dst) override {
    if (src == dst || bytes == 0) return;
    if (rank() == src) call(t_.send(t_.user, buf, static_cast<int64_t>(bytes), dst), "send");
    else call(t_.recv(t_.user, buf, static_cast<int64_t>(bytes), src), "recv");
  }

 private:
  static void call(int rc, const char* what) {
    if (rc != 0) throw NcclError(std::string("host transport ") + what + " failed (" + std::to_string(rc) + ")");
  }
  char* stage(size_t bytes) {
    if (bytes > cap_) {
      if (pinned_) DFCG_CUDA(cudaFreeHost(pinned_));
      pinned_ = nullptr;
      DFCG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&pinned_), bytes));
      cap_ = bytes;
    }
    return pinned_;
  }
  dfcg_host_transport t_;
  char* pinned_ = nullptr;
  size_t cap_ = 0;
};

}  // namespace

int Comm::selftest() {
  // host-only pattern: a broadcast from every root, then a ring of point-to-point messages
  // through the callbacks (HostComm) or the NCCL scratch path; every rank checks what it got
  const int n = size(), r = rank();
  int bad = 0;
  for (int root = 0; root < n; ++root) {
    std::vector<std::int64_t> v(257, r == root ? 1000 * root + 7 : -1);
    bcast_host(v.data(), sizeof(std::int64_t) * v.size(), root);
    for (auto x : v) bad += x != 1000 * root + 7;
  }
  // ring of point-to-point messages in one global order (src = 0, 1, ...): rank q sends to q + 1
  for (int src = 0; src < n && n > 1; ++src) {
    const int dst = (src + 1) % n;
    if (r != src && r != dst) continue;
    std::vector<std::int64_t> v(1031, r == src ? 77 * src + 1 : -1);
    p2p_host(v.data(), sizeof(std::int64_t) * v.size(), src, dst);
    if (r == dst)
      for (auto x : v) bad += x != 77 * src + 1;
  }
  return bad;
}

void nccl_unique_id(unsigned char id[128]) {
  ncclUniqueId uid;
  nccl_check(nccl().GetUniqueId(&uid), "ncclGetUniqueId");
  std::memcpy(id, &uid, 128);
}

std::unique_ptr<Comm> make_nccl_comm(int nranks, int rank, const unsigned char id[128], int device) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("comm: need 0 <= rank < nranks");
  return std::make_unique<NcclComm>(nranks, rank, id, device);
}

std::unique_ptr<Comm> make_host_comm(int nranks, int rank, const dfcg_host_transport& t) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("comm: need 0 <= rank < nranks");
  return std::make_unique<HostComm>(nranks, rank, t);
}

std::vector<int> assign_blocks_lpt(const std::vector<i64>& nnz, int nranks) {
  if (nranks < 1) throw std::invalid_argument("assign_blocks: nranks must be >= 1");
  std::vector<size_t> ord(nnz.size());
  std::iota(ord.begin(), ord.end(), size_t{0});
  std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return nnz[a] > nnz[b]; });
  std::vector<i64> load(static_cast<size_t>(nranks), 0);
  std::vector<int> count(static_cast<size_t>(nranks), 0), owner(nnz.size(), 0);
  for (size_t g : ord) {
    int best = 0;
    for (int q = 1; q < nranks; ++q) {
      // least load; ties: fewer blocks (empty blocks still cost a slot), then the lower rank
      if (load[q] < load[best] || (load[q] == load[best] && count[q] < count[best])) best = q;
    }
    owner[g] = best;
    load[best] += std::max<i64>(nnz[g], 0);
    ++count[best];
  }
  return owner;
}

}  // namespace dfcg
