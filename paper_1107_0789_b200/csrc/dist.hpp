// Multi-GPU transport for the DFC combine (one process per GPU).
//
// The reference runs every subproblem on one machine (parallel_for worker threads,
// P/include/dfc/dfc.hpp:84-147); the multi-GPU split keeps its semantics: the t F-step
// subproblems are independent (no exchange during the solve), and only the C step moves
// factors between ranks: a broadcast of the anchor basis U_b (m x k_b) and a
// gather of the per-block projected rows (w_g x k_b), or the R-hat factors for DFC-Nys.
//
// Two transports behind one interface, both stream-ordered on device buffers:
//   NcclComm  NCCL over NVLink / NVSwitch (libnccl.so.2 loaded at run time; the communicator is
//             created from an ncclUniqueId the caller distributes, e.g. with torch.distributed);
//   HostComm  caller-provided host callbacks (dfcg_host_transport): device data is staged through
//             pinned host memory — the CPU (gloo) test transport and a fallback for boxes
//             without NCCL.
#pragma once

#include <memory>
#include <vector>

#include "../../include/dfcg.h"
#include "common.cuh"

namespace dfcg {

struct NcclError : std::runtime_error {  // -> DFCG_ENCCL at the C ABI
  using std::runtime_error::runtime_error;
};

class Comm {
 public:
  Comm(int nranks, int rank) : nranks_(nranks), rank_(rank) {}
  virtual ~Comm() = default;
  int size() const { return nranks_; }
  int rank() const { return rank_; }

  // bytes at buf (device) from `root` to every rank, ordered on stream s
  virtual void bcast(void* buf, size_t bytes, int root, cudaStream_t s) = 0;

  // A batch of point-to-point transfers. Every rank passes the SAME global list (the ops it is
  // not part of are skipped): NCCL issues its own ops in one group, the host transport walks the
  // list in order, so blocking sends and receives pair up without deadlock.
  struct Xfer {
    int src, dst;
    void* send_buf;  // valid on src (device)
    void* recv_buf;  // valid on dst (device)
    size_t bytes;
  };
  virtual void exchange(const std::vector<Xfer>& ops, cudaStream_t s) = 0;

  // host-side scalars (block reports, ranks): bytes at host buffer from root
  virtual void bcast_host(void* buf, size_t bytes, int root) = 0;
  // host buffer from src to dst (both ranks call it; others must not)
  virtual void p2p_host(void* buf, size_t bytes, int src, int dst) = 0;

  // test hook: host-only traffic pattern through the transport (no CUDA), returns 0 when every
  // rank received the expected bytes
  int selftest();

 private:
  int nranks_, rank_;
};

void nccl_unique_id(unsigned char id[128]);
std::unique_ptr<Comm> make_nccl_comm(int nranks, int rank, const unsigned char id[128], int device);
std::unique_ptr<Comm> make_host_comm(int nranks, int rank, const dfcg_host_transport& t);

// Longest-processing-time assignment of subproblems to ranks by observation count: blocks in
// descending nnz (ties: lower index first), each to the currently least-loaded rank (ties:
// lower rank). Deterministic, so every rank computes the same owner table.
std::vector<int> assign_blocks_lpt(const std::vector<i64>& nnz, int nranks);

}  // namespace dfcg
