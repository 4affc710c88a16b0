// exchange.hpp -- collectives among the shards of a sharded plan step.
//
// A sharded planner splits the candidates of every restart into contiguous,
// increasing ranges, shard r of W owning [n r / W, n (r + 1) / W)
// (src/planner.cpp:280-281 splits its worker ranges the same way). A round
// needs two exchanges (round.cpp):
//   1. allreduce_min_u64 of the packed per-restart winners (keypack.h), in
//      the stream between the rollout and the window select, so every shard
//      anchors its near-tie window on the GLOBAL FP32 winner;
//   2. allgather of each shard's exact (FP64, reference arithmetic) best per
//      restart after each certification pass, so every shard takes the same
//      certification decision and returns the same winner
//      (the ordered merge of src/planner.cpp:310-321).
// Implementations: NCCL (one communicator per GPU, NVLink; the ranks are
// processes or threads) and host memory (shards that are threads of one
// process on the SAME device, where NCCL refuses duplicate GPUs: the 1-GPU
// test box). NCCL is loaded at run time (libnccl.so.2, the copy torch
// loaded if any), so the library links without it.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace ppcapi {

struct Exchange {
  int rank = 0, world = 1;
  virtual ~Exchange() = default;
  // elementwise min of n uint64 at the DEVICE buffer dbuf over all ranks, in
  // place, ordered on `stream` (no host synchronization needed by NCCL)
  virtual void allreduce_min_u64(uint64_t* dbuf, int n, cudaStream_t stream) = 0;
  // HOST buffers: recv[w * bytes .. (w + 1) * bytes) = rank w's send;
  // returns when recv is complete
  virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t stream) = 0;
  virtual const char* kind() const = 0;
};

// Shards that are threads of one process: rendezvous in host memory.
struct ThreadGroup {
  explicit ThreadGroup(int w) : world(w), slots(static_cast<size_t>(w)) {}
  void barrier();  // throws once abort() was called
  void abort();    // a shard failed: release (and fail) every waiting shard
  void reset();    // before a round: no shard is waiting
  int world;
  bool aborted = false;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<std::vector<unsigned char>> slots;
};

std::unique_ptr<Exchange> make_thread_exchange(std::shared_ptr<ThreadGroup> g, int rank);

// NCCL. unique_id is ncclUniqueId (128 bytes).
constexpr int kNcclIdBytes = 128;
bool nccl_available(std::string* why = nullptr);
void nccl_unique_id(unsigned char out[kNcclIdBytes]);
// one rank of a communicator (the device must be current)
std::unique_ptr<Exchange> make_nccl_exchange(const unsigned char id[kNcclIdBytes], int world,
                                             int rank);
// a communicator over `n` distinct devices of this process (ncclCommInitAll)
std::vector<std::unique_ptr<Exchange>> make_nccl_exchanges(const int* devices, int n);

}  // namespace ppcapi
