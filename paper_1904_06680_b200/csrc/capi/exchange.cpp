// exchange.cpp -- NCCL and host-memory implementations of the shard
// exchange (exchange.hpp).
#include "exchange.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>

namespace ppcapi {

// ------------------------------------------------------------- threads ----
void ThreadGroup::barrier() {
  std::unique_lock<std::mutex> lock(mu);
  if (aborted) throw std::runtime_error("sharded round aborted by another shard");
  const uint64_t gen = generation;
  if (++arrived == world) {
    arrived = 0;
    ++generation;
    cv.notify_all();
    return;
  }
  cv.wait(lock, [&] { return generation != gen || aborted; });
  if (generation == gen) throw std::runtime_error("sharded round aborted by another shard");
}

void ThreadGroup::reset() {
  std::lock_guard<std::mutex> lock(mu);
  aborted = false;
  arrived = 0;
}

void ThreadGroup::abort() {
  std::lock_guard<std::mutex> lock(mu);
  aborted = true;
  cv.notify_all();
}

namespace {

void cuda_ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

class ThreadExchange final : public Exchange {
 public:
  ThreadExchange(std::shared_ptr<ThreadGroup> g, int r) : g_(std::move(g)) {
    rank = r;
    world = g_->world;
  }
  const char* kind() const override { return "host"; }

  void allreduce_min_u64(uint64_t* dbuf, int n, cudaStream_t stream) override {
    std::vector<uint64_t> mine(static_cast<size_t>(n));
    cuda_ck(cudaMemcpyAsync(mine.data(), dbuf, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost,
                            stream),
            "exchange D2H");
    cuda_ck(cudaStreamSynchronize(stream), "exchange sync");
    std::vector<unsigned char> all(static_cast<size_t>(world) * sizeof(uint64_t) * n);
    gather(mine.data(), all.data(), sizeof(uint64_t) * n);
    const uint64_t* a = reinterpret_cast<const uint64_t*>(all.data());
    for (int w = 0; w < world; ++w) {
      for (int i = 0; i < n; ++i) mine[i] = std::min(mine[i], a[static_cast<size_t>(w) * n + i]);
    }
    cuda_ck(cudaMemcpyAsync(dbuf, mine.data(), sizeof(uint64_t) * n, cudaMemcpyHostToDevice,
                            stream),
            "exchange H2D");
    cuda_ck(cudaStreamSynchronize(stream), "exchange sync");
  }

  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t) override {
    gather(send, recv, bytes);
  }

 private:
  void gather(const void* send, void* recv, size_t bytes) {
    {
      std::lock_guard<std::mutex> lock(g_->mu);
      auto& s = g_->slots[static_cast<size_t>(rank)];
      s.assign(static_cast<const unsigned char*>(send),
               static_cast<const unsigned char*>(send) + bytes);
    }
    g_->barrier();  // every slot written
    {
      std::lock_guard<std::mutex> lock(g_->mu);
      for (int w = 0; w < world; ++w) {
        const auto& s = g_->slots[static_cast<size_t>(w)];
        if (s.size() != bytes) throw std::logic_error("exchange size mismatch between shards");
        std::memcpy(static_cast<unsigned char*>(recv) + static_cast<size_t>(w) * bytes, s.data(),
                    bytes);
      }
    }
    g_->barrier();  // every slot read before the next exchange overwrites it
  }
  std::shared_ptr<ThreadGroup> g_;
};

// ---------------------------------------------------------------- NCCL ----
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string why;
  bool ok = false;
};

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    // the copy torch (or another library) already mapped, else the system's
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (lib == nullptr) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (lib == nullptr) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (lib == nullptr) {
      a.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return a;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(lib, name));
      if (fn == nullptr) a.why = std::string("NCCL symbol missing: ") + name;
    };
    sym(a.get_unique_id, "ncclGetUniqueId");
    sym(a.comm_init_rank, "ncclCommInitRank");
    sym(a.comm_init_all, "ncclCommInitAll");
    sym(a.comm_destroy, "ncclCommDestroy");
    sym(a.all_reduce, "ncclAllReduce");
    sym(a.all_gather, "ncclAllGather");
    sym(a.error_string, "ncclGetErrorString");
    a.ok = a.why.empty();
    return a;
  }();
  return api;
}

void nccl_ck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    throw std::runtime_error(std::string(what) + ": " + nccl().error_string(r));
  }
}

const NcclApi& need_nccl() {
  const NcclApi& a = nccl();
  if (!a.ok) throw std::runtime_error("NCCL unavailable: " + a.why);
  return a;
}

class NcclExchange final : public Exchange {
 public:
  NcclExchange(ncclComm_t c, int r, int w) : comm_(c) {
    rank = r;
    world = w;
  }
  ~NcclExchange() override {
    if (d_send_ != nullptr) cudaFree(d_send_);
    if (d_recv_ != nullptr) cudaFree(d_recv_);
    if (comm_ != nullptr) nccl().comm_destroy(comm_);
  }
  const char* kind() const override { return "nccl"; }

  void allreduce_min_u64(uint64_t* dbuf, int n, cudaStream_t stream) override {
    nccl_ck(nccl().all_reduce(dbuf, dbuf, static_cast<size_t>(n), ncclUint64, ncclMin, comm_,
                              stream),
            "ncclAllReduce(min, uint64)");
  }

  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t stream) override {
    if (bytes > cap_) {
      if (d_send_ != nullptr) cudaFree(d_send_);
      if (d_recv_ != nullptr) cudaFree(d_recv_);
      d_send_ = d_recv_ = nullptr;
      cap_ = 0;
      cuda_ck(cudaMalloc(&d_send_, bytes), "exchange buffer");
      cuda_ck(cudaMalloc(&d_recv_, bytes * static_cast<size_t>(world)), "exchange buffer");
      cap_ = bytes;
    }
    cuda_ck(cudaMemcpyAsync(d_send_, send, bytes, cudaMemcpyHostToDevice, stream), "exchange H2D");
    nccl_ck(nccl().all_gather(d_send_, d_recv_, bytes, ncclUint8, comm_, stream), "ncclAllGather");
    cuda_ck(cudaMemcpyAsync(recv, d_recv_, bytes * static_cast<size_t>(world),
                            cudaMemcpyDeviceToHost, stream),
            "exchange D2H");
    cuda_ck(cudaStreamSynchronize(stream), "exchange sync");
  }

 private:
  ncclComm_t comm_ = nullptr;
  void* d_send_ = nullptr;
  void* d_recv_ = nullptr;
  size_t cap_ = 0;
};

}  // namespace

std::unique_ptr<Exchange> make_thread_exchange(std::shared_ptr<ThreadGroup> g, int rank) {
  return std::make_unique<ThreadExchange>(std::move(g), rank);
}

bool nccl_available(std::string* why) {
  const NcclApi& a = nccl();
  if (!a.ok && why != nullptr) *why = a.why;
  return a.ok;
}

void nccl_unique_id(unsigned char out[kNcclIdBytes]) {
  static_assert(sizeof(ncclUniqueId) == kNcclIdBytes, "ncclUniqueId size");
  ncclUniqueId id;
  nccl_ck(need_nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, kNcclIdBytes);
}

std::unique_ptr<Exchange> make_nccl_exchange(const unsigned char id[kNcclIdBytes], int world,
                                             int rank) {
  ncclUniqueId uid;
  std::memcpy(&uid, id, kNcclIdBytes);
  ncclComm_t c = nullptr;
  nccl_ck(need_nccl().comm_init_rank(&c, world, uid, rank), "ncclCommInitRank");
  return std::make_unique<NcclExchange>(c, rank, world);
}

std::vector<std::unique_ptr<Exchange>> make_nccl_exchanges(const int* devices, int n) {
  std::vector<ncclComm_t> comms(static_cast<size_t>(n), nullptr);
  nccl_ck(need_nccl().comm_init_all(comms.data(), n, devices), "ncclCommInitAll");
  std::vector<std::unique_ptr<Exchange>> out;
  for (int k = 0; k < n; ++k) out.push_back(std::make_unique<NcclExchange>(comms[k], k, n));
  return out;
}

}  // namespace ppcapi
