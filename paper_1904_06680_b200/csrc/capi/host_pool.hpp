// host_pool.hpp -- the process-wide host worker pool: the certification's
// exact re-evaluation of near ties (round.cpp) and the parallel loops of the
// field binning (field.cpp) share it.
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace ppcapi {

// Fork-join pool for the host's exact re-evaluation of near-tie candidates.
// prewarm() is called when a round is launched: the workers wake and spin
// for the job (up to a few ms) while the GPU works, so the fork itself costs
// no thread wake-up latency.
class HostPool {
 public:
  explicit HostPool(int n) {
    for (int i = 1; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lock(mu_);
      stop_.store(true);
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  int size() const { return static_cast<int>(workers_.size()) + 1; }
  void prewarm() {
    {
      std::lock_guard<std::mutex> lock(mu_);
      warm_.fetch_add(1);
    }
    cv_.notify_all();
  }
  // fn(i) for i in [0, n), spread over the workers and the caller.
  void run(int n, const std::function<void(int)>& fn) {
    fn_ = &fn;
    n_ = n;
    next_.store(0);
    done_.store(0);
    {
      std::lock_guard<std::mutex> lock(mu_);
      job_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    drain();
    const int workers = static_cast<int>(workers_.size());
    while (done_.load(std::memory_order_acquire) < workers) std::this_thread::yield();
  }

 private:
  void drain() {
    for (int i; (i = next_.fetch_add(1)) < n_;) (*fn_)(i);
  }
  void loop() {
    uint64_t seen_job = 0, seen_warm = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lock(mu_);
        cv_.wait(lock, [&] {
          return stop_.load() || job_.load() != seen_job || warm_.load() != seen_warm;
        });
        if (stop_.load()) return;
        seen_warm = warm_.load();
      }
      const auto t0 = std::chrono::steady_clock::now();
      while (job_.load(std::memory_order_acquire) == seen_job && !stop_.load() &&
             std::chrono::steady_clock::now() - t0 < std::chrono::milliseconds(5)) {
      }
      if (job_.load(std::memory_order_acquire) != seen_job) {
        seen_job = job_.load(std::memory_order_acquire);
        drain();
        done_.fetch_add(1, std::memory_order_release);
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_;
  const std::function<void(int)>* fn_ = nullptr;
  std::atomic<int> next_{0}, done_{0};
  int n_ = 0;
  std::atomic<uint64_t> job_{0}, warm_{0};
  std::atomic<bool> stop_{false};
};

// One certification pool per process, shared by every planner handle (a
// run_sweep drives several planners at once; one pool per planner would
// oversubscribe the host with spinning workers). One thread per host core
// but one; callers take turns (lock()), a certification is tens of us.
struct SharedPool {
  std::mutex mu;
  std::unique_ptr<HostPool> pool;
};
inline SharedPool& shared_pool() {
  static SharedPool* sp = [] {
    auto* p = new SharedPool;  // never destroyed: planners may outlive statics
    const unsigned hc = std::thread::hardware_concurrency();
    p->pool = std::make_unique<HostPool>(static_cast<int>(std::max(1u, hc > 1 ? hc - 1 : 1u)));
    return p;
  }();
  return *sp;
}

}  // namespace ppcapi
