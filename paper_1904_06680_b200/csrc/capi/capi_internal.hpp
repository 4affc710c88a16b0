// capi_internal.hpp -- internals shared by the C-ABI implementation files
// (not installed; the boundary is include/paraplan_cuda.h):
//   capi.cpp        the extern "C" entry points, construction, the plan step
//   upload.cpp      snapshots -> round constants + binned field images (HBM)
//   round.cpp       one sampling round on the device + certified re-ranking
//   host_exact.cpp  the reference's FP64 rollout and sampling on the host
// All compiled with -ffp-contract=off -fno-math-errno.
#pragma once

#include "paraplan_cuda.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../cuda/device_api.h"
#include "exchange.hpp"
#include "field.hpp"
#include "paraplan/geometry.hpp"
#include "paraplan/planner.hpp"
#include "paraplan/policy.hpp"
#include "paraplan/rng.hpp"
#include "host_pool.hpp"  // HostPool, shared_pool()

namespace ppcapi {

inline thread_local std::string g_error;  // pp_last_error()

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NoDevice : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
  }
}

template <class F>
pp_status guarded(F&& f) {
  try {
    f();
    return PP_OK;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return PP_INVALID_ARGUMENT;
  } catch (const NoDevice& e) {
    g_error = e.what();
    return PP_NO_DEVICE;
  } catch (const CudaError& e) {
    g_error = e.what();
    return PP_CUDA_ERROR;
  } catch (const std::exception& e) {
    g_error = e.what();
    return PP_RUNTIME_ERROR;
  }
}

// Device buffer that only grows.
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  // Returns true when the buffer was (re)allocated.
  bool reserve(size_t bytes, const char* what) {
    if (bytes <= cap) return false;
    if (p != nullptr) cudaFree(p);
    p = nullptr;
    cap = 0;
    ck(cudaMalloc(&p, bytes), what);
    cap = bytes;
    return true;
  }
  void release() {
    if (p != nullptr) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
  void reserve(size_t bytes, const char* what) {
    if (bytes <= cap) return;
    if (p != nullptr) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    ck(cudaMallocHost(&p, bytes), what);
    cap = bytes;
  }
  void release() {
    if (p != nullptr) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

inline paraplan::VehicleParams params_of(const pp_vehicle& v) {
  paraplan::VehicleParams p;
  p.l_f = v.l_f;
  p.l_r = v.l_r;
  p.delta_max = v.delta_max;
  p.delta_rate_max = v.delta_rate_max;
  p.u_v_min = v.u_v_min;
  p.u_v_max = v.u_v_max;
  p.overhang_front = v.overhang_front;
  p.overhang_rear = v.overhang_rear;
  p.half_width = v.half_width;
  p.T_s = v.T_s;
  return p;
}

inline paraplan::PlannerConfig config_of(const pp_config& c) {
  paraplan::PlannerConfig cfg;
  cfg.H = c.H;
  cfg.n_restarts = c.n_restarts;
  cfg.n_iter_max = c.n_iter_max;
  cfg.n_candidates = c.n_candidates;
  cfg.n_obst_pts = c.n_obst_pts;
  cfg.tol = {c.eps_xi, c.eps_eta, c.eps_phi, c.eps_v};
  cfg.sigma_log_low = c.sigma_log_low;
  cfg.sigma_log_high = c.sigma_log_high;
  cfg.master_seed = c.master_seed;
  cfg.early_exit = c.early_exit != 0;
  cfg.threads = c.threads;
  cfg.precision = c.precision;
  cfg.device = c.device;
  cfg.refine = c.refine != 0;
  return cfg;
}

struct Key {
  int cls = 0;
  double k1 = 0.0, k2 = 0.0;
};


inline bool key_better(const Key& a, const Key& b) {  // src/planner.cpp:40-44
  if (a.cls != b.cls) return a.cls > b.cls;
  if (a.k1 != b.k1) return a.k1 > b.k1;
  return a.k2 > b.k2;
}

constexpr int kSelCap = 1 << 16;    // initial selection capacity per launch (grows)
constexpr int kSelMax = 1 << 24;    // largest selection (beyond it: the FP64 round)
using ppdev::kSelFirst;             // copied back with the round result
// Round block (device, one allocation; its head is copied back in ONE D2H):
// [counters u32 x 16][exec u64 x 4 + pad][Rec x kMaxRestartsPerLaunch]
// [unflagged Rec x kMaxRestartsPerLaunch][packed keys][selected indices int64 x kSelFirst]
constexpr size_t kExecOff = 64;
constexpr size_t kRecOff = 128;
// [Rec x kMaxRestartsPerLaunch] best unflagged per restart (keys_only rounds)
constexpr size_t kFreeOff = kRecOff + sizeof(ppdev::Rec) * ppdev::kMaxRestartsPerLaunch;
// [uint64 x 2 x kMaxRestartsPerLaunch] packed winners of a sharded round
// (keypack.h), reduced across the shards in place
constexpr size_t kPackOff =
    (kFreeOff + sizeof(ppdev::Rec) * ppdev::kMaxRestartsPerLaunch + 63) / 64 * 64;
// [uint32 x kMaxRestartsPerLaunch] goal-horizon cut state (kCutNone between
// rounds) and [uint32 x kMaxRestartsPerLaunch] the round's final cut per
// restart (device_api.h kCutTGoal)
constexpr size_t kCutOff =
    (kPackOff + sizeof(uint64_t) * 2 * ppdev::kMaxRestartsPerLaunch + 63) / 64 * 64;
constexpr size_t kCutPubOff = kCutOff + sizeof(uint32_t) * ppdev::kMaxRestartsPerLaunch;
constexpr size_t kSelOff =
    (kCutPubOff + sizeof(uint32_t) * ppdev::kMaxRestartsPerLaunch + 63) / 64 * 64;
// rollouts of a restart stop cut_slack() states after its earliest t_goal
// (PARAPLAN_GOAL_CUT=0: never; PARAPLAN_CUT_SLACK overrides the slack, a
// negative one for tests of the redo path)
inline int cut_slack() {
  static const int v = [] {
    const char* e = std::getenv("PARAPLAN_CUT_SLACK");
    return e != nullptr ? std::atoi(e) : 2;
  }();
  return v;
}
// PARAPLAN_FLUSH_EVERY=k: a fixed flush period (A/B experiments only)
inline int flush_every_fixed() {
  static const int v = [] {
    const char* e = std::getenv("PARAPLAN_FLUSH_EVERY");
    return e != nullptr ? std::max(1, std::atoi(e)) : 0;
  }();
  return v;
}
inline bool goal_cut_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("PARAPLAN_GOAL_CUT");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return v;
}
constexpr size_t kRoundBytes = kSelOff + sizeof(int64_t) * kSelFirst;
// behind the round block (not in its D2H): an FP64 list round's final cut
// per source restart [uint32 x kMaxRestartsPerLaunch] and its filter's pick
// count, copied back by the certification
constexpr size_t kListCutOff = kRoundBytes;
constexpr size_t kListCountOff = kListCutOff + sizeof(uint32_t) * ppdev::kMaxRestartsPerLaunch;
constexpr size_t kListTailBytes = 512;
constexpr size_t kRoundAlloc = kRoundBytes + kListTailBytes;

// FP32 rounds are certified for every class up to this horizon, beyond it for
// class-2 (reaching) windows only (round.cpp: the error model).
inline int fp32_max_h() {
  static const int v = [] {
    const char* e = std::getenv("PARAPLAN_FP32_MAX_H");
    return e != nullptr ? std::atoi(e) : 40;
  }();
  return v;
}

// PARAPLAN_TRACE=1: one stderr line per certification pass; 2: also the
// host-side phase times of every plan step (diagnostics).
inline int trace_level() {
  static const int v = [] {
    const char* e = std::getenv("PARAPLAN_TRACE");
    return e != nullptr ? std::atoi(e) : 0;
  }();
  return v;
}
inline bool trace_on() { return trace_level() > 0; }

struct PhaseClock {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  char buf[1024] = {};
  int len = 0;
  void mark(const char* what) {
    if (trace_level() < 2 || len >= static_cast<int>(sizeof(buf)) - 1) return;
    const double us =
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    const int n = std::snprintf(buf + len, sizeof(buf) - len, " %s=%.1f", what, us);
    if (n > 0) len = std::min(static_cast<int>(sizeof(buf)) - 1, len + n);
  }
  void flush() {
    if (trace_level() >= 2) std::fprintf(stderr, "[paraplan] plan_step us:%s\n", buf);
  }
};
// the plan step being traced on this thread (planners may run on several
// threads at once, e.g. run_sweep)
inline thread_local PhaseClock* g_clock = nullptr;
inline void phase(const char* what) {
  if (g_clock != nullptr) g_clock->mark(what);
}

}  // namespace ppcapi

// The planner handle behind the opaque pp_handle of the C-ABI.
struct pp_handle {
  pp_model model{};
  std::vector<int32_t> sizes;
  paraplan::VehicleParams params;
  paraplan::PlannerConfig cfg;
  paraplan::NormConstants norm;
  std::unique_ptr<paraplan::MlpPolicy> policy;
  paraplan::ChassisPolytope chassis;
  ppfield::Box box;  // the same rectangle as (front, rear, half width)
  int P = 0;
  ppdev::NetKind kind = ppdev::NetKind::kGeneric;
  int device = 0;
  int sms = 148;  // multiprocessors of `device` (queried at construction)
  int refine_blocks = 0;  // resident refine_kernel CTAs per SM (0: not queried yet)
  bool fp64 = false;
  // FP32 planner: the last certified round needed FP64 (class 0/1 anchors
  // beyond the FP32 error envelope); the next round starts in FP64
  bool prefer_fp64 = false;
  // the next round runs every rollout to its end (a cut round whose
  // certificate the cut would break is redone so)
  bool no_cut = false;
  // the last round's winner reached the goal: the next round runs the cut's
  // kernel (round.cpp)
  bool expect_reach = true;
  // rollout warps flush finished lanes every flush_every-th iteration, sized
  // from the last round's mean rollout length (round.cpp)
  int flush_every = 3;
  int flush_min = 0;

  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // a deferred field goes up on `side` while the generator runs on `stream`;
  // the rollout waits on ev_field (the dependent launch of the rollout after
  // the generator stays intact)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_field = nullptr;
  bool field_via_side = false, field_event = false;
  ppcapi::DevBuf d_field, d_params, d_round, d_tiles, d_samples, d_scratch, d_injected, d_theta, d_skeys,
      d_sel, d_bound, d_movers, d_bin, d_selmore, d_reflist, d_listkeys, d_listout, d_listpick;
  int sel_cap = 1 << 16;  // selection capacity of this handle (kSelCap, grown on overflow)
  ppcapi::HostBuf h_field, h_params, h_round, h_bound, h_movers, h_listkeys;

  // near-tie re-ranking (PlannerConfig::refine): needs the host snapshot
  bool rerank = true;
  const pp_snapshot* snapshot = nullptr;  // -> snap_copy once a snapshot is resident
  pp_snapshot snap_copy{};
  std::vector<double> snap_warm;
  double sel_rho = 1e-3;   // FP32 window: cost <= best * (1 + rho) + 1e-6
  ppcapi::HostPool* pool = nullptr;  // exact re-evaluation of near ties (shared_pool())
  double dmarg32 = 2e-5;   // FP32 margin below which a worse-side verdict may flip
  // The certification's FP64 rollouts of each certified restart winner in
  // the current plan step (stats + trajectory, recorded while the window is
  // re-evaluated). The FP64 epilogue copies the final winner's instead of
  // re-simulating it: same function, same theta, same snapshot.
  struct WinnerRollout {
    int restart = -1, iter = -1, candidate = -1;
    pp_rollout_stats stats{};
    std::vector<double> traj;
    int32_t len = 0;
  };
  std::vector<WinnerRollout> winner_rollouts;
  std::vector<double> cert_traj;  // per window member, (H + 1) x 4 doubles
  std::vector<pp_rollout_stats> cert_stats;
  std::vector<int32_t> cert_len;

  // resident snapshot
  bool snap_valid = false;
  std::map<int64_t, ppdev::LaunchShape> shapes;  // occupancy per (smem, grid mode, precision)
  // plan_step: the field of the snapshot is binned and uploaded while the
  // theta generator runs (consumed by the first round of the step)
  std::function<void()> pending_field;
  // several GPUs in one process: the other shards' handles (this handle is
  // shard 0), a pool running one shard per thread, and each shard's
  // snapshot upload of the current plan step (done on its own thread)
  std::vector<pp_handle*> shards;
  std::unique_ptr<ppcapi::HostPool> shard_pool;
  // Sharded plan step: this handle evaluates shard `shard_rank` of
  // `shard_world` of every round's candidates and exchanges with the other
  // shards through `xchg` (NCCL, or host memory for shards sharing a
  // device); set by pp_comm_init (one process per GPU) or at construction
  // for PlannerConfig::devices (one thread per shard). The exchange is used
  // by plan steps only (xchg_active), never by pp_evaluate's explicit ranges.
  std::unique_ptr<ppcapi::Exchange> xchg;
  std::shared_ptr<ppcapi::ThreadGroup> thread_group;  // primary: host exchange of its shards
  int shard_rank = 0, shard_world = 1;
  bool xchg_active = false;
  std::function<void()> pending_upload;
  ppdev::RoundArgs base{};
  int field_smem_bytes = 0;

  pp_timing timing{};
  // resident obstacle field: FP64 binned image (host) + device images
  ppfield::Binned field;
  bool field64_ready = false;
  ppcapi::DevBuf d_field64;
  ppcapi::HostBuf h_field64;
};

namespace ppcapi {

// refine_kernel: every resident CTA of 128 threads (queried once per handle)
inline int refine_grid(pp_handle* h) {
  if (h->refine_blocks == 0) h->refine_blocks = ppdev::refine_occupancy(h->kind);
  return h->sms * h->refine_blocks;
}

// upload.cpp
void finish_field(pp_handle* h, ppdev::RoundArgs& a);
const void* ensure_field64(pp_handle* h);
void keep_snapshot(pp_handle* h, const pp_snapshot& s);
void set_round_constants(pp_handle* h, const pp_snapshot& s);
void upload_field_rows(pp_handle* h, const pp_snapshot& s, ppdev::RoundArgs& a);
void upload_points(pp_handle* h, const pp_snapshot_points& p, bool defer = false);
void upload_snapshot(pp_handle* h, const pp_snapshot& s, bool defer = false);

// round.cpp
void upload_params(pp_handle* h, ppdev::RoundArgs& a, const uint64_t* prefix, int n_prefix,
                   const double* center);
void grow_selection(pp_handle* h, ppdev::RoundArgs& a, int cap);
uint64_t key_prefix(uint64_t seed, uint64_t t, uint64_t r, uint64_t i);
ppdev::LaunchShape launch_shape(pp_handle* h, bool fp64, int field_smem, int kind);
void consume_pending_field(pp_handle* h, bool side = false);
void run_round_launch(pp_handle* h, uint64_t t, int iter, int r0, int rc, const double* center,
                      int64_t c0, int64_t c1, const double* injected, pp_record* out,
                      pp_rollout_stats* per_sample, bool force_fp64 = false);
// shard_mode: 0 unsharded; 1 sharded, the first window anchored on the
// packed global winners (in-stream allreduce); 2 sharded, anchors exchanged
// on the host first (no packed keys: n_candidates > 2^22 or H > 255)
void certify_round(pp_handle* h, ppdev::RoundArgs& a, uint64_t t, int iter, int r0, int rc,
                   const double* center, int64_t c0, int64_t c1, const double* injected,
                   pp_record* out, bool fp64, uint32_t n_sel, int shard_mode = 0);
void run_round(pp_handle* h, uint64_t t, int iter, int r0, int rc, const double* center,
               int64_t c0, int64_t c1, const double* injected, pp_record* out,
               pp_rollout_stats* per_sample);

// host_exact.cpp
void host_rollout(const pp_handle* h, const pp_snapshot& s, const double* theta,
                  pp_rollout_stats* out, double* traj, int32_t cap, int32_t* traj_len);
void host_sample(const pp_handle* h, const double* center, uint64_t t, int restart, int iter,
                 int cand, double* out, int len = -1);
bool host_stops_at_state0(const pp_handle* h, const pp_snapshot& s, pp_rollout_stats* out);

}  // namespace ppcapi
