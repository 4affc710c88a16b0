// capi.cpp -- implementation of the C-ABI in include/paraplan_cuda.h.
//
// Host side of Planner::plan_step (src/planner.cpp:238-351 in the reference):
//   * validation with the reference's messages,
//   * snapshot staging (pinned host -> HBM, one copy per tick),
//   * the restart x iteration schedule: with n_iter_max == 1 every candidate
//     of every restart is independent (each restart re-centres on the warm
//     start, :271-277) and the whole tick is ONE kernel launch; iterations
//     >= 1 centre on the incumbent and run as dependent rounds,
//   * the ordered, strict-better merge of round winners (:310-330),
//   * the FP64 epilogue (:339-350) on the host, bit-identical to the
//     reference because best_theta is regenerated with the host KeyedRng and
//     re-simulated through the same FP64 primitives.
// Compiled with -ffp-contract=off -fno-math-errno.
#include "paraplan_cuda.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <map>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "../cuda/device_api.h"
#include "field.hpp"
#include "paraplan/geometry.hpp"
#include "paraplan/planner.hpp"
#include "paraplan/policy.hpp"
#include "paraplan/rng.hpp"

namespace {

thread_local std::string g_error;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NoDevice : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
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

paraplan::VehicleParams params_of(const pp_vehicle& v) {
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

paraplan::PlannerConfig config_of(const pp_config& c) {
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

bool key_better(const Key& a, const Key& b) {  // src/planner.cpp:40-44
  if (a.cls != b.cls) return a.cls > b.cls;
  if (a.k1 != b.k1) return a.k1 > b.k1;
  return a.k2 > b.k2;
}

}  // namespace

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
  bool fp64 = false;

  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // a deferred field goes up on `side` while the generator runs on `stream`;
  // the rollout waits on ev_field (the dependent launch of the rollout after
  // the generator stays intact)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_field = nullptr;
  bool field_via_side = false, field_event = false;
  DevBuf d_field, d_params, d_round, d_tiles, d_samples, d_scratch, d_injected, d_theta, d_skeys,
      d_sel, d_bound, d_movers, d_bin;
  HostBuf h_field, h_params, h_round, h_bound, h_movers;

  // near-tie re-ranking (PlannerConfig::refine): needs the host snapshot
  bool rerank = true;
  const pp_snapshot* snapshot = nullptr;  // -> snap_copy once a snapshot is resident
  pp_snapshot snap_copy{};
  std::vector<double> snap_warm;
  double sel_rho = 1e-3;   // FP32 window: cost <= best * (1 + rho) + 1e-6
  std::unique_ptr<HostPool> pool;  // exact re-evaluation of near ties
  double dmarg32 = 2e-5;   // FP32 margin below which a worse-side verdict may flip

  // resident snapshot
  bool snap_valid = false;
  std::map<int64_t, ppdev::LaunchShape> shapes;  // occupancy per (smem, grid mode, precision)
  // plan_step: the field of the snapshot is binned and uploaded while the
  // theta generator runs (consumed by the first round of the step)
  std::function<void()> pending_field;
  ppdev::RoundArgs base{};
  int field_smem_bytes = 0;

  pp_timing timing{};
  // resident obstacle field: FP64 binned image (host) + device images
  ppfield::Binned field;
  bool field64_ready = false;
  DevBuf d_field64;
  HostBuf h_field64;
};

namespace {

// Round constants in the compute precision (rounded once from FP64).
template <typename Real>
void fill_consts(const ppdev::RoundArgs& a, ppdev::ConstsT<Real>* k) {
  k->gx = Real(a.gx);
  k->gy = Real(a.gy);
  k->gphi = Real(a.gphi);
  k->gv = Real(a.gv);
  k->gcos = Real(a.gcos);
  k->gsin = Real(a.gsin);
  k->v0 = Real(a.v0);
  k->act0 = Real(a.act0);
  k->pa0 = Real(a.pa0);
  k->inv_xi = Real(1.0 / a.d_xi);
  k->inv_eta = Real(1.0 / a.d_eta);
  k->inv_phi = Real(1.0 / a.d_phi);
  k->inv_v = Real(1.0 / a.d_v);
  k->d_xi = a.d_xi;
  k->d_eta = a.d_eta;
  k->d_phi = a.d_phi;
  k->d_v = a.d_v;
  k->eps_xi = Real(a.eps_xi);
  k->eps_eta = Real(a.eps_eta);
  k->eps_phi = Real(a.eps_phi);
  k->eps_v = Real(a.eps_v);
  k->dmax = Real(a.delta_max);
  k->window = Real(a.window);
  k->l_r = Real(a.l_r);
  k->wb = Real(a.wheelbase);
  k->Ts = Real(a.T_s);
  k->umin = Real(a.u_v_min);
  k->umax = Real(a.u_v_max);
  k->fe = Real(a.fe);
  k->re = Real(a.re);
  k->hw = Real(a.hw);
  k->r2 = Real(a.r2);
  const double cull = std::sqrt(a.r2) + 1e-3;
  k->cull = Real(cull);
  k->bx0 = Real(a.grid_x0);
  k->by0 = Real(a.grid_y0);
  k->binv = Real(1.0 / a.grid_g);
  k->qpad = Real(a.grid_g / 8.0);
  // a discrete verdict whose margin is below this may flip under rounding
  k->dmarg = sizeof(Real) == sizeof(float) ? Real(a.dmarg32) : Real(1e-9);
  k->bcx = Real(0.5 * (a.fe - a.re));
  k->bhx = Real(0.5 * (a.fe + a.re));
  k->inv_wb = Real(1.0 / a.wheelbase);
  k->wb_d = a.wheelbase;
  k->tan_small = a.delta_max <= 0.785 ? 1 : 0;
}

// Device image of h->field in the compute precision (one H2D); the FP64 image
// for the near-tie re-ranking is uploaded only when a round needs it.
void finish_field(pp_handle* h, ppdev::RoundArgs& a) {
  const ppfield::Binned& b = h->field;
  a.field_ns = b.Ns;
  a.field_nd = b.Nd;
  a.grid_nx = b.nx;
  a.grid_ny = b.ny;
  a.grid_x0 = b.x0;
  a.grid_y0 = b.y0;
  a.grid_g = b.g;
  a.grid_mode = b.mode();
  const size_t elem = h->fp64 ? sizeof(double) : sizeof(float);
  const ppfield::Layout l = ppfield::layout(b, elem), l64 = ppfield::layout(b, sizeof(double));
  a.lay = {static_cast<int64_t>(l.dpts), static_cast<int64_t>(l.sst), static_cast<int64_t>(l.dst),
           static_cast<int64_t>(l.sbox), static_cast<int64_t>(l.bytes)};
  a.lay64 = {static_cast<int64_t>(l64.dpts), static_cast<int64_t>(l64.sst),
             static_cast<int64_t>(l64.dst), static_cast<int64_t>(l64.sbox),
             static_cast<int64_t>(l64.bytes)};
  a.field = nullptr;
  a.field64 = nullptr;
  h->field64_ready = false;
  if (b.points() > 0) {
    h->h_field.reserve(l.bytes, "pinned field");
    h->d_field.reserve(l.bytes, "device field");
    cudaStream_t st = h->field_via_side ? h->side : h->stream;
    if (b.dyn_deferred) {
      // the device bins the movers itself: upload the static parts and the
      // raw movers only (csrc/cuda/binning_f64.cu)
      ppfield::pack(b, h->fp64, h->h_field.p, false);
      unsigned char* hf = static_cast<unsigned char*>(h->h_field.p);
      unsigned char* df = static_cast<unsigned char*>(h->d_field.p);
      const auto part = [&](size_t lo, size_t hi) {
        if (hi > lo) {
          ck(cudaMemcpyAsync(df + lo, hf + lo, hi - lo, cudaMemcpyHostToDevice, st), "field H2D");
          h->timing.h2d_bytes += static_cast<int64_t>(hi - lo);
        }
      };
      part(0, l.dpts);       // static points
      part(l.sst, l.dst);    // static starts
      part(l.sbox, l.bytes); // static cell boxes
      const size_t mb = sizeof(double) * b.dbase.size();
      h->h_movers.reserve(mb, "pinned movers");
      h->d_movers.reserve(mb, "device movers");
      std::memcpy(h->h_movers.p, b.dbase.data(), mb);
      ck(cudaMemcpyAsync(h->d_movers.p, h->h_movers.p, mb, cudaMemcpyHostToDevice, st),
         "movers H2D");
      h->timing.h2d_bytes += static_cast<int64_t>(mb);
      h->d_bin.reserve(sizeof(int32_t) * static_cast<size_t>(b.rows) * b.cells(), "bin cursors");
      ppdev::BinArgs ba{};
      ba.movers = static_cast<const double*>(h->d_movers.p);
      ba.Nd = b.Nd;
      ba.rows = b.rows;
      ba.nx = b.nx;
      ba.ny = b.ny;
      ba.x0 = b.x0;
      ba.y0 = b.y0;
      ba.inv_g = 1.0 / b.g;
      ba.dpts = df + l.dpts;
      ba.dst = reinterpret_cast<int32_t*>(df + l.dst);
      ba.cursor = static_cast<int32_t*>(h->d_bin.p);
      ba.fp64 = h->fp64 ? 1 : 0;
      ck(static_cast<cudaError_t>(ppdev::bin_movers(ba, st)), "mover binning");
      h->timing.launches += 3;
    } else {
      ppfield::pack(b, h->fp64, h->h_field.p);
      ck(cudaMemcpyAsync(h->d_field.p, h->h_field.p, l.bytes, cudaMemcpyHostToDevice, st),
         "field H2D");
      h->timing.h2d_bytes += static_cast<int64_t>(l.bytes);
    }
    if (h->field_via_side) {
      ck(cudaEventRecord(h->ev_field, h->side), "field event");
      h->field_event = true;
    }
    a.field = h->d_field.p;
    if (h->fp64) {
      a.field64 = h->d_field.p;
      h->field64_ready = true;
    }
  }
  a.dmarg32 = h->dmarg32;
  fill_consts(a, &a.kf);
  fill_consts(a, &a.kd);
  // stage the field in shared memory when it fits; larger fields are read
  // through L1/L2
  h->field_smem_bytes = (b.points() > 0 && l.bytes <= 40 * 1024) ? static_cast<int>(l.bytes) : 0;
}

// FP64 field image on the device (FP32 rounds that need the FP64 refine or
// the FP64 fallback).
const void* ensure_field64(pp_handle* h) {
  if (h->field.points() == 0) return nullptr;
  ppfield::bin_dynamic(h->field);
  if (!h->field64_ready) {
    const ppfield::Layout l64 = ppfield::layout(h->field, sizeof(double));
    h->h_field64.reserve(l64.bytes, "pinned field64");
    h->d_field64.reserve(l64.bytes, "device field64");
    ppfield::pack(h->field, true, h->h_field64.p);
    ck(cudaMemcpyAsync(h->d_field64.p, h->h_field64.p, l64.bytes, cudaMemcpyHostToDevice,
                       h->stream),
       "field64 H2D");
    h->timing.h2d_bytes += static_cast<int64_t>(l64.bytes);
    h->field64_ready = true;
  }
  return h->d_field64.p;
}

void set_round_constants(pp_handle* h, const pp_snapshot& s);
void upload_field_rows(pp_handle* h, const pp_snapshot& s, ppdev::RoundArgs& a);

// Mover sets of at least this many positions (rows x movers) are binned on
// the device in a plan step.
int64_t device_bin_min() {
  static const int64_t v = [] {
    const char* e = std::getenv("PARAPLAN_DEVICE_BIN_MIN");
    return e != nullptr ? std::atoll(e) : int64_t{1} << 16;
  }();
  return v;
}

// Host copy of the snapshot scalars (+ warm start) for the epilogue and the
// certification; the field lives in h->field.
void keep_snapshot(pp_handle* h, const pp_snapshot& s) {
  h->snap_copy = s;
  h->snap_copy.field_xy = nullptr;
  h->snap_copy.field_H = h->cfg.H;
  h->snap_warm.assign(s.warm_theta, s.warm_theta + std::max(0, s.warm_theta_len));
  h->snap_copy.warm_theta = h->snap_warm.data();
  h->snapshot = &h->snap_copy;
  h->snap_valid = true;
}

// Snapshot with raw anchor-frame obstacle points: the field is the
// reference's extrapolate(points, H, T_s) (src/geometry.cpp:43-61), built
// straight into the binned static/dynamic form.
void upload_points(pp_handle* h, const pp_snapshot_points& p, bool defer = false) {
  const auto& cfg = h->cfg;
  if (p.n_points < 0) throw std::invalid_argument("malformed obstacle points");
  if (p.n_points > 0 && p.points == nullptr) throw std::invalid_argument("null obstacle points");
  pp_snapshot s{};
  s.ev_x = p.ev_x;
  s.ev_y = p.ev_y;
  s.ev_phi = p.ev_phi;
  s.ev_v = p.ev_v;
  s.actuator_delta = p.actuator_delta;
  s.prev_a0 = p.prev_a0;
  s.prev_a1 = p.prev_a1;
  s.goal_x = p.goal_x;
  s.goal_y = p.goal_y;
  s.goal_phi = p.goal_phi;
  s.goal_v = p.goal_v;
  s.field_xy = nullptr;
  s.field_H = cfg.H;
  s.n_points = p.n_points;
  s.warm_theta = p.warm_theta;
  s.warm_theta_len = p.warm_theta_len;
  set_round_constants(h, s);
  keep_snapshot(h, s);
  // In a plan step the device bins large mover sets itself and the host
  // bins its exact FP64 image while the round runs.
  auto field = [h, p, defer] {
    ppdev::RoundArgs& a = h->base;
    a.n_points = p.n_points;
    const double cull = std::sqrt(a.r2) + 1e-3;
    ppfield::from_points(h->field, p.points, p.n_points, h->cfg.H + 1, p.T_s, cull, defer);
    if (h->field.dyn_deferred &&
        static_cast<int64_t>(h->field.Nd) * h->field.rows < device_bin_min()) {
      ppfield::bin_dynamic(h->field);  // small: the host bins it at once
    }
    finish_field(h, a);
  };
  if (defer) {
    h->pending_field = field;
  } else {
    field();
  }
}

// Goal transform and constants of a snapshot (src/planner.cpp:70-81).
void upload_snapshot(pp_handle* h, const pp_snapshot& s, bool defer = false) {
  const auto& cfg = h->cfg;
  if (s.n_points < 0 || s.field_H < 0) throw std::invalid_argument("malformed obstacle field");
  if (s.n_points > 0 && s.field_H < cfg.H) {
    // The reference would read past the field (geometry.hpp:82-85).
    throw std::invalid_argument("obstacle field shorter than the planning horizon");
  }
  if (s.n_points > 0 && s.field_xy == nullptr) throw std::invalid_argument("null obstacle field");
  set_round_constants(h, s);
  keep_snapshot(h, s);
  if (defer) {
    h->pending_field = [h, s] { upload_field_rows(h, s, h->base); };
  } else {
    upload_field_rows(h, s, h->base);
  }
}

void set_round_constants(pp_handle* h, const pp_snapshot& s) {
  const auto& cfg = h->cfg;
  ppdev::RoundArgs& a = h->base;
  a = ppdev::RoundArgs{};
  const paraplan::Pose2 anchor{s.ev_x, s.ev_y, s.ev_phi};
  const paraplan::Vec2 g = paraplan::to_ev_frame(anchor, {s.goal_x, s.goal_y});
  a.gx = g.x;
  a.gy = g.y;
  a.gphi = s.goal_phi - anchor.phi;
  a.gv = s.goal_v;
  a.gcos = std::cos(a.gphi);
  a.gsin = std::sin(a.gphi);
  a.v0 = s.ev_v;
  a.act0 = s.actuator_delta;
  a.pa0 = s.prev_a0;
  a.d_xi = h->norm.d_xi;
  a.d_eta = h->norm.d_eta;
  a.d_phi = h->norm.d_phi;
  a.d_v = h->norm.d_v;
  a.eps_xi = cfg.tol.eps_xi;
  a.eps_eta = cfg.tol.eps_eta;
  a.eps_phi = cfg.tol.eps_phi;
  a.eps_v = cfg.tol.eps_v;
  const auto& p = h->params;
  a.delta_max = p.delta_max;
  a.window = p.delta_rate_max * p.T_s;
  a.l_r = p.l_r;
  a.wheelbase = p.l_f + p.l_r;
  a.T_s = p.T_s;
  a.u_v_min = p.u_v_min;
  a.u_v_max = p.u_v_max;
  a.fe = p.front_extent();
  a.re = p.rear_extent();
  a.hw = p.half_width;
  const double radius = h->chassis.bounding_radius();
  a.r2 = radius * radius;
  a.sig_lo = cfg.sigma_log_low;
  a.sig_span = cfg.sigma_log_high - cfg.sigma_log_low;
  a.H = cfg.H;
  a.n_params = h->P;
  a.n_layers = static_cast<int32_t>(h->sizes.size());
  for (size_t i = 0; i < h->sizes.size(); ++i) a.sizes[i] = h->sizes[i];
  // the generator's start features need the constants before the field
  a.dmarg32 = h->dmarg32;
  fill_consts(a, &a.kf);
  fill_consts(a, &a.kd);
}

void upload_field_rows(pp_handle* h, const pp_snapshot& s, ppdev::RoundArgs& a) {
  const auto& cfg = h->cfg;
  // Only rows 0..H are ever read (src/planner.cpp:139 at h <= H): split
  // into static and dynamic points and bin them (csrc/capi/field.hpp).
  const int N = s.n_points;
  a.n_points = N;
  const double cull = std::sqrt(a.r2) + 1e-3;
  if (N > 0) {
    ppfield::from_rows(h->field, s.field_xy, cfg.H + 1, N, cull);
  } else {
    h->field = ppfield::Binned{};
    h->field.rows = cfg.H + 1;
    h->field.cull = cull;
  }
  finish_field(h, a);
}

// key prefix fold^4(seed, t, restart, iter) (src/rng.cpp:26-34 minus the
// candidate fold, which the kernel applies).
uint64_t key_prefix(uint64_t seed, uint64_t t, uint64_t r, uint64_t i) {
  // KeyedRng's state after four folds == prefix; reuse the public class on a
  // dummy candidate would fold a fifth time, so recompute here.
  constexpr uint64_t G = 0x9E3779B97F4A7C15ULL;
  auto mix = [](uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  };
  auto fold = [&](uint64_t hh, uint64_t f) { return mix(hh ^ (mix(f) + G + (hh << 6) + (hh >> 2))); };
  uint64_t hh = mix(seed + G);
  hh = fold(hh, t);
  hh = fold(hh, r);
  hh = fold(hh, i);
  return hh;
}

constexpr int ppdev_warps() { return 4; }  // warps per CTA (rollout.cuh kBlock / 32)

void host_rollout(const pp_handle* h, const pp_snapshot& s, const double* theta,
                  pp_rollout_stats* out, double* traj, int32_t cap, int32_t* traj_len);
void host_sample(const pp_handle* h, const double* center, uint64_t t, int restart, int iter,
                 int cand, double* out, int len = -1);

void certify_round(pp_handle* h, ppdev::RoundArgs& a, uint64_t t, int iter, int r0, int rc,
                   const double* center, int64_t c0, int64_t c1, const double* injected,
                   pp_record* out, bool fp64, uint32_t n_sel);

constexpr int kSelCap = 1 << 16;    // near-tie candidates re-ranked per launch
constexpr int kSelFirst = 512;      // copied back with the round result
// Round block (device, one allocation; its head is copied back in ONE D2H):
// [counters u32 x 16][exec u64 x 4 + pad][Rec x kMaxRestartsPerLaunch]
// [unflagged Rec x kMaxRestartsPerLaunch][selected indices int64 x kSelCap]
constexpr size_t kExecOff = 64;
constexpr size_t kRecOff = 128;
// [Rec x kMaxRestartsPerLaunch] best unflagged per restart (keys_only rounds)
constexpr size_t kFreeOff = kRecOff + sizeof(ppdev::Rec) * ppdev::kMaxRestartsPerLaunch;
constexpr size_t kSelOff =
    (kFreeOff + sizeof(ppdev::Rec) * ppdev::kMaxRestartsPerLaunch + 63) / 64 * 64;
constexpr size_t kRoundBytes = kSelOff + sizeof(int64_t) * kSelCap;
constexpr int kRefineGrid = 148 * 2;

// PARAPLAN_TRACE=1: one stderr line per certification pass; 2: also the
// host-side phase times of every plan step (diagnostics).
int trace_level() {
  static const int v = [] {
    const char* e = std::getenv("PARAPLAN_TRACE");
    return e != nullptr ? std::atoi(e) : 0;
  }();
  return v;
}
bool trace_on() { return trace_level() > 0; }

struct PhaseClock {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  char buf[256];
  int len = 0;
  void mark(const char* what) {
    if (trace_level() < 2) return;
    const double us =
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    len += std::snprintf(buf + len, sizeof(buf) - len, " %s=%.1f", what, us);
  }
  void flush() {
    if (trace_level() >= 2) std::fprintf(stderr, "[paraplan] plan_step us:%s\n", buf);
  }
};
PhaseClock* g_clock = nullptr;  // the plan step being traced (one driver thread per handle)
void phase(const char* what) {
  if (g_clock != nullptr) g_clock->mark(what);
}

// Windows up to this size are re-evaluated on the host pool (exact FP64
// rollouts, 16 workers); wider ones get the FP64 device kernel first.
int host_max() {
  static const int v = [] {
    const char* e = std::getenv("PARAPLAN_HOST_MAX");
    return e != nullptr ? std::atoi(e) : 1024;
  }();
  return v;
}

// Occupancy of the rollout kernel for (precision, staged field size, grid
// mode), queried once per handle.
ppdev::LaunchShape launch_shape(pp_handle* h, bool fp64, int field_smem, int grid_mode) {
  const int64_t key = (static_cast<int64_t>(field_smem) << 8) | (grid_mode << 1) | (fp64 ? 1 : 0);
  auto found = h->shapes.find(key);
  if (found == h->shapes.end()) {
    ppdev::LaunchShape sh{};
    const int rcode = fp64 ? ppdev::shape_f64(h->kind, h->device, field_smem, grid_mode, &sh)
                           : ppdev::shape_f32(h->kind, h->device, field_smem, grid_mode, &sh);
    ck(static_cast<cudaError_t>(rcode), "occupancy query");
    found = h->shapes.emplace(key, sh).first;
  }
  return found->second;
}

void consume_pending_field(pp_handle* h, bool side = false) {
  std::function<void()> f = std::move(h->pending_field);
  h->pending_field = nullptr;
  h->field_via_side = side;
  h->field_event = false;
  try {
    f();
  } catch (...) {
    h->field_via_side = false;
    throw;
  }
  h->field_via_side = false;
  if (h->field_event) {
    ck(cudaStreamWaitEvent(h->stream, h->ev_field, 0), "field wait");
    h->field_event = false;
  }
  phase("field");
}

// One sampling round on the device: restarts [r0, r0+rc), candidates
// [c0, c1) of each, iteration `iter`, centred on `center` (or injected theta).
// With re-ranking on, the round is followed by the near-tie window select,
// the FP64 re-evaluation of the window and a host re-rank of FP64 near-ties
// in the reference's own arithmetic, so the winner is the reference's.
void run_round_launch(pp_handle* h, uint64_t t, int iter, int r0, int rc, const double* center,
                      int64_t c0, int64_t c1, const double* injected, pp_record* out,
                      pp_rollout_stats* per_sample, bool force_fp64 = false) {
  const int64_t count = c1 - c0;
  const bool fp64 = h->fp64 || force_fp64;
  const bool rerank = h->rerank && h->snapshot != nullptr;
  // the schedule (refill: generator + rollout) and the theta record width do
  // not depend on the field
  const ppdev::LaunchShape shape0 = launch_shape(h, fp64, 0, 0);
  // a pending field is binned while the generator runs; without a generator
  // (lockstep) or for an FP64 redo it is needed now
  if (h->pending_field && (!shape0.refill || force_fp64)) consume_pending_field(h);
  ppdev::RoundArgs a = h->base;
  if (force_fp64 && !h->fp64) {
    a.field = ensure_field64(h);
    a.lay = a.lay64;
  }
  a.restart_count = rc;
  a.cand_begin = c0;
  a.count = count;
  a.queue_bytes = 0;

  // params block: [prefix u64 x rc][center f64 x P]
  const size_t pbytes = sizeof(uint64_t) * rc + sizeof(double) * h->P;
  h->h_params.reserve(pbytes, "pinned params");
  h->d_params.reserve(pbytes, "device params");
  uint64_t* hp = static_cast<uint64_t*>(h->h_params.p);
  for (int r = 0; r < rc; ++r) {
    hp[r] = key_prefix(h->cfg.master_seed, t, static_cast<uint64_t>(r0 + r),
                       static_cast<uint64_t>(iter));
  }
  double* hc = reinterpret_cast<double*>(hp + rc);
  if (center != nullptr) {
    std::memcpy(hc, center, sizeof(double) * h->P);
  } else {
    std::fill(hc, hc + h->P, 0.0);
  }
  ck(cudaMemcpyAsync(h->d_params.p, h->h_params.p, pbytes, cudaMemcpyHostToDevice, h->stream),
     "params H2D");
  h->timing.h2d_bytes += static_cast<int64_t>(pbytes);
  a.key_prefix = static_cast<const uint64_t*>(h->d_params.p);
  a.center = reinterpret_cast<const double*>(static_cast<uint64_t*>(h->d_params.p) + rc);

  if (injected != nullptr) {
    const size_t ib = sizeof(double) * h->P * static_cast<size_t>(count);
    h->d_injected.reserve(ib, "device theta");
    ck(cudaMemcpyAsync(h->d_injected.p, injected, ib, cudaMemcpyHostToDevice, h->stream),
       "theta H2D");
    h->timing.h2d_bytes += static_cast<int64_t>(ib);
    a.injected = static_cast<const double*>(h->d_injected.p);
  }

  // the round block: counters, work counters, per-restart winners and the
  // selected window, copied back together
  char* dres = static_cast<char*>(h->d_round.p);
  a.counters = reinterpret_cast<uint32_t*>(dres);
  a.exec = reinterpret_cast<unsigned long long*>(dres + kExecOff);
  a.out = reinterpret_cast<ppdev::Rec*>(dres + kRecOff);
  const size_t rbytes = rerank ? kSelOff + sizeof(int64_t) * kSelFirst
                               : kRecOff + sizeof(ppdev::Rec) * rc;
  if (per_sample != nullptr) {
    h->d_samples.reserve(sizeof(ppdev::SampleOut) * rc * static_cast<size_t>(count),
                         "per-sample buffer");
    a.per_sample = static_cast<ppdev::SampleOut*>(h->d_samples.p);
  }
  const size_t total = static_cast<size_t>(count) * rc;
  if (shape0.refill) {
    const size_t esz = fp64 ? sizeof(double) : sizeof(float);
    h->d_theta.reserve(total * shape0.theta_elem * esz, "theta buffer");
    a.theta_buf = h->d_theta.p;  // [total][theta_elem]: theta, first action, pad
    a.first_buf = nullptr;
  }
  // several restarts on the refill schedule: winners from the sample keys
  const bool keys_only = shape0.refill && rc > 1;
  a.keys_only = keys_only ? 1 : 0;
  a.out_free = keys_only && rerank ? reinterpret_cast<ppdev::Rec*>(dres + kFreeOff) : nullptr;
  if (rerank || keys_only) {
    h->d_skeys.reserve(total * (fp64 ? sizeof(ppdev::SKey) : sizeof(ppdev::SKey32)), "sample keys");
    a.skeys = h->d_skeys.p;
    a.skey32 = fp64 ? 0 : 1;
  }
  if (rerank) {
    h->d_sel.reserve(kSelCap * sizeof(ppdev::SelRec), "selection");
    a.sel_out = static_cast<ppdev::SelRec*>(h->d_sel.p);
    a.sel_list = reinterpret_cast<int64_t*>(dres + kSelOff);
    a.sel_cap = kSelCap;
    a.refine_grid = kRefineGrid;
    a.sel_rho = fp64 ? 1e-11 : h->sel_rho;
    a.sel_alpha = fp64 ? 1e-13 : 1e-6;
  }

  ck(cudaEventRecord(h->ev0, h->stream), "event");
  ck(static_cast<cudaError_t>(fp64 ? ppdev::launch_generate_f64(h->kind, a, h->stream)
                                   : ppdev::launch_generate_f32(h->kind, a, h->stream)),
     "theta generator launch");
  if (h->pending_field) {  // bin + upload the field while the generator runs
    consume_pending_field(h, true);
    const ppdev::RoundArgs& b = h->base;
    a.field = b.field;
    a.field64 = b.field64;
    a.n_points = b.n_points;
    a.field_ns = b.field_ns;
    a.field_nd = b.field_nd;
    a.grid_nx = b.grid_nx;
    a.grid_ny = b.grid_ny;
    a.grid_mode = b.grid_mode;
    a.grid_x0 = b.grid_x0;
    a.grid_y0 = b.grid_y0;
    a.grid_g = b.grid_g;
    a.lay = b.lay;
    a.lay64 = b.lay64;
    a.kf = b.kf;
    a.kd = b.kd;
  }
  const int field_smem = (force_fp64 && !h->fp64) ? 0 : h->field_smem_bytes;
  const ppdev::LaunchShape shape = launch_shape(h, fp64, field_smem, a.grid_mode);
  // refill: 32-candidate batches; lockstep: one tile of `block` candidates
  const int unit = shape.refill ? 32 : shape.block;
  const int64_t tpr64 = (count + unit - 1) / unit;
  if (tpr64 * rc > (int64_t{1} << 30)) throw std::invalid_argument("sampling round too large");
  a.tiles_per_restart = static_cast<int32_t>(tpr64);
  a.n_tiles = static_cast<int32_t>(tpr64 * rc);
  a.block = shape.block;
  a.grid = std::max(1, std::min(shape.grid, shape.refill ? (a.n_tiles + ppdev_warps() - 1) /
                                                               ppdev_warps()
                                                         : a.n_tiles));
  a.field_smem_bytes = field_smem;
  // tile records (x2 for keys_only: best and best unflagged)
  const size_t n_recs = shape.refill ? 2 * static_cast<size_t>(rc) * std::max(a.grid, 148 * 4)
                                    : static_cast<size_t>(a.n_tiles);
  h->d_tiles.reserve(sizeof(ppdev::Rec) * n_recs, "tile records");
  a.tile_recs = static_cast<ppdev::Rec*>(h->d_tiles.p);
  // theta in a global per-lane column (NetGlobal): any architecture without
  // a register specialisation in this precision ([5,10,10,2] has one in FP32)
  const bool generic = h->kind == ppdev::NetKind::kGeneric ||
                       (fp64 && h->kind == ppdev::NetKind::k5_10_10_2);
  if (generic || rerank) {
    const size_t lanes = std::max<size_t>(generic ? static_cast<size_t>(a.grid) * a.block : 0,
                                          rerank ? kRefineGrid * 128 : 0);
    h->d_scratch.reserve(lanes * h->P * sizeof(double), "theta scratch");
    a.theta_scratch = static_cast<float*>(h->d_scratch.p);
    a.theta_scratch64 = static_cast<double*>(h->d_scratch.p);
  }
  ck(static_cast<cudaError_t>(fp64 ? ppdev::launch_rollout_f64(h->kind, a, h->stream)
                                   : ppdev::launch_rollout_f32(h->kind, a, h->stream)),
     "sampling kernel launch");
  if (rerank) {
    // the selection counter was re-armed by the rollout kernel's last CTA
    ck(static_cast<cudaError_t>(ppdev::launch_select(a, h->stream)), "window select launch");
    if (!h->pool) {
      const unsigned hc = std::thread::hardware_concurrency();
      h->pool = std::make_unique<HostPool>(static_cast<int>(std::min(16u, std::max(1u, hc))));
    }
    h->pool->prewarm();  // workers spin while the GPU samples
  }
  ck(cudaEventRecord(h->ev1, h->stream), "event");
  // one D2H: counters (selection count), work counters, winners and the
  // first kSelFirst selected indices
  ck(cudaMemcpyAsync(h->h_round.p, h->d_round.p, rbytes, cudaMemcpyDeviceToHost, h->stream),
     "result D2H");
  phase("enqueued");
  // the host's exact image of device-binned movers, while the round runs
  if (h->field.dyn_deferred) {
    ppfield::bin_dynamic(h->field);
    phase("host-binned");
  }
  uint32_t n_sel = 0;
  h->timing.d2h_bytes += static_cast<int64_t>(rbytes);
  if (per_sample != nullptr) {
    const size_t sb = sizeof(ppdev::SampleOut) * rc * static_cast<size_t>(count);
    ck(cudaMemcpyAsync(per_sample, h->d_samples.p, sb, cudaMemcpyDeviceToHost, h->stream),
       "per-sample D2H");
    h->timing.d2h_bytes += static_cast<int64_t>(sb);
  }
  ck(cudaStreamSynchronize(h->stream), "sampling kernel");
  phase("synced");
  float ms = 0.f;
  ck(cudaEventElapsedTime(&ms, h->ev0, h->ev1), "event timing");
  h->timing.kernel_ms += ms;
  h->timing.launches += (shape.refill ? 2 : 1) + (rerank ? 1 : 0) + (keys_only ? 1 : 0);
  h->timing.samples += count * rc;
  const char* hres = static_cast<const char*>(h->h_round.p);
  const unsigned long long* ex = reinterpret_cast<const unsigned long long*>(hres + kExecOff);
  h->timing.executed_steps += static_cast<int64_t>(ex[2]);
  h->timing.checked_states += static_cast<int64_t>(ex[3]);
  const ppdev::Rec* recs = reinterpret_cast<const ppdev::Rec*>(hres + kRecOff);
  for (int r = 0; r < rc; ++r) {
    out[r].cls = recs[r].cls;
    out[r].candidate = recs[r].cand;
    out[r].restart = r0 + r;
    out[r].iter = iter;
    out[r].k1 = recs[r].k1;
    out[r].k2 = recs[r].k2;
  }
  if (!rerank) return;

  n_sel = reinterpret_cast<const uint32_t*>(hres)[2];
  const auto c_t0 = std::chrono::steady_clock::now();
  certify_round(h, a, t, iter, r0, rc, center, c0, c1, injected, out, fp64, n_sel);
  phase("certified");
  h->timing.certify_ms +=
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - c_t0).count();
}

// Certified re-ranking (PlannerConfig::refine). The FP32 keys are trusted
// only up to a relative error rho/2 (+ alpha/2), and discrete verdicts that
// rounding could flip toward a BETTER outcome are flagged by the kernel and
// always selected; flips toward a worse outcome only hurt the candidate
// itself. Each pass evaluates the window's new members in the reference's
// own FP64 arithmetic on the host (the device FP64 kernel first when the
// window is wide) and certifies a restart when its exact best beats every
// unselected candidate's optimistic bound; otherwise the window widens.
// Windows that overflow, or restarts still uncertified after the last pass,
// are redone as an FP64 round.
void certify_round(pp_handle* h, ppdev::RoundArgs& a, uint64_t t, int iter, int r0, int rc,
                   const double* center, int64_t c0, int64_t c1, const double* injected,
                   pp_record* out, bool fp64, uint32_t n_sel) {
  const int64_t count = c1 - c0;
  const pp_snapshot& snap = *h->snapshot;
  std::vector<double> ctr(h->P, 0.0);
  if (center != nullptr) ctr.assign(center, center + h->P);
  struct Exact {
    int cls;
    int t_goal;
    double cost;  // terminal cost (cls 0/1) or path length (cls 2)
    double k1, k2;
  };
  std::unordered_map<int64_t, Exact> known;
  auto exact_of = [&](int64_t s) {  // the reference's own FP64 arithmetic
    const int r = static_cast<int>(s / count);
    const int cand = static_cast<int>(c0 + (s - r * count));
    std::vector<double> theta(h->P);
    if (injected != nullptr) {
      std::memcpy(theta.data(), injected + static_cast<size_t>(cand - c0) * h->P,
                  sizeof(double) * h->P);
    } else {
      host_sample(h, ctr.data(), t, r0 + r, iter, cand, theta.data(), -1);
    }
    pp_rollout_stats st{};
    host_rollout(h, snap, theta.data(), &st, nullptr, 0, nullptr);
    Exact e;
    e.cls = st.collided ? 0 : (st.reached ? 2 : 1);
    e.t_goal = st.t_goal;
    e.cost = e.cls == 2 ? st.path_length : st.terminal_cost;
    e.k1 = e.cls == 2 ? -static_cast<double>(st.t_goal) : -st.terminal_cost;
    e.k2 = e.cls == 2 ? -st.path_length : 0.0;
    return e;
  };
  if (!h->pool) {
    const unsigned hc = std::thread::hardware_concurrency();
    h->pool = std::make_unique<HostPool>(static_cast<int>(std::min(16u, std::max(1u, hc))));
  }
  const double rho = a.sel_rho, alpha = a.sel_alpha;
  std::vector<ppdev::SelBound> bound(rc);
  // the first window is built around each restart's best unflagged
  // candidate when the round reports it (keys_only), else its winner
  const ppdev::Rec* free_recs =
      a.out_free != nullptr
          ? reinterpret_cast<const ppdev::Rec*>(static_cast<const char*>(h->h_round.p) + kFreeOff)
          : nullptr;
  for (int r = 0; r < rc; ++r) {
    pp_record o = out[r];
    if (free_recs != nullptr && free_recs[r].cls >= 0) {
      o.cls = free_recs[r].cls;
      o.k1 = free_recs[r].k1;
      o.k2 = free_recs[r].k2;
    }
    bound[r].cls = o.cls;
    bound[r].t_goal = o.cls == 2 ? static_cast<int>(-o.k1) : 0;
    bound[r].thr = (o.cls == 2 ? -o.k2 : -o.k1) * (1.0 + rho) + alpha;
  }
  std::vector<char> certified(rc, 0);
  std::vector<int64_t> list;
  constexpr int kPasses = 6;
  for (int pass = 0; pass < kPasses; ++pass) {
    if (pass > 0) {  // widened select over the uncertified restarts
      h->d_bound.reserve(sizeof(ppdev::SelBound) * rc, "window bounds");
      h->h_bound.reserve(sizeof(ppdev::SelBound) * rc, "pinned bounds");
      std::memcpy(h->h_bound.p, bound.data(), sizeof(ppdev::SelBound) * rc);
      ck(cudaMemcpyAsync(h->d_bound.p, h->h_bound.p, sizeof(ppdev::SelBound) * rc,
                         cudaMemcpyHostToDevice, h->stream),
         "bounds H2D");
      a.sel_bound = static_cast<const ppdev::SelBound*>(h->d_bound.p);
      ck(cudaMemsetAsync(a.counters + 2, 0, sizeof(uint32_t), h->stream), "selection counter");
      ck(static_cast<cudaError_t>(ppdev::launch_select(a, h->stream)), "window select launch");
      ck(cudaMemcpyAsync(h->h_round.p, h->d_round.p, kSelOff + sizeof(int64_t) * kSelFirst,
                         cudaMemcpyDeviceToHost, h->stream),
         "selection D2H");
      ck(cudaStreamSynchronize(h->stream), "window select");
      h->timing.launches += 1;
      n_sel = static_cast<const uint32_t*>(h->h_round.p)[2];
    }
    if (n_sel > static_cast<uint32_t>(kSelCap)) {
      if (trace_on()) {
        std::fprintf(stderr, "[paraplan] t=%llu iter=%d pass=%d selected=%u: window overflow\n",
                     static_cast<unsigned long long>(t), iter, pass, n_sel);
      }
      break;
    }
    if (n_sel > static_cast<uint32_t>(kSelFirst)) {
      ck(cudaMemcpy(reinterpret_cast<int64_t*>(static_cast<char*>(h->h_round.p) + kSelOff) + kSelFirst,
                    a.sel_list + kSelFirst, sizeof(int64_t) * (n_sel - kSelFirst),
                    cudaMemcpyDeviceToHost),
         "selection D2H");
    }
    const int64_t* sl =
        reinterpret_cast<const int64_t*>(static_cast<const char*>(h->h_round.p) + kSelOff);
    list.clear();
    for (uint32_t i = 0; i < n_sel; ++i) {
      if (known.find(sl[i]) == known.end()) list.push_back(sl[i]);
    }
    std::sort(list.begin(), list.end());
    list.erase(std::unique(list.begin(), list.end()), list.end());
    h->timing.refined += static_cast<int32_t>(list.size());
    std::vector<Exact> got(list.size());
    if (list.size() <= static_cast<size_t>(host_max())) {
      h->pool->run(static_cast<int>(list.size()), [&](int i) { got[i] = exact_of(list[i]); });
    } else {
      // wide window: FP64 keys from the device, exact host keys for the FP64
      // near-ties of each restart's best
      ck(cudaMemcpyAsync(a.sel_list, list.data(), sizeof(int64_t) * list.size(),
                         cudaMemcpyHostToDevice, h->stream),
         "refine list H2D");
      const uint32_t n_list = static_cast<uint32_t>(list.size());
      ck(cudaMemcpyAsync(a.counters + 2, &n_list, sizeof(uint32_t), cudaMemcpyHostToDevice,
                         h->stream),
         "refine count H2D");
      a.field64 = ensure_field64(h);
      ck(static_cast<cudaError_t>(ppdev::launch_refine(h->kind, a, h->stream)), "refine launch");
      std::vector<ppdev::SelRec> dev(list.size());
      ck(cudaMemcpyAsync(dev.data(), a.sel_out, sizeof(ppdev::SelRec) * list.size(),
                         cudaMemcpyDeviceToHost, h->stream),
         "refine D2H");
      ck(cudaStreamSynchronize(h->stream), "refine kernel");
      h->timing.launches += 1;
      std::vector<int> best(rc, -1);
      for (size_t i = 0; i < dev.size(); ++i) {
        got[i] = Exact{dev[i].cls, dev[i].cls == 2 ? static_cast<int>(-dev[i].k1) : -1,
                       dev[i].cls == 2 ? -dev[i].k2 : -dev[i].k1, dev[i].k1, dev[i].k2};
        const int r = dev[i].restart;
        if (best[r] < 0 || key_better({got[i].cls, got[i].k1, got[i].k2},
                                      {got[best[r]].cls, got[best[r]].k1, got[best[r]].k2})) {
          best[r] = static_cast<int>(i);
        }
      }
      std::vector<int> ties;
      for (size_t i = 0; i < dev.size(); ++i) {
        const Exact& b = got[best[dev[i].restart]];
        const double tol = 1e-12;
        if (got[i].cls == b.cls && std::abs(got[i].k1 - b.k1) <= tol * std::max(1.0, std::abs(b.k1)) &&
            std::abs(got[i].k2 - b.k2) <= tol * std::max(1.0, std::abs(b.k2))) {
          ties.push_back(static_cast<int>(i));
        }
      }
      h->pool->run(static_cast<int>(ties.size()),
                   [&](int j) { got[ties[j]] = exact_of(list[ties[j]]); });
    }
    for (size_t i = 0; i < list.size(); ++i) known[list[i]] = got[i];

    // certify or widen each uncertified restart
    bool all = true;
    for (int r = 0; r < rc; ++r) {
      if (certified[r]) continue;
      const ppdev::SelBound& bd = bound[r];
      int64_t win = -1;
      const Exact* e = nullptr;
      for (const auto& kv : known) {
        if (kv.first / count != r) continue;
        const Exact& q = kv.second;
        if (e == nullptr || key_better({q.cls, q.k1, q.k2}, {e->cls, e->k1, e->k2}) ||
            (q.cls == e->cls && q.k1 == e->k1 && q.k2 == e->k2 && kv.first < win)) {
          e = &q;
          win = kv.first;
        }
      }
      const double slack = 0.5 * (rho * bd.thr + alpha);
      bool ok = false;
      if (e != nullptr) {
        if (e->cls > bd.cls) {
          ok = true;  // only a flagged (always selected) candidate can rise a class
        } else if (e->cls == bd.cls) {
          ok = (bd.cls == 2 && e->t_goal < bd.t_goal) ||
               ((bd.cls != 2 || e->t_goal == bd.t_goal) && e->cost <= bd.thr - slack);
        }
      }
      if (ok) {
        certified[r] = 1;
        out[r].cls = e->cls;
        out[r].candidate = static_cast<int>(c0 + (win - r * count));
        out[r].k1 = e->k1;
        out[r].k2 = e->k2;
        bound[r].cls = -1;  // select nothing more for this restart
        continue;
      }
      all = false;
      if (trace_level() >= 2) {
        std::fprintf(stderr,
                     "[paraplan]   restart %d open: window cls %d t_goal %d thr %.9g slack %.3g; "
                     "exact best cls %d t_goal %d cost %.9g\n",
                     r0 + r, bd.cls, bd.t_goal, bd.thr, slack, e ? e->cls : -9,
                     e ? e->t_goal : -9, e ? e->cost : 0.0);
      }
      const bool same = e != nullptr && e->cls == bd.cls && (bd.cls != 2 || e->t_goal == bd.t_goal);
      const double widened = bd.thr * 1.25 + alpha;
      bound[r].thr = same ? std::max(e->cost * (1.0 + rho) + alpha, widened) : widened;
    }
    if (trace_on()) {
      std::fprintf(stderr, "[paraplan] t=%llu iter=%d pass=%d selected=%u new=%zu certified=%s\n",
                   static_cast<unsigned long long>(t), iter, pass, n_sel, list.size(),
                   all ? "all" : "no");
    }
    if (all) return;
  }
  // overflowed or not certified: redo the round in FP64
  if (trace_on()) {
    std::fprintf(stderr, "[paraplan] t=%llu iter=%d: FP64 fallback round\n",
                 static_cast<unsigned long long>(t), iter);
  }
  if (fp64) throw std::runtime_error("near-tie re-ranking could not certify an FP64 round");
  h->timing.refined = -1;
  run_round_launch(h, t, iter, r0, rc, center, c0, c1, injected, out, nullptr, true);
}

void run_round(pp_handle* h, uint64_t t, int iter, int r0, int rc, const double* center,
               int64_t c0, int64_t c1, const double* injected, pp_record* out,
               pp_rollout_stats* per_sample) {
  if (!h->snap_valid) throw std::invalid_argument("no snapshot uploaded");
  if (rc < 1 || c1 < c0) throw std::invalid_argument("empty sampling round");
  // the refill kernel keeps per-restart tables in shared memory: chunk
  for (int done = 0; done < rc; done += ppdev::kMaxRestartsPerLaunch) {
    const int n = std::min(ppdev::kMaxRestartsPerLaunch, rc - done);
    run_round_launch(h, t, iter, r0 + done, n, center, c0, c1, injected, out + done,
                     per_sample == nullptr ? nullptr : per_sample + done * (c1 - c0));
  }
}


// Host FP64 rollout: src/planner.cpp:66-191 expressed through the public
// primitives (bit-identical under -ffp-contract=off; the reference's own
// selfcheck::resimulate_rollout relies on the same equivalence).
void host_rollout(const pp_handle* h, const pp_snapshot& s, const double* theta,
                  pp_rollout_stats* out, double* traj, int32_t cap, int32_t* traj_len) {
  using namespace paraplan;
  const auto& p = h->params;
  const auto& cfg = h->cfg;
  const Pose2 anchor{s.ev_x, s.ev_y, s.ev_phi};
  const Vec2 gp = to_ev_frame(anchor, {s.goal_x, s.goal_y});
  const GoalSetpoint goal{gp.x, gp.y, s.goal_phi - anchor.phi, s.goal_v};
  const double gc = std::cos(goal.phi), gs = std::sin(goal.phi);
  const std::span<const double> th(theta, h->P);
  const int N = s.n_points;
  if (s.field_xy == nullptr && h->field.dyn_deferred) {
    throw std::logic_error("obstacle field used before its moving points were binned");
  }
  if (N > 0 && s.field_xy != nullptr && s.field_H < cfg.H) {
    throw std::invalid_argument("obstacle field shorter than the planning horizon");
  }

  VehicleState z{0.0, 0.0, 0.0, s.ev_v};
  ActuatorState act{s.actuator_delta};
  double prev_a0 = s.prev_a0;
  std::memset(out, 0, sizeof(*out));
  out->t_goal = -1;
  int32_t n = 0;
  auto push = [&](const VehicleState& st) {
    if (traj != nullptr && n < cap) {
      traj[4 * n + 0] = st.x;
      traj[4 * n + 1] = st.y;
      traj[4 * n + 2] = st.phi;
      traj[4 * n + 3] = st.v;
    }
    ++n;
  };
  push(z);
  const ControlAction first = h->policy->forward(th, build_features(z, goal, prev_a0, h->norm));
  out->first_a0 = first.a0;
  out->first_a1 = first.a1;
  double path = 0.0;
  for (int k = 0;; ++k) {
    if (N > 0) {
      // the resident snapshot (field_xy == nullptr) goes through the binned
      // field; a caller's snapshot is scanned point by point
      bool hit;
      if (s.field_xy == nullptr) {
        hit = ppfield::collides(h->field, h->chassis, h->box, k, z.x, z.y, z.phi);
      } else {
        const std::span<const Vec2> row(
            reinterpret_cast<const Vec2*>(s.field_xy) + static_cast<size_t>(k) * N, N);
        hit = collision({z.x, z.y, z.phi}, row, h->chassis);
      }
      if (hit) {
        out->collided = 1;
        break;
      }
    }
    const double gdx = goal.x - z.x, gdy = goal.y - z.y;
    if (std::abs(gc * gdx + gs * gdy) <= cfg.tol.eps_xi &&
        std::abs(-gs * gdx + gc * gdy) <= cfg.tol.eps_eta &&
        std::abs(wrap_angle(goal.phi - z.phi)) <= cfg.tol.eps_phi &&
        std::abs(goal.v - z.v) <= cfg.tol.eps_v) {
      out->reached = 1;
      out->t_goal = k;
      break;
    }
    if (k == cfg.H) break;
    const ControlAction a =
        k == 0 ? first : h->policy->forward(th, build_features(z, goal, prev_a0, h->norm));
    const Controls u = map_controls(a, act, p);
    const VehicleState nz = step(z, u.delta, u.u_v, p);
    const double dx = nz.x - z.x, dy = nz.y - z.y;
    path += std::sqrt(dx * dx + dy * dy);
    z = nz;
    act.delta = u.delta;
    prev_a0 = a.a0;
    push(z);
  }
  out->path_length = path;
  out->terminal_cost = std::abs(goal.x - z.x) / h->norm.d_xi +
                       std::abs(goal.y - z.y) / h->norm.d_eta +
                       std::abs(wrap_angle(goal.phi - z.phi)) / h->norm.d_phi +
                       std::abs(goal.v - z.v) / h->norm.d_v;
  out->steps = n - 1;
  if (traj_len != nullptr) *traj_len = n;
}

void host_sample(const pp_handle* h, const double* center, uint64_t t, int restart, int iter,
                 int cand, double* out, int len) {
  if (len < 0) len = h->P;
  if (cand == 0) {
    std::memcpy(out, center, sizeof(double) * len);
    return;
  }
  paraplan::KeyedRng rng(h->cfg.master_seed, t, static_cast<uint64_t>(restart),
                         static_cast<uint64_t>(iter), static_cast<uint64_t>(cand));
  const double sigma = std::pow(
      10.0, h->cfg.sigma_log_low + rng.next_unit() * (h->cfg.sigma_log_high - h->cfg.sigma_log_low));
  for (int i = 0; i < len; ++i) out[i] = center[i] + sigma * rng.next_normal();
}

}  // namespace

extern "C" {

int32_t pp_abi_version(void) { return PP_ABI_VERSION; }

const char* pp_last_error(void) { return g_error.c_str(); }

int32_t pp_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// Warm-up at construction (the reference starts its thread pool in its
// constructor as well): one obstacle-free round at the configured size
// allocates the round buffers, loads the kernels and starts the host pool,
// and the 2-D field kernels are loaded too, so the first plan_step pays for
// none of it. Failures here are left for the first real call to report.
void prewarm(pp_handle* h) {
  if (const char* e = std::getenv("PARAPLAN_PREWARM"); e != nullptr && std::atoi(e) == 0) return;
  try {
    pp_snapshot s{};
    s.goal_x = 1e3;
    s.field_H = h->cfg.H;
    upload_snapshot(h, s);
    const int rc = std::min(h->cfg.n_restarts, 64);
    std::vector<pp_record> rec(rc);
    run_round(h, 0, 0, 0, rc, nullptr, 0, h->cfg.n_candidates, nullptr, rec.data(), nullptr);
    for (int mode = 1; mode <= 2; ++mode) {
      ppdev::LaunchShape sh{};
      if (h->fp64) {
        ppdev::shape_f64(h->kind, h->device, 0, mode, &sh);
      } else {
        ppdev::shape_f32(h->kind, h->device, 0, mode, &sh);
      }
    }
    ck(cudaStreamSynchronize(h->stream), "warm-up");
  } catch (...) {
    cudaGetLastError();
  }
  h->snap_valid = false;
  h->snapshot = nullptr;
  h->timing = pp_timing{};
}

pp_status pp_create(const pp_model* m, pp_handle** out) {
  if (out != nullptr) *out = nullptr;
  pp_handle* h = nullptr;
  const pp_status st = guarded([&] {
    if (m == nullptr || out == nullptr) throw std::invalid_argument("null argument");
    auto hp = std::make_unique<pp_handle>();
    hp->model = *m;
    hp->sizes.assign(m->layer_sizes, m->layer_sizes + std::max(0, m->n_layers));
    hp->model.layer_sizes = hp->sizes.data();
    hp->params = params_of(m->vehicle);
    hp->cfg = config_of(m->config);
    hp->norm = {m->norm.d_xi, m->norm.d_eta, m->norm.d_phi, m->norm.d_v};
    paraplan::MlpArchitecture arch;
    arch.layer_sizes.assign(hp->sizes.begin(), hp->sizes.end());
    if (static_cast<int>(arch.layer_sizes.size()) > ppdev::kMaxLayers) {
      throw std::invalid_argument("at most 16 layers are supported");
    }
    // Same validation order as the reference constructor (planner.cpp:46-58).
    hp->policy = std::make_unique<paraplan::MlpPolicy>(arch);
    hp->params.validate();
    hp->cfg.validate();
    hp->chassis = paraplan::ChassisPolytope::rectangle(hp->params);
    hp->box = {hp->params.front_extent(), hp->params.rear_extent(), hp->params.half_width};
    hp->P = hp->policy->param_count();
    hp->kind = ppdev::classify(hp->sizes.data(), static_cast<int32_t>(hp->sizes.size()));
    hp->fp64 = hp->cfg.precision == 64;
    hp->rerank = hp->cfg.refine;
    if (const char* e = std::getenv("PARAPLAN_SEL_RHO")) hp->sel_rho = std::atof(e);
    if (const char* e = std::getenv("PARAPLAN_DMARG")) hp->dmarg32 = std::atof(e);
    hp->device = hp->cfg.device;

    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      throw NoDevice("no CUDA device: the paraplan B200 planner has no CPU fallback");
    }
    if (hp->device >= n) throw std::invalid_argument("CUDA device ordinal out of range");
    cudaDeviceProp prop{};
    ck(cudaGetDeviceProperties(&prop, hp->device), "device query");
    if (prop.major != 10) {
      throw NoDevice(std::string("device ") + prop.name +
                     " is not sm_100 (B200); kernels are built for sm_100a only");
    }
    ck(cudaSetDevice(hp->device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&hp->stream, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreate(&hp->ev0), "event");
    ck(cudaEventCreate(&hp->ev1), "event");
    ck(cudaStreamCreateWithFlags(&hp->side, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&hp->ev_field, cudaEventDisableTiming), "event");
    hp->d_round.reserve(kRoundBytes, "round block");
    ck(cudaMemsetAsync(hp->d_round.p, 0, kRoundBytes, hp->stream), "round block");
    hp->h_round.reserve(kRoundBytes, "pinned round block");
    ck(cudaStreamSynchronize(hp->stream), "init");
    h = hp.release();
  });
  if (st == PP_OK) {
    prewarm(h);
    *out = h;
  }
  return st;
}

void pp_destroy(pp_handle* h) {
  if (h == nullptr) return;
  cudaSetDevice(h->device);
  if (h->stream != nullptr) cudaStreamSynchronize(h->stream);
  for (DevBuf* b : {&h->d_field, &h->d_params, &h->d_round, &h->d_tiles, &h->d_movers, &h->d_bin,
                    &h->d_samples, &h->d_scratch, &h->d_injected, &h->d_theta, &h->d_skeys,
                    &h->d_sel, &h->d_bound, &h->d_field64}) {
    b->release();
  }
  for (HostBuf* b : {&h->h_field, &h->h_params, &h->h_round, &h->h_bound, &h->h_movers,
                     &h->h_field64}) {
    b->release();
  }
  if (h->side != nullptr) cudaStreamSynchronize(h->side);
  if (h->ev_field != nullptr) cudaEventDestroy(h->ev_field);
  if (h->side != nullptr) cudaStreamDestroy(h->side);
  if (h->ev0 != nullptr) cudaEventDestroy(h->ev0);
  if (h->ev1 != nullptr) cudaEventDestroy(h->ev1);
  if (h->stream != nullptr) cudaStreamDestroy(h->stream);
  delete h;
}

int32_t pp_param_count(const pp_handle* h) { return h == nullptr ? 0 : h->P; }

void* pp_stream(const pp_handle* h) { return h == nullptr ? nullptr : h->stream; }

pp_status pp_last_timing(const pp_handle* h, pp_timing* out) {
  if (h == nullptr || out == nullptr) return PP_INVALID_ARGUMENT;
  *out = h->timing;
  return PP_OK;
}

pp_status pp_upload_snapshot(pp_handle* h, const pp_snapshot* snap) {
  return guarded([&] {
    if (h == nullptr || snap == nullptr) throw std::invalid_argument("null argument");
    ck(cudaSetDevice(h->device), "cudaSetDevice");
    upload_snapshot(h, *snap);
    ck(cudaStreamSynchronize(h->stream), "snapshot H2D");
  });
}

pp_status pp_evaluate(pp_handle* h, const pp_snapshot* snap, uint64_t t, int32_t iter,
                      int32_t restart_begin, int32_t restart_count, const double* center,
                      int64_t cand_begin, int64_t cand_end, pp_record* out,
                      pp_rollout_stats* per_sample) {
  return guarded([&] {
    if (h == nullptr || out == nullptr) throw std::invalid_argument("null argument");
    if (cand_begin < 0 || cand_end > h->cfg.n_candidates || restart_begin < 0 ||
        restart_begin + restart_count > h->cfg.n_restarts || iter < 0 ||
        iter >= h->cfg.n_iter_max) {
      throw std::invalid_argument("sampling round outside the configured budget");
    }
    ck(cudaSetDevice(h->device), "cudaSetDevice");
    h->timing = pp_timing{};
    if (snap != nullptr) upload_snapshot(h, *snap);
    if (cand_end <= cand_begin) {
      for (int r = 0; r < restart_count; ++r) {
        out[r] = pp_record{-1, -1, restart_begin + r, iter, 0.0, 0.0};
      }
      return;
    }
    run_round(h, t, iter, restart_begin, restart_count, center, cand_begin, cand_end, nullptr,
              out, per_sample);
  });
}

pp_status pp_eval_theta(pp_handle* h, const pp_snapshot* snap, const double* theta, int64_t n,
                        pp_rollout_stats* out) {
  return guarded([&] {
    if (h == nullptr || theta == nullptr || out == nullptr) {
      throw std::invalid_argument("null argument");
    }
    ck(cudaSetDevice(h->device), "cudaSetDevice");
    h->timing = pp_timing{};
    if (snap != nullptr) upload_snapshot(h, *snap);
    if (n <= 0) return;
    pp_record rec{};
    run_round(h, 0, 0, 0, 1, nullptr, 0, n, theta, &rec, out);
  });
}

pp_status pp_rollout(const pp_handle* h, const pp_snapshot* snap, const double* theta,
                     int32_t theta_len, pp_rollout_stats* out, double* traj, int32_t traj_cap,
                     int32_t* traj_len) {
  return guarded([&] {
    if (h == nullptr || snap == nullptr || theta == nullptr || out == nullptr) {
      throw std::invalid_argument("null argument");
    }
    if (theta_len != h->P) throw std::invalid_argument("parameter vector size mismatch");
    host_rollout(h, *snap, theta, out, traj, traj_cap, traj_len);
  });
}

pp_status pp_sample_candidate(const pp_handle* h, const double* center, int32_t len, uint64_t t,
                              int32_t restart, int32_t iter, int32_t candidate, double* out) {
  return guarded([&] {
    if (h == nullptr || center == nullptr || out == nullptr) {
      throw std::invalid_argument("null argument");
    }
    if (len < 0) throw std::invalid_argument("candidate buffer size mismatch");
    host_sample(h, center, t, restart, iter, candidate, out, len);
  });
}

double pp_perturbation_sigma(const pp_handle* h, uint64_t t, int32_t restart, int32_t iter,
                             int32_t candidate) {
  paraplan::KeyedRng rng(h->cfg.master_seed, t, static_cast<uint64_t>(restart),
                         static_cast<uint64_t>(iter), static_cast<uint64_t>(candidate));
  return std::pow(10.0, h->cfg.sigma_log_low +
                            rng.next_unit() * (h->cfg.sigma_log_high - h->cfg.sigma_log_low));
}

int32_t pp_key_better(int32_t cls_a, double k1_a, double k2_a, int32_t cls_b, double k1_b,
                      double k2_b) {
  return key_better({cls_a, k1_a, k2_a}, {cls_b, k1_b, k2_b}) ? 1 : 0;
}

// Ordered merge (src/planner.cpp:310-321): records come from disjoint,
// increasing index ranges, so a strict-better scan keeps the lowest index.
pp_status pp_merge_records(const pp_record* recs, int32_t n, pp_record* out) {
  if (out == nullptr || (n > 0 && recs == nullptr)) return PP_INVALID_ARGUMENT;
  pp_record m{-1, -1, -1, -1, 0.0, 0.0};
  for (int32_t i = 0; i < n; ++i) {
    if (recs[i].candidate < 0) continue;
    if (m.candidate < 0 ||
        key_better({recs[i].cls, recs[i].k1, recs[i].k2}, {m.cls, m.k1, m.k2})) {
      m = recs[i];
    }
  }
  *out = m;
  return PP_OK;
}

}  // extern "C"

namespace {

// Planner::plan_step after the snapshot is resident (src/planner.cpp:238-351).
void plan_step_resident(pp_handle* h, uint64_t t, pp_plan_output* out) {
  const int P = h->P;
  const auto& cfg = h->cfg;
  const pp_snapshot& snap = *h->snapshot;
  std::vector<double> init_center(P, 0.0);
  if (snap.warm_theta_len == P) init_center.assign(snap.warm_theta, snap.warm_theta + P);

  const int R = cfg.n_restarts, I = cfg.n_iter_max, n = cfg.n_candidates;
  // Iteration 0 of every restart centres on the warm start: one launch.
  std::vector<pp_record> first(R);
  run_round(h, t, 0, 0, R, init_center.data(), 0, n, nullptr, first.data(), nullptr);

  Key best;
  bool best_valid = false, any_free = false;
  std::vector<double> best_theta(P, 0.0), center(P, 0.0), theta(P);
  pp_record win{-1, -1, -1, -1, 0.0, 0.0};
  int64_t evaluated = 0;
  bool done = false;
  for (int r = 0; r < R && !done; ++r) {
    for (int it = 0; it < I; ++it) {
      pp_record rec;
      if (it == 0) {
        center = init_center;
        rec = first[r];
      } else {
        if (best_valid) center = best_theta;  // :275-276
        run_round(h, t, it, r, 1, center.data(), 0, n, nullptr, &rec, nullptr);
      }
      evaluated += n;
      any_free = any_free || rec.cls >= 1;
      const Key k{rec.cls, rec.k1, rec.k2};
      if (!best_valid || key_better(k, best)) {  // :324-330
        host_sample(h, center.data(), t, r, it, rec.candidate, theta.data());
        best = k;
        best_theta = theta;
        best_valid = true;
        win = rec;
      }
      if (cfg.early_exit && best_valid && best.cls == 2) {  // :332-334
        done = true;
        break;
      }
    }
  }

  // FP64 epilogue (:339-350).
  phase("merged");
  out->evaluated = evaluated;
  if (out->best_theta != nullptr) std::memcpy(out->best_theta, best_theta.data(), sizeof(double) * P);
  int32_t len = 0;
  host_rollout(h, snap, best_theta.data(), &out->predicted, out->trajectory, cfg.H + 1, &len);
  out->trajectory_len = len;
  out->success = out->predicted.reached && !out->predicted.collided;
  if (any_free) {
    out->action_a0 = out->predicted.first_a0;
    out->action_a1 = out->predicted.first_a1;
  } else {
    out->action_a0 = snap.actuator_delta / h->params.delta_max;
    out->action_a1 = -1.0;
  }
  out->winner = win;
}

// A deferred field never outlives its plan step (its source is the caller's
// snapshot), nor does the phase clock.
struct PendingGuard {
  pp_handle* h;
  explicit PendingGuard(pp_handle* hh) : h(hh) {}
  ~PendingGuard() {
    h->pending_field = nullptr;
    g_clock = nullptr;
  }
};

void check_warm(const pp_handle* h, int32_t len) {
  if (len != 0 && len != h->P) {
    throw std::invalid_argument("warm start vector size mismatch");  // :240-244
  }
}

}  // namespace

extern "C" {

pp_status pp_plan_step(pp_handle* h, const pp_snapshot* snap, uint64_t t, pp_plan_output* out) {
  return guarded([&] {
    if (h == nullptr || snap == nullptr || out == nullptr) {
      throw std::invalid_argument("null argument");
    }
    check_warm(h, snap->warm_theta_len);
    ck(cudaSetDevice(h->device), "cudaSetDevice");
    h->timing = pp_timing{};
    PhaseClock clock;
    g_clock = &clock;
    PendingGuard pending(h);
    upload_snapshot(h, *snap, true);  // field binned while the generator runs
    phase("upload");
    plan_step_resident(h, t, out);
    phase("done");
    g_clock = nullptr;
    clock.flush();
  });
}

pp_status pp_upload_points(pp_handle* h, const pp_snapshot_points* snap) {
  return guarded([&] {
    if (h == nullptr || snap == nullptr) throw std::invalid_argument("null argument");
    ck(cudaSetDevice(h->device), "cudaSetDevice");
    upload_points(h, *snap);
    ck(cudaStreamSynchronize(h->stream), "snapshot H2D");
  });
}

pp_status pp_plan_step_points(pp_handle* h, const pp_snapshot_points* snap, uint64_t t,
                              pp_plan_output* out) {
  return guarded([&] {
    if (h == nullptr || snap == nullptr || out == nullptr) {
      throw std::invalid_argument("null argument");
    }
    check_warm(h, snap->warm_theta_len);
    ck(cudaSetDevice(h->device), "cudaSetDevice");
    h->timing = pp_timing{};
    PhaseClock clock;
    g_clock = &clock;
    PendingGuard pending(h);
    upload_points(h, *snap, true);  // field binned while the generator runs
    phase("upload");
    plan_step_resident(h, t, out);
    phase("done");
    g_clock = nullptr;
    clock.flush();
  });
}

pp_status pp_measure_fp32_peak(int32_t device, double* tflops, double* sm_mhz) {
  return guarded([&] {
    if (tflops == nullptr || sm_mhz == nullptr) throw std::invalid_argument("null argument");
    if (pp_device_count() <= device) throw NoDevice("no such CUDA device");
    ck(static_cast<cudaError_t>(ppdev::measure_ffma(device, tflops, sm_mhz)), "ffma probe");
  });
}

}  // extern "C"

namespace ppdev {
NetKind classify(const int32_t* s, int32_t n) {
  if (n == 3 && s[0] == 5 && s[2] == 2) {
    if (s[1] == 2) return NetKind::k5_2_2;
    if (s[1] == 10) return NetKind::k5_10_2;
  }
  if (n == 4 && s[0] == 5 && s[1] == 10 && s[2] == 10 && s[3] == 2) return NetKind::k5_10_10_2;
  return NetKind::kGeneric;
}
}  // namespace ppdev
