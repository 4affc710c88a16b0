// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the *unmodified* reference planner, compiled from the
// reference's own sources under /root/reference/proj by oracle/Makefile into
// oracle/_ref/libparaplan_ref.so. It speaks the same PODs as the product
// boundary (include/paraplan_cuda.h) so a test can hand the identical model /
// snapshot to both sides. Only tests/, __graft_entry__.smoke() and bench.py's
// CPU-baseline leg may load it.
//
// Every entry point forwards to the reference API:
//   ref_plan_step        -> Planner::plan_step        (src/planner.cpp:238-351)
//   ref_rollout          -> Planner::rollout          (src/planner.cpp:193-205)
//   ref_sample_candidate -> Planner::sample_candidate (src/planner.cpp:207-226)
//   ref_eval_candidates  -> sample_candidate + rollout per candidate, i.e. the
//                           per-sample work of evaluate_block (:279-301)
//   ref_rng_*            -> KeyedRng                  (src/rng.cpp:26-58)
//   ref_selfchecks       -> run_selfchecks            (src/selfcheck.cpp:325-332)
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "paraplan/mission.hpp"
#include "paraplan/planner.hpp"
#include "paraplan/rng.hpp"
#include "paraplan/scenario.hpp"
#include "paraplan/selfcheck.hpp"
#include "paraplan_cuda.h"
#include "thread_pool.hpp"  // the reference pool (src/thread_pool.hpp)

#include <chrono>
#include <random>
#include <thread>

using namespace paraplan;

namespace {

thread_local std::string g_err;

struct RefPlanner {
  std::unique_ptr<Planner> planner;
};

VehicleParams to_params(const pp_vehicle& v) {
  VehicleParams p;
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

PlannerConfig to_config(const pp_config& c) {
  PlannerConfig cfg;
  cfg.H = c.H;
  cfg.n_restarts = c.n_restarts;
  cfg.n_iter_max = c.n_iter_max;
  cfg.n_candidates = c.n_candidates;
  cfg.n_obst_pts = c.n_obst_pts;
  cfg.tol.eps_xi = c.eps_xi;
  cfg.tol.eps_eta = c.eps_eta;
  cfg.tol.eps_phi = c.eps_phi;
  cfg.tol.eps_v = c.eps_v;
  cfg.sigma_log_low = c.sigma_log_low;
  cfg.sigma_log_high = c.sigma_log_high;
  cfg.master_seed = c.master_seed;
  cfg.early_exit = c.early_exit != 0;
  cfg.threads = c.threads;
  return cfg;
}

PlanningSnapshot to_snapshot(const pp_snapshot& s) {
  PlanningSnapshot snap;
  snap.ev_state = {s.ev_x, s.ev_y, s.ev_phi, s.ev_v};
  snap.actuator.delta = s.actuator_delta;
  snap.prev_action = {s.prev_a0, s.prev_a1};
  snap.goal = {s.goal_x, s.goal_y, s.goal_phi, s.goal_v};
  ExtrapolatedField& f = snap.obstacle_field;
  f.anchor = {s.ev_x, s.ev_y, s.ev_phi};
  f.H = s.field_H;
  f.n_points = s.n_points;
  const std::size_t count = static_cast<std::size_t>(s.field_H + 1) * s.n_points;
  f.positions.resize(count);
  for (std::size_t i = 0; i < count; ++i) {
    f.positions[i] = {s.field_xy[2 * i], s.field_xy[2 * i + 1]};
  }
  if (s.warm_theta_len > 0) {
    snap.warm_theta.assign(s.warm_theta, s.warm_theta + s.warm_theta_len);
  }
  return snap;
}

void fill_stats(const RolloutResult& r, pp_rollout_stats* o) {
  o->reached = r.reached;
  o->t_goal = r.t_goal;
  o->collided = r.collided;
  o->steps = static_cast<int32_t>(r.trajectory.size()) - 1;
  o->path_length = r.path_length;
  o->terminal_cost = r.terminal_cost;
  o->first_a0 = r.first_action.a0;
  o->first_a1 = r.first_action.a1;
}

int32_t copy_traj(const RolloutResult& r, double* traj, int32_t cap) {
  const int32_t n = static_cast<int32_t>(r.trajectory.size());
  if (traj != nullptr) {
    for (int32_t i = 0; i < n && i < cap; ++i) {
      traj[4 * i + 0] = r.trajectory[i].x;
      traj[4 * i + 1] = r.trajectory[i].y;
      traj[4 * i + 2] = r.trajectory[i].phi;
      traj[4 * i + 3] = r.trajectory[i].v;
    }
  }
  return n;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void* ref_create(const pp_model* m) {
  RefPlanner* rp = new RefPlanner;
  const int rc = guarded([&] {
    MlpArchitecture arch;
    arch.layer_sizes.assign(m->layer_sizes, m->layer_sizes + m->n_layers);
    rp->planner = std::make_unique<Planner>(to_params(m->vehicle), arch,
                                            to_config(m->config),
                                            NormConstants{m->norm.d_xi, m->norm.d_eta,
                                                          m->norm.d_phi, m->norm.d_v});
  });
  if (rc != 0) {
    delete rp;
    return nullptr;
  }
  return rp;
}

void ref_destroy(void* h) { delete static_cast<RefPlanner*>(h); }

int ref_param_count(void* h) { return static_cast<RefPlanner*>(h)->planner->param_count(); }

int ref_plan_step(void* h, const pp_snapshot* s, uint64_t t, pp_plan_output* out) {
  return guarded([&] {
    const Planner& p = *static_cast<RefPlanner*>(h)->planner;
    const PlanningSnapshot snap = to_snapshot(*s);
    const PlannerOutput o = p.plan_step(snap, t);
    if (out->best_theta != nullptr) {
      std::memcpy(out->best_theta, o.best_theta.data(), o.best_theta.size() * sizeof(double));
    }
    out->trajectory_len = copy_traj(o.predicted, out->trajectory, p.config().H + 1);
    out->success = o.success;
    out->action_a0 = o.action.a0;
    out->action_a1 = o.action.a1;
    fill_stats(o.predicted, &out->predicted);
    out->evaluated = o.evaluated;
    const ScoreKey k = score(o.predicted);
    out->winner = {k.cls, -1, -1, -1, k.k1, k.k2};
  });
}

int ref_rollout(void* h, const pp_snapshot* s, const double* theta, int32_t len,
                pp_rollout_stats* out, double* traj, int32_t cap, int32_t* traj_len) {
  return guarded([&] {
    const Planner& p = *static_cast<RefPlanner*>(h)->planner;
    const PlanningSnapshot snap = to_snapshot(*s);
    const RolloutResult r = p.rollout(std::span<const double>(theta, len), snap);
    fill_stats(r, out);
    const int32_t n = copy_traj(r, traj, cap);
    if (traj_len != nullptr) *traj_len = n;
  });
}

int ref_sample_candidate(void* h, const double* center, int32_t len, uint64_t t,
                         int32_t restart, int32_t iter, int32_t cand, double* out) {
  return guarded([&] {
    const Planner& p = *static_cast<RefPlanner*>(h)->planner;
    p.sample_candidate(std::span<double>(out, len), std::span<const double>(center, len), t,
                       restart, iter, cand);
  });
}

double ref_perturbation_sigma(void* h, uint64_t t, int32_t r, int32_t i, int32_t c) {
  return static_cast<RefPlanner*>(h)->planner->perturbation_sigma(t, r, i, c);
}

// Per-candidate stats of one sampling round, exactly as evaluate_block
// computes them (sample_candidate, then the rollout of that theta).
int ref_eval_candidates(void* h, const pp_snapshot* s, uint64_t t, int32_t iter,
                        int32_t restart, const double* center, int64_t c_begin,
                        int64_t c_end, pp_rollout_stats* out) {
  return guarded([&] {
    const Planner& p = *static_cast<RefPlanner*>(h)->planner;
    const PlanningSnapshot snap = to_snapshot(*s);
    const int np = p.param_count();
    std::vector<double> ctr(center, center + np);
    std::vector<double> theta(np);
    for (int64_t c = c_begin; c < c_end; ++c) {
      p.sample_candidate(theta, ctr, t, restart, iter, static_cast<int>(c));
      fill_stats(p.rollout(theta, snap), &out[c - c_begin]);
    }
  });
}

int ref_eval_theta(void* h, const pp_snapshot* s, const double* theta, int64_t n,
                   pp_rollout_stats* out) {
  return guarded([&] {
    const Planner& p = *static_cast<RefPlanner*>(h)->planner;
    const PlanningSnapshot snap = to_snapshot(*s);
    const int np = p.param_count();
    for (int64_t i = 0; i < n; ++i) {
      fill_stats(p.rollout(std::span<const double>(theta + i * np, np), snap), &out[i]);
    }
  });
}

// KeyedRng draws: kind 0 = next_u64, 1 = next_unit, 2 = next_normal.
void ref_rng_stream(uint64_t seed, uint64_t t, uint64_t r, uint64_t i, uint64_t c,
                    int32_t kind, int32_t n, void* out) {
  KeyedRng rng(seed, t, r, i, c);
  for (int32_t k = 0; k < n; ++k) {
    if (kind == 0) {
      static_cast<uint64_t*>(out)[k] = rng.next_u64();
    } else if (kind == 1) {
      static_cast<double*>(out)[k] = rng.next_unit();
    } else {
      static_cast<double*>(out)[k] = rng.next_normal();
    }
  }
}

// "name:PASS:detail\n" lines into buf; returns the number of failed checks.
int ref_selfchecks(char* buf, int32_t cap) {
  int failed = 0;
  std::string text;
  for (const CheckResult& c : run_selfchecks()) {
    failed += c.pass ? 0 : 1;
    text += c.name + (c.pass ? ":PASS:" : ":FAIL:") + c.detail + "\n";
  }
  std::snprintf(buf, cap, "%s", text.c_str());
  return failed;
}

// Snapshot of tick t of a builtin mission exactly as run_mission builds it
// (select_goal -> sense -> extrapolate, src/mission.cpp:124-144). The field
// is written to field_xy (capacity cap doubles); returns n_points or -1.
int ref_builtin_snapshot(const char* name, int32_t t, int32_t H, int32_t n_obst_pts,
                         int32_t drop_dynamic, pp_snapshot* out, double* field_xy,
                         int64_t cap) {
  int n = -1;
  guarded([&] {
    const ScenarioSpec spec = builtin_scenario(name);
    Mission m = spec.mission;
    if (drop_dynamic) m.dynamic_points.clear();
    const VehicleParams params;
    const VehicleState ev = m.initial_state;
    const GoalSelection sel = select_goal(m, ev, 0, GoalTolerance{});
    const std::vector<ObstaclePoint> pts = sense(m, ev, t, n_obst_pts, params.T_s);
    const ExtrapolatedField f = extrapolate(pts, H, params.T_s, {ev.x, ev.y, ev.phi});
    out->ev_x = ev.x;
    out->ev_y = ev.y;
    out->ev_phi = ev.phi;
    out->ev_v = ev.v;
    out->actuator_delta = 0.0;
    out->prev_a0 = 0.0;
    out->prev_a1 = idle_longitudinal(params);
    out->goal_x = sel.goal.x;
    out->goal_y = sel.goal.y;
    out->goal_phi = sel.goal.phi;
    out->goal_v = sel.goal.v;
    out->field_H = f.H;
    out->n_points = f.n_points;
    out->warm_theta = nullptr;
    out->warm_theta_len = 0;
    if (static_cast<int64_t>(2 * f.positions.size()) > cap) throw std::runtime_error("cap");
    for (std::size_t k = 0; k < f.positions.size(); ++k) {
      field_xy[2 * k] = f.positions[k].x;
      field_xy[2 * k + 1] = f.positions[k].y;
    }
    out->field_xy = field_xy;
    n = f.n_points;
  });
  return n;
}

// Snapshot of tick t of a caller-described mission, built by the reference's
// own select_goal -> sense -> extrapolate (src/mission.cpp:124-144). The
// mission: waypoints (x, y, phi, v) x n_wp, static and dynamic points
// (x, y, heading, speed) in the world frame, EV state (x, y, phi, v). Used by
// bench.py's reference arm so that process loads only oracle/_ref.
int ref_mission_snapshot(const double* waypoints, int32_t n_wp, const double* static_pts,
                         int32_t n_static, const double* dyn_pts, int32_t n_dyn,
                         const double* ev_state, int32_t t, int32_t H, int32_t n_obst_pts,
                         pp_snapshot* out, double* field_xy, int64_t cap) {
  int n = -1;
  guarded([&] {
    Mission m;
    for (int32_t i = 0; i < n_wp; ++i) {
      const double* w = waypoints + 4 * i;
      m.waypoints.push_back(GoalSetpoint{w[0], w[1], w[2], w[3]});
    }
    for (int32_t i = 0; i < n_static; ++i) {
      const double* q = static_pts + 4 * i;
      m.static_points.push_back(ObstaclePoint{q[0], q[1], q[2], q[3]});
    }
    for (int32_t i = 0; i < n_dyn; ++i) {
      const double* q = dyn_pts + 4 * i;
      m.dynamic_points.push_back(ObstaclePoint{q[0], q[1], q[2], q[3]});
    }
    m.initial_state = VehicleState{ev_state[0], ev_state[1], ev_state[2], ev_state[3]};
    const VehicleParams params;
    const VehicleState ev = m.initial_state;
    const GoalSelection sel = select_goal(m, ev, 0, GoalTolerance{});
    const std::vector<ObstaclePoint> pts = sense(m, ev, t, n_obst_pts, params.T_s);
    const ExtrapolatedField f = extrapolate(pts, H, params.T_s, {ev.x, ev.y, ev.phi});
    out->ev_x = ev.x;
    out->ev_y = ev.y;
    out->ev_phi = ev.phi;
    out->ev_v = ev.v;
    out->actuator_delta = 0.0;
    out->prev_a0 = 0.0;
    out->prev_a1 = idle_longitudinal(params);
    out->goal_x = sel.goal.x;
    out->goal_y = sel.goal.y;
    out->goal_phi = sel.goal.phi;
    out->goal_v = sel.goal.v;
    out->field_H = f.H;
    out->n_points = f.n_points;
    out->warm_theta = nullptr;
    out->warm_theta_len = 0;
    if (static_cast<int64_t>(2 * f.positions.size()) > cap) throw std::runtime_error("cap");
    for (std::size_t k = 0; k < f.positions.size(); ++k) {
      field_xy[2 * k] = f.positions[k].x;
      field_xy[2 * k + 1] = f.positions[k].y;
    }
    out->field_xy = field_xy;
    n = f.n_points;
  });
  return n;
}

// Parallel-efficiency calibration of the host: each of
// `threads` workers runs `ms` milliseconds' worth (single-thread calibrated)
// of independent spin work; returns the wall-clock milliseconds of the whole
// fork-join. pool = 0: raw std::thread per worker; pool = 1: the reference's
// own detail::ThreadPool (src/thread_pool.hpp:33-49), worker 0 on the caller.
double ref_spin_calibration(int32_t threads, double ms, int32_t pool) {
  using clk = std::chrono::steady_clock;
  auto spin = [](uint64_t n) {
    volatile uint64_t x = 0x9E3779B97F4A7C15ull;
    for (uint64_t i = 0; i < n; ++i) x = x * 6364136223846793005ull + 1442695040888963407ull;
    return x;
  };
  // iterations per millisecond on one thread
  uint64_t n = 1 << 16;
  for (;;) {
    const auto t0 = clk::now();
    spin(n);
    const double dt = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
    if (dt > 5.0) {
      n = static_cast<uint64_t>(static_cast<double>(n) * ms / dt);
      break;
    }
    n *= 2;
  }
  const int w = threads < 1 ? 1 : threads;
  const auto t0 = clk::now();
  if (pool != 0) {
    static thread_local std::unique_ptr<paraplan::detail::ThreadPool> tp;
    if (!tp || tp->workers() != w) tp = std::make_unique<paraplan::detail::ThreadPool>(w);
    const auto t1 = clk::now();
    tp->run([&](int) { spin(n); });
    return std::chrono::duration<double, std::milli>(clk::now() - t1).count();
  }
  std::vector<std::thread> ts;
  for (int i = 1; i < w; ++i) ts.emplace_back([&] { spin(n); });
  spin(n);
  for (auto& t : ts) t.join();
  return std::chrono::duration<double, std::milli>(clk::now() - t0).count();
}

// Snapshot i (0-based) of the reference's acceptance criterion 9 sequence
// (tests/acceptance_test.cpp:271-334): mt19937_64(4242), the same
// distributions drawn in the same order, points extrapolated over H = 60 by
// the reference's extrapolate. warm (capacity 18) receives the warm start
// when the sequence draws one (*warm_len = 18, else 0). Returns n_points.
int ref_acceptance9_snapshot(int32_t index, int32_t H, pp_snapshot* out, double* field_xy,
                             int64_t cap, double* warm, int32_t* warm_len) {
  int n = -1;
  guarded([&] {
    constexpr double pi = 3.141592653589793;
    std::mt19937_64 rng(4242);
    std::uniform_real_distribution<double> pos(-20.0, 20.0);
    std::uniform_real_distribution<double> ang(-2.0 * pi, 2.0 * pi);
    std::uniform_real_distribution<double> vel(-8.0, 12.0);
    std::uniform_real_distribution<double> unit(-1.0, 1.0);
    std::uniform_int_distribution<int> n_pts(0, 12);
    for (int i = 0; i <= index; ++i) {
      PlanningSnapshot snap;
      snap.ev_state.x = pos(rng);
      snap.ev_state.y = pos(rng);
      snap.ev_state.phi = ang(rng);
      snap.ev_state.v = vel(rng);
      snap.actuator.delta = 0.6 * unit(rng);
      snap.prev_action.a0 = 0.9 * unit(rng);
      snap.prev_action.a1 = 0.9 * unit(rng);
      snap.goal.x = snap.ev_state.x + pos(rng);
      snap.goal.y = snap.ev_state.y + pos(rng);
      snap.goal.phi = ang(rng);
      snap.goal.v = vel(rng);
      std::vector<ObstaclePoint> pts;
      const int count = n_pts(rng);
      for (int j = 0; j < count; ++j) {
        ObstaclePoint q;
        q.x = snap.ev_state.x + pos(rng);
        q.y = snap.ev_state.y + pos(rng);
        q.heading = ang(rng);
        q.speed = std::abs(vel(rng));
        pts.push_back(q);
      }
      const ExtrapolatedField f =
          extrapolate(pts, H, 0.1, {snap.ev_state.x, snap.ev_state.y, snap.ev_state.phi});
      std::vector<double> wt;
      if (unit(rng) > 0.0) {
        wt.resize(18);
        for (double& w : wt) w = unit(rng);
      }
      if (i < index) continue;
      out->ev_x = snap.ev_state.x;
      out->ev_y = snap.ev_state.y;
      out->ev_phi = snap.ev_state.phi;
      out->ev_v = snap.ev_state.v;
      out->actuator_delta = snap.actuator.delta;
      out->prev_a0 = snap.prev_action.a0;
      out->prev_a1 = snap.prev_action.a1;
      out->goal_x = snap.goal.x;
      out->goal_y = snap.goal.y;
      out->goal_phi = snap.goal.phi;
      out->goal_v = snap.goal.v;
      out->field_H = f.H;
      out->n_points = f.n_points;
      if (static_cast<int64_t>(2 * f.positions.size()) > cap) throw std::runtime_error("cap");
      for (std::size_t k = 0; k < f.positions.size(); ++k) {
        field_xy[2 * k] = f.positions[k].x;
        field_xy[2 * k + 1] = f.positions[k].y;
      }
      out->field_xy = field_xy;
      *warm_len = static_cast<int32_t>(wt.size());
      for (std::size_t k = 0; k < wt.size(); ++k) warm[k] = wt[k];
      out->warm_theta = wt.empty() ? nullptr : warm;
      out->warm_theta_len = static_cast<int32_t>(wt.size());
      n = f.n_points;
    }
  });
  return n;
}

// Closed-loop mission through the reference run_mission; per-tick records as
// 8 doubles (t, x, y, phi, v, a0, a1, delta). Returns the record count.
int ref_run_mission_builtin(const char* name, int32_t H, int32_t n_candidates,
                            int32_t n_restarts, double time_limit, uint64_t seed,
                            int32_t threads, double* rec, int32_t cap, double* tau_avg) {
  int count = -1;
  guarded([&] {
    ScenarioSpec spec = builtin_scenario(name);
    PlannerConfig cfg = spec.planner;
    cfg.H = H;
    cfg.n_candidates = n_candidates;
    cfg.n_restarts = n_restarts;
    cfg.threads = threads;
    Mission m = spec.mission;
    if (time_limit >= 0) m.time_limit = time_limit;
    const SimulationLog log = run_mission(m, cfg, spec.arch, seed);
    count = static_cast<int>(log.records.size());
    for (int k = 0; k < count && k < cap; ++k) {
      const TickRecord& r = log.records[k];
      double* o = rec + 8 * k;
      o[0] = r.t;
      o[1] = r.state.x;
      o[2] = r.state.y;
      o[3] = r.state.phi;
      o[4] = r.state.v;
      o[5] = r.action.a0;
      o[6] = r.action.a1;
      o[7] = r.delta;
    }
    if (tau_avg != nullptr) *tau_avg = log.stats.tau_avg;
  });
  return count;
}

// The reference's serialize_scenario of a builtin scenario into buf (the
// length is returned; -1 on error).
int ref_serialize_builtin(const char* name, char* buf, int32_t cap) {
  int n = -1;
  guarded([&] {
    const std::string text = serialize_scenario(builtin_scenario(name));
    n = static_cast<int>(text.size());
    if (n < cap) std::memcpy(buf, text.data(), text.size() + 1);
  });
  return n;
}

// The reference's run_sweep on a builtin scenario with a reduced budget:
// every output file (scenario JSON, report JSON, per-seed CSV and xy) is
// written to out_dir exactly as the reference writes it.
int ref_run_sweep_builtin(const char* name, int32_t H, int32_t n_candidates, int32_t n_restarts,
                          double time_limit, const uint64_t* seeds, int32_t n_seeds,
                          int32_t threads, const char* out_dir) {
  int ok = -1;
  guarded([&] {
    ScenarioSpec spec = builtin_scenario(name);
    spec.planner.H = H;
    spec.planner.n_candidates = n_candidates;
    spec.planner.n_restarts = n_restarts;
    if (time_limit >= 0) spec.mission.time_limit = time_limit;
    spec.seeds.assign(seeds, seeds + n_seeds);
    run_sweep(spec, out_dir, threads);
    ok = 0;
  });
  return ok;
}

}  // extern "C"
