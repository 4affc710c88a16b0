// planner.cpp -- paraplan::Planner, the drop-in C++ facade over the C-ABI.
//
// Same constructor / method contract as the reference Planner
// (src/planner.cpp:46-58, 193-351): validation throws std::invalid_argument
// with the reference messages; plan_step runs on the device (pp_plan_step);
// rollout / sample_candidate / perturbation_sigma are the host FP64 paths.
// A missing or non-sm_100 GPU is a std::runtime_error at construction: the
// planner never falls back to the CPU.
#include "paraplan/planner.hpp"

#include <stdexcept>
#include <string>

#include "paraplan_cuda.h"

namespace paraplan {

namespace {

void throw_status(pp_status st) {
  if (st == PP_OK) return;
  const std::string msg = pp_last_error();
  if (st == PP_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

pp_snapshot pack(const PlanningSnapshot& s) {
  pp_snapshot c{};
  c.ev_x = s.ev_state.x;
  c.ev_y = s.ev_state.y;
  c.ev_phi = s.ev_state.phi;
  c.ev_v = s.ev_state.v;
  c.actuator_delta = s.actuator.delta;
  c.prev_a0 = s.prev_action.a0;
  c.prev_a1 = s.prev_action.a1;
  c.goal_x = s.goal.x;
  c.goal_y = s.goal.y;
  c.goal_phi = s.goal.phi;
  c.goal_v = s.goal.v;
  static_assert(sizeof(Vec2) == 2 * sizeof(double), "Vec2 must be two packed doubles");
  c.field_xy = s.obstacle_field.positions.empty()
                   ? nullptr
                   : reinterpret_cast<const double*>(s.obstacle_field.positions.data());
  c.field_H = s.obstacle_field.H;
  c.n_points = s.obstacle_field.n_points;
  if (c.n_points > 0 &&
      s.obstacle_field.positions.size() <
          static_cast<std::size_t>(s.obstacle_field.H + 1) * c.n_points) {
    throw std::invalid_argument("obstacle field has fewer positions than (H+1) x n_points");
  }
  c.warm_theta = s.warm_theta.empty() ? nullptr : s.warm_theta.data();
  c.warm_theta_len = static_cast<int32_t>(s.warm_theta.size());
  return c;
}

pp_model model_of(const VehicleParams& p, const MlpArchitecture& arch, const PlannerConfig& cfg,
                  const NormConstants& norm, std::vector<int32_t>& sizes) {
  pp_model m{};
  m.vehicle = {p.l_f,           p.l_r,          p.delta_max,     p.delta_rate_max,
               p.u_v_min,       p.u_v_max,      p.overhang_front, p.overhang_rear,
               p.half_width,    p.T_s};
  m.norm = {norm.d_xi, norm.d_eta, norm.d_phi, norm.d_v};
  pp_config& c = m.config;
  c.H = cfg.H;
  c.n_restarts = cfg.n_restarts;
  c.n_iter_max = cfg.n_iter_max;
  c.n_candidates = cfg.n_candidates;
  c.n_obst_pts = cfg.n_obst_pts;
  c.early_exit = cfg.early_exit ? 1 : 0;
  c.eps_xi = cfg.tol.eps_xi;
  c.eps_eta = cfg.tol.eps_eta;
  c.eps_phi = cfg.tol.eps_phi;
  c.eps_v = cfg.tol.eps_v;
  c.sigma_log_low = cfg.sigma_log_low;
  c.sigma_log_high = cfg.sigma_log_high;
  c.master_seed = cfg.master_seed;
  c.threads = cfg.threads;
  c.precision = cfg.precision;
  c.device = cfg.device;
  c.refine = cfg.refine ? 1 : 0;
  if (cfg.devices.size() > PP_MAX_DEVICES) throw std::invalid_argument("at most 8 devices per planner");
  c.n_devices = static_cast<int32_t>(cfg.devices.size());
  for (size_t k = 0; k < cfg.devices.size(); ++k) c.devices[k] = cfg.devices[k];
  sizes.assign(arch.layer_sizes.begin(), arch.layer_sizes.end());
  m.layer_sizes = sizes.data();
  m.n_layers = static_cast<int32_t>(sizes.size());
  return m;
}

}  // namespace

Planner::Planner(const VehicleParams& params, const MlpArchitecture& arch,
                 const PlannerConfig& cfg, const NormConstants& norm)
    : params_(params),
      cfg_(cfg),
      norm_(norm),
      policy_(arch),
      chassis_(ChassisPolytope::rectangle(params)) {
  params_.validate();
  cfg_.validate();
  std::vector<int32_t> sizes;
  const pp_model m = model_of(params_, arch, cfg_, norm_, sizes);
  throw_status(pp_create(&m, &handle_));
}

Planner::~Planner() { pp_destroy(handle_); }

namespace {
PlannerOutput unpack(const pp_plan_output& o, const std::vector<double>& traj,
                     std::vector<double> best_theta);
}

PlannerOutput Planner::plan_step(const PlanningSnapshot& snap, std::uint64_t t) const {
  const int np = param_count();
  if (!snap.warm_theta.empty() && static_cast<int>(snap.warm_theta.size()) != np) {
    throw std::invalid_argument("warm start vector size mismatch");
  }
  const pp_snapshot s = pack(snap);
  std::vector<double> theta(np, 0.0);
  std::vector<double> traj(static_cast<std::size_t>(cfg_.H + 1) * 4);
  pp_plan_output o{};
  o.best_theta = theta.data();
  o.trajectory = traj.data();
  throw_status(pp_plan_step(handle_, &s, t, &o));
  return unpack(o, traj, std::move(theta));
}

PlannerOutput Planner::plan_step_points(const PlanningSnapshot& snap,
                                        std::span<const ObstaclePoint> points,
                                        std::uint64_t t) const {
  const int np = param_count();
  if (!snap.warm_theta.empty() && static_cast<int>(snap.warm_theta.size()) != np) {
    throw std::invalid_argument("warm start vector size mismatch");
  }
  static_assert(sizeof(ObstaclePoint) == 4 * sizeof(double), "ObstaclePoint must be 4 doubles");
  pp_snapshot_points s{};
  s.ev_x = snap.ev_state.x;
  s.ev_y = snap.ev_state.y;
  s.ev_phi = snap.ev_state.phi;
  s.ev_v = snap.ev_state.v;
  s.actuator_delta = snap.actuator.delta;
  s.prev_a0 = snap.prev_action.a0;
  s.prev_a1 = snap.prev_action.a1;
  s.goal_x = snap.goal.x;
  s.goal_y = snap.goal.y;
  s.goal_phi = snap.goal.phi;
  s.goal_v = snap.goal.v;
  s.points = points.empty() ? nullptr : reinterpret_cast<const double*>(points.data());
  s.n_points = static_cast<int32_t>(points.size());
  s.T_s = params_.T_s;
  s.warm_theta = snap.warm_theta.empty() ? nullptr : snap.warm_theta.data();
  s.warm_theta_len = static_cast<int32_t>(snap.warm_theta.size());
  std::vector<double> theta(np, 0.0);
  std::vector<double> traj(static_cast<std::size_t>(cfg_.H + 1) * 4);
  pp_plan_output o{};
  o.best_theta = theta.data();
  o.trajectory = traj.data();
  throw_status(pp_plan_step_points(handle_, &s, t, &o));
  return unpack(o, traj, std::move(theta));
}

namespace {
PlannerOutput unpack(const pp_plan_output& o, const std::vector<double>& traj,
                     std::vector<double> best_theta) {
  PlannerOutput out;
  out.best_theta = std::move(best_theta);
  out.evaluated = o.evaluated;
  out.success = o.success != 0;
  out.action = {o.action_a0, o.action_a1};
  RolloutResult& r = out.predicted;
  r.reached = o.predicted.reached != 0;
  r.t_goal = o.predicted.t_goal;
  r.collided = o.predicted.collided != 0;
  r.path_length = o.predicted.path_length;
  r.terminal_cost = o.predicted.terminal_cost;
  r.first_action = {o.predicted.first_a0, o.predicted.first_a1};
  r.trajectory.resize(o.trajectory_len);
  for (int i = 0; i < o.trajectory_len; ++i) {
    r.trajectory[i] = {traj[4 * i], traj[4 * i + 1], traj[4 * i + 2], traj[4 * i + 3]};
  }
  return out;
}
}  // namespace

RolloutResult Planner::rollout(std::span<const double> theta, const PlanningSnapshot& snap) const {
  if (static_cast<int>(theta.size()) != param_count()) {
    throw std::invalid_argument("parameter vector size mismatch");
  }
  const pp_snapshot s = pack(snap);
  std::vector<double> traj(static_cast<std::size_t>(cfg_.H + 1) * 4);
  pp_rollout_stats st{};
  int32_t len = 0;
  throw_status(pp_rollout(handle_, &s, theta.data(), static_cast<int32_t>(theta.size()), &st,
                          traj.data(), cfg_.H + 1, &len));
  RolloutResult r;
  r.reached = st.reached != 0;
  r.t_goal = st.t_goal;
  r.collided = st.collided != 0;
  r.path_length = st.path_length;
  r.terminal_cost = st.terminal_cost;
  r.first_action = {st.first_a0, st.first_a1};
  r.trajectory.resize(len);
  for (int i = 0; i < len; ++i) {
    r.trajectory[i] = {traj[4 * i], traj[4 * i + 1], traj[4 * i + 2], traj[4 * i + 3]};
  }
  return r;
}

void Planner::sample_candidate(std::span<double> out, std::span<const double> center,
                               std::uint64_t t, int restart, int iter, int candidate) const {
  if (out.size() != center.size()) throw std::invalid_argument("candidate buffer size mismatch");
  throw_status(pp_sample_candidate(handle_, center.data(), static_cast<int32_t>(center.size()), t,
                                   restart, iter, candidate, out.data()));
}

double Planner::perturbation_sigma(std::uint64_t t, int restart, int iter, int candidate) const {
  return pp_perturbation_sigma(handle_, t, restart, iter, candidate);
}

}  // namespace paraplan
