// host_exact.cpp -- the reference's FP64 rollout (src/planner.cpp:66-191)
// and candidate sampling (:207-226) on the host, through the public
// primitives: the epilogue and the exact evaluations of the certification.
#include "capi_internal.hpp"

namespace ppcapi {

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

// The checks of state 0 alone (src/planner.cpp:137-153 at h = 0), which no
// candidate's theta can influence: returns true when every rollout stops
// there, with the (common) exact key's stats in *out.
bool host_stops_at_state0(const pp_handle* h, const pp_snapshot& s, pp_rollout_stats* out) {
  using namespace paraplan;
  const auto& cfg = h->cfg;
  const Pose2 anchor{s.ev_x, s.ev_y, s.ev_phi};
  const Vec2 gp = to_ev_frame(anchor, {s.goal_x, s.goal_y});
  const GoalSetpoint goal{gp.x, gp.y, s.goal_phi - anchor.phi, s.goal_v};
  const double gc = std::cos(goal.phi), gs = std::sin(goal.phi);
  const VehicleState z{0.0, 0.0, 0.0, s.ev_v};
  std::memset(out, 0, sizeof(*out));
  out->t_goal = -1;
  bool stop = false;
  if (s.n_points > 0) {
    bool hit;
    if (s.field_xy == nullptr) {
      hit = ppfield::collides(h->field, h->chassis, h->box, 0, z.x, z.y, z.phi);
    } else {
      const std::span<const Vec2> row(reinterpret_cast<const Vec2*>(s.field_xy), s.n_points);
      hit = collision({z.x, z.y, z.phi}, row, h->chassis);
    }
    if (hit) {
      out->collided = 1;
      stop = true;
    }
  }
  if (!stop) {
    const double gdx = goal.x - z.x, gdy = goal.y - z.y;
    if (std::abs(gc * gdx + gs * gdy) <= cfg.tol.eps_xi &&
        std::abs(-gs * gdx + gc * gdy) <= cfg.tol.eps_eta &&
        std::abs(wrap_angle(goal.phi - z.phi)) <= cfg.tol.eps_phi &&
        std::abs(goal.v - z.v) <= cfg.tol.eps_v) {
      out->reached = 1;
      out->t_goal = 0;
      stop = true;
    }
  }
  if (!stop && cfg.H != 0) return false;
  out->terminal_cost = std::abs(goal.x - z.x) / h->norm.d_xi +
                       std::abs(goal.y - z.y) / h->norm.d_eta +
                       std::abs(wrap_angle(goal.phi - z.phi)) / h->norm.d_phi +
                       std::abs(goal.v - z.v) / h->norm.d_v;
  return true;
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

}  // namespace ppcapi
