// primitives.cpp -- host FP64 primitives of the public C++ API.
//
// These are the functions the FP64 epilogue of plan_step re-simulates the
// winner with, so every expression keeps the reference's evaluation order
// and the file is compiled with -ffp-contract=off -fno-math-errno (as the
// reference, src/CMakeLists.txt:15-17): results are bit-identical to the
// reference on the same libm. Citations are to /root/reference/proj.
#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "paraplan/dynamics.hpp"
#include "paraplan/geometry.hpp"
#include "paraplan/planner.hpp"
#include "paraplan/policy.hpp"
#include "paraplan/rng.hpp"

namespace paraplan {

namespace {
constexpr double kPi = std::numbers::pi;
constexpr std::uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

std::uint64_t splitmix_finalize(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

std::uint64_t combine(std::uint64_t h, std::uint64_t field) {
  return splitmix_finalize(h ^ (splitmix_finalize(field) + kGamma + (h << 6) + (h >> 2)));
}

void require(bool ok, const char* what) {
  if (!ok) throw std::invalid_argument(what);
}
}  // namespace

// ------------------------------------------------------------ dynamics ---
// src/dynamics.cpp:9-28
void VehicleParams::validate() const {
  require(l_f > 0.0 && l_r > 0.0, "axle distances must be positive");
  require(delta_max > 0.0 && delta_max < kPi / 2.0, "delta_max must lie in (0, pi/2)");
  require(delta_rate_max > 0.0, "delta_rate_max must be positive");
  require(u_v_min < 0.0 && 0.0 < u_v_max, "acceleration range must straddle zero");
  require(overhang_front >= 0.0 && overhang_rear >= 0.0 && half_width > 0.0,
          "chassis dimensions out of range");
  require(T_s > 0.0, "T_s must be positive");
}

// src/dynamics.cpp:30-43
Controls map_controls(const ControlAction& a, const ActuatorState& act, const VehicleParams& p) {
  const double steer = std::clamp(a.a0, -1.0, 1.0);
  const double drive = std::clamp(a.a1, -1.0, 1.0);
  const double slew = p.delta_rate_max * p.T_s;
  Controls u;
  u.delta = std::clamp(p.delta_max * steer, act.delta - slew, act.delta + slew);
  u.delta = std::clamp(u.delta, -p.delta_max, p.delta_max);
  const double w = 0.5 * (drive + 1.0);
  u.u_v = (1.0 - w) * p.u_v_min + w * p.u_v_max;
  return u;
}

// src/dynamics.cpp:45-62 (tb = tan(beta), beta never evaluated)
VehicleState step(const VehicleState& z, double delta, double u_v, const VehicleParams& p) {
  const double td = std::tan(delta);
  const double tb = p.l_r * td / (p.l_f + p.l_r);
  const double c = std::cos(z.phi);
  const double s = std::sin(z.phi);
  VehicleState n;
  n.x = z.x + p.T_s * z.v * (c - tb * s);
  n.y = z.y + p.T_s * z.v * (s + tb * c);
  n.phi = z.phi + p.T_s * z.v * td / (p.l_f + p.l_r);
  n.v = z.v + p.T_s * u_v;
  return n;
}

// src/dynamics.cpp:64-66
double idle_longitudinal(const VehicleParams& p) {
  return -1.0 - 2.0 * p.u_v_min / (p.u_v_max - p.u_v_min);
}

// ------------------------------------------------------------ geometry ---
// src/geometry.cpp:9-13
double wrap_angle(double a) {
  const double r = std::remainder(a, 2.0 * kPi);
  return r <= -kPi ? r + 2.0 * kPi : r;
}

// src/geometry.cpp:15-28
Vec2 to_ev_frame(const Pose2& anchor, const Vec2& world_pt) {
  const double dx = world_pt.x - anchor.x;
  const double dy = world_pt.y - anchor.y;
  const double c = std::cos(anchor.phi);
  const double s = std::sin(anchor.phi);
  return {c * dx + s * dy, -s * dx + c * dy};
}

Vec2 from_ev_frame(const Pose2& anchor, const Vec2& ev_pt) {
  const double c = std::cos(anchor.phi);
  const double s = std::sin(anchor.phi);
  return {anchor.x + c * ev_pt.x - s * ev_pt.y, anchor.y + s * ev_pt.x + c * ev_pt.y};
}

// src/geometry.cpp:30-41
ChassisPolytope ChassisPolytope::rectangle(const VehicleParams& p) {
  ChassisPolytope poly;
  const double front = p.front_extent(), rear = p.rear_extent();
  poly.planes_.push_back({1.0, 0.0, front});
  poly.planes_.push_back({-1.0, 0.0, rear});
  poly.planes_.push_back({0.0, 1.0, p.half_width});
  poly.planes_.push_back({0.0, -1.0, p.half_width});
  poly.bounding_radius_ = std::hypot(std::max(front, rear), p.half_width);
  return poly;
}

// src/geometry.cpp:43-61
ExtrapolatedField extrapolate(std::span<const ObstaclePoint> pts, int H, double T_s,
                              const Pose2& anchor) {
  if (H < 0) throw std::invalid_argument("horizon must be non-negative");
  ExtrapolatedField f;
  f.anchor = anchor;
  f.H = H;
  f.T_s = T_s;
  f.n_points = static_cast<int>(pts.size());
  const std::size_t n = pts.size();
  f.positions.resize(static_cast<std::size_t>(H + 1) * n);
  for (std::size_t j = 0; j < n; ++j) {
    const double vx = T_s * pts[j].speed * std::cos(pts[j].heading);
    const double vy = T_s * pts[j].speed * std::sin(pts[j].heading);
    for (int h = 0; h <= H; ++h) {
      f.positions[static_cast<std::size_t>(h) * n + j] = {pts[j].x + h * vx, pts[j].y + h * vy};
    }
  }
  return f;
}

// src/geometry.cpp:63-81
bool collision(const Pose2& pose, std::span<const Vec2> pts, const ChassisPolytope& chassis) {
  const double c = std::cos(pose.phi);
  const double s = std::sin(pose.phi);
  const double r2 = chassis.bounding_radius() * chassis.bounding_radius();
  for (const Vec2& m : pts) {
    const double dx = m.x - pose.x;
    const double dy = m.y - pose.y;
    if (dx * dx + dy * dy >= r2) continue;
    if (chassis.contains({c * dx + s * dy, -s * dx + c * dy})) return true;
  }
  return false;
}

bool collision(const Pose2& pose, std::span<const Vec2> pts, const VehicleParams& p) {
  return collision(pose, pts, ChassisPolytope::rectangle(p));
}

// -------------------------------------------------------------- policy ---
// src/policy.cpp:11-26
void MlpArchitecture::validate() const {
  require(layer_sizes.size() >= 2, "architecture needs at least 2 layers");
  require(layer_sizes.front() == 5, "input layer must have 5 units");
  require(layer_sizes.back() == 2, "output layer must have 2 units");
  for (int n : layer_sizes) {
    require(n > 0 && n <= MlpPolicy::kMaxWidth, "layer sizes must be in [1, 256]");
  }
}

// src/policy.cpp:28-34
int param_count(const MlpArchitecture& arch) {
  int total = 0;
  const auto& s = arch.layer_sizes;
  for (std::size_t l = 1; l < s.size(); ++l) total += (s[l - 1] + 1) * s[l];
  return total;
}

// src/policy.cpp:36-46
FeatureVector build_features(const VehicleState& ev, const GoalSetpoint& goal, double prev_a0,
                             const NormConstants& nc) {
  FeatureVector f;
  f[0] = (goal.x - ev.x) / nc.d_xi;
  f[1] = (goal.y - ev.y) / nc.d_eta;
  f[2] = wrap_angle(goal.phi - ev.phi) / nc.d_phi;
  f[3] = (goal.v - ev.v) / nc.d_v;
  f[4] = prev_a0;
  return f;
}

MlpPolicy::MlpPolicy(MlpArchitecture arch) : arch_(std::move(arch)) {
  arch_.validate();
  n_params_ = paraplan::param_count(arch_);
}

// src/policy.cpp:53-80
ControlAction MlpPolicy::forward(std::span<const double> theta, const FeatureVector& s) const {
  if (static_cast<int>(theta.size()) != n_params_) {
    throw std::invalid_argument("parameter vector size mismatch");
  }
  double ping[kMaxWidth];
  double pong[kMaxWidth];
  std::copy(s.begin(), s.end(), ping);
  double* in = ping;
  double* out = pong;
  const double* w = theta.data();
  const auto& sizes = arch_.layer_sizes;
  for (std::size_t l = 1; l < sizes.size(); ++l) {
    const int n_in = sizes[l - 1], n_out = sizes[l];
    const double* bias = w + static_cast<std::size_t>(n_in) * n_out;
    for (int o = 0; o < n_out; ++o) {
      double acc = bias[o];
      const double* row = w + static_cast<std::size_t>(o) * n_in;
      for (int i = 0; i < n_in; ++i) acc += row[i] * in[i];
      out[o] = std::tanh(acc);
    }
    w = bias + n_out;
    std::swap(in, out);
  }
  return {in[0], in[1]};
}

// ----------------------------------------------------------------- rng ---
// src/rng.cpp:26-58
KeyedRng::KeyedRng(std::uint64_t seed, std::uint64_t t, std::uint64_t restart,
                   std::uint64_t iter, std::uint64_t candidate) {
  std::uint64_t h = splitmix_finalize(seed + kGamma);
  for (std::uint64_t field : {t, restart, iter, candidate}) h = combine(h, field);
  state_ = h;
}

std::uint64_t KeyedRng::next_u64() {
  state_ += kGamma;
  return splitmix_finalize(state_);
}

double KeyedRng::next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

double KeyedRng::next_normal() {
  if (has_spare_) {
    has_spare_ = false;
    return spare_;
  }
  const double u1 = 1.0 - next_unit();
  const double u2 = next_unit();
  const double radius = std::sqrt(-2.0 * std::log(u1));
  const double angle = 2.0 * kPi * u2;
  spare_ = radius * std::sin(angle);
  has_spare_ = true;
  return radius * std::cos(angle);
}

// ---------------------------------------------------------- planner cfg ---
// src/planner.cpp:12-25 (+ the device extensions)
void PlannerConfig::validate() const {
  require(H >= 1, "H must be >= 1");
  require(n_candidates >= 1, "n must be >= 1");
  require(n_restarts >= 1, "N_restarts must be >= 1");
  require(n_iter_max >= 1, "N_iter_max must be >= 1");
  require(n_obst_pts >= 0, "N_obstPts must be >= 0");
  require(threads >= 1, "threads must be >= 1");
  require(sigma_log_low <= sigma_log_high, "sigma range must be ordered");
  require(tol.eps_xi > 0 && tol.eps_eta > 0 && tol.eps_phi > 0 && tol.eps_v > 0,
          "goal tolerances must be positive");
  require(precision == 32 || precision == 64, "precision must be 32 or 64");
  require(device >= 0, "device must be >= 0");
}

// src/planner.cpp:27-44
ScoreKey score(const RolloutResult& r) {
  ScoreKey k;
  k.cls = r.collided ? 0 : (r.reached ? 2 : 1);
  if (k.cls == 2) {
    k.k1 = -static_cast<double>(r.t_goal);
    k.k2 = -r.path_length;
  } else {
    k.k1 = -r.terminal_cost;
  }
  return k;
}

bool better(const ScoreKey& a, const ScoreKey& b) {
  if (a.cls != b.cls) return a.cls > b.cls;
  if (a.k1 != b.k1) return a.k1 > b.k1;
  return a.k2 > b.k2;
}

}  // namespace paraplan
