// upload.cpp -- a snapshot into the planner: round constants (goal in the
// anchor frame, src/planner.cpp:70-81) and the obstacle field, split into
// static and dynamic points and binned (field.hpp), packed into the device
// image in the compute precision and copied to HBM; large mover sets are
// binned by the device itself (csrc/cuda/binning_f64.cu).
#include "capi_internal.hpp"

namespace ppcapi {

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
  k->ts_umid = Real(a.T_s * 0.5 * (a.u_v_min + a.u_v_max));
  k->ts_uhalf = Real(a.T_s * 0.5 * (a.u_v_max - a.u_v_min));
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
  // FP64: 1e-12 absolute (~1000x a state's FP64 error after one step)
  k->dmarg = sizeof(Real) == sizeof(float) ? Real(a.dmarg32) : Real(1e-12);
  // the relative drift of the state after h steps, bounded like a class-2
  // window's rho: FP32 1e-3 (h / 150)^2, at least 2e-6 (>= 8x the measured
  // path error at every h); FP64 1e-9 (h / 150)^2, at least 1e-12 (the
  // measured FP64 cost error at the winners is <= 5.1e-10 at h = 200). Short
  // FP32 horizons keep the fixed band (their drift stays below it)
  k->dmarg_rel = sizeof(Real) == sizeof(float) ? Real(a.H > fp32_max_h() ? 1e-3 : 0.0)
                                               : Real(1e-9);
  k->dmarg_floor = sizeof(Real) == sizeof(float) ? Real(2e-6) : Real(1e-12);
  k->bcx = Real(0.5 * (a.fe - a.re));
  k->bhx = Real(0.5 * (a.fe + a.re));
  k->inv_wb = Real(1.0 / a.wheelbase);
  k->wb_d = a.wheelbase;
  k->tan_small = a.delta_max <= 0.785 ? 1 : 0;
  k->flag_miss = 0;  // per round (round.cpp)
  k->H = a.H;
  k->any_pts = a.field_ns + a.field_nd > 0 ? 1 : 0;
  const bool dyn = a.field_nd > 0;  // field_query.cuh bind_shared: the staged part
  k->k3_row_bytes = dyn ? static_cast<uint32_t>(a.field_dstride * 2 * sizeof(Real)) : 0u;
  k->k3_st_row_bytes = dyn ? static_cast<uint32_t>((a.grid_nx + 1) * sizeof(int)) : 0u;
  k->xtop = Real(a.grid_nx - 1);
  k->ytop = Real(a.grid_ny - 1);
}

// Device image of h->field in the compute precision (one H2D); the FP64 image
// for the near-tie re-ranking is uploaded only when a round needs it.
void finish_field(pp_handle* h, ppdev::RoundArgs& a) {
  {  // single-part x-bucket fields: sentinel padding for kernel kind 3
    ppfield::Binned& m = h->field;
    const bool one_part = m.Ns == 0 || m.Nd == 0;
    const bool pad = m.mode() == 0 && one_part && !m.dyn_deferred;
    // a window starts at a point index <= N and the warp reads up to its
    // longest window rounded up to a whole group: N + kK3Group - 1 sentinels
    m.pad_s = pad && m.Nd == 0 ? m.Ns + ppdev::kK3Group - 1 : 0;
    m.pad_d = pad && m.Ns == 0 ? m.Nd + ppdev::kK3Group - 1 : 0;
  }
  const ppfield::Binned& b = h->field;
  a.field_ns = b.Ns;
  a.field_nd = b.Nd;
  a.field_dstride = b.Nd + b.pad_d;
  a.field_padded = (b.pad_s > 0 || b.pad_d > 0) ? 1 : 0;
  a.grid_nx = b.nx;
  a.grid_ny = b.ny;
  a.grid_x0 = b.x0;
  a.grid_y0 = b.y0;
  a.grid_g = b.g;
  a.grid_mode = b.mode();
  // cooperative window scans pay where a window holds many points: dense
  // static clouds (cell boxes), or 2-D grids averaging >= 1 point per cell
  a.coop = b.mode() == 2 ||
           (b.mode() == 1 && b.Ns + static_cast<double>(b.Nd) >= static_cast<double>(b.cells()));
  const size_t elem = h->fp64 ? sizeof(double) : sizeof(float);
  const ppfield::Layout l = ppfield::layout(b, elem), l64 = ppfield::layout(b, sizeof(double));
  a.lay = {static_cast<int64_t>(l.dpts), static_cast<int64_t>(l.sst), static_cast<int64_t>(l.dst),
           static_cast<int64_t>(l.sbox), static_cast<int64_t>(l.cst), static_cast<int64_t>(l.cbox),
           static_cast<int64_t>(l.bytes)};
  a.lay64 = {static_cast<int64_t>(l64.dpts), static_cast<int64_t>(l64.sst),
             static_cast<int64_t>(l64.dst), static_cast<int64_t>(l64.sbox),
             static_cast<int64_t>(l64.cst), static_cast<int64_t>(l64.cbox),
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
      phase("packed");
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
      part(l.sbox, l.bytes); // static cell and chunk boxes
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
      ba.sms = h->sms;
      ck(static_cast<cudaError_t>(ppdev::bin_movers(ba, st)), "mover binning");
      h->timing.launches += 3;
    } else {
      ppfield::pack(b, h->fp64, h->h_field.p);
      phase("field-packed");
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
void upload_points(pp_handle* h, const pp_snapshot_points& p, bool defer) {
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
    phase("points-binned");
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
void upload_snapshot(pp_handle* h, const pp_snapshot& s, bool defer) {
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
  a.sms = h->sms;
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
    phase("rows-binned");
  } else {
    h->field = ppfield::Binned{};
    h->field.rows = cfg.H + 1;
    h->field.cull = cull;
  }
  finish_field(h, a);
}

}  // namespace ppcapi
