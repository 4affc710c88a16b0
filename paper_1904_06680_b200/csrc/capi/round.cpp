// round.cpp -- one sampling round on the device (generator -> rollout ->
// window select, src/planner.cpp:259-336 for one restart x iteration block)
// and the certified re-ranking of its winners in the reference's FP64
// arithmetic (PlannerConfig::refine).
#include "capi_internal.hpp"

namespace ppcapi {

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


// Selection buffers of capacity `cap`: the indices beyond the round block's
// first kSelFirst, the refine kernel's input list and its FP64 keys.
void grow_selection(pp_handle* h, ppdev::RoundArgs& a, int cap) {
  h->sel_cap = std::max(h->sel_cap, cap);
  h->d_selmore.reserve(sizeof(int64_t) * (h->sel_cap - kSelFirst), "selection");
  h->d_reflist.reserve(sizeof(int64_t) * h->sel_cap, "refine list");
  h->d_sel.reserve(sizeof(ppdev::SelRec) * h->sel_cap, "refine keys");
  a.sel_more = static_cast<int64_t*>(h->d_selmore.p);
  a.ref_list = static_cast<const int64_t*>(h->d_reflist.p);
  a.sel_out = static_cast<ppdev::SelRec*>(h->d_sel.p);
  a.sel_cap = h->sel_cap;
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

// The certification's error model (measured: profiles/r2_error_model*.json,
// tests/measure_fp_error.py). The device rollout's relative cost
// error against the reference's own FP64 arithmetic, at the exact winner:
//   FP32, class 2 (reached; cost = path length), any H:   <= 2.1e-5
//   FP32, class 0/1 (cost = terminal cost), H <= 30:      <= 1.4e-6
//   FP32, class 0/1, H >= 60:  up to 2.2e-2 (H 60) ... 0.5 (H 200): chaotic
//                              amplification through saturated steering
//   FP64 (no contraction), class 0/1: <= 2e-12 (H <= 60), <= 5.6e-9 (H 200);
//   class 2: <= 1.1e-13
// So an FP32 round is certified with rho = 1e-3 only where that envelope
// holds with a wide margin: every class up to H = fp32_max_h() (40), class 2
// beyond. A longer round whose anchor is of class 0/1 is redone in FP64, and
// FP64 rounds use rho64(H).
// FP64 windows: class 0/1 anchors (terminal cost) by the horizon; class 2
// (path length of a reaching rollout, measured FP64 error <= 1.1e-13)
double rho64(int H) { return H <= 60 ? 1e-9 : 1e-6; }
constexpr double kRho64Reached = 1e-11;
constexpr double kRho64ReachedFloor = 2e-14;

// Occupancy of the rollout kernel for (precision, staged field size, grid
// mode), queried once per handle.
ppdev::LaunchShape launch_shape(pp_handle* h, bool fp64, int field_smem, int kind) {
  const int64_t key = (static_cast<int64_t>(field_smem) << 8) | (kind << 1) | (fp64 ? 1 : 0);
  auto found = h->shapes.find(key);
  if (found == h->shapes.end()) {
    ppdev::LaunchShape sh{};
    const int rcode = fp64 ? ppdev::shape_f64(h->kind, h->device, field_smem, kind, &sh)
                           : ppdev::shape_f32(h->kind, h->device, field_smem, kind, &sh);
    ck(static_cast<cudaError_t>(rcode), "occupancy query");
    found = h->shapes.emplace(key, sh).first;
  }
  return found->second;
}

void consume_pending_field(pp_handle* h, bool side) {
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
// The round's params block, [prefix u64 x n_prefix][centre f64 x P][centre
// rounded to f32 x P] (the FP32 generator adds sigma * N(0,1) to the float
// centre; the host's (float) rounding is the device's), on the handle's
// stream; a.key_prefix / a.center / a.center_f point into it.
void upload_params(pp_handle* h, ppdev::RoundArgs& a, const uint64_t* prefix, int n_prefix,
                   const double* center) {
  const size_t pbytes = sizeof(uint64_t) * n_prefix + sizeof(double) * h->P + sizeof(float) * h->P;
  h->h_params.reserve(pbytes, "pinned params");
  h->d_params.reserve(pbytes, "device params");
  uint64_t* hp = static_cast<uint64_t*>(h->h_params.p);
  std::memcpy(hp, prefix, sizeof(uint64_t) * n_prefix);
  double* hc = reinterpret_cast<double*>(hp + n_prefix);
  float* hf = reinterpret_cast<float*>(hc + h->P);
  for (int i = 0; i < h->P; ++i) {
    hc[i] = center != nullptr ? center[i] : 0.0;
    hf[i] = static_cast<float>(hc[i]);
  }
  ck(cudaMemcpyAsync(h->d_params.p, h->h_params.p, pbytes, cudaMemcpyHostToDevice, h->stream),
     "params H2D");
  h->timing.h2d_bytes += static_cast<int64_t>(pbytes);
  const uint64_t* dp = static_cast<const uint64_t*>(h->d_params.p);
  a.key_prefix = dp;
  a.center = reinterpret_cast<const double*>(dp + n_prefix);
  a.center_f = reinterpret_cast<const float*>(a.center + h->P);
}

void run_round_launch(pp_handle* h, uint64_t t, int iter, int r0, int rc, const double* center,
                      int64_t c0, int64_t c1, const double* injected, pp_record* out,
                      pp_rollout_stats* per_sample, bool force_fp64) {
  const int64_t count = c1 - c0;
  // the last round of this planner needed FP64 (class 0/1 beyond the FP32
  // envelope): start in FP64 (a closed loop's ticks look alike)
  if (!h->fp64 && h->prefer_fp64 && h->rerank && h->snapshot != nullptr &&
      per_sample == nullptr && h->cfg.H > fp32_max_h()) {
    force_fp64 = true;
  }
  const bool fp64 = h->fp64 || force_fp64;
  const bool rerank = h->rerank && h->snapshot != nullptr;
  // the schedule (refill: generator + rollout) and the theta record width do
  // not depend on the field
  const ppdev::LaunchShape shape0 = launch_shape(h, fp64, 0, 0);
  // a pending field is binned while the generator runs; without a generator
  // (lockstep) or for an FP64 redo it is needed now
  if (h->pending_field && (!shape0.refill || force_fp64)) consume_pending_field(h);
  ppdev::RoundArgs a = h->base;
  if (a.sms <= 0) throw std::logic_error("round constants without a device SM count");
  if (force_fp64 && !h->fp64) {
    a.field = ensure_field64(h);
    a.lay = a.lay64;
  }
  a.restart_count = rc;
  a.cand_begin = c0;
  a.count = count;
  a.queue_bytes = 0;

  std::vector<uint64_t> prefixes(rc);
  for (int r = 0; r < rc; ++r) {
    prefixes[r] = key_prefix(h->cfg.master_seed, t, static_cast<uint64_t>(r0 + r),
                             static_cast<uint64_t>(iter));
  }
  upload_params(h, a, prefixes.data(), rc, center);

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
    a.theta_buf = h->d_theta.p;  // [total][theta_elem]: theta, state 1, pad
    a.first_buf = nullptr;
  }
  // goal-horizon cut (refill schedule; per-sample rounds keep every rollout)
  // (with the cut's kernel only when the planner's last round reached: a
  // round nobody reaches runs ~6% faster without its instructions)
  const bool cut = shape0.refill && per_sample == nullptr && !h->no_cut && goal_cut_enabled() &&
                   h->expect_reach;
  a.goal_cut = cut ? reinterpret_cast<uint32_t*>(dres + kCutOff) : nullptr;
  a.cut_pub = reinterpret_cast<uint32_t*>(dres + kCutPubOff);
  a.cut_slack = cut_slack();
  a.cut_slots = rc;
  a.flush_every = flush_every_fixed() > 0 ? flush_every_fixed() : h->flush_every;
  a.flush_min = flush_every_fixed() > 0 ? 0 : h->flush_min;
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
    grow_selection(h, a, h->sel_cap);
    a.sel_list = reinterpret_cast<int64_t*>(dres + kSelOff);
    a.refine_grid = refine_grid(h);
    a.sel_rho = fp64 ? rho64(h->cfg.H) : h->sel_rho;
    a.sel_rho2 = fp64 ? kRho64Reached : h->sel_rho;
    a.sel_rho2_floor = fp64 ? kRho64ReachedFloor : 2e-6;
    a.rho2_by_tgoal = 1;
    a.sel_alpha = fp64 ? 1e-13 : 1e-6;
  }

  phase("buffers");
  ck(cudaEventRecord(h->ev0, h->stream), "event");
  ck(static_cast<cudaError_t>(fp64 ? ppdev::launch_generate_f64(h->kind, a, h->stream)
                                   : ppdev::launch_generate_f32(h->kind, a, h->stream)),
     "theta generator launch");
  phase("generator");
  if (h->pending_field) {  // bin + upload the field while the generator runs
    consume_pending_field(h, true);
    const ppdev::RoundArgs& b = h->base;
    a.field = b.field;
    a.field64 = b.field64;
    a.n_points = b.n_points;
    a.field_ns = b.field_ns;
    a.field_nd = b.field_nd;
    a.field_dstride = b.field_dstride;
    a.field_padded = b.field_padded;
    a.grid_nx = b.grid_nx;
    a.grid_ny = b.grid_ny;
    a.grid_mode = b.grid_mode;
    a.coop = b.coop;
    a.grid_x0 = b.grid_x0;
    a.grid_y0 = b.grid_y0;
    a.grid_g = b.grid_g;
    a.lay = b.lay;
    a.lay64 = b.lay64;
    a.kf = b.kf;
    a.kd = b.kd;
  }
  const int field_smem = (force_fp64 && !h->fp64) ? 0 : h->field_smem_bytes;
  const ppdev::LaunchShape shape = launch_shape(
      h, fp64, field_smem, ppdev::grid_kind(a.grid_mode, field_smem, a.field_ns, a.field_nd,
                                        a.field_padded));
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
  const size_t n_recs = shape.refill ? 2 * static_cast<size_t>(rc) * std::max(a.grid, h->sms * 4)
                                    : static_cast<size_t>(a.n_tiles);
  h->d_tiles.reserve(sizeof(ppdev::Rec) * n_recs, "tile records");
  a.tile_recs = static_cast<ppdev::Rec*>(h->d_tiles.p);
  // theta in a global per-lane column (NetGlobal): any architecture without
  // a register specialisation in this precision ([5,10,10,2] has one in FP32)
  const bool generic = h->kind == ppdev::NetKind::kGeneric ||
                       (fp64 && h->kind == ppdev::NetKind::k5_10_10_2);
  if (generic || rerank) {
    const size_t lanes = std::max<size_t>(generic ? static_cast<size_t>(a.grid) * a.block : 0,
                                          rerank ? refine_grid(h) * 128 : 0);
    h->d_scratch.reserve(lanes * h->P * sizeof(double), "theta scratch");
    a.theta_scratch = static_cast<float*>(h->d_scratch.p);
    a.theta_scratch64 = static_cast<double*>(h->d_scratch.p);
  }
  // several restarts: narrow collision misses are marginal too (step.cuh)
  a.kf.flag_miss = rc > 1 ? 1 : 0;
  a.kd.flag_miss = rc > 1 ? 1 : 0;
  ck(static_cast<cudaError_t>(fp64 ? ppdev::launch_rollout_f64(h->kind, a, h->stream)
                                   : ppdev::launch_rollout_f32(h->kind, a, h->stream)),
     "sampling kernel launch");
  // sharded plan step: the shards exchange their per-restart winners
  const bool sharded = h->xchg_active && h->xchg != nullptr;
  const bool packed = sharded && rerank && injected == nullptr &&
                      h->cfg.n_candidates <= ppdev::kPackMaxCandidates &&
                      h->cfg.H <= ppdev::kPackMaxTGoal;
  if (rerank) {
    if (packed) {
      // one min-allreduce of the packed winners in the stream, then every
      // shard's window is anchored on the global best (keypack.h)
      a.pkeys = reinterpret_cast<uint64_t*>(dres + kPackOff);
      ck(static_cast<cudaError_t>(ppdev::launch_pack_keys(a, h->stream)), "pack keys launch");
      h->xchg->allreduce_min_u64(a.pkeys, 2 * rc, h->stream);
      a.sel_packed = 1;
      h->timing.launches += 2;
    }
    // the selection counter was re-armed by the rollout kernel's last CTA;
    // sharded rounds without packed keys select after a host exchange
    // (certify_round)
    if (!sharded || packed) {
      ck(static_cast<cudaError_t>(ppdev::launch_select(a, h->stream)), "window select launch");
    }
    if (h->pool == nullptr) h->pool = shared_pool().pool.get();
  }
  // one D2H: counters (selection count), work counters, winners and the
  // first kSelFirst selected indices, stored into pinned host memory by a
  // dependent kernel right behind the last round kernel (no event between
  // them, which would break the programmatic dependency)
  ck(static_cast<cudaError_t>(
         ppdev::launch_copy_out(h->d_round.p, h->h_round.p, (rbytes + 15) / 16 * 16, kExecOff,
                                h->stream)),
     "result D2H");
  ck(cudaEventRecord(h->ev1, h->stream), "event");
  phase("enqueued");
  // the host's exact image of device-binned movers, while the round runs
  if (h->field.dyn_deferred) {
    ppfield::bin_dynamic(h->field);
    phase("host-binned");
  }
  // then the certification's workers spin while the GPU finishes (woken
  // after the binning, whose threads they would otherwise crowd out)
  if (rerank) h->pool->prewarm();
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
  // the round's device span: first kernel start to the result store
  // (copy_out_kernel), else the events around the launches (no generator)
  const char* hres = static_cast<const char*>(h->h_round.p);
  const unsigned long long* ex = reinterpret_cast<const unsigned long long*>(hres + kExecOff);
  double ms = 1e-6 * static_cast<double>(ex[ppdev::kExecRoundT0]);
  if (ex[ppdev::kExecRoundT0] == 0ull) {
    float ems = 0.f;
    ck(cudaEventElapsedTime(&ems, h->ev0, h->ev1), "event timing");
    ms = ems;
  }
  phase("evtime");
  if (trace_level() >= 2) std::fprintf(stderr, "[paraplan] round gpu us: %.1f\n", 1e3 * ms);
  h->timing.kernel_ms += ms;
  h->timing.launches += (shape.refill ? 2 : 1) + (rerank && (!sharded || packed) ? 1 : 0) +
                        (keys_only ? 1 : 0) + 1;
  h->timing.samples += count * rc;
  h->timing.executed_steps += static_cast<int64_t>(ex[2]);
  // the next round's flush rule, from this round's mean rollout length
  // (measured on B200: rollouts of ~9 steps (C5 H=10) flush best every 2
  // iterations, ~11-13 steps (C2, C5 H >= 30) every 3, ~20 and more (C4)
  // once 6 lanes wait, else every 6)
  if (count * rc > 0 && ex[2] > 0) {
    const double mean = static_cast<double>(ex[2]) / static_cast<double>(count * rc);
    h->flush_every = mean <= 10.0 ? 2 : (mean <= 16.0 ? 3 : 6);
    h->flush_min = mean <= 16.0 ? 0 : 6;
  }
  h->timing.checked_states += static_cast<int64_t>(ex[3]);
  h->timing.rollout_ms += 1e-6 * static_cast<double>(ex[6]);
  const ppdev::Rec* recs = reinterpret_cast<const ppdev::Rec*>(hres + kRecOff);
  bool reached = false;
  for (int r = 0; r < rc; ++r) reached = reached || recs[r].cls == 2;
  if (per_sample == nullptr) h->expect_reach = reached;
  for (int r = 0; r < rc; ++r) {
    out[r].cls = recs[r].cls;
    out[r].candidate = recs[r].cand;
    out[r].restart = r0 + r;
    out[r].iter = iter;
    out[r].k1 = recs[r].k1;
    out[r].k2 = recs[r].k2;
  }
  if (!rerank) return;

  phase("outs");
  n_sel = reinterpret_cast<const uint32_t*>(hres)[2];
  const auto c_t0 = std::chrono::steady_clock::now();
  certify_round(h, a, t, iter, r0, rc, center, c0, c1, injected, out, fp64, n_sel,
                sharded ? (packed ? 1 : 2) : 0);
  phase("certified");
  h->timing.certify_ms +=
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - c_t0).count();
}

// FP64 re-evaluation of the n window members listed in h->d_reflist (flat
// indices of the round `a`, rc restarts of `count` candidates, candidates
// starting at c0): a list round of the FP64 generator + refill rollout (the
// FP64 round's own kernels and per-candidate cost, at full occupancy, with the
// goal-horizon cut per source restart), keys only, then the device filter
// (launch_list_filter) keeps each restart's FP64 near-ties (within 2 x their
// tolerance) and the FP64-flagged members. Only those come back: list[i] the
// member, dev[i] its FP64 key, mstep[i] the earliest state whose FP64 verdict
// came within the FP64 band of flipping (ppdev::kNoStep: none), mpath[i] the
// path up to there. Returns the list round's cut per restart (kCutNone: none).
std::vector<uint32_t> eval_list_fp64(pp_handle* h, const ppdev::RoundArgs& a, int64_t n,
                                     int64_t count, int64_t c0, int rc,
                                     std::vector<int64_t>& list,
                                     std::vector<ppdev::SelRec>& dev,
                                     std::vector<uint32_t>& mstep, std::vector<float>& mpath) {
  ppdev::RoundArgs L = a;
  L.list = static_cast<const int64_t*>(h->d_reflist.p);
  L.list_count = count;
  L.count = n;
  L.restart_count = 1;
  L.cand_begin = c0;
  L.field = ensure_field64(h);
  L.field64 = L.field;
  L.lay = L.lay64;
  L.field_smem_bytes = 0;
  L.per_sample = nullptr;
  L.keys_only = 1;
  L.out_free = nullptr;
  L.sel_packed = 0;
  L.pkeys = nullptr;
  L.skey32 = 0;
  char* dres = static_cast<char*>(h->d_round.p);
  // the list round is one slot: cut only lists from a round of one restart
  L.goal_cut = rc == 1 && !h->no_cut && goal_cut_enabled()
                   ? reinterpret_cast<uint32_t*>(dres + kCutOff)
                   : nullptr;
  L.cut_pub = reinterpret_cast<uint32_t*>(dres + kListCutOff);
  L.cut_slack = cut_slack();
  L.cut_slots = 1;
  // sized to the selection capacity: a closed loop's windows grow tick by tick
  const size_t cap = std::max<size_t>(n, h->sel_cap);
  h->d_listkeys.reserve(sizeof(ppdev::SKey) * cap, "list keys");
  h->d_listout.reserve(sizeof(ppdev::Rec) * 2, "list winner");
  L.skeys = h->d_listkeys.p;
  L.out = static_cast<ppdev::Rec*>(h->d_listout.p);
  const ppdev::LaunchShape s0 = launch_shape(h, true, 0, 0);
  h->d_theta.reserve(static_cast<size_t>(n) * s0.theta_elem * sizeof(double), "theta buffer");
  L.theta_buf = h->d_theta.p;
  const ppdev::LaunchShape shape =
      launch_shape(h, true, 0, ppdev::grid_kind(L.grid_mode, 0, L.field_ns, L.field_nd));
  const int64_t tiles = (n + 31) / 32;
  L.tiles_per_restart = static_cast<int32_t>(tiles);
  L.n_tiles = static_cast<int32_t>(tiles);
  L.block = shape.block;
  L.grid = std::max(1, std::min(shape.grid, static_cast<int>((tiles + ppdev_warps() - 1) /
                                                             ppdev_warps())));
  // the FP64 margin flags as an FP64 round's (narrow misses too: a member
  // must never look robust when its exact class could differ)
  L.kd.flag_miss = 1;
  ck(static_cast<cudaError_t>(ppdev::launch_generate_f64(h->kind, L, h->stream)),
     "list generator launch");
  ck(static_cast<cudaError_t>(ppdev::launch_rollout_f64(h->kind, L, h->stream)),
     "list rollout launch");
  // the filter: scratch [rank u32 x 64][cost u64 x 64], then the picks
  constexpr size_t kScratch = 1024;  // as the prewarm's reservation (capi.cpp)
  h->d_listpick.reserve(kScratch + sizeof(ppdev::ListPick) * cap, "list picks");
  char* dp = static_cast<char*>(h->d_listpick.p);
  ck(cudaMemsetAsync(dp, 0xff, kScratch, h->stream), "list filter scratch");
  ck(cudaMemsetAsync(dres + kListCountOff, 0, sizeof(uint32_t), h->stream), "list filter count");
  ppdev::ListFilterArgs f{};
  f.keys = static_cast<const ppdev::SKey*>(h->d_listkeys.p);
  f.list = L.list;
  f.n = n;
  f.list_count = count;
  f.rho = rho64(h->cfg.H);
  f.rho2 = kRho64Reached;
  f.rho2_floor = kRho64ReachedFloor;
  f.rank = reinterpret_cast<uint32_t*>(dp);
  f.cost = reinterpret_cast<unsigned long long*>(dp + 256);
  f.count = reinterpret_cast<uint32_t*>(dres + kListCountOff);
  f.out = reinterpret_cast<ppdev::ListPick*>(dp + kScratch);
  f.sms = h->sms;
  ck(static_cast<cudaError_t>(ppdev::launch_list_filter(f, h->stream)), "list filter launch");
  char* hres = static_cast<char*>(h->h_round.p);
  ck(cudaMemcpyAsync(hres + kListCutOff, dres + kListCutOff, kListTailBytes,
                     cudaMemcpyDeviceToHost, h->stream),
     "list cut D2H");
  ck(cudaStreamSynchronize(h->stream), "list round");
  h->timing.launches += 6;
  const uint32_t m = *reinterpret_cast<const uint32_t*>(hres + kListCountOff);
  std::vector<uint32_t> cut(rc, ppdev::kCutNone);
  if (L.goal_cut != nullptr) {
    std::memcpy(cut.data(), hres + kListCutOff, sizeof(uint32_t) * rc);
  }
  h->h_listkeys.reserve(sizeof(ppdev::ListPick) * std::max<size_t>(m, 1), "pinned list picks");
  const ppdev::ListPick* picks = static_cast<const ppdev::ListPick*>(h->h_listkeys.p);
  if (m > 0) {
    ck(cudaMemcpyAsync(h->h_listkeys.p, f.out, sizeof(ppdev::ListPick) * m,
                       cudaMemcpyDeviceToHost, h->stream),
       "list picks D2H");
    ck(cudaStreamSynchronize(h->stream), "list picks");
  }
  phase("list-gpu");
  list.resize(m);
  dev.resize(m);
  mstep.resize(m);
  mpath.resize(m);
  for (uint32_t i = 0; i < m; ++i) {
    const ppdev::SKey& k = picks[i].key;
    ppdev::SelRec& d = dev[i];
    list[i] = picks[i].flat;
    d.cls = ppdev::meta_cls(k.meta);
    const int tg = ppdev::meta_tgoal(k.meta);
    d.k1 = d.cls == 2 ? -static_cast<double>(tg) : -k.cost;
    d.k2 = d.cls == 2 ? -k.cost : 0.0;
    mstep[i] = ppdev::meta_mstep(k.meta);
    mpath[i] = ppdev::bits_float(k.mpath);
  }
  return cut;
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
//
// Sharded (shard_mode != 0): every shard selects its own candidates against
// the same bounds, evaluates them, and the shards all-gather their exact
// per-restart bests after each pass (XBest), so every shard takes the same
// decision and returns the same winner -- the global exact best, ties to the
// lowest index as the reference's ordered merge (src/planner.cpp:310-321).

namespace {

// One shard's exact best of a restart in a certification pass.
struct XBest {
  int32_t cls, t_goal;  // cls -1: no window member
  double cost, k1, k2;
  int64_t cand;       // candidate index within the restart
  int32_t overflow;   // the shard's window overflowed this pass
  uint32_t cut;       // the shard's goal-horizon cut of the restart (kCutNone: none)
};

}  // namespace

void certify_round(pp_handle* h, ppdev::RoundArgs& a, uint64_t t, int iter, int r0, int rc,
                   const double* center, int64_t c0, int64_t c1, const double* injected,
                   pp_record* out, bool fp64, uint32_t n_sel, int shard_mode) {
  const int64_t count = c1 - c0;
  const pp_snapshot& snap = *h->snapshot;
  Exchange* xg = shard_mode != 0 ? h->xchg.get() : nullptr;
  std::vector<double> ctr(h->P, 0.0);
  if (center != nullptr) ctr.assign(center, center + h->P);
  phase("cert-enter");
  struct Exact {
    int cls;
    int t_goal;
    double cost;  // terminal cost (cls 0/1) or path length (cls 2)
    double k1, k2;
    int slot;  // its recorded trajectory in h->cert_traj, or -1
  };
  // Trajectories of the window members are recorded for the epilogue while
  // they fit a small arena (2 MB: C2's 43 members x 31 states; up to 326
  // members at H=200); wider windows keep only their keys and the epilogue
  // re-simulates its winner.
  const size_t stride = static_cast<size_t>(h->cfg.H + 1) * 4;
  constexpr size_t kTrajArena = size_t{1} << 18;  // doubles (2 MB)
  int slots = 0;
  auto take_slots = [&](size_t n) {
    if (injected != nullptr || (slots + n) * stride > kTrajArena) return -1;
    const int base = slots;
    slots += static_cast<int>(n);
    if (h->cert_stats.size() < static_cast<size_t>(slots)) {
      h->cert_traj.resize(std::max(h->cert_traj.size(), slots * stride));
      h->cert_stats.resize(slots);
      h->cert_len.resize(slots);
    }
    return base;
  };
  // exact keys of every candidate evaluated so far, by increasing flat
  // index (restart-major): a restart's entries are one contiguous range
  std::vector<std::pair<int64_t, Exact>> known;
  const auto by_index = [](const std::pair<int64_t, Exact>& kv, int64_t s) { return kv.first < s; };
  auto exact_of = [&](int64_t s, int slot) {  // the reference's own FP64 arithmetic
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
    if (slot >= 0) {
      host_rollout(h, snap, theta.data(), &st, h->cert_traj.data() + slot * stride, h->cfg.H + 1,
                   &h->cert_len[slot]);
      h->cert_stats[slot] = st;
    } else {
      host_rollout(h, snap, theta.data(), &st, nullptr, 0, nullptr);
    }
    Exact e;
    e.slot = slot;
    e.cls = st.collided ? 0 : (st.reached ? 2 : 1);
    e.t_goal = st.t_goal;
    e.cost = e.cls == 2 ? st.path_length : st.terminal_cost;
    e.k1 = e.cls == 2 ? -static_cast<double>(st.t_goal) : -st.terminal_cost;
    e.k2 = e.cls == 2 ? -st.path_length : 0.0;
    return e;
  };
  if (h->pool == nullptr) h->pool = shared_pool().pool.get();
  phase("cert-setup");
  // Every rollout starts from the same state 0, so the checks at state 0
  // (collision with field row 0, then the goal box; src/planner.cpp:137-152)
  // do not depend on theta. If they stop the rollout there, every candidate
  // of the round has the same exact key, and each restart's winner is its
  // lowest index (strict-better scans, :295, :316) -- candidate 0 of a
  // sharded round, whose shard 0 starts there. The window would hold the
  // whole round (equal keys), so the round is certified directly (the same
  // decision on every shard, no exchange).
  {
    pp_rollout_stats st{};
    if (host_stops_at_state0(h, snap, &st)) {
      const int cls = st.collided ? 0 : (st.reached ? 2 : 1);
      const double k1 = cls == 2 ? -static_cast<double>(st.t_goal) : -st.terminal_cost;
      const double k2 = cls == 2 ? -st.path_length : 0.0;
      for (int r = 0; r < rc; ++r) {
        out[r].cls = cls;
        out[r].candidate = xg != nullptr ? 0 : static_cast<int>(c0);
        out[r].k1 = k1;
        out[r].k2 = k2;
      }
      if (trace_on()) {
        std::fprintf(stderr, "[paraplan] t=%llu iter=%d: every rollout stops at state 0\n",
                     static_cast<unsigned long long>(t), iter);
      }
      return;
    }
  }
  phase("state0");
  const double alpha = a.sel_alpha;
  const auto rho_of = [&](int cls, int t_goal) {
    return cls != 2 ? a.sel_rho
                    : (a.rho2_by_tgoal ? ppdev::rho2_of(a.sel_rho2, a.sel_rho2_floor, t_goal)
                                       : a.sel_rho2);
  };
  const char* hres = static_cast<const char*>(h->h_round.p);
  const uint32_t* cut_pub = reinterpret_cast<const uint32_t*>(hres + kCutPubOff);
  std::vector<ppdev::SelBound> bound(rc);
  auto set_bound = [&](int r, int cls, int t_goal, double cost) {
    bound[r].cls = cls;
    bound[r].t_goal = cls == 2 ? t_goal : 0;
    bound[r].thr = cost * (1.0 + rho_of(cls, t_goal)) + alpha;  // as select_kernel
  };
  if (shard_mode == 1) {
    // the packed global winners the select kernel anchored on (keypack.h)
    const uint64_t* pk = reinterpret_cast<const uint64_t*>(hres + kPackOff);
    for (int r = 0; r < rc; ++r) {
      const uint64_t pf = pk[rc + r];
      const ppdev::Unpacked u = ppdev::unpack_key(pf != ppdev::kPackEmpty ? pf : pk[r]);
      set_bound(r, u.cls, u.t_goal, static_cast<double>(u.cost));
    }
  } else {
    // the first window is built around each restart's best unflagged
    // candidate when the round reports it (keys_only), else its winner
    const ppdev::Rec* free_recs =
        a.out_free != nullptr ? reinterpret_cast<const ppdev::Rec*>(hres + kFreeOff) : nullptr;
    std::vector<XBest> mine(rc), all;
    for (int r = 0; r < rc; ++r) {
      pp_record o = out[r];
      if (free_recs != nullptr && free_recs[r].cls >= 0) {
        o.cls = free_recs[r].cls;
        o.k1 = free_recs[r].k1;
        o.k2 = free_recs[r].k2;
        o.candidate = free_recs[r].cand;
      }
      mine[r] = XBest{o.cls, o.cls == 2 ? static_cast<int>(-o.k1) : 0,
                      o.cls == 2 ? -o.k2 : -o.k1, o.k1, o.k2, o.candidate, 0, 0};
    }
    if (shard_mode == 2) {  // the global anchors through a host exchange
      all.resize(static_cast<size_t>(rc) * xg->world);
      xg->allgather(mine.data(), all.data(), sizeof(XBest) * rc, h->stream);
      for (int r = 0; r < rc; ++r) {
        XBest g = all[r];
        for (int w = 1; w < xg->world; ++w) {
          const XBest& q = all[static_cast<size_t>(w) * rc + r];
          if (q.cls < 0) continue;
          if (g.cls < 0 || key_better({q.cls, q.k1, q.k2}, {g.cls, g.k1, g.k2})) g = q;
        }
        mine[r] = g;
      }
    }
    for (int r = 0; r < rc; ++r) set_bound(r, mine[r].cls, mine[r].t_goal, mine[r].cost);
  }
  // an FP32 planner's FP64 round: would FP32 have done (class 2 anchors)?
  if (fp64 && !h->fp64) {
    bool terminal = false;
    for (int r = 0; r < rc; ++r) terminal = terminal || (bound[r].cls >= 0 && bound[r].cls < 2);
    h->prefer_fp64 = terminal;
  }
  // outside the FP32 envelope (class 0/1 anchors beyond fp32_max_h): the
  // round is redone in FP64 (every shard decides alike: global anchors)
  if (!fp64 && h->cfg.H > fp32_max_h()) {
    bool terminal = false;
    for (int r = 0; r < rc; ++r) terminal = terminal || (bound[r].cls >= 0 && bound[r].cls < 2);
    if (terminal) {
      if (trace_on()) {
        std::fprintf(stderr, "[paraplan] t=%llu iter=%d: class 0/1 at H=%d: FP64 round\n",
                     static_cast<unsigned long long>(t), iter, h->cfg.H);
      }
      h->timing.fp64_rounds += 1;
      h->prefer_fp64 = true;
      run_round_launch(h, t, iter, r0, rc, center, c0, c1, injected, out, nullptr, true);
      return;
    }
  }
  phase("bounds");
  std::vector<char> certified(rc, 0);
  // per restart: the earliest cut of the round and of its list rounds
  std::vector<uint32_t> cut_eff(rc, ppdev::kCutNone);
  if (a.goal_cut != nullptr) std::copy(cut_pub, cut_pub + rc, cut_eff.begin());
  std::vector<int64_t> list;
  std::vector<XBest> xmine(rc), xall;
  bool widened = shard_mode == 2;  // no select ran yet
  constexpr int kPasses = 6;
  for (int pass = 0; pass < kPasses; ++pass) {
    auto reselect = [&] {  // the select kernel with the current bounds
      if (a.sel_bound != nullptr || pass > 0 || widened) {
        h->d_bound.reserve(sizeof(ppdev::SelBound) * rc, "window bounds");
        h->h_bound.reserve(sizeof(ppdev::SelBound) * rc, "pinned bounds");
        std::memcpy(h->h_bound.p, bound.data(), sizeof(ppdev::SelBound) * rc);
        ck(cudaMemcpyAsync(h->d_bound.p, h->h_bound.p, sizeof(ppdev::SelBound) * rc,
                           cudaMemcpyHostToDevice, h->stream),
           "bounds H2D");
        a.sel_bound = static_cast<const ppdev::SelBound*>(h->d_bound.p);
      }
      ck(cudaMemsetAsync(a.counters + 2, 0, sizeof(uint32_t), h->stream), "selection counter");
      ck(static_cast<cudaError_t>(ppdev::launch_select(a, h->stream)), "window select launch");
      ck(cudaMemcpyAsync(h->h_round.p, h->d_round.p, kSelOff + sizeof(int64_t) * kSelFirst,
                         cudaMemcpyDeviceToHost, h->stream),
         "selection D2H");
      ck(cudaStreamSynchronize(h->stream), "window select");
      h->timing.launches += 1;
      n_sel = static_cast<const uint32_t*>(h->h_round.p)[2];
      widened = false;
    };
    if (pass > 0 || widened) reselect();  // (widened) window of the uncertified restarts
    // a window wider than the selection buffers: grow them, select again
    while (n_sel > static_cast<uint32_t>(h->sel_cap) && n_sel <= static_cast<uint32_t>(kSelMax)) {
      if (trace_on()) {
        std::fprintf(stderr, "[paraplan] t=%llu iter=%d pass=%d selected=%u: selection grows\n",
                     static_cast<unsigned long long>(t), iter, pass, n_sel);
      }
      grow_selection(h, a, static_cast<int>(std::min<uint32_t>(
                               static_cast<uint32_t>(kSelMax), n_sel + n_sel / 4)));
      reselect();
    }
    const bool overflow = n_sel > static_cast<uint32_t>(h->sel_cap);
    if (overflow && trace_on()) {
      std::fprintf(stderr, "[paraplan] t=%llu iter=%d pass=%d selected=%u: window overflow\n",
                   static_cast<unsigned long long>(t), iter, pass, n_sel);
    }
    list.clear();
    // a wide first-pass window stays on the device: the FP64 list round reads
    // the selection in place and only the members the host must see return
    const bool refill64 = launch_shape(h, true, 0, 0).refill != 0;
    const bool dev_list =
        !overflow && known.empty() && refill64 && n_sel > static_cast<uint32_t>(host_max());
    if (!overflow && !dev_list) {
      std::vector<int64_t> sl(n_sel);
      std::memcpy(sl.data(), static_cast<const char*>(h->h_round.p) + kSelOff,
                  sizeof(int64_t) * std::min<uint32_t>(n_sel, kSelFirst));
      if (n_sel > static_cast<uint32_t>(kSelFirst)) {
        ck(cudaMemcpy(sl.data() + kSelFirst, a.sel_more, sizeof(int64_t) * (n_sel - kSelFirst),
                      cudaMemcpyDeviceToHost),
           "selection D2H");
      }
      list.reserve(n_sel);
      for (uint32_t i = 0; i < n_sel; ++i) {
        if (known.empty()) {
          list.push_back(sl[i]);
          continue;
        }
        const auto it = std::lower_bound(known.begin(), known.end(), sl[i], by_index);
        if (it == known.end() || it->first != sl[i]) list.push_back(sl[i]);
      }
      // the device appends in no particular order; a wide window is ordered
      // after its FP64 pass, on the members it keeps
      if (list.size() <= static_cast<size_t>(host_max())) std::sort(list.begin(), list.end());
    }
    const size_t n_new = dev_list ? n_sel : list.size();
    h->timing.refined += static_cast<int32_t>(n_new);
    phase("list");
    if (trace_level() >= 3 && !list.empty() && !fp64) {  // window composition
      std::vector<ppdev::SKey32> ks(list.size());
      for (size_t i = 0; i < list.size(); ++i) {
        ck(cudaMemcpy(&ks[i], static_cast<const ppdev::SKey32*>(a.skeys) + list[i],
                      sizeof(ppdev::SKey32), cudaMemcpyDeviceToHost),
           "trace D2H");
        if (i >= 20000) break;
      }
      const size_t m = std::min<size_t>(list.size(), 20001);
      size_t flagged = 0, incost = 0, ms_hist[4] = {0, 0, 0, 0};
      for (size_t i = 0; i < m; ++i) {
        const int r = static_cast<int>(list[i] / count);
        const uint32_t ms = ppdev::meta_mstep(ks[i].meta);
        if (ms != ppdev::kNoStep) {
          ++flagged;
          ms_hist[std::min<uint32_t>(ms, 3)]++;
        }
        if (ppdev::meta_cls(ks[i].meta) == bound[r].cls && ks[i].cost <= bound[r].thr) ++incost;
      }
      std::fprintf(stderr,
                   "[paraplan]   window %zu (sampled %zu): anchor cls %d t_goal %d thr %.9g; "
                   "flagged %zu (mstep 0/1/2/3+: %zu %zu %zu %zu), within thr %zu\n",
                   list.size(), m, bound[0].cls, bound[0].t_goal, bound[0].thr, flagged, ms_hist[0],
                   ms_hist[1], ms_hist[2], ms_hist[3], incost);
    }
    std::vector<Exact> got;
    if (!dev_list && list.size() <= static_cast<size_t>(host_max())) {
      got.resize(list.size());
      const int base = take_slots(list.size());
      std::lock_guard<std::mutex> turn(shared_pool().mu);
      h->pool->run(static_cast<int>(list.size()), [&](int i) {
        got[i] = exact_of(list[i], base < 0 ? -1 : base + i);
      });
    } else {
      // wide window: FP64 keys from the device, exact host keys for the FP64
      // near-ties of each restart's best and the FP64-flagged members
      if (dev_list) {  // the selection, in place: round block head + sel_more
        const char* dsel = static_cast<const char*>(h->d_round.p) + kSelOff;
        const size_t head = std::min<uint32_t>(n_sel, kSelFirst);
        ck(cudaMemcpyAsync(h->d_reflist.p, dsel, sizeof(int64_t) * head,
                           cudaMemcpyDeviceToDevice, h->stream),
           "refine list D2D");
        if (n_sel > static_cast<uint32_t>(kSelFirst)) {
          ck(cudaMemcpyAsync(static_cast<int64_t*>(h->d_reflist.p) + kSelFirst, a.sel_more,
                             sizeof(int64_t) * (n_sel - kSelFirst), cudaMemcpyDeviceToDevice,
                             h->stream),
             "refine list D2D");
        }
      } else {
        ck(cudaMemcpyAsync(h->d_reflist.p, list.data(), sizeof(int64_t) * list.size(),
                           cudaMemcpyHostToDevice, h->stream),
           "refine list H2D");
      }
      std::vector<ppdev::SelRec> dev;
      std::vector<uint32_t> mstep;
      std::vector<float> mpath;
      if (refill64) {
        const size_t n_listed = n_new;
        const std::vector<uint32_t> lcut =
            eval_list_fp64(h, a, static_cast<int64_t>(n_listed), count, c0, rc, list, dev, mstep,
                           mpath);
        for (int r = 0; r < rc; ++r) cut_eff[r] = std::min(cut_eff[r], lcut[r]);
        for (size_t i = 0; i < list.size(); ++i) {
          dev[i].restart = static_cast<int32_t>(list[i] / count);
          dev[i].cand = static_cast<int32_t>(c0 + (list[i] - dev[i].restart * count));
        }
        if (trace_on()) {
          std::fprintf(stderr, "[paraplan]   wide window %zu: %zu picked on the device\n", n_listed,
                       list.size());
        }
      } else {  // generic architectures: one lockstep FP64 rollout per lane
        dev.resize(list.size());
        mstep.assign(list.size(), ppdev::kNoStep);
        mpath.assign(list.size(), 0.0f);
        const uint32_t n_list = static_cast<uint32_t>(list.size());
        ck(cudaMemcpyAsync(a.counters + 2, &n_list, sizeof(uint32_t), cudaMemcpyHostToDevice,
                           h->stream),
           "refine count H2D");
        a.field64 = ensure_field64(h);
        ck(static_cast<cudaError_t>(ppdev::launch_refine(h->kind, a, h->stream)),
           "refine launch");
        ck(cudaMemcpyAsync(dev.data(), a.sel_out, sizeof(ppdev::SelRec) * list.size(),
                           cudaMemcpyDeviceToHost, h->stream),
           "refine D2H");
        ck(cudaStreamSynchronize(h->stream), "refine kernel");
        h->timing.launches += 1;
      }
      got.resize(list.size());
      phase("refine64");
      std::vector<int> best(rc, -1);
      for (size_t i = 0; i < dev.size(); ++i) {
        got[i] = Exact{dev[i].cls, dev[i].cls == 2 ? static_cast<int>(-dev[i].k1) : -1,
                       dev[i].cls == 2 ? -dev[i].k2 : -dev[i].k1, dev[i].k1, dev[i].k2, -1};
        const int r = dev[i].restart;
        if (best[r] < 0 || key_better({got[i].cls, got[i].k1, got[i].k2},
                                      {got[best[r]].cls, got[best[r]].k1, got[best[r]].k2}) ||
            (!key_better({got[best[r]].cls, got[best[r]].k1, got[best[r]].k2},
                         {got[i].cls, got[i].k1, got[i].k2}) &&
             list[i] < list[best[r]])) {
          best[r] = static_cast<int>(i);
        }
      }
      // The members to evaluate exactly: the FP64 near-ties of each
      // restart's best, and every member whose FP64 verdict came within the
      // FP64 margin of flipping (it may rise a class). The rest are worse
      // than the best by more than two FP64 error bounds, so exactly worse
      // too, and are dropped. Near-ties whose FP64 keys are bitwise equal
      // (e.g. rollouts whose steering saturates identically: the same
      // trajectory) are one group: its lowest index is evaluated and the
      // others, identical rollouts that lose the index tie-break, dropped.
      // Flagged members group the same way, by key and flagged state.
      phase("best");
      std::vector<int> keep;
      {
        struct GroupKey {
          int r, cls;
          double k1, k2;
          uint32_t ms;
          bool operator<(const GroupKey& o) const {
            if (r != o.r) return r < o.r;
            if (cls != o.cls) return cls < o.cls;
            if (k1 != o.k1) return k1 < o.k1;
            return k2 < o.k2;
          }
        };
        struct GroupHash {
          size_t operator()(const GroupKey& g) const {
            uint64_t a, b;
            std::memcpy(&a, &g.k1, 8);
            std::memcpy(&b, &g.k2, 8);
            return std::hash<uint64_t>()(a * 0x9E3779B97F4A7C15ull ^ b ^
                                         (static_cast<uint64_t>(g.r) << 20 | g.ms << 2 | g.cls));
          }
        };
        struct GroupEq {
          bool operator()(const GroupKey& x, const GroupKey& y) const {
            return x.r == y.r && x.cls == y.cls && x.k1 == y.k1 && x.k2 == y.k2 && x.ms == y.ms;
          }
        };
        // -> member of the lowest index
        std::unordered_map<GroupKey, int, GroupHash, GroupEq> groups;
        for (size_t i = 0; i < dev.size(); ++i) {
          const Exact& b = got[best[dev[i].restart]];
          const double tol =
              b.cls == 2 ? ppdev::rho2_of(kRho64Reached, kRho64ReachedFloor, b.t_goal)
                         : rho64(h->cfg.H);
          const bool flag = mstep[i] != ppdev::kNoStep;
          if (flag || (got[i].cls == b.cls &&
                       std::abs(got[i].k1 - b.k1) <= tol * std::max(1.0, std::abs(b.k1)) &&
                       std::abs(got[i].k2 - b.k2) <= tol * std::max(1.0, std::abs(b.k2)))) {
            const GroupKey g{dev[i].restart, got[i].cls, got[i].k1, got[i].k2,
                             flag ? mstep[i] : ppdev::kNoStep};
            auto it = groups.find(g);
            if (it == groups.end()) {
              groups.emplace(g, static_cast<int>(i));
            } else if (list[i] < list[it->second]) {
              it->second = static_cast<int>(i);
            }
          }
        }
        for (const auto& kv : groups) keep.push_back(kv.second);
        std::sort(keep.begin(), keep.end(), [&](int x, int y) { return list[x] < list[y]; });
        keep.erase(std::unique(keep.begin(), keep.end()), keep.end());
      }
      // Phase A: the near-tie groups, exactly; their exact best per restart.
      // Phase B: a flagged member is evaluated only if its most optimistic
      // exact key could still beat (or tie) that best: a flip at its flagged
      // state reaches there with the path so far (mpath, a lower bound; the
      // path only grows), or its own FP64 key within the FP64 tolerance.
      phase("groups");
      std::vector<int> ka, kb;
      for (int i : keep) (mstep[i] == ppdev::kNoStep ? ka : kb).push_back(i);
      const auto eval_exact = [&](const std::vector<int>& idx, std::vector<Exact>& out) {
        out.resize(idx.size());
        const int base = take_slots(idx.size());
        std::lock_guard<std::mutex> turn(shared_pool().mu);
        h->pool->run(static_cast<int>(idx.size()), [&](int j) {
          out[j] = exact_of(list[idx[j]], base < 0 ? -1 : base + j);
        });
      };
      std::vector<Exact> got_a, got_b;
      eval_exact(ka, got_a);
      phase("exactA");
      std::vector<int> estar(rc, -1);  // per restart: best of phase A (index into ka)
      for (size_t j = 0; j < ka.size(); ++j) {
        const int r = dev[ka[j]].restart;
        const Exact& q = got_a[j];
        if (estar[r] < 0 || key_better({q.cls, q.k1, q.k2},
                                       {got_a[estar[r]].cls, got_a[estar[r]].k1,
                                        got_a[estar[r]].k2})) {
          estar[r] = static_cast<int>(j);
        }
      }
      std::vector<int> kb_eval;
      for (int i : kb) {
        const int r = dev[i].restart;
        if (estar[r] < 0) {
          kb_eval.push_back(i);
          continue;
        }
        const double tol = got[i].cls == 2
                               ? ppdev::rho2_of(kRho64Reached, kRho64ReachedFloor, got[i].t_goal)
                               : rho64(h->cfg.H);
        const Key flip{2, -static_cast<double>(mstep[i]),
                       -static_cast<double>(mpath[i]) * (1.0 - 1e-12)};
        const Key own = got[i].cls == 2 ? Key{2, got[i].k1, -got[i].cost * (1.0 - tol)}
                                        : Key{got[i].cls, -got[i].cost * (1.0 - tol), 0.0};
        const Key opt = key_better(flip, own) ? flip : own;
        const Exact& e = got_a[estar[r]];
        if (!key_better({e.cls, e.k1, e.k2}, opt)) kb_eval.push_back(i);
      }
      eval_exact(kb_eval, got_b);
      std::vector<std::pair<int64_t, Exact>> kept;
      kept.reserve(ka.size() + kb_eval.size());
      for (size_t j = 0; j < ka.size(); ++j) kept.emplace_back(list[ka[j]], got_a[j]);
      for (size_t j = 0; j < kb_eval.size(); ++j) kept.emplace_back(list[kb_eval[j]], got_b[j]);
      std::sort(kept.begin(), kept.end(),
                [](const auto& x, const auto& y) { return x.first < y.first; });
      std::vector<int64_t> kept_list(kept.size());
      std::vector<Exact> kept_got(kept.size());
      for (size_t j = 0; j < kept.size(); ++j) {
        kept_list[j] = kept[j].first;
        kept_got[j] = kept[j].second;
      }
      if (trace_on()) {
        std::fprintf(stderr, "[paraplan]   wide window %zu: %zu near-tie groups and %zu of %zu "
                             "FP64-flagged members to the host (best cls %d t_goal %d)\n",
                     list.size(), ka.size(), kb_eval.size(), kb.size(),
                     best.empty() ? -1 : got[best[0]].cls, best.empty() ? -1 : got[best[0]].t_goal);
      }
      list.swap(kept_list);
      got.swap(kept_got);
    }
    phase("exact");
    {  // merge the (sorted, new) list into the known keys
      std::vector<std::pair<int64_t, Exact>> merged;
      merged.reserve(known.size() + list.size());
      size_t k = 0;
      for (size_t i = 0; i < list.size(); ++i) {
        while (k < known.size() && known[k].first < list[i]) merged.push_back(known[k++]);
        merged.emplace_back(list[i], got[i]);
      }
      while (k < known.size()) merged.push_back(known[k++]);
      known.swap(merged);
    }

    // each uncertified restart's exact best (this shard's, then the global)
    std::vector<const Exact*> local(rc, nullptr);
    std::vector<int64_t> local_win(rc, -1);
    for (int r = 0; r < rc; ++r) {
      if (certified[r]) continue;
      // increasing index order: among equal keys the first (lowest) wins
      const auto hi = std::lower_bound(known.begin(), known.end(), (r + 1) * count, by_index);
      for (auto it = std::lower_bound(known.begin(), known.end(), r * count, by_index); it != hi;
           ++it) {
        const Exact& q = it->second;
        if (local[r] == nullptr ||
            key_better({q.cls, q.k1, q.k2}, {local[r]->cls, local[r]->k1, local[r]->k2})) {
          local[r] = &q;
          local_win[r] = it->first;
        }
      }
    }
    for (int r = 0; r < rc; ++r) {
      const Exact* e = local[r];
      const uint32_t cut = cut_eff[r];
      xmine[r] = e == nullptr
                     ? XBest{-1, 0, 0.0, 0.0, 0.0, -1, overflow ? 1 : 0, cut}
                     : XBest{e->cls, e->t_goal, e->cost, e->k1, e->k2,
                             c0 + (local_win[r] - r * count), overflow ? 1 : 0, cut};
    }
    bool any_overflow = overflow;
    std::vector<XBest> gbest(xmine);
    if (xg != nullptr) {  // the same decision on every shard
      xall.resize(static_cast<size_t>(rc) * xg->world);
      xg->allgather(xmine.data(), xall.data(), sizeof(XBest) * rc, h->stream);
      for (int r = 0; r < rc; ++r) {
        XBest g{-1, 0, 0.0, 0.0, 0.0, -1, 0, ppdev::kCutNone};
        uint32_t cut = ppdev::kCutNone;
        for (int w = 0; w < xg->world; ++w) {  // shard order = index order
          const XBest& q = xall[static_cast<size_t>(w) * rc + r];
          any_overflow = any_overflow || q.overflow != 0;
          cut = std::min(cut, q.cut);
          if (q.cls < 0) continue;
          if (g.cls < 0 || key_better({q.cls, q.k1, q.k2}, {g.cls, g.k1, g.k2})) g = q;
        }
        g.cut = cut;
        gbest[r] = g;
      }
    }
    if (any_overflow) break;

    // certify or widen each uncertified restart
    bool all = true, cut_broken = false;
    for (int r = 0; r < rc; ++r) {
      if (certified[r]) continue;
      const ppdev::SelBound& bd = bound[r];
      const XBest& e = gbest[r];
      const double rho = rho_of(bd.cls, bd.t_goal);
      const double slack = 0.5 * (rho * bd.thr + alpha);
      bool ok = false;
      if (e.cls >= 0) {
        if (e.cls > bd.cls) {
          ok = true;  // only a flagged (always selected) candidate can rise a class
        } else if (e.cls == bd.cls) {
          ok = (bd.cls == 2 && e.t_goal < bd.t_goal) ||
               ((bd.cls != 2 || e.t_goal == bd.t_goal) && e.cost <= bd.thr - slack);
        }
      }
      // A cut rollout has not reached the goal by its restart's (shard's)
      // earliest t_goal + cut_slack() (device_api.h), so no exact key places
      // it ahead of an exact best that reaches by then -- unless it is
      // flagged at or before the window's t_goal, and then it is in the
      // window. An exact best reaching later (or not at all) has no such
      // guarantee: the round is redone without the cut.
      if (ok && e.cut != ppdev::kCutNone &&
          !(e.cls == 2 && static_cast<int64_t>(e.t_goal) <= int64_t{e.cut} + cut_slack())) {
        cut_broken = true;
        ok = false;
      }
      if (ok) {
        certified[r] = 1;
        out[r].cls = e.cls;
        out[r].candidate = static_cast<int>(e.cand);
        out[r].k1 = e.k1;
        out[r].k2 = e.k2;
        const Exact* le = local[r];
        if (le != nullptr && le->slot >= 0 && c0 + (local_win[r] - r * count) == e.cand) {
          pp_handle::WinnerRollout w;  // the winner is this shard's: keep its rollout
          w.restart = out[r].restart;
          w.iter = out[r].iter;
          w.candidate = out[r].candidate;
          w.stats = h->cert_stats[le->slot];
          w.len = h->cert_len[le->slot];
          const double* tr = h->cert_traj.data() + le->slot * stride;
          w.traj.assign(tr, tr + static_cast<size_t>(std::min<int32_t>(w.len, h->cfg.H + 1)) * 4);
          h->winner_rollouts.push_back(std::move(w));
        }
        bound[r].cls = -1;  // select nothing more for this restart
        continue;
      }
      all = false;
      if (trace_level() >= 2) {
        std::fprintf(stderr,
                     "[paraplan]   restart %d open: window cls %d t_goal %d thr %.9g slack %.3g; "
                     "exact best cls %d t_goal %d cost %.9g\n",
                     r0 + r, bd.cls, bd.t_goal, bd.thr, slack, e.cls, e.t_goal, e.cost);
      }
      const bool same = e.cls >= 0 && e.cls == bd.cls && (bd.cls != 2 || e.t_goal == bd.t_goal);
      const double wider = bd.thr * 1.25 + alpha;
      bound[r].thr = same ? std::max(e.cost * (1.0 + rho) + alpha, wider) : wider;
    }
    if (cut_broken) {
      if (trace_on()) {
        std::fprintf(stderr, "[paraplan] t=%llu iter=%d: the goal cut does not hold, round redone\n",
                     static_cast<unsigned long long>(t), iter);
      }
      h->no_cut = true;
      try {
        run_round_launch(h, t, iter, r0, rc, center, c0, c1, injected, out, nullptr, fp64);
      } catch (...) {
        h->no_cut = false;
        throw;
      }
      h->no_cut = false;
      return;
    }
    if (trace_on()) {
      std::fprintf(stderr, "[paraplan] t=%llu iter=%d pass=%d selected=%u new=%zu certified=%s\n",
                   static_cast<unsigned long long>(t), iter, pass, n_sel, list.size(),
                   all ? "all" : "no");
    }
    if (all) return;
  }
  // overflowed or not certified (on any shard): redo the round in FP64
  if (trace_on()) {
    std::fprintf(stderr, "[paraplan] t=%llu iter=%d: FP64 fallback round\n",
                 static_cast<unsigned long long>(t), iter);
  }
  if (fp64) throw std::runtime_error("near-tie re-ranking could not certify an FP64 round");
  h->timing.refined = -1;
  h->timing.fp64_rounds += 1;
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

}  // namespace ppcapi
