// capi.cpp -- the C-ABI of include/paraplan_cuda.h: construction and
// teardown, snapshots, sampling rounds, the plan step, diagnostics.
//
// Host side of Planner::plan_step (src/planner.cpp:238-351 in the reference):
//   * validation with the reference's messages,
//   * snapshot staging (pinned host -> HBM, one copy per tick),
//   * the restart x iteration schedule: with n_iter_max == 1 every candidate
//     of every restart is independent (each restart re-centres on the warm
//     start, :271-277) and the whole tick is ONE round; iterations >= 1
//     centre on the incumbent and run as dependent rounds,
//   * the ordered, strict-better merge of round winners (:310-330),
//   * the FP64 epilogue (:339-350) on the host, bit-identical to the
//     reference because best_theta is regenerated with the host KeyedRng and
//     re-simulated through the same FP64 primitives.
// Internals: capi_internal.hpp (upload.cpp, round.cpp, host_exact.cpp).
#include "capi_internal.hpp"

using namespace ppcapi;

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
    h->winner_rollouts.clear();  // kept by plan steps only
    run_round(h, 0, 0, 0, rc, nullptr, 0, h->cfg.n_candidates, nullptr, rec.data(), nullptr);
    // the other grid modes, and (FP32 planners) the FP64 kernels of the
    // certification's fallback round
    for (int mode = 0; mode <= 2; ++mode) {
      ppdev::LaunchShape sh{};
      ppdev::shape_f64(h->kind, h->device, 0, mode, &sh);
      if (!h->fp64) ppdev::shape_f32(h->kind, h->device, 0, mode, &sh);
    }
    ppdev::LaunchShape sh{};  // x-buckets staged in shared memory
    if (h->fp64) ppdev::shape_f64(h->kind, h->device, 16, 3, &sh);
    else ppdev::shape_f32(h->kind, h->device, 16, 3, &sh);
    ck(cudaStreamSynchronize(h->stream), "warm-up");
    // An FP32 planner whose certification overflows redoes the round in
    // FP64, with twice the theta record and key sizes. Growing those buffers
    // at that tick cost 0.25-0.8 s on B200 (C3 tick 38), so rounds of up to
    // 2^23 candidates reserve the FP64 sizes here.
    const size_t total = static_cast<size_t>(h->cfg.n_candidates) * std::max(1, rc);
    if (!h->fp64 && h->rerank && total <= (size_t{1} << 23)) {
      const ppdev::LaunchShape s64 = launch_shape(h, true, 0, 0);
      if (s64.refill) h->d_theta.reserve(total * s64.theta_elem * sizeof(double), "theta buffer");
      h->d_skeys.reserve(total * sizeof(ppdev::SKey), "sample keys");
    }
    // selection buffers for a window of the whole round (up to kSelMax): a
    // closed loop's near-goal ticks select most of a round, and growing
    // pinned and device buffers mid-tick cost tens of ms
    if (h->rerank) {
      ppdev::RoundArgs scratch{};
      const int cap = static_cast<int>(std::min<size_t>(total, kSelMax));
      grow_selection(h, scratch, std::max(cap, kSelCap));
      h->d_listkeys.reserve(sizeof(ppdev::SKey) * h->sel_cap, "list keys");
      h->d_listout.reserve(sizeof(ppdev::Rec) * 2, "list winner");
      h->d_listpick.reserve(1024 + sizeof(ppdev::ListPick) * h->sel_cap, "list picks");
      // (the picks of a wide window are its near-ties and flagged members:
      // few; a larger set grows the pinned buffer when it happens)
      h->h_listkeys.reserve(sizeof(ppdev::ListPick) * std::min(h->sel_cap, 1 << 16),
                            "pinned list picks");
      // the filter's kernels load on first use: load them now (an empty list)
      ppdev::ListFilterArgs f{};
      f.list_count = 1;
      f.sms = h->sms;
      ck(static_cast<cudaError_t>(ppdev::launch_list_filter(f, h->stream)), "filter warm-up");
      ck(cudaStreamSynchronize(h->stream), "filter warm-up");
    }
  } catch (...) {
    cudaGetLastError();
  }
  h->snap_valid = false;
  h->snapshot = nullptr;
  h->timing = pp_timing{};
  h->prefer_fp64 = false;  // the warm-up's fake snapshot says nothing about real ticks
  h->expect_reach = true;
  h->flush_every = 3;
  h->flush_min = 0;
}

// The exchange of an in-process sharded planner (PlannerConfig::devices):
// NCCL over the listed GPUs when they are distinct and NCCL loads, else host
// memory (shards sharing a GPU: NCCL refuses duplicate devices).
// PARAPLAN_EXCHANGE=host|nccl forces one (A/B and tests).
void attach_shard_exchanges(pp_handle* h, const pp_model& m) {
  const int S = static_cast<int>(h->shards.size()) + 1;
  std::vector<pp_handle*> all{h};
  all.insert(all.end(), h->shards.begin(), h->shards.end());
  std::vector<int> devs;
  for (pp_handle* g : all) devs.push_back(g->device);
  std::vector<int> sorted(devs);
  std::sort(sorted.begin(), sorted.end());
  const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
  const char* env = std::getenv("PARAPLAN_EXCHANGE");
  const std::string want = env != nullptr ? env : "";
  bool use_nccl = distinct && want != "host" && nccl_available();
  if (want == "nccl" && !use_nccl) {
    std::string why = distinct ? "" : "shards share a device";
    nccl_available(&why);
    throw std::invalid_argument("PARAPLAN_EXCHANGE=nccl: " + why);
  }
  if (use_nccl) {
    auto ex = make_nccl_exchanges(devs.data(), S);
    for (int k = 0; k < S; ++k) all[k]->xchg = std::move(ex[k]);
  } else {
    h->thread_group = std::make_shared<ThreadGroup>(S);
    for (int k = 0; k < S; ++k) all[k]->xchg = make_thread_exchange(h->thread_group, k);
  }
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
    if (hp->cfg.H > ppdev::kMaxKeyHorizon) {  // the 15-bit state fields of the sample keys
      throw std::invalid_argument("the device planner supports horizons H <= 32766");
    }
    hp->chassis = paraplan::ChassisPolytope::rectangle(hp->params);
    hp->box = {hp->params.front_extent(), hp->params.rear_extent(), hp->params.half_width};
    hp->P = hp->policy->param_count();
    hp->kind = ppdev::classify(hp->sizes.data(), static_cast<int32_t>(hp->sizes.size()));
    hp->fp64 = hp->cfg.precision == 64;
    hp->rerank = hp->cfg.refine;
    if (const char* e = std::getenv("PARAPLAN_SEL_RHO")) hp->sel_rho = std::atof(e);
    if (const char* e = std::getenv("PARAPLAN_DMARG")) hp->dmarg32 = std::atof(e);
    hp->device = hp->cfg.device;
    const int n_dev = m->config.n_devices;
    if (n_dev > PP_MAX_DEVICES) throw std::invalid_argument("at most 8 devices per planner");
    if (n_dev > 1) hp->device = m->config.devices[0];

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
    ck(cudaDeviceGetAttribute(&hp->sms, cudaDevAttrMultiProcessorCount, hp->device), "SM count");
    hp->base.sms = hp->sms;
    ck(cudaStreamCreateWithFlags(&hp->stream, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreate(&hp->ev0), "event");
    ck(cudaEventCreate(&hp->ev1), "event");
    ck(cudaStreamCreateWithFlags(&hp->side, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&hp->ev_field, cudaEventDisableTiming), "event");
    hp->d_round.reserve(kRoundAlloc, "round block");
    ck(cudaMemsetAsync(hp->d_round.p, 0, kRoundAlloc, hp->stream), "round block");
    ck(cudaMemsetAsync(static_cast<char*>(hp->d_round.p) + kCutOff, 0xff,
                       sizeof(uint32_t) * ppdev::kMaxRestartsPerLaunch, hp->stream),
       "goal cut");
    hp->h_round.reserve(kRoundAlloc, "pinned round block");
    ck(cudaStreamSynchronize(hp->stream), "init");
    h = hp.release();
  });
  if (st == PP_OK) {
    prewarm(h);
    // the other shards: the same model on devices[1..n) (a shard's error,
    // e.g. a missing device, is the planner's)
    pp_status sst = PP_OK;
    for (int k = 1; k < m->config.n_devices && sst == PP_OK; ++k) {
      pp_model mk = *m;
      mk.config.n_devices = 0;
      mk.config.device = m->config.devices[k];
      pp_handle* g = nullptr;
      sst = pp_create(&mk, &g);
      if (sst == PP_OK) h->shards.push_back(g);
    }
    if (sst == PP_OK && !h->shards.empty()) {
      sst = guarded([&] {
        h->shard_pool = std::make_unique<HostPool>(static_cast<int>(h->shards.size()) + 1);
        attach_shard_exchanges(h, *m);
      });
    }
    if (sst != PP_OK) {
      const std::string msg = pp_last_error();
      pp_destroy(h);
      g_error = msg;
      return sst;
    }
    *out = h;
  }
  return st;
}

void pp_destroy(pp_handle* h) {
  if (h == nullptr) return;
  h->shard_pool.reset();
  for (pp_handle* g : h->shards) pp_destroy(g);
  h->shards.clear();
  cudaSetDevice(h->device);
  if (h->stream != nullptr) cudaStreamSynchronize(h->stream);
  for (DevBuf* b : {&h->d_field, &h->d_params, &h->d_round, &h->d_tiles, &h->d_movers, &h->d_bin,
                    &h->d_samples, &h->d_scratch, &h->d_injected, &h->d_theta, &h->d_skeys,
                    &h->d_sel, &h->d_bound, &h->d_field64, &h->d_selmore, &h->d_reflist,
                    &h->d_listkeys, &h->d_listout, &h->d_listpick}) {
    b->release();
  }
  for (HostBuf* b : {&h->h_field, &h->h_params, &h->h_round, &h->h_bound, &h->h_movers,
                     &h->h_listkeys,
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
    h->winner_rollouts.clear();  // kept by plan steps only
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
    h->winner_rollouts.clear();  // kept by plan steps only
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
  if (h == nullptr) {  // no status out-parameter: NaN marks the invalid handle
    g_error = "null argument";
    return std::nan("");
  }
  paraplan::KeyedRng rng(h->cfg.master_seed, t, static_cast<uint64_t>(restart),
                         static_cast<uint64_t>(iter), static_cast<uint64_t>(candidate));
  return std::pow(10.0, h->cfg.sigma_log_low +
                            rng.next_unit() * (h->cfg.sigma_log_high - h->cfg.sigma_log_low));
}

pp_status pp_draw_theta(pp_handle* h, const double* center, int32_t len, uint64_t t,
                        int32_t restart, int32_t iter, int64_t cand_begin, int64_t cand_end,
                        double* out) {
  return guarded([&] {
    if (h == nullptr || center == nullptr || out == nullptr) {
      throw std::invalid_argument("null argument");
    }
    if (len != h->P) throw std::invalid_argument("candidate buffer size mismatch");
    if (cand_begin < 0 || cand_end < cand_begin || restart < 0 || iter < 0) {
      throw std::invalid_argument("candidate range out of bounds");
    }
    const int64_t n = cand_end - cand_begin;
    if (n == 0) return;
    ck(cudaSetDevice(h->device), "cudaSetDevice");
    ppdev::RoundArgs a{};
    a.sms = h->sms;
    a.sig_lo = h->cfg.sigma_log_low;
    a.sig_span = h->cfg.sigma_log_high - h->cfg.sigma_log_low;
    a.n_params = h->P;
    a.count = n;
    a.restart_count = 1;
    a.cand_begin = cand_begin;
    const uint64_t prefix = key_prefix(h->cfg.master_seed, t, static_cast<uint64_t>(restart),
                                       static_cast<uint64_t>(iter));
    upload_params(h, a, &prefix, 1, center);
    const size_t esz = h->fp64 ? sizeof(double) : sizeof(float);
    const size_t bytes = esz * h->P * static_cast<size_t>(n);
    h->d_samples.reserve(bytes, "theta draws");
    ck(static_cast<cudaError_t>(h->fp64 ? ppdev::launch_draw_f64(a, h->d_samples.p, h->stream)
                                        : ppdev::launch_draw_f32(a, h->d_samples.p, h->stream)),
       "theta draw launch");
    std::vector<unsigned char> host(bytes);
    ck(cudaMemcpyAsync(host.data(), h->d_samples.p, bytes, cudaMemcpyDeviceToHost, h->stream),
       "theta D2H");
    ck(cudaStreamSynchronize(h->stream), "theta draws");
    const size_t m = static_cast<size_t>(h->P) * n;
    if (h->fp64) {
      std::memcpy(out, host.data(), bytes);
    } else {
      const float* f = reinterpret_cast<const float*>(host.data());
      for (size_t i = 0; i < m; ++i) out[i] = static_cast<double>(f[i]);
    }
  });
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

// One sampling round over every shard of the planner. Shard k of S
// evaluates candidates [n k / S, n (k + 1) / S) of each restart, and the
// shards exchange their winners and exact keys (round.cpp certify_round,
// exchange.hpp) so that every shard returns the same, global winner: the
// reference's ordered merge of its worker ranges (src/planner.cpp:280-281,
// 310-321). Shards are either the threads of this process (PlannerConfig
// devices, one handle per device) or the processes of a communicator
// (pp_comm_init, one process per GPU). One shard: run_round.
struct ExchangeScope {  // the exchange serves plan steps only
  pp_handle* g;
  explicit ExchangeScope(pp_handle* gg) : g(gg) { g->xchg_active = g->xchg != nullptr; }
  ~ExchangeScope() { g->xchg_active = false; }
};

void run_round_shards(pp_handle* h, uint64_t t, int iter, int r0, int rc, const double* center,
                      int64_t n, pp_record* out) {
  if (h->xchg != nullptr && h->shards.empty()) {  // one rank of a communicator
    ExchangeScope scope(h);
    const int64_t c0 = n * h->shard_rank / h->shard_world;
    const int64_t c1 = n * (h->shard_rank + 1) / h->shard_world;
    run_round(h, t, iter, r0, rc, center, c0, c1, nullptr, out, nullptr);
    return;
  }
  if (h->shards.empty()) {
    run_round(h, t, iter, r0, rc, center, 0, n, nullptr, out, nullptr);
    return;
  }
  const int S = static_cast<int>(h->shards.size()) + 1;
  std::vector<std::vector<pp_record>> recs(S, std::vector<pp_record>(rc));
  std::vector<std::exception_ptr> errs(S);
  if (h->thread_group) h->thread_group->reset();
  h->shard_pool->run(S, [&](int k) {
    pp_handle* g = k == 0 ? h : h->shards[k - 1];
    try {
      ck(cudaSetDevice(g->device), "cudaSetDevice");
      if (g->pending_upload) {  // this plan step's snapshot, on the shard's own thread
        std::function<void()> up = std::move(g->pending_upload);
        g->pending_upload = nullptr;
        up();
      }
      ExchangeScope scope(g);
      run_round(g, t, iter, r0, rc, center, n * k / S, n * (k + 1) / S, nullptr, recs[k].data(),
                nullptr);
    } catch (...) {
      errs[k] = std::current_exception();
      if (h->thread_group) h->thread_group->abort();  // release the other shards
    }
  });
  ck(cudaSetDevice(h->device), "cudaSetDevice");
  for (auto& e : errs) {
    if (e) std::rethrow_exception(e);
  }
  // every shard certified the same global winners
  for (int r = 0; r < rc; ++r) {
    for (int k = 1; k < S; ++k) {
      if (recs[k][r].candidate != recs[0][r].candidate || recs[k][r].cls != recs[0][r].cls) {
        throw std::logic_error("sharded round: shards disagree on the winner");
      }
    }
    out[r] = recs[0][r];
  }
}

// The shards' timings folded into the planner's (kernel time: the slowest
// shard, the shards run concurrently).
void gather_shard_timing(pp_handle* h) {
  for (pp_handle* g : h->shards) {
    const pp_timing& q = g->timing;
    h->timing.kernel_ms = std::max(h->timing.kernel_ms, q.kernel_ms);
    h->timing.rollout_ms = std::max(h->timing.rollout_ms, q.rollout_ms);
    h->timing.executed_steps += q.executed_steps;
    h->timing.checked_states += q.checked_states;
    h->timing.samples += q.samples;
    h->timing.launches += q.launches;
    h->timing.refined += std::max(q.refined, 0);
    h->timing.fp64_rounds = std::max(h->timing.fp64_rounds, q.fp64_rounds);
    h->timing.h2d_bytes += q.h2d_bytes;
    h->timing.d2h_bytes += q.d2h_bytes;
    g->timing = pp_timing{};
  }
}

void plan_step_resident(pp_handle* h, uint64_t t, pp_plan_output* out) {
  const int P = h->P;
  const auto& cfg = h->cfg;
  const pp_snapshot& snap = *h->snapshot;
  std::vector<double> init_center(P, 0.0);
  if (snap.warm_theta_len == P) init_center.assign(snap.warm_theta, snap.warm_theta + P);

  const int R = cfg.n_restarts, I = cfg.n_iter_max, n = cfg.n_candidates;
  h->winner_rollouts.clear();
  for (pp_handle* g : h->shards) g->winner_rollouts.clear();
  // Iteration 0 of every restart centres on the warm start: one launch.
  std::vector<pp_record> first(R);
  run_round_shards(h, t, 0, 0, R, init_center.data(), n, first.data());

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
        run_round_shards(h, t, it, r, 1, center.data(), n, &rec);
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
  gather_shard_timing(h);
  phase("merged");
  out->evaluated = evaluated;
  if (out->best_theta != nullptr) std::memcpy(out->best_theta, best_theta.data(), sizeof(double) * P);
  int32_t len = 0;
  // the certification already ran this rollout when the winner was one of
  // its window members (any shard): copy it
  const pp_handle::WinnerRollout* done_w = nullptr;
  for (size_t k = 0; k <= h->shards.size() && done_w == nullptr && win.candidate >= 0; ++k) {
    const pp_handle* g = k == 0 ? h : h->shards[k - 1];
    for (const auto& w : g->winner_rollouts) {
      if (w.restart == win.restart && w.iter == win.iter && w.candidate == win.candidate) {
        done_w = &w;
        break;
      }
    }
  }
  if (done_w != nullptr) {
    out->predicted = done_w->stats;
    len = done_w->len;
    if (out->trajectory != nullptr) {
      std::memcpy(out->trajectory, done_w->traj.data(), sizeof(double) * done_w->traj.size());
    }
  } else {
    host_rollout(h, snap, best_theta.data(), &out->predicted, out->trajectory, cfg.H + 1, &len);
  }
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
    for (pp_handle* g : h->shards) {
      g->pending_upload = nullptr;
      g->pending_field = nullptr;
    }
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
    for (pp_handle* g : h->shards) {
      g->timing = pp_timing{};
      g->pending_upload = [g, snap] { upload_snapshot(g, *snap, true); };
    }
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
    for (pp_handle* g : h->shards) {
      g->timing = pp_timing{};
      g->pending_upload = [g, snap] { upload_points(g, *snap, true); };
    }
    phase("upload");
    plan_step_resident(h, t, out);
    phase("done");
    g_clock = nullptr;
    clock.flush();
  });
}

pp_status pp_comm_unique_id(uint8_t* out) {
  return guarded([&] {
    if (out == nullptr) throw std::invalid_argument("null argument");
    std::string why;
    if (!nccl_available(&why)) throw std::runtime_error("NCCL unavailable: " + why);
    nccl_unique_id(out);
  });
}

pp_status pp_comm_init(pp_handle* h, const uint8_t* id, int32_t world, int32_t rank) {
  return guarded([&] {
    if (h == nullptr || id == nullptr) throw std::invalid_argument("null argument");
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("bad rank / world");
    if (!h->shards.empty()) {
      throw std::invalid_argument("a planner over several devices cannot join a communicator");
    }
    if (h->cfg.n_candidates < world) {
      throw std::invalid_argument("fewer candidates than ranks");
    }
    ck(cudaSetDevice(h->device), "cudaSetDevice");
    h->xchg.reset();
    h->xchg = make_nccl_exchange(id, world, rank);
    h->shard_rank = rank;
    h->shard_world = world;
  });
}

uint64_t pp_pack_key(int32_t cls, int32_t t_goal, float cost, uint32_t candidate) {
  return ppdev::pack_key(cls, t_goal, cost, candidate);
}

void pp_unpack_key(uint64_t key, int32_t* cls, int32_t* t_goal, float* cost,
                   uint32_t* candidate) {
  const ppdev::Unpacked u = ppdev::unpack_key(key);
  if (cls != nullptr) *cls = u.cls;
  if (t_goal != nullptr) *t_goal = u.t_goal;
  if (cost != nullptr) *cost = u.cost;
  if (candidate != nullptr) *candidate = u.idx;
}

const char* pp_exchange_kind(const pp_handle* h) {
  if (h == nullptr || h->xchg == nullptr) return "none";
  return h->xchg->kind();
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
