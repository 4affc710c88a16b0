// rollout.cuh -- the fused per-control-step sampler kernels (sm_100a).
//
// One lane per candidate. Per candidate a lane
//   1. derives the keyed SplitMix64 stream in closed form and draws
//      theta = center + sigma * N(0,1) (src/rng.cpp:26-58,
//      src/planner.cpp:207-226), rounded once to Real (sample.cuh),
//   2. rolls the kinematic bicycle over the horizon with the reference's
//      exact check order (src/planner.cpp:66-191): collision vs obstacle row h,
//      inclusive goal box in the goal frame, horizon stop, tanh MLP ->
//      map_controls -> explicit Euler (step.cuh, nets.cuh),
//   3. scores the rollout (src/planner.cpp:27-44); the round reduces to the
//      lexicographically best candidate per restart, ties to the lowest index
//      (reduce.cuh).
//
// The obstacle field arrives binned on a cell grid (csrc/capi/field.hpp) and
// is staged once per CTA in shared memory by a TMA bulk copy when it fits. A
// collision query visits only the cells under the chassis's bounding box:
// every other point lies outside the rectangle, so the reference's test
// would reject it too and the verdict is unchanged (field_query.cuh).
//
// Two schedules:
//   generate_kernel + refill_kernel (theta in registers: [5,2,2], [5,10,2],
//     FP32 [5,10,10,2]): the generator draws theta and the first action of
//     every candidate at full SIMT width into an L2-sized buffer; in the
//     rollout kernel (a dependent launch) persistent warps claim
//     restart-aligned 32-candidate batches and a lane whose rollout ends
//     loads the next candidate at once, so lanes never idle behind the
//     longest rollout of their warp. With one restart, lane bests flush into
//     per-warp tables and the last CTA reduces the CTA records; with several,
//     the rollout writes sample keys only and reduce_keys_kernel forms the
//     per-restart winners.
//   lockstep_kernel (any architecture, theta in a global column per lane):
//     one candidate per lane per tile, last-CTA reduction.
// select_kernel takes the near-tie window of the certified re-ranking,
// refine_kernel evaluates a wide window in FP64.
//
// Real = float: throughput path (FMA contraction on). Real = double: parity
// path (rollout_f64.cu is compiled with --fmad=false so each add/mul rounds
// like the reference's -ffp-contract=off build).
#pragma once

#include "reduce.cuh"
#include "sample.cuh"

namespace ppdev {

// --------------------------------------------------- generate kernel ----
// theta (rounded to Real), the first action and the state it leads to
// (state 1) of every candidate of the round, one thread per candidate at full
// SIMT width: the FP64 RNG lives here and not in the rollout kernel, so the
// rollout kernel stays register-light, and a rollout starts at state 1.
// Layout: one record of rec_width(P) Reals per candidate, [theta 0..P-1]
// [x y phi v act pa0 path of state 1][f0 f1: the first action][pad], so a
// refilling lane loads it with 16-byte vector loads; the flat index is
// s = r * count + local (restart-major).
constexpr int kRecState = 9;
template <typename Real>
constexpr int rec_width(int P) {
  return ((P + kRecState) * static_cast<int>(sizeof(Real)) + 15) / 16 * 16 /
         static_cast<int>(sizeof(Real));
}
template <typename Real>
__device__ __forceinline__ void store_state(const Lane<Real>& L, Real* v) {
  v[0] = L.x;
  v[1] = L.y;
  v[2] = L.phi;
  v[3] = L.v;
  v[4] = L.act;
  v[5] = L.pa0;
  v[6] = L.path;
  v[7] = L.f0;
  v[8] = L.f1;
}
// a lane at state 1 from its record
template <typename Real>
__device__ __forceinline__ void load_state(Lane<Real>& L, const Real* v) {
  L.x = v[0];
  L.y = v[1];
  L.phi = v[2];
  L.v = v[3];
  L.act = v[4];
  L.pa0 = v[5];
  L.path = v[6];
  L.h = 1;
  L.mstep = kNoStep;
  L.mpath = Real(0);
}
template <typename Real>
using Vec16 = typename std::conditional<sizeof(Real) == 4, float4, double2>::type;

// One candidate's record: theta of restart r, local candidate `local`, and
// its first action, written to record slot s.
template <typename Real, class Net>
__device__ __forceinline__ void generate_one(const RoundArgs& a, const Consts<Real>& K,
                                             const Real s0[5], int r, int64_t local, int64_t s) {
  constexpr int P = Net::P;
  constexpr int W = rec_width<Real>(P);
  constexpr int V = W * static_cast<int>(sizeof(Real)) / 16;
  Vec16<Real>* recs = static_cast<Vec16<Real>*>(a.theta_buf);
  union {
    Real v[W];
    Vec16<Real> q[V];
  } rec;
  draw_theta<Real, P>(a, __ldg(a.key_prefix + r), a.injected ? local : a.cand_begin + local, P,
                      [&](int i, Real v) { rec.v[i] = v; });
  Net n;
#pragma unroll
  for (int i = 0; i < P; ++i) n.w[i] = rec.v[i];
  Real f0, f1;
  n.eval(s0, f0, f1);  // first action (src/planner.cpp:130-132)
  Lane<Real> L;
  L.start(K, f0, f1);
  first_step(L, K);
  store_state(L, rec.v + P);
  if constexpr (prescaled<Real, Net>(true)) {
    const Real in_scale[5] = {K.inv_xi * Real(2.8853900817779268), K.inv_eta * Real(2.8853900817779268),
                              K.inv_phi * Real(2.8853900817779268), K.inv_v * Real(2.8853900817779268),
                              Real(2.8853900817779268)};
    prescale<Net>(rec.v, in_scale);
  }
#pragma unroll
  for (int i = P + kRecState; i < W; ++i) rec.v[i] = Real(0);
  const unsigned long long keep = l2_keep_policy();
#pragma unroll
  for (int j = 0; j < V; ++j) st_rec(recs + s * V + j, rec.q[j], keep);
}

// Resident 256-thread CTAs per SM the generator's register cap must allow:
// FP32 [5,2,2] PARAPLAN_GEN_MINB; FP32 [5,10,2] (a 91-float record)
// PARAPLAN_GEN_MINB_MID (2: 128 registers, a little spill, measured on B200:
// its C2 round 0.557 -> 0.453 ms against 1 CTA at 232 registers; 3 CTAs
// spill 328 B and give 0.507); the rest 1 (FP64 [5,2,2] needs 102 registers,
// 2 CTAs anyway; 3 CTAs measured no faster)
template <typename Real, class Net>
constexpr int gen_min_blocks() {
  return sizeof(Real) != 4 ? 1
         : Net::P <= 24    ? PARAPLAN_GEN_MINB
         : Net::P <= PARAPLAN_GEN_MID_MAXP ? PARAPLAN_GEN_MINB_MID
                           : 1;
}

template <typename Real, class Net>
__global__ void __launch_bounds__(256, gen_min_blocks<Real, Net>())
    generate_kernel(const RoundArgs a) {
  constexpr int P = Net::P;
  constexpr int W = rec_width<Real>(P);
  constexpr int V = W * static_cast<int>(sizeof(Real)) / 16;
  const Consts<Real>& K = consts_of<Real>(a);
  // the round's device start (copy_out_kernel publishes the round's span)
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.exec != nullptr) a.exec[kExecRoundT0] = global_ns();
  Real s0[5];
  start_features(K, s0);
  Vec16<Real>* recs = static_cast<Vec16<Real>*>(a.theta_buf);
  const int64_t total = a.count * a.restart_count;
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < total;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // restart of flat index s (32-bit division when the round is small); a
    // list round draws item s = candidate list[s] of the listed round
    const int64_t flat = a.list != nullptr ? a.list[s] : s;
    const int64_t cnt = a.list != nullptr ? a.list_count : a.count;
    const int r = flat < cnt ? 0  // one restart (and a list of one): no division
                  : flat <= 0x7fffffff && cnt <= 0x7fffffff
                      ? static_cast<int>(static_cast<uint32_t>(flat) / static_cast<uint32_t>(cnt))
                      : static_cast<int>(flat / cnt);
    const int64_t local = flat - static_cast<int64_t>(r) * cnt;
    generate_one<Real, Net>(a, K, s0, r, local, s);
  }
  (void)recs;
}

// ------------------------------------------------------ refill kernel ----
// Resident CTAs per SM the register allocation must allow: [5,2,2] in FP32
// fits 6 (<= 85 registers), wider nets and FP64 need more registers.
template <typename Real, class Net>
constexpr int refill_min_blocks(int grid = 3) {
  return sizeof(Real) == 4
             ? (Net::kP <= 24 ? (grid == 1 || grid == 2 ? PARAPLAN_REFILL_MINB_2D : PARAPLAN_REFILL_MINB)
                              : (Net::kP <= 100 ? PARAPLAN_REFILL_MINB_MID : PARAPLAN_REFILL_MINB_BIG))
             : (Net::kP <= 24 ? PARAPLAN_REFILL64_MINB : 2);
}

// A relaxed load of a restart's goal cut (the value other lanes lower with
// atomicMin); `tag` (loop-variant) keeps it from being hoisted out of the
// loop.
__device__ __forceinline__ uint32_t ld_cut(const uint32_t* p, int tag) {
  uint32_t v;
  asm("ld.relaxed.gpu.global.u32 %0, [%1]; // %2" : "=r"(v) : "l"(p), "r"(tag));
  return v;
}

// kCut: with the goal-horizon cut (a.goal_cut set); without it the loop
// carries none of its instructions (~6% of a C2 rollout that never reaches).
template <typename Real, class Net, int kGrid, bool kCut>
__global__ void __launch_bounds__(kBlock, refill_min_blocks<Real, Net>(kGrid))
    refill_kernel(const RoundArgs a) {
  constexpr int P = Net::kP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Key table[kWarps][kMaxRestartsPerLaunch];
  __shared__ Key red[32];
  __shared__ unsigned long long red_sum[32];

  mark_start(a);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const Consts<Real>& K = consts_of<Real>(a);
  const int H = K.H;
  for (int i = threadIdx.x; i < kWarps * kMaxRestartsPerLaunch; i += blockDim.x) {
    (&table[0][0])[i] = empty_key();
  }
  const Field<Real> f = stage_field<Real, kGrid>(a, smem_raw);
  wait_prior_grid();  // the generator's theta records

  const int bpr = a.tiles_per_restart;  // 32-candidate batches per restart
  const unsigned total_batches = static_cast<unsigned>(a.n_tiles);
  constexpr int W = rec_width<Real>(P);
  constexpr int V = W * static_cast<int>(sizeof(Real)) / 16;
  const Vec16<Real>* recs = static_cast<const Vec16<Real>*>(a.theta_buf);
  const unsigned long long drop = l2_drop_policy();

  Net net;
#pragma unroll
  for (int i = 0; i < P; ++i) net.w[i] = Real(0);
  // state 0 is every candidate's: its checks run once per thread (the
  // verdicts every lane would compute); lanes start at state 1 (the
  // generator's record), or, when state 0 already stops, end there
  Lane<Real> L;
  L.start(K, Real(0), Real(0));  // idle lanes step a valid (discarded) state
  L.ephi = M<Real>::wrap(K.gphi - Real(0));
  const int cls0 = check_state<Real, kGrid>(L, K, f, H, true, Real(0), Real(1));
  L.mstep = kNoStep;
  const Real ephi0 = L.ephi;
  bool active = false;
  int my_r = 0;
  int my_c = 0;  // local candidate index within [0, count)
  LaneKey<Real> best = lane_empty<Real>();
  int best_r = -1;
  int q_head = 32, q_count = 0, q_r = 0, q_c0 = 0;
  bool exhausted = false;
  // per lane: a few candidates x H. The checked states are the steps plus
  // one per candidate (L.h + 1 each), added once for the whole round
  unsigned n_steps = 0;
  const bool track = a.keys_only == 0;  // lane bests (one restart) or keys only
  // lane bests can cross restarts only when a launch holds several
  const bool cross = track && a.restart_count > 1;
  // goal-horizon cut (kCut): a lane stops at state cut_at = its restart's
  // earliest t_goal (as this lane last saw it) + slack. The restart's value
  // is loaded every 8 iterations before the step and folded in after it (no
  // wait on the load); a lane that reaches lowers it at once. With several
  // restarts a lane forgets the cut when it takes a new candidate (a list
  // round is one slot: the host cuts list rounds of one restart only).
  uint32_t* const goal_cut = kCut ? a.goal_cut : nullptr;
  constexpr int kNoCut = 0x7fffffff;
  int cut_at = kNoCut;
  unsigned iter = 0;

  // A lane whose rollout ends parks its class in `pend`; its keys are written
  // and it is refilled at the warp's next flush, every a.flush_every-th
  // iteration. The flush code runs for the whole warp whenever any lane
  // needs it, so batching it trades parked lane-steps for fewer flushes
  // (the host sizes it from the last round's mean rollout length).
  int pend = -1;  // class of a finished rollout (| 4: cut) awaiting its keys
  int flush_cd = 1;
  for (;;) {
    // every a.flush_every-th iteration (a countdown); the goal-cut variant,
    // whose rounds can hold long rollouts, also once a.flush_min lanes wait
    bool flush_now = --flush_cd <= 0;
    if (kCut && a.flush_min > 0) {
      flush_now |= __popc(__ballot_sync(kFull, !active)) >= a.flush_min;
    }
    if (flush_now) flush_cd = a.flush_every;
    if (flush_now) {
      // -------- finished lanes: keys and lane bests --------
      // lane bests are per restart: flush the old one before crossing over
      if (cross) {
        bool flush = pend >= 0 && best.cls >= 0 && best_r != my_r;
        if (__any_sync(kFull, flush)) flush_bests(flush, best, best_r, table[warp], lane);
      }
      if (pend >= 0) {
        const int cls = pend & 3;
        const bool cut = (pend & 4) != 0;
        const Real term = terminal_cost(L, K);
        const int tg = cut ? kCutTGoal : L.h;
        if (track) {
          const LaneKey<Real> k =
              make_lane_key<Real>(cls, tg, L.path, term, static_cast<int>(a.cand_begin + my_c));
          if (best.cls < 0 || prefer(k, best)) {
            best = k;
            best_r = my_r;
          }
        }
        n_steps += static_cast<unsigned>(L.h);
        if (a.per_sample != nullptr) {
          // the first action from the record (not kept in the lane's registers)
          const Real* rv = reinterpret_cast<const Real*>(recs) +
                           (static_cast<int64_t>(my_r) * a.count + my_c) * W + P;
          write_sample(a, static_cast<int64_t>(my_r) * a.count + my_c, cls, L, term, rv[7], rv[8]);
        }
        write_skey(a, static_cast<int64_t>(my_r) * a.count + my_c, cls, L, term, tg);
        pend = -1;
      }
      // -------- hand the warp's current batch to idle lanes --------
      const unsigned need = __ballot_sync(kFull, !active);
      if (need != 0u) {
        if (q_head >= q_count && !exhausted) {
          unsigned b = 0;
          if (lane == 0) b = atomicAdd(&a.counters[0], 1u);
          b = __shfl_sync(kFull, b, 0);
          if (b >= total_batches) {
            exhausted = true;
          } else {
            q_r = a.restart_count == 1 ? 0 : static_cast<int>(b) / bpr;
            q_c0 = (static_cast<int>(b) - q_r * bpr) * 32;
            const int64_t left = a.count - q_c0;
            q_count = left < 32 ? static_cast<int>(left) : 32;
            q_head = 0;
            // the batch's records into L1: the lanes refill from it over the
            // next iterations (all but the first few hit L1)
            if (lane < q_count) {
              const char* rp = reinterpret_cast<const char*>(
                  recs + (static_cast<int64_t>(q_r) * a.count + q_c0 + lane) * V);
              prefetch_l1(rp);
              prefetch_l1(rp + W * static_cast<int>(sizeof(Real)) - 1);
            }
          }
        }
        const int avail = q_count - q_head;
        if (avail > 0) {
          const int rank = __popc(need & ((1u << lane) - 1u));
          if (!active && rank < avail) {
            my_r = q_r;
            my_c = q_c0 + q_head + rank;
            const int64_t sidx = static_cast<int64_t>(my_r) * a.count + my_c;
            // contiguous 16-byte aligned record: V vector loads
            union {
              Real v[W];
              Vec16<Real> q[V];
            } rec;
#pragma unroll
            for (int j = 0; j < V; ++j) rec.q[j] = ld_rec(recs + sidx * V + j, drop);
#pragma unroll
            for (int i = 0; i < P; ++i) net.w[i] = rec.v[i];
            if (cls0 < 0) {
              load_state(L, rec.v + P);
            } else {
              L.start(K, Real(0), Real(0));
              L.ephi = ephi0;
            }
            active = true;
            if (kCut && a.restart_count > 1) cut_at = kNoCut;
          }
          q_head += __popc(need) < avail ? __popc(need) : avail;
        }
      }
      // stream exhausted, all lanes done and flushed (only a flush can end
      // the loop: between flushes a lane that stops parks in `pend`)
      if (!__any_sync(kFull, active || pend >= 0)) break;
    }

    // -------- one rollout state per lane --------
    uint32_t cut_ld = kCutNone;  // used after the step
    if (kCut && (++iter & 7u) == 0u) cut_ld = ld_cut(goal_cut + my_r, static_cast<int>(iter));
    // every lane steps (idle lanes only at the stream tail, results unused).
    // When state 0 already stops (cls0 >= 0) the lanes hold state 0, whose
    // checks give cls0 again and whose transition is not committed
    int cls = advance<Real, kGrid, Net, false>(L, net, K, f, H, active);
    bool cut = false;
    if constexpr (kCut) {
      if (cut_ld != kCutNone) cut_at = min(cut_at, static_cast<int>(cut_ld) + a.cut_slack);
      // cut: states 0..h checked without reaching, h >= the restart's
      // earliest t_goal + slack (a lane's view is never below the final one)
      cut = active && cls < 0 && L.h >= cut_at;
      if (active && cls == 2 && L.h + a.cut_slack < cut_at) {
        cut_at = L.h + a.cut_slack;
        atomicMin(goal_cut + my_r, static_cast<uint32_t>(L.h));
      }
      if (cut) cls = 2;
    }
    if (active && cls >= 0) {
      pend = cls | (cut ? 4 : 0);
      active = false;
    }
  }

  // -------- flush lane bests, combine warps, publish CTA records --------
  mark_end(a);
  const unsigned long long steps = block_sum(static_cast<unsigned long long>(n_steps), red_sum);
  if (threadIdx.x == 0) {
    atomicAdd(&a.exec[0], steps);
    atomicAdd(&a.exec[1], steps + (blockIdx.x == 0 ? static_cast<unsigned long long>(
                                                         a.count * a.restart_count)
                                                   : 0ull));
  }
  if (!track) return;  // reduce_keys_kernel forms the winners
  bool flush = best.cls >= 0;
  flush_bests(flush, best, best_r, table[warp], lane);
  __syncthreads();
  for (int r = threadIdx.x; r < a.restart_count; r += blockDim.x) {
    Key k = table[0][r];
    for (int w = 1; w < kWarps; ++w) {
      if (table[w][r].cls >= 0 && (k.cls < 0 || prefer(table[w][r], k))) k = table[w][r];
    }
    a.tile_recs[static_cast<size_t>(r) * gridDim.x + blockIdx.x] = Rec{k.cls, k.idx, k.k1, k.k2};
  }
  finish_round(a, a.tile_recs, static_cast<int>(gridDim.x), red);
}

// Per-restart winners from the sample keys (RoundArgs::keys_only): block
// (x, r) reduces chunk x of restart r; the last block reduces the chunks.
// The keys are the rollout's own: (cls, t_goal, FP32 cost) give the same
// (cls, k1, k2) as make_key, and the index is the slot's.
static __global__ void __launch_bounds__(256) reduce_keys_kernel(const RoundArgs a) {
  __shared__ Key red[32];
  wait_prior_grid();  // the rollout's keys
  const int r = blockIdx.y;
  const int64_t chunk = (a.count + gridDim.x - 1) / gridDim.x;
  const int64_t lo = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t hi = lo + chunk < a.count ? lo + chunk : a.count;
  Key k = empty_key(), kf = empty_key();  // best, best not flagged marginal
  for (int64_t c = lo + threadIdx.x; c < hi; c += blockDim.x) {
    const int64_t slot = static_cast<int64_t>(r) * a.count + c;
    double cost;
    uint32_t meta;
    if (a.skey32) {
      const SKey32 q = static_cast<const SKey32*>(a.skeys)[slot];
      cost = static_cast<double>(q.cost);
      meta = q.meta;
    } else {
      const SKey q = static_cast<const SKey*>(a.skeys)[slot];
      cost = q.cost;
      meta = q.meta;
    }
    Key o;
    o.cls = meta_cls(meta);
    o.idx = static_cast<int>(a.cand_begin + c);
    if (o.cls == 2) {
      o.k1 = -static_cast<double>(meta_tgoal(meta));
      o.k2 = -cost;
    } else {
      o.k1 = -cost;
      o.k2 = 0.0;
    }
    if (k.cls < 0 || prefer(o, k)) k = o;
    if (!meta_flagged(meta) && (kf.cls < 0 || prefer(o, kf))) kf = o;
  }
  k = block_best(k, red);
  kf = block_best(kf, red);
  const unsigned n_src = gridDim.x;
  Rec* tiles_free = a.tile_recs + static_cast<size_t>(a.restart_count) * n_src;
  if (threadIdx.x == 0) {
    a.tile_recs[static_cast<size_t>(r) * n_src + blockIdx.x] = Rec{k.cls, k.idx, k.k1, k.k2};
    tiles_free[static_cast<size_t>(r) * n_src + blockIdx.x] = Rec{kf.cls, kf.idx, kf.k1, kf.k2};
  }
  if (!last_block(a)) return;
  reduce_recs_warps(a, a.tile_recs, static_cast<int>(n_src), a.out);
  if (a.out_free != nullptr) reduce_recs_warps(a, tiles_free, static_cast<int>(n_src), a.out_free);
  publish_round(a);
}

// ---------------------------------------------------- lockstep kernel ----
template <typename Real, class Net>
struct NetFactory;

template <typename Real, int H1>
struct NetFactory<Real, NetReg<Real, H1>> {
  static __device__ __forceinline__ NetReg<Real, H1> make(const RoundArgs&) { return {}; }
};
template <typename Real, int A, int B>
struct NetFactory<Real, NetReg3<Real, A, B>> {
  static __device__ __forceinline__ NetReg3<Real, A, B> make(const RoundArgs&) { return {}; }
};

template <typename Real>
struct Scratch;
template <>
struct Scratch<float> {
  static __device__ __forceinline__ float* ptr(const RoundArgs& a) { return a.theta_scratch; }
};
template <>
struct Scratch<double> {
  static __device__ __forceinline__ double* ptr(const RoundArgs& a) { return a.theta_scratch64; }
};

template <typename Real>
struct NetFactory<Real, NetGlobal<Real>> {
  static __device__ __forceinline__ NetGlobal<Real> make(const RoundArgs& a) {
    NetGlobal<Real> n;
    n.stride = a.grid * a.block;
    n.col = Scratch<Real>::ptr(a) + blockIdx.x * a.block + threadIdx.x;
    n.sizes = a.sizes;
    n.n_layers = a.n_layers;
    return n;
  }
};

template <typename Real, class Net, int kGrid>
__global__ void __launch_bounds__(kBlock) lockstep_kernel(const RoundArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Key red[32];
  __shared__ unsigned long long red_sum[32];
  __shared__ int s_tile;

  mark_start(a);
  const Consts<Real>& K = consts_of<Real>(a);
  const int H = K.H;
  const int P = a.n_params;
  const Field<Real> f = stage_field<Real, kGrid>(a, smem_raw);
  Real s0[5];
  start_features(K, s0);

  Net net = NetFactory<Real, Net>::make(a);
  unsigned long long n_steps = 0, n_states = 0;
  for (;;) {
    if (threadIdx.x == 0) s_tile = static_cast<int>(atomicAdd(&a.counters[0], 1u));
    __syncthreads();
    const int tile = s_tile;
    __syncthreads();
    if (tile >= a.n_tiles) break;
    const int r = tile / a.tiles_per_restart;
    const int64_t local =
        static_cast<int64_t>(tile - r * a.tiles_per_restart) * blockDim.x + threadIdx.x;
    Key key = empty_key();
    const bool valid = local < a.count;
    const int64_t c = a.cand_begin + (valid ? local : 0);
    draw_theta<Real, Net::kP>(a, __ldg(a.key_prefix + r), a.injected ? (valid ? local : 0) : c,
                              P, [&](int i, Real v) { net.set(i, v); });
    Real f0, f1;
    net.eval(s0, f0, f1);
    Lane<Real> L;
    L.start(K, f0, f1);
    int cls = -1;
    // lanes keep stepping (and discarding) until the whole warp is done
    while (__any_sync(kFull, cls < 0)) {
      const int k = advance<Real, kGrid>(L, net, K, f, H);
      if (cls < 0) cls = k;
    }
    if (valid) {
      const Real term = terminal_cost(L, K);
      key = make_key<Real>(cls, L.h, L.path, term, static_cast<int>(c));
      n_steps += static_cast<unsigned long long>(L.h);
      n_states += static_cast<unsigned long long>(L.h + 1);
      if (a.per_sample != nullptr) {
        write_sample(a, static_cast<int64_t>(r) * a.count + local, cls, L, term, L.f0, L.f1);
      }
      write_skey(a, static_cast<int64_t>(r) * a.count + local, cls, L, term);
    }
    const Key best = block_best(key, red);
    // tile records are restart-major: [r][tile within restart]
    if (threadIdx.x == 0) a.tile_recs[tile] = Rec{best.cls, best.idx, best.k1, best.k2};
  }
  mark_end(a);
  const unsigned long long steps = block_sum(static_cast<unsigned long long>(n_steps), red_sum);
  const unsigned long long states = block_sum(static_cast<unsigned long long>(n_states), red_sum);
  if (threadIdx.x == 0) {
    atomicAdd(&a.exec[0], steps);
    atomicAdd(&a.exec[1], states);
  }
  finish_round(a, a.tile_recs, a.tiles_per_restart, red);
}

// ------------------------------------------------------ select kernel ----
// Near-tie window of every restart: candidates of the winner's class whose
// key lies within (1 + rho) * cost + alpha of the round winner, plus every
// candidate flagged marginal. Indices are appended to a.sel_list.
static __global__ void __launch_bounds__(256) select_kernel(const RoundArgs a) {
  wait_prior_grid();  // the rollout's keys and winners
  const int64_t total = a.count * a.restart_count;
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < total;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = a.restart_count == 1
                      ? 0
                      : (total <= 0x7fffffff ? static_cast<int>(static_cast<uint32_t>(s) /
                                                                 static_cast<uint32_t>(a.count))
                                             : static_cast<int>(s / a.count));
    SelBound bd;
    if (a.sel_bound != nullptr) {  // widened window of a later pass
      bd = a.sel_bound[r];
    } else if (a.sel_packed) {  // sharded: around the GLOBAL best unflagged candidate
      const uint64_t pf = a.pkeys[a.restart_count + r];
      const Unpacked u = unpack_key(pf != kPackEmpty ? pf : a.pkeys[r]);
      bd.cls = u.cls;
      bd.t_goal = u.cls == 2 ? u.t_goal : 0;
      const double rho = u.cls != 2       ? a.sel_rho
                         : a.rho2_by_tgoal ? rho2_of(a.sel_rho2, a.sel_rho2_floor, u.t_goal)
                                           : a.sel_rho2;
      bd.thr = static_cast<double>(u.cost) * (1.0 + rho) + a.sel_alpha;
    } else {  // first pass: around the round winner (its best unflagged candidate)
      const Rec b = (a.out_free != nullptr && a.out_free[r].cls >= 0) ? a.out_free[r] : a.out[r];
      bd.cls = b.cls;
      bd.t_goal = b.cls == 2 ? static_cast<int>(-b.k1) : 0;
      const double rho = b.cls != 2       ? a.sel_rho
                         : a.rho2_by_tgoal ? rho2_of(a.sel_rho2, a.sel_rho2_floor, bd.t_goal)
                                           : a.sel_rho2;
      bd.thr = (b.cls == 2 ? -b.k2 : -b.k1) * (1.0 + rho) + a.sel_alpha;
    }
    SKey k;
    if (a.skey32) {
      const SKey32 k32 = static_cast<const SKey32*>(a.skeys)[s];
      k.cost = static_cast<double>(k32.cost);
      k.meta = k32.meta;
    } else {
      k = static_cast<const SKey*>(a.skeys)[s];
    }
    const int cls = meta_cls(k.meta);
    // flagged: a flip could improve it -- before a class-2 anchor's t_goal
    const uint32_t ms = meta_mstep(k.meta);
    bool take = bd.cls >= 0 && ms != kNoStep &&
                (bd.cls != 2 || ms <= static_cast<uint32_t>(bd.t_goal));
    if (cls == bd.cls && k.cost <= bd.thr) {
      take |= cls != 2 || meta_tgoal(k.meta) == bd.t_goal;
    }
    if (take) {
      const unsigned i = atomicAdd(&a.counters[2], 1u);
      if (i < static_cast<unsigned>(a.sel_cap)) {
        if (i < static_cast<unsigned>(kSelFirst)) {
          a.sel_list[i] = s;
        } else {
          a.sel_more[i - kSelFirst] = s;
        }
      }
    }
  }
}

// Packed keys of the per-restart winners (keypack.h): [best][best unflagged]
// per restart, for the cross-shard min-reduction. FP64 costs round up.
static __global__ void __launch_bounds__(128) pack_keys_kernel(const RoundArgs a) {
  wait_prior_grid();  // the round's winners
  for (int r = threadIdx.x; r < a.restart_count; r += blockDim.x) {
    for (int which = 0; which < 2; ++which) {
      const Rec b = which == 0 ? a.out[r] : (a.out_free != nullptr ? a.out_free[r] : a.out[r]);
      const double cost = b.cls == 2 ? -b.k2 : -b.k1;
      a.pkeys[which * a.restart_count + r] =
          pack_key(b.cls, b.cls == 2 ? static_cast<int>(-b.k1) : 0, __double2float_ru(cost),
                   static_cast<uint32_t>(b.cand));
    }
  }
}

// ------------------------------------------------------ refine kernel ----
// FP64 re-evaluation of the selected candidates (theta redrawn in FP64,
// FP64 field). One lane per candidate, warp-synchronous stepping.
template <class Net64>
struct RefineNet;
template <int H1>
struct RefineNet<NetReg<double, H1>> {
  static __device__ __forceinline__ NetReg<double, H1> make(const RoundArgs&) { return {}; }
};
template <>
struct RefineNet<NetGlobal<double>> {
  static __device__ __forceinline__ NetGlobal<double> make(const RoundArgs& a) {
    NetGlobal<double> n;
    n.stride = gridDim.x * blockDim.x;
    n.col = a.theta_scratch64 + blockIdx.x * blockDim.x + threadIdx.x;
    n.sizes = a.sizes;
    n.n_layers = a.n_layers;
    return n;
  }
};

template <class Net64, int kGrid>
__global__ void __launch_bounds__(128) refine_kernel(const RoundArgs a) {
  const Consts<double>& K = a.kd;
  const unsigned n_sel = min(__ldcg(&a.counters[2]), static_cast<unsigned>(a.sel_cap));
  const Field<double> f = field_at<double>(a, a.field64, a.lay64);
  double s0[5];
  start_features(K, s0);
  Net64 net = RefineNet<Net64>::make(a);
  // warp-uniform bound so every lane of a live warp keeps stepping
  // warps numbered block-fastest, so a short window spreads over every SM
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned base = ((threadIdx.x >> 5) * gridDim.x + blockIdx.x) * 32u; base < n_sel;
       base += stride) {
    const unsigned i = base + (threadIdx.x & 31u);
    const bool valid = i < n_sel;
    const int64_t s = a.ref_list[valid ? i : base];
    const int r = static_cast<int>(s / a.count);
    const int64_t local = s - static_cast<int64_t>(r) * a.count;
    draw_theta<double, Net64::kP>(a, __ldg(a.key_prefix + r),
                                  a.injected ? local : a.cand_begin + local, a.n_params,
                                  [&](int j, double v) { net.set(j, v); });
    double f0, f1;
    net.eval(s0, f0, f1);
    Lane<double> L;
    L.start(K, f0, f1);
    int cls = -1;
    while (__any_sync(kFull, cls < 0)) {
      const int k = advance<double, kGrid>(L, net, K, f, a.H);
      if (cls < 0) cls = k;
    }
    if (valid) {
      const double term = terminal_cost(L, K);
      const Key k = make_key<double>(cls, L.h, L.path, term, static_cast<int>(a.cand_begin + local));
      a.sel_out[i] = SelRec{k.cls, k.idx, r, 0, k.k1, k.k2};
    }
  }
}

// -------------------------------------------------------- theta draws ----
// The device's own theta draws of candidates [cand_begin, cand_begin + count)
// of restart 0 of the round (key prefix a.key_prefix[0]), P Reals per
// candidate: the RNG parity dump (pp_draw_theta).
template <typename Real>
static __global__ void __launch_bounds__(256) draw_kernel(const RoundArgs a, Real* out) {
  const int P = a.n_params;
  for (int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; c < a.count;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    Real* o = out + c * P;
    draw_theta<Real, 0>(a, __ldg(a.key_prefix), a.cand_begin + c, P,
                        [&](int i, Real v) { o[i] = v; });
  }
}

template <typename Real>
int launch_draw_impl(const RoundArgs& a, void* out, void* stream) {
  const int blocks = static_cast<int>(std::min<int64_t>((a.count + 255) / 256, std::max(a.sms, 1) * 8));
  draw_kernel<Real><<<std::max(blocks, 1), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      a, static_cast<Real*>(out));
  return static_cast<int>(cudaGetLastError());
}

// ------------------------------------------------------------ launch ----
// Register-resident nets use the refill schedule; PARAPLAN_SCHEDULE=lockstep
// forces the lockstep schedule (A/B measurements only).
inline bool force_lockstep() {
  static const bool v = [] {
    const char* e = std::getenv("PARAPLAN_SCHEDULE");
    return e != nullptr && std::strcmp(e, "lockstep") == 0;
  }();
  return v;
}

template <class Net>
bool refill_schedule() {
  return Net::kP > 0 && !force_lockstep();
}

using KernelFn = void (*)(const RoundArgs);

// Launch with programmatic stream serialization when `pdl` (the kernel calls
// wait_prior_grid() before reading its predecessor's output).
inline cudaError_t launch_dependent(KernelFn k, int grid, int block, size_t smem, cudaStream_t st,
                                    bool pdl, const RoundArgs& a) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(static_cast<unsigned>(block));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, a);
}

template <typename Real, class Net, int kGrid>
KernelFn kernel_of_g(bool cut) {
  if constexpr (Net::kP > 0) {
    if (refill_schedule<Net>()) {
      return cut ? refill_kernel<Real, Net, kGrid, true> : refill_kernel<Real, Net, kGrid, false>;
    }
  }
  return lockstep_kernel<Real, Net, kGrid>;
}

// grid mode of the field (0 x-buckets, 1 2-D, 2 2-D with cell boxes) -- a
// separate instantiation each, so the small-field kernel stays lean.
template <typename Real, class Net>
KernelFn kernel_of(int kind, bool cut = true) {
  switch (kind) {
    case 3:
      return kernel_of_g<Real, Net, 3>(cut);
    case 2:
      return kernel_of_g<Real, Net, 2>(cut);
    case 1:
      return kernel_of_g<Real, Net, 1>(cut);
    default:
      return kernel_of_g<Real, Net, 0>(cut);
  }
}

// Stage 1 of a round: the theta generator (refill schedule only; a no-op
// for the lockstep schedule, which draws theta itself).
template <typename Real, class Net>
int launch_generate_impl(const RoundArgs& a, void* stream) {
  if constexpr (Net::kP > 0) {
    if (refill_schedule<Net>()) {
      const int64_t total = a.count * a.restart_count;
      const int gen_blocks = static_cast<int>((total + 255) / 256);
      generate_kernel<Real, Net><<<gen_blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
      return static_cast<int>(cudaGetLastError());
    }
  }
  return 0;
}

// Stage 2: the rollout. After the generator it is a dependent launch (the
// rollout CTAs stage the field while the generator drains, then wait for its
// records).
template <typename Real, class Net>
int launch_rollout_impl(const RoundArgs& a, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto k = kernel_of<Real, Net>(grid_kind(a.grid_mode, a.field_smem_bytes, a.field_ns, a.field_nd,
                                               a.field_padded),
                                 a.goal_cut != nullptr);
  const size_t smem = static_cast<size_t>(a.field_smem_bytes);
  if (smem > 32 * 1024) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  }
  bool after_generate = false;
  if constexpr (Net::kP > 0) after_generate = refill_schedule<Net>();
  cudaError_t e = launch_dependent(k, a.grid, a.block, smem, st, after_generate, a);
  if (e == cudaSuccess && a.keys_only) {
    // about four blocks per SM over all restarts
    const int64_t per = std::max<int64_t>(1, std::min<int64_t>((a.count + 2047) / 2048,
                                                              std::max(a.sms, 1) * 4 / a.restart_count));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(per), static_cast<unsigned>(a.restart_count));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, reduce_keys_kernel, a);
  }
  return static_cast<int>(e);
}

// Near-tie window of a finished round (a dependent launch after the rollout).
inline int launch_select_impl(const RoundArgs& a, void* stream) {
  const int64_t total = a.count * a.restart_count;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, std::max(a.sms, 1) * PARAPLAN_SELECT_BPS));
  return static_cast<int>(
      launch_dependent(select_kernel, blocks, 256, 0, static_cast<cudaStream_t>(stream), true, a));
}

// FP64 re-evaluation of the selected window.
template <class Net64>
int launch_refine_impl(const RoundArgs& a, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (a.grid_mode == 2) {
    refine_kernel<Net64, 2><<<a.refine_grid, 128, 0, st>>>(a);
  } else if (a.grid_mode == 1) {
    refine_kernel<Net64, 1><<<a.refine_grid, 128, 0, st>>>(a);
  } else {
    refine_kernel<Net64, 0><<<a.refine_grid, 128, 0, st>>>(a);
  }
  return static_cast<int>(cudaGetLastError());
}

// Resident refine_kernel CTAs per SM (the smallest over the grid modes), so
// a wide window fills the GPU.
template <class Net64>
int refine_occupancy_impl() {
  int occ = 1 << 30;
  for (KernelFn k : {refine_kernel<Net64, 0>, refine_kernel<Net64, 1>, refine_kernel<Net64, 2>}) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, 128, 0) != cudaSuccess) return 2;
    occ = std::min(occ, b);
  }
  return std::max(1, occ);
}

template <typename Real, class Net>
int shape_impl(int device, int field_bytes, int grid, LaunchShape* out) {
  auto k = kernel_of<Real, Net>(grid);
  const bool refill = refill_schedule<Net>();
  const int smem_bytes = field_bytes;
  out->queue_bytes = 0;
  out->theta_elem = refill ? rec_width<Real>(Net::kP) : 0;  // Reals per candidate record
  int sms = 0, blocks = 0;
  cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return static_cast<int>(e);
  if (smem_bytes > 32 * 1024) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, kBlock, smem_bytes);
  if (e != cudaSuccess) return static_cast<int>(e);
  int smem_optin = 0;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  out->block = kBlock;
  out->grid = sms * (blocks > 0 ? blocks : 1);
  out->smem_limit = smem_optin;
  out->refill = refill ? 1 : 0;
  return 0;
}

}  // namespace ppdev
