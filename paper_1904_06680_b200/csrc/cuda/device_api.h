// device_api.h -- host-visible interface of the sm_100a kernels (no CUDA
// types; streams are passed as void*). Implemented in rollout_f32.cu /
// rollout_f64.cu (one instantiation of rollout.cuh each) and peak.cu.
#pragma once

#include <cstdint>

#include "keypack.h"

namespace ppdev {

constexpr int kMaxLayers = 16;
constexpr int kMaxRestartsPerLaunch = 64;  // per-warp restart tables of the refill kernel
constexpr int kSelFirst = 512;  // selected indices stored in the round block (copied back with it)

// Per-sample output of the parity/debug path (same layout as pp_rollout_stats).
struct SampleOut {
  int32_t reached, t_goal, collided, steps;
  double path_length, terminal_cost, first_a0, first_a1;
};

// Compact per-sample key for the near-tie window: 16 bytes for FP64 rounds,
// 8 bytes (SKey32) for FP32 rounds, whose costs are floats anyway.
struct SKey {
  double cost;    // terminal cost (cls 0/1) or path length (cls 2)
  uint32_t meta;  // make_meta below
  uint32_t mpath; // FP64 rounds: float bits of the path up to the flagged state, rounded down
};

// meta of a sample key: cls (2 bits) | t_goal (15 bits, class 2) | the
// earliest state index at which a discrete verdict that could IMPROVE the
// candidate came within the flag band of flipping (a narrow goal miss, a
// narrow collision hit; 15 bits, kNoStep = none). A class-2 window anchored
// at t_goal T needs only the flags at states <= T: a later flip reaches later.
constexpr uint32_t kNoStep = 0x7fff;
constexpr int kMaxKeyHorizon = 0x7ffe;  // H the 15-bit fields hold
PP_HD uint32_t make_meta(int cls, int t_goal, uint32_t mstep) {
  return static_cast<uint32_t>(cls) | (static_cast<uint32_t>(cls == 2 ? t_goal : 0) << 2) |
         (mstep << 17);
}
// Goal-horizon cut (refill schedule): once a rollout of a restart reaches the
// goal at state T, no candidate of that restart that has not reached it by
// state T + slack can win (class 2 ranks first, then the earliest t_goal), so
// its lane stops there. Its key is class 2 with t_goal kCutTGoal, behind
// every real t_goal (H <= kMaxKeyHorizon); its flags up to the cut are kept.
constexpr int kCutTGoal = 0x7fff;
constexpr uint32_t kCutNone = 0xffffffffu;
PP_HD int meta_cls(uint32_t m) { return static_cast<int>(m & 3u); }
PP_HD int meta_tgoal(uint32_t m) { return static_cast<int>((m >> 2) & 0x7fffu); }
PP_HD uint32_t meta_mstep(uint32_t m) { return m >> 17; }
PP_HD bool meta_flagged(uint32_t m) { return (m >> 17) != kNoStep; }

// rho of a window anchored on a class-2 candidate reaching at t_goal T. The
// relative error of a reaching rollout's path grows with T (measured,
// profiles/r2_error_model*.json; FP32: 1.6e-7 at T <= 6, 3e-7 at T = 20-40,
// 1.3e-6 at T = 78, 2.1e-5 at T = 125; FP64: <= 1.1e-13): base (T / 150)^2,
// at least `floor` -- FP32 base 1e-3, floor 2e-6; FP64 base 1e-11, floor
// 2e-14 -- >= 8x the measured error at every T. Host and device evaluate it
// alike (no FMA contraction in either translation unit).
PP_HD double rho2_of(double base, double floor, int T) {
  const double f = static_cast<double>(T) / 150.0;
  const double r = base * (f * f < 1.0 ? f * f : 1.0);
  return r > floor ? r : floor;
}
struct SKey32 {
  float cost;
  uint32_t meta;
};

// Window of one restart for a widened select pass: class, t_goal (class 2)
// and cost threshold; cls = -1 selects nothing (restart certified).
struct SelBound {
  int32_t cls, t_goal;
  double thr;
};

// FP64 re-evaluated key of a selected candidate.
struct SelRec {
  int32_t cls, cand, restart, pad;
  double k1, k2;
};

// Winner of a tile / of a restart segment. cls = -1 marks "no candidate".
struct Rec {
  int32_t cls;
  int32_t cand;  // index within the restart
  double k1, k2;
};

// Kernel kind 3 scans a lane's x-bucket window kK3Group points per step of
// its loop, with no remainder pass: the sentinel padding after each part of
// the staged image holds N + kK3Group - 1 points (csrc/capi/upload.cpp).
#ifndef PARAPLAN_K3_GROUP
#define PARAPLAN_K3_GROUP 2
#endif
constexpr int kK3Group = PARAPLAN_K3_GROUP;

// Round constants in the compute precision, filled once per snapshot on the
// host and read by the kernels straight from the parameter (constant) bank,
// so they cost no registers.
template <typename Real>
struct alignas(16) ConstsT {
  // The fields a rollout step reads come first, four to a 16-byte group in
  // the order the step uses them, so the FP32 kernels fetch them from the
  // parameter bank with few vector loads (LDCU.128) per iteration.
  Real gx, gy, gcos, gsin;            // goal in the anchor frame (planner.cpp:70-81)
  Real gphi, gv, eps_xi, eps_eta;     // + GoalTolerance
  Real eps_phi, eps_v, dmax, window;  // VehicleParams-derived
  Real l_r, Ts, inv_wb, ts_umid;      // inv_wb: 1 / wheelbase (FP32 path multiplies);
  Real ts_uhalf;                      // ts_umid, ts_uhalf: T_s (umin + umax) / 2, T_s (umax - umin) / 2
  Real bx0, binv, qpad;  // cell grid of the field: origin, 1 / cell size; box query pad: cell / 8
  Real bcx, bhx, hw;     // rectangle centre offset (fe - re)/2, half length (fe + re)/2, half width
  Real dmarg;            // |margin| below which a discrete verdict is "marginal"
  Real dmarg_rel;        // + this x the path so far: the flag band widens with the distance
                         // travelled (the measured relative drift of a rollout's state)
  Real dmarg_floor;      // the band's relative drift is at least this
  int32_t flag_miss;     // several restarts: narrow collision MISSES are marginal too
  int32_t tan_small;     // delta_max <= pi/4: tan by polynomial ratio (FP32)
  // round shape the step reads (copies of RoundArgs values, same group rule)
  int32_t H;             // horizon
  int32_t any_pts;       // field_ns + field_nd > 0
  uint32_t k3_row_bytes;     // kernel kind 3: bytes of one dynamic point row (0: static part)
  uint32_t k3_st_row_bytes;  // kernel kind 3: bytes of one row of cell starts (0: static part)
  Real xtop, ytop;       // grid_nx - 1, grid_ny - 1 (the last cell column / row)
  // the rest: start state, feature scales, FP64-only divisors
  Real v0, act0, pa0;    // initial carry (planner.cpp:123-125)
  Real inv_xi, inv_eta, inv_phi, inv_v;
  Real wb, umin, umax;
  Real fe, re, r2;       // chassis half-planes, squared bounding radius
  Real cull;             // collision x-window half width: bounding radius + 1e-3
  Real by0;              // cell grid origin (y)
  double d_xi, d_eta, d_phi, d_v;  // NormConstants (FP64 path divides)
  double wb_d;           // wheelbase (FP64 path divides, src/dynamics.cpp:52-55)
};

// Byte offsets of the parts of a field image.
struct FieldLayout {
  int64_t dpts, sst, dst, sbox, cst, cbox, bytes;
};

// Everything one sampling round needs. Scalars are FP64 here; the FP32
// kernel rounds them once at kernel entry.
struct RoundArgs {
  // goal in the anchor frame (planner.cpp:70-81)
  double gx, gy, gphi, gv, gcos, gsin;
  // initial carry (planner.cpp:123-125)
  double v0, act0, pa0;
  // NormConstants
  double d_xi, d_eta, d_phi, d_v;
  // GoalTolerance
  double eps_xi, eps_eta, eps_phi, eps_v;
  // VehicleParams-derived
  double delta_max, window, l_r, wheelbase, T_s, u_v_min, u_v_max;
  double fe, re, hw, r2;  // chassis half-planes and squared bounding radius
  // sigma = 10^(lo + u * span)
  double sig_lo, sig_span;
  ConstsT<float> kf;
  ConstsT<double> kd;
  int32_t H;
  int32_t n_points;  // 0 disables the collision test (planner.cpp:74)
  int32_t n_params;
  int32_t n_layers;
  int32_t sizes[kMaxLayers];
  // sampling round: restarts [0, restart_count) of this call, candidates
  // [cand_begin, cand_begin + count) of each restart
  int32_t restart_count;
  int64_t cand_begin;
  int64_t count;
  const uint64_t* key_prefix;  // device [restart_count]: fold^4(seed, t, r, iter)
  const double* center;        // device [n_params]
  const float* center_f;       // device [n_params]: center rounded to float
  const double* injected;      // device [count * n_params] or null (RNG off)
  // Obstacle field image (see csrc/capi/field.hpp): [static pts Real2 x Ns]
  // [dynamic pts Real2 x (H+1) x Nd][static starts int32 x (cells+1)]
  // [dynamic starts int32 x (H+1) x (cells+1)][static cell boxes Real4 x
  // cells, grid_mode 2 only], points in cell order.
  const void* field;
  int32_t field_ns, field_nd;  // static points, dynamic points per row
  int32_t field_dstride;       // points per dynamic row in the image (Nd + sentinels)
  int32_t field_padded;        // the image carries sentinels (kernel kind 3 needs them)
  int32_t grid_nx, grid_ny;    // cells (grid_ny == 1: x-buckets)
  int32_t grid_mode;           // 0 x-buckets, 1 2-D by column, 2 2-D with static cell boxes
  int32_t coop;                // 2-D grids: warps with few live lanes scan windows together
  double grid_x0, grid_y0, grid_g;  // grid origin and cell size (host side)
  FieldLayout lay;             // byte offsets of the compute-precision image
  FieldLayout lay64;           // byte offsets of the FP64 image (field64)
  // scratch / outputs (device)
  Rec* tile_recs;              // restart-major: [r][tile] (lockstep) or [r][CTA] (refill)
  Rec* out;                    // [restart_count]
  uint32_t* counters;          // [2]: tile ticket, done ticket (self-resetting)
  unsigned long long* exec;    // [4]: accumulators (steps, states), published totals
  SampleOut* per_sample;       // [restart_count * count] or null
  float* theta_scratch;        // generic-arch path: [n_params * grid_threads]
  double* theta_scratch64;
  int32_t grid;                // blocks launched (persistent)
  int32_t block;               // threads per block
  int32_t tiles_per_restart;
  int32_t n_tiles;
  int32_t field_smem_bytes;    // 0 = read the field from global/L2
  int32_t queue_bytes;         // unused (0)
  void* theta_buf;             // refill schedule: [P][total] theta in Real
  void* first_buf;             // refill schedule: [2][total] first action in Real
  // near-tie re-ranking (null skeys = off)
  void* skeys;                 // [restart_count * count] SKey (FP64) or SKey32 (FP32)
  int32_t skey32;              // skeys holds SKey32
  // several restarts (refill schedule): the rollout only writes the sample
  // keys, and reduce_keys_kernel forms the per-restart winners from them
  // (lanes crossing restarts would otherwise flush their bests every batch)
  int32_t keys_only;
  // keys_only: per restart also the best candidate NOT flagged marginal; the
  // first window is built around it (flagged candidates are always in the
  // window), so a flagged FP32 winner that the exact arithmetic demotes
  // does not force extra widening passes
  Rec* out_free;
  const void* field64;         // FP64 image of the field (same layout as `field`)
  int64_t* sel_list;           // [kSelFirst] the first selected flat indices (round block)
  int64_t* sel_more;           // [sel_cap - kSelFirst] the rest of them
  const int64_t* ref_list;     // [counters[2]] the members refine_kernel evaluates
  SelRec* sel_out;             // [sel_cap] their FP64 keys
  int32_t sel_cap;             // selection capacity (grown by the host on overflow)
  int32_t refine_grid;
  double sel_rho, sel_alpha;   // window: cost <= best * (1 + rho) + alpha
  double sel_rho2;             // rho of windows anchored on a class-2 (reached) candidate
  int32_t rho2_by_tgoal;       // rho2 grows with the anchor's t_goal (rho2_of)
  double sel_rho2_floor;
  // list rounds (the certification's FP64 re-evaluation of a wide window):
  // item i of the round is the flat candidate list[i] (restart-major over
  // list_count candidates per restart) of the round the list came from; the
  // round itself is one "restart" of count = n items, keys_only
  const int64_t* list;
  int64_t list_count;

  const SelBound* sel_bound;   // null: first pass (window around a.out)
  double dmarg32;              // FP32 marginal threshold (host side, copied into kf)
  int32_t sms;                 // multiprocessors of the device (launch sizing)
  // sharded plan step (one shard of the candidates per GPU): the packed
  // per-restart winners [best x restart_count][best unflagged x
  // restart_count] (keypack.h), reduced across the shards in place by the
  // exchange; select_kernel then anchors each restart's first window on the
  // GLOBAL best unflagged candidate (sel_packed != 0)
  int32_t sel_packed;
  uint64_t* pkeys;
  // goal-horizon cut (kCutTGoal above; null: every rollout runs to its end):
  // goal_cut[r] the earliest t_goal seen so far in restart r (kCutNone: none;
  // a list round has one slot, and is cut only when its list comes from a
  // round of one restart), re-armed by the round's last block after copying
  // slots [0, cut_slots) to cut_pub
  uint32_t* goal_cut;
  uint32_t* cut_pub;
  int32_t cut_slack;
  int32_t cut_slots;
  // refill schedule: a warp writes its finished lanes' keys and refills them
  // every flush_every-th iteration (>= 1), or (flush_min > 0) as soon as
  // flush_min of its lanes wait
  int32_t flush_every;
  int32_t flush_min;
};

// RoundArgs::exec slot of the round's device start stamp (generate_kernel)
constexpr int kExecRoundT0 = 7;

// Architecture dispatch of the specialised kernels.
enum class NetKind : int { kGeneric = 0, k5_2_2 = 1, k5_10_2 = 2, k5_10_10_2 = 3 };
NetKind classify(const int32_t* sizes, int32_t n_layers);

// Grid sizing: persistent blocks = min(n_tiles, SMs x resident blocks/SM).
struct LaunchShape {
  int32_t grid, block, smem_limit;
  int32_t refill;       // 1: refill_kernel (32-candidate batches), 0: lockstep tiles
  int32_t queue_bytes;  // unused (0)
  int32_t theta_elem;   // refill: Real elements per candidate in theta_buf + first_buf
};
// field_bytes = shared-memory image of the field (0 = read from L2).
// Returns 0 or a cudaError_t.
// grid: the field uses the 2-D cell grid (separate kernel instantiation).
// Rollout kernel kind of a field: its grid mode (0 x-buckets, 1 2-D by
// column, 2 2-D with cell boxes), or 3 = x-buckets staged in shared memory
// with a single part (all points static or all dynamic: small mixed clouds
// are made all-dynamic by the binning, csrc/capi/field.cpp kSmall).
#ifndef PARAPLAN_SMEM_FIELD
#define PARAPLAN_SMEM_FIELD 1
#endif
inline int grid_kind(int mode, int field_smem_bytes, int ns, int nd, int padded = 1) {
#if PARAPLAN_SMEM_FIELD
  return mode == 0 && field_smem_bytes > 0 && (ns == 0 || nd == 0) && padded ? 3 : mode;
#else
  return mode;
#endif
}
// `grid` is the kernel kind (grid_kind).
int shape_f32(NetKind k, int device, int field_bytes, int grid, LaunchShape* out);
int shape_f64(NetKind k, int device, int field_bytes, int grid, LaunchShape* out);

// Enqueue one sampling round on `stream` in two stages: the theta generator
// (needs no field), then the rollout (needs the field). Returns 0 or a
// cudaError_t.
int launch_generate_f32(NetKind k, const RoundArgs& a, void* stream);
int launch_generate_f64(NetKind k, const RoundArgs& a, void* stream);
int launch_rollout_f32(NetKind k, const RoundArgs& a, void* stream);
int launch_rollout_f64(NetKind k, const RoundArgs& a, void* stream);

// The device's theta draws of candidates [cand_begin, cand_begin + count) of
// the restart whose key prefix is key_prefix[0] (P Reals each, into `out`).
int launch_draw_f32(const RoundArgs& a, void* out, void* stream);
int launch_draw_f64(const RoundArgs& a, void* out, void* stream);

// Near-tie window after a round: counters[2] receives the number of selected
// candidates, sel_list their flat indices.
int launch_select(const RoundArgs& a, void* stream);
// Packed keys of the round's per-restart winners into a.pkeys (a dependent
// launch after the rollout / per-restart reduction).
int launch_pack_keys(const RoundArgs& a, void* stream);
// Wide-window filter after an FP64 list round (csrc/capi/round.cpp
// certify_round): per source restart, the members' best rank (2 - cls,
// t_goal) and the best cost at that rank; then every member that is flagged
// or within 2 x tol of its restart's best (a superset of the host's FP64
// near-ties, tol = rho of the best's class and t_goal) is appended to `out`.
struct ListPick {
  int64_t flat;  // the member (flat index of the listed round)
  SKey key;      // its FP64 key
};
struct ListFilterArgs {
  const SKey* keys;     // [n] the list round's keys
  const int64_t* list;  // [n] flat indices, restart-major over list_count
  int64_t n, list_count;
  double rho;                // class 0/1 tolerance
  double rho2, rho2_floor;   // class 2: rho2_of(rho2, rho2_floor, t_goal)
  uint32_t* rank;            // [kMaxRestartsPerLaunch] scratch, 0xff..
  unsigned long long* cost;  // [kMaxRestartsPerLaunch] scratch, 0xff..
  uint32_t* count;           // picked members (0 on entry)
  ListPick* out;             // [n]
  int32_t sms;
};
int launch_list_filter(const ListFilterArgs& f, void* stream);
// Copy `bytes` (a multiple of 16) of the device round block into pinned host
// memory with SM stores, after the previous kernel on `stream` (dependent
// launch behind the round's last kernel). Slot kExecRoundT0 of the
// block's exec counters (at `exec_off` bytes) holds the device time the
// round's first kernel started (0: no stamp); the host copy receives the
// round's span in ns there instead, and the device slot is cleared.
int launch_copy_out(const void* src, void* host_dst, size_t bytes, size_t exec_off, void* stream);
// FP64 re-evaluation of the selected candidates into sel_out.
int launch_refine(NetKind k, const RoundArgs& a, void* stream);
// Resident refine_kernel CTAs of 128 threads per SM.
int refine_occupancy(NetKind k);

// Device binning of the dynamic rows of a raw-points field (field.hpp's
// layout): row r of mover k sits at x + r * step (FP64, no contraction: the
// host's positions bit for bit), rounded to the image precision, in the
// cell order of the host's grid. Counts, per-row scan, scatter.
struct BinArgs {
  const double* movers;  // Nd x 4: x, y, step x, step y
  int32_t Nd, rows, nx, ny;
  double x0, y0, inv_g;
  void* dpts;            // rows x Nd: float2 (fp64 == 0) or double2
  int32_t* dst;          // rows x (cells + 1) starts
  int32_t* cursor;       // rows x cells scratch
  int32_t fp64;
  int32_t sms;  // multiprocessors of the device (launch sizing)
};
int bin_movers(const BinArgs& a, void* stream);

// FFMA throughput probe (the FP32 roofline denominator).
int measure_ffma(int device, double* tflops, double* sm_mhz);

}  // namespace ppdev
