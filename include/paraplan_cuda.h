/*
 * paraplan_cuda.h -- the C-ABI boundary of the B200 sampling planner.
 *
 * Plain C: fixed-width PODs, caller-owned buffers, int status codes. No C++,
 * torch or CUDA types cross this boundary. Everything above it (the C++
 * `paraplan::Planner` facade in include/paraplan/planner.hpp, the pybind11
 * module `paraplan._core`, ctypes callers) is a thin wrapper.
 *
 * Entry points and the reference interface each one replaces
 * (paths relative to the reference's proj/ tree):
 *
 *   pp_create / pp_destroy      Planner::Planner / ~Planner
 *                               (src/planner.cpp:46-58, include/paraplan/planner.hpp:90-92)
 *   pp_plan_step                Planner::plan_step        (src/planner.cpp:238-351)
 *   pp_plan_step_points         plan_step of extrapolate(points) (src/mission.cpp:142-158)
 *   pp_rollout                  Planner::rollout          (src/planner.cpp:193-205)
 *   pp_sample_candidate         Planner::sample_candidate (src/planner.cpp:207-226)
 *   pp_perturbation_sigma       Planner::perturbation_sigma (src/planner.cpp:228-236)
 *   pp_evaluate                 one sampling round = evaluate_block over a candidate
 *                               shard + the ordered merge (src/planner.cpp:279-321);
 *                               the unit the multi-GPU path shards
 *   pp_eval_theta               Planner::rollout over an injected theta batch
 *                               (parity / debug path; src/planner.cpp:193-205)
 *   pp_merge_records            ordered merge of shard winners (src/planner.cpp:310-321)
 *   pp_key_better               better(ScoreKey, ScoreKey) (src/planner.cpp:40-44)
 *
 * Error behaviour mirrors the reference: configuration errors that the
 * reference reports with std::invalid_argument come back as
 * PP_INVALID_ARGUMENT with the reference's message in pp_last_error();
 * CUDA failures are PP_CUDA_ERROR. There is no CPU fallback: without a
 * usable sm_100 device pp_create fails with PP_NO_DEVICE.
 */
#ifndef PARAPLAN_CUDA_H_
#define PARAPLAN_CUDA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PP_ABI_VERSION 2
#define PP_MAX_DEVICES 8

typedef enum pp_status {
  PP_OK = 0,
  PP_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  PP_RUNTIME_ERROR = 2,    /* reference: std::runtime_error   */
  PP_CUDA_ERROR = 3,
  PP_NO_DEVICE = 4
} pp_status;

/* Arithmetic of the device sampling pass. The returned plan (best_theta,
 * predicted rollout, action) is always recomputed on the host in FP64 with
 * the reference's expression order, so it is bit-identical to the reference
 * whenever the winning candidate index is. */
typedef enum pp_precision {
  PP_FP32 = 32, /* FP32 rollout; winner window re-ranked in FP64 (see refine) */
  PP_FP64 = 64  /* FP64 rollout on the device */
} pp_precision;

/* VehicleParams (include/paraplan/dynamics.hpp:9-27) */
typedef struct pp_vehicle {
  double l_f, l_r;
  double delta_max, delta_rate_max;
  double u_v_min, u_v_max;
  double overhang_front, overhang_rear, half_width;
  double T_s;
} pp_vehicle;

/* NormConstants (include/paraplan/policy.hpp:34-39) */
typedef struct pp_norm {
  double d_xi, d_eta, d_phi, d_v;
} pp_norm;

/* PlannerConfig + GoalTolerance (include/paraplan/planner.hpp:14-35), plus
 * the device-side knobs that the reference does not have (trailing). */
typedef struct pp_config {
  int32_t H;
  int32_t n_restarts;
  int32_t n_iter_max;
  int32_t n_candidates;
  int32_t n_obst_pts;
  int32_t early_exit; /* bool */
  double eps_xi, eps_eta, eps_phi, eps_v;
  double sigma_log_low, sigma_log_high;
  uint64_t master_seed;
  int32_t threads;   /* accepted and validated; the device path ignores it */
  int32_t precision; /* pp_precision */
  int32_t device;    /* CUDA ordinal */
  int32_t refine;    /* FP32 only: re-rank the near-tie window in FP64 (1 = on) */
  /* Several GPUs in one process (n_devices > 1; else `device` alone): the
   * candidates of every sampling round are split into contiguous shards,
   * shard k on devices[k]; the shard winners (each certified) are merged in
   * shard order, as the reference merges its worker ranges
   * (src/planner.cpp:280-281, 310-321), so the plan is the single-GPU one. */
  int32_t n_devices;
  int32_t devices[PP_MAX_DEVICES];
} pp_config;

/* Planner constructor arguments. layer_sizes is MlpArchitecture::layer_sizes
 * (include/paraplan/policy.hpp:21-27); it is copied by pp_create. */
typedef struct pp_model {
  pp_vehicle vehicle;
  pp_norm norm;
  pp_config config;
  const int32_t* layer_sizes;
  int32_t n_layers;
} pp_model;

/* PlanningSnapshot (include/paraplan/planner.hpp:39-46). field_xy is
 * ExtrapolatedField::positions flattened: (field_H+1) * n_points (x, y)
 * pairs, row-major in h, anchor frame. warm_theta_len == 0 means "start from
 * the zero vector". All pointers are borrowed for the duration of the call. */
typedef struct pp_snapshot {
  double ev_x, ev_y, ev_phi, ev_v;
  double actuator_delta;
  double prev_a0, prev_a1;
  double goal_x, goal_y, goal_phi, goal_v;
  const double* field_xy;
  int32_t field_H;
  int32_t n_points;
  const double* warm_theta;
  int32_t warm_theta_len;
  int32_t _pad;
} pp_snapshot;

/* Snapshot with raw obstacle points instead of an extrapolated field: the
 * anchor-frame points sense() returns (x, y, heading, speed) x n_points. The
 * planner extrapolates them exactly as extrapolate(points, H, T_s)
 * (src/geometry.cpp:43-61) would, so results equal pp_plan_step on that
 * field; static points are stored once and nothing (H+1) x N crosses the
 * boundary. */
typedef struct pp_snapshot_points {
  double ev_x, ev_y, ev_phi, ev_v;
  double actuator_delta;
  double prev_a0, prev_a1;
  double goal_x, goal_y, goal_phi, goal_v;
  const double* points;
  int32_t n_points;
  int32_t _pad;
  double T_s;
  const double* warm_theta;
  int32_t warm_theta_len;
  int32_t _pad2;
} pp_snapshot_points;

/* RolloutResult without the trajectory (include/paraplan/planner.hpp:48-56).
 * steps = dynamics steps simulated (trajectory length - 1). */
typedef struct pp_rollout_stats {
  int32_t reached;
  int32_t t_goal;
  int32_t collided;
  int32_t steps;
  double path_length;
  double terminal_cost;
  double first_a0, first_a1;
} pp_rollout_stats;

/* Winner of one sampling round over a candidate range: ScoreKey
 * (planner.hpp:62-66) + the candidate index within its restart. */
typedef struct pp_record {
  int32_t cls;       /* 2 reached, 1 collision-free, 0 collided; -1 = empty */
  int32_t candidate; /* index within the restart, -1 = empty range */
  int32_t restart;
  int32_t iter;
  double k1, k2;
} pp_record;

/* PlannerOutput (include/paraplan/planner.hpp:71-77) with caller buffers:
 * best_theta holds param_count doubles, trajectory (H+1)*4 doubles
 * (x, y, phi, v per state). */
typedef struct pp_plan_output {
  double* best_theta;
  double* trajectory;
  int32_t trajectory_len; /* out: number of states */
  int32_t success;
  double action_a0, action_a1;
  pp_rollout_stats predicted;
  int64_t evaluated;
  pp_record winner; /* diagnostic: the incumbent key and its (restart, iter, candidate) */
} pp_plan_output;

/* Per-call device accounting (for the benchmark and the roofline). */
typedef struct pp_timing {
  double kernel_ms;        /* device time of the sampling rounds: first kernel start to the
                              result store (%globaltimer; CUDA events around the launches
                              when a round has no generator kernel) */
  int64_t executed_steps;  /* sum over samples of dynamics steps simulated */
  int64_t checked_states;  /* sum over samples of states tested (steps + 1) */
  int64_t samples;         /* candidates evaluated on the device */
  int32_t launches;        /* kernels launched by the call */
  int32_t refined;         /* FP32 candidates re-ranked in FP64 */
  int64_t h2d_bytes, d2h_bytes;
  double certify_ms;       /* host time of the certified re-ranking (wall) */
  double rollout_ms;       /* device span of the rollout kernel alone (%globaltimer,
                              first CTA start to last CTA end) */
  int32_t fp64_rounds;     /* FP32 rounds redone in FP64 (outside the FP32 error
                              envelope, or not certified) */
  int32_t _pad;
} pp_timing;

typedef struct pp_handle pp_handle;

pp_status pp_create(const pp_model* model, pp_handle** out);
void pp_destroy(pp_handle* h);

/* Thread-local message of the last failed call on this thread. */
const char* pp_last_error(void);

int32_t pp_param_count(const pp_handle* h);
int32_t pp_abi_version(void);

/* Planner::plan_step. Uploads the snapshot, runs every sampling round on the
 * device, merges in the reference order and recomputes the plan on the host
 * in FP64. */
pp_status pp_plan_step(pp_handle* h, const pp_snapshot* snap, uint64_t t,
                       pp_plan_output* out);

/* pp_plan_step on a raw-points snapshot (same results as on the
 * extrapolated field); run_mission's tick uses it. */
pp_status pp_plan_step_points(pp_handle* h, const pp_snapshot_points* snap, uint64_t t,
                              pp_plan_output* out);
pp_status pp_upload_points(pp_handle* h, const pp_snapshot_points* snap);

/* Planner::rollout (host FP64, bit-identical to the reference). traj may be
 * NULL; otherwise it holds traj_cap states of 4 doubles. */
pp_status pp_rollout(const pp_handle* h, const pp_snapshot* snap,
                     const double* theta, int32_t theta_len,
                     pp_rollout_stats* out, double* traj, int32_t traj_cap,
                     int32_t* traj_len);

pp_status pp_sample_candidate(const pp_handle* h, const double* center,
                              int32_t len, uint64_t t, int32_t restart,
                              int32_t iter, int32_t candidate, double* out);
/* NaN for a null handle (pp_last_error() says so). */
double pp_perturbation_sigma(const pp_handle* h, uint64_t t, int32_t restart,
                             int32_t iter, int32_t candidate);

/* RNG parity dump: the theta the DEVICE draws for candidates [cand_begin,
 * cand_end) of (t, restart, iter) around `center` (len doubles), as the
 * rollout kernels use them (precision 64: the reference's FP64 draws, equal
 * to pp_sample_candidate; precision 32: the FP32 transform of the same
 * integer stream). out holds (cand_end - cand_begin) x len doubles.
 * Replaces nothing in the reference: the device side of
 * Planner::sample_candidate (planner.hpp:110-113, src/planner.cpp:207-226). */
pp_status pp_draw_theta(pp_handle* h, const double* center, int32_t len, uint64_t t,
                        int32_t restart, int32_t iter, int64_t cand_begin,
                        int64_t cand_end, double* out);

/* Copies the snapshot to the device (pinned staging, one H2D). A NULL
 * snapshot in pp_evaluate reuses the resident one. */
pp_status pp_upload_snapshot(pp_handle* h, const pp_snapshot* snap);

/* One sampling round (iteration `iter`) for restarts
 * [restart_begin, restart_begin + restart_count) over candidates
 * [cand_begin, cand_end) of each restart, centred on `center`
 * (param_count doubles). Writes one winner record per restart.
 * per_sample (optional) receives restart_count * (cand_end - cand_begin)
 * stats, restart-major. */
pp_status pp_evaluate(pp_handle* h, const pp_snapshot* snap, uint64_t t,
                      int32_t iter, int32_t restart_begin,
                      int32_t restart_count, const double* center,
                      int64_t cand_begin, int64_t cand_end, pp_record* out,
                      pp_rollout_stats* per_sample);

/* Device rollout of n injected parameter vectors (row-major n x
 * param_count doubles). No RNG involved: "identical sampled parameters". */
pp_status pp_eval_theta(pp_handle* h, const pp_snapshot* snap,
                        const double* theta, int64_t n,
                        pp_rollout_stats* out);

/* Ordered merge of n records (lowest index wins ties): the reference's
 * worker merge. Empty records (candidate < 0) are skipped. */
pp_status pp_merge_records(const pp_record* recs, int32_t n, pp_record* out);
int32_t pp_key_better(int32_t cls_a, double k1_a, double k2_a, int32_t cls_b,
                      double k1_b, double k2_b);

pp_status pp_last_timing(const pp_handle* h, pp_timing* out);

/* The device stream every kernel of this handle runs on (cudaStream_t). */
void* pp_stream(const pp_handle* h);

/* Number of visible CUDA devices (0 without a GPU; never fails). */
int32_t pp_device_count(void);

/* ---- One process per GPU (torch.distributed / MPI style launch) ----------
 * The candidates of every sampling round are split into contiguous shards,
 * rank r of W owning [n r / W, n (r + 1) / W) of each restart. Each rank
 * evaluates its shard on its own GPU; the per-restart winners are combined by
 * ONE ncclAllReduce(ncclMin, uint64) on a packed (class, t_goal, FP32 cost,
 * index) key (n_candidates <= 2^22, H <= 255; else an all-gather of the
 * records), and the certification's exact keys by an ncclAllGather, so every
 * rank returns the same plan -- the reference's ordered merge of contiguous
 * worker ranges (src/planner.cpp:280-281, 310-321). Every rank calls
 * pp_plan_step / pp_plan_step_points with the same snapshot and t. */
/* Rank 0 makes the NCCL unique id (128 bytes); the caller shares it. */
pp_status pp_comm_unique_id(uint8_t* out128);
/* Joins rank `rank` of a `world`-rank communicator (a one-rank communicator
 * runs the same exchange path on one GPU). */
pp_status pp_comm_init(pp_handle* h, const uint8_t* id128, int32_t world, int32_t rank);
/* The packed key of the winner allreduce (no device needed): smaller is
 * better in the reference's order (better(), src/planner.cpp:40-44), ties to
 * the lower candidate index. cls -1 packs to UINT64_MAX. */
uint64_t pp_pack_key(int32_t cls, int32_t t_goal, float cost, uint32_t candidate);
void pp_unpack_key(uint64_t key, int32_t* cls, int32_t* t_goal, float* cost,
                   uint32_t* candidate);
/* The exchange between the planner's shards: "nccl", "host" (shards of one
 * process sharing a GPU) or "none" (one shard). */
const char* pp_exchange_kind(const pp_handle* h);

/* Measured FP32 FMA throughput of `device` in TFLOP/s (FFMA loop, 2 flop per
 * FMA) -- the roofline denominator of the rollout kernel. */
pp_status pp_measure_fp32_peak(int32_t device, double* tflops, double* sm_mhz);

#ifdef __cplusplus
}
#endif

#endif /* PARAPLAN_CUDA_H_ */
