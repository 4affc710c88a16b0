/*
 * paraplan_oracle.h -- TEST INFRASTRUCTURE: a plain-C, FP64, CPU restatement
 * of the reference planner's hot path (Planner::plan_step and the functions
 * under it), used only as the parity checker by tests/, __graft_entry__.smoke()
 * and bench.py's CPU-baseline leg. The product never links or calls it.
 *
 * Parity of this restatement is pinned against the reference compiled from
 * its own sources (oracle/_ref/libparaplan_ref.so, see oracle/Makefile) and
 * against the golden vectors committed under tests/golden/.
 */
#ifndef PARAPLAN_ORACLE_H_
#define PARAPLAN_ORACLE_H_

#include <stdint.h>

#include "paraplan_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

uint64_t po_rng_draw(uint64_t seed, uint64_t t, uint64_t r, uint64_t i, uint64_t c,
                     int32_t k);
void po_rng_stream(uint64_t seed, uint64_t t, uint64_t r, uint64_t i, uint64_t c,
                   int32_t kind, int32_t n, void* out);

int32_t po_param_count(const pp_model* m);
int po_validate(const pp_model* m, char* msg, int32_t cap);

void po_sample_candidate(const pp_model* m, const double* center, uint64_t t,
                         int32_t restart, int32_t iter, int32_t cand, double* out);

/* traj may be NULL; otherwise it holds H+1 states of 4 doubles. */
void po_rollout(const pp_model* m, const pp_snapshot* s, const double* theta,
                pp_rollout_stats* out, double* traj, int32_t* traj_len);

void po_eval_candidates(const pp_model* m, const pp_snapshot* s, uint64_t t,
                        int32_t iter, int32_t restart, const double* center,
                        int64_t c_begin, int64_t c_end, pp_rollout_stats* out);
void po_eval_candidates_mt(const pp_model* m, const pp_snapshot* s, uint64_t t,
                           int32_t iter, int32_t restart, const double* center,
                           int64_t c_begin, int64_t c_end, int32_t threads,
                           pp_rollout_stats* out);

/* threads > 1 uses OpenMP over contiguous candidate blocks with the
 * reference's ordered merge (bit-identical to threads == 1). */
int po_plan_step(const pp_model* m, const pp_snapshot* s, uint64_t t,
                 int32_t threads, pp_plan_output* out);

int32_t po_better(int32_t cls_a, double k1_a, double k2_a, int32_t cls_b,
                  double k1_b, double k2_b);

#ifdef __cplusplus
}
#endif

#endif
