/*
 * paraplan_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C, FP64 restatement of the reference planner's hot path. Each
 * function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). Built with -ffp-contract=off -fno-math-errno like the
 * reference (src/CMakeLists.txt:15-17) and every expression is evaluated in
 * the reference's order, so results are bit-identical to the reference on the
 * same libm. Pinned by tests/test_oracle.py against oracle/_ref (the reference
 * compiled from its own sources) and tests/golden/*.json.
 *
 * Nothing in the product links this file.
 */
#include "paraplan_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define PO_PI 3.141592653589793
#define PO_MAX_WIDTH 256

/* ---------------------------------------------------------------- RNG --- */
/* src/rng.cpp:9 (golden-ratio increment) */
static const uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

/* src/rng.cpp:11-18: SplitMix64 finaliser */
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* src/rng.cpp:20-22: hash-combine of one key field */
static uint64_t fold(uint64_t h, uint64_t field) {
  return mix64(h ^ (mix64(field) + kGamma + (h << 6) + (h >> 2)));
}

typedef struct {
  uint64_t state;
  double spare;
  int has_spare;
} po_rng;

/* src/rng.cpp:26-35: key order seed -> t -> restart -> iter -> candidate */
static void rng_init(po_rng* g, uint64_t seed, uint64_t t, uint64_t r, uint64_t i,
                     uint64_t c) {
  uint64_t h = mix64(seed + kGamma);
  h = fold(h, t);
  h = fold(h, r);
  h = fold(h, i);
  h = fold(h, c);
  g->state = h;
  g->spare = 0.0;
  g->has_spare = 0;
}

/* src/rng.cpp:37-40 */
static uint64_t rng_u64(po_rng* g) {
  g->state += kGamma;
  return mix64(g->state);
}

/* src/rng.cpp:42-44: 53-bit uniform in [0, 1) */
static double rng_unit(po_rng* g) { return (double)(rng_u64(g) >> 11) * 0x1.0p-53; }

/* src/rng.cpp:46-58: Box-Muller, u1 = 1 - unit first, cos value returned,
 * sin value cached */
static double rng_normal(po_rng* g) {
  double u1, u2, r, t;
  if (g->has_spare) {
    g->has_spare = 0;
    return g->spare;
  }
  u1 = 1.0 - rng_unit(g);
  u2 = rng_unit(g);
  r = sqrt(-2.0 * log(u1));
  t = 2.0 * PO_PI * u2;
  g->spare = r * sin(t);
  g->has_spare = 1;
  return r * cos(t);
}

uint64_t po_rng_draw(uint64_t seed, uint64_t t, uint64_t r, uint64_t i, uint64_t c,
                     int32_t k) {
  po_rng g;
  uint64_t v = 0;
  int32_t j;
  rng_init(&g, seed, t, r, i, c);
  for (j = 0; j <= k; ++j) v = rng_u64(&g);
  return v;
}

void po_rng_stream(uint64_t seed, uint64_t t, uint64_t r, uint64_t i, uint64_t c,
                   int32_t kind, int32_t n, void* out) {
  po_rng g;
  int32_t k;
  rng_init(&g, seed, t, r, i, c);
  for (k = 0; k < n; ++k) {
    if (kind == 0) {
      ((uint64_t*)out)[k] = rng_u64(&g);
    } else if (kind == 1) {
      ((double*)out)[k] = rng_unit(&g);
    } else {
      ((double*)out)[k] = rng_normal(&g);
    }
  }
}

/* ------------------------------------------------------- validation --- */
/* src/policy.cpp:28-34 */
int32_t po_param_count(const pp_model* m) {
  int32_t total = 0, l;
  for (l = 0; l + 1 < m->n_layers; ++l) {
    total += (m->layer_sizes[l] + 1) * m->layer_sizes[l + 1];
  }
  return total;
}

#define PO_FAIL(text)                          \
  do {                                         \
    if (msg) snprintf(msg, cap, "%s", text);   \
    return 1;                                  \
  } while (0)

/* src/dynamics.cpp:9-28, src/planner.cpp:12-25, src/policy.cpp:11-26 */
int po_validate(const pp_model* m, char* msg, int32_t cap) {
  const pp_vehicle* v = &m->vehicle;
  const pp_config* c = &m->config;
  int32_t l;
  if (m->n_layers < 2) PO_FAIL("architecture needs at least 2 layers");
  if (m->layer_sizes[0] != 5) PO_FAIL("input layer must have 5 units");
  if (m->layer_sizes[m->n_layers - 1] != 2) PO_FAIL("output layer must have 2 units");
  for (l = 0; l < m->n_layers; ++l) {
    if (m->layer_sizes[l] <= 0 || m->layer_sizes[l] > PO_MAX_WIDTH) {
      PO_FAIL("layer sizes must be in [1, 256]");
    }
  }
  if (!(v->l_f > 0.0) || !(v->l_r > 0.0)) PO_FAIL("axle distances must be positive");
  if (!(v->delta_max > 0.0 && v->delta_max < PO_PI / 2.0)) {
    PO_FAIL("delta_max must lie in (0, pi/2)");
  }
  if (!(v->delta_rate_max > 0.0)) PO_FAIL("delta_rate_max must be positive");
  if (!(v->u_v_min < 0.0 && 0.0 < v->u_v_max)) {
    PO_FAIL("acceleration range must straddle zero");
  }
  if (!(v->overhang_front >= 0.0 && v->overhang_rear >= 0.0 && v->half_width > 0.0)) {
    PO_FAIL("chassis dimensions out of range");
  }
  if (!(v->T_s > 0.0)) PO_FAIL("T_s must be positive");
  if (c->H < 1) PO_FAIL("H must be >= 1");
  if (c->n_candidates < 1) PO_FAIL("n must be >= 1");
  if (c->n_restarts < 1) PO_FAIL("N_restarts must be >= 1");
  if (c->n_iter_max < 1) PO_FAIL("N_iter_max must be >= 1");
  if (c->n_obst_pts < 0) PO_FAIL("N_obstPts must be >= 0");
  if (c->threads < 1) PO_FAIL("threads must be >= 1");
  if (!(c->sigma_log_low <= c->sigma_log_high)) PO_FAIL("sigma range must be ordered");
  if (!(c->eps_xi > 0 && c->eps_eta > 0 && c->eps_phi > 0 && c->eps_v > 0)) {
    PO_FAIL("goal tolerances must be positive");
  }
  return 0;
}

/* ------------------------------------------------------- candidates --- */
/* src/planner.cpp:207-226: candidate 0 is the centre; otherwise sigma is the
 * first draw (10^U(lo, hi)) and each coordinate adds sigma * N(0, 1). */
void po_sample_candidate(const pp_model* m, const double* center, uint64_t t,
                         int32_t restart, int32_t iter, int32_t cand, double* out) {
  const int32_t np = po_param_count(m);
  const double lo = m->config.sigma_log_low, hi = m->config.sigma_log_high;
  po_rng g;
  double sigma;
  int32_t i;
  if (cand == 0) {
    memcpy(out, center, sizeof(double) * (size_t)np);
    return;
  }
  rng_init(&g, m->config.master_seed, t, (uint64_t)restart, (uint64_t)iter,
           (uint64_t)cand);
  sigma = pow(10.0, lo + rng_unit(&g) * (hi - lo));
  for (i = 0; i < np; ++i) out[i] = center[i] + sigma * rng_normal(&g);
}

/* ---------------------------------------------------------- rollout --- */
/* src/geometry.cpp:9-13 */
static double wrap(double a) {
  const double r = remainder(a, 2.0 * PO_PI);
  return r <= -PO_PI ? r + 2.0 * PO_PI : r;
}

static double clampd(double v, double lo, double hi) {
  return v < lo ? lo : (hi < v ? hi : v); /* std::clamp semantics */
}

/* src/policy.cpp:53-80 (tanh on every layer, accumulation b + sum_i w_i x_i
 * in ascending i) */
static void mlp(const pp_model* m, const double* theta, const double s[5], double* a0,
                double* a1) {
  double buf[2][PO_MAX_WIDTH];
  int cur = 0;
  size_t off = 0;
  int32_t l, o, i;
  for (i = 0; i < 5; ++i) buf[0][i] = s[i];
  for (l = 0; l + 1 < m->n_layers; ++l) {
    const int32_t nin = m->layer_sizes[l], nout = m->layer_sizes[l + 1];
    const double* w = theta + off;
    const double* b = w + (size_t)nin * nout;
    for (o = 0; o < nout; ++o) {
      double acc = b[o];
      for (i = 0; i < nin; ++i) acc += w[(size_t)o * nin + i] * buf[cur][i];
      buf[1 - cur][o] = tanh(acc);
    }
    off += (size_t)(nin + 1) * nout;
    cur = 1 - cur;
  }
  *a0 = buf[cur][0];
  *a1 = buf[cur][1];
}

typedef struct {
  double gx, gy, gphi, gv, gcos, gsin;
} po_goal;

/* src/geometry.cpp:15-21 + src/planner.cpp:70-73: goal in the anchor frame,
 * heading difference left unwrapped */
static po_goal goal_in_anchor(const pp_snapshot* s) {
  po_goal g;
  const double dx = s->goal_x - s->ev_x, dy = s->goal_y - s->ev_y;
  const double c = cos(s->ev_phi), sn = sin(s->ev_phi);
  g.gx = c * dx + sn * dy;
  g.gy = -sn * dx + c * dy;
  g.gphi = s->goal_phi - s->ev_phi;
  g.gv = s->goal_v;
  g.gcos = cos(g.gphi); /* src/planner.cpp:80-81 */
  g.gsin = sin(g.gphi);
  return g;
}

/* src/planner.cpp:116-121 == src/policy.cpp:36-46 */
static void features(const pp_model* m, const po_goal* g, const double z[4],
                     double prev_a0, double s[5]) {
  s[0] = (g->gx - z[0]) / m->norm.d_xi;
  s[1] = (g->gy - z[1]) / m->norm.d_eta;
  s[2] = wrap(g->gphi - z[2]) / m->norm.d_phi;
  s[3] = (g->gv - z[3]) / m->norm.d_v;
  s[4] = prev_a0;
}

/* src/geometry.cpp:30-41 (rectangle half-planes, bounding radius) and
 * :63-76 (prefilter dx^2+dy^2 >= r^2 skips; strict containment) */
static int collides(const pp_model* m, double x, double y, double phi, const double* pts,
                    int32_t n) {
  const pp_vehicle* v = &m->vehicle;
  const double fe = v->l_f + v->overhang_front, re = v->l_r + v->overhang_rear;
  const double hw = v->half_width;
  const double radius = hypot(fe > re ? fe : re, hw);
  const double r2 = radius * radius;
  const double c = cos(phi), s = sin(phi);
  const double planes[4][3] = {{1.0, 0.0, fe}, {-1.0, 0.0, re}, {0.0, 1.0, hw}, {0.0, -1.0, hw}};
  int32_t j, k;
  for (j = 0; j < n; ++j) {
    const double dx = pts[2 * j] - x, dy = pts[2 * j + 1] - y;
    double bx, by;
    int inside = 1;
    if (dx * dx + dy * dy >= r2) continue;
    bx = c * dx + s * dy;
    by = -s * dx + c * dy;
    for (k = 0; k < 4; ++k) {
      if (!(planes[k][0] * bx + planes[k][1] * by < planes[k][2])) {
        inside = 0;
        break;
      }
    }
    if (inside) return 1;
  }
  return 0;
}

/* src/planner.cpp:66-191 (simulate): per state h, collision first (only when
 * the field has points), then the inclusive goal box in the goal frame, then
 * the horizon stop, then network -> map_controls -> explicit Euler. */
void po_rollout(const pp_model* m, const pp_snapshot* s, const double* theta,
                pp_rollout_stats* out, double* traj, int32_t* traj_len) {
  const pp_vehicle* v = &m->vehicle;
  const pp_config* cfg = &m->config;
  const po_goal g = goal_in_anchor(s);
  const double window = v->delta_rate_max * v->T_s;
  const double wheelbase = v->l_f + v->l_r;
  double z[4] = {0.0, 0.0, 0.0, s->ev_v};
  double act = s->actuator_delta, prev_a0 = s->prev_a0;
  double feat[5], a0, a1, f0, f1;
  int32_t h, n_traj = 0;

  memset(out, 0, sizeof(*out));
  out->t_goal = -1;
  if (traj) memcpy(traj + 4 * n_traj, z, sizeof(z));
  ++n_traj;

  features(m, &g, z, prev_a0, feat); /* :130-132 first action before the loop */
  mlp(m, theta, feat, &f0, &f1);
  out->first_a0 = f0;
  out->first_a1 = f1;

  for (h = 0;; ++h) {
    if (s->n_points > 0 &&
        collides(m, z[0], z[1], z[2], s->field_xy + (size_t)2 * h * s->n_points,
                 s->n_points)) {
      out->collided = 1;
      break;
    }
    {
      const double gdx = g.gx - z[0], gdy = g.gy - z[1];
      if (fabs(g.gcos * gdx + g.gsin * gdy) <= cfg->eps_xi &&
          fabs(-g.gsin * gdx + g.gcos * gdy) <= cfg->eps_eta &&
          fabs(wrap(g.gphi - z[2])) <= cfg->eps_phi && fabs(g.gv - z[3]) <= cfg->eps_v) {
        out->reached = 1;
        out->t_goal = h;
        break;
      }
    }
    if (h == cfg->H) break;

    if (h == 0) {
      a0 = f0;
      a1 = f1;
    } else {
      features(m, &g, z, prev_a0, feat);
      mlp(m, theta, feat, &a0, &a1);
    }
    {
      /* map_controls (src/dynamics.cpp:30-43) */
      const double c0 = clampd(a0, -1.0, 1.0), c1 = clampd(a1, -1.0, 1.0);
      double delta = clampd(v->delta_max * c0, act - window, act + window);
      double w, u_v, tan_d, tb, c, sn, nx, ny, nphi, nv, dx, dy;
      delta = clampd(delta, -v->delta_max, v->delta_max);
      w = 0.5 * (c1 + 1.0);
      u_v = (1.0 - w) * v->u_v_min + w * v->u_v_max;
      /* explicit Euler, kinematic bicycle (src/dynamics.cpp:45-62) */
      tan_d = tan(delta);
      tb = v->l_r * tan_d / wheelbase;
      c = cos(z[2]);
      sn = sin(z[2]);
      nx = z[0] + v->T_s * z[3] * (c - tb * sn);
      ny = z[1] + v->T_s * z[3] * (sn + tb * c);
      nphi = z[2] + v->T_s * z[3] * tan_d / wheelbase;
      nv = z[3] + v->T_s * u_v;
      dx = nx - z[0];
      dy = ny - z[1];
      out->path_length += sqrt(dx * dx + dy * dy); /* :177-179 */
      z[0] = nx;
      z[1] = ny;
      z[2] = nphi;
      z[3] = nv;
      act = delta;  /* realised steering (:181) */
      prev_a0 = a0; /* raw network output (:182) */
    }
    if (traj) memcpy(traj + 4 * n_traj, z, sizeof(z));
    ++n_traj;
  }
  /* :186-189 */
  out->terminal_cost = fabs(g.gx - z[0]) / m->norm.d_xi + fabs(g.gy - z[1]) / m->norm.d_eta +
                       fabs(wrap(g.gphi - z[2])) / m->norm.d_phi +
                       fabs(g.gv - z[3]) / m->norm.d_v;
  out->steps = n_traj - 1;
  if (traj_len) *traj_len = n_traj;
}

/* ------------------------------------------------------------ score --- */
typedef struct {
  int32_t cls;
  double k1, k2;
} po_key;

/* src/planner.cpp:27-38 */
static po_key score(const pp_rollout_stats* r) {
  po_key k;
  k.cls = r->collided ? 0 : (r->reached ? 2 : 1);
  if (k.cls == 2) {
    k.k1 = -(double)r->t_goal;
    k.k2 = -r->path_length;
  } else {
    k.k1 = -r->terminal_cost;
    k.k2 = 0.0;
  }
  return k;
}

/* src/planner.cpp:40-44 */
int32_t po_better(int32_t cls_a, double k1_a, double k2_a, int32_t cls_b, double k1_b,
                  double k2_b) {
  if (cls_a != cls_b) return cls_a > cls_b;
  if (k1_a != k1_b) return k1_a > k1_b;
  return k2_a > k2_b;
}

void po_eval_candidates(const pp_model* m, const pp_snapshot* s, uint64_t t, int32_t iter,
                        int32_t restart, const double* center, int64_t c_begin,
                        int64_t c_end, pp_rollout_stats* out) {
  po_eval_candidates_mt(m, s, t, iter, restart, center, c_begin, c_end, 1, out);
}

/* Per-candidate stats are independent of the worker split (each candidate
 * is its own sample_candidate + rollout), so any thread count gives the same
 * bits. */
void po_eval_candidates_mt(const pp_model* m, const pp_snapshot* s, uint64_t t, int32_t iter,
                           int32_t restart, const double* center, int64_t c_begin,
                           int64_t c_end, int32_t threads, pp_rollout_stats* out) {
  const int32_t np = po_param_count(m);
  const int32_t workers = threads < 1 ? 1 : threads;
  int64_t c;
#pragma omp parallel num_threads(workers) if (workers > 1)
  {
    double* theta = (double*)malloc(sizeof(double) * (size_t)np);
#pragma omp for schedule(dynamic, 64)
    for (c = c_begin; c < c_end; ++c) {
      po_sample_candidate(m, center, t, restart, iter, (int32_t)c, theta);
      po_rollout(m, s, theta, &out[c - c_begin], NULL, NULL);
    }
    free(theta);
  }
}

typedef struct {
  po_key key;
  int32_t cand;
  int32_t any_free;
} po_local;

/* src/planner.cpp:279-301: one worker's contiguous block, strict better */
static po_local eval_block(const pp_model* m, const pp_snapshot* s, uint64_t t,
                           int32_t restart, int32_t iter, const double* center,
                           int32_t begin, int32_t end, double* theta) {
  po_local loc;
  int32_t c;
  loc.cand = -1;
  loc.any_free = 0;
  loc.key.cls = 0;
  loc.key.k1 = loc.key.k2 = 0.0;
  for (c = begin; c < end; ++c) {
    pp_rollout_stats st;
    po_key k;
    po_sample_candidate(m, center, t, restart, iter, c, theta);
    po_rollout(m, s, theta, &st, NULL, NULL);
    k = score(&st);
    loc.any_free = loc.any_free || !st.collided;
    if (loc.cand < 0 || po_better(k.cls, k.k1, k.k2, loc.key.cls, loc.key.k1, loc.key.k2)) {
      loc.key = k;
      loc.cand = c;
    }
  }
  return loc;
}

/* src/planner.cpp:238-351 */
int po_plan_step(const pp_model* m, const pp_snapshot* s, uint64_t t, int32_t threads,
                 pp_plan_output* out) {
  const pp_config* cfg = &m->config;
  const pp_vehicle* v = &m->vehicle;
  const int32_t np = po_param_count(m);
  const int32_t n = cfg->n_candidates;
  const int32_t workers = threads < 1 ? 1 : threads;
  double* init_center = (double*)calloc((size_t)np, sizeof(double));
  double* center = (double*)malloc(sizeof(double) * (size_t)np);
  double* best_theta = (double*)calloc((size_t)np, sizeof(double));
  po_local* locals = (po_local*)malloc(sizeof(po_local) * (size_t)workers);
  po_key best_key;
  int best_valid = 0, any_free = 0;
  int64_t evaluated = 0;
  int32_t restart, iter, w, traj_len = 0;
  int32_t win_r = -1, win_i = -1, win_c = -1;

  best_key.cls = 0;
  best_key.k1 = best_key.k2 = 0.0;
  if (s->warm_theta_len != 0 && s->warm_theta_len != np) {
    free(init_center);
    free(center);
    free(best_theta);
    free(locals);
    return 1; /* "warm start vector size mismatch" (:240-244) */
  }
  if (s->warm_theta_len == np) memcpy(init_center, s->warm_theta, sizeof(double) * (size_t)np);

  for (restart = 0; restart < cfg->n_restarts; ++restart) {
    for (iter = 0; iter < cfg->n_iter_max; ++iter) {
      po_local merged;
      /* :273-277 every restart re-centres on the warm start; iterations climb
       * on the incumbent */
      if (iter == 0) {
        memcpy(center, init_center, sizeof(double) * (size_t)np);
      } else if (best_valid) {
        memcpy(center, best_theta, sizeof(double) * (size_t)np);
      }
#pragma omp parallel for num_threads(workers) schedule(static, 1) if (workers > 1)
      for (w = 0; w < workers; ++w) {
        const int32_t begin = (int32_t)((int64_t)n * w / workers);
        const int32_t end = (int32_t)((int64_t)n * (w + 1) / workers);
        double* theta = (double*)malloc(sizeof(double) * (size_t)np);
        locals[w] = eval_block(m, s, t, restart, iter, center, begin, end, theta);
        free(theta);
      }
      evaluated += n;
      /* :310-321 ordered merge */
      merged.cand = -1;
      merged.any_free = 0;
      merged.key = best_key;
      for (w = 0; w < workers; ++w) {
        if (locals[w].cand < 0) continue;
        merged.any_free = merged.any_free || locals[w].any_free;
        if (merged.cand < 0 || po_better(locals[w].key.cls, locals[w].key.k1, locals[w].key.k2,
                                         merged.key.cls, merged.key.k1, merged.key.k2)) {
          merged.key = locals[w].key;
          merged.cand = locals[w].cand;
        }
      }
      any_free = any_free || merged.any_free;
      /* :324-330 strict comparison keeps the earlier incumbent */
      if (!best_valid || po_better(merged.key.cls, merged.key.k1, merged.key.k2, best_key.cls,
                                   best_key.k1, best_key.k2)) {
        po_sample_candidate(m, center, t, restart, iter, merged.cand, best_theta);
        best_key = merged.key;
        best_valid = 1;
        win_r = restart;
        win_i = iter;
        win_c = merged.cand;
      }
      if (cfg->early_exit && best_valid && best_key.cls == 2) goto done; /* :332-334 */
    }
  }
done:
  /* :339-350 FP64 epilogue on the winner */
  out->evaluated = evaluated;
  if (out->best_theta) memcpy(out->best_theta, best_theta, sizeof(double) * (size_t)np);
  po_rollout(m, s, best_theta, &out->predicted, out->trajectory, &traj_len);
  out->trajectory_len = traj_len;
  out->success = out->predicted.reached && !out->predicted.collided;
  if (any_free) {
    out->action_a0 = out->predicted.first_a0;
    out->action_a1 = out->predicted.first_a1;
  } else {
    out->action_a0 = s->actuator_delta / v->delta_max;
    out->action_a1 = -1.0;
  }
  out->winner.cls = best_key.cls;
  out->winner.k1 = best_key.k1;
  out->winner.k2 = best_key.k2;
  out->winner.restart = win_r;
  out->winner.iter = win_i;
  out->winner.candidate = win_c;
  free(init_center);
  free(center);
  free(best_theta);
  free(locals);
  return 0;
}
