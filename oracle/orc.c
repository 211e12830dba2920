/* orc.c -- fp64 scalar CPU ORACLE (test infrastructure only; see orc.h).
 *
 * Plain, slow, obviously-correct loops.  No blocking, no bounding spheres,
 * no early-exit reordering beyond what the definitions state.  FK is a chain
 * product of 4x4 homogeneous matrices (a different formulation from the GPU's
 * 3x4 affine updates).
 */
#include "orc.h"

#define ORC_MAX_DOF 64
/* per-robot stride of the configuration buffers: room for the longest chain (reading c.9:
 * one joint value per joint; the ABI allows MRV_MAX_DOF = 16 joints) */
#define ORC_QSTRIDE ORC_MAX_DOF

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* 4x4 homogeneous matrices                                           */
/* ------------------------------------------------------------------ */

typedef struct { double a[4][4]; } mat4;

static mat4 mat4_identity(void) {
  mat4 m;
  memset(&m, 0, sizeof m);
  for (int i = 0; i < 4; ++i) m.a[i][i] = 1.0;
  return m;
}

/* row-major 3x4 fp32 (the input table layout) -> 4x4 double */
static mat4 mat4_from_3x4(const float* p) {
  mat4 m = mat4_identity();
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 4; ++j) m.a[i][j] = (double)p[4 * i + j];
  return m;
}

static mat4 mat4_mul(const mat4* x, const mat4* y) {
  mat4 r;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      double s = 0.0;
      for (int k = 0; k < 4; ++k) s += x->a[i][k] * y->a[k][j];
      r.a[i][j] = s;
    }
  return r;
}

static mat4 mat4_rotz(double th) {
  mat4 m = mat4_identity();
  m.a[0][0] = cos(th); m.a[0][1] = -sin(th);
  m.a[1][0] = sin(th); m.a[1][1] = cos(th);
  return m;
}

static mat4 mat4_transz(double d) {
  mat4 m = mat4_identity();
  m.a[2][3] = d;
  return m;
}

static void mat4_apply(const mat4* m, const double* o, double* out) {
  for (int i = 0; i < 3; ++i) out[i] = m->a[i][0] * o[0] + m->a[i][1] * o[1] + m->a[i][2] * o[2] + m->a[i][3];
}

/* Rotation of a (not necessarily unit) quaternion (w, x, y, z), s = 2/(q.q)
 * (reading c.8). */
static mat4 mat4_from_pose_quat(const double* p, const double* q) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  double s = 2.0 / (w * w + x * x + y * y + z * z);
  mat4 m = mat4_identity();
  m.a[0][0] = 1.0 - s * (y * y + z * z); m.a[0][1] = s * (x * y - w * z);       m.a[0][2] = s * (x * z + w * y);
  m.a[1][0] = s * (x * y + w * z);       m.a[1][1] = 1.0 - s * (x * x + z * z); m.a[1][2] = s * (y * z - w * x);
  m.a[2][0] = s * (x * z - w * y);       m.a[2][1] = s * (y * z + w * x);       m.a[2][2] = 1.0 - s * (x * x + y * y);
  m.a[0][3] = p[0]; m.a[1][3] = p[1]; m.a[2][3] = p[2];
  return m;
}

/* ------------------------------------------------------------------ */
/* Interpolation (reading c.4; slerp reading c.8)                      */
/* ------------------------------------------------------------------ */

static int32_t motion_T(const orc_scene* sc, const orc_motions* mo, int64_t m) {
  if (mo->robot_timesteps) {
    int32_t T = 1;
    for (int r = 0; r < sc->n_robots; ++r)
      if (mo->robot_timesteps[m * sc->n_robots + r] > T) T = mo->robot_timesteps[m * sc->n_robots + r];
    return T;
  }
  return mo->n_timesteps ? mo->n_timesteps[m] : mo->fixed_timesteps;
}

static int32_t robot_T(const orc_scene* sc, const orc_motions* mo, int64_t m, int32_t r) {
  return mo->robot_timesteps ? mo->robot_timesteps[m * sc->n_robots + r] : motion_T(sc, mo, m);
}

static const float* wp_ptr(const orc_scene* sc, const orc_motions* mo, int64_t m, int32_t r, int32_t k) {
  return mo->waypoints + (((m * sc->n_robots + r) * (int64_t)mo->K + k) * mo->S);
}

void orc_interp(const orc_scene* sc, const orc_motions* mo, int64_t m, int32_t r, int32_t t, double* q) {
  const orc_robot* rb = &sc->robots[r];
  const int32_t T = robot_T(sc, mo, m, r), K = mo->K, dof = rb->dof;
  if (t > T - 1) t = T - 1;   /* stay at the goal after the robot's own path ends */
  if (T == 1 || K == 1) {
    const float* w = wp_ptr(sc, mo, m, r, 0);
    for (int d = 0; d < dof; ++d) q[d] = (double)w[d];
    return;
  }
  /* knot k sits at t_k = k (T-1)/(K-1): integer segment select, exact at knots */
  const int64_t num = (int64_t)t * (K - 1);
  const int64_t seg = num / (T - 1), rem = num % (T - 1);
  const float* w0 = wp_ptr(sc, mo, m, r, (int32_t)seg);
  if (rem == 0) {
    for (int d = 0; d < dof; ++d) q[d] = (double)w0[d];
    return;
  }
  const float* w1 = wp_ptr(sc, mo, m, r, (int32_t)seg + 1);
  const double u = (double)rem / (double)(T - 1);
  const int nlin = rb->kind == ORC_SE3 ? 3 : dof;
  for (int d = 0; d < nlin; ++d) q[d] = (double)w0[d] + u * ((double)w1[d] - (double)w0[d]);
  if (rb->kind == ORC_SE3) {
    double a[4], b[4], dm = 0.0, dp = 0.0;
    for (int d = 0; d < 4; ++d) {
      a[d] = w0[3 + d];
      b[d] = w1[3 + d];
      dm += (b[d] - a[d]) * (b[d] - a[d]);
      dp += (b[d] + a[d]) * (b[d] + a[d]);
    }
    const double om = 2.0 * atan2(sqrt(dm), sqrt(dp));
    const double so = sin(om);
    double ca, cb;
    if (so < 1e-6) {
      ca = 1.0 - u; cb = u;
    } else {
      ca = sin((1.0 - u) * om) / so; cb = sin(u * om) / so;
    }
    for (int d = 0; d < 4; ++d) q[3 + d] = ca * a[d] + cb * b[d];
  }
}

/* ------------------------------------------------------------------ */
/* Forward kinematics (reading c.9)                      */
/* ------------------------------------------------------------------ */

void orc_fk(const orc_robot* rb, const double* q, double* xyz) {
  if (rb->kind == ORC_CHAIN) {
    mat4 frames[ORC_MAX_DOF];
    mat4 T = rb->base ? mat4_from_3x4(rb->base) : mat4_identity();
    for (int j = 0; j < rb->dof; ++j) {
      mat4 O = mat4_from_3x4(rb->joint_origin + 12 * j);
      mat4 J = rb->joint_type[j] == 1 ? mat4_transz(q[j]) : mat4_rotz(q[j]);
      mat4 TO = mat4_mul(&T, &O);
      T = mat4_mul(&TO, &J);
      frames[j] = T;
    }
    for (int k = 0; k < rb->n_spheres; ++k) {
      double o[3] = {rb->sphere[4 * k], rb->sphere[4 * k + 1], rb->sphere[4 * k + 2]};
      mat4_apply(&frames[rb->sphere_link[k]], o, xyz + 3 * k);
    }
    return;
  }
  mat4 H;
  if (rb->kind == ORC_SE2) {
    H = mat4_rotz(q[2]);
    H.a[0][3] = q[0];
    H.a[1][3] = q[1];
  } else {
    H = mat4_from_pose_quat(q, q + 3);
  }
  for (int k = 0; k < rb->n_spheres; ++k) {
    double o[3] = {rb->sphere[4 * k], rb->sphere[4 * k + 1], rb->sphere[4 * k + 2]};
    mat4_apply(&H, o, xyz + 3 * k);
  }
}

static int total_spheres(const orc_scene* sc) {
  int n = 0;
  for (int r = 0; r < sc->n_robots; ++r) n += sc->robots[r].n_spheres;
  return n;
}

static void centres_from_configs(const orc_scene* sc, const double* qall /* [n][ORC_QSTRIDE] */, double* xyz) {
  int off = 0;
  for (int r = 0; r < sc->n_robots; ++r) {
    orc_fk(&sc->robots[r], qall + ORC_QSTRIDE * r, xyz + 3 * off);
    off += sc->robots[r].n_spheres;
  }
}

void orc_centres_at(const orc_scene* sc, const orc_motions* mo, int64_t m, int32_t t, double* xyz) {
  double* qall = (double*)malloc(sizeof(double) * ORC_QSTRIDE * (size_t)sc->n_robots);
  for (int r = 0; r < sc->n_robots; ++r) orc_interp(sc, mo, m, r, t, qall + ORC_QSTRIDE * r);
  centres_from_configs(sc, qall, xyz);
  free(qall);
}

/* ------------------------------------------------------------------ */
/* Collision predicates (strict, reading c.1/c.2) and separations       */
/* ------------------------------------------------------------------ */

/* sphere c (radius r) vs sphere o (radius R): strict overlap d^2 < (r+R)^2 */
static int sph_sph(const double* c, double r, const double* o, double R, double* sep) {
  const double dx = c[0] - o[0], dy = c[1] - o[1], dz = c[2] - o[2];
  const double d2 = dx * dx + dy * dy + dz * dz, rs = r + R;
  if (sep) *sep = sqrt(d2) - rs;
  return d2 < rs * rs;
}

/* sphere c (radius r) vs AABB [lo, hi]: e_k = max(lo_k - c_k, 0, c_k - hi_k),
 * strict overlap sum e_k^2 < r^2 */
static int sph_box(const double* c, double r, const float* box, double* sep) {
  double s = 0.0;
  for (int k = 0; k < 3; ++k) {
    double e = 0.0;
    if ((double)box[k] - c[k] > e) e = (double)box[k] - c[k];
    if (c[k] - (double)box[3 + k] > e) e = c[k] - (double)box[3 + k];
    s += e * e;
  }
  if (sep) *sep = sqrt(s) - r;
  return s < r * r;
}

/* robot r (centres at xyz_r) vs environment (mode & ORC_ENV_OBSTACLES) and vs
 * itself on its self-collision link pairs (mode & ORC_ENV_SELF); returns strict hit,
 * min sep */
static int env_eval_mode(const orc_scene* sc, int r, const double* xyz_r, double* min_sep, int want_sep, int mode) {
  const orc_robot* rb = &sc->robots[r];
  int hit = 0;
  double ms = INFINITY, sep;
  if (mode & ORC_ENV_OBSTACLES) {
    for (int k = 0; k < rb->n_spheres; ++k) {
      const double rad = rb->sphere[4 * k + 3];
      for (int o = 0; o < sc->n_obs_spheres; ++o) {
        double oc[3] = {sc->obs_spheres[4 * o], sc->obs_spheres[4 * o + 1], sc->obs_spheres[4 * o + 2]};
        if (sph_sph(xyz_r + 3 * k, rad, oc, sc->obs_spheres[4 * o + 3], want_sep ? &sep : NULL)) hit = 1;
        if (want_sep && sep < ms) ms = sep;
        if (hit && !want_sep) return 1;
      }
      for (int b = 0; b < sc->n_boxes; ++b) {
        if (sph_box(xyz_r + 3 * k, rad, sc->boxes + 6 * b, want_sep ? &sep : NULL)) hit = 1;
        if (want_sep && sep < ms) ms = sep;
        if (hit && !want_sep) return 1;
      }
    }
  }
  if (mode & ORC_ENV_SELF) {
    for (int p = 0; p < rb->n_self_pairs; ++p) {
      const int la = rb->self_pairs[2 * p], lb = rb->self_pairs[2 * p + 1];
      for (int k = 0; k < rb->n_spheres; ++k) {
        if (rb->sphere_link[k] != la) continue;
        for (int l = 0; l < rb->n_spheres; ++l) {
          if (rb->sphere_link[l] != lb) continue;
          if (sph_sph(xyz_r + 3 * k, rb->sphere[4 * k + 3], xyz_r + 3 * l, rb->sphere[4 * l + 3],
                      want_sep ? &sep : NULL))
            hit = 1;
          if (want_sep && sep < ms) ms = sep;
          if (hit && !want_sep) return 1;
        }
      }
    }
  }
  if (min_sep) *min_sep = ms;
  return hit;
}


/* robots i, j (centres xi, xj): strict hit, min sep */
static int pair_eval(const orc_scene* sc, int i, int j, const double* xi, const double* xj, double* min_sep,
                     int want_sep) {
  const orc_robot* a = &sc->robots[i];
  const orc_robot* b = &sc->robots[j];
  int hit = 0;
  double ms = INFINITY, sep;
  for (int k = 0; k < a->n_spheres; ++k)
    for (int l = 0; l < b->n_spheres; ++l) {
      if (sph_sph(xi + 3 * k, a->sphere[4 * k + 3], xj + 3 * l, b->sphere[4 * l + 3], want_sep ? &sep : NULL))
        hit = 1;
      if (want_sep && sep < ms) ms = sep;
      if (hit && !want_sep) return 1;
    }
  if (min_sep) *min_sep = ms;
  return hit;
}

static int* sphere_offsets(const orc_scene* sc) {
  int* off = (int*)malloc(sizeof(int) * (size_t)(sc->n_robots + 1));
  off[0] = 0;
  for (int r = 0; r < sc->n_robots; ++r) off[r + 1] = off[r] + sc->robots[r].n_spheres;
  return off;
}

void orc_state_tables(const orc_scene* sc, const orc_motions* mo, int64_t m, int32_t check_env, int32_t* env_hit,
                      double* env_sep, int32_t* pair_hit, double* pair_sep) {
  const int n = sc->n_robots, P = n * (n - 1) / 2;
  const int32_t T = motion_T(sc, mo, m);
  int* off = sphere_offsets(sc);
  double* xyz = (double*)malloc(sizeof(double) * 3 * (size_t)off[n]);
  for (int32_t t = 0; t < T; ++t) {
    orc_centres_at(sc, mo, m, t, xyz);
    for (int r = 0; r < n; ++r) {
      double s = INFINITY;
      int h = 0;
      if (check_env) h = env_eval_mode(sc, r, xyz + 3 * off[r], &s, 1, check_env);
      env_hit[(int64_t)t * n + r] = h;
      env_sep[(int64_t)t * n + r] = s;
    }
    int p = 0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j, ++p) {
        double s;
        pair_hit[(int64_t)t * P + p] = pair_eval(sc, i, j, xyz + 3 * off[i], xyz + 3 * off[j], &s, 1);
        pair_sep[(int64_t)t * P + p] = s;
      }
  }
  free(xyz);
  free(off);
}

double orc_pair_sep(const orc_scene* sc, const orc_motions* mo, int64_t m, int32_t t, int32_t i, int32_t j) {
  int* off = sphere_offsets(sc);
  double* xyz = (double*)malloc(sizeof(double) * 3 * (size_t)off[sc->n_robots]);
  orc_centres_at(sc, mo, m, t, xyz);
  double s;
  pair_eval(sc, i, j, xyz + 3 * off[i], xyz + 3 * off[j], &s, 1);
  free(xyz);
  free(off);
  return s;
}

/* ------------------------------------------------------------------ */
/* Thread pool over items                                              */
/* ------------------------------------------------------------------ */

typedef struct {
  void (*fn)(void* ctx, int64_t item, double* xyz, double* qbuf, int64_t* work);
  void* ctx;
  int64_t n_items;
  atomic_llong next;
  atomic_llong work;
  int n_spheres_total;
  int n_robots;
} pool_job;

static void* pool_worker(void* arg) {
  pool_job* job = (pool_job*)arg;
  double* xyz = (double*)malloc(sizeof(double) * 3 * (size_t)(job->n_spheres_total + 1));
  double* qbuf = (double*)malloc(sizeof(double) * ORC_QSTRIDE * (size_t)(job->n_robots + 1));
  int64_t work = 0;
  for (;;) {
    int64_t it = atomic_fetch_add(&job->next, 16);
    if (it >= job->n_items) break;
    int64_t end = it + 16 < job->n_items ? it + 16 : job->n_items;
    for (; it < end; ++it) job->fn(job->ctx, it, xyz, qbuf, &work);
  }
  atomic_fetch_add(&job->work, work);
  free(xyz);
  free(qbuf);
  return NULL;
}

static int64_t run_pool(const orc_scene* sc, int64_t n_items, int32_t n_threads,
                        void (*fn)(void*, int64_t, double*, double*, int64_t*), void* ctx) {
  pool_job job;
  job.fn = fn;
  job.ctx = ctx;
  job.n_items = n_items;
  atomic_init(&job.next, 0);
  atomic_init(&job.work, 0);
  job.n_spheres_total = total_spheres(sc);
  job.n_robots = sc->n_robots;
  if (n_threads < 1) n_threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
  for (int i = 1; i < n_threads; ++i) pthread_create(&th[i], NULL, pool_worker, &job);
  pool_worker(&job);
  for (int i = 1; i < n_threads; ++i) pthread_join(th[i], NULL);
  free(th);
  return atomic_load(&job.work);
}

/* ------------------------------------------------------------------ */
/* Composite configuration evaluation (pool acceptance)                */
/* ------------------------------------------------------------------ */

typedef struct {
  const orc_scene* sc;
  const float* q;
  int32_t S, check_env;
  double* min_sep;
  uint8_t* hit;
} cfg_ctx;

static void cfg_item(void* vctx, int64_t it, double* xyz, double* qbuf, int64_t* work) {
  cfg_ctx* c = (cfg_ctx*)vctx;
  const orc_scene* sc = c->sc;
  const int n = sc->n_robots;
  (void)work;
  for (int r = 0; r < n; ++r)
    for (int d = 0; d < sc->robots[r].dof; ++d) qbuf[ORC_QSTRIDE * r + d] = c->q[(it * n + r) * c->S + d];
  centres_from_configs(sc, qbuf, xyz);
  double ms = INFINITY, s;
  int hit = 0, off_i = 0;
  for (int i = 0; i < n; ++i) {
    if (c->check_env) {
      hit |= env_eval_mode(sc, i, xyz + 3 * off_i, &s, 1, c->check_env);
      if (s < ms) ms = s;
    }
    int off_j = off_i + sc->robots[i].n_spheres;
    for (int j = i + 1; j < n; ++j) {
      hit |= pair_eval(sc, i, j, xyz + 3 * off_i, xyz + 3 * off_j, &s, 1);
      if (s < ms) ms = s;
      off_j += sc->robots[j].n_spheres;
    }
    off_i += sc->robots[i].n_spheres;
  }
  c->min_sep[it] = ms;
  c->hit[it] = (uint8_t)hit;
}

void orc_config_eval(const orc_scene* sc, const float* q, int64_t N, int32_t S, int32_t check_env, int32_t n_threads,
                     double* min_sep, uint8_t* hit) {
  cfg_ctx c = {sc, q, S, check_env, min_sep, hit};
  run_pool(sc, N, n_threads, cfg_item, &c);
}

/* ------------------------------------------------------------------ */
/* Plain-definition MotVal / FFC with band classification              */
/* ------------------------------------------------------------------ */

typedef struct {
  const orc_scene* sc;
  const orc_motions* mo;
  int32_t check_env;
  double band;
  uint8_t *valid, *cls, *def_hit;
  uint32_t *key, *k_lo, *k_hi;
  uint8_t* amb;
  int32_t full_scan;        /* classify every state, not only up to the first definite hit */
  int32_t *amb_states, *scanned;   /* optional per-motion counts (NULL = not wanted) */
} q_ctx;

static void state_centres(const orc_scene* sc, const orc_motions* mo, int64_t m, int32_t t, double* qbuf,
                          double* xyz) {
  for (int r = 0; r < sc->n_robots; ++r) orc_interp(sc, mo, m, r, t, qbuf + ORC_QSTRIDE * r);
  centres_from_configs(sc, qbuf, xyz);
}

static void motval_item(void* vctx, int64_t m, double* xyz, double* qbuf, int64_t* work) {
  q_ctx* c = (q_ctx*)vctx;
  const orc_scene* sc = c->sc;
  const int n = sc->n_robots;
  const int32_t T = motion_T(sc, c->mo, m);
  int valid = 1, amb_state = 0, def = 0;
  int32_t n_amb = 0, n_scan = 0;
  for (int32_t t = 0; t < T && (!def || c->full_scan); ++t) {
    ++n_scan;
    state_centres(sc, c->mo, m, t, qbuf, xyz);
    ++*work;
    double ms = INFINITY, s;
    int strict = 0, off_i = 0;
    for (int i = 0; i < n; ++i) {
      if (c->check_env) {
        strict |= env_eval_mode(sc, i, xyz + 3 * off_i, &s, 1, c->check_env);
        if (s < ms) ms = s;
      }
      int off_j = off_i + sc->robots[i].n_spheres;
      for (int j = i + 1; j < n; ++j) {
        strict |= pair_eval(sc, i, j, xyz + 3 * off_i, xyz + 3 * off_j, &s, 1);
        if (s < ms) ms = s;
        off_j += sc->robots[j].n_spheres;
      }
      off_i += sc->robots[i].n_spheres;
    }
    if (strict) valid = 0;
    if (ms > -c->band && ms < c->band) ++n_amb;   /* the state's min sep is within the band */
    if (ms <= -c->band) def = 1;            /* unambiguously invalid: may stop */
    else if (ms < c->band) amb_state = 1;   /* within the band of contact */
  }
  c->valid[m] = (uint8_t)valid;
  c->cls[m] = (uint8_t)(!def && amb_state);
  c->def_hit[m] = (uint8_t)def;
  if (c->amb_states) c->amb_states[m] = n_amb;
  if (c->scanned) c->scanned[m] = n_scan;
}

void orc_motval_batch_ex(const orc_scene* sc, const orc_motions* mo, int32_t check_env, double band, int32_t full_scan,
                         int32_t n_threads, uint8_t* valid, uint8_t* cls, uint8_t* def_hit, int32_t* amb_states,
                         int32_t* scanned) {
  q_ctx c;
  memset(&c, 0, sizeof c);
  c.sc = sc; c.mo = mo; c.check_env = check_env; c.band = band; c.full_scan = full_scan;
  c.valid = valid; c.cls = cls; c.def_hit = def_hit; c.amb_states = amb_states; c.scanned = scanned;
  run_pool(sc, mo->M, n_threads, motval_item, &c);
}

void orc_motval_batch(const orc_scene* sc, const orc_motions* mo, int32_t check_env, double band, int32_t n_threads,
                      uint8_t* valid, uint8_t* cls, uint8_t* def_hit) {
  orc_motval_batch_ex(sc, mo, check_env, band, 0, n_threads, valid, cls, def_hit, NULL, NULL);
}

static void ffc_item(void* vctx, int64_t m, double* xyz, double* qbuf, int64_t* work) {
  q_ctx* c = (q_ctx*)vctx;
  const orc_scene* sc = c->sc;
  const int n = sc->n_robots;
  const uint32_t P = (uint32_t)(n * (n - 1) / 2);
  const int32_t T = motion_T(sc, c->mo, m);
  uint32_t k_or = ORC_NONE, k_lo = ORC_NONE, k_hi = ORC_NONE;
  int amb = 0;
  int32_t n_amb = 0, n_scan = 0;
  for (int32_t t = 0; t < T && (k_hi == ORC_NONE || c->full_scan) && P > 0; ++t) {
    state_centres(sc, c->mo, m, t, qbuf, xyz);
    ++*work;
    ++n_scan;
    int amb_t = 0;
    uint32_t p = 0;
    int off_i = 0;
    for (int i = 0; i < n; ++i) {
      int off_j = off_i + sc->robots[i].n_spheres;
      for (int j = i + 1; j < n; ++j, ++p) {
        double s;
        const int hit = pair_eval(sc, i, j, xyz + 3 * off_i, xyz + 3 * off_j, &s, 1);
        const uint32_t key = (uint32_t)t * P + p;
        if (hit && k_or == ORC_NONE) k_or = key;
        if (s < c->band && k_lo == ORC_NONE) k_lo = key;
        if (s <= -c->band && k_hi == ORC_NONE) k_hi = key;
        if (s > -c->band && s < c->band) {
          amb_t = 1;
          if (k_or == ORC_NONE || key <= k_or) amb = 1;
        }
        off_j += sc->robots[j].n_spheres;
      }
      off_i += sc->robots[i].n_spheres;
    }
    n_amb += amb_t;
  }
  c->key[m] = k_or;
  c->k_lo[m] = k_lo;
  c->k_hi[m] = k_hi;
  c->amb[m] = (uint8_t)amb;
  if (c->amb_states) c->amb_states[m] = n_amb;
  if (c->scanned) c->scanned[m] = n_scan;
}

void orc_ffc_batch_ex(const orc_scene* sc, const orc_motions* mo, double band, int32_t full_scan, int32_t n_threads,
                      uint32_t* key, uint32_t* k_lo, uint32_t* k_hi, uint8_t* amb, int32_t* amb_states,
                      int32_t* scanned) {
  q_ctx c;
  memset(&c, 0, sizeof c);
  c.sc = sc; c.mo = mo; c.band = band; c.full_scan = full_scan;
  c.key = key; c.k_lo = k_lo; c.k_hi = k_hi; c.amb = amb; c.amb_states = amb_states; c.scanned = scanned;
  run_pool(sc, mo->M, n_threads, ffc_item, &c);
}

void orc_ffc_batch(const orc_scene* sc, const orc_motions* mo, double band, int32_t n_threads, uint32_t* key,
                   uint32_t* k_lo, uint32_t* k_hi, uint8_t* amb) {
  orc_ffc_batch_ex(sc, mo, band, 0, n_threads, key, k_lo, k_hi, amb, NULL, NULL);
}

/* ------------------------------------------------------------------ */
/* CPU baseline: sequential linear scan, exit at first strict hit      */
/* ------------------------------------------------------------------ */

static void base_motval_item(void* vctx, int64_t m, double* xyz, double* qbuf, int64_t* work) {
  q_ctx* c = (q_ctx*)vctx;
  const orc_scene* sc = c->sc;
  const int n = sc->n_robots;
  const int32_t T = motion_T(sc, c->mo, m);
  int valid = 1;
  for (int32_t t = 0; t < T && valid; ++t) {
    state_centres(sc, c->mo, m, t, qbuf, xyz);
    ++*work;
    int off_i = 0;
    for (int i = 0; i < n && valid; ++i) {
      if (c->check_env && env_eval_mode(sc, i, xyz + 3 * off_i, NULL, 0, c->check_env)) valid = 0;
      int off_j = off_i + sc->robots[i].n_spheres;
      for (int j = i + 1; j < n && valid; ++j) {
        if (pair_eval(sc, i, j, xyz + 3 * off_i, xyz + 3 * off_j, NULL, 0)) valid = 0;
        off_j += sc->robots[j].n_spheres;
      }
      off_i += sc->robots[i].n_spheres;
    }
  }
  c->valid[m] = (uint8_t)valid;
}

int64_t orc_baseline_motval(const orc_scene* sc, const orc_motions* mo, int32_t check_env, int32_t n_threads,
                            uint8_t* valid) {
  q_ctx c;
  memset(&c, 0, sizeof c);
  c.sc = sc; c.mo = mo; c.check_env = check_env; c.valid = valid;
  return run_pool(sc, mo->M, n_threads, base_motval_item, &c);
}

static void base_ffc_item(void* vctx, int64_t m, double* xyz, double* qbuf, int64_t* work) {
  q_ctx* c = (q_ctx*)vctx;
  const orc_scene* sc = c->sc;
  const int n = sc->n_robots;
  const uint32_t P = (uint32_t)(n * (n - 1) / 2);
  const int32_t T = motion_T(sc, c->mo, m);
  uint32_t key = ORC_NONE;
  for (int32_t t = 0; t < T && key == ORC_NONE && P > 0; ++t) {
    state_centres(sc, c->mo, m, t, qbuf, xyz);
    ++*work;
    uint32_t p = 0;
    int off_i = 0;
    for (int i = 0; i < n && key == ORC_NONE; ++i) {
      int off_j = off_i + sc->robots[i].n_spheres;
      for (int j = i + 1; j < n && key == ORC_NONE; ++j, ++p) {
        if (pair_eval(sc, i, j, xyz + 3 * off_i, xyz + 3 * off_j, NULL, 0)) key = (uint32_t)t * P + p;
        off_j += sc->robots[j].n_spheres;
      }
      off_i += sc->robots[i].n_spheres;
    }
  }
  c->key[m] = key;
}

int64_t orc_baseline_ffc(const orc_scene* sc, const orc_motions* mo, int32_t n_threads, uint32_t* key) {
  q_ctx c;
  memset(&c, 0, sizeof c);
  c.sc = sc; c.mo = mo; c.key = key;
  return run_pool(sc, mo->M, n_threads, base_ffc_item, &c);
}

/* ------------------------------------------------------------------ */
/* PP-ST-RRT MotVal variant                         */
/* ------------------------------------------------------------------ */

typedef struct {
  const orc_scene* sc;
  orc_scene one;              /* the focus robot alone: the candidates' waypoint layout */
  int32_t focus;
  uint64_t partners;
  const orc_motions* cand;
  const int32_t* t_start;
  const orc_motions* paths;
  int32_t horizon, check_env;
  double band;
  uint8_t *valid, *cls, *def_hit;
} pp_ctx;

static void pp_item(void* vctx, int64_t m, double* xyz, double* qbuf, int64_t* work) {
  pp_ctx* c = (pp_ctx*)vctx;
  const orc_scene* sc = c->sc;
  const int n = sc->n_robots, f = c->focus;
  int off[ORC_MAX_DOF + 1];   /* sphere offsets (n <= 64 robots) */
  int* offp = off;
  int* heap = NULL;
  if (n + 1 > ORC_MAX_DOF + 1) offp = heap = (int*)malloc(sizeof(int) * (size_t)(n + 1));
  offp[0] = 0;
  for (int r = 0; r < n; ++r) offp[r + 1] = offp[r] + sc->robots[r].n_spheres;
  const int32_t T = motion_T(&c->one, c->cand, m);
  int valid = 1, amb_state = 0, def = 0;
  for (int32_t t = 0; t < T && !def; ++t) {
    ++*work;
    /* the focus robot at its candidate's local timestep t ... */
    orc_interp(&c->one, c->cand, m, 0, t, qbuf);
    orc_fk(&sc->robots[f], qbuf, xyz + 3 * offp[f]);
    /* ... the higher-priority robots on their fixed paths at the absolute timestep
     * t_start + t ("higher priority paths are treated as dynamic obstacles"),
     * held at the horizon's last timestep beyond it */
    int32_t ta = c->t_start[m] + t;
    if (ta > c->horizon - 1) ta = c->horizon - 1;
    for (int r = 0; r < n; ++r) {
      if (r == f || !((c->partners >> r) & 1u)) continue;
      orc_interp(sc, c->paths, 0, r, ta, qbuf);
      orc_fk(&sc->robots[r], qbuf, xyz + 3 * offp[r]);
    }
    double ms = INFINITY, s;
    int strict = 0;
    /* outer loop: only the current robot (its obstacle / self checks) ... */
    if (c->check_env) {
      strict |= env_eval_mode(sc, f, xyz + 3 * offp[f], &s, 1, c->check_env);
      if (s < ms) ms = s;
    }
    /* ... inner loop: only the higher-priority robots */
    for (int r = 0; r < n; ++r) {
      if (r == f || !((c->partners >> r) & 1u)) continue;
      const int i = r < f ? r : f, j = r < f ? f : r;
      strict |= pair_eval(sc, i, j, xyz + 3 * offp[i], xyz + 3 * offp[j], &s, 1);
      if (s < ms) ms = s;
    }
    if (strict) valid = 0;
    if (ms <= -c->band) def = 1;
    else if (ms < c->band) amb_state = 1;
  }
  c->valid[m] = (uint8_t)valid;
  c->cls[m] = (uint8_t)(!def && amb_state);
  c->def_hit[m] = (uint8_t)def;
  free(heap);
}

void orc_pp_motval_batch(const orc_scene* sc, int32_t focus, uint64_t partner_mask, const orc_motions* cand,
                         const int32_t* t_start, const orc_motions* paths, int32_t horizon, int32_t check_env,
                         double band, int32_t n_threads, uint8_t* valid, uint8_t* cls, uint8_t* def_hit) {
  pp_ctx c;
  memset(&c, 0, sizeof c);
  c.sc = sc;
  c.one.n_robots = 1;
  c.one.robots = &sc->robots[focus];
  c.focus = focus;
  c.partners = partner_mask & ~(1ull << focus);
  c.cand = cand; c.t_start = t_start; c.paths = paths;
  c.horizon = horizon; c.check_env = check_env; c.band = band;
  c.valid = valid; c.cls = cls; c.def_hit = def_hit;
  run_pool(sc, cand->M, n_threads, pp_item, &c);
}
