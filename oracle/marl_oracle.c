/* TEST INFRASTRUCTURE ONLY -- CPU oracle for the batched env-step hot path.
 * See marl_oracle.h for scope, pinning and the output layout.  Every routine
 * cites the reference file:line it restates (paths relative to
 * /root/reference/proj/core/).  Built with -ffp-contract=off and no -march,
 * like the reference's CMake Release build (proj/CMakeLists.txt:7-9), so the
 * fp64 operation sequence and glibc libm calls are the reference's own. */
#define _GNU_SOURCE
#include "marl_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}
const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ PRNG */

static inline uint32_t rotl32(uint32_t x, int r) { return (x << r) | (x >> (32 - r)); }

/* prng.cpp:93-114 */
void orc_threefry(uint32_t k0, uint32_t k1, uint32_t x0, uint32_t x1, uint32_t* y) {
  static const int rot[8] = {13, 15, 26, 6, 17, 29, 16, 24};
  const uint32_t ks[3] = {k0, k1, 0x1BD11BDAu ^ k0 ^ k1};
  x0 += ks[0];
  x1 += ks[1];
  for (int blk = 0; blk < 5; ++blk) {
    int base = (blk & 1) ? 4 : 0;
    for (int r = 0; r < 4; ++r) {
      x0 += x1;
      x1 = rotl32(x1, rot[base + r]);
      x1 ^= x0;
    }
    x0 += ks[(blk + 1) % 3];
    x1 += ks[(blk + 2) % 3] + (uint32_t)(blk + 1);
  }
  y[0] = x0;
  y[1] = x1;
}

/* prng.cpp:76-81 block_at */
static uint64_t block_at(const uint32_t* key, uint64_t off) {
  uint64_t ctr = (((uint64_t)key[3] << 32) | key[2]) + off;
  uint32_t y[2];
  orc_threefry(key[0], key[1], (uint32_t)(ctr & 0xffffffffu), (uint32_t)(ctr >> 32), y);
  return ((uint64_t)y[0] << 32) | y[1];
}

static const uint64_t kSplitBase = (uint64_t)1 << 63; /* prng.cpp:84 */

uint64_t orc_bits(const uint32_t key[4], uint64_t i) { return block_at(key, i); } /* prng.cpp:145 */

/* child i of prng::split (prng.cpp:147-157) */
void orc_split_child(const uint32_t key[4], uint64_t i, uint32_t* out) {
  uint64_t a = block_at(key, kSplitBase + 2 * i);
  uint64_t b = block_at(key, kSplitBase + 2 * i + 1);
  out[0] = (uint32_t)(a >> 32);
  out[1] = (uint32_t)(a & 0xffffffffu);
  out[2] = (uint32_t)(b & 0xffffffffu);
  out[3] = (uint32_t)(b >> 32);
}

void orc_split(const uint32_t key[4], uint64_t n, uint32_t* out) {
  for (uint64_t i = 0; i < n; ++i) orc_split_child(key, i, out + 4 * i);
}

/* prng.cpp:159-167 */
void orc_fold_in(const uint32_t key[4], uint64_t d, uint32_t* out) {
  uint64_t base = kSplitBase + ((uint64_t)1 << 62);
  uint64_t a = block_at(key, base + 2 * d);
  uint64_t b = block_at(key, base + 2 * d + 1);
  out[0] = (uint32_t)(a >> 32);
  out[1] = (uint32_t)(a & 0xffffffffu);
  out[2] = (uint32_t)(b & 0xffffffffu);
  out[3] = (uint32_t)(b >> 32);
}

static inline double to_unit(uint64_t block) { return (double)(block >> 11) * 0x1.0p-53; } /* prng.cpp:86-89 */

/* prng.cpp:169-178 (element j of uniform(key, n, lo, hi)) */
static double uniform_at(const uint32_t* key, uint64_t j, double lo, double hi) {
  double v = lo + to_unit(block_at(key, j)) * (hi - lo);
  if (v >= hi) v = nextafter(hi, lo);
  return v;
}
double orc_uniform1(const uint32_t key[4], double lo, double hi) { return uniform_at(key, 0, lo, hi); }

/* prng.cpp:182-190 */
static int randint1(const uint32_t* key, int lo, int hi) {
  uint64_t range = (uint64_t)((int64_t)hi - (int64_t)lo);
  return (int)((int64_t)lo + (int64_t)(block_at(key, 0) % range));
}
/* prng.cpp:237-240 */
static int bernoulli(const uint32_t* key, double p) { return to_unit(block_at(key, 0)) < p; }

/* ------------------------------------------------------------ common bits */

static inline double dmin(double a, double b) { return (b < a) ? b : a; }  /* std::min */
static inline double dmax(double a, double b) { return (a < b) ? b : a; }  /* std::max */
static inline double dclamp(double v, double lo, double hi) {              /* std::clamp */
  return (v < lo) ? lo : (hi < v) ? hi : v;
}

typedef struct {
  uint64_t h;
} fnv;
static inline void fnv_mix(fnv* f, uint64_t v) { f->h = (f->h ^ v) * 1099511628211ull; }
static inline void fnv_mixd(fnv* f, double d) {
  uint64_t b;
  memcpy(&b, &d, 8);
  fnv_mix(f, b);
}

/* ------------------------------------------------------------------- MPE */
/* mpe.cpp:13-18 */
#define MPE_DT 0.1
#define MPE_DAMPING 0.25
#define MPE_CONTACT_FORCE 1e2
#define MPE_CONTACT_MARGIN 1e-3
#define MPE_DEFAULT_SENS 5.0
#define MPE_EPISODE 25
#define MPE_MAXE 8

typedef struct { /* mpe.cpp:21-29 */
  double size;
  int movable, collide;
  double accel, max_speed;
  int silent, adversary;
} mpe_spec;

typedef struct { /* mpe.cpp:31-37 */
  double pos[2 * MPE_MAXE];
  double vel[2 * MPE_MAXE];
  double comm[MPE_MAXE * 3];
  int goal;
  int steps;
} mpe_state;

typedef struct {
  int scenario, coop_prey;
  int n_agents, n_landmarks, n_entities, dim_c;
  mpe_spec spec[MPE_MAXE];
} mpe_env;

static void mpe_init(mpe_env* e, int scenario, int coop) { /* mpe.cpp:45-79 */
  memset(e, 0, sizeof *e);
  e->scenario = scenario;
  e->coop_prey = (scenario == ORC_MPE_TAG) ? coop : 0;
  mpe_spec lm = {0.05, 0, 1, -1, -1, 1, 0};
  if (scenario == ORC_MPE_SPREAD) {
    e->dim_c = 2;
    e->n_agents = 3;
    for (int i = 0; i < 3; ++i) e->spec[i] = (mpe_spec){0.15, 1, 1, -1, -1, 1, 0};
    e->n_landmarks = 3;
    for (int i = 0; i < 3; ++i) {
      e->spec[3 + i] = lm;
      e->spec[3 + i].collide = 0;
    }
  } else if (scenario == ORC_MPE_SPEAKER_LISTENER) {
    e->dim_c = 3;
    e->n_agents = 2;
    e->spec[0] = (mpe_spec){0.075, 0, 0, -1, -1, 0, 0};
    e->spec[1] = (mpe_spec){0.075, 1, 0, -1, -1, 1, 0};
    e->n_landmarks = 3;
    for (int i = 0; i < 3; ++i) e->spec[2 + i] = (mpe_spec){0.04, 0, 0, -1, -1, 1, 0};
  } else {
    e->dim_c = 2;
    e->n_agents = 4;
    for (int i = 0; i < 3; ++i) e->spec[i] = (mpe_spec){0.075, 1, 1, 3.0, 1.0, 1, 1};
    e->spec[3] = (mpe_spec){0.05, 1, 1, 4.0, 1.3, 1, 0};
    e->n_landmarks = 2;
    for (int i = 0; i < 2; ++i) e->spec[4 + i] = (mpe_spec){0.2, 0, 1, -1, -1, 1, 0};
  }
  e->n_entities = e->n_agents + e->n_landmarks;
}

static int mpe_obs_size(const mpe_env* e, int i) { /* mpe.cpp:278-285 */
  if (e->scenario == ORC_MPE_SPREAD) return 4 + 2 * e->n_landmarks + 4 * (e->n_agents - 1);
  if (e->scenario == ORC_MPE_SPEAKER_LISTENER) return i == 0 ? e->n_landmarks : 2 + 2 * e->n_landmarks + e->dim_c;
  return 4 + 2 * e->n_landmarks + 2 * (e->n_agents - 1) + 2 * (e->spec[i].adversary ? 1 : 0);
}
static int mpe_n_actions(const mpe_env* e, int i) { /* mpe.cpp:91-99 (discrete) */
  return e->spec[i].movable ? 5 : e->dim_c;
}

static double logaddexp0(double z) { /* mpe.cpp:39-41 */
  return z > 0 ? z + log1p(exp(-z)) : log1p(exp(z));
}

static double lm_pos(const mpe_env* e, const mpe_state* s, int j, int axis) { /* mpe.cpp:287-289 */
  return s->pos[2 * (e->n_agents + j) + axis];
}

static void mpe_observe(const mpe_env* e, const mpe_state* s, int i, float* out) { /* mpe.cpp:291-334 */
  double o[64];
  int k = 0;
  if (e->scenario == ORC_MPE_SPEAKER_LISTENER && i == 0) {
    for (int j = 0; j < e->n_landmarks; ++j) o[k++] = j == s->goal ? 1.0 : 0.0;
  } else if (e->scenario == ORC_MPE_SPEAKER_LISTENER) {
    o[k++] = s->vel[2 * i];
    o[k++] = s->vel[2 * i + 1];
    for (int j = 0; j < e->n_landmarks; ++j) {
      o[k++] = lm_pos(e, s, j, 0) - s->pos[2 * i];
      o[k++] = lm_pos(e, s, j, 1) - s->pos[2 * i + 1];
    }
    for (int c = 0; c < e->dim_c; ++c) o[k++] = s->comm[c];
  } else {
    o[k++] = s->vel[2 * i];
    o[k++] = s->vel[2 * i + 1];
    o[k++] = s->pos[2 * i];
    o[k++] = s->pos[2 * i + 1];
    for (int j = 0; j < e->n_landmarks; ++j) {
      o[k++] = lm_pos(e, s, j, 0) - s->pos[2 * i];
      o[k++] = lm_pos(e, s, j, 1) - s->pos[2 * i + 1];
    }
    for (int j = 0; j < e->n_agents; ++j) {
      if (j == i) continue;
      o[k++] = s->pos[2 * j] - s->pos[2 * i];
      o[k++] = s->pos[2 * j + 1] - s->pos[2 * i + 1];
    }
    if (e->scenario == ORC_MPE_SPREAD) {
      for (int j = 0; j < e->n_agents; ++j) {
        if (j == i) continue;
        for (int c = 0; c < e->dim_c; ++c) o[k++] = s->comm[j * e->dim_c + c];
      }
    } else {
      for (int j = 0; j < e->n_agents; ++j) {
        if (j == i || e->spec[j].adversary) continue;
        o[k++] = s->vel[2 * j];
        o[k++] = s->vel[2 * j + 1];
      }
    }
  }
  for (int q = 0; q < k; ++q) out[q] = (float)o[q];
}

static int mpe_collide(const mpe_env* e, const mpe_state* s, int a, int b) { /* mpe.cpp:342-346 */
  double dx = s->pos[2 * a] - s->pos[2 * b];
  double dy = s->pos[2 * a + 1] - s->pos[2 * b + 1];
  return sqrt(dx * dx + dy * dy) < e->spec[a].size + e->spec[b].size;
}

static double bound_penalty(double x) { /* mpe.cpp:348-352 */
  if (x < 0.9) return 0.0;
  if (x < 1.0) return (x - 0.9) * 10.0;
  return dmin(exp(2.0 * x - 2.0), 10.0);
}

static double mpe_reward(const mpe_env* e, const mpe_state* s, int i) { /* mpe.cpp:354-384 */
  if (e->scenario == ORC_MPE_SPREAD) {
    double rew = 0.0;
    for (int j = 0; j < e->n_landmarks; ++j) {
      double best = 1e18;
      for (int a = 0; a < e->n_agents; ++a) {
        double dx = s->pos[2 * a] - lm_pos(e, s, j, 0);
        double dy = s->pos[2 * a + 1] - lm_pos(e, s, j, 1);
        best = dmin(best, sqrt(dx * dx + dy * dy));
      }
      rew -= best;
    }
    for (int a = 0; a < e->n_agents; ++a)
      if (a != i && mpe_collide(e, s, a, i)) rew -= 1.0;
    return rew;
  }
  if (e->scenario == ORC_MPE_SPEAKER_LISTENER) {
    double dx = s->pos[2] - lm_pos(e, s, s->goal, 0);
    double dy = s->pos[3] - lm_pos(e, s, s->goal, 1);
    return -(dx * dx + dy * dy);
  }
  double touches = 0.0;
  for (int a = 0; a < 3; ++a)
    if (mpe_collide(e, s, a, 3)) touches += 1.0;
  if (e->coop_prey || e->spec[i].adversary) return 10.0 * touches;
  double rew = -10.0 * touches;
  rew -= bound_penalty(fabs(s->pos[2 * i]));
  rew -= bound_penalty(fabs(s->pos[2 * i + 1]));
  return rew;
}

static void mpe_reset(const mpe_env* e, const uint32_t* key, mpe_state* s) { /* mpe.cpp:107-124 */
  memset(s, 0, sizeof *s);
  s->goal = -1;
  for (int i = 0; i < e->n_entities; ++i) {
    uint32_t kid[4];
    orc_split_child(key, (uint64_t)i, kid);
    double lim = i < e->n_agents ? 1.0 : 0.9;
    s->pos[2 * i] = uniform_at(kid, 0, -lim, lim);
    s->pos[2 * i + 1] = uniform_at(kid, 1, -lim, lim);
  }
  if (e->scenario == ORC_MPE_SPEAKER_LISTENER) {
    uint32_t kid[4];
    orc_split_child(key, (uint64_t)e->n_entities, kid);
    s->goal = randint1(kid, 0, e->n_landmarks);
  }
}

/* mpe.cpp:126-227; returns done */
static int mpe_step(const mpe_env* e, const mpe_state* prev, const int32_t* act, mpe_state* next,
                    double* rewards) {
  *next = *prev;
  double force[2 * MPE_MAXE];
  for (int q = 0; q < 2 * e->n_entities; ++q) force[q] = 0.0;
  for (int i = 0; i < e->n_agents; ++i) {
    const mpe_spec* sp = &e->spec[i];
    double u[2] = {0.0, 0.0};
    if (sp->movable) {
      int a = act[i];
      if (a == 1) u[0] = -1.0;
      if (a == 2) u[0] = +1.0;
      if (a == 3) u[1] = -1.0;
      if (a == 4) u[1] = +1.0;
      double sens = sp->accel > 0 ? sp->accel : MPE_DEFAULT_SENS;
      force[2 * i] += u[0] * sens;
      force[2 * i + 1] += u[1] * sens;
    }
    if (!sp->silent) {
      double* c = &next->comm[i * e->dim_c];
      for (int k = 0; k < e->dim_c; ++k) c[k] = 0.0;
      c[act[i]] = 1.0;
    }
  }
  for (int a = 0; a < e->n_entities; ++a) {
    for (int b = a + 1; b < e->n_entities; ++b) {
      if (!e->spec[a].collide || !e->spec[b].collide) continue;
      double dx = next->pos[2 * a] - next->pos[2 * b];
      double dy = next->pos[2 * a + 1] - next->pos[2 * b + 1];
      double dist = sqrt(dx * dx + dy * dy);
      if (dist < 1e-9) dist = 1e-9;
      double dist_min = e->spec[a].size + e->spec[b].size;
      double pen = logaddexp0(-(dist - dist_min) / MPE_CONTACT_MARGIN) * MPE_CONTACT_MARGIN;
      double fx = MPE_CONTACT_FORCE * dx / dist * pen;
      double fy = MPE_CONTACT_FORCE * dy / dist * pen;
      if (e->spec[a].movable) {
        force[2 * a] += fx;
        force[2 * a + 1] += fy;
      }
      if (e->spec[b].movable) {
        force[2 * b] -= fx;
        force[2 * b + 1] -= fy;
      }
    }
  }
  for (int i = 0; i < e->n_agents; ++i) {
    const mpe_spec* sp = &e->spec[i];
    if (!sp->movable) continue;
    double* v = &next->vel[2 * i];
    v[0] *= (1.0 - MPE_DAMPING);
    v[1] *= (1.0 - MPE_DAMPING);
    v[0] += force[2 * i] * MPE_DT;
    v[1] += force[2 * i + 1] * MPE_DT;
    if (sp->max_speed > 0) {
      double speed = sqrt(v[0] * v[0] + v[1] * v[1]);
      if (speed > sp->max_speed) {
        v[0] = v[0] / speed * sp->max_speed;
        v[1] = v[1] / speed * sp->max_speed;
      }
    }
    next->pos[2 * i] += v[0] * MPE_DT;
    next->pos[2 * i + 1] += v[1] * MPE_DT;
  }
  next->steps = prev->steps + 1;
  for (int i = 0; i < e->n_agents; ++i) rewards[i] = mpe_reward(e, next, i);
  return next->steps >= MPE_EPISODE;
}

static uint64_t mpe_hash(const mpe_env* e, const mpe_state* s) { /* mpe.cpp:254-269 */
  fnv f = {1469598103934665603ull};
  for (int q = 0; q < 2 * e->n_entities; ++q) fnv_mixd(&f, s->pos[q]);
  for (int q = 0; q < 2 * e->n_agents; ++q) fnv_mixd(&f, s->vel[q]);
  for (int q = 0; q < e->dim_c * e->n_agents; ++q) fnv_mixd(&f, s->comm[q]);
  fnv_mix(&f, (uint64_t)s->steps);
  fnv_mix(&f, (uint64_t)(int64_t)s->goal);
  return f.h;
}

/* ------------------------------------------------------------------ SMAX */
#define SMAX_DT (1.0 / 16.0) /* smax.cpp:17-19 */
#define SMAX_TICKS 8
#define SMAX_SEP_TOL 1e-6
enum { kMoveNorth = 0, kMoveSouth = 1, kMoveEast = 2, kMoveWest = 3, kStop = 4, kAttackBase = 5 };
enum { ST_HEALTH = 0, ST_DAMAGE, ST_COOLDOWN, ST_SPEED, ST_SIGHT, ST_RANGE, ST_RADIUS };

typedef struct {
  int na, ne, n;
  const int8_t* types;
  double (*stats)[7];
  double map, jitter;
  int max_steps, enemy_controlled;
} smax_env;

typedef struct { /* smax.cpp:53-61, arrays point into per-env storage */
  double *x, *y, *health, *cooldown;
  int8_t* type;
  int16_t *prev_action, *ai_target;
  int8_t* ai_sweep;
  int* t;
  int8_t* winner;
} smax_view;

static inline int team_of(const smax_env* e, int u) { return u < e->na ? 0 : 1; } /* smax.cpp:344 */
static inline double st(const smax_env* e, const smax_view* s, int u, int f) {
  return e->stats[s->type[u]][f];
}

static double center_dist(const smax_view* s, int a, int b) { /* smax.cpp:494-496 */
  return hypot(s->x[a] - s->x[b], s->y[a] - s->y[b]);
}
static int in_attack_range(const smax_env* e, const smax_view* s, int sh, int tg) { /* smax.cpp:497-501 */
  double reach = st(e, s, sh, ST_RANGE) + st(e, s, sh, ST_RADIUS) + st(e, s, tg, ST_RADIUS);
  return center_dist(s, sh, tg) <= reach;
}

static double max_overlap(const smax_env* e, const smax_view* s) { /* smax.cpp:569-580 */
  double worst = 0.0;
  for (int a = 0; a < e->n; ++a) {
    if (s->health[a] <= 0.0) continue;
    for (int b = a + 1; b < e->n; ++b) {
      if (s->health[b] <= 0.0) continue;
      double sum = st(e, s, a, ST_RADIUS) + st(e, s, b, ST_RADIUS);
      worst = dmax(worst, sum - center_dist(s, a, b));
    }
  }
  return worst;
}

static void separate(const smax_env* e, smax_view* s, int to_fixpoint) { /* smax.cpp:542-567 */
  for (int pass = 0; pass < (to_fixpoint ? 256 : 1); ++pass) {
    for (int a = 0; a < e->n; ++a) {
      if (s->health[a] <= 0.0) continue;
      for (int b = a + 1; b < e->n; ++b) {
        if (s->health[b] <= 0.0) continue;
        double ra = st(e, s, a, ST_RADIUS), rb = st(e, s, b, ST_RADIUS);
        double dx = s->x[b] - s->x[a], dy = s->y[b] - s->y[a];
        double d = hypot(dx, dy);
        double overlap = ra + rb - d;
        if (overlap <= 0.0) continue;
        double nx = 1.0, ny = 0.0;
        if (d > 1e-12) {
          nx = dx / d;
          ny = dy / d;
        }
        double push = 0.5 * overlap;
        s->x[a] = dclamp(s->x[a] - nx * push, ra, e->map - ra);
        s->y[a] = dclamp(s->y[a] - ny * push, ra, e->map - ra);
        s->x[b] = dclamp(s->x[b] + nx * push, rb, e->map - rb);
        s->y[b] = dclamp(s->y[b] + ny * push, rb, e->map - rb);
      }
    }
    if (!to_fixpoint || max_overlap(e, s) <= SMAX_SEP_TOL) break;
  }
}

static void smax_place(const smax_env* e, smax_view* s, int u, double bx, double by) { /* smax.cpp:481-485 */
  double r = st(e, s, u, ST_RADIUS);
  s->x[u] = dclamp(bx, r, e->map - r);
  s->y[u] = dclamp(by, r, e->map - r);
}
static void place_jittered(const smax_env* e, smax_view* s, int u, double bx, double by,
                           const uint32_t* key) { /* smax.cpp:486-492 */
  if (e->jitter > 0.0) {
    uint32_t k[4];
    orc_fold_in(key, 3000 + 2 * (uint64_t)u, k);
    bx += uniform_at(k, 0, -e->jitter, e->jitter);
    orc_fold_in(key, 3001 + 2 * (uint64_t)u, k);
    by += uniform_at(k, 0, -e->jitter, e->jitter);
  }
  smax_place(e, s, u, bx, by);
}

static void smax_reset(const smax_env* e, const uint32_t* key, smax_view* s) { /* smax.cpp:163-193 */
  for (int u = 0; u < e->n; ++u) {
    s->type[u] = e->types[u];
    s->x[u] = 0.0;
    s->y[u] = 0.0;
  }
  /* spawn_clusters, smax.cpp:448-454 */
  for (int i = 0; i < e->na; ++i)
    place_jittered(e, s, i, 0.25 * e->map - 1.5 * (i / 5), 0.5 * e->map + 1.5 * (i % 5 - 2), key);
  for (int i = 0; i < e->ne; ++i)
    place_jittered(e, s, e->na + i, 0.75 * e->map + 1.5 * (i / 5), 0.5 * e->map + 1.5 * (i % 5 - 2), key);
  for (int u = 0; u < e->n; ++u) {
    s->health[u] = st(e, s, u, ST_HEALTH);
    s->cooldown[u] = 0.0;
    s->prev_action[u] = kStop;
    s->ai_target[u] = -1;
    s->ai_sweep[u] = -1;
  }
  *s->t = 0;
  *s->winner = -1;
  separate(e, s, 1);
}

static int smax_n_actions(const smax_env* e, int u) { /* smax.cpp:153-155 */
  return kAttackBase + (team_of(e, u) == 0 ? e->ne : e->na);
}

static void smax_legal(const smax_env* e, const smax_view* s, int u, uint8_t* mask) { /* smax.cpp:195-211 */
  int opp_start = team_of(e, u) == 0 ? e->na : 0;
  int opp_n = team_of(e, u) == 0 ? e->ne : e->na;
  for (int q = 0; q < kAttackBase + opp_n; ++q) mask[q] = 0;
  if (*s->winner != -1) return;
  mask[kStop] = 1;
  if (s->health[u] <= 0.0) return;
  for (int m = 0; m < kStop; ++m) mask[m] = 1;
  for (int k = 0; k < opp_n; ++k) {
    int o = opp_start + k;
    if (s->health[o] > 0.0 && in_attack_range(e, s, u, o)) mask[kAttackBase + k] = 1;
  }
}

static int heuristic_action(const smax_env* e, const smax_view* s, int u, int* target,
                            int* sweep) { /* smax.cpp:374-419 */
  if (s->health[u] <= 0.0) return kStop;
  int team = team_of(e, u);
  int opp_start = team == 0 ? e->na : 0;
  int opp_n = team == 0 ? e->ne : e->na;
  double sight = st(e, s, u, ST_SIGHT);
#define VISIBLE(k) (s->health[opp_start + (k)] > 0.0 && center_dist(s, u, opp_start + (k)) <= sight)
  if (*target < 0 || *target >= opp_n || !VISIBLE(*target)) {
    *target = -1;
    double best = 0.0;
    for (int k = 0; k < opp_n; ++k) {
      if (VISIBLE(k) && in_attack_range(e, s, u, opp_start + k)) {
        *target = k;
        break;
      }
    }
    if (*target < 0) {
      for (int k = 0; k < opp_n; ++k) {
        if (!VISIBLE(k)) continue;
        double d = center_dist(s, u, opp_start + k);
        if (*target < 0 || d < best) {
          *target = k;
          best = d;
        }
      }
    }
  }
#undef VISIBLE
  if (*target >= 0) {
    int o = opp_start + *target;
    if (in_attack_range(e, s, u, o)) return kAttackBase + *target;
    double dx = s->x[o] - s->x[u];
    double dy = s->y[o] - s->y[u];
    if (fabs(dx) >= fabs(dy)) return dx > 0 ? kMoveEast : kMoveWest;
    return dy > 0 ? kMoveNorth : kMoveSouth;
  }
  if (*sweep < 0) *sweep = team == 0 ? kMoveEast : kMoveWest;
  if (s->x[u] <= 1.0) *sweep = kMoveEast;
  if (s->x[u] >= e->map - 1.0) *sweep = kMoveWest;
  return *sweep;
}

static void simulate_tick(const smax_env* e, smax_view* s, const int* act, int final_tick,
                          double* damage, double* health0) { /* smax.cpp:503-537 */
  static const double dir_x[4] = {0.0, 0.0, 1.0, -1.0};
  static const double dir_y[4] = {1.0, -1.0, 0.0, 0.0};
  for (int u = 0; u < e->n; ++u)
    if (s->health[u] > 0.0) s->cooldown[u] = dmax(0.0, s->cooldown[u] - SMAX_DT);
  for (int u = 0; u < e->n; ++u) {
    if (s->health[u] <= 0.0 || act[u] > kMoveWest) continue;
    double sp = st(e, s, u, ST_SPEED), r = st(e, s, u, ST_RADIUS);
    s->x[u] = dclamp(s->x[u] + sp * SMAX_DT * dir_x[act[u]], r, e->map - r);
    s->y[u] = dclamp(s->y[u] + sp * SMAX_DT * dir_y[act[u]], r, e->map - r);
  }
  for (int u = 0; u < e->n; ++u) {
    damage[u] = 0.0;
    health0[u] = s->health[u];
  }
  for (int u = 0; u < e->n; ++u) {
    if (health0[u] <= 0.0 || act[u] < kAttackBase) continue;
    int o = (team_of(e, u) == 0 ? e->na : 0) + (act[u] - kAttackBase);
    if (health0[o] <= 0.0 || !in_attack_range(e, s, u, o)) continue;
    if (s->cooldown[u] > 0.0) continue;
    damage[o] += st(e, s, u, ST_DAMAGE);
    s->cooldown[u] = st(e, s, u, ST_COOLDOWN);
  }
  for (int u = 0; u < e->n; ++u)
    if (damage[u] > 0.0) s->health[u] = dmax(0.0, health0[u] - damage[u]);
  separate(e, s, final_tick);
}

static int alive_count(const smax_env* e, const smax_view* s, int team) { /* smax.cpp:582-587 */
  int c = 0;
  for (int u = team == 0 ? 0 : e->na, end = team == 0 ? e->na : e->n; u < end; ++u)
    c += s->health[u] > 0.0 ? 1 : 0;
  return c;
}

static double smax_pool(const smax_env* e, const smax_view* s, int team) { /* smax.cpp:365-372 */
  double total = 0.0;
  for (int u = team == 0 ? 0 : e->na, end = team == 0 ? e->na : e->n; u < end; ++u) {
    total += s->health[u] / st(e, s, u, ST_HEALTH);
    total += s->health[u] > 0.0 ? 1.0 : 0.0;
  }
  return total;
}

static void smax_observe(const smax_env* e, const smax_view* s, int me, float* o) { /* smax.cpp:601-634 */
  int size = 10 + 17 * (e->n - 1);
  for (int q = 0; q < size; ++q) o[q] = 0.0f;
  if (s->health[me] <= 0.0) return;
  double mh = st(e, s, me, ST_HEALTH), mc = st(e, s, me, ST_COOLDOWN), sight = st(e, s, me, ST_SIGHT);
  int k = 0;
  o[k++] = (float)(s->health[me] / mh);
  o[k++] = (float)(s->cooldown[me] / mc);
  o[k++] = (float)(s->x[me] / e->map);
  o[k++] = (float)(s->y[me] / e->map);
  for (int i = 0; i < 6; ++i) o[k++] = i == s->type[me] ? 1.0f : 0.0f;
  int team = team_of(e, me);
  for (int pass = 0; pass < 2; ++pass) {
    for (int u = 0; u < e->n; ++u) {
      int want = pass == 0 ? (u != me && team_of(e, u) == team) : (team_of(e, u) != team);
      if (!want) continue;
      int vis = s->health[u] > 0.0 && center_dist(s, me, u) <= sight;
      if (!vis) {
        k += 17;
        continue;
      }
      o[k++] = 1.0f;
      o[k++] = (float)((s->x[u] - s->x[me]) / sight);
      o[k++] = (float)((s->y[u] - s->y[me]) / sight);
      o[k++] = (float)(s->health[u] / st(e, s, u, ST_HEALTH));
      o[k++] = (float)(s->cooldown[u] / st(e, s, u, ST_COOLDOWN));
      for (int i = 0; i < 6; ++i) o[k++] = i == s->type[u] ? 1.0f : 0.0f;
      int pa = s->prev_action[u];
      int bucket = pa <= kStop ? pa : kStop + 1; /* smax.cpp:589 */
      for (int i = 0; i < 6; ++i) o[k++] = i == bucket ? 1.0f : 0.0f;
    }
  }
}

static uint64_t smax_hash(const smax_env* e, const smax_view* s) { /* smax.cpp:312-337 */
  fnv f = {1469598103934665603ull};
  for (int u = 0; u < e->n; ++u) {
    fnv_mixd(&f, s->x[u]);
    fnv_mixd(&f, s->y[u]);
    fnv_mixd(&f, s->health[u]);
    fnv_mixd(&f, s->cooldown[u]);
    fnv_mix(&f, (uint64_t)(uint8_t)s->type[u]);
    fnv_mix(&f, (uint64_t)(uint16_t)s->prev_action[u]);
    fnv_mix(&f, (uint64_t)(uint16_t)s->ai_target[u]);
    fnv_mix(&f, (uint64_t)(uint8_t)s->ai_sweep[u]);
  }
  fnv_mix(&f, (uint64_t)*s->t);
  fnv_mix(&f, (uint64_t)(uint8_t)*s->winner);
  return f.h;
}

/* ------------------------------------------------------------ Overcooked */
enum { kUp = 0, kDown = 1, kLeft = 2, kRight = 3, kStay = 4, kInteract = 5 }; /* overcooked.cpp:16 */
enum { kNone = 0, kOnion = 1, kPlate = 2, kSoup = 3 };                         /* overcooked.cpp:21 */
static const int kDr[4] = {-1, 1, 0, 0}, kDc[4] = {0, 0, -1, 1};
#define OC_MAXC 256
#define OC_PLANES 27

typedef struct { /* overcooked.cpp:60-68 */
  int h, w;
  char kind[OC_MAXC];
  int spawn[2];
  int n_pots, pot_cells[OC_MAXC];
  int n_counters, counter_cells[OC_MAXC];
  int pot_index[OC_MAXC], counter_index[OC_MAXC];
} oc_layout;

typedef struct {
  oc_layout lay;
  int max_steps, cook_time, random_conflicts;
  double delivery_reward, sh_onion, sh_plate, sh_soup;
} oc_env;

typedef struct { /* overcooked.cpp:131-139 */
  int pos[2], facing[2], held[2];
  int* pot_onions;
  int* pot_timer;
  int* counter_item;
  int* t;
} oc_view;

static int oc_parse(const char* text, oc_layout* L) { /* overcooked.cpp:70-129 */
  char rows[64][128];
  int nr = 0, len = 0;
  memset(L, 0, sizeof *L);
  for (const char* c = text;; ++c) {
    if (*c == '\n' || *c == 0) {
      if (len > 0) {
        if (nr >= 64) return fail(2, "layout too tall");
        rows[nr][len] = 0;
        ++nr;
      }
      len = 0;
      if (*c == 0) break;
    } else {
      if (len >= 127) return fail(2, "layout too wide");
      rows[nr][len++] = *c;
    }
  }
  if (nr < 3) return fail(2, "layout needs at least 3 rows");
  L->h = nr;
  L->w = (int)strlen(rows[0]);
  if (L->h * L->w > OC_MAXC) return fail(2, "layout too large");
  for (int r = 0; r < nr; ++r)
    if ((int)strlen(rows[r]) != L->w) return fail(2, "layout rows must all have the same width");
  L->spawn[0] = L->spawn[1] = -1;
  for (int r = 0; r < L->h; ++r)
    for (int c = 0; c < L->w; ++c) {
      char ch = rows[r][c];
      int cell = r * L->w + c;
      switch (ch) {
        case 'X': case 'O': case 'D': case 'P': case 'S':
          L->kind[cell] = ch;
          if (ch == 'P') L->pot_cells[L->n_pots++] = cell;
          if (ch == 'X') L->counter_cells[L->n_counters++] = cell;
          break;
        case ' ':
          L->kind[cell] = ' ';
          break;
        case '1': case '2': {
          int idx = ch - '1';
          if (L->spawn[idx] != -1) return fail(2, "duplicate spawn digit in layout");
          L->spawn[idx] = cell;
          L->kind[cell] = ' ';
          break;
        }
        default:
          return fail(2, "unknown layout character");
      }
    }
  if (L->spawn[0] < 0 || L->spawn[1] < 0) return fail(2, "layout needs spawn digits 1 and 2");
  const char need[4] = {'P', 'O', 'D', 'S'};
  for (int q = 0; q < 4; ++q) {
    int found = 0;
    for (int c = 0; c < L->h * L->w; ++c) found |= L->kind[c] == need[q];
    if (!found) return fail(2, "layout needs at least one of each P, O, D, S");
  }
  for (int r = 0; r < L->h; ++r)
    for (int c = 0; c < L->w; ++c)
      if ((r == 0 || c == 0 || r == L->h - 1 || c == L->w - 1) && L->kind[r * L->w + c] == ' ')
        return fail(2, "layout border must be walls/stations, not floor");
  /* lower_bound lookups of overcooked.cpp:386-393 (cells are ascending) */
  for (int p = 0; p < L->n_pots; ++p) L->pot_index[L->pot_cells[p]] = p;
  for (int k = 0; k < L->n_counters; ++k) L->counter_index[L->counter_cells[k]] = k;
  return 0;
}

static void oc_reset(const oc_env* e, oc_view* s) { /* overcooked.cpp:193-204 */
  s->pos[0] = e->lay.spawn[0];
  s->pos[1] = e->lay.spawn[1];
  s->facing[0] = s->facing[1] = kUp;
  s->held[0] = s->held[1] = kNone;
  for (int p = 0; p < e->lay.n_pots; ++p) s->pot_onions[p] = s->pot_timer[p] = 0;
  for (int k = 0; k < e->lay.n_counters; ++k) s->counter_item[k] = kNone;
  *s->t = 0;
}

static void oc_encode(const oc_env* e, const oc_view* s, int me, float* o) { /* overcooked.cpp:395-427 */
  const oc_layout* L = &e->lay;
  int cells = L->h * L->w;
  for (int q = 0; q < OC_PLANES * cells + 1; ++q) o[q] = 0.0f;
#define PUT(plane, cell, v) (o[(plane) * cells + (cell)] = (v))
  int other = 1 - me;
  PUT(0, s->pos[me], 1.0f);
  PUT(1, s->pos[other], 1.0f);
  PUT(2 + s->facing[me], s->pos[me], 1.0f);
  PUT(6 + s->facing[other], s->pos[other], 1.0f);
  for (int cell = 0; cell < cells; ++cell) {
    switch (L->kind[cell]) {
      case 'X': PUT(10, cell, 1.0f); break;
      case 'O': PUT(11, cell, 1.0f); break;
      case 'D': PUT(12, cell, 1.0f); break;
      case 'P': PUT(13, cell, 1.0f); break;
      case 'S': PUT(14, cell, 1.0f); break;
      default: break;
    }
  }
  for (int p = 0; p < L->n_pots; ++p) {
    int cell = L->pot_cells[p];
    PUT(15, cell, (float)s->pot_onions[p]);
    PUT(16, cell, (float)s->pot_timer[p] / (float)e->cook_time);
    if (s->pot_onions[p] == 3 && s->pot_timer[p] == 0) PUT(17, cell, 1.0f);
  }
  if (s->held[me] != kNone) PUT(18 + s->held[me] - 1, s->pos[me], 1.0f);
  if (s->held[other] != kNone) PUT(21 + s->held[other] - 1, s->pos[other], 1.0f);
  for (int k = 0; k < L->n_counters; ++k)
    if (s->counter_item[k] != kNone) PUT(24 + s->counter_item[k] - 1, L->counter_cells[k], 1.0f);
#undef PUT
  o[OC_PLANES * cells] = (float)*s->t / (float)e->max_steps;
}

/* overcooked.cpp:206-313; s holds prev on entry and next on exit */
static int oc_step(const oc_env* e, const uint32_t* key, oc_view* s, const int32_t* act,
                   double* reward, double* shaped, int* deliveries_out) {
  const oc_layout* L = &e->lay;
  int prev_pos[2] = {s->pos[0], s->pos[1]};
  for (int p = 0; p < L->n_pots; ++p)
    if (s->pot_onions[p] == 3 && s->pot_timer[p] > 0) s->pot_timer[p] -= 1;
  int want[2] = {s->pos[0], s->pos[1]};
  for (int i = 0; i < 2; ++i) {
    if (act[i] > kRight) continue;
    s->facing[i] = act[i];
    int r = s->pos[i] / L->w + kDr[act[i]];
    int c = s->pos[i] % L->w + kDc[act[i]];
    if (L->kind[r * L->w + c] == ' ') want[i] = r * L->w + c;
  }
  int swap = want[0] == prev_pos[1] && want[1] == prev_pos[0] && want[0] != prev_pos[0];
  if (want[0] == want[1] || swap) {
    if (e->random_conflicts && !swap && want[0] != prev_pos[0] && want[1] != prev_pos[1]) {
      int loser = bernoulli(key, 0.5) ? 0 : 1;
      want[loser] = prev_pos[loser];
    } else {
      want[0] = prev_pos[0];
      want[1] = prev_pos[1];
    }
  }
  s->pos[0] = want[0];
  s->pos[1] = want[1];
  shaped[0] = shaped[1] = 0.0;
  int deliveries = 0;
  for (int i = 0; i < 2; ++i) {
    if (act[i] != kInteract) continue;
    int r = s->pos[i] / L->w + kDr[s->facing[i]];
    int c = s->pos[i] % L->w + kDc[s->facing[i]];
    int cell = r * L->w + c;
    switch (L->kind[cell]) {
      case 'O':
        if (s->held[i] == kNone) s->held[i] = kOnion;
        break;
      case 'D':
        if (s->held[i] == kNone) {
          s->held[i] = kPlate;
          shaped[i] += e->sh_plate;
        }
        break;
      case 'P': {
        int p = L->pot_index[cell];
        if (s->held[i] == kOnion && s->pot_onions[p] < 3) {
          s->pot_onions[p] += 1;
          s->held[i] = kNone;
          shaped[i] += e->sh_onion;
          if (s->pot_onions[p] == 3) s->pot_timer[p] = e->cook_time;
        } else if (s->held[i] == kPlate && s->pot_onions[p] == 3 && s->pot_timer[p] == 0) {
          s->held[i] = kSoup;
          s->pot_onions[p] = 0;
          shaped[i] += e->sh_soup;
        }
        break;
      }
      case 'S':
        if (s->held[i] == kSoup) {
          s->held[i] = kNone;
          deliveries += 1;
        }
        break;
      case 'X': {
        int k = L->counter_index[cell];
        if (s->held[i] != kNone && s->counter_item[k] == kNone) {
          s->counter_item[k] = s->held[i];
          s->held[i] = kNone;
        } else if (s->held[i] == kNone && s->counter_item[k] != kNone) {
          s->held[i] = s->counter_item[k];
          s->counter_item[k] = kNone;
        }
        break;
      }
      default:
        break;
    }
  }
  *s->t += 1;
  *reward = e->delivery_reward * deliveries;
  *deliveries_out = deliveries;
  return *s->t >= e->max_steps;
}

static uint64_t oc_hash(const oc_env* e, const oc_view* s) { /* overcooked.cpp:348-364 */
  fnv f = {1469598103934665603ull};
  for (int i = 0; i < 2; ++i) {
    fnv_mix(&f, (uint64_t)s->pos[i]);
    fnv_mix(&f, (uint64_t)s->facing[i]);
    fnv_mix(&f, (uint64_t)s->held[i]);
  }
  for (int p = 0; p < e->lay.n_pots; ++p) {
    fnv_mix(&f, (uint64_t)s->pot_onions[p]);
    fnv_mix(&f, (uint64_t)s->pot_timer[p]);
  }
  for (int k = 0; k < e->lay.n_counters; ++k) fnv_mix(&f, (uint64_t)s->counter_item[k]);
  fnv_mix(&f, (uint64_t)*s->t);
  return f.h;
}

/* ------------------------------------------------------------ VectorEnv */

struct orc_venv {
  int family;
  int64_t n, off, gn;
  int A, obs_dim, n_act, n_info;
  mpe_env mpe;
  smax_env smax;
  int8_t smax_types[128];
  double smax_stats[6][7];
  oc_env oc;
  /* per-env storage */
  mpe_state* mpe_s;
  double* sx; /* [n][4][U] x,y,health,cooldown */
  int8_t* stype;
  int16_t *sprev, *starget;
  int8_t* ssweep;
  int* st_t;
  int8_t* swinner;
  int* oc_ints; /* per env: pos2 facing2 held2 t pots*2 counters */
  int oc_stride;
  /* VectorEnv::BatchedState (vector_env.hpp:13-20) */
  uint32_t* keys;
  double* ep_ret;
  int32_t* ep_len;
  float* scratch_obs;
};

static smax_view smax_at(orc_venv* v, int64_t i) {
  int U = v->smax.n;
  smax_view s;
  double* base = v->sx + (size_t)i * 4 * U;
  s.x = base;
  s.y = base + U;
  s.health = base + 2 * U;
  s.cooldown = base + 3 * U;
  s.type = v->stype + (size_t)i * U;
  s.prev_action = v->sprev + (size_t)i * U;
  s.ai_target = v->starget + (size_t)i * U;
  s.ai_sweep = v->ssweep + (size_t)i * U;
  s.t = v->st_t + i;
  s.winner = v->swinner + i;
  return s;
}

static oc_view oc_at(orc_venv* v, int64_t i) {
  oc_view s;
  int* b = v->oc_ints + (size_t)i * v->oc_stride;
  s.pos[0] = b[0];
  s.pos[1] = b[1];
  s.facing[0] = b[2];
  s.facing[1] = b[3];
  s.held[0] = b[4];
  s.held[1] = b[5];
  s.t = b + 6;
  s.pot_onions = b + 7;
  s.pot_timer = b + 7 + v->oc.lay.n_pots;
  s.counter_item = b + 7 + 2 * v->oc.lay.n_pots;
  return s;
}
static void oc_store(orc_venv* v, int64_t i, const oc_view* s) {
  int* b = v->oc_ints + (size_t)i * v->oc_stride;
  b[0] = s->pos[0];
  b[1] = s->pos[1];
  b[2] = s->facing[0];
  b[3] = s->facing[1];
  b[4] = s->held[0];
  b[5] = s->held[1];
}

int orc_create(const orc_params* p, int64_t n_envs, int64_t global_offset, int64_t global_n,
               orc_venv** out) {
  if (n_envs < 1) return fail(3, "VectorEnv: n_envs must be >= 1");
  if (global_offset < 0 || global_offset + n_envs > global_n) return fail(3, "bad shard range");
  orc_venv* v = calloc(1, sizeof *v);
  v->family = p->family;
  v->n = n_envs;
  v->off = global_offset;
  v->gn = global_n;
  if (p->family == ORC_MPE) {
    mpe_init(&v->mpe, p->mpe_scenario, p->mpe_coop_prey);
    v->A = v->mpe.n_agents;
    for (int i = 0; i < v->A; ++i) {
      if (mpe_obs_size(&v->mpe, i) > v->obs_dim) v->obs_dim = mpe_obs_size(&v->mpe, i);
      if (mpe_n_actions(&v->mpe, i) > v->n_act) v->n_act = mpe_n_actions(&v->mpe, i);
    }
    v->n_info = 0;
    v->mpe_s = calloc((size_t)n_envs, sizeof(mpe_state));
  } else if (p->family == ORC_SMAX) {
    smax_env* e = &v->smax;
    e->na = p->smax_n_ally;
    e->ne = p->smax_n_enemy;
    e->n = e->na + e->ne;
    if (e->n > 128 || e->na < 1 || e->ne < 1) { free(v); return fail(2, "bad SMAX roster"); }
    memcpy(v->smax_types, p->smax_types, sizeof v->smax_types);
    memcpy(v->smax_stats, p->smax_stats, sizeof v->smax_stats);
    e->types = v->smax_types;
    e->stats = v->smax_stats;
    e->map = p->smax_map;
    e->jitter = p->smax_jitter;
    e->max_steps = p->smax_max_steps;
    e->enemy_controlled = p->smax_enemy_controlled;
    v->A = e->na + (e->enemy_controlled ? e->ne : 0);
    v->obs_dim = 10 + 17 * (e->n - 1);
    v->n_act = kAttackBase + (e->enemy_controlled && e->na > e->ne ? e->na : e->ne);
    v->n_info = 3;
    int U = e->n;
    v->sx = calloc((size_t)n_envs * 4 * U, sizeof(double));
    v->stype = calloc((size_t)n_envs * U, 1);
    v->sprev = calloc((size_t)n_envs * U, 2);
    v->starget = calloc((size_t)n_envs * U, 2);
    v->ssweep = calloc((size_t)n_envs * U, 1);
    v->st_t = calloc((size_t)n_envs, sizeof(int));
    v->swinner = calloc((size_t)n_envs, 1);
  } else if (p->family == ORC_OVERCOOKED) {
    oc_env* e = &v->oc;
    int rc = oc_parse(p->oc_layout, &e->lay);
    if (rc) { free(v); return rc; }
    e->max_steps = p->oc_max_steps;
    e->cook_time = p->oc_cook_time;
    e->delivery_reward = p->oc_delivery_reward;
    e->sh_onion = p->oc_shaping_onion;
    e->sh_plate = p->oc_shaping_plate;
    e->sh_soup = p->oc_shaping_soup;
    e->random_conflicts = p->oc_random_conflicts;
    if (e->max_steps < 1) { free(v); return fail(2, "overcooked: max_steps must be >= 1"); }
    if (e->cook_time < 1) { free(v); return fail(2, "overcooked: cook_time must be >= 1"); }
    v->A = 2;
    v->obs_dim = OC_PLANES * e->lay.h * e->lay.w + 1;
    v->n_act = 6;
    v->n_info = 2;
    v->oc_stride = 7 + 2 * e->lay.n_pots + e->lay.n_counters;
    v->oc_ints = calloc((size_t)n_envs * v->oc_stride, sizeof(int));
  } else {
    free(v);
    return fail(1, "unknown family");
  }
  v->keys = calloc((size_t)n_envs * 4, sizeof(uint32_t));
  v->ep_ret = calloc((size_t)n_envs, sizeof(double));
  v->ep_len = calloc((size_t)n_envs, sizeof(int32_t));
  v->scratch_obs = calloc((size_t)v->A * v->obs_dim, sizeof(float));
  *out = v;
  return 0;
}

void orc_destroy(orc_venv* v) {
  if (!v) return;
  free(v->mpe_s);
  free(v->sx);
  free(v->stype);
  free(v->sprev);
  free(v->starget);
  free(v->ssweep);
  free(v->st_t);
  free(v->swinner);
  free(v->oc_ints);
  free(v->keys);
  free(v->ep_ret);
  free(v->ep_len);
  free(v->scratch_obs);
  free(v);
}

void orc_spec(const orc_venv* v, int* n_agents, int* obs_dim, int* n_act, int* n_info) {
  *n_agents = v->A;
  *obs_dim = v->obs_dim;
  *n_act = v->n_act;
  *n_info = v->n_info;
}

/* env.reset for env i into its slot; writes padded obs rows */
static void env_reset(orc_venv* v, int64_t i, const uint32_t* key, float* obs) {
  size_t row = (size_t)v->obs_dim;
  if (obs) memset(obs, 0, sizeof(float) * row * v->A);
  if (v->family == ORC_MPE) {
    mpe_reset(&v->mpe, key, &v->mpe_s[i]);
    if (obs)
      for (int a = 0; a < v->A; ++a) mpe_observe(&v->mpe, &v->mpe_s[i], a, obs + a * row);
  } else if (v->family == ORC_SMAX) {
    smax_view s = smax_at(v, i);
    smax_reset(&v->smax, key, &s);
    if (obs)
      for (int a = 0; a < v->A; ++a) smax_observe(&v->smax, &s, a, obs + a * row);
  } else {
    oc_view s = oc_at(v, i);
    oc_reset(&v->oc, &s);
    oc_store(v, i, &s);
    if (obs)
      for (int a = 0; a < 2; ++a) oc_encode(&v->oc, &s, a, obs + a * row);
  }
}

int orc_reset(orc_venv* v, const uint32_t key[4], float* obs) { /* vector_env.cpp:51-70 */
  uint32_t carry_parent[4];
  orc_fold_in(key, 1, carry_parent);
  for (int64_t i = 0; i < v->n; ++i) {
    uint64_t g = (uint64_t)(v->off + i);
    uint32_t rk[4];
    orc_split_child(key, g, rk);
    orc_split_child(carry_parent, g, v->keys + 4 * i);
    v->ep_ret[i] = 0.0;
    v->ep_len[i] = 0;
    env_reset(v, i, rk, obs ? obs + (size_t)i * v->A * v->obs_dim : NULL);
  }
  return 0;
}

static void env_legal(orc_venv* v, int64_t i, int a, uint8_t* mask) {
  if (v->family == ORC_SMAX) {
    smax_view s = smax_at(v, i);
    int u = a; /* agent order = unit order (smax.cpp:143-145) */
    smax_legal(&v->smax, &s, u, mask);
    for (int q = smax_n_actions(&v->smax, u); q < v->n_act; ++q) mask[q] = 0;
  } else {
    int n = v->family == ORC_MPE ? mpe_n_actions(&v->mpe, a) : 6;
    for (int q = 0; q < v->n_act; ++q) mask[q] = q < n; /* env.hpp:71-73 default */
  }
}

int orc_legal(orc_venv* v, uint8_t* legal) {
  for (int64_t i = 0; i < v->n; ++i)
    for (int a = 0; a < v->A; ++a) env_legal(v, i, a, legal + ((size_t)i * v->A + a) * v->n_act);
  return 0;
}

int orc_random_actions(orc_venv* v, const uint32_t step_key[4], int32_t* actions) { /* vector_env.cpp:169-187 */
  uint8_t mask[256];
  for (int64_t i = 0; i < v->n; ++i) {
    uint32_t ek[4];
    orc_split_child(step_key, (uint64_t)(v->off + i), ek);
    for (int a = 0; a < v->A; ++a) {
      env_legal(v, i, a, mask);
      /* legal_uniform, vector_env.cpp:21-32 */
      int n_legal = 0;
      for (int q = 0; q < v->n_act; ++q) n_legal += mask[q] ? 1 : 0;
      if (n_legal == 0) return fail(3, "no legal action available");
      int pick = (int)(orc_bits(ek, (uint64_t)a) % (uint64_t)n_legal), chosen = v->n_act - 1;
      for (int q = 0; q < v->n_act; ++q) {
        if (!mask[q]) continue;
        if (pick == 0) { chosen = q; break; }
        --pick;
      }
      actions[i * v->A + a] = chosen;
    }
  }
  return 0;
}

static int env_n_actions(orc_venv* v, int a) {
  if (v->family == ORC_MPE) return mpe_n_actions(&v->mpe, a);
  if (v->family == ORC_SMAX) return smax_n_actions(&v->smax, a);
  return 6;
}

/* VectorEnv::step, vector_env.cpp:72-129 */
int orc_step(orc_venv* v, const int32_t* actions, float* obs, double* rewards, uint8_t* dones,
             uint8_t* finished, float* final_obs, double* final_returns, int32_t* final_lengths,
             double* infos) {
  int A = v->A;
  size_t row = (size_t)v->obs_dim;
  /* Env::validate_actions (env.cpp:7-14) for the whole batch first */
  for (int64_t i = 0; i < v->n; ++i)
    for (int a = 0; a < A; ++a) {
      int32_t x = actions[i * A + a];
      if (x < 0 || x >= env_n_actions(v, a)) return fail(3, "action is outside its action space");
    }
  double rew[128];
  double inf[128 * 3];
  for (int64_t i = 0; i < v->n; ++i) {
    uint32_t k0[4], k1[4], k2[4]; /* split(carry, 3): step / auto-reset / carry */
    orc_split_child(v->keys + 4 * i, 0, k0);
    orc_split_child(v->keys + 4 * i, 1, k1);
    orc_split_child(v->keys + 4 * i, 2, k2);
    const int32_t* act = actions + i * A;
    float* ob = v->scratch_obs;
    memset(ob, 0, sizeof(float) * row * A);
    int done = 0;
    if (v->family == ORC_MPE) {
      mpe_state next;
      done = mpe_step(&v->mpe, &v->mpe_s[i], act, &next, rew);
      v->mpe_s[i] = next;
      for (int a = 0; a < A; ++a) mpe_observe(&v->mpe, &next, a, ob + a * row);
    } else if (v->family == ORC_SMAX) {
      const smax_env* e = &v->smax;
      smax_view s = smax_at(v, i);
      int U = e->n;
      /* keep prev for reward_map and the heuristic (smax.cpp:224-240) */
      double prev_buf[4 * 128];
      int8_t prev_type[128];
      int16_t prev_pa[128], prev_tg[128];
      int8_t prev_sw[128];
      int prev_t = *s.t;
      int8_t prev_w = *s.winner;
      memcpy(prev_buf, s.x, sizeof(double) * 4 * U);
      memcpy(prev_type, s.type, (size_t)U);
      memcpy(prev_pa, s.prev_action, 2 * (size_t)U);
      memcpy(prev_tg, s.ai_target, 2 * (size_t)U);
      memcpy(prev_sw, s.ai_sweep, (size_t)U);
      smax_view prev = {prev_buf, prev_buf + U, prev_buf + 2 * U, prev_buf + 3 * U, prev_type,
                        prev_pa, prev_tg, prev_sw, &prev_t, &prev_w};
      int act_u[128];
      for (int u = 0; u < U; ++u) act_u[u] = kStop;
      for (int q = 0; q < e->na; ++q) act_u[q] = act[q];
      if (e->enemy_controlled) {
        for (int q = 0; q < e->ne; ++q) act_u[e->na + q] = act[e->na + q];
      } else {
        for (int q = 0; q < e->ne; ++q) {
          int u = e->na + q;
          int tg = prev.ai_target[u], sw = prev.ai_sweep[u];
          act_u[u] = heuristic_action(e, &prev, u, &tg, &sw);
          s.ai_target[u] = (int16_t)tg;
          s.ai_sweep[u] = (int8_t)sw;
        }
      }
      double dmg[128], h0[128];
      for (int tick = 0; tick < SMAX_TICKS; ++tick) simulate_tick(e, &s, act_u, tick == SMAX_TICKS - 1, dmg, h0);
      for (int u = 0; u < U; ++u) s.prev_action[u] = (int16_t)act_u[u];
      *s.t = prev_t + 1;
      int aa = alive_count(e, &s, 0), ea = alive_count(e, &s, 1);
      if (aa == 0 && ea == 0) *s.winner = 2;
      else if (ea == 0) *s.winner = 0;
      else if (aa == 0) *s.winner = 1;
      else if (*s.t >= e->max_steps) *s.winner = 2;
      for (int a = 0; a < A; ++a) smax_observe(e, &s, a, ob + a * row);
      /* reward_map, smax.cpp:352-363 */
      double ally_r = 0.5 * (smax_pool(e, &prev, 1) - smax_pool(e, &s, 1)) / (2.0 * e->ne);
      double enemy_r = 0.5 * (smax_pool(e, &prev, 0) - smax_pool(e, &s, 0)) / (2.0 * e->na);
      if (prev_w == -1 && *s.winner == 0) ally_r += 0.5;
      if (prev_w == -1 && *s.winner == 1) enemy_r += 0.5;
      for (int a = 0; a < A; ++a) {
        int team = team_of(e, a);
        rew[a] = team == 0 ? ally_r : enemy_r;
        inf[a * 3 + 0] = s.health[a] > 0.0 ? 1.0 : 0.0;   /* alive */
        inf[a * 3 + 1] = *s.winner == team ? 1.0 : 0.0;   /* battle_won */
        inf[a * 3 + 2] = *s.winner == 2 ? 1.0 : 0.0;      /* draw */
      }
      done = *s.winner != -1;
    } else {
      oc_view s = oc_at(v, i);
      double team, shaped[2];
      int deliv;
      done = oc_step(&v->oc, k0, &s, act, &team, shaped, &deliv);
      oc_store(v, i, &s);
      for (int a = 0; a < 2; ++a) {
        oc_encode(&v->oc, &s, a, ob + a * row);
        rew[a] = team;
        inf[a * 2 + 0] = (double)deliv;   /* deliveries */
        inf[a * 2 + 1] = shaped[a];       /* shaped_reward */
      }
    }
    /* team_reward (vector_env.cpp:14-18) + bookkeeping (vector_env.cpp:99-125) */
    double sum = 0;
    for (int a = 0; a < A; ++a) sum += rew[a];
    double ep_return = v->ep_ret[i] + sum / (double)A;
    int ep_length = v->ep_len[i] + 1;
    if (rewards) memcpy(rewards + i * A, rew, sizeof(double) * A);
    if (infos && v->n_info) memcpy(infos + i * A * v->n_info, inf, sizeof(double) * A * v->n_info);
    if (dones) {
      for (int a = 0; a < A; ++a) dones[i * (A + 1) + a] = (uint8_t)done;
      dones[i * (A + 1) + A] = (uint8_t)done;
    }
    if (finished) finished[i] = (uint8_t)done;
    if (done) {
      if (final_obs) memcpy(final_obs + (size_t)i * A * row, ob, sizeof(float) * row * A);
      if (final_returns) final_returns[i] = ep_return;
      if (final_lengths) final_lengths[i] = ep_length;
      env_reset(v, i, k1, obs ? obs + (size_t)i * A * row : NULL);
      v->ep_ret[i] = 0.0;
      v->ep_len[i] = 0;
    } else {
      if (obs) memcpy(obs + (size_t)i * A * row, ob, sizeof(float) * row * A);
      if (final_returns) final_returns[i] = 0.0;
      if (final_lengths) final_lengths[i] = 0;
      v->ep_ret[i] = ep_return;
      v->ep_len[i] = ep_length;
    }
    memcpy(v->keys + 4 * i, k2, sizeof k2);
  }
  return 0;
}

void orc_keys(const orc_venv* v, uint32_t* keys) { memcpy(keys, v->keys, sizeof(uint32_t) * 4 * (size_t)v->n); }
void orc_episode(const orc_venv* v, double* returns, int32_t* lengths) {
  if (returns) memcpy(returns, v->ep_ret, sizeof(double) * (size_t)v->n);
  if (lengths) memcpy(lengths, v->ep_len, sizeof(int32_t) * (size_t)v->n);
}
void orc_state_hash(const orc_venv* v, uint64_t* hashes) {
  orc_venv* m = (orc_venv*)v;
  for (int64_t i = 0; i < v->n; ++i) {
    if (v->family == ORC_MPE) hashes[i] = mpe_hash(&v->mpe, &v->mpe_s[i]);
    else if (v->family == ORC_SMAX) {
      smax_view s = smax_at(m, i);
      hashes[i] = smax_hash(&v->smax, &s);
    } else {
      oc_view s = oc_at(m, i);
      hashes[i] = oc_hash(&v->oc, &s);
    }
  }
}

int orc_smax_units(const orc_venv* v, int64_t env, double* x, double* y, double* health, double* cooldown) {
  if (v->family != ORC_SMAX) return fail(3, "not a SMAX env");
  smax_view s = smax_at((orc_venv*)v, env);
  int U = v->smax.n;
  memcpy(x, s.x, sizeof(double) * U);
  memcpy(y, s.y, sizeof(double) * U);
  memcpy(health, s.health, sizeof(double) * U);
  memcpy(cooldown, s.cooldown, sizeof(double) * U);
  return 0;
}
int orc_smax_winner(const orc_venv* v, int64_t env) {
  return v->family == ORC_SMAX ? v->swinner[env] : -2;
}
