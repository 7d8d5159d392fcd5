/* ut_oracle.c -- TEST INFRASTRUCTURE: plain-C restatement of the reference's
 * batched environment step (utrack, /root/reference/proj/core). Used only as the
 * checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
 *
 * Every function cites the reference lines it restates. Numerical contract: one
 * IEEE op per source operation, no contraction (-ffp-contract=off), sequential
 * reductions, glibc fp64 libm, correctly-rounded fp32 log/sin/cos -- the same
 * definition as oracle/eigen_shim (so this file and oracle/_ref agree bit for bit,
 * tests/test_oracle_pinning.py).
 *
 * Batch semantics follow VecEnv (vecenv.cpp) with one declared superset: the
 * self-driven step (step_policy) also refreshes obs/global/infos/final_obs, which
 * the reference leaves stale (vecenv.cpp:118-143 gathers masks only).
 */
#include "ut_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define UTO_PI 3.14159265358979323846
#define UTO_TWO_PI (2.0 * UTO_PI)

static _Thread_local char g_err[512];

static int set_err(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}
const char* uto_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ RNG --- */
/* rng.hpp:127-133 */
static uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* rng.hpp:30-38 */
uint64_t uto_derive_key(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  const uint64_t v[4] = {a, b, c, d};
  uint64_t h = 0x9e3779b97f4a7c15ull;
  for (int i = 0; i < 4; ++i) {
    h ^= splitmix64(v[i] + h);
    h = (h << 23) | (h >> 41);
  }
  return splitmix64(h);
}

/* rng.hpp:116-131, 141-158: Philox4x32-10, counter {block lo, hi, stream lo, hi} */
void uto_philox_block(uint64_t key, uint64_t stream, uint64_t block, uint32_t out[4]) {
  uint32_t c0 = (uint32_t)block, c1 = (uint32_t)(block >> 32);
  uint32_t c2 = (uint32_t)stream, c3 = (uint32_t)(stream >> 32);
  uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

typedef struct {
  uint64_t key, stream, pos;
  int have_spare;
  double spare;
  uint32_t buf[4];
  int buf_valid;
} uto_rng;

static void rng_init(uto_rng* r, uint64_t key, uint64_t stream) {
  memset(r, 0, sizeof *r);
  r->key = key;
  r->stream = stream;
}
/* rng.hpp:40-48 */
static uint32_t next_u32(uto_rng* r) {
  const int lane = (int)(r->pos & 3);
  if (lane == 0 || !r->buf_valid) {
    uto_philox_block(r->key, r->stream, r->pos >> 2, r->buf);
    r->buf_valid = 1;
  }
  ++r->pos;
  return r->buf[lane];
}
/* rng.hpp:50-54 */
static uint64_t next_u64(uto_rng* r) {
  const uint64_t lo = next_u32(r);
  const uint64_t hi = next_u32(r);
  return (hi << 32) | lo;
}
/* rng.hpp:57-64 */
static double uniform(uto_rng* r) { return (double)(next_u64(r) >> 11) * 0x1.0p-53; }
static double uniform_pos(uto_rng* r) { return 1.0 - uniform(r); }
static double uniform_range(uto_rng* r, double lo, double hi) { return lo + (hi - lo) * uniform(r); }
/* rng.hpp:67-79 */
static double normal(uto_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  const double u1 = uniform_pos(r);
  const double u2 = uniform(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double a = UTO_TWO_PI * u2;
  r->spare = rad * sin(a);
  r->have_spare = 1;
  return rad * cos(a);
}
/* rng.hpp:82-96 */
static uint32_t uniform_int(uto_rng* r, uint32_t n) {
  uint64_t x = next_u32(r);
  uint64_t m = x * n;
  uint32_t l = (uint32_t)m;
  if (l < n) {
    const uint32_t floor_ = (uint32_t)(-n) % n;
    while (l < floor_) {
      x = next_u32(r);
      m = x * n;
      l = (uint32_t)m;
    }
  }
  return (uint32_t)(m >> 32);
}
/* rng.hpp:99-104, then the int cast at the call sites (env.cpp:206, 296): the
 * u64 -> int conversion keeps the low 32 bits (GCC/nvcc behaviour), made explicit. */
static int32_t geometric_i32(uto_rng* r, double mean_value) {
  const double p = 1.0 / mean_value;
  const double u = uniform_pos(r);
  const double k = ceil(log(u) / log1p(-p));
  const uint64_t g = k < 1.0 ? 1u : (uint64_t)k;
  return (int32_t)(uint32_t)g;
}
/* rng.hpp:106-112 */
static void rng_restore(uto_rng* r, uint64_t pos, int have_spare, double spare) {
  r->pos = pos;
  r->have_spare = have_spare;
  r->spare = spare;
  r->buf_valid = 0;
}

/* --------------------------------------- correctly-rounded fp32 math --- */
float uto_cr_logf(float x) { return (float)log((double)x); }
float uto_cr_cosf(float x) { return (float)cos((double)x); }
float uto_cr_sinf(float x) { return (float)sin((double)x); }

/* The whole 2^24-point input grid of one noise transcendental (tracking.cpp:29-36):
 * kind 0: log(((i)+1) 2^-24); 1: cos(2pi_f i 2^-24); 2: sin(2pi_f i 2^-24). */
void uto_cr_grid(int kind, float* out) {
  const float two_pi_f = 2.0f * (float)UTO_PI;
  for (uint32_t i = 0; i < (1u << 24); ++i) {
    if (kind == 0 || kind == 3) {
      const float l = uto_cr_logf((float)(i + 1u) * 0x1.0p-24f);
      out[i] = kind == 0 ? l : sqrtf(-2.0f * l);
    } else {
      const float a = two_pi_f * ((float)i * 0x1.0p-24f);
      out[i] = kind == 1 ? uto_cr_cosf(a) : uto_cr_sinf(a);
    }
  }
}

/* ---------------------------------------------------------- kinematics --- */
/* kinematics.cpp:13-18 */
static double wrap_angle(double psi) {
  double w = fmod(psi + UTO_PI, UTO_TWO_PI);
  if (w <= 0.0) w += UTO_TWO_PI;
  return w - UTO_PI;
}

typedef struct {
  double x, y, z, heading, speed;
  int32_t rudder;
} uto_vehicle;

/* kinematics.cpp:42-49 */
static void advance_vehicle(uto_vehicle* v, double dpsi, double dt, double noise) {
  v->heading = wrap_angle(v->heading + dpsi + noise);
  v->x += v->speed * dt * cos(v->heading);
  v->y += v->speed * dt * sin(v->heading);
}

/* Eigen fixed-size redux order (see eigen_shim): x^2 + (y^2 + z^2) */
static double norm3(double dx, double dy, double dz) { return sqrt(dx * dx + (dy * dy + dz * dz)); }
static double norm2(double dx, double dy) { return sqrt(dx * dx + dy * dy); }

/* --------------------------------------------------------- config --- */
/* env_config.hpp:36-80 */
void uto_config_default(ut_env_config* c) {
  memset(c, 0, sizeof *c);
  c->n_agents = 1;
  c->n_targets = 1;
  c->horizon = 128;
  c->dt = 30.0;
  c->agent_speed = 1.0;
  c->target_speed_frac = 0.3;
  c->target_speed_frac_max = 0.0;
  c->target_turn_interval = 20.0;
  c->detection_range = 450.0;
  c->comm_range = 1500.0;
  c->comm_drop_prob = 0.1;
  c->range_noise_std = 3.0;
  c->eps_min = 10.0;
  c->eps_max = 50.0;
  c->d_min = 50.0;
  c->d_safe = 10.0;
  c->reward_mode = UT_REWARD_TRACKING;
  c->spawn_min_sep = 50.0;
  c->spawn_max_sep = 200.0;
  c->perturbation_std = 0.0;
  c->target_depth_min = 10.0;
  c->target_depth_max = 60.0;
  c->lost_steps = 20;
  c->heading_model_kind = UT_HEADING_DEFAULT;
  c->heading_noise_std = 0.02;
  c->pf.n_particles = 1024;
  c->pf.process_noise_pos = 1.0;
  c->pf.process_noise_vel = 0.05;
  c->pf.speed_margin = 1.2;
  c->pf.init_radius = 450.0;
}

/* Default model bucket (speed, dt): OLS over synth_calibration(speeds, dts, 201, 0, 0)
 * rows of that bucket (kinematics.cpp:58-111, 131-154, 180-186). Returns 0 if the
 * (speed, dt) pair is not a shipped bucket. */
static int default_bucket(double speed, double dt, double* a_out, double* b_out) {
  static const double speeds[] = {0.5, 0.75, 1.0, 1.25, 1.5, 2.0};
  static const double dts[] = {10.0, 15.0, 30.0, 60.0};
  int found = 0;
  for (int i = 0; i < 6; ++i)
    if (speeds[i] == speed) found |= 1;
  for (int i = 0; i < 4; ++i)
    if (dts[i] == dt) found |= 2;
  if (found != 3) return 0;
  const int rows = 201;
  const double kmax = 0.24, gain = 0.15;
  double sx = 0.0, sy = 0.0, sxx = 0.0, sxy = 0.0;
  for (int i = 0; i < rows; ++i) {
    const double t = (double)i / (rows - 1);
    const double gamma = -kmax + 2.0 * kmax * t;             /* kinematics.cpp:137 */
    const double dpsi = gain * speed * dt * tan(gamma) + 0.0; /* kinematics.cpp:119, 140-141 */
    sx += gamma;
    sy += dpsi;
    sxx += gamma * gamma;
    sxy += gamma * dpsi;
  }
  const double n = (double)rows;
  const double denom = n * sxx - sx * sx;
  const double a = (n * sxy - sx * sy) / denom;
  const double b = (sy - a * sx) / n;
  *a_out = a;
  *b_out = b;
  return 1;
}

/* EnvConfig::finalize (env.cpp:40-65) + max turn (env.cpp:115-116) */
int uto_config_finalize(ut_env_config* c) {
#define UTO_REQ(cond, msg) \
  if (!(cond)) return set_err(UT_ERR_CONFIG, "%s", msg)
  if (c->heading_noise_std < 0.0) return set_err(UT_ERR_CONFIG, "heading model noise_std must be >= 0");
  UTO_REQ(c->n_agents >= 1, "env.n_agents must be >= 1");
  UTO_REQ(c->n_targets >= 1, "env.n_targets must be >= 1");
  UTO_REQ(c->horizon >= 1, "env.horizon must be >= 1");
  UTO_REQ(c->dt > 0.0, "env.dt must be > 0");
  UTO_REQ(c->agent_speed > 0.0, "env.agent_speed must be > 0");
  UTO_REQ(c->target_speed_frac >= 0.0, "env.target_speed_frac must be >= 0");
  UTO_REQ(c->target_turn_interval >= 1.0, "env.target_turn_interval must be >= 1 step");
  UTO_REQ(c->eps_min < c->eps_max, "env.eps_min must be < env.eps_max");
  UTO_REQ(c->spawn_min_sep < c->spawn_max_sep, "env.spawn_min_sep must be < env.spawn_max_sep");
  UTO_REQ(!(c->comm_drop_prob < 0.0 || c->comm_drop_prob > 1.0), "env.comm_drop_prob must be in [0, 1]");
  UTO_REQ(c->range_noise_std >= 0.0, "env.range_noise_std must be >= 0");
  UTO_REQ(!(c->target_depth_min < 0.0 || c->target_depth_max < c->target_depth_min),
          "env.target_depth band must satisfy 0 <= min <= max");
  UTO_REQ(c->lost_steps >= 1, "env.lost_steps must be >= 1");
  UTO_REQ(c->pf.n_particles >= 1, "env.pf.n_particles must be >= 1");
  UTO_REQ(c->pf.init_radius > 0.0, "env.pf.init_radius must be > 0");
#undef UTO_REQ
  if (c->heading_model_kind == UT_HEADING_DEFAULT) {
    double a, b;
    if (!default_bucket(c->agent_speed, c->dt, &a, &b))
      return set_err(UT_ERR_CONFIG, "heading model has no bucket for (speed=%g m/s, dt=%g s)", c->agent_speed, c->dt);
    c->heading_a = a;
    c->heading_b = b;
  }
  c->max_turn_per_step = fabs(c->heading_a * 0.24 + c->heading_b);
  return UT_OK;
}

/* ------------------------------------------------------------- state --- */
typedef struct {
  double x, y, z, heading;
  int32_t age;
  uint8_t valid;
} uto_info; /* env.hpp:19-25 */

typedef struct {
  double ox, oy, r2, sigma;
} uto_meas; /* tracking.hpp:14-19 */

typedef struct {
  uto_rng rng;
  double max_speed;
  double est_x, est_y, spread; /* TrackEstimate, tracking.hpp:29-33 */
  int32_t age;
  uint8_t ever;
} uto_set;

typedef struct {
  int64_t index; /* global env index (stream key) */
  uto_rng rng, bench;
  double episode_target_speed;
  int32_t step;
  uto_vehicle* agents;   /* [A] */
  uto_vehicle* targets;  /* [T] */
  int32_t* countdown;    /* [T] TargetMotion */
  double* cmd_heading;   /* [T] */
  int32_t* miss_streak;  /* [T] */
  uto_info* info;        /* [A][A] */
  uto_set* sets;         /* [A][T] */
  uint8_t* present;      /* [A][T] meas_present_ */
  uint8_t* fresh;        /* [A][T] meas_fresh_age_ */
  uto_meas* meas;        /* [A][T] */
  /* StepOutput (env.hpp:53-60) */
  double reward;
  uint8_t done, collision;
  double *err, *dist;
  uint8_t* lost;
  double episode_return; /* stats only */
  double ev_dist, ev_err; /* evaluation accumulators (curriculum.cpp:286-325) */
  int ev_flags;
} uto_env;

struct uto_vecenv {
  ut_env_config cfg;
  int64_t n;
  int32_t A, T, R, P;
  uto_env* envs;
  double *px, *py, *vx, *vy, *w; /* [set][P] */
  /* scratch */
  float* noise;  /* 4P */
  double *loglik, *sx, *sy, *svx, *svy;
  /* batch buffers (vecenv.hpp:79-84), column-major */
  double *obs, *final_obs, *global;
  double* rewards;
  uint8_t *dones, *masks;
  double stats[UT_N_STATS];
};

static int64_t set_index(const uto_vecenv* v, int64_t e, int a, int t) {
  return (e * v->A + a) * v->T + t;
}

/* ----------------------------------------------------- particle filter --- */
typedef struct {
  double *px, *py, *vx, *vy, *w;
  int64_t n;
  uto_set* s;
} pfview;

static pfview pf_view(uto_vecenv* v, int64_t e, int a, int t) {
  const int64_t si = set_index(v, e, a, t);
  pfview p;
  p.n = v->P;
  p.px = v->px + si * v->P;
  p.py = v->py + si * v->P;
  p.vx = v->vx + si * v->P;
  p.vy = v->vy + si * v->P;
  p.w = v->w + si * v->P;
  p.s = &v->envs[e].sets[a * v->T + t];
  return p;
}

/* tracking.cpp:76-92 */
static void pf_reinit(pfview* p, double cx, double cy, double radius, double max_speed) {
  p->s->max_speed = max_speed;
  const double inv = 1.0 / (double)p->n;
  for (int64_t i = 0; i < p->n; ++i) p->w[i] = inv;
  for (int64_t i = 0; i < p->n; ++i) {
    const double r = radius * sqrt(uniform(&p->s->rng));
    const double a = UTO_TWO_PI * uniform(&p->s->rng);
    p->px[i] = cx + r * cos(a);
    p->py[i] = cy + r * sin(a);
    const double sp = max_speed * uniform(&p->s->rng);
    const double d = UTO_TWO_PI * uniform(&p->s->rng);
    p->vx[i] = sp * cos(d);
    p->vy[i] = sp * sin(d);
  }
}

/* tracking.cpp:24-37 */
static void fill_normals(uto_rng* rng, float* out, int64_t m) {
  const int64_t half = m / 2;
  float* stage = (float*)malloc(sizeof(float) * (size_t)m);
  float* u1 = stage;
  float* u2 = stage + half;
  for (int64_t i = 0; i < half; ++i) u1[i] = (float)((next_u32(rng) >> 8) + 1) * 0x1.0p-24f;
  for (int64_t i = 0; i < half; ++i) u2[i] = (float)(next_u32(rng) >> 8) * 0x1.0p-24f;
  const float two_pi_f = 2.0f * (float)UTO_PI;
  for (int64_t i = 0; i < half; ++i) {
    const float r = sqrtf((-2.0f) * uto_cr_logf(u1[i]));
    const float a = two_pi_f * u2[i];
    out[i] = r * uto_cr_cosf(a);
    out[half + i] = r * uto_cr_sinf(a);
  }
  free(stage);
}

void uto_fill_normals(uint64_t key, uint64_t stream, uint64_t pos, int64_t n, float* out) {
  uto_rng r;
  rng_init(&r, key, stream);
  rng_restore(&r, pos, 0, 0.0);
  fill_normals(&r, out, 4 * n);
}

/* tracking.cpp:94-117 */
static void pf_predict(uto_vecenv* v, pfview* p, double dt, double pn, double vn) {
  const int64_t n = p->n;
  for (int64_t i = 0; i < n; ++i) p->px[i] = p->px[i] + p->vx[i] * dt;
  for (int64_t i = 0; i < n; ++i) p->py[i] = p->py[i] + p->vy[i] * dt;
  if (pn > 0.0 || vn > 0.0) {
    fill_normals(&p->s->rng, v->noise, 4 * n);
    for (int64_t i = 0; i < n; ++i) p->px[i] = p->px[i] + pn * (double)v->noise[i];
    for (int64_t i = 0; i < n; ++i) p->py[i] = p->py[i] + pn * (double)v->noise[n + i];
    for (int64_t i = 0; i < n; ++i) p->vx[i] = p->vx[i] + vn * (double)v->noise[2 * n + i];
    for (int64_t i = 0; i < n; ++i) p->vy[i] = p->vy[i] + vn * (double)v->noise[3 * n + i];
  }
  if (p->s->max_speed > 0.0) {
    const double ms = p->s->max_speed;
    for (int64_t i = 0; i < n; ++i) {
      const double s = sqrt(p->vx[i] * p->vx[i] + p->vy[i] * p->vy[i]);
      const double f = (s > ms) ? ms / s : 1.0;
      p->vx[i] = p->vx[i] * f;
      p->vy[i] = p->vy[i] * f;
    }
  }
}

/* tracking.cpp:119-143 with a single measurement (the env always passes one) */
static int pf_update(uto_vecenv* v, pfview* p, const uto_meas* m) {
  const int64_t n = p->n;
  double* ll = v->loglik;
  for (int64_t i = 0; i < n; ++i) {
    const double dx = p->px[i] - m->ox, dy = p->py[i] - m->oy;
    const double d = sqrt(dx * dx + dy * dy);
    const double q = (d - m->r2) / m->sigma;
    ll[i] = 0.0 - 0.5 * (q * q);
  }
  double shift = ll[0];
  for (int64_t i = 1; i < n; ++i)
    if (ll[i] > shift) shift = ll[i];
  if (isfinite(shift)) {
    for (int64_t i = 0; i < n; ++i) p->w[i] = p->w[i] * exp(ll[i] - shift);
    double sum = p->w[0];
    for (int64_t i = 1; i < n; ++i) sum = sum + p->w[i];
    if (isfinite(sum) && sum > 0.0) {
      for (int64_t i = 0; i < n; ++i) p->w[i] = p->w[i] / sum;
      return 0;
    }
  }
  const double inv = 1.0 / (double)n;
  for (int64_t i = 0; i < n; ++i) p->w[i] = inv;
  return 1;
}

/* tracking.cpp:145-178 */
static int pf_maybe_resample(uto_vecenv* v, pfview* p) {
  const int64_t n = p->n;
  double s2 = p->w[0] * p->w[0];
  for (int64_t i = 1; i < n; ++i) s2 = s2 + p->w[i] * p->w[i];
  const double ess = 1.0 / s2;
  if (getenv("UTO_TRACE")) fprintf(stderr, "[oracle] ess=%.17g resample=%d pos=%llu\n", ess, ess < (double)n / 2.0,
                                   (unsigned long long)p->s->rng.pos);
  if (!(ess < (double)n / 2.0)) return 0;
  const double u0 = uniform(&p->s->rng);
  const double inv_n = 1.0 / (double)n;
  int64_t i = 0;
  double cum = p->w[0];
  for (int64_t j = 0; j < n; ++j) {
    const double u = ((double)j + u0) * inv_n;
    while (cum < u && i < n - 1) {
      ++i;
      cum += p->w[i];
    }
    v->sx[j] = p->px[i];
    v->sy[j] = p->py[i];
    v->svx[j] = p->vx[i];
    v->svy[j] = p->vy[i];
  }
  memcpy(p->px, v->sx, sizeof(double) * (size_t)n);
  memcpy(p->py, v->sy, sizeof(double) * (size_t)n);
  memcpy(p->vx, v->svx, sizeof(double) * (size_t)n);
  memcpy(p->vy, v->svy, sizeof(double) * (size_t)n);
  for (int64_t k = 0; k < n; ++k) p->w[k] = inv_n;
  return 1;
}

/* tracking.cpp:180-188 */
static void pf_estimate(pfview* p) {
  const int64_t n = p->n;
  double mx = p->w[0] * p->px[0];
  for (int64_t i = 1; i < n; ++i) mx = mx + p->w[i] * p->px[i];
  double my = p->w[0] * p->py[0];
  for (int64_t i = 1; i < n; ++i) my = my + p->w[i] * p->py[i];
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double dx = p->px[i] - mx, dy = p->py[i] - my;
    const double term = p->w[i] * (dx * dx + dy * dy);
    acc = (i == 0) ? term : acc + term;
  }
  p->s->est_x = mx;
  p->s->est_y = my;
  p->s->spread = sqrt(acc);
}

/* --------------------------------------------------------- environment --- */
static double rudder_angle(int idx) { return -0.24 + 0.12 * idx; } /* env.cpp:67-72 */
static int valid_action(int rudder, int act) {                     /* env.cpp:74-81 */
  return act >= 0 && act < UT_NUM_ACTIONS && abs(act - rudder) <= 1;
}

/* env.cpp:83-90 */
static double tracking_reward_single(double e, const ut_env_config* c) {
  if (e < c->eps_min) return 1.0;
  if (e > c->eps_max) return 0.0;
  const double t = (e - c->eps_min) / (c->eps_max - c->eps_min);
  if (t >= 1.0) return 0.0;
  return exp(-2.0 * t / (1.0 - t));
}

static void setc(double* m, int64_t rows, int64_t r, int c, double x) { m[(int64_t)c * rows + r] = x; }

/* env.cpp:412-453, written straight into the batch buffer rows
 * ((e * A + agent) * R + row) (vecenv.cpp:47-53) */
static void build_observation(uto_vecenv* v, int64_t e, int agent, double* obs) {
  const uto_env* E = &v->envs[e];
  const int A = v->A, T = v->T, R = v->R;
  const int64_t rows = v->n * A * R;
  const int64_t base = (e * A + agent) * R;
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < UT_FEATURE_DIM; ++c) setc(obs, rows, base + r, c, 0.0);
  const uto_vehicle* self = &E->agents[agent];
  for (int j = 0; j < A; ++j) {
    const int64_t row = base + j;
    if (j == agent) {
      setc(obs, rows, row, 3, sin(self->heading));
      setc(obs, rows, row, 4, cos(self->heading));
      setc(obs, rows, row, 5, self->speed / 1.0);
      setc(obs, rows, row, 6, 1.0);
      setc(obs, rows, row, 9, 1.0);
      continue;
    }
    setc(obs, rows, row, 7, 1.0);
    const uto_info* in = &E->info[agent * A + j];
    if (!in->valid) continue;
    setc(obs, rows, row, 0, (in->x - self->x) / 1000.0);
    setc(obs, rows, row, 1, (in->y - self->y) / 1000.0);
    setc(obs, rows, row, 2, (in->z - self->z) / 1000.0);
    setc(obs, rows, row, 3, sin(in->heading));
    setc(obs, rows, row, 4, cos(in->heading));
    setc(obs, rows, row, 5, v->cfg.agent_speed / 1.0);
    setc(obs, rows, row, 9, 1.0);
    setc(obs, rows, row, 10, (double)in->age / 10.0);
  }
  for (int t = 0; t < T; ++t) {
    const int64_t row = base + A + t;
    setc(obs, rows, row, 8, 1.0);
    const uto_set* s = &E->sets[agent * T + t];
    if (!s->ever) continue;
    const uto_vehicle* tv = &E->targets[t];
    setc(obs, rows, row, 0, (s->est_x - self->x) / 1000.0);
    setc(obs, rows, row, 1, (s->est_y - self->y) / 1000.0);
    setc(obs, rows, row, 2, (tv->z - self->z) / 1000.0);
    setc(obs, rows, row, 9, 1.0);
    setc(obs, rows, row, 10, (double)s->age / 10.0);
    setc(obs, rows, row, 11, s->spread / 100.0);
  }
}

/* env.cpp:455-471 into rows (e * R + row) (vecenv.cpp:55) */
static void build_global_state(uto_vecenv* v, int64_t e) {
  const uto_env* E = &v->envs[e];
  const int A = v->A, R = v->R;
  const int64_t rows = v->n * R;
  for (int r = 0; r < R; ++r) {
    const uto_vehicle* x = r < A ? &E->agents[r] : &E->targets[r - A];
    const int64_t row = e * R + r;
    for (int c = 0; c < UT_FEATURE_DIM; ++c) setc(v->global, rows, row, c, 0.0);
    setc(v->global, rows, row, 0, x->x / 1000.0);
    setc(v->global, rows, row, 1, x->y / 1000.0);
    setc(v->global, rows, row, 2, x->z / 1000.0);
    setc(v->global, rows, row, 3, sin(x->heading));
    setc(v->global, rows, row, 4, cos(x->heading));
    setc(v->global, rows, row, 5, x->speed / 1.0);
    setc(v->global, rows, row, r < A ? 7 : 8, 1.0);
    setc(v->global, rows, row, 9, 1.0);
  }
}

static void gather(uto_vecenv* v, int64_t e) {
  for (int a = 0; a < v->A; ++a) build_observation(v, e, a, v->obs);
  build_global_state(v, e);
}
static void gather_masks(uto_vecenv* v, int64_t e) { /* vecenv.cpp:58-67 */
  for (int a = 0; a < v->A; ++a)
    for (int k = 0; k < UT_NUM_ACTIONS; ++k)
      v->masks[(e * v->A + a) * UT_NUM_ACTIONS + k] = (uint8_t)valid_action(v->envs[e].agents[a].rudder, k);
}

/* env.cpp:153-233 */
static int spawn(uto_vecenv* v, int64_t e) {
  uto_env* E = &v->envs[e];
  const ut_env_config* c = &v->cfg;
  const int A = v->A, T = v->T, R = v->R;
  const double lo = c->agent_speed * c->target_speed_frac;
  const double hi = c->agent_speed * (c->target_speed_frac_max > c->target_speed_frac ? c->target_speed_frac_max
                                                                                       : c->target_speed_frac);
  E->episode_target_speed = lo;
  if (hi > lo) E->episode_target_speed = uniform_range(&E->rng, lo, hi);

  const double disc_r = c->spawn_max_sep / 2.0;
  double px[64], py[64];
  double* qx = R <= 64 ? px : (double*)malloc(sizeof(double) * (size_t)R);
  double* qy = R <= 64 ? py : (double*)malloc(sizeof(double) * (size_t)R);
  int placed = 0;
  for (int attempt = 0; attempt < 1000 && !placed; ++attempt) {
    for (int i = 0; i < R; ++i) {
      const double r = disc_r * sqrt(uniform(&E->rng));
      const double a = UTO_TWO_PI * uniform(&E->rng);
      qx[i] = r * cos(a);
      qy[i] = r * sin(a);
    }
    placed = 1;
    for (int i = 0; i + 1 < R && placed; ++i)
      for (int j = i + 1; j < R && placed; ++j)
        if (norm2(qx[i] - qx[j], qy[i] - qy[j]) < c->spawn_min_sep) placed = 0;
  }
  if (!placed) {
    if (qx != px) free(qx), free(qy);
    return set_err(UT_ERR_CONFIG, "spawn infeasible after 1000 attempts: %d entities with separation in [%g, %g] m",
                   R, c->spawn_min_sep, c->spawn_max_sep);
  }
  for (int a = 0; a < A; ++a) {
    uto_vehicle* ag = &E->agents[a];
    ag->x = qx[a];
    ag->y = qy[a];
    ag->z = 0.0;
    ag->heading = wrap_angle(UTO_TWO_PI * uniform(&E->rng));
    ag->speed = c->agent_speed;
    ag->rudder = 2;
  }
  for (int t = 0; t < T; ++t) {
    uto_vehicle* tv = &E->targets[t];
    const double depth = uniform_range(&E->rng, c->target_depth_min, c->target_depth_max);
    tv->x = qx[A + t];
    tv->y = qy[A + t];
    tv->z = depth;
    tv->heading = wrap_angle(UTO_TWO_PI * uniform(&E->rng));
    tv->speed = E->episode_target_speed;
    tv->rudder = 2;
    E->cmd_heading[t] = tv->heading;
    E->countdown[t] = geometric_i32(&E->rng, c->target_turn_interval);
  }
  if (qx != px) free(qx), free(qy);

  const double particle_speed = c->pf.speed_margin * E->episode_target_speed;
  for (int a = 0; a < A; ++a) {
    for (int j = 0; j < A; ++j) memset(&E->info[a * A + j], 0, sizeof(uto_info));
    for (int t = 0; t < T; ++t) {
      pfview p = pf_view(v, e, a, t);
      pf_reinit(&p, E->agents[a].x, E->agents[a].y, c->pf.init_radius, particle_speed);
      pf_estimate(&p);
      p.s->age = 0;
      p.s->ever = 0;
    }
  }
  for (int t = 0; t < T; ++t) E->miss_streak[t] = 0;
  memset(E->present, 0, (size_t)(A * T));
  E->step = 0;
  E->reward = 0.0;
  E->done = 0;
  E->collision = 0;
  E->episode_return = 0.0;
  E->ev_dist = 0.0;
  E->ev_err = 0.0;
  E->ev_flags = 0;
  return UT_OK;
}

/* env.cpp:289-304 */
static void move_targets(uto_vecenv* v, uto_env* E) {
  const ut_env_config* c = &v->cfg;
  for (int t = 0; t < v->T; ++t) {
    uto_vehicle* tv = &E->targets[t];
    if (E->countdown[t] <= 0) {
      E->cmd_heading[t] = wrap_angle(UTO_TWO_PI * uniform(&E->rng));
      E->countdown[t] = geometric_i32(&E->rng, c->target_turn_interval);
    }
    const double want = wrap_angle(E->cmd_heading[t] - tv->heading);
    const double mt = c->max_turn_per_step;
    const double dpsi = want < -mt ? -mt : (mt < want ? mt : want); /* std::clamp */
    const double sigma = c->heading_noise_std;
    const double noise = sigma > 0.0 ? sigma * normal(&E->rng) : 0.0;
    advance_vehicle(tv, dpsi, c->dt, noise);
    E->countdown[t] -= 1;
  }
}

/* env.cpp:306-316 */
static void move_agents(uto_vecenv* v, uto_env* E, const int32_t* actions) {
  const ut_env_config* c = &v->cfg;
  for (int a = 0; a < v->A; ++a) {
    uto_vehicle* ag = &E->agents[a];
    ag->rudder = actions[a];
    const double gamma = rudder_angle(ag->rudder);
    const double sigma = c->heading_noise_std;
    double noise = sigma > 0.0 ? sigma * normal(&E->rng) : 0.0;
    if (c->perturbation_std > 0.0) noise += c->perturbation_std * normal(&E->rng);
    const double dpsi = c->heading_a * gamma + c->heading_b; /* kinematics.cpp:36-40 */
    advance_vehicle(ag, dpsi, c->dt, noise);
  }
}

/* env.cpp:318-347 */
static void measure_ranges(uto_vecenv* v, uto_env* E) {
  const ut_env_config* c = &v->cfg;
  const int A = v->A, T = v->T;
  for (int t = 0; t < T; ++t) {
    int detected = 0;
    for (int a = 0; a < A; ++a) {
      const int idx = a * T + t;
      E->present[idx] = 0;
      const uto_vehicle* av = &E->agents[a];
      const uto_vehicle* tv = &E->targets[t];
      const double dist3 = norm3(av->x - tv->x, av->y - tv->y, av->z - tv->z);
      if (dist3 > c->detection_range) continue;
      if (c->comm_drop_prob > 0.0 && uniform(&E->rng) < c->comm_drop_prob) continue;
      double r3 = dist3;
      if (c->range_noise_std > 0.0) r3 += c->range_noise_std * normal(&E->rng);
      r3 = r3 < 0.0 ? 0.0 : r3; /* std::max(r3, 0.0) */
      const double dd = tv->z - av->z;
      const double sq = r3 * r3 - dd * dd; /* tracking.cpp:9-14 */
      const double r2 = sq <= 0.0 ? 0.0 : sqrt(sq);
      uto_meas* m = &E->meas[idx];
      m->ox = av->x;
      m->oy = av->y;
      m->r2 = r2;
      m->sigma = c->range_noise_std < 0.1 ? 0.1 : c->range_noise_std;
      E->present[idx] = 1;
      detected = 1;
    }
    E->miss_streak[t] = detected ? 0 : E->miss_streak[t] + 1;
  }
}

/* env.cpp:349-363 */
static void filter_step(uto_vecenv* v, int64_t e) {
  uto_env* E = &v->envs[e];
  const ut_env_config* c = &v->cfg;
  for (int a = 0; a < v->A; ++a)
    for (int t = 0; t < v->T; ++t) {
      const int idx = a * v->T + t;
      pfview p = pf_view(v, e, a, t);
      pf_predict(v, &p, c->dt, c->pf.process_noise_pos, c->pf.process_noise_vel);
      E->fresh[idx] = 0;
      if (E->present[idx]) {
        pf_update(v, &p, &E->meas[idx]);
        v->stats[UT_STAT_PF_UPDATES] += 1.0;
        E->fresh[idx] = 1;
      }
    }
}

/* env.cpp:365-410 */
static void exchange_comms(uto_vecenv* v, int64_t e) {
  uto_env* E = &v->envs[e];
  const ut_env_config* c = &v->cfg;
  const int A = v->A, T = v->T;
  for (int i = 0; i < A * A; ++i) E->info[i].age += 1;
  for (int r = 0; r < A; ++r) {
    for (int s = 0; s < A; ++s) {
      if (s == r) continue;
      const uto_vehicle* rv = &E->agents[r];
      const uto_vehicle* sv = &E->agents[s];
      if (norm3(rv->x - sv->x, rv->y - sv->y, rv->z - sv->z) > c->comm_range) continue;
      if (c->comm_drop_prob > 0.0 && uniform(&E->rng) < c->comm_drop_prob) continue;
      uto_info* in = &E->info[r * A + s];
      in->x = sv->x;
      in->y = sv->y;
      in->z = sv->z;
      in->heading = sv->heading;
      in->age = 0;
      in->valid = 1;
      for (int t = 0; t < T; ++t) {
        if (!E->present[s * T + t]) continue;
        pfview p = pf_view(v, e, r, t);
        pf_update(v, &p, &E->meas[s * T + t]);
        v->stats[UT_STAT_PF_UPDATES] += 1.0;
        E->fresh[r * T + t] = 1;
      }
    }
  }
  for (int a = 0; a < A; ++a)
    for (int t = 0; t < T; ++t) {
      const int idx = a * T + t;
      pfview p = pf_view(v, e, a, t);
      v->stats[UT_STAT_PF_RESAMPLES] += (double)pf_maybe_resample(v, &p);
      const int32_t prev_age = p.s->age;
      pf_estimate(&p);
      p.s->age = E->fresh[idx] ? 0 : prev_age + 1;
      p.s->ever = (uint8_t)(p.s->ever || E->fresh[idx]);
    }
}

/* env.cpp:473-505 */
static void compute_reward_and_info(uto_vecenv* v, uto_env* E) {
  const ut_env_config* c = &v->cfg;
  const int A = v->A, T = v->T;
  for (int t = 0; t < T; ++t) {
    const uto_vehicle* tv = &E->targets[t];
    double best_err = INFINITY;
    for (int a = 0; a < A; ++a) {
      const uto_set* s = &E->sets[a * T + t];
      const double d = norm2(s->est_x - tv->x, s->est_y - tv->y);
      best_err = d < best_err ? d : best_err; /* std::min */
    }
    E->err[t] = best_err;
    double best_dist = INFINITY;
    for (int a = 0; a < A; ++a) {
      const double d = hypot(E->agents[a].x - tv->x, E->agents[a].y - tv->y);
      best_dist = d < best_dist ? d : best_dist;
    }
    E->dist[t] = best_dist;
    E->lost[t] = (uint8_t)(E->miss_streak[t] >= c->lost_steps);
  }
  int crash = 0;
  for (int i = 0; i + 1 < A && !crash; ++i)
    for (int j = i + 1; j < A && !crash; ++j) {
      const uto_vehicle *p = &E->agents[i], *q = &E->agents[j];
      if (norm3(p->x - q->x, p->y - q->y, p->z - q->z) < c->d_safe) crash = 1;
    }
  E->collision = (uint8_t)crash;
  if (crash) {
    E->reward = -1.0;
  } else if (c->reward_mode == UT_REWARD_TRACKING) {
    double sum = 0.0;
    for (int t = 0; t < T; ++t) sum += tracking_reward_single(E->err[t], c);
    E->reward = sum / (double)T;
  } else {
    double sum = 0.0;
    for (int t = 0; t < T; ++t) sum += (E->dist[t] <= c->d_min) ? 1.0 : 0.0;
    E->reward = sum / (double)T;
  }
  E->step += 1;
  E->done = (uint8_t)(E->step >= c->horizon);
}

/* Environment::step phases (env.cpp:250-279) after validation, then the
 * VecEnv bookkeeping (vecenv.cpp:95-115) */
static int env_step(uto_vecenv* v, int64_t e, const int32_t* actions) {
  uto_env* E = &v->envs[e];
  move_targets(v, E);
  move_agents(v, E, actions);
  measure_ranges(v, E);
  filter_step(v, e);
  exchange_comms(v, e);
  gather(v, e); /* build_global_state + build_observation */
  compute_reward_and_info(v, E);

  v->rewards[e] = E->reward;
  v->dones[e] = E->done;
  double err_mean = 0.0;
  for (int t = 0; t < v->T; ++t) err_mean += E->err[t];
  v->stats[UT_STAT_ENV_STEPS] += 1.0;
  v->stats[UT_STAT_REWARD_SUM] += E->reward;
  v->stats[UT_STAT_TRACK_ERR_SUM] += err_mean / (double)v->T;
  v->stats[UT_STAT_COLLISION_STEPS] += E->collision;
  for (int t = 0; t < v->T; ++t) v->stats[UT_STAT_LOST_TARGET_STEPS] += E->lost[t];
  E->episode_return += E->reward;
  /* curriculum::evaluate's per-episode accumulation (curriculum.cpp:307-325) */
  {
    int lost_any = 0;
    for (int t = 0; t < v->T; ++t) {
      E->ev_err += E->err[t];
      lost_any |= E->lost[t];
    }
    for (int a = 0; a < v->A; ++a)
      for (int t = 0; t < v->T; ++t)
        E->ev_dist += hypot(E->agents[a].x - E->targets[t].x, E->agents[a].y - E->targets[t].y);
    E->ev_flags |= (E->collision ? 1 : 0) | (lost_any ? 2 : 0);
  }
  if (E->done) {
    v->stats[UT_STAT_EPISODES_DONE] += 1.0;
    v->stats[UT_STAT_EPISODE_RETURN_SUM] += E->episode_return;
    {
      const double md = E->ev_dist / ((double)v->cfg.horizon * v->A * v->T);
      const double me = E->ev_err / ((double)v->cfg.horizon * v->T);
      v->stats[UT_STAT_EVAL_DIST_SUM] += md;
      v->stats[UT_STAT_EVAL_DIST_SQ] += md * md;
      v->stats[UT_STAT_EVAL_ERR_SUM] += me;
      v->stats[UT_STAT_EVAL_ERR_SQ] += me * me;
      v->stats[UT_STAT_EVAL_COLLIDED_EPISODES] += (E->ev_flags & 1) ? 1.0 : 0.0;
      v->stats[UT_STAT_EVAL_LOST_EPISODES] += (E->ev_flags & 2) ? 1.0 : 0.0;
      E->ev_dist = E->ev_err = 0.0;
      E->ev_flags = 0;
    }
    for (int a = 0; a < v->A; ++a) build_observation(v, e, a, v->final_obs);
    const double rew = E->reward;
    const uint8_t col = E->collision;
    const int rc = spawn(v, e);
    if (rc) return rc;
    /* spawn() resets out_.reward/done/collision (env.cpp:222-224) but the batch
     * info keeps this step's values (vecenv.cpp:96-104) */
    E->reward = rew;
    E->collision = col;
    E->done = 1;
    gather(v, e);
  }
  gather_masks(v, e);
  return UT_OK;
}

/* ---------------------------------------------------------------- API --- */
static void free_env(uto_env* E) {
  free(E->agents);
  free(E->targets);
  free(E->countdown);
  free(E->cmd_heading);
  free(E->miss_streak);
  free(E->info);
  free(E->sets);
  free(E->present);
  free(E->fresh);
  free(E->meas);
  free(E->err);
  free(E->dist);
  free(E->lost);
}

void uto_destroy(uto_vecenv* v) {
  if (!v) return;
  if (v->envs)
    for (int64_t e = 0; e < v->n; ++e) free_env(&v->envs[e]);
  free(v->envs);
  free(v->px), free(v->py), free(v->vx), free(v->vy), free(v->w);
  free(v->noise), free(v->loglik), free(v->sx), free(v->sy), free(v->svx), free(v->svy);
  free(v->obs), free(v->final_obs), free(v->global), free(v->rewards), free(v->dones), free(v->masks);
  free(v);
}

#define UTO_ALLOC(ptr, count) ((ptr) = calloc((size_t)(count), sizeof(*(ptr))))

/* VecEnv ctor (vecenv.cpp:7-45) over Environment ctors (env.cpp:110-151) */
int uto_create(const ut_env_config* cfg, int64_t n_envs, uint64_t seed, int64_t offset, uto_vecenv** out) {
  if (n_envs < 1) return set_err(UT_ERR_CONFIG, "vecenv: n_envs must be >= 1");
  ut_env_config c = *cfg;
  int rc = uto_config_finalize(&c);
  if (rc) return rc;
  uto_vecenv* v = calloc(1, sizeof *v);
  v->cfg = c;
  v->n = n_envs;
  v->A = c.n_agents;
  v->T = c.n_targets;
  v->R = c.n_agents + c.n_targets;
  v->P = c.pf.n_particles;
  const int64_t sets = n_envs * v->A * v->T, P = v->P;
  UTO_ALLOC(v->envs, n_envs);
  UTO_ALLOC(v->px, sets * P);
  UTO_ALLOC(v->py, sets * P);
  UTO_ALLOC(v->vx, sets * P);
  UTO_ALLOC(v->vy, sets * P);
  UTO_ALLOC(v->w, sets * P);
  UTO_ALLOC(v->noise, 4 * P);
  UTO_ALLOC(v->loglik, P);
  UTO_ALLOC(v->sx, P);
  UTO_ALLOC(v->sy, P);
  UTO_ALLOC(v->svx, P);
  UTO_ALLOC(v->svy, P);
  UTO_ALLOC(v->obs, n_envs * v->A * v->R * UT_FEATURE_DIM);
  UTO_ALLOC(v->final_obs, n_envs * v->A * v->R * UT_FEATURE_DIM);
  UTO_ALLOC(v->global, n_envs * v->R * UT_FEATURE_DIM);
  UTO_ALLOC(v->rewards, n_envs);
  UTO_ALLOC(v->dones, n_envs);
  UTO_ALLOC(v->masks, n_envs * v->A * UT_NUM_ACTIONS);
  if (!v->px || !v->w || !v->obs) {
    uto_destroy(v);
    return set_err(UT_ERR_RUNTIME, "oracle: out of memory");
  }
  const int A = v->A, T = v->T;
  for (int64_t e = 0; e < n_envs; ++e) {
    uto_env* E = &v->envs[e];
    const uint64_t gi = (uint64_t)(offset + e);
    E->index = (int64_t)gi;
    rng_init(&E->rng, uto_derive_key(seed, 0x656e76u, gi, 0), gi);
    rng_init(&E->bench, uto_derive_key(seed, 0x62656e63u, gi, 0), gi); /* vecenv.cpp:18-21 */
    UTO_ALLOC(E->agents, A);
    UTO_ALLOC(E->targets, T);
    UTO_ALLOC(E->countdown, T);
    UTO_ALLOC(E->cmd_heading, T);
    UTO_ALLOC(E->miss_streak, T);
    UTO_ALLOC(E->info, A * A);
    UTO_ALLOC(E->sets, A * T);
    UTO_ALLOC(E->present, A * T);
    UTO_ALLOC(E->fresh, A * T);
    UTO_ALLOC(E->meas, A * T);
    UTO_ALLOC(E->err, T);
    UTO_ALLOC(E->dist, T);
    UTO_ALLOC(E->lost, T);
    for (int a = 0; a < A; ++a) E->agents[a].rudder = 2;
    for (int t = 0; t < T; ++t) E->targets[t].rudder = 2;
    for (int a = 0; a < A; ++a)
      for (int t = 0; t < T; ++t) {
        const uint64_t pair = (uint64_t)(a * T + t);
        pfview p = pf_view(v, e, a, t);
        rng_init(&p.s->rng, uto_derive_key(seed, 0x7066u, gi, pair), pair);
        pf_reinit(&p, 0.0, 0.0, c.pf.init_radius, 1.0); /* pf::init (tracking.cpp:43-67) */
      }
    rc = spawn(v, e);
    if (rc) {
      uto_destroy(v);
      return rc;
    }
    gather(v, e);
    gather_masks(v, e);
  }
  *out = v;
  return UT_OK;
}

int uto_reset_all(uto_vecenv* v) { /* vecenv.cpp:69-77 */
  for (int64_t e = 0; e < v->n; ++e) {
    const int rc = spawn(v, e);
    if (rc) return rc;
    gather(v, e);
    gather_masks(v, e);
    v->rewards[e] = 0.0;
    v->dones[e] = 0;
  }
  return UT_OK;
}

/* VecEnv::step (vecenv.cpp:79-116); all actions validated first (see ut_env.h) */
int uto_step(uto_vecenv* v, const int32_t* actions) {
  for (int64_t e = 0; e < v->n; ++e)
    for (int a = 0; a < v->A; ++a) {
      const int act = actions[e * v->A + a];
      const int rud = v->envs[e].agents[a].rudder;
      if (!valid_action(rud, act))
        return set_err(UT_ERR_CONTRACT, "env %lld: step: invalid action %d for agent %d at rudder index %d",
                       (long long)e, act, a, rud);
    }
  for (int64_t e = 0; e < v->n; ++e) {
    const int rc = env_step(v, e, actions + e * v->A);
    if (rc) return rc;
  }
  return UT_OK;
}

/* VecEnv::step_policy (vecenv.cpp:118-143), random policy only */
int uto_step_policy(uto_vecenv* v, int policy, int n_steps) {
  if (policy != UT_POLICY_RANDOM) return set_err(UT_ERR_CONTRACT, "oracle: only the random policy is restated");
  int32_t acts[256];
  for (int k = 0; k < n_steps; ++k)
    for (int64_t e = 0; e < v->n; ++e) {
      uto_env* E = &v->envs[e];
      for (int a = 0; a < v->A; ++a) {
        int legal[UT_NUM_ACTIONS], nl = 0;
        for (int q = 0; q < UT_NUM_ACTIONS; ++q)
          if (valid_action(E->agents[a].rudder, q)) legal[nl++] = q;
        acts[a] = legal[uniform_int(&E->bench, (uint32_t)nl)];
      }
      const int rc = env_step(v, e, acts);
      if (rc) return rc;
    }
  return UT_OK;
}

int uto_refresh_outputs(uto_vecenv* v) {
  for (int64_t e = 0; e < v->n; ++e) {
    gather(v, e);
    gather_masks(v, e);
  }
  return UT_OK;
}

int uto_copy_outputs(uto_vecenv* v, const ut_host_outputs* d) {
  const int64_t n = v->n;
  const int A = v->A, T = v->T, R = v->R;
  (void)T;
  if (d->obs) memcpy(d->obs, v->obs, sizeof(double) * (size_t)(n * A * R * UT_FEATURE_DIM));
  if (d->final_obs) memcpy(d->final_obs, v->final_obs, sizeof(double) * (size_t)(n * A * R * UT_FEATURE_DIM));
  if (d->global_state) memcpy(d->global_state, v->global, sizeof(double) * (size_t)(n * R * UT_FEATURE_DIM));
  if (d->rewards) memcpy(d->rewards, v->rewards, sizeof(double) * (size_t)n);
  if (d->dones) memcpy(d->dones, v->dones, (size_t)n);
  if (d->masks) memcpy(d->masks, v->masks, (size_t)(n * A * UT_NUM_ACTIONS));
  for (int64_t e = 0; e < n; ++e) {
    const uto_env* E = &v->envs[e];
    for (int t = 0; t < T; ++t) {
      if (d->tracking_error) d->tracking_error[e * T + t] = E->err[t];
      if (d->min_agent_dist) d->min_agent_dist[e * T + t] = E->dist[t];
      if (d->target_lost) d->target_lost[e * T + t] = E->lost[t];
    }
    if (d->collision) d->collision[e] = E->collision;
    if (d->step) d->step[e] = E->step;
  }
  return UT_OK;
}

int uto_eval_acc(uto_vecenv* v, int64_t e, double out[3]) {
  if (e < 0 || e >= v->n) return set_err(UT_ERR_CONTRACT, "eval_acc: env out of range");
  out[0] = v->envs[e].ev_dist;
  out[1] = v->envs[e].ev_err;
  out[2] = (double)v->envs[e].ev_flags;
  return UT_OK;
}

int uto_stats(uto_vecenv* v, double out[UT_N_STATS]) {
  memcpy(out, v->stats, sizeof v->stats);
  return UT_OK;
}

/* env.cpp:550-593 */
int uto_serialize(uto_vecenv* v, int64_t e, double* b, size_t cap, size_t* len) {
  const int A = v->A, T = v->T, P = v->P;
  const size_t need = (size_t)(5 + 6 * A + 9 * T + A * (6 * A + T * (9 + 5 * P)));
  *len = need;
  if (!b) return UT_OK;
  if (cap < need) return set_err(UT_ERR_DATA, "serialize: buffer too small");
  const uto_env* E = &v->envs[e];
  size_t i = 0;
  b[i++] = (double)E->step;
  b[i++] = E->episode_target_speed;
  b[i++] = (double)E->rng.pos;
  b[i++] = E->rng.have_spare ? 1.0 : 0.0;
  b[i++] = E->rng.spare;
  for (int a = 0; a < A; ++a) {
    const uto_vehicle* x = &E->agents[a];
    b[i++] = x->x, b[i++] = x->y, b[i++] = x->z, b[i++] = x->heading, b[i++] = x->speed;
    b[i++] = (double)x->rudder;
  }
  for (int t = 0; t < T; ++t) {
    const uto_vehicle* x = &E->targets[t];
    b[i++] = x->x, b[i++] = x->y, b[i++] = x->z, b[i++] = x->heading, b[i++] = x->speed;
    b[i++] = (double)x->rudder;
    b[i++] = (double)E->countdown[t];
    b[i++] = E->cmd_heading[t];
  }
  for (int t = 0; t < T; ++t) b[i++] = (double)E->miss_streak[t];
  for (int a = 0; a < A; ++a) {
    for (int j = 0; j < A; ++j) {
      const uto_info* in = &E->info[a * A + j];
      b[i++] = in->x, b[i++] = in->y, b[i++] = in->z, b[i++] = in->heading;
      b[i++] = (double)in->age;
      b[i++] = in->valid ? 1.0 : 0.0;
    }
    for (int t = 0; t < T; ++t) {
      const uto_set* s = &E->sets[a * T + t];
      b[i++] = s->est_x, b[i++] = s->est_y, b[i++] = s->spread;
      b[i++] = (double)s->age;
      b[i++] = s->ever ? 1.0 : 0.0;
      b[i++] = (double)s->rng.pos;
      b[i++] = s->rng.have_spare ? 1.0 : 0.0;
      b[i++] = s->rng.spare;
      b[i++] = s->max_speed;
      const int64_t si = set_index(v, e, a, t) * P;
      const double* fields[5] = {v->px + si, v->py + si, v->vx + si, v->vy + si, v->w + si};
      for (int f = 0; f < 5; ++f)
        for (int k = 0; k < P; ++k) b[i++] = fields[f][k];
    }
  }
  return UT_OK;
}

/* env.cpp:595-659 */
int uto_deserialize(uto_vecenv* v, int64_t e, const double* b, size_t len) {
  const int A = v->A, T = v->T, P = v->P;
  const size_t need = (size_t)(5 + 6 * A + 9 * T + A * (6 * A + T * (9 + 5 * P)));
  if (len < need) return set_err(UT_ERR_DATA, "environment state blob truncated");
  if (len > need) return set_err(UT_ERR_DATA, "environment state blob has trailing data");
  uto_env* E = &v->envs[e];
  size_t i = 0;
  E->step = (int32_t)b[i++];
  E->episode_target_speed = b[i++];
  {
    const uint64_t pos = (uint64_t)b[i++];
    const int hs = b[i++] != 0.0;
    const double sp = b[i++];
    rng_restore(&E->rng, pos, hs, sp);
  }
  for (int a = 0; a < A; ++a) {
    uto_vehicle* x = &E->agents[a];
    x->x = b[i++], x->y = b[i++], x->z = b[i++], x->heading = b[i++], x->speed = b[i++];
    x->rudder = (int32_t)b[i++];
  }
  for (int t = 0; t < T; ++t) {
    uto_vehicle* x = &E->targets[t];
    x->x = b[i++], x->y = b[i++], x->z = b[i++], x->heading = b[i++], x->speed = b[i++];
    x->rudder = (int32_t)b[i++];
    E->countdown[t] = (int32_t)b[i++];
    E->cmd_heading[t] = b[i++];
  }
  for (int t = 0; t < T; ++t) E->miss_streak[t] = (int32_t)b[i++];
  for (int a = 0; a < A; ++a) {
    for (int j = 0; j < A; ++j) {
      uto_info* in = &E->info[a * A + j];
      in->x = b[i++], in->y = b[i++], in->z = b[i++], in->heading = b[i++];
      in->age = (int32_t)b[i++];
      in->valid = b[i++] != 0.0;
    }
    for (int t = 0; t < T; ++t) {
      uto_set* s = &E->sets[a * T + t];
      s->est_x = b[i++], s->est_y = b[i++], s->spread = b[i++];
      s->age = (int32_t)b[i++];
      s->ever = b[i++] != 0.0;
      const uint64_t pos = (uint64_t)b[i++];
      const int hs = b[i++] != 0.0;
      const double sp = b[i++];
      rng_restore(&s->rng, pos, hs, sp);
      s->max_speed = b[i++];
      const int64_t si = set_index(v, e, a, t) * P;
      double* fields[5] = {v->px + si, v->py + si, v->vx + si, v->vy + si, v->w + si};
      for (int f = 0; f < 5; ++f)
        for (int k = 0; k < P; ++k) fields[f][k] = b[i++];
    }
  }
  gather(v, e);
  return UT_OK;
}
