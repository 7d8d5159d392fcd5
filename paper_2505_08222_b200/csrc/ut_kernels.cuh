// ut_kernels.cuh -- the fused environment-step kernel and its helpers.
//
// One CTA steps one environment end to end (north_star "one fused kernel per
// step"): the env record is staged in shared memory, one thread runs the serial
// env-stream prologue (Appendix A order: targets, agents, pings, comm drops),
// then the whole CTA runs every particle set of the env with the set held in
// registers -- PPT consecutive particles per thread (128-bit coalesced loads and
// stores, each set read once and written once per step) -- then the epilogue
// (reward, done, tokens, masks) and, for finished envs, the auto-reset (spawn +
// particle re-init) before the record is written back.
//
// Per set the work is: predict (Philox words generated one set ahead into a
// double-buffered smem area, correctly rounded fp32 Box-Muller), ONE merged pass
// for all of this step's range updates (per-stage maxima kept so the reference's
// sequential semantics hold; the exact sequential path runs whenever an
// intermediate underflow could matter), ESS from the same reduction, systematic
// resample (scan + search), estimate in one shifted reduction.
#pragma once
#include "ut_device.cuh"

namespace ut {

enum StepMode : int { MODE_EXTERNAL = -1, MODE_RANDOM = 0, MODE_SCRIPTED = 1 };
enum DevStatus : int { ST_OK = 0, ST_SPAWN_INFEASIBLE = 2 };
constexpr int kMaxMerged = 8;   // merged update handles up to 8 measurements per set
constexpr int kMeasStride = 8;  // ox, oy, r2, sigma, 1/sigma (+pad)
constexpr double kMergeFloor = 0x1p-860;  // see the merged-update argument in step_set

// ------------------------------------------------------------ smem carve ---
struct Smem {
  double2* tab_log;    // [128]
  double2* tab_sc;     // [64]
  double* rec;
  double* meas;        // [A*T][kMeasStride]
  double* red;         // kRedDoubles: BlockReducer buffers + scan warp sums
  double* bc;          // 16 broadcast slots
  double* qxy;         // [2 * R] spawn scratch
  int* act;            // [A]
  uint8_t* present;    // [A*T]
  uint8_t* link;       // [A*A]
  uint8_t* mcount;     // [A*T] measurements applied to each set this step
  uint8_t* mlist;      // [A*T][A] their meas indices in application order
  uint32_t* words[2];  // Philox words, double buffered: 4P + 2 (+ 8 slack)
  double* cum;         // [P] resample scan
  double* st;          // [4P] resample staging
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline size_t words_bytes(int P) {
  // predict uses 4P words + 2 for the resample u0; one extra block covers a
  // misaligned start. (Re-init's 8P words use the resample area instead.)
  return align16((size_t)4 * (4 * (size_t)P + 2 + 8));
}
__host__ __device__ inline size_t resample_bytes(int P) {
  const size_t a = sizeof(double) * 5 * (size_t)P;  // cum + 4 staged fields
  const size_t b = (size_t)4 * (8 * (size_t)P + 8);  // re-init words
  return align16(a > b ? a : b);
}

__host__ __device__ inline size_t smem_bytes(int rec_words, int A, int T, int P) {
  const int R = A + T;
  size_t s = 0;
  s += sizeof(double2) * (128 + 64);
  s += align16(sizeof(double) * rec_words);
  s += align16(sizeof(double) * kMeasStride * A * T);
  s += align16(sizeof(double) * kRedDoubles);
  s += align16(sizeof(double) * 16);
  s += align16(sizeof(double) * 2 * R);
  s += align16(sizeof(int) * A);
  s += align16(A * T) + align16(A * A) + align16(A * T) + align16(A * T * A);
  s += 2 * words_bytes(P);
  s += resample_bytes(P);
  return s;
}

__device__ inline Smem carve(unsigned char* base, int rec_words, int A, int T, int P) {
  Smem S;
  const int R = A + T;
  size_t o = 0;
  S.tab_log = (double2*)(base + o);
  o += sizeof(double2) * 128;
  S.tab_sc = (double2*)(base + o);
  o += sizeof(double2) * 64;
  S.rec = (double*)(base + o);
  o += align16(sizeof(double) * rec_words);
  S.meas = (double*)(base + o);
  o += align16(sizeof(double) * kMeasStride * A * T);
  S.red = (double*)(base + o);
  o += align16(sizeof(double) * kRedDoubles);
  S.bc = (double*)(base + o);
  o += align16(sizeof(double) * 16);
  S.qxy = (double*)(base + o);
  o += align16(sizeof(double) * 2 * R);
  S.act = (int*)(base + o);
  o += align16(sizeof(int) * A);
  S.present = base + o;
  o += align16(A * T);
  S.link = base + o;
  o += align16(A * A);
  S.mcount = base + o;
  o += align16(A * T);
  S.mlist = base + o;
  o += align16(A * T * A);
  S.words[0] = (uint32_t*)(base + o);
  o += words_bytes(P);
  S.words[1] = (uint32_t*)(base + o);
  o += words_bytes(P);
  S.cum = (double*)(base + o);
  S.st = S.cum + P;
  return S;
}

__device__ __forceinline__ const DevConfig& cfg_of(const DevBatch& B, int64_t e) {
  return B.cfgs[B.cfg_of_env ? B.cfg_of_env[e] : 0];
}
__device__ __forceinline__ int64_t rec_off(const DevBatch& B, int64_t e) {
  return B.rec_offset ? B.rec_offset[e] : e * (int64_t)B.cfgs[0].rec_words;
}
__device__ __forceinline__ int64_t set_off(const DevBatch& B, int64_t e) {
  return B.set_offset ? B.set_offset[e] : e * (int64_t)(B.cfgs[0].A * B.cfgs[0].T);
}

__device__ __forceinline__ void load_tables(const Smem& S) {
  for (int i = threadIdx.x; i < 128; i += blockDim.x) S.tab_log[i] = make_double2(kLogTab[2 * i], kLogTab[2 * i + 1]);
  for (int i = threadIdx.x; i < 64; i += blockDim.x) S.tab_sc[i] = make_double2(kSinCosTab[2 * i], kSinCosTab[2 * i + 1]);
}

// --------------------------------------------------- serial env prologue ---
// Environment::scripted_action (env.cpp:511-543) for every agent, on the
// pre-step state (VecEnv::step_policy computes all actions first, vecenv.cpp:123-124).
__device__ __noinline__ void scripted_actions(const DevConfig& c, const double* rec, int* act) {
  const int A = c.A, T = c.T, AT = A * T;
  const double* ag = rec + c.o_agent;
  const double* trk = rec + c.o_track;
  for (int a = 0; a < A; ++a) {
    const double sx = ag[V_X * A + a], sy = ag[V_Y * A + a], sh = ag[V_HEAD * A + a];
    const int rud = (int)ag[V_RUDDER * A + a];
    double gx = sx, gy = sy, best = CUDART_INF;
    for (int t = 0; t < T; ++t) {
      const int si = a * T + t;
      const double ex = trk[K_EX * AT + si], ey = trk[K_EY * AT + si];
      const double d = norm2(ex - sx, ey - sy);
      const double penalty = trk[K_EVER * AT + si] != 0.0 ? 0.0 : 1e6;
      if (d + penalty < best) {
        best = d + penalty;
        gx = ex;
        gy = ey;
      }
    }
    const double desired = atan2(gy - sy, gx - sx);
    int best_act = rud;
    double best_mis = CUDART_INF;
    for (int i = 0; i < 5; ++i) {
      if (abs(i - rud) > 1) continue;
      const double dpsi = c.head_a * (-0.24 + 0.12 * i) + c.head_b;
      const double mis = fabs(wrap_angle(sh + dpsi - desired));
      if (mis < best_mis) {
        best_mis = mis;
        best_act = i;
      }
    }
    act[a] = best_act;
  }
}

// Actions + move_targets + move_agents + measure_ranges + comm decisions, in
// the reference's env-stream draw order, then the per-set
// measurement schedule. Thread 0 only.
__device__ __noinline__ void env_prologue(const DevConfig& c, const DevBatch& B, const Smem& S, int64_t e, int64_t gi,
                             int mode) {
  const int A = c.A, T = c.T;
  double* rec = S.rec;
  double* ag = rec + c.o_agent;
  double* tg = rec + c.o_target;
  double* miss = rec + c.o_miss;
  double* info = rec + c.o_info;
  const int AA = A * A;
  SerialRng rng;
  rng.init(derive_key(B.seed, kTagEnv, (uint64_t)gi, 0), (uint64_t)gi, (uint64_t)rec[R_ENV_POS],
           rec[R_ENV_HAVE_SPARE] != 0.0, rec[R_ENV_SPARE]);

  // actions: VecEnv::step_policy (vecenv.cpp:118-135) or the caller's
  if (mode == MODE_RANDOM) {
    SerialRng b;
    b.init(derive_key(B.seed, kTagBench, (uint64_t)gi, 0), (uint64_t)gi, (uint64_t)rec[R_BENCH_POS], false, 0.0);
    for (int a = 0; a < A; ++a) {
      const int rud = (int)ag[V_RUDDER * A + a];
      int legal[5], nl = 0;
      for (int q = 0; q < 5; ++q)
        if (abs(q - rud) <= 1) legal[nl++] = q;
      S.act[a] = legal[b.uniform_int((uint32_t)nl)];
    }
    rec[R_BENCH_POS] = (double)b.pos;
  } else if (mode == MODE_SCRIPTED) {
    scripted_actions(c, rec, S.act);
  } else {
    for (int a = 0; a < A; ++a) S.act[a] = B.actions[e * B.A_max + a];
  }

  // move_targets (env.cpp:289-304)
  for (int t = 0; t < T; ++t) {
    if (tg[V_COUNTDOWN * T + t] <= 0.0) {
      tg[V_CMD * T + t] = wrap_angle(kTwoPi * rng.uniform());
      tg[V_COUNTDOWN * T + t] = (double)rng.geometric_i32(c.turn_interval);
    }
    const double want = wrap_angle(tg[V_CMD * T + t] - tg[V_HEAD * T + t]);
    const double mt = c.max_turn;
    const double dpsi = want < -mt ? -mt : (mt < want ? mt : want);
    const double noise = c.head_noise > 0.0 ? c.head_noise * rng.normal() : 0.0;
    // advance_vehicle (kinematics.cpp:42-49)
    const double h = wrap_angle(tg[V_HEAD * T + t] + dpsi + noise);
    tg[V_HEAD * T + t] = h;
    tg[V_X * T + t] += tg[V_SPEED * T + t] * c.dt * cos(h);
    tg[V_Y * T + t] += tg[V_SPEED * T + t] * c.dt * sin(h);
    tg[V_COUNTDOWN * T + t] -= 1.0;
  }
  // move_agents (env.cpp:306-316) + step_vehicle (kinematics.cpp:51-56)
  for (int a = 0; a < A; ++a) {
    const int rud = S.act[a];
    ag[V_RUDDER * A + a] = (double)rud;
    const double gamma = -0.24 + 0.12 * rud;
    double noise = c.head_noise > 0.0 ? c.head_noise * rng.normal() : 0.0;
    if (c.pert_std > 0.0) noise += c.pert_std * rng.normal();
    const double dpsi = c.head_a * gamma + c.head_b;
    const double h = wrap_angle(ag[V_HEAD * A + a] + dpsi + noise);
    ag[V_HEAD * A + a] = h;
    ag[V_X * A + a] += ag[V_SPEED * A + a] * c.dt * cos(h);
    ag[V_Y * A + a] += ag[V_SPEED * A + a] * c.dt * sin(h);
  }
  // measure_ranges (env.cpp:318-347): targets outer, agents inner
  for (int t = 0; t < T; ++t) {
    bool detected = false;
    for (int a = 0; a < A; ++a) {
      const int idx = a * T + t;
      S.present[idx] = 0;
      const double ax = ag[V_X * A + a], ay = ag[V_Y * A + a], az = ag[V_Z * A + a];
      const double tz = tg[V_Z * T + t];
      const double dist3 = norm3(ax - tg[V_X * T + t], ay - tg[V_Y * T + t], az - tz);
      if (dist3 > c.det_range) continue;
      if (c.drop > 0.0 && rng.uniform() < c.drop) continue;
      double r3 = dist3;
      if (c.range_noise > 0.0) r3 += c.range_noise * rng.normal();
      r3 = r3 < 0.0 ? 0.0 : r3;
      const double dd = tz - az;
      const double sq = r3 * r3 - dd * dd;  // slant_to_horizontal (tracking.cpp:9-14)
      double* m = S.meas + kMeasStride * idx;
      m[0] = ax;
      m[1] = ay;
      m[2] = sq <= 0.0 ? 0.0 : sqrt(sq);
      m[3] = c.sigma_meas;
      m[4] = 1.0 / c.sigma_meas;
      S.present[idx] = 1;
      detected = true;
    }
    miss[t] = detected ? 0.0 : miss[t] + 1.0;
  }
  // exchange_comms decisions (env.cpp:365-383)
  for (int i = 0; i < AA; ++i) info[I_AGE * AA + i] += 1.0;
  for (int r = 0; r < A; ++r)
    for (int s = 0; s < A; ++s) {
      S.link[r * A + s] = 0;
      if (s == r) continue;
      const double sx = ag[V_X * A + s], sy = ag[V_Y * A + s], sz = ag[V_Z * A + s];
      if (norm3(ag[V_X * A + r] - sx, ag[V_Y * A + r] - sy, ag[V_Z * A + r] - sz) > c.comm_range) continue;
      if (c.drop > 0.0 && rng.uniform() < c.drop) continue;
      const int k = r * A + s;
      info[I_X * AA + k] = sx;
      info[I_Y * AA + k] = sy;
      info[I_Z * AA + k] = sz;
      info[I_HEAD * AA + k] = ag[V_HEAD * A + s];
      info[I_AGE * AA + k] = 0.0;
      info[I_VALID * AA + k] = 1.0;
      S.link[k] = 1;
    }
  // per-set update schedule: own ping first (env.cpp:356-360), then the fused
  // senders in ascending order (env.cpp:370-392)
  for (int a = 0; a < A; ++a)
    for (int t = 0; t < T; ++t) {
      const int si = a * T + t;
      int n = 0;
      if (S.present[si]) S.mlist[si * A + n++] = (uint8_t)si;
      for (int s = 0; s < A; ++s)
        if (s != a && S.link[a * A + s] && S.present[s * T + t]) S.mlist[si * A + n++] = (uint8_t)(s * T + t);
      S.mcount[si] = (uint8_t)n;
    }
  rec[R_ENV_POS] = (double)rng.pos;
  rec[R_ENV_HAVE_SPARE] = rng.have_spare ? 1.0 : 0.0;
  rec[R_ENV_SPARE] = rng.spare;
}

// -------------------------------------------------- particle-set phases ---
template <int PPT>
struct SetRegs {
  double px[PPT], py[PPT], vx[PPT], vy[PPT], w[PPT];
};

// Words [pos, pos + n_words) of one stream into smem (no barrier):
// word(pos + m) == words[(pos & 3) + m].
__device__ __forceinline__ void gen_words(uint32_t* words, uint64_t key, uint64_t stream, uint64_t pos,
                                          uint64_t n_words) {
  const uint64_t b0 = pos >> 2;
  const int nb = (int)(((pos + n_words - 1) >> 2) - b0 + 1);
  uint4* w4 = reinterpret_cast<uint4*>(words);
  for (int i = threadIdx.x; i < nb; i += blockDim.x) w4[i] = philox(key, stream, b0 + (uint64_t)i);
}

// 4 consecutive words starting at idx (idx % 4 uniform across the warp).
__device__ __forceinline__ uint4 lds_words4(const uint32_t* w, int idx) {
  if ((idx & 3) == 0) return *reinterpret_cast<const uint4*>(w + idx);
  if ((idx & 1) == 0) {
    const uint2 a = *reinterpret_cast<const uint2*>(w + idx);
    const uint2 b = *reinterpret_cast<const uint2*>(w + idx + 2);
    return make_uint4(a.x, a.y, b.x, b.y);
  }
  return make_uint4(w[idx], w[idx + 1], w[idx + 2], w[idx + 3]);
}

template <int PPT>
__device__ __forceinline__ void load_set(SetRegs<PPT>& s, const DevBatch& B, size_t base, int k0, int P) {
  if (PPT == 4 && k0 + 4 <= P && (P & 3) == 0) {
    const double2* px = reinterpret_cast<const double2*>(B.px + base + k0);
    const double2* py = reinterpret_cast<const double2*>(B.py + base + k0);
    const double2* vx = reinterpret_cast<const double2*>(B.vx + base + k0);
    const double2* vy = reinterpret_cast<const double2*>(B.vy + base + k0);
    const double2* w = reinterpret_cast<const double2*>(B.w + base + k0);
    double2 t[10] = {px[0], px[1], py[0], py[1], vx[0], vx[1], vy[0], vy[1], w[0], w[1]};
    s.px[0] = t[0].x, s.px[1] = t[0].y, s.px[2] = t[1].x, s.px[3] = t[1].y;
    s.py[0] = t[2].x, s.py[1] = t[2].y, s.py[2] = t[3].x, s.py[3] = t[3].y;
    s.vx[0] = t[4].x, s.vx[1] = t[4].y, s.vx[2] = t[5].x, s.vx[3] = t[5].y;
    s.vy[0] = t[6].x, s.vy[1] = t[6].y, s.vy[2] = t[7].x, s.vy[3] = t[7].y;
    s.w[0] = t[8].x, s.w[1] = t[8].y, s.w[2] = t[9].x, s.w[3] = t[9].y;
    return;
  }
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const int k = k0 + j;
    if (k < P) {
      s.px[j] = B.px[base + k];
      s.py[j] = B.py[base + k];
      s.vx[j] = B.vx[base + k];
      s.vy[j] = B.vy[base + k];
      s.w[j] = B.w[base + k];
    } else {
      s.px[j] = s.py[j] = s.vx[j] = s.vy[j] = s.w[j] = 0.0;
    }
  }
}

template <int PPT>
__device__ __forceinline__ void store_set(const SetRegs<PPT>& s, const DevBatch& B, size_t base, int k0, int P) {
  if (PPT == 4 && k0 + 4 <= P && (P & 3) == 0) {
    double2* px = reinterpret_cast<double2*>(B.px + base + k0);
    double2* py = reinterpret_cast<double2*>(B.py + base + k0);
    double2* vx = reinterpret_cast<double2*>(B.vx + base + k0);
    double2* vy = reinterpret_cast<double2*>(B.vy + base + k0);
    double2* w = reinterpret_cast<double2*>(B.w + base + k0);
    px[0] = make_double2(s.px[0], s.px[1]);
    px[1] = make_double2(s.px[2], s.px[3]);
    py[0] = make_double2(s.py[0], s.py[1]);
    py[1] = make_double2(s.py[2], s.py[3]);
    vx[0] = make_double2(s.vx[0], s.vx[1]);
    vx[1] = make_double2(s.vx[2], s.vx[3]);
    vy[0] = make_double2(s.vy[0], s.vy[1]);
    vy[1] = make_double2(s.vy[2], s.vy[3]);
    w[0] = make_double2(s.w[0], s.w[1]);
    w[1] = make_double2(s.w[2], s.w[3]);
    return;
  }
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const int k = k0 + j;
    if (k < P) {
      B.px[base + k] = s.px[j];
      B.py[base + k] = s.py[j];
      B.vx[base + k] = s.vx[j];
      B.vy[base + k] = s.vy[j];
      B.w[base + k] = s.w[j];
    }
  }
}

// pf::update with one measurement (tracking.cpp:119-143) -- the exact
// sequential path.
template <int PPT>
__device__ __noinline__ void pf_update_seq(SetRegs<PPT>& s, const double* m, int k0, int P, BlockReducer& R) {
  const double ox = m[0], oy = m[1], r2 = m[2], sig = m[3];
  double ll[PPT];
  double mx = -CUDART_INF;
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    if (k0 + j < P) {
      const double dx = s.px[j] - ox, dy = s.py[j] - oy;
      const double d = sqrt(dx * dx + dy * dy);
      const double q = (d - r2) / sig;
      ll[j] = 0.0 - 0.5 * (q * q);
      mx = ll[j] > mx ? ll[j] : mx;
    } else {
      ll[j] = -CUDART_INF;
    }
  }
  const double shift = R.max(mx);
  if (isfinite(shift)) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (k0 + j < P) {
        s.w[j] = s.w[j] * exp(ll[j] - shift);
        acc = acc + s.w[j];
      }
    }
    const double sum = R.sum(acc);
    if (isfinite(sum) && sum > 0.0) {
#pragma unroll
      for (int j = 0; j < PPT; ++j) s.w[j] = s.w[j] / sum;
      return;
    }
  }
  const double inv = 1.0 / (double)P;
#pragma unroll
  for (int j = 0; j < PPT; ++j) s.w[j] = k0 + j < P ? inv : 0.0;
}

// pf::estimate (tracking.cpp:180-188) in ONE reduction: moments about the set's
// previous estimate (cx, cy), mean = c + sum w (p - c), spread^2 = second moment
// minus the squared shift; exact second pass when that subtraction could lose
// more than ~1e-11 relative.
template <int PPT>
__device__ __forceinline__ double3 pf_estimate(const SetRegs<PPT>& s, int k0, int P, double cx, double cy,
                                               BlockReducer& R) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    if (k0 + j < P) {
      const double dx = s.px[j] - cx, dy = s.py[j] - cy;
      a0 = a0 + s.w[j] * dx;
      a1 = a1 + s.w[j] * dy;
      a2 = a2 + s.w[j] * (dx * dx + dy * dy);
    }
  }
  const double3 m = R.sum3(a0, a1, a2);
  const double mx = cx + m.x, my = cy + m.y;
  const double shift2 = m.x * m.x + m.y * m.y;
  const double var = m.z - shift2;
  if (var > 1e-5 * shift2) return make_double3(mx, my, sqrt(var));
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    if (k0 + j < P) {
      const double dx = s.px[j] - mx, dy = s.py[j] - my;
      acc = acc + s.w[j] * (dx * dx + dy * dy);
    }
  }
  return make_double3(mx, my, sqrt(R.sum(acc)));
}

// pf::resample (tracking.cpp:147-170): inclusive scan of w in index order, then
// output j takes the first particle whose cumulative weight reaches (j + u0)/n,
// clamped to n - 1 (the reference's monotone two-pointer walk): a binary search
// for the thread's first output, a forward walk for the rest.
template <int PPT>
__device__ void pf_resample(SetRegs<PPT>& s, int k0, int P, double u0, const Smem& S) {
  const int tid = threadIdx.x, NT = blockDim.x;
  double* cum = S.cum;
  double* st = S.st;
  double* wsum = S.red + 2 * kRedSlots;
  double loc[PPT];
  double run = 0.0;
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int k = k0 + q;
    if (k < P) {
      st[k] = s.px[q];
      st[P + k] = s.py[q];
      st[2 * P + k] = s.vx[q];
      st[3 * P + k] = s.vy[q];
      run = q == 0 ? s.w[q] : run + s.w[q];
    }
    loc[q] = run;
  }
  const int lane = tid & 31, warp = tid >> 5;
  double incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl = incl + y;
  }
  double excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = 0.0;
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  double woff = 0.0;
  for (int v = 0; v < warp; ++v) woff = woff + wsum[v];
  const double base = woff + excl;
#pragma unroll
  for (int q = 0; q < PPT; ++q)
    if (k0 + q < P) cum[k0 + q] = base + loc[q];
  (void)NT;
  __syncthreads();
  const double inv_n = 1.0 / (double)P;
  if (k0 < P) {
    const double u = ((double)k0 + u0) * inv_n;
    int a = 0, b = P - 1;
    while (a < b) {
      const int mid = (a + b) >> 1;
      if (cum[mid] < u)
        a = mid + 1;
      else
        b = mid;
    }
    int i = a;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int j = k0 + q;
      if (j < P) {
        const double uj = ((double)j + u0) * inv_n;
        // lower_bound over [i, P-1]: usually i or i+1; otherwise a binary search
        // (a plain forward walk diverges over runs of zero-weight particles)
        if (i < P - 1 && cum[i] < uj) {
          ++i;
          if (i < P - 1 && cum[i] < uj) {
            int lo = i + 1, hi = P - 1;
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              if (cum[mid] < uj)
                lo = mid + 1;
              else
                hi = mid;
            }
            i = lo;
          }
        }
        s.px[q] = st[i];
        s.py[q] = st[P + i];
        s.vx[q] = st[2 * P + i];
        s.vy[q] = st[3 * P + i];
        s.w[q] = inv_n;
      }
    }
  }
  __syncthreads();
}

// filter_step (env.cpp:349-363) + fused comm updates (env.cpp:385-392) +
// finalize (env.cpp:397-409) for ONE set. `wb` is this set's words buffer; the
// next set's words (if any) are generated into the other buffer on the way.
template <int PPT>
__device__ void step_set(const DevConfig& c, const DevBatch& B, const Smem& S, BlockReducer& R, int64_t gi,
                         int64_t gset, int a, int t, int wb, double* stat) {
  const int P = c.P, tid = threadIdx.x, A = c.A, T = c.T, AT = A * T;
  const int si = a * T + t;
  const int k0 = tid * PPT;
  double* trk = S.rec + c.o_track;
  uint64_t pos = (uint64_t)trk[K_POS * AT + si];
  const double ms = trk[K_MAXSPEED * AT + si];
  const uint64_t key = derive_key(B.seed, kTagPf, (uint64_t)gi, (uint64_t)si);
  const size_t base = (size_t)gset * P;
  const uint32_t* words = S.words[wb];
  const int off = (int)(pos & 3);

  SetRegs<PPT> s;
  load_set<PPT>(s, B, base, k0, P);

  // Next set's words into the other buffer (made visible by this set's barriers).
  if (si + 1 < AT) {
    const uint64_t npos = (uint64_t)trk[K_POS * AT + si + 1];
    gen_words(S.words[wb ^ 1], derive_key(B.seed, kTagPf, (uint64_t)gi, (uint64_t)(si + 1)), (uint64_t)(si + 1),
              npos, (c.noise_on ? 4ull * (uint64_t)P : 0ull) + 2ull);
  }

  // ---- pf::predict (tracking.cpp:94-117)
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    s.px[j] = s.px[j] + s.vx[j] * c.dt;
    s.py[j] = s.py[j] + s.vy[j] * c.dt;
  }
  if (c.noise_on) {
    const float two_pi_f = 2.0f * 3.14159265358979323846f;
    // fill_normals: pair i uses u1 = word(pos + i), u2 = word(pos + 2P + i);
    // particle k takes cos of pairs k and P+k, sin of pairs k and P+k.
    uint4 W[4];
    if (PPT == 4 && k0 + 4 <= P) {
#pragma unroll
      for (int q = 0; q < 4; ++q) W[q] = lds_words4(words, off + q * P + k0);
    }
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const int k = k0 + j;
      if (k < P) {
        uint32_t w1a, w1b, w2a, w2b;
        if (PPT == 4 && k0 + 4 <= P) {
          w1a = lane_of(W[0], j);
          w1b = lane_of(W[1], j);
          w2a = lane_of(W[2], j);
          w2b = lane_of(W[3], j);
        } else {
          w1a = words[off + k];
          w1b = words[off + P + k];
          w2a = words[off + 2 * P + k];
          w2b = words[off + 3 * P + k];
        }
        float zpx, zvx, zpy, zvy;  // out[k], out[2P+k] / out[P+k], out[3P+k]
        bool ok = box_muller_fast(w1a, w2a, S.tab_log, S.tab_sc, zpx, zvx);
        ok &= box_muller_fast(w1b, w2b, S.tab_log, S.tab_sc, zpy, zvy);
        if (!ok) {  // an uncertain rounding (p ~ 1e-4 per particle): exact fp64 libm path
          box_muller_slow(w1a, w2a, zpx, zvx);
          box_muller_slow(w1b, w2b, zpy, zvy);
        }
        s.px[j] = s.px[j] + c.pn * (double)zpx;
        s.py[j] = s.py[j] + c.pn * (double)zpy;
        s.vx[j] = s.vx[j] + c.vn * (double)zvx;
        s.vy[j] = s.vy[j] + c.vn * (double)zvy;
      }
    }
  }
  if (ms > 0.0) {
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const double sp = sqrt(s.vx[j] * s.vx[j] + s.vy[j] * s.vy[j]);
      const double f = sp > ms ? ms / sp : 1.0;
      s.vx[j] = s.vx[j] * f;
      s.vy[j] = s.vy[j] * f;
    }
  }
  const int u0_idx = off + (c.noise_on ? 4 * P : 0);  // resample draw follows predict's 4P
  if (c.noise_on) pos += 4ull * (uint64_t)P;

  // ---- range updates: own ping, then fused senders (env.cpp:356-360, 385-392)
  const int nm = S.mcount[si];
  const uint8_t* ml = S.mlist + si * A;
  bool have_ess = false;
  double ess = 0.0;
  bool exact = nm > kMaxMerged || B.force_exact;
  if (nm > 0 && !exact) {
    // Merged pass. With L_i = sum_j ll_ij and s_j = max_i ll_ij, the sequential
    // reference computes e_i / sum(e) with e_i = w_i exp(L_i - sum_j s_j), up to
    // rounding, unless an intermediate product underflows. Every intermediate
    // product of particle i is >= e_i (each ll - s <= 0, each stage sum <= 1).
    // Particles with e_i < 2^-60 max(e) are invisible in every fp64 sum either
    // way; all others have products >= 2^-60 max(e) >= 2^-920 (normal) when
    // max(e) >= 2^-860, and no stage can degenerate. So under that check the
    // merged result equals the sequential one to rounding; otherwise (or with a
    // non-finite shift) the exact sequential path runs.
    double L[PPT];
#pragma unroll
    for (int q = 0; q < PPT; ++q) L[q] = 0.0;
    double* mb = R.buf();  // per-stage warp maxima, [stage * 32 + warp]
    const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
#pragma unroll 1
    for (int j = 0; j < nm; ++j) {
      const double* m = S.meas + kMeasStride * ml[j];
      const double ox = m[0], oy = m[1], r2 = m[2], sig = m[3], rsig = m[4];
      double mj = -CUDART_INF;
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        if (k0 + q < P) {
          const double dx = s.px[q] - ox, dy = s.py[q] - oy;
          const double d = sqrt(dx * dx + dy * dy);
          const double qv = div_rcp(d - r2, sig, rsig);
          const double ll = 0.0 - 0.5 * (qv * qv);
          L[q] = L[q] + ll;
          mj = ll > mj ? ll : mj;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double u = __shfl_xor_sync(0xffffffffu, mj, o);
        mj = u > mj ? u : mj;
      }
      if (lane == 0) mb[j * 32 + warp] = mj;
    }
    __syncthreads();
    double shift = 0.0;  // sum_j s_j, in stage order
#pragma unroll 1
    for (int j = 0; j < nm; ++j) {
      double sj = lane < nw ? mb[j * 32 + lane] : -CUDART_INF;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double u = __shfl_xor_sync(0xffffffffu, sj, o);
        sj = u > sj ? u : sj;
      }
      shift = j == 0 ? sj : shift + sj;
    }
    if (!isfinite(shift)) {
      exact = true;
    } else {
      double e[PPT], ls = 0.0, lq = 0.0, lm = 0.0;
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        e[q] = 0.0;
        if (k0 + q < P) {
          e[q] = s.w[q] * exp(L[q] - shift);
          ls = ls + e[q];
          lq = lq + e[q] * e[q];
          lm = e[q] > lm ? e[q] : lm;
        }
      }
      const double3 r = R.sum2_max(ls, lq, lm);
      if (isfinite(r.x) && r.x > 0.0 && r.z >= kMergeFloor) {
        const double rcp = 1.0 / r.x;
#pragma unroll
        for (int q = 0; q < PPT; ++q) s.w[q] = div_rcp(e[q], r.x, rcp);
        // ESS = sum^2 / sum(e^2) unless the squares may have underflowed
        if (r.z >= 0x1p-200) {
          ess = (r.x * r.x) / r.y;
          have_ess = true;
        }
      } else {
        exact = true;
      }
    }
    if (exact && tid == 0) stat[2] += 1.0;
  }
  if (exact) {
    for (int j = 0; j < nm; ++j) pf_update_seq<PPT>(s, S.meas + kMeasStride * ml[j], k0, P, R);
  }
  const bool fresh = nm > 0;

  // ---- pf::maybe_resample (tracking.cpp:172-178)
  bool resampled = false;
  const bool ess_known_ok = nm == 0 && trk[K_ESSOK * AT + si] != 0.0;
  if (!ess_known_ok) {
    if (!have_ess) {
      double w2 = 0.0;
#pragma unroll
      for (int q = 0; q < PPT; ++q) w2 = w2 + s.w[q] * s.w[q];
      ess = 1.0 / R.sum(w2);
    }
    if (ess < (double)P / 2.0) {
      const uint64_t lo = words[u0_idx], hi = words[u0_idx + 1];
      const double u0 = (double)(((hi << 32) | lo) >> 11) * 0x1.0p-53;
      pos += 2;
      pf_resample<PPT>(s, k0, P, u0, S);
      resampled = true;
    }
  }

  if (B.trace_env == gi - B.env_index_offset && tid == 0)
    printf("[trace env %lld set %d] nm=%d exact=%d have_ess=%d ess=%.17g resampled=%d pos=%llu\n",
           (long long)(gi - B.env_index_offset), si, nm, (int)exact, (int)have_ess, ess, (int)resampled,
           (unsigned long long)pos);

  // ---- estimate (env.cpp:403-407)
  const double3 est = pf_estimate<PPT>(s, k0, P, trk[K_EX * AT + si], trk[K_EY * AT + si], R);
  store_set<PPT>(s, B, base, k0, P);
  if (tid == 0) {
    trk[K_EX * AT + si] = est.x;
    trk[K_EY * AT + si] = est.y;
    trk[K_SPREAD * AT + si] = est.z;
    trk[K_AGE * AT + si] = fresh ? 0.0 : trk[K_AGE * AT + si] + 1.0;
    trk[K_EVER * AT + si] = (trk[K_EVER * AT + si] != 0.0 || fresh) ? 1.0 : 0.0;
    trk[K_POS * AT + si] = (double)pos;
    trk[K_ESSOK * AT + si] = 1.0;  // maybe_resample ran: ESS >= P/2 or weights uniform
    stat[0] += (double)nm;
    stat[1] += resampled ? 1.0 : 0.0;
  }
}

// pf::reinit (tracking.cpp:76-92) + estimate for one set (spawn, env.cpp:214-220).
template <int PPT>
__device__ void reinit_set(const DevConfig& c, const DevBatch& B, const Smem& S, BlockReducer& R, int64_t gi,
                           int64_t gset, int si, double cx, double cy, double vmax) {
  const int P = c.P, tid = threadIdx.x, AT = c.A * c.T;
  const int k0 = tid * PPT;
  double* trk = S.rec + c.o_track;
  uint64_t pos = (uint64_t)trk[K_POS * AT + si];
  const uint64_t key = derive_key(B.seed, kTagPf, (uint64_t)gi, (uint64_t)si);
  uint32_t* words = reinterpret_cast<uint32_t*>(S.cum);  // the resample area
  __syncthreads();  // that area may still be read by the previous phase
  gen_words(words, key, (uint64_t)si, pos, 8ull * (uint64_t)P);
  __syncthreads();
  const int off = (int)(pos & 3);
  const double inv = 1.0 / (double)P;
  const double radius = c.init_radius;
  SetRegs<PPT> s;
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const int k = k0 + j;
    s.px[j] = s.py[j] = s.vx[j] = s.vy[j] = s.w[j] = 0.0;
    if (k < P) {
      const uint32_t* q = words + off + 8 * k;
      auto u = [&](int i) {
        const uint64_t lo = q[2 * i], hi = q[2 * i + 1];
        return (double)(((hi << 32) | lo) >> 11) * 0x1.0p-53;
      };
      const double r = radius * sqrt(u(0));
      const double an = kTwoPi * u(1);
      double sa, ca;
      sincos(an, &sa, &ca);
      s.px[j] = cx + r * ca;
      s.py[j] = cy + r * sa;
      const double sp = vmax * u(2);
      const double d = kTwoPi * u(3);
      double sd, cd;
      sincos(d, &sd, &cd);
      s.vx[j] = sp * cd;
      s.vy[j] = sp * sd;
      s.w[j] = inv;
    }
  }
  pos += 8ull * (uint64_t)P;
  const double3 est = pf_estimate<PPT>(s, k0, P, cx, cy, R);
  store_set<PPT>(s, B, (size_t)gset * P, k0, P);
  if (tid == 0) {
    trk[K_EX * AT + si] = est.x;
    trk[K_EY * AT + si] = est.y;
    trk[K_SPREAD * AT + si] = est.z;
    trk[K_AGE * AT + si] = 0.0;
    trk[K_EVER * AT + si] = 0.0;
    trk[K_POS * AT + si] = (double)pos;
    trk[K_MAXSPEED * AT + si] = vmax;
    trk[K_ESSOK * AT + si] = 1.0;
  }
  __syncthreads();
}

// ------------------------------------------------------------- spawn ---
// Environment::spawn, serial part (env.cpp:155-212, 221-224). Thread 0 only.
// Returns false when the rejection sampling fails (ConfigError in the reference).
__device__ __noinline__ bool spawn_serial(const DevConfig& c, const DevBatch& B, const Smem& S, int64_t gi) {
  const int A = c.A, T = c.T, R = c.R, AA = A * A;
  double* rec = S.rec;
  double* ag = rec + c.o_agent;
  double* tg = rec + c.o_target;
  SerialRng rng;
  rng.init(derive_key(B.seed, kTagEnv, (uint64_t)gi, 0), (uint64_t)gi, (uint64_t)rec[R_ENV_POS],
           rec[R_ENV_HAVE_SPARE] != 0.0, rec[R_ENV_SPARE]);
  double eps = c.tgt_lo;
  if (c.tgt_hi > c.tgt_lo) eps = rng.uniform(c.tgt_lo, c.tgt_hi);
  rec[R_EP_SPEED] = eps;
  double* qx = S.qxy;
  double* qy = S.qxy + R;
  bool placed = false;
  for (int attempt = 0; attempt < 1000 && !placed; ++attempt) {
    for (int i = 0; i < R; ++i) {
      const double r = c.disc_r * sqrt(rng.uniform());
      const double an = kTwoPi * rng.uniform();
      double sa, ca;
      sincos(an, &sa, &ca);
      qx[i] = r * ca;
      qy[i] = r * sa;
    }
    placed = true;
    for (int i = 0; i + 1 < R && placed; ++i)
      for (int j = i + 1; j < R && placed; ++j)
        if (norm2(qx[i] - qx[j], qy[i] - qy[j]) < c.min_sep) placed = false;
  }
  if (!placed) {
    rec[R_ENV_POS] = (double)rng.pos;
    return false;
  }
  for (int a = 0; a < A; ++a) {
    ag[V_X * A + a] = qx[a];
    ag[V_Y * A + a] = qy[a];
    ag[V_Z * A + a] = 0.0;
    ag[V_HEAD * A + a] = wrap_angle(kTwoPi * rng.uniform());
    ag[V_SPEED * A + a] = c.agent_speed;
    ag[V_RUDDER * A + a] = 2.0;
  }
  for (int t = 0; t < T; ++t) {
    const double depth = rng.uniform(c.depth_min, c.depth_max);
    tg[V_X * T + t] = qx[A + t];
    tg[V_Y * T + t] = qy[A + t];
    tg[V_Z * T + t] = depth;
    const double h = wrap_angle(kTwoPi * rng.uniform());
    tg[V_HEAD * T + t] = h;
    tg[V_SPEED * T + t] = eps;
    tg[V_RUDDER * T + t] = 2.0;
    tg[V_CMD * T + t] = h;
    tg[V_COUNTDOWN * T + t] = (double)rng.geometric_i32(c.turn_interval);
  }
  double* info = rec + c.o_info;
  for (int f = 0; f < I_NFIELD; ++f)
    for (int i = 0; i < AA; ++i) info[f * AA + i] = 0.0;
  for (int t = 0; t < T; ++t) rec[c.o_miss + t] = 0.0;
  rec[R_STEP] = 0.0;
  rec[R_EP_RETURN] = 0.0;
  rec[R_ENV_POS] = (double)rng.pos;
  rec[R_ENV_HAVE_SPARE] = rng.have_spare ? 1.0 : 0.0;
  rec[R_ENV_SPARE] = rng.spare;
  return true;
}

// Full spawn: serial part + every set's re-init. All threads. Returns false on
// spawn failure (CTA-uniform).
template <int PPT>
__device__ __noinline__ bool spawn_env(const DevConfig& c, const DevBatch& B, const Smem& S, BlockReducer& R, int64_t e,
                          int64_t gi) {
  if (threadIdx.x == 0) S.bc[8] = spawn_serial(c, B, S, gi) ? 1.0 : 0.0;
  __syncthreads();
  if (S.bc[8] == 0.0) return false;
  const int A = c.A, T = c.T;
  const double vmax = c.speed_margin * S.rec[R_EP_SPEED];
  const int64_t so = set_off(B, e);
  for (int a = 0; a < A; ++a) {
    const double cx = S.rec[c.o_agent + V_X * A + a], cy = S.rec[c.o_agent + V_Y * A + a];
    for (int t = 0; t < T; ++t) reinit_set<PPT>(c, B, S, R, gi, so + a * T + t, a * T + t, cx, cy, vmax);
  }
  return true;
}

// --------------------------------------------------------- outputs ---
// build_observation (env.cpp:412-453) / build_global_state (env.cpp:455-471) for
// env e into the batch layout (vecenv.cpp:47-56), plus masks (vecenv.cpp:58-67).
__device__ __noinline__ void write_tokens(const DevConfig& c, const DevBatch& B, const double* rec, int64_t e, double* obs,
                             bool with_global, bool with_masks) {
  const int A = c.A, T = c.T, R = c.R, Am = B.A_max, Rm = B.R_max, AA = A * A, AT = A * T;
  const double* ag = rec + c.o_agent;
  const double* tg = rec + c.o_target;
  const double* info = rec + c.o_info;
  const double* trk = rec + c.o_track;
  for (int p = threadIdx.x; p < Am * Rm; p += blockDim.x) {
    const int a = p / Rm, r = p - (p / Rm) * Rm;
    double v[12];
#pragma unroll
    for (int q = 0; q < 12; ++q) v[q] = 0.0;
    if (a < A && r < R) {
      const double sx = ag[V_X * A + a], sy = ag[V_Y * A + a], sz = ag[V_Z * A + a];
      if (r < A) {
        if (r == a) {
          double sh, ch;
          sincos(ag[V_HEAD * A + a], &sh, &ch);
          v[3] = sh;
          v[4] = ch;
          v[5] = ag[V_SPEED * A + a] / 1.0;
          v[6] = 1.0;
          v[9] = 1.0;
        } else {
          v[7] = 1.0;
          const int k = a * A + r;
          if (info[I_VALID * AA + k] != 0.0) {
            v[0] = (info[I_X * AA + k] - sx) / 1000.0;
            v[1] = (info[I_Y * AA + k] - sy) / 1000.0;
            v[2] = (info[I_Z * AA + k] - sz) / 1000.0;
            double sh, ch;
            sincos(info[I_HEAD * AA + k], &sh, &ch);
            v[3] = sh;
            v[4] = ch;
            v[5] = c.agent_speed / 1.0;
            v[9] = 1.0;
            v[10] = info[I_AGE * AA + k] / 10.0;
          }
        }
      } else {
        const int t = r - A, si = a * T + t;
        v[8] = 1.0;
        if (trk[K_EVER * AT + si] != 0.0) {
          v[0] = (trk[K_EX * AT + si] - sx) / 1000.0;
          v[1] = (trk[K_EY * AT + si] - sy) / 1000.0;
          v[2] = (tg[V_Z * T + t] - sz) / 1000.0;
          v[9] = 1.0;
          v[10] = trk[K_AGE * AT + si] / 10.0;
          v[11] = trk[K_SPREAD * AT + si] / 100.0;
        }
      }
    }
    const int64_t row = (e * Am + a) * Rm + r;
#pragma unroll
    for (int q = 0; q < 12; ++q) obs[(int64_t)q * B.obs_rows + row] = v[q];
  }
  if (with_global) {
    for (int r = threadIdx.x; r < Rm; r += blockDim.x) {
      double v[12];
#pragma unroll
      for (int q = 0; q < 12; ++q) v[q] = 0.0;
      if (r < R) {
        const bool is_agent = r < A;
        const double* src = is_agent ? ag : tg;
        const int n = is_agent ? A : T, i = is_agent ? r : r - A;
        v[0] = src[V_X * n + i] / 1000.0;
        v[1] = src[V_Y * n + i] / 1000.0;
        v[2] = src[V_Z * n + i] / 1000.0;
        double sh, ch;
        sincos(src[V_HEAD * n + i], &sh, &ch);
        v[3] = sh;
        v[4] = ch;
        v[5] = src[V_SPEED * n + i] / 1.0;
        v[is_agent ? 7 : 8] = 1.0;
        v[9] = 1.0;
      }
      const int64_t row = e * Rm + r;
#pragma unroll
      for (int q = 0; q < 12; ++q) B.global[(int64_t)q * B.global_rows + row] = v[q];
    }
  }
  if (with_masks) {
    for (int p = threadIdx.x; p < Am * 5; p += blockDim.x) {
      const int a = p / 5, k = p - (p / 5) * 5;
      uint8_t m = 0;
      if (a < A) m = abs(k - (int)ag[V_RUDDER * A + a]) <= 1 ? 1 : 0;
      B.masks[e * Am * 5 + p] = m;
    }
  }
}

// compute_reward_and_info (env.cpp:473-505) + VecEnv bookkeeping
// (vecenv.cpp:95-104) + device statistics. Thread 0 only. Returns done.
__device__ __noinline__ bool env_epilogue(const DevConfig& c, const DevBatch& B, const Smem& S, int64_t e) {
  const int A = c.A, T = c.T, AT = A * T, Tm = B.T_max;
  double* rec = S.rec;
  const double* ag = rec + c.o_agent;
  const double* tg = rec + c.o_target;
  const double* trk = rec + c.o_track;
  double reward_sum = 0.0, follow_sum = 0.0, err_sum = 0.0, lost_n = 0.0;
  for (int t = 0; t < T; ++t) {
    const double tx = tg[V_X * T + t], ty = tg[V_Y * T + t];
    double best_err = CUDART_INF, best_dist = CUDART_INF;
    for (int a = 0; a < A; ++a) {
      const int si = a * T + t;
      const double d = norm2(trk[K_EX * AT + si] - tx, trk[K_EY * AT + si] - ty);
      best_err = d < best_err ? d : best_err;
    }
    for (int a = 0; a < A; ++a) {
      const double d = hypot(ag[V_X * A + a] - tx, ag[V_Y * A + a] - ty);
      best_dist = d < best_dist ? d : best_dist;
    }
    const bool lost = rec[c.o_miss + t] >= (double)c.lost_steps;
    B.track_err[e * Tm + t] = best_err;
    B.min_dist[e * Tm + t] = best_dist;
    B.lost[e * Tm + t] = lost ? 1 : 0;
    // tracking_reward_single (env.cpp:83-90)
    double rt;
    if (best_err < c.eps_min) {
      rt = 1.0;
    } else if (best_err > c.eps_max) {
      rt = 0.0;
    } else {
      const double tt = (best_err - c.eps_min) / (c.eps_max - c.eps_min);
      rt = tt >= 1.0 ? 0.0 : exp(-2.0 * tt / (1.0 - tt));
    }
    reward_sum += rt;
    follow_sum += best_dist <= c.d_min ? 1.0 : 0.0;
    err_sum += best_err;
    lost_n += lost ? 1.0 : 0.0;
  }
  for (int t = T; t < Tm; ++t) {
    B.track_err[e * Tm + t] = 0.0;
    B.min_dist[e * Tm + t] = 0.0;
    B.lost[e * Tm + t] = 0;
  }
  bool crash = false;  // crash_check (env.cpp:99-104)
  for (int i = 0; i + 1 < A && !crash; ++i)
    for (int j = i + 1; j < A && !crash; ++j)
      if (norm3(ag[V_X * A + i] - ag[V_X * A + j], ag[V_Y * A + i] - ag[V_Y * A + j],
                ag[V_Z * A + i] - ag[V_Z * A + j]) < c.d_safe)
        crash = true;
  double reward;
  if (crash)
    reward = -1.0;
  else if (c.reward_mode == 0)
    reward = reward_sum / (double)T;
  else
    reward = follow_sum / (double)T;
  const double step = rec[R_STEP] + 1.0;
  rec[R_STEP] = step;
  const bool done = step >= (double)c.horizon;
  B.rewards[e] = reward;
  B.dones[e] = done ? 1 : 0;
  B.collision[e] = crash ? 1 : 0;
  // statistics (marl.cpp:288-306 accumulators)
  double* st = rec + c.o_stats;
  st[0] += 1.0;
  st[1] += reward;
  st[2] += err_sum / (double)T;
  st[5] += crash ? 1.0 : 0.0;
  st[6] += lost_n;
  rec[R_EP_RETURN] += reward;
  if (done) {
    st[3] += 1.0;
    st[4] += rec[R_EP_RETURN];
  }
  return done;
}

__device__ __forceinline__ void copy_rec(double* dst, const double* src, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// ================================================================ kernels ===
// The fused step: one CTA per env.
#ifndef UT_STEP_MIN_BLOCKS
#define UT_STEP_MIN_BLOCKS 2
#endif
template <int PPT>
__global__ void __launch_bounds__(256, UT_STEP_MIN_BLOCKS) step_kernel(DevBatch B, int mode, int32_t* status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t e = blockIdx.x;
  const DevConfig& c = cfg_of(B, e);
  const Smem S = carve(smem_raw, c.rec_words, c.A, c.T, c.P);
  BlockReducer R{S.red, 0};
  const int64_t gi = B.env_index_offset + e;
  double* grec = B.rec + rec_off(B, e);
  const long long tc0 = clock64();
  load_tables(S);
  copy_rec(S.rec, grec, c.rec_words);
  __syncthreads();
  if (threadIdx.x == 0) env_prologue(c, B, S, e, gi, mode);
  // first set's words, generated while thread 0 runs the prologue
  {
    const int AT = c.A * c.T;
    const uint64_t pos0 = (uint64_t)S.rec[c.o_track + K_POS * AT];
    gen_words(S.words[0], derive_key(B.seed, kTagPf, (uint64_t)gi, 0), 0, pos0,
              (c.noise_on ? 4ull * (uint64_t)c.P : 0ull) + 2ull);
  }
  __syncthreads();

  const long long tc1 = clock64();

  const int64_t so = set_off(B, e);
  double stat[3] = {0.0, 0.0, 0.0};
  int wb = 0;
  for (int a = 0; a < c.A; ++a)
    for (int t = 0; t < c.T; ++t) {
      step_set<PPT>(c, B, S, R, gi, so + a * c.T + t, a, t, wb, stat);
      wb ^= 1;
    }
  __syncthreads();
  const long long tc2 = clock64();

  if (threadIdx.x == 0) {
    S.rec[c.o_stats + 7] += stat[0];
    S.rec[c.o_stats + 8] += stat[1];
    S.rec[c.o_stats + 9] += stat[2];
    S.bc[9] = env_epilogue(c, B, S, e) ? 1.0 : 0.0;
  }
  __syncthreads();
  const bool done = S.bc[9] != 0.0;
  write_tokens(c, B, S.rec, e, B.obs, true, !done);
  long long tc3 = clock64(), tc4 = tc3;
  if (done) {
    write_tokens(c, B, S.rec, e, B.final_obs, false, false);
    __syncthreads();
    if (!spawn_env<PPT>(c, B, S, R, e, gi)) {
      if (threadIdx.x == 0) atomicMax(status, (int)ST_SPAWN_INFEASIBLE);
    }
    __syncthreads();
    write_tokens(c, B, S.rec, e, B.obs, true, true);
    tc4 = clock64();
  }
  if (threadIdx.x == 0) B.step[e] = (int32_t)S.rec[R_STEP];
  __syncthreads();
  copy_rec(grec, S.rec, c.rec_words);
  if (B.phase_cycles && threadIdx.x == 0) {
    unsigned long long* pc = B.phase_cycles + e * kPhaseCount;
    pc[PH_PROLOGUE] += (unsigned long long)(tc1 - tc0);
    pc[PH_FILTER] += (unsigned long long)(tc2 - tc1);
    pc[PH_OUTPUT] += (unsigned long long)(tc3 - tc2);
    pc[PH_RESET] += (unsigned long long)(tc4 - tc3);
  }
}

// Environment ctor / reset (env.cpp:110-151, 153-233) for every env. When
// `ctor` is set the record starts zeroed and each set's stream is advanced past
// pf::init's 8P draws (tracking.cpp:43-67), whose values spawn overwrites.
template <int PPT>
__global__ void reset_kernel(DevBatch B, int ctor, int32_t* status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t e = blockIdx.x;
  const DevConfig& c = cfg_of(B, e);
  const Smem S = carve(smem_raw, c.rec_words, c.A, c.T, c.P);
  BlockReducer R{S.red, 0};
  const int64_t gi = B.env_index_offset + e;
  double* grec = B.rec + rec_off(B, e);
  if (ctor) {
    for (int i = threadIdx.x; i < c.rec_words; i += blockDim.x) S.rec[i] = 0.0;
    __syncthreads();
    const int AT = c.A * c.T;
    for (int i = threadIdx.x; i < AT; i += blockDim.x) {
      S.rec[c.o_track + K_POS * AT + i] = 8.0 * (double)c.P;
      S.rec[c.o_track + K_MAXSPEED * AT + i] = 1.0;
    }
    for (int a = threadIdx.x; a < c.A; a += blockDim.x) S.rec[c.o_agent + V_RUDDER * c.A + a] = 2.0;
    for (int t = threadIdx.x; t < c.T; t += blockDim.x) S.rec[c.o_target + V_RUDDER * c.T + t] = 2.0;
  } else {
    copy_rec(S.rec, grec, c.rec_words);
  }
  __syncthreads();
  if (!spawn_env<PPT>(c, B, S, R, e, gi)) {
    if (threadIdx.x == 0) atomicMax(status, (int)ST_SPAWN_INFEASIBLE);
  }
  __syncthreads();
  write_tokens(c, B, S.rec, e, B.obs, true, true);
  if (threadIdx.x == 0) {
    B.rewards[e] = 0.0;
    B.dones[e] = 0;
    B.step[e] = (int32_t)S.rec[R_STEP];
  }
  __syncthreads();
  copy_rec(grec, S.rec, c.rec_words);
}

// VecEnv::refresh_outputs (vecenv.cpp:145-150).
__global__ void tokens_kernel(DevBatch B) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t e = blockIdx.x;
  const DevConfig& c = cfg_of(B, e);
  double* rec = reinterpret_cast<double*>(smem_raw);
  copy_rec(rec, B.rec + rec_off(B, e), c.rec_words);
  __syncthreads();
  write_tokens(c, B, rec, e, B.obs, true, true);
  if (threadIdx.x == 0) B.step[e] = (int32_t)rec[R_STEP];
}

// Action validation for VecEnv::step (env.cpp:236-248) before anything moves.
__global__ void validate_kernel(DevBatch B) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= B.n_envs) return;
  const DevConfig& c = cfg_of(B, e);
  const double* rec = B.rec + rec_off(B, e);
  for (int a = 0; a < c.A; ++a) {
    const int act = B.actions[e * B.A_max + a];
    const int rud = (int)rec[c.o_agent + V_RUDDER * c.A + a];
    if (act < 0 || act >= 5 || abs(act - rud) > 1) {
      atomicMin(B.error_env, (int32_t)e);
      return;
    }
  }
}

// Sum of the per-env statistics (deterministic single-CTA tree), optional reset.
__global__ void stats_kernel(DevBatch B, double* out, int reset) {
  __shared__ double red[kRedDoubles];
  BlockReducer R{red, 0};
  for (int k = 0; k < kStatCount; ++k) {
    double acc = 0.0;
    for (int64_t e = threadIdx.x; e < B.n_envs; e += blockDim.x) {
      const DevConfig& c = cfg_of(B, e);
      double* st = B.rec + rec_off(B, e) + c.o_stats;
      acc = acc + st[k];
      if (reset) st[k] = 0.0;
    }
    const double s = R.sum(acc);
    if (threadIdx.x == 0) out[k] = s;
  }
}

}  // namespace ut
