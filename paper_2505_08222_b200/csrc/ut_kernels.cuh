// ut_kernels.cuh -- the fused environment-step kernel and its helpers.
//
// One persistent, cooperative launch per step ("one fused kernel per step",
// north_star), in phases separated by grid barriers. Phases 1, 3 and 4 walk the
// CTA's contiguous env range in chunks of blockDim.x envs; phase 2 takes envs one
// at a time from a global counter, so every CTA stays busy until the end:
//
//   1. PROLOGUE  one env per THREAD: actions, move_targets, move_agents,
//      measure_ranges and the comm-drop decisions, in the reference's serial
//      env-stream order, on that env's structure-of-arrays
//      record (coalesced across the threads of the chunk). The ping schedule is
//      handed to phase 2 through a small per-env scratch.
//   2. FILTER    the whole CTA streams through every particle set of each env it
//      claims (an env's sets are contiguous in HBM), each set held in
//      registers -- PPT consecutive particles per thread, 128-bit loads/stores,
//      read once and written once per step: predict (Philox words generated one
//      set ahead, correctly rounded fp32 Box-Muller), ONE merged pass for all of
//      the set's range updates (the reference's sequential semantics preserved,
//      exact sequential path when an intermediate underflow could matter), ESS
//      from the same reduction, systematic resample, estimate.
//   3. OUTPUT    one env per thread: reward, done, info, stats; then tokens,
//      global state and masks with one thread per token row.
//   4. RESET     finished envs: spawn (one env per thread) + particle re-init
//      (whole CTA per set) + fresh tokens.
#pragma once
#include <cooperative_groups.h>

#include "ut_device.cuh"

namespace ut {
namespace cg = cooperative_groups;

enum StepMode : int { MODE_EXTERNAL = -1, MODE_RANDOM = 0, MODE_SCRIPTED = 1 };
enum DevStatus : int { ST_OK = 0, ST_SPAWN_INFEASIBLE = 2 };
constexpr int kMaxMerged = 8;     // merged update handles up to 8 measurements per set
constexpr int kMbStride = 36;     // stage-maxima row stride (uint32; 8 x 36 fit one reducer buffer)
static_assert(kMaxMerged * kMbStride <= 2 * kRedSlots, "stage maxima exceed a reducer buffer");
constexpr int kMeasStride = 8;    // ox, oy, r2, sigma, -1/(2 sigma^2) (+pad)
constexpr int kMaxEntities = 64;  // spawn scratch per thread
constexpr double kMergeFloor = 0x1p-860;  // see the merged-update argument in step_set
constexpr int kChunkFlagDone = 1, kChunkFlagSpawned = 2;
constexpr int kBcStatUpdates = 8, kBcStatResamples = 9, kBcStatExact = 10;  // Smem::bc slots
constexpr int kBcClaim = 11;  // the filter phase's claimed envs (int), two slots used in turn

// Strided view of one env's record: word w at p[w * n_envs].
struct Rec {
  double* p;
  int64_t s;
  __device__ __forceinline__ double& operator[](int w) const { return p[(int64_t)w * s]; }
};
__device__ __forceinline__ Rec rec_of(const DevBatch& B, int64_t e) { return Rec{B.rec + e, B.n_envs}; }

#define AG(f, a) rec[c.o_agent + (f) * c.sA + (a)]
#define TG(f, t) rec[c.o_target + (f) * c.sT + (t)]
#define INFO(f, k) rec[c.o_info + (f) * c.sA * c.sA + (k)]
#define TRK(f, ti) rec[c.o_track + (f) * c.sA * c.sT + (ti)]
#define STAT(k) rec[c.o_stats + (k)]

// ------------------------------------------------------------ smem carve ---
// staged per-set scalars (Smem::trk)
enum : int { TK_POS = 0, TK_MAXSPEED, TK_EX, TK_EY, TK_ESSOK, TK_AGE, TK_EVER, TK_KEY, kTrkStride };

struct Smem {
  double2* tab_log;  // [128]
  double2* tab_sc;   // [64][8] (replicated, see sincos_table)
  double* tab_exp;   // [32][16] (replicated, see exp_neg)
  DevConfig* cfg;    // config of the env being filtered
  double* red;       // kRedDoubles: BlockReducer buffers + scan warp sums
  double* bc;        // 16 broadcast slots (0: resample draw; kBcStat*: the env's filter statistics)
  double* meas;      // [sA*sT][kMeasStride] pings of the env being filtered
  uint16_t* mcount;  // [sA*sT] measurements applied to each set this step
  uint16_t* mlist;   // [sA*sT][sA] their meas indices in application order
  double* trk;       // [sA*sT][kTrkStride] the sets' track scalars + PF stream keys
  uint8_t* flags;    // [blockDim] per-env chunk flags
  uint4* bnd;        // [A*T][4 nw + 2] the env's warp-boundary Philox blocks (stage_bnd)
  uint64_t* mbar;    // TMA completion barrier
  uint32_t mbar_sa, pf_sa;  // their shared-window addresses (computed once)
  double* pf;        // [5][P] TMA-prefetched next particle set
  double* cum;       // [P] resample scan | re-init words
  double* st;        // [4P] resample staging
  double2* park;     // [2][P/2] vx, vy of the merged pass, pair-chunked (park_field)
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }


// Fixed-size part of the layout for a particle capacity NP (compile-time
// offsets: every access is an LDS/STS with an immediate offset). The
// fleet-sized regions follow at runtime offsets.
template <int NP>
struct FixedSmem {
  double2 tab_log[128];
  double2 tab_sc[64 * 8];
  double tab_exp[32 * 16];
  double red[kRedDoubles];
  double bc[16];
  uint64_t mbar[2];
  // phase timers (thread 0): the phases, barrier waits, the running section's
  // start, and the launch's start clock / globaltimer. Kept in the dynamic
  // block like everything else: the kernels share out-of-line device functions
  // that address shared memory at fixed offsets, so no kernel may add static
  // shared variables in front of the dynamic block.
  long long ph[kPhaseWait + 4];
  // one particle set: the TMA landing zone of the set being read, then (once
  // every thread holds its particles) the staging of the exact update and the
  // resample, and in the reset phase the re-init words
  double pf[5 * NP];
  // vx / vy parked during the merged pass's likelihood stages, in lane-contiguous
  // 16-byte chunks (the set buffer's own-slot layout puts a quarter-warp's 128-bit
  // accesses on half the banks)
  double2 park[NP];
  DevConfig cfg;
};

// Philox blocks of one set's noise that a warp's lanes do not cover themselves
// (stage_bnd): for each of the 4 segments, the block after each warp's range;
// then the two blocks holding the resample draw.
__host__ __device__ constexpr int bnd_per_set(int nw) { return 4 * nw + 2; }

template <int NP>
__host__ __device__ inline size_t smem_bytes(int sA, int sT, int nt) {
  size_t s = align16(sizeof(FixedSmem<NP>));
  s += align16(sizeof(double) * kMeasStride * sA * sT);
  s += align16(sizeof(uint16_t) * sA * sT);
  s += align16(sizeof(uint16_t) * sA * sT * sA);
  s += align16(sizeof(double) * kTrkStride * sA * sT);
  s += align16(nt);
  s += sizeof(uint4) * sA * sT * bnd_per_set(nt / 32);
  return s;
}

template <int NP>
__device__ __forceinline__ Smem carve(unsigned char* base, int sA, int sT) {
  FixedSmem<NP>& F = *reinterpret_cast<FixedSmem<NP>*>(base);
  Smem S;
  S.tab_log = F.tab_log;
  S.tab_sc = F.tab_sc;
  S.tab_exp = F.tab_exp;
  S.cfg = &F.cfg;
  S.red = F.red;
  S.bc = F.bc;
  S.mbar = F.mbar;
  S.mbar_sa = smem_addr(F.mbar);
  S.pf_sa = smem_addr(F.pf);
  S.pf = F.pf;
  S.st = F.pf;
  S.cum = F.pf + 4 * NP;
  S.park = F.park;
  size_t o = align16(sizeof(FixedSmem<NP>));
  S.meas = (double*)(base + o);
  o += align16(sizeof(double) * kMeasStride * sA * sT);
  S.mcount = (uint16_t*)(base + o);
  o += align16(sizeof(uint16_t) * sA * sT);
  S.mlist = (uint16_t*)(base + o);
  o += align16(sizeof(uint16_t) * sA * sT * sA);
  S.trk = (double*)(base + o);
  o += align16(sizeof(double) * kTrkStride * sA * sT);
  S.flags = base + o;
  o += align16(blockDim.x);
  S.bnd = reinterpret_cast<uint4*>(base + o);
  return S;
}

template <int NP>
__device__ __forceinline__ Smem carve_dyn(int sA, int sT) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  return carve<NP>(smem_raw, sA, sT);
}

__device__ __forceinline__ const DevConfig& cfg_of(const DevBatch& B, int64_t e) {
  return B.cfgs[B.cfg_of_env ? B.cfg_of_env[e] : 0];
}
__device__ __forceinline__ int64_t set_off(const DevBatch& B, int64_t e) {
  return B.set_offset ? B.set_offset[e] : e * (int64_t)(B.cfgs[0].A * B.cfgs[0].T);
}

// Phase timing (PhaseTimer, env.cpp:18-36, enabled when B.phase_cycles is set):
// thread 0 of the CTA closes the running section into phase k and opens the
// next; the CTA's sums are flushed to B.phase_cycles at the end of the launch.
constexpr int kPhLast = kPhaseWait + 1;  // Smem::ph slots: running section start, then launch start clock / ns
__device__ __forceinline__ long long* ph_slots() {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  return reinterpret_cast<FixedSmem<256>*>(smem_raw)->ph;  // offset independent of NP (precedes pf)
}
__device__ __forceinline__ void ph_mark(const DevBatch& B, int k) {
  if (threadIdx.x == 0 && B.phase_cycles != nullptr) {
    long long* g_ph = ph_slots();
    const long long now = clock64();
    g_ph[k] += now - g_ph[kPhLast];
    g_ph[kPhLast] = now;
  }
}
// The same for a section that belongs to two phases in the ratio num : den - num.
__device__ __forceinline__ void ph_mark_split(const DevBatch& B, int k1, int k2, int num, int den) {
  if (threadIdx.x == 0 && B.phase_cycles != nullptr) {
    long long* g_ph = ph_slots();
    const long long now = clock64();
    const long long d = now - g_ph[kPhLast];
    const long long d1 = den > 0 ? d * num / den : d;
    g_ph[k1] += d1;
    g_ph[k2] += d - d1;
    g_ph[kPhLast] = now;
  }
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void load_tables(const Smem& S) {
  for (int i = threadIdx.x; i < 128; i += blockDim.x) S.tab_log[i] = make_double2(kLogTab[2 * i], kLogTab[2 * i + 1]);
  for (int i = threadIdx.x; i < 64 * 8; i += blockDim.x)
    S.tab_sc[i] = make_double2(kSinCosTab[2 * (i >> 3)], kSinCosTab[2 * (i >> 3) + 1]);
  for (int i = threadIdx.x; i < 32 * 16; i += blockDim.x) S.tab_exp[i] = kExp2Tab[i >> 4];
}

// The CTA's contiguous env range.
__device__ __forceinline__ void cta_range(int64_t n, int64_t& lo, int64_t& hi) {
  const int64_t base = n / gridDim.x, extra = n % gridDim.x, b = blockIdx.x;
  lo = b * base + (b < extra ? b : extra);
  hi = lo + base + (b < extra ? 1 : 0);
}

// ------------------------------------------------ per-env serial phases ---
// Environment::scripted_action (env.cpp:511-543) on the pre-step state of agent
// a (only its own pose and tracks are read, so it may run right before a moves).
__device__ __noinline__ int scripted_action(const DevConfig& c, const Rec& rec, int a) {
  const int T = c.T;
  const double sx = AG(V_X, a), sy = AG(V_Y, a), sh = AG(V_HEAD, a);
  const int rud = (int)AG(V_RUDDER, a);
  double gx = sx, gy = sy, best = CUDART_INF;
  for (int t = 0; t < T; ++t) {
    const int ti = a * c.sT + t;
    const double ex = TRK(K_EX, ti), ey = TRK(K_EY, ti);
    const double d = norm2(ex - sx, ey - sy);
    const double penalty = TRK(K_EVER, ti) != 0.0 ? 0.0 : 1e6;
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
  return best_act;
}

// Actions + move_targets + move_agents + measure_ranges + comm decisions for
// env e, in the reference's env-stream draw order. Writes
// the ping schedule (horizontal ranges, present and link flags) to scratch.
__device__ __noinline__ void env_prologue(const DevConfig& c, const DevBatch& B, int64_t e, int64_t gi, int mode) {
  const Rec rec = rec_of(B, e);
  const int A = c.A, T = c.T, sA = c.sA, sT = c.sT, AA = sA * sA;
  double* r2 = B.sched_r2 + e * (int64_t)(sA * sT);
  uint8_t* present = B.sched_flags + e * (int64_t)(sA * sT + AA);
  uint8_t* link = present + sA * sT;
  SerialRng rng;
  rng.init(derive_key(B.seed, kTagEnv, (uint64_t)gi, 0), (uint64_t)gi, (uint64_t)rec[R_ENV_POS],
           rec[R_ENV_HAVE_SPARE] != 0.0, rec[R_ENV_SPARE]);

  // move_targets (env.cpp:289-304)
  for (int t = 0; t < T; ++t) {
    if (TG(V_COUNTDOWN, t) <= 0.0) {
      TG(V_CMD, t) = wrap_angle(kTwoPi * rng.uniform());
      TG(V_COUNTDOWN, t) = (double)rng.geometric_i32(c.turn_interval);
    }
    const double want = wrap_angle(TG(V_CMD, t) - TG(V_HEAD, t));
    const double mt = c.max_turn;
    const double dpsi = want < -mt ? -mt : (mt < want ? mt : want);
    const double noise = c.head_noise > 0.0 ? c.head_noise * rng.normal() : 0.0;
    // advance_vehicle (kinematics.cpp:42-49)
    const double h = wrap_angle(TG(V_HEAD, t) + dpsi + noise);
    TG(V_HEAD, t) = h;
    TG(V_X, t) += TG(V_SPEED, t) * c.dt * cos(h);
    TG(V_Y, t) += TG(V_SPEED, t) * c.dt * sin(h);
    TG(V_COUNTDOWN, t) -= 1.0;
  }
  ph_mark(B, PH_TARGETS);
  // actions (VecEnv::step_policy vecenv.cpp:118-135 or the caller's) + move_agents
  // (env.cpp:306-316, step_vehicle kinematics.cpp:51-56). The bench stream is
  // separate from the env stream and every action depends only on the agent's
  // own pre-step state, so choosing each action right before its agent moves
  // draws exactly the reference's values.
  SerialRng bench;
  if (mode == MODE_RANDOM)
    bench.init(derive_key(B.seed, kTagBench, (uint64_t)gi, 0), (uint64_t)gi, (uint64_t)rec[R_BENCH_POS], false, 0.0);
  for (int a = 0; a < A; ++a) {
    int act;
    if (mode == MODE_RANDOM) {
      const int rud = (int)AG(V_RUDDER, a);
      const int lo = rud > 0 ? rud - 1 : 0, hi = rud < 4 ? rud + 1 : 4;
      act = lo + (int)bench.uniform_int((uint32_t)(hi - lo + 1));
    } else if (mode == MODE_SCRIPTED) {
      act = scripted_action(c, rec, a);
    } else {
      act = B.actions[e * B.A_max + a];
    }
    AG(V_RUDDER, a) = (double)act;
    const double gamma = -0.24 + 0.12 * act;
    double noise = c.head_noise > 0.0 ? c.head_noise * rng.normal() : 0.0;
    if (c.pert_std > 0.0) noise += c.pert_std * rng.normal();
    const double dpsi = c.head_a * gamma + c.head_b;
    const double h = wrap_angle(AG(V_HEAD, a) + dpsi + noise);
    AG(V_HEAD, a) = h;
    AG(V_X, a) += AG(V_SPEED, a) * c.dt * cos(h);
    AG(V_Y, a) += AG(V_SPEED, a) * c.dt * sin(h);
  }
  if (mode == MODE_RANDOM) rec[R_BENCH_POS] = (double)bench.pos;
  ph_mark(B, PH_AGENTS);
  // measure_ranges (env.cpp:318-347): targets outer, agents inner
  for (int t = 0; t < T; ++t) {
    bool detected = false;
    const double tx = TG(V_X, t), ty = TG(V_Y, t), tz = TG(V_Z, t);
    for (int a = 0; a < A; ++a) {
      const int idx = a * sT + t;
      present[idx] = 0;
      const double ax = AG(V_X, a), ay = AG(V_Y, a), az = AG(V_Z, a);
      const double dist3 = norm3(ax - tx, ay - ty, az - tz);
      if (dist3 > c.det_range) continue;
      if (c.drop > 0.0 && rng.uniform() < c.drop) continue;
      double r3 = dist3;
      if (c.range_noise > 0.0) r3 += c.range_noise * rng.normal();
      r3 = r3 < 0.0 ? 0.0 : r3;
      const double dd = tz - az;
      const double sq = r3 * r3 - dd * dd;  // slant_to_horizontal (tracking.cpp:9-14)
      r2[idx] = sq <= 0.0 ? 0.0 : sqrt(sq);
      present[idx] = 1;
      detected = true;
    }
    rec[c.o_miss + t] = detected ? 0.0 : rec[c.o_miss + t] + 1.0;
  }
  ph_mark(B, PH_MEASURE);
  // exchange_comms decisions (env.cpp:365-383); AgentInfo ages first
  for (int r = 0; r < A; ++r)
    for (int s = 0; s < A; ++s) INFO(I_AGE, r * sA + s) += 1.0;
  for (int r = 0; r < A; ++r) {
    const double rx = AG(V_X, r), ry = AG(V_Y, r), rz = AG(V_Z, r);
    for (int s = 0; s < A; ++s) {
      const int k = r * sA + s;
      link[k] = 0;
      if (s == r) continue;
      const double sx = AG(V_X, s), sy = AG(V_Y, s), sz = AG(V_Z, s);
      if (norm3(rx - sx, ry - sy, rz - sz) > c.comm_range) continue;
      if (c.drop > 0.0 && rng.uniform() < c.drop) continue;
      INFO(I_X, k) = sx;
      INFO(I_Y, k) = sy;
      INFO(I_Z, k) = sz;
      INFO(I_HEAD, k) = AG(V_HEAD, s);
      INFO(I_AGE, k) = 0.0;
      INFO(I_VALID, k) = 1.0;
      link[k] = 1;
    }
  }
  rec[R_ENV_POS] = (double)rng.pos;
  rec[R_ENV_HAVE_SPARE] = rng.have_spare ? 1.0 : 0.0;
  rec[R_ENV_SPARE] = rng.spare;
  ph_mark(B, PH_COMMS);
}

// compute_reward_and_info (env.cpp:473-505) + VecEnv bookkeeping
// (vecenv.cpp:95-104) + device statistics for env e. Returns done.
// append_trajectory_rows (trajectory.cpp:13-66) for env e after its step: agents,
// then targets with the best-informed track (first agent with the smallest
// error, as the reward attributes it) and this step's tracking error.
__device__ __noinline__ void write_trajectory(const DevConfig& c, const DevBatch& B, int64_t e, double reward,
                                              bool crash, double step) {
  const Rec rec = rec_of(B, e);
  const int A = c.A, T = c.T;
  double* out = B.traj + (e - B.traj_lo) * (int64_t)B.R_max * kTrajFields;
  for (int r = 0; r < B.R_max; ++r) {
    double* row = out + (int64_t)r * kTrajFields;
    for (int f = 0; f < kTrajFields; ++f) row[f] = 0.0;
    row[TJ_STEP] = r < A + T ? step : -1.0;  // -1: padding row of a smaller fleet
    if (r >= A + T) continue;
    const bool tgt = r >= A;
    const int i = tgt ? r - A : r;
    row[TJ_X] = tgt ? TG(V_X, i) : AG(V_X, i);
    row[TJ_Y] = tgt ? TG(V_Y, i) : AG(V_Y, i);
    row[TJ_Z] = tgt ? TG(V_Z, i) : AG(V_Z, i);
    row[TJ_HEAD] = tgt ? TG(V_HEAD, i) : AG(V_HEAD, i);
    row[TJ_REWARD] = reward;
    row[TJ_COLLISION] = crash ? 1.0 : 0.0;
    row[TJ_IS_TARGET] = tgt ? 1.0 : 0.0;
    if (tgt) {
      double best = CUDART_INF;
      for (int a = 0; a < A; ++a) {
        const int ti = a * c.sT + i;
        const double d = norm2(TRK(K_EX, ti) - TG(V_X, i), TRK(K_EY, ti) - TG(V_Y, i));
        if (d < best) {
          best = d;
          row[TJ_HAS_EST] = 1.0;
          row[TJ_EST_X] = TRK(K_EX, ti);
          row[TJ_EST_Y] = TRK(K_EY, ti);
        }
      }
      row[TJ_ERR] = best;  // out.tracking_error[t] (step > 0)
    }
  }
}

__device__ __noinline__ bool env_epilogue(const DevConfig& c, const DevBatch& B, int64_t e) {
  const Rec rec = rec_of(B, e);
  const int A = c.A, T = c.T, Tm = B.T_max;
  double reward_sum = 0.0, follow_sum = 0.0, err_sum = 0.0, lost_n = 0.0, dist_all = 0.0;
  for (int t = 0; t < T; ++t) {
    const double tx = TG(V_X, t), ty = TG(V_Y, t);
    double best_err = CUDART_INF, best_dist = CUDART_INF;
    for (int a = 0; a < A; ++a) {
      const int ti = a * c.sT + t;
      const double d = norm2(TRK(K_EX, ti) - tx, TRK(K_EY, ti) - ty);
      best_err = d < best_err ? d : best_err;
    }
    for (int a = 0; a < A; ++a) {
      const double d = hypot(AG(V_X, a) - tx, AG(V_Y, a) - ty);
      best_dist = d < best_dist ? d : best_dist;
      dist_all = dist_all + d;
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
      if (norm3(AG(V_X, i) - AG(V_X, j), AG(V_Y, i) - AG(V_Y, j), AG(V_Z, i) - AG(V_Z, j)) < c.d_safe) crash = true;
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
  B.step[e] = (int32_t)step;
  // statistics (marl.cpp:288-306 accumulators)
  STAT(0) += 1.0;
  STAT(1) += reward;
  STAT(2) += err_sum / (double)T;
  STAT(5) += crash ? 1.0 : 0.0;
  STAT(6) += lost_n;
  rec[R_EP_RETURN] += reward;
  if (B.traj && e >= B.traj_lo && e < B.traj_hi) write_trajectory(c, B, e, reward, crash, step);
  // evaluation accumulators (curriculum.cpp:307-325, agents outer over targets
  // there; here targets outer -- a different summation order of the same terms)
  rec[R_EV_DIST] += dist_all;
  rec[R_EV_ERR] += err_sum;
  rec[R_EV_FLAGS] = (double)((int)rec[R_EV_FLAGS] | (crash ? 1 : 0) | (lost_n > 0.0 ? 2 : 0));
  if (done) {
    STAT(3) += 1.0;
    STAT(4) += rec[R_EP_RETURN];
    // per-episode means over the horizon's steps (curriculum.cpp:327-328)
    const double md = rec[R_EV_DIST] / ((double)c.horizon * A * T);
    const double me = rec[R_EV_ERR] / ((double)c.horizon * T);
    const int fl = (int)rec[R_EV_FLAGS];
    STAT(10) += md;
    STAT(11) += md * md;
    STAT(12) += me;
    STAT(13) += me * me;
    STAT(14) += (fl & 1) ? 1.0 : 0.0;
    STAT(15) += (fl & 2) ? 1.0 : 0.0;
    rec[R_EV_DIST] = 0.0;
    rec[R_EV_ERR] = 0.0;
    rec[R_EV_FLAGS] = 0.0;
  }
  return done;
}

// Environment::spawn, serial part (env.cpp:155-212, 221-224) for env e.
// Returns false when the rejection sampling fails (ConfigError in the reference).
__device__ __noinline__ bool spawn_serial(const DevConfig& c, const DevBatch& B, int64_t e, int64_t gi) {
  const Rec rec = rec_of(B, e);
  const int A = c.A, T = c.T, R = c.R, sA = c.sA;
  SerialRng rng;
  rng.init(derive_key(B.seed, kTagEnv, (uint64_t)gi, 0), (uint64_t)gi, (uint64_t)rec[R_ENV_POS],
           rec[R_ENV_HAVE_SPARE] != 0.0, rec[R_ENV_SPARE]);
  double eps = c.tgt_lo;
  if (c.tgt_hi > c.tgt_lo) eps = rng.uniform(c.tgt_lo, c.tgt_hi);
  rec[R_EP_SPEED] = eps;
  double qx[kMaxEntities], qy[kMaxEntities];
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
    AG(V_X, a) = qx[a];
    AG(V_Y, a) = qy[a];
    AG(V_Z, a) = 0.0;
    AG(V_HEAD, a) = wrap_angle(kTwoPi * rng.uniform());
    AG(V_SPEED, a) = c.agent_speed;
    AG(V_RUDDER, a) = 2.0;
  }
  for (int t = 0; t < T; ++t) {
    const double depth = rng.uniform(c.depth_min, c.depth_max);
    TG(V_X, t) = qx[A + t];
    TG(V_Y, t) = qy[A + t];
    TG(V_Z, t) = depth;
    const double h = wrap_angle(kTwoPi * rng.uniform());
    TG(V_HEAD, t) = h;
    TG(V_SPEED, t) = eps;
    TG(V_RUDDER, t) = 2.0;
    TG(V_CMD, t) = h;
    TG(V_COUNTDOWN, t) = (double)rng.geometric_i32(c.turn_interval);
  }
  for (int f = 0; f < I_NFIELD; ++f)
    for (int r = 0; r < A; ++r)
      for (int s = 0; s < A; ++s) INFO(f, r * sA + s) = 0.0;
  for (int t = 0; t < T; ++t) rec[c.o_miss + t] = 0.0;
  rec[R_STEP] = 0.0;
  rec[R_EP_RETURN] = 0.0;
  rec[R_EV_DIST] = 0.0;
  rec[R_EV_ERR] = 0.0;
  rec[R_EV_FLAGS] = 0.0;
  rec[R_ENV_POS] = (double)rng.pos;
  rec[R_ENV_HAVE_SPARE] = rng.have_spare ? 1.0 : 0.0;
  rec[R_ENV_SPARE] = rng.spare;
  return true;
}

// ----------------------------------------------------------- outputs ---
// build_observation (env.cpp:412-453) for (env, agent, row) into the batch
// layout (vecenv.cpp:47-53); padding rows of mixed fleets are zero.
__device__ __forceinline__ void token_row(const DevConfig& c, const Rec& rec, int a, int r, double v[12]) {
#pragma unroll
  for (int q = 0; q < 12; ++q) v[q] = 0.0;
  const int A = c.A, R = c.R;
  if (a >= A || r >= R) return;
  const double sx = AG(V_X, a), sy = AG(V_Y, a), sz = AG(V_Z, a);
  if (r < A) {
    if (r == a) {
      double sh, ch;
      sincos(AG(V_HEAD, a), &sh, &ch);
      v[3] = sh;
      v[4] = ch;
      v[5] = AG(V_SPEED, a) / 1.0;
      v[6] = 1.0;
      v[9] = 1.0;
    } else {
      v[7] = 1.0;
      const int k = a * c.sA + r;
      if (INFO(I_VALID, k) != 0.0) {
        v[0] = (INFO(I_X, k) - sx) / 1000.0;
        v[1] = (INFO(I_Y, k) - sy) / 1000.0;
        v[2] = (INFO(I_Z, k) - sz) / 1000.0;
        double sh, ch;
        sincos(INFO(I_HEAD, k), &sh, &ch);
        v[3] = sh;
        v[4] = ch;
        v[5] = c.agent_speed / 1.0;
        v[9] = 1.0;
        v[10] = INFO(I_AGE, k) / 10.0;
      }
    }
  } else {
    const int t = r - A, ti = a * c.sT + t;
    v[8] = 1.0;
    if (TRK(K_EVER, ti) != 0.0) {
      v[0] = (TRK(K_EX, ti) - sx) / 1000.0;
      v[1] = (TRK(K_EY, ti) - sy) / 1000.0;
      v[2] = (TG(V_Z, t) - sz) / 1000.0;
      v[9] = 1.0;
      v[10] = TRK(K_AGE, ti) / 10.0;
      v[11] = TRK(K_SPREAD, ti) / 100.0;
    }
  }
}

// build_global_state (env.cpp:455-471) row r of env e (vecenv.cpp:55).
__device__ __forceinline__ void global_row(const DevConfig& c, const Rec& rec, int r, double v[12]) {
#pragma unroll
  for (int q = 0; q < 12; ++q) v[q] = 0.0;
  if (r >= c.R) return;
  const bool is_agent = r < c.A;
  const int base = is_agent ? c.o_agent : c.o_target, stride = is_agent ? c.sA : c.sT;
  const int i = is_agent ? r : r - c.A;
  v[0] = rec[base + V_X * stride + i] / 1000.0;
  v[1] = rec[base + V_Y * stride + i] / 1000.0;
  v[2] = rec[base + V_Z * stride + i] / 1000.0;
  double sh, ch;
  sincos(rec[base + V_HEAD * stride + i], &sh, &ch);
  v[3] = sh;
  v[4] = ch;
  v[5] = rec[base + V_SPEED * stride + i] / 1.0;
  v[is_agent ? 7 : 8] = 1.0;
  v[9] = 1.0;
}

// Tokens / global rows / masks (vecenv.cpp:47-67) of envs [e0, e1), one thread
// per row. `sel` (optional) restricts to envs whose chunk flag has that bit;
// `final_obs` writes the observation rows into the final_obs buffer only.
__device__ __noinline__ void write_outputs(const DevBatch& B, int64_t e0, int64_t e1, const uint8_t* flags, int sel,
                                           bool final_obs) {
  const int Am = B.A_max, Rm = B.R_max;
  const int64_t n = e1 - e0;
  double* obs = final_obs ? B.final_obs : B.obs;
  for (int64_t p = threadIdx.x; p < n * Am * Rm; p += blockDim.x) {
    const int64_t le = p / (Am * Rm);
    if (sel && !(flags[le] & sel)) continue;
    const int q = (int)(p - le * Am * Rm), a = q / Rm, r = q - (q / Rm) * Rm;
    const int64_t e = e0 + le;
    double v[12];
    token_row(cfg_of(B, e), rec_of(B, e), a, r, v);
    const int64_t row = (e * Am + a) * Rm + r;
#pragma unroll
    for (int k = 0; k < 12; ++k) obs[(int64_t)k * B.obs_rows + row] = v[k];
  }
  if (final_obs) return;
  for (int64_t p = threadIdx.x; p < n * Rm; p += blockDim.x) {
    const int64_t le = p / Rm;
    if (sel && !(flags[le] & sel)) continue;
    const int r = (int)(p - le * Rm);
    const int64_t e = e0 + le;
    double v[12];
    global_row(cfg_of(B, e), rec_of(B, e), r, v);
    const int64_t row = e * Rm + r;
#pragma unroll
    for (int k = 0; k < 12; ++k) B.global[(int64_t)k * B.global_rows + row] = v[k];
  }
  for (int64_t p = threadIdx.x; p < n * Am * 5; p += blockDim.x) {
    const int64_t le = p / (Am * 5);
    if (sel && !(flags[le] & sel)) continue;
    const int q = (int)(p - le * Am * 5), a = q / 5, k = q - (q / 5) * 5;
    const int64_t e = e0 + le;
    const DevConfig& c = cfg_of(B, e);
    const Rec rec = rec_of(B, e);
    B.masks[e * Am * 5 + q] = (a < c.A && abs(k - (int)AG(V_RUDDER, a)) <= 1) ? 1 : 0;
  }
}

// Double-buffered outputs: this step's set last held the outputs of two steps
// ago; the terminal rows written into the other set at the previous step (its
// envs with done set) are copied over, so every set holds every env's latest
// terminal observation (the single buffer's semantics) without a full-buffer copy.
__device__ __noinline__ void copy_final_rows(const DevBatch& B, int64_t e0, int64_t e1) {
  const int Am = B.A_max, Rm = B.R_max;
  const int64_t n = e1 - e0;
  for (int64_t p = threadIdx.x; p < n * Am * Rm; p += blockDim.x) {
    const int64_t e = e0 + p / (Am * Rm);
    if (!B.prev_dones[e]) continue;
    const int64_t row = e * Am * Rm + (p - (p / (Am * Rm)) * Am * Rm);
#pragma unroll
    for (int k = 0; k < 12; ++k) B.final_obs[(int64_t)k * B.obs_rows + row] = B.prev_final_obs[(int64_t)k * B.obs_rows + row];
  }
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

__device__ __forceinline__ void words_at(uint4 x, uint4 y, int off, uint32_t w[4]) {
  // 4 consecutive words starting at lane `off` of block x, continuing into y
  // (branch-free: a 2-word then a 1-word shift of the window)
  const bool s2 = off & 2, s1 = off & 1;
  const uint32_t a0 = s2 ? x.z : x.x, a1 = s2 ? x.w : x.y, a2 = s2 ? y.x : x.z, a3 = s2 ? y.y : x.w,
                 a4 = s2 ? y.z : y.x;
  w[0] = s1 ? a1 : a0;
  w[1] = s1 ? a2 : a1;
  w[2] = s1 ? a3 : a2;
  w[3] = s1 ? a4 : a3;
}

// pf::update with one measurement (tracking.cpp:119-143) -- the exact
// sequential path, out of line and working on this thread's particles staged in
// shared memory (px at st[k], py at st[P+k], w at cum[k]). Returns the reducer
// parity.
template <int PPT>
__device__ __noinline__ int pf_update_seq(const double* m, int k0, int P, const double* st, double* wts, double* red,
                                          int parity) {
  BlockReducer R{red, parity};
  const double ox = m[0], oy = m[1], r2 = m[2], sig = m[3];
  double ll[PPT];
  double mx = -CUDART_INF;
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const int k = k0 + j;
    if (k < P) {
      const double dx = st[k] - ox, dy = st[P + k] - oy;
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
      const int k = k0 + j;
      if (k < P) {
        wts[k] = wts[k] * exp(ll[j] - shift);
        acc = acc + wts[k];
      }
    }
    const double sum = R.sum(acc);
    if (isfinite(sum) && sum > 0.0) {
#pragma unroll
      for (int j = 0; j < PPT; ++j)
        if (k0 + j < P) wts[k0 + j] = wts[k0 + j] / sum;
      return R.parity;
    }
  }
  const double inv = 1.0 / (double)P;
#pragma unroll
  for (int j = 0; j < PPT; ++j)
    if (k0 + j < P) wts[k0 + j] = inv;
  return R.parity;
}

// pf::estimate (tracking.cpp:180-188) in ONE reduction: moments about the set's
// previous estimate (cx, cy), mean = c + sum w (p - c), spread^2 = second moment
// minus the squared shift; exact second pass when that subtraction could lose
// more than ~1e-11 relative. Returns (mean x, mean y, spread^2): the caller takes
// the square root in the one thread that writes the record.
template <int PPT, bool FULL, int NW>
__device__ __forceinline__ double3 pf_estimate(const SetRegs<PPT>& s, int k0, int P, double cx, double cy,
                                               BlockReducer& R, bool uniform = false, double inv_n = 0.0) {
  // -0.0 is the exact identity of IEEE addition, so the first term's add folds
  // away (0.0 + x is not an identity: x = -0.0)
  double a0 = -0.0, a1 = -0.0, a2 = -0.0;
  if (uniform) {  // weights all 1/n (just resampled): plain moments, scaled once
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (FULL || k0 + j < P) {
        const double dx = s.px[j] - cx, dy = s.py[j] - cy;
        a0 = a0 + dx;
        a1 = a1 + dy;
        a2 = fma(dx, dx, a2);
        a2 = fma(dy, dy, a2);
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (FULL || k0 + j < P) {
        const double dx = s.px[j] - cx, dy = s.py[j] - cy;
        a0 = a0 + s.w[j] * dx;
        a1 = a1 + s.w[j] * dy;
        a2 = a2 + s.w[j] * (dx * dx + dy * dy);
      }
    }
  }
  double3 m = R.sum3<NW>(a0, a1, a2);
  if (uniform) m.x = m.x * inv_n, m.y = m.y * inv_n, m.z = m.z * inv_n;
  const double mx = cx + m.x, my = cy + m.y;
  const double shift2 = m.x * m.x + m.y * m.y;
  const double var = m.z - shift2;
  // var > 0 here; far above 2^-960 for any spread a set can have
  if (var > 1e-5 * shift2) return make_double3(mx, my, var);
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    if (FULL || k0 + j < P) {
      const double dx = s.px[j] - mx, dy = s.py[j] - my;
      acc = acc + s.w[j] * (dx * dx + dy * dy);
    }
  }
  return make_double3(mx, my, R.sum<NW>(acc));  // >= 0: 0 or far above 2^-960
}

// Stage this thread's particles for the resample gather: particle k = k0 + q of
// thread t at q * NT + t, so each field's stores are lane-contiguous
// (conflict-free); positions and velocities as pairs, one 128-bit access each.
template <int PPT, bool FULL, int NW>
__device__ __forceinline__ void resample_stage(const SetRegs<PPT>& s, int k0, int P, const Smem& S) {
  const int tid = threadIdx.x;
  const int NT = NW > 0 ? NW * 32 : (int)blockDim.x;
  const int FS = NT * PPT;
  double2* st2 = reinterpret_cast<double2*>(S.st);  // [FS] (px, py), then [FS] (vx, vy)
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    if (FULL || k0 + q < P) {
      st2[q * NT + tid] = make_double2(s.px[q], s.py[q]);
      st2[FS + q * NT + tid] = make_double2(s.vx[q], s.vy[q]);
    }
  }
}

// Zero this thread's resample marks (S.cum as int[P]; before a barrier that
// precedes the marking, and after every thread's last read of the set buffer's
// w field, which the marks alias).
template <int PPT, bool FULL>
__device__ __forceinline__ void resample_zero_marks(int k0, int P, const Smem& S) {
  static_assert(PPT % 4 == 0, "mark zeroing takes whole int4s");
  int* mark = reinterpret_cast<int*>(S.cum);
  if (FULL || k0 < P) {
#pragma unroll
    for (int i = 0; i < PPT; i += 4) *reinterpret_cast<int4*>(mark + k0 + i) = make_int4(0, 0, 0, 0);
  }
}

// The selection half of pf::resample (tracking.cpp:147-170), once the marks are
// zeroed and the particles staged (both ordered by a barrier before the marks
// are set). Particle k = k0 + q has cumulative weight times n equal to
// loc[q] * scale + c0 - (1 - u0); output j takes the first particle whose
// cumulative weight reaches (j + u0)/n, clamped to n - 1 (the reference's
// monotone two-pointer walk).
// With count(c) = #{j : u_j <= c}, the outputs [count(cum[i-1]), count(cum[i]))
// are particle i's: particle k marks count(cum[k]) with k + 1 (the max wins
// where zero-weight particles share a boundary) and a prefix max over the marks
// (0 where unmarked) hands every output its source; outputs past
// count(cum[n-2]) fall to n - 1.
// count(c) = floor(c n - u0) + 1, clamped to [0, n]. It can differ from the
// count against the rounded u_j = (j + u0)/n only when c n - u0 lies within
// ~1e-13 of an integer; the block-tree cumulative weights already differ
// from the reference's sequential ones by ~1e-15 (x n = 1e-12), so exact
// boundary tests would not make a flip any less likely.
// As cum n + (1 - u0) >= 0, truncation gives the +1 and the clamp at 0 for
// free: count = min(n, trunc(loc scale + c0)).
template <int PPT, bool FULL, int NW>
__device__ void resample_select(SetRegs<PPT>& s, int k0, int P, const double (&loc)[PPT], double c0, double scale,
                                double inv_n, const Smem& S) {
  const int tid = threadIdx.x;
  int* mark = reinterpret_cast<int*>(S.cum);  // [P] source marks of the outputs
  const int NT = NW > 0 ? NW * 32 : (int)blockDim.x;
  const int FS = NT * PPT;
  const double2* st2 = reinterpret_cast<const double2*>(S.st);
  const int lane = tid & 31, warp = tid >> 5;
  int hq[PPT];  // count(cum[k]); P = no mark (the last particle, padding)
#pragma unroll
  for (int q = 0; q < PPT; ++q)
    hq[q] = k0 + q < P - 1 ? min(P, __double2int_rz(fma(loc[q], scale, c0))) : P;
  // Of a run of consecutive particles with the same count only the last one's
  // mark survives the max, so only it issues the atomic (lane 31's last always
  // does): the same marks with ~P spread atomics instead of P + conflicts.
  int nxt = __shfl_down_sync(0xffffffffu, hq[0], 1);
  if (lane == 31) nxt = -1;
  // Unconditional: a lane without a mark adds max(., 0) -- a no-op, marks are
  // >= 0 -- at its own lane-contiguous slot (no bank conflicts), so the warp
  // issues the reduction without a branch around it (ptxas does not predicate
  // ATOMS: a predicated red.shared becomes BSSY / BRA / BSYNC).
  const int NTm = NW > 0 ? NW * 32 : (int)blockDim.x;
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int hn = q + 1 < PPT ? hq[q + 1] : nxt;
    const bool p = hq[q] < P && hq[q] != hn;
    int* adr = p ? mark + min(hq[q], P - 1) : mark + ((q * NTm + tid) & (P - 1));
    atomicMax(adr, p ? k0 + q + 1 : 0);
  }
  ut_bar();
  int r[PPT];
#pragma unroll
  for (int i = 0; i < PPT; i += 4) {
    const int4 m4 = (FULL || k0 < P) ? *reinterpret_cast<const int4*>(mark + k0 + i) : make_int4(0, 0, 0, 0);
    r[i] = i == 0 ? m4.x : max(m4.x, r[i - 1]);
    r[i + 1] = max(m4.y, r[i]);
    r[i + 2] = max(m4.z, r[i + 1]);
    r[i + 3] = max(m4.w, r[i + 2]);
  }
  // Across lanes: the marks are increasing wherever they are set (counts grow
  // with the particle index), so the prefix max before a lane is the value of
  // the nearest lower lane holding a mark -- one ballot and one shuffle instead
  // of a five-level max scan.
  const int mi = r[PPT - 1];
  const unsigned nz = __ballot_sync(0xffffffffu, mi != 0);
  const unsigned below = nz & ((1u << lane) - 1u);
  const int src = below ? 31 - __clz(below) : lane;
  const int top = nz ? 31 - __clz(nz) : 0;
  int mex = __shfl_sync(0xffffffffu, mi, src);
  const int wtop = __shfl_sync(0xffffffffu, mi, top);
  if (!below) mex = -1;
  int* wmx = reinterpret_cast<int*>(S.red + 2 * kRedSlots + 96);
  st_shared_if(lane == 31, reinterpret_cast<uint32_t*>(wmx) + warp, (uint32_t)wtop);
  ut_bar();
  if constexpr (NW > 0 && NW % 4 == 0) {  // the warp maxima as int4 loads
#pragma unroll
    for (int v = 0; v < NW; v += 4) {
      const int4 m4 = *reinterpret_cast<const int4*>(wmx + v);
      if (v < warp) mex = max(mex, m4.x);
      if (v + 1 < warp) mex = max(mex, m4.y);
      if (v + 2 < warp) mex = max(mex, m4.z);
      if (v + 3 < warp) mex = max(mex, m4.w);
    }
  } else if constexpr (NW > 0) {
#pragma unroll
    for (int v = 0; v < NW - 1; ++v)
      if (v < warp) mex = max(mex, wmx[v]);
  } else {
    for (int v = 0; v < warp; ++v) mex = max(mex, wmx[v]);
  }
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    if (FULL || k0 + q < P) {
      const int i = max(mex, r[q]);
      const int j = (i & (PPT - 1)) * NT + i / PPT;
      const double2 p2 = st2[j], v2 = st2[FS + j];
      s.px[q] = p2.x, s.py[q] = p2.y;
      s.vx[q] = v2.x, s.vy[q] = v2.y;
      s.w[q] = inv_n;
    }
  }
  // the set buffer is next written by the prefetch after this set's estimate barrier
}

// pf::resample (tracking.cpp:147-170) on normalised weights: inclusive scan of
// w in index order (thread, warp, block), then the selection.
template <int PPT, bool FULL, int NW>
__device__ void pf_resample(SetRegs<PPT>& s, int k0, int P, double u0, double inv_n, const Smem& S) {
  const int tid = threadIdx.x;
  double* wsum = S.red + 2 * kRedSlots;  // [32] warp totals, then [32] int warp maxima at +96
  resample_stage<PPT, FULL, NW>(s, k0, P, S);
  double loc[PPT];
  double run = 0.0;
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    if (FULL || k0 + q < P) run = q == 0 ? s.w[q] : run + s.w[q];
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
  st_shared_if(lane == 31, wsum + warp, incl);
  resample_zero_marks<PPT, FULL>(k0, P, S);
  ut_bar();
  double woff = -0.0;  // cum[k] = (sum of earlier warps' totals + excl) + loc[q]; -0.0: see pf_estimate
  if constexpr (NW > 0) {
#pragma unroll
    for (int v = 0; v < NW - 1; ++v)
      if (v < warp) woff = woff + wsum[v];
  } else {
    for (int v = 0; v < warp; ++v) woff = woff + wsum[v];
  }
  const double base = woff + excl;
  resample_select<PPT, FULL, NW>(s, k0, P, loc, fma(base, (double)P, 1.0 - u0), (double)P, inv_n, S);
}

// One field of this thread's PPT consecutive particles to / from the set
// buffer (128-bit accesses; k0 is a multiple of PPT).
template <int PPT>
__device__ __forceinline__ void store_field(double* f, int k0, const double (&v)[PPT]) {
#pragma unroll
  for (int q = 0; q < PPT; q += 2) *reinterpret_cast<double2*>(f + k0 + q) = make_double2(v[q], v[q + 1]);
}
template <int PPT>
__device__ __forceinline__ void load_field(const double* f, int k0, double (&v)[PPT]) {
#pragma unroll
  for (int q = 0; q < PPT; q += 2) {
    const double2 t = *reinterpret_cast<const double2*>(f + k0 + q);
    v[q] = t.x, v[q + 1] = t.y;
  }
}

// One field of this thread's PPT particles to / from a parking area of pair
// chunks: particles (k0 + q, k0 + q + 1) at chunk (q / 2) NT + tid, so a warp's
// 128-bit accesses are contiguous (conflict-free).
template <int PPT>
__device__ __forceinline__ void park_field(double2* f, int nt, const double (&v)[PPT]) {
#pragma unroll
  for (int q = 0; q < PPT; q += 2) f[(q / 2) * nt + threadIdx.x] = make_double2(v[q], v[q + 1]);
}
template <int PPT>
__device__ __forceinline__ void unpark_field(const double2* f, int nt, double (&v)[PPT]) {
#pragma unroll
  for (int q = 0; q < PPT; q += 2) {
    const double2 t = f[(q / 2) * nt + threadIdx.x];
    v[q] = t.x, v[q + 1] = t.y;
  }
}

// Per-phase cycle profile of the particle-set loop (debug builds with
// -DUT_SET_PROFILE only; thread 0 of each CTA, read by ut_debug_set_profile).
constexpr int kSetProfSlots = 12;
#ifdef UT_SET_PROFILE
__shared__ long long g_sp_acc[kSetProfSlots + 1];
__device__ unsigned long long g_setprof[kSetProfSlots];
#define SETPROF(k)                                  \
  if (threadIdx.x == 0) {                           \
    const long long _n = clock64();                 \
    g_sp_acc[k] += _n - g_sp_acc[kSetProfSlots];    \
    g_sp_acc[kSetProfSlots] = _n;                   \
  }
#else
#define SETPROF(k)
#endif

// Issue the TMA prefetch of particle set g (5 fields x P doubles) into S.pf.
__device__ __forceinline__ void prefetch_set(const DevBatch& B, const Smem& S, int64_t g, int P) {
  UT_SHAKE(5);
  const uint32_t bytes = (uint32_t)(sizeof(double) * P);
  const size_t off = (size_t)g * P;
  fence_proxy_async();
  mbar_expect_tx_sa(S.mbar_sa, 5u * bytes);
  bulk_g2s_sa(S.pf_sa, B.px + off, bytes, S.mbar_sa);
  bulk_g2s_sa(S.pf_sa + bytes, B.py + off, bytes, S.mbar_sa);
  bulk_g2s_sa(S.pf_sa + 2 * bytes, B.vx + off, bytes, S.mbar_sa);
  bulk_g2s_sa(S.pf_sa + 3 * bytes, B.vy + off, bytes, S.mbar_sa);
  bulk_g2s_sa(S.pf_sa + 4 * bytes, B.w + off, bytes, S.mbar_sa);
}

// filter_step (env.cpp:349-363) + fused comm updates (env.cpp:385-392) +
// finalize (env.cpp:397-409) for set (a, t) of env e (global set index gset).
// FULL (P == blockDim * PPT, P % 4 == 0): the set arrives in S.pf by TMA
// (phase `tphase`), the Philox blocks are computed in registers and the next
// set `next` (>= 0) is prefetched into S.pf after this set's last barrier.
template <int PPT, bool FULL, int NW>
__device__ void step_set(const DevConfig& c, const DevBatch& B, const Smem& S, BlockReducer& R, int e, int gset,
                         int a, int t, uint32_t& tphase, int next) {
  const int P = c.P, tid = threadIdx.x, T = c.T;
  const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int ps = a * T + t;     // PF stream id / set within the env (env.cpp:130-133)
  const int ti = a * c.sT + t;  // track index in the record
  const int k0 = tid * PPT;
  const double* tk = S.trk + kTrkStride * ti;  // staged by stage_env
  // pos, the max speed, the particle base and the record are (re)derived where
  // used, so nothing long-lived occupies registers across the noise phase
  const uint64_t pos = (uint64_t)tk[TK_POS];
  const uint64_t key = (uint64_t)__double_as_longlong(tk[TK_KEY]);
  const int off = (int)(pos & 3);
  const bool noise = FULL || c.noise_on != 0;  // FULL instances run only with noise (host side)
  const uint64_t u0p = pos + (noise ? 4ull * (uint64_t)P : 0ull);  // resample draw follows predict

  // ---- particles into registers (FULL: after the noise is drawn, below, so the
  // Box-Muller pairs of all PPT particles can be interleaved)
  SetRegs<PPT> s;
  if (!FULL) {
    const size_t base = (size_t)gset * P;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const int k = k0 + j;
      s.px[j] = s.py[j] = s.vx[j] = s.vy[j] = s.w[j] = 0.0;
      if (k < P) {
        s.px[j] = B.px[base + k];
        s.py[j] = B.py[base + k];
        s.vx[j] = B.vx[base + k];
        s.vy[j] = B.vy[base + k];
        s.w[j] = B.w[base + k];
      }
    }
  }

  // ---- Philox words of fill_normals (tracking.cpp:24-37): particle k needs the
  // words at pos + s*P + k for segments s = 0..3. FULL: thread t computes the
  // NB = PPT/4 aligned blocks pos/4 + s*P/4 + NB*t + i of each segment; a
  // misaligned stream takes its remaining words from the next lane's first
  // block (shuffle). Lane 31 needs the block after its warp's range in each
  // segment: stage_bnd computed those (and the resample draw's blocks) for
  // every set of the env at once, spread over the whole CTA.
  constexpr int NB = PPT / 4 > 0 ? PPT / 4 : 1;
  uint4 blk[4][NB];
  const uint4* bnd = S.bnd + ps * bnd_per_set(nw);
  if (FULL && noise) {
    uint64_t bq[4 * NB];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int i = 0; i < NB; ++i)
        bq[q * NB + i] = (pos >> 2) + (uint64_t)q * (uint64_t)(P / 4) + (uint64_t)(NB * tid + i);
    uint4 bo[4 * NB];
    philox_n<4 * NB>(key, (uint64_t)ps, bq, bo);
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int i = 0; i < NB; ++i) blk[q][i] = bo[q * NB + i];
    if (warp == nw - 1 && lane == 3) {
      uint32_t w2[4];
      words_at(bnd[4 * nw], bnd[4 * nw + 1], off, w2);
      reinterpret_cast<uint32_t*>(S.bc)[0] = w2[0];
      reinterpret_cast<uint32_t*>(S.bc)[1] = w2[1];
    }
  } else if (tid == 0) {  // the resample draw, broadcast through smem
    const uint4 x = philox(key, (uint64_t)ps, u0p >> 2);
    const int o = (int)(u0p & 3);
    const uint4 y = o == 3 ? philox(key, (uint64_t)ps, (u0p >> 2) + 1) : x;
    uint32_t w2[4];
    words_at(x, y, o, w2);
    reinterpret_cast<uint32_t*>(S.bc)[0] = w2[0];
    reinterpret_cast<uint32_t*>(S.bc)[1] = w2[1];
  }
  // S.bc is read before the resample, after at least one block barrier; the
  // previous set's reads of it precede its estimate barrier.

  // ---- pf::predict (tracking.cpp:94-117): the normals first
  float zpx[PPT], zpy[PPT], zvx[PPT], zvy[PPT];  // out[k], out[P+k], out[2P+k], out[3P+k]
  if (noise) {
    uint32_t W[4][PPT];  // [segment][particle]
    if (FULL && (off == 0 || off == 2)) {
      // The stream positions of the particle sets stay even (4P per predict, 2
      // per resample, 8P at init), so the window starts at word 0 or 2 of the
      // thread's first block (block-uniform): no shuffles and no selects at 0,
      // two shuffles and a compile-time shift at 2.
      static_assert(PPT % 4 == 0, "the FULL path takes whole Philox blocks");
      if (off == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            W[q][4 * i] = blk[q][i].x, W[q][4 * i + 1] = blk[q][i].y;
            W[q][4 * i + 2] = blk[q][i].z, W[q][4 * i + 3] = blk[q][i].w;
          }
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t nx = __shfl_down_sync(0xffffffffu, blk[q][0].x, 1);
          uint32_t ny = __shfl_down_sync(0xffffffffu, blk[q][0].y, 1);
          if (lane == 31) {  // the block after the warp's range (stage_bnd)
            const uint4 xq = bnd[q * nw + warp];
            nx = xq.x, ny = xq.y;
          }
          uint32_t a[4 * NB + 2];
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            a[4 * i] = blk[q][i].x, a[4 * i + 1] = blk[q][i].y, a[4 * i + 2] = blk[q][i].z, a[4 * i + 3] = blk[q][i].w;
          }
          a[4 * NB] = nx, a[4 * NB + 1] = ny;
#pragma unroll
          for (int j = 0; j < PPT; ++j) W[q][j] = a[j + 2];
        }
      }
    } else if (FULL) {  // any other start word (an injected state): the general window
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        // this thread's window: its NB blocks, then the next lane's first block
        uint4 nb;
        nb.x = __shfl_down_sync(0xffffffffu, blk[q][0].x, 1);
        nb.y = __shfl_down_sync(0xffffffffu, blk[q][0].y, 1);
        nb.z = __shfl_down_sync(0xffffffffu, blk[q][0].z, 1);
        const uint4 xq = bnd[q * nw + warp];  // broadcast load, selected on lane 31
        if (off != 0 && lane == 31) nb = xq;
        uint32_t a[4 * NB + 3];
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          a[4 * i] = blk[q][i].x, a[4 * i + 1] = blk[q][i].y, a[4 * i + 2] = blk[q][i].z, a[4 * i + 3] = blk[q][i].w;
        }
        a[4 * NB] = nb.x, a[4 * NB + 1] = nb.y, a[4 * NB + 2] = nb.z;
        // word j of the window starting at `off` (branch-free: a 2-word, then a
        // 1-word shift)
        const bool s2 = off & 2, s1 = off & 1;
        uint32_t b[PPT + 1];
#pragma unroll
        for (int j = 0; j <= PPT; ++j) b[j] = s2 ? a[j + 2] : a[j];
#pragma unroll
        for (int j = 0; j < PPT; ++j) W[q][j] = s1 ? b[j + 1] : b[j];
      }
    } else {
#pragma unroll
      for (int j = 0; j < PPT; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          W[q][j] = k0 + j < P ? word_at(key, (uint64_t)ps, pos + (uint64_t)q * (uint64_t)P + (uint64_t)(k0 + j)) : 0u;
    }
    // pair k: u1 = word(pos+k), u2 = word(pos+2P+k); pair P+k: segments 1, 3
    uint32_t bad = 0;  // pairs with an uncertain rounding: exact fp64 libm path
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      bad |= box_muller_fast(W[0][j], W[2][j], S.tab_log, S.tab_sc, zpx[j], zvx[j]) ? 0u : 1u << (2 * j);
      bad |= box_muller_fast(W[1][j], W[3][j], S.tab_log, S.tab_sc, zpy[j], zvy[j]) ? 0u : 2u << (2 * j);
    }
    if (bad) {
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        if (bad & (1u << (2 * j))) {
          const float2 z = box_muller_slow(W[0][j], W[2][j]);
          zpx[j] = z.x, zvx[j] = z.y;
        }
        if (bad & (2u << (2 * j))) {
          const float2 z = box_muller_slow(W[1][j], W[3][j]);
          zpy[j] = z.x, zvy[j] = z.y;
        }
      }
    }
  }
  const int nm = S.mcount[ti];
  bool exact = nm > kMaxMerged || B.force_exact;
  // merged pass: w, vx, vy leave the registers during the likelihood stages
  // (the set buffer keeps them in this thread's own slots until the barrier
  // after which the staging may start)
  const bool merged = nm > 0 && !exact;
  const int NPf = (int)(S.cum - S.pf) / 4;  // field stride of the set buffer
  const int NT = NW > 0 ? NW * 32 : (int)blockDim.x;
  if (FULL) {
    SETPROF(0);
    mbar_wait_sa(S.mbar_sa, tphase);
    UT_SHAKE(6);
    SETPROF(1);
    tphase ^= 1u;
#pragma unroll
    for (int q = 0; q < PPT; q += 2) {
      const double2 x = *reinterpret_cast<const double2*>(S.pf + k0 + q);
      const double2 y = *reinterpret_cast<const double2*>(S.pf + P + k0 + q);
      const double2 u = *reinterpret_cast<const double2*>(S.pf + 2 * P + k0 + q);
      const double2 v = *reinterpret_cast<const double2*>(S.pf + 3 * P + k0 + q);
      s.px[q] = x.x, s.px[q + 1] = x.y, s.py[q] = y.x, s.py[q + 1] = y.y;
      s.vx[q] = u.x, s.vx[q + 1] = u.y, s.vy[q] = v.x, s.vy[q + 1] = v.y;
    }
    if (!merged) load_field<PPT>(S.pf + 4 * NPf, k0, s.w);
  }
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    if (FULL || k0 + j < P) {
      s.px[j] = s.px[j] + s.vx[j] * c.dt;
      s.py[j] = s.py[j] + s.vy[j] * c.dt;
      if (noise) {
        s.px[j] = s.px[j] + c.pn * (double)zpx[j];
        s.py[j] = s.py[j] + c.pn * (double)zpy[j];
        s.vx[j] = s.vx[j] + c.vn * (double)zvx[j];
        s.vy[j] = s.vy[j] + c.vn * (double)zvy[j];
      }
    }
  }
  const double ms = tk[TK_MAXSPEED];
  // No clamp when ms <= 0 (tracking.cpp:105). A speed^2 at or below lo < ms^2
  // (exactly: RN(ms^2) (1 - 2^-50) rounded stays below it) has RN(sqrt) <= ms,
  // so f = 1 and the particle is unchanged: warps with no particle above lo
  // skip the correctly rounded sqrt and division (about half of them: the fast
  // particles cluster after resampling). Otherwise branch-free per particle (sp
  // = 0 gives a quotient the select drops).
  // The test runs on the high words (for doubles >= 0 their order is the integer
  // order, and hi(v2) < hi(lo) implies v2 < lo; ties and NaN only send a warp
  // to the exact branch): integer compares, where an "any v2 > lo" over doubles
  // compiles to an fp64 max reduction with NaN fix-ups.
  const double lo = (ms * ms) * (1.0 - 0x1p-50);
  const int lo_hi = __double2hiint(lo);
  double v2[PPT];
  bool over = false;
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    v2[j] = s.vx[j] * s.vx[j] + s.vy[j] * s.vy[j];
    over |= __double2hiint(v2[j]) >= lo_hi;
  }
  if (ms > 0.0 && __any_sync(0xffffffffu, over)) {
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const double sp = sqrt_rn_clamp(v2[j]);
      const double qt = div_rn_clamp(ms, sp);
      const double f = sp > ms ? qt : 1.0;
      s.vx[j] = s.vx[j] * f;
      s.vy[j] = s.vy[j] * f;
    }
  }
  ph_mark(B, PH_FILTER);

  // ---- range updates: own ping, then fused senders (env.cpp:356-360, 385-392)
  SETPROF(2);
  const uint16_t* ml = S.mlist + ti * c.sA;
  bool have_ess = false, resampled = false, w_early = false;
  double ess = 0.0;
  if (merged) {
    park_field<PPT>(S.park, NT, s.vx);
    park_field<PPT>(S.park + NT * (PPT / 2), NT, s.vy);
    if (!FULL) store_field<PPT>(S.pf + 4 * NPf, k0, s.w);
  }
  if (nm > 0 && !exact) {
    // Merged pass. With L_i = sum_j ll_ij and s_j = max_i ll_ij, the sequential
    // reference computes e_i / sum(e) with e_i = w_i exp(L_i - sum_j s_j), up to
    // rounding, unless an intermediate product underflows. Every intermediate
    // product of particle i is >= e_i (each ll - s <= 0, each stage sum <= 1).
    // Particles with e_i < 2^-60 max(e) are invisible in every fp64 sum either
    // way; all others have products >= 2^-60 max(e) >= 2^-920 (normal) when
    // max(e) >= 2^-860, and no stage can degenerate. So under that check the
    // merged result equals the sequential one to rounding; otherwise (or with a
    // non-finite shift) the exact sequential path runs. The argument holds for
    // any UPPER BOUND s'_j >= s_j (e only shrinks, the guard stays
    // conservative), so the stage maxima are taken from the high words only.
    double L[PPT];
#pragma unroll
    for (int q = 0; q < PPT; ++q) L[q] = -0.0;  // sum_j tq_j^2 (-0.0: see pf_estimate)
    // per-stage warp maxima, [stage * kMbStride + warp]: the stride keeps the
    // stage lanes' 128-bit reads below on distinct banks
    float* mb = reinterpret_cast<float*>(R.buf());
    // Every measurement of the env has the same noise (c2 = -1/(2 sigma^2), one
    // config per env), so sum_j ll_ij = c2 sum_j tq_ij^2 with tq = d - r: one fma
    // per particle and stage, the product by c2 (and the shift) folded into the
    // exp's argument later -- the same log-likelihood to a few ulp.
    // The stage maximum s_j = c2 min_i tq_ij^2 comes from the smallest |tq|:
    // its high word (sign cleared; doubles >= 0 order like their bits) read back
    // with a zero low word is a lower bound lb_j of min |tq|, so c2 lb_j^2 is an
    // upper bound s'_j of s_j. One unsigned min per particle, one REDUX per stage.
    const double c2 = S.meas[kMeasStride * ml[0] + 4];
    auto stage = [&](int j) -> uint32_t {
      const double* m = S.meas + kMeasStride * ml[j];
      const double ox = m[0], oy = m[1], r2 = m[2];
      uint32_t mj = 0xFFFFFFFFu;
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        if (FULL || k0 + q < P) {
          const double dx = s.px[q] - ox, dy = s.py[q] - oy;
          const double d = sqrt_dist(fma(dx, dx, dy * dy));
          const double tq = d - r2;
          L[q] = fma(tq, tq, L[q]);
          mj = min(mj, (uint32_t)__double2hiint(tq) & 0x7FFFFFFFu);
        }
      }
      return mj;
    };
    auto stage_max = [&](int j, uint32_t mj) {
      mj = redux_min_u32(mj);
      st_shared_if(lane == 0, reinterpret_cast<uint32_t*>(mb) + j * kMbStride + warp, mj);
    };
    // two stages per iteration so their distance / sqrt chains interleave (the
    // warp reductions, whose divergence check fences the scheduler, follow both)
#pragma unroll 1
    for (int j = 0; j + 1 < nm; j += 2) {
      const uint32_t m0 = stage(j);
      const uint32_t m1 = stage(j + 1);
      stage_max(j, m0);
      stage_max(j + 1, m1);
    }
    if (nm & 1) stage_max(nm - 1, stage(nm - 1));
    if (merged) load_field<PPT>(S.pf + 4 * NPf, k0, s.w);
    SETPROF(3);
    ut_bar();
    double shift = 0.0;  // sum_j s'_j, in stage order
    const uint32_t* mbu = reinterpret_cast<const uint32_t*>(mb);
    // lane j < nm combines stage j's warp maxima once; the stage-order sum then
    // takes them lane by lane (the same operands in the same order)
    uint32_t hl = 0xFFFFFFFFu;
    if (lane < nm) {
      if constexpr (NW > 0 && NW % 4 == 0) {
#pragma unroll
        for (int v = 0; v < NW; v += 4) {
          const uint4 m4 = *reinterpret_cast<const uint4*>(mbu + lane * kMbStride + v);
          hl = min(hl, min(min(m4.x, m4.y), min(m4.z, m4.w)));
        }
      } else {
        for (int v = 0; v < nw; ++v) hl = min(hl, mbu[lane * kMbStride + v]);
      }
    }
    // the sum over lanes 0..7 (nm <= kMaxMerged = 8) by an xor butterfly (every
    // lane of the group ends with the same operands in the same pairing), then
    // lane 0's total to the warp
    {
      const double lb = __hiloint2double((int)hl, 0);
      double sj = lane < nm ? c2 * (lb * lb) : 0.0;  // >= max_i ll_ij
      sj = sj + __shfl_xor_sync(0xffffffffu, sj, 4);
      sj = sj + __shfl_xor_sync(0xffffffffu, sj, 2);
      sj = sj + __shfl_xor_sync(0xffffffffu, sj, 1);
      shift = __shfl_sync(0xffffffffu, sj, 0);
    }
    if (!isfinite(shift)) {
      exact = true;
      if (merged) {  // before the exact path's staging barrier
        unpark_field<PPT>(S.park, NT, s.vx);
        unpark_field<PPT>(S.park + NT * (PPT / 2), NT, s.vy);
      }
    } else {
      // e, its running sums (the resample scan's thread part) and squares; the
      // weight total then comes from the scan's warp totals, so the weight sums
      // and the resample's scan share one barrier
      double e[PPT], loc[PPT], run = -0.0, lq = -0.0;  // -0.0: see pf_estimate
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        e[q] = 0.0;
        if (FULL || k0 + q < P) {
          e[q] = s.w[q] * exp_neg(fma(L[q], c2, -shift), S.tab_exp);  // L = sum tq^2 here
          run = run + e[q];
          lq = lq + e[q] * e[q];
        }
        loc[q] = run;
      }
      if (merged) {
        unpark_field<PPT>(S.park, NT, s.vx);
        unpark_field<PPT>(S.park + NT * (PPT / 2), NT, s.vy);
      }
      SETPROF(4);
      double incl = run;  // the warp's inclusive scan of the thread totals
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl = incl + y;
      }
      // the thread's exclusive prefix as incl - run (no shuffle; it differs from
      // the previous lane's incl by rounding only, which the resample's marks
      // tolerate: counts only need to be consistent within a thread)
      const double excl = incl - run;
      lq = warp_sum(lq);
      const double* tw = R.buf();  // [0, 32) warp totals of e, [32, 64) of e^2
      st_shared_if(lane == 31, const_cast<double*>(tw) + warp, incl);
      st_shared_if(lane == 0, const_cast<double*>(tw) + 32 + warp, lq);
      // the marks alias the set buffer's w field, which every thread reloaded
      // before the stage barrier
      resample_zero_marks<PPT, FULL>(k0, P, S);
      ut_bar();
      // the warp totals once in registers: the block total (warp_partials_sum's
      // tree) and, for a resample, the earlier warps' share come from the same loads
      constexpr int NWT = NW >= 2 && (NW & (NW - 1)) == 0 ? NW : 1;
      double tv[NWT];
      double ls;
      if constexpr (NWT > 1) {
#pragma unroll
        for (int i = 0; i < NWT; i += 2) {
          const double2 t2 = *reinterpret_cast<const double2*>(tw + i);
          tv[i] = t2.x, tv[i + 1] = t2.y;
        }
        double v[NWT];
#pragma unroll
        for (int i = 0; i < NWT; ++i) v[i] = tv[i];
#pragma unroll
        for (int st = 1; st < NWT; st *= 2)
#pragma unroll
          for (int i = 0; i < NWT; i += 2 * st) v[i] = v[i] + v[i + st];
        ls = v[0];
      } else {
        ls = warp_partials_sum<NW>(tw);
      }
      const double lsq = warp_partials_sum<NW>(tw + 32);
      SETPROF(5);
      // the guards on max(e) from the sum: sum >= 2^-850 gives max >= sum / P >=
      // 2^-860 (P <= 1024), sum >= 2^-190 gives max >= 2^-200
      const bool guard_ok = isfinite(ls) && ls >= 0x1p-850;
      const bool ess_ok = ls >= 0x1p-190;
      if (guard_ok) {
        // ls in [2^-850, P] and ls^2, lsq >= 2^-400 where the ESS is formed:
        // the branch-free IEEE divisions apply
        const double rcp = div_rn_clamp(1.0, ls);
        // ESS = sum^2 / sum(e^2) < P / 2 unless the squares may have underflowed,
        // tested without the division: P / 2 is a power of two, so the product
        // is exact (the two forms differ only where sum^2 / sum(e^2) rounds up
        // onto P / 2, ~2^-53 relative)
        const bool low_ess = ess_ok && ls * ls < ((double)P / 2.0) * lsq;
        if (ess_ok) {
          ess = low_ess ? 0.0 : (double)P;  // only its side of P / 2 is used below
          have_ess = true;
        }
        if (low_ess) {
          // pf::maybe_resample's resample on the scan above: cum(k) n =
          // (woff + excl + loc) P / sum, the weights never normalised
          double woff = -0.0;
          if constexpr (NWT > 1) {
#pragma unroll
            for (int v = 0; v < NWT - 1; ++v)
              if (v < warp) woff = woff + tv[v];
          } else {
            for (int v = 0; v < warp; ++v) woff = woff + tw[v];
          }
          const uint64_t u0_lo = reinterpret_cast<const uint32_t*>(S.bc)[0];
          const uint64_t u0_hi = reinterpret_cast<const uint32_t*>(S.bc)[1];
          const double u0 = (double)(((u0_hi << 32) | u0_lo) >> 11) * 0x1.0p-53;
          const double scale = (double)P * rcp;
          if (FULL) {  // the resampled weights are all 1/n: stored now, draining under the gather
            const size_t wb = (size_t)gset * P;
#pragma unroll
            for (int q = 0; q < PPT; q += 4) st_global_v4(B.w + wb + k0 + q, c.inv_P, c.inv_P, c.inv_P, c.inv_P);
            w_early = true;
          }
          resample_stage<PPT, FULL, NW>(s, k0, P, S);
          resample_select<PPT, FULL, NW>(s, k0, P, loc, fma(woff + excl, scale, 1.0 - u0), scale, c.inv_P, S);
          SETPROF(7);
          resampled = true;
        } else {
#pragma unroll
          // (e / sum to ~1 ulp: the merged weights carry the rounding of the tree
          // sums and of exp anyway; the resample's strata see 1e-16 either way)
          for (int q = 0; q < PPT; ++q) s.w[q] = e[q] * rcp;
        }
      } else {
        exact = true;
      }
    }
  }
  if (exact && nm > 0) {
    if (tid == 0) S.bc[kBcStatExact] += 1.0;
    ut_bar();  // every thread holds its particles: S.pf becomes the staging area
#pragma unroll
    for (int q = 0; q < PPT; ++q)
      if (FULL || k0 + q < P) {
        S.st[k0 + q] = s.px[q];
        S.st[P + k0 + q] = s.py[q];
        S.cum[k0 + q] = s.w[q];
      }
    for (int j = 0; j < nm; ++j)
      R.parity = pf_update_seq<PPT>(S.meas + kMeasStride * ml[j], k0, P, S.st, S.cum, R.red, R.parity);
#pragma unroll
    for (int q = 0; q < PPT; ++q)
      if (FULL || k0 + q < P) s.w[q] = S.cum[k0 + q];
    ut_bar();  // the staging area is reused by the resample
  }
  const bool fresh = nm > 0;
  // the update pass: the own ping's share is filter_step, the senders' comms
  ph_mark_split(B, PH_FILTER, PH_COMMS, nm > 0 && ml[0] == ti ? 1 : 0, nm);

  // ---- pf::maybe_resample (tracking.cpp:172-178). With no update this step the
  // weights are the ones last step's maybe_resample already vetted (ESS >= P/2),
  // so the reference's recomputation cannot resample: skipped unless the state
  // was injected.
  SETPROF(6);
  const bool ess_known_ok = (nm == 0 && tk[TK_ESSOK] != 0.0) || resampled;
  if (!ess_known_ok) {
    if (!have_ess) {
      double w2 = 0.0;
#pragma unroll
      for (int q = 0; q < PPT; ++q) w2 = w2 + s.w[q] * s.w[q];
      ess = 1.0 / R.sum<NW>(w2);
    }
    if (ess < (double)P / 2.0) {
      const uint64_t u0_lo = reinterpret_cast<const uint32_t*>(S.bc)[0];
      const uint64_t u0_hi = reinterpret_cast<const uint32_t*>(S.bc)[1];
      const double u0 = (double)(((u0_hi << 32) | u0_lo) >> 11) * 0x1.0p-53;
      pf_resample<PPT, FULL, NW>(s, k0, P, u0, c.inv_P, S);
      SETPROF(7);
      resampled = true;
    }
  }

  if (!FULL && B.trace_env == (int64_t)e && tid == 0)  // trace: generic instance only
    printf("[trace env %lld set %d] nm=%d exact=%d have_ess=%d ess=%.17g resampled=%d pos=%llu\n",
           (long long)e, ps, nm, (int)exact, (int)have_ess, ess, (int)resampled,
           (unsigned long long)pos);  // at set start

  // ---- the set back to HBM (ahead of the estimate, which only reads the
  // registers: the store queue drains under the estimate's reduction)
  const size_t base = (size_t)gset * P;
  if (FULL) {
    // 256-bit stores (STG.E.ENL2.256): one per field and 4 particles
#pragma unroll
    for (int q = 0; q < PPT; q += 4) {
      // the fields the estimate does not read first: their registers, freed
      // first, are the ones the estimate's temporaries get
      st_global_v4(B.vx + base + k0 + q, s.vx[q], s.vx[q + 1], s.vx[q + 2], s.vx[q + 3]);
      st_global_v4(B.vy + base + k0 + q, s.vy[q], s.vy[q + 1], s.vy[q + 2], s.vy[q + 3]);
      // w: stored at the resample decision (w_early), or unchanged since the
      // load (no update and no resample this step)
      if (!w_early && !(nm == 0 && tk[TK_ESSOK] != 0.0))
        st_global_v4(B.w + base + k0 + q, s.w[q], s.w[q + 1], s.w[q + 2], s.w[q + 3]);
      // px, py: after the estimate, which reads them (see there)
    }
  } else {
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
  // ---- estimate (env.cpp:403-407)
  // The set buffer is free once every thread is past the estimate barrier: the
  // next set of this chunk is prefetched into it then (generic-proxy writes to
  // it are fenced against the async-proxy copy first).
  if (FULL) fence_proxy_async();
  SETPROF(8);
  const double3 est = pf_estimate<PPT, FULL, NW>(s, k0, P, tk[TK_EX], tk[TK_EY], R, resampled, c.inv_P);
  // the positions stored only now: they stay live for the estimate anyway, and
  // the estimate's temporaries no longer wait (WAR, long scoreboard) for 256-bit
  // stores still reading the registers they are given
  if (FULL) {
#pragma unroll
    for (int q = 0; q < PPT; q += 4) {
      st_global_v4(B.px + base + k0 + q, s.px[q], s.px[q + 1], s.px[q + 2], s.px[q + 3]);
      st_global_v4(B.py + base + k0 + q, s.py[q], s.py[q + 1], s.py[q + 2], s.py[q + 3]);
    }
  }
  SETPROF(9);
  if (FULL && tid == 0 && next >= 0) prefetch_set(B, S, next, P);
  if (tid == 0) {
    const Rec rec = rec_of(B, e);
    TRK(K_EX, ti) = est.x;
    TRK(K_EY, ti) = est.y;
    TRK(K_SPREAD, ti) = sqrt_rn_clamp(est.z);  // the spread^2 -> spread in the one thread writing it
    TRK(K_AGE, ti) = fresh ? 0.0 : tk[TK_AGE] + 1.0;
    TRK(K_EVER, ti) = (tk[TK_EVER] != 0.0 || fresh) ? 1.0 : 0.0;
    // stream position: 4P predict draws, 2 for a resample (tracking.cpp:24-37, 160)
    TRK(K_POS, ti) = tk[TK_POS] + (noise ? 4.0 * (double)P : 0.0) + (resampled ? 2.0 : 0.0);
    TRK(K_ESSOK, ti) = 1.0;  // maybe_resample ran: ESS >= P/2 or weights uniform
    S.bc[kBcStatUpdates] += (double)nm;
    S.bc[kBcStatResamples] += resampled ? 1.0 : 0.0;
  }
  ph_mark(B, PH_COMMS);  // maybe_resample + estimate (env.cpp:397-409)
  SETPROF(10);
}

// The warp-boundary Philox blocks of every set of the staged env (the FULL
// instance's noise, step_set): per set, for each segment q and warp w the block
// pos/4 + q P/4 + NB 32 (w + 1), then pos/4 + P and pos/4 + P + 1 (the resample
// draw at pos + 4P). Spread over the whole CTA as 4 interleaved chains per
// thread, once per env, instead of a fifth chain in every thread of every set.
// Needs the env's staged track scalars (S.trk); caller syncs before and after.
template <int PPT>
__device__ __noinline__ void stage_bnd(const DevConfig& c, const Smem& S) {
  constexpr int NB = PPT / 4 > 0 ? PPT / 4 : 1;
  const int nw = blockDim.x >> 5, per = bnd_per_set(nw), P = c.P;
  const int total = c.A * c.T * per;
  for (int i0 = threadIdx.x; i0 < total; i0 += 4 * blockDim.x) {
    uint32_t c0[4], c1[4], c2[4], c3[4], k0[4], k1[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int item = min(i0 + j * (int)blockDim.x, total - 1);
      const int ps = item / per, r = item - ps * per;
      const int a = ps / c.T, t = ps - a * c.T;
      const double* tk = S.trk + kTrkStride * (a * c.sT + t);
      const uint64_t pos = (uint64_t)tk[TK_POS];
      const uint64_t key = (uint64_t)__double_as_longlong(tk[TK_KEY]);
      const int q = r / nw, w = r - q * nw;
      const uint64_t blk = r < 4 * nw
                               ? (pos >> 2) + (uint64_t)q * (uint64_t)(P / 4) + (uint64_t)(NB * 32 * (w + 1))
                               : (pos >> 2) + (uint64_t)P + (uint64_t)(r - 4 * nw);
      c0[j] = (uint32_t)blk, c1[j] = (uint32_t)(blk >> 32);
      c2[j] = (uint32_t)ps, c3[j] = 0u;
      k0[j] = (uint32_t)key, k1[j] = (uint32_t)(key >> 32);
    }
    philox_keys<4>(c0, c1, c2, c3, k0, k1);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int item = i0 + j * (int)blockDim.x;
      if (item < total) S.bnd[item] = make_uint4(c0[j], c1[j], c2[j], c3[j]);
    }
  }
}

// L2 prefetch of the record words and ping schedule stage_env will read for env
// e (one address per thread), issued an env ahead so the staging's scattered
// loads (one 32-B sector per word of the structure-of-arrays record) hit L2.
__device__ __forceinline__ void prefetch_env(const DevBatch& B, int64_t e) {
  const DevConfig& c = cfg_of(B, e);
  const int A = c.A, T = c.T, i = threadIdx.x;
  const double* p = nullptr;
  if (i < A) {
    p = B.rec + (int64_t)(c.o_agent + V_X * c.sA + i) * B.n_envs + e;
  } else if (i < 2 * A) {
    p = B.rec + (int64_t)(c.o_agent + V_Y * c.sA + (i - A)) * B.n_envs + e;
  } else if (i < 2 * A + 7 * A * T) {
    const int j = i - 2 * A, f = j / (A * T), s = j - f * (A * T), a = s / T, t = s - a * T;
    // the staged fields K_POS, K_MAXSPEED, K_EX, K_EY, K_ESSOK, K_AGE, K_EVER as 4-bit codes
    constexpr uint32_t kF = K_POS | K_MAXSPEED << 4 | K_EX << 8 | K_EY << 12 | K_ESSOK << 16 | K_AGE << 20 |
                            K_EVER << 24;
    const int fld = (int)((kF >> (4 * f)) & 15u);
    p = B.rec + (int64_t)(c.o_track + fld * c.sA * c.sT + a * c.sT + t) * B.n_envs + e;
  } else if (i == 2 * A + 7 * A * T) {
    p = B.sched_r2 + e * (int64_t)(c.sA * c.sT);
  } else if (i == 2 * A + 7 * A * T + 1) {
    p = reinterpret_cast<const double*>(B.sched_flags + e * (int64_t)(c.sA * c.sT + c.sA * c.sA));
  }
  if (p) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Stage env e's config and ping schedule for the particle phase: measurement
// rows and the per-set update lists (own ping, then senders in ascending order).
// Caller syncs.
__device__ __forceinline__ void stage_env(const DevConfig& cg, const DevBatch& B, const Smem& S, const Rec& rec,
                                         int64_t e) {
  const DevConfig& c = cg;
  const int A = c.A, T = c.T, sA = c.sA, sT = c.sT;
  const double* r2 = B.sched_r2 + e * (int64_t)(sA * sT);
  const uint8_t* present = B.sched_flags + e * (int64_t)(sA * sT + sA * sA);
  const uint8_t* link = present + sA * sT;
  for (int i = threadIdx.x; i < (int)(sizeof(DevConfig) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(S.cfg)[i] = reinterpret_cast<const uint32_t*>(&cg)[i];
  if (threadIdx.x == 0) S.bc[kBcStatUpdates] = S.bc[kBcStatResamples] = S.bc[kBcStatExact] = 0.0;
  for (int i = threadIdx.x; i < A * T; i += blockDim.x) {
    const int a = i / T, t = i - (i / T) * T, ti = a * sT + t;
    double* m = S.meas + kMeasStride * ti;
    m[0] = AG(V_X, a);
    m[1] = AG(V_Y, a);
    m[2] = r2[ti];
    m[3] = c.sigma_meas;
    m[4] = -0.5 / (c.sigma_meas * c.sigma_meas);
    int n = 0;
    uint16_t* ml = S.mlist + ti * sA;
    if (present[ti]) ml[n++] = (uint16_t)ti;
    for (int s = 0; s < A; ++s)
      if (s != a && link[a * sA + s] && present[s * sT + t]) ml[n++] = (uint16_t)(s * sT + t);
    S.mcount[ti] = (uint16_t)n;
    double* tk = S.trk + kTrkStride * ti;
    tk[TK_POS] = TRK(K_POS, ti);
    tk[TK_MAXSPEED] = TRK(K_MAXSPEED, ti);
    tk[TK_EX] = TRK(K_EX, ti);
    tk[TK_EY] = TRK(K_EY, ti);
    tk[TK_ESSOK] = TRK(K_ESSOK, ti);
    tk[TK_AGE] = TRK(K_AGE, ti);
    tk[TK_EVER] = TRK(K_EVER, ti);
    tk[TK_KEY] = __longlong_as_double((long long)derive_key(B.seed, kTagPf, (uint64_t)(B.env_index_offset + e),
                                                            (uint64_t)(a * T + t)));
  }
}

// pf::reinit (tracking.cpp:76-92) of one particle from its 8 stream words:
// r = R sqrt(u0), a = 2 pi u1 -> position; s = vmax u2, d = 2 pi u3 -> velocity.
__device__ __forceinline__ void reinit_particle(const uint32_t* q, double cx, double cy, double radius, double vmax,
                                                const double2* tab_sc, double& px, double& py, double& vx,
                                                double& vy) {
  const double r = radius * sqrt_rn_clamp(uniform_from_words(q[0], q[1]));
  const double an = kTwoPi * uniform_from_words(q[2], q[3]);
  double sa, ca;
  sincos_table_d(an, tab_sc, sa, ca);
  px = cx + r * ca;
  py = cy + r * sa;
  const double sp = vmax * uniform_from_words(q[4], q[5]);
  const double d = kTwoPi * uniform_from_words(q[6], q[7]);
  double sd, cd;
  sincos_table_d(d, tab_sc, sd, cd);
  vx = sp * cd;
  vy = sp * sd;
}

// pf::reinit (tracking.cpp:76-92) + estimate for one set (spawn, env.cpp:214-220).
// FULL (P == NW * 32 * PPT): each thread's PPT consecutive particles draw their
// 8 PPT words straight from 2 PPT + 1 Philox blocks in registers (one spare
// block covers a stream position that is not a multiple of 4), the set goes to
// HBM with 256-bit stores and the estimate is one block reduction. Otherwise
// the words are staged through shared memory.
template <int PPT, bool FULL, int NW>
__device__ void reinit_set(const DevConfig& c, const DevBatch& B, const Smem& S, BlockReducer& R, const Rec& rec,
                           int64_t gi, int64_t gset, int a, int t, double cx, double cy, double vmax) {
  const int P = c.P, tid = threadIdx.x;
  const int ps = a * c.T + t, ti = a * c.sT + t;
  const int k0 = tid * PPT;
  const uint64_t pos = (uint64_t)TRK(K_POS, ti);
  const uint64_t key = derive_key(B.seed, kTagPf, (uint64_t)gi, (uint64_t)ps);
  const int off = (int)(pos & 3);
  const double radius = c.init_radius;
  SetRegs<PPT> s;
  if constexpr (FULL) {
    constexpr int NBK = 2 * PPT + 1;
    uint64_t bq[NBK];
    uint4 bo[NBK];
#pragma unroll
    for (int i = 0; i < NBK; ++i) bq[i] = (pos >> 2) + (uint64_t)(2 * k0 + i);
    philox_n<NBK>(key, (uint64_t)ps, bq, bo);
    uint32_t wv[4 * NBK];
#pragma unroll
    for (int i = 0; i < NBK; ++i) wv[4 * i] = bo[i].x, wv[4 * i + 1] = bo[i].y, wv[4 * i + 2] = bo[i].z, wv[4 * i + 3] = bo[i].w;
    // the window of words starting at `off` (branch-free 2-word, then 1-word shift)
    const bool s2 = off & 2, s1 = off & 1;
    uint32_t b[8 * PPT + 1];
#pragma unroll
    for (int j = 0; j <= 8 * PPT; ++j) b[j] = s2 ? wv[j + 2] : wv[j];
    uint32_t W[8 * PPT];
#pragma unroll
    for (int j = 0; j < 8 * PPT; ++j) W[j] = s1 ? b[j + 1] : b[j];
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      reinit_particle(W + 8 * j, cx, cy, radius, vmax, S.tab_sc, s.px[j], s.py[j], s.vx[j], s.vy[j]);
      s.w[j] = c.inv_P;
    }
  } else {
    uint32_t* words = reinterpret_cast<uint32_t*>(S.pf);  // the set buffer (no prefetch in flight here)
    ut_bar();  // that area may still be read by the previous set
    gen_words(words, key, (uint64_t)ps, pos, 8ull * (uint64_t)P);
    ut_bar();
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const int k = k0 + j;
      s.px[j] = s.py[j] = s.vx[j] = s.vy[j] = s.w[j] = 0.0;
      if (k < P) {
        reinit_particle(words + off + 8 * k, cx, cy, radius, vmax, S.tab_sc, s.px[j], s.py[j], s.vx[j], s.vy[j]);
        s.w[j] = c.inv_P;
      }
    }
  }
  // estimate (tracking.cpp:180-188) of the uniform-weight cloud about its centre
  const double3 est = pf_estimate<PPT, FULL, NW>(s, k0, P, cx, cy, R, true, c.inv_P);
  const size_t base = (size_t)gset * P;
  if constexpr (FULL) {
#pragma unroll
    for (int q = 0; q < PPT; q += 4) {
      // the fields the estimate does not read first: their registers, freed
      // first, are the ones the estimate's temporaries get
      st_global_v4(B.vx + base + k0 + q, s.vx[q], s.vx[q + 1], s.vx[q + 2], s.vx[q + 3]);
      st_global_v4(B.vy + base + k0 + q, s.vy[q], s.vy[q + 1], s.vy[q + 2], s.vy[q + 3]);
      st_global_v4(B.w + base + k0 + q, s.w[q], s.w[q + 1], s.w[q + 2], s.w[q + 3]);
      st_global_v4(B.px + base + k0 + q, s.px[q], s.px[q + 1], s.px[q + 2], s.px[q + 3]);
      st_global_v4(B.py + base + k0 + q, s.py[q], s.py[q + 1], s.py[q + 2], s.py[q + 3]);
    }
  } else {
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
  if (tid == 0) {
    TRK(K_EX, ti) = est.x;
    TRK(K_EY, ti) = est.y;
    TRK(K_SPREAD, ti) = sqrt_rn_clamp(est.z);  // the spread^2 -> spread in the one thread writing it
    TRK(K_AGE, ti) = 0.0;
    TRK(K_EVER, ti) = 0.0;
    TRK(K_POS, ti) = (double)(pos + 8ull * (uint64_t)P);
    TRK(K_MAXSPEED, ti) = vmax;
    TRK(K_ESSOK, ti) = 1.0;
  }
}

// Re-init every set of the chunk's envs flagged kChunkFlagSpawned (out of line:
// works on the global copy of the batch descriptor and the dynamic smem; the
// sincos table is in place).
// Inlined into each kernel: as an out-of-line function called from the step
// kernel (shared with the generic step instance) the particle registers of
// all but the first particle per thread came back wrong (every set, on the
// device; the same function called from the reset kernel was right, and
// inlining fixes it) -- kept inline until that is understood.
template <int PPT, int NP, int KTAG>
__device__ __forceinline__ void reinit_chunk(const DevBatch& B, int64_t e0, int64_t e1) {
  const Smem S = carve_dyn<NP>(B.cfgs[0].sA, B.cfgs[0].sT);
  BlockReducer R{S.red, 0};
  constexpr int NW = NP / (32 * PPT);
  const bool full = B.P == NP && (int)blockDim.x == NW * 32;
  for (int64_t e = e0; e < e1; ++e) {
    if (!(S.flags[e - e0] & kChunkFlagSpawned)) continue;
    const DevConfig& c = cfg_of(B, e);
    const Rec rec = rec_of(B, e);
    const int64_t gi = B.env_index_offset + e;
    const double vmax = c.speed_margin * rec[R_EP_SPEED];
    const int64_t so = set_off(B, e);
    for (int a = 0; a < c.A; ++a) {
      const double cx = AG(V_X, a), cy = AG(V_Y, a);
      for (int t = 0; t < c.T; ++t) {
        if (full)
          reinit_set<PPT, true, NW>(c, B, S, R, rec, gi, so + a * c.T + t, a, t, cx, cy, vmax);
        else
          reinit_set<PPT, false, 0>(c, B, S, R, rec, gi, so + a * c.T + t, a, t, cx, cy, vmax);
      }
    }
  }
  ut_bar();
}

// ================================================================ kernels ===
#ifndef UT_STEP_MIN_BLOCKS
#define UT_STEP_MIN_BLOCKS 2
#endif

// The fused step.
template <int PPT, int NP, bool FULL>
__global__ void __launch_bounds__(1024 / PPT, UT_STEP_MIN_BLOCKS) step_kernel(DevBatch B, int mode, int32_t* status) {
  // external actions: nothing moves unless every action passed validate_kernel
  // (launched just before on the same stream; vecenv.cpp:88-93 validates all first)
  if (mode == MODE_EXTERNAL && *B.error_env != INT_MAX) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Smem S = carve<NP>(smem_raw, B.cfgs[0].sA, B.cfgs[0].sT);
  const DevBatch& Bg = *B.self;  // cold paths read the global copy
  BlockReducer R{S.red, 0};
  load_tables(S);
  if (FULL && threadIdx.x == 0) mbar_init(S.mbar, 1);
  // env and set indices fit in 32 bits (checked at creation)
  int lo, hi;
  {
    int64_t lo64, hi64;
    cta_range(B.n_envs, lo64, hi64);
    lo = (int)lo64, hi = (int)hi64;
  }
  ut_bar();
  uint32_t tphase = 0;
#ifdef UT_SET_PROFILE
  if (threadIdx.x == 0)
    for (int k = 0; k <= kSetProfSlots; ++k) g_sp_acc[k] = k == kSetProfSlots ? clock64() : 0;
#endif
  // phase timing (thread 0, shared memory: nothing live in registers)
  const bool timing = B.phase_cycles != nullptr;
  if (timing && threadIdx.x == 0) {
    long long* g_ph = ph_slots();
    for (int k = 0; k <= kPhaseWait; ++k) g_ph[k] = 0;
    g_ph[kPhLast] = g_ph[kPhLast + 1] = clock64();
    g_ph[kPhLast + 2] = (long long)globaltimer_ns();
  }
  // Three phases separated by grid-wide barriers (cooperative launch: every CTA
  // is resident): the env prologues of the CTA's static env range; the particle
  // filters, envs handed out one at a time by a global counter so the grid
  // finishes together (a static split left the slowest CTA 5 % behind the
  // mean); then outputs and auto-resets of the static range.
  cg::grid_group grid = cg::this_grid();
  const int n = (int)B.n_envs;
  // ---- 1. prologue, one env per thread
  for (int e0 = lo; e0 < hi; e0 += blockDim.x) {
    const int e = e0 + threadIdx.x;
    if (e < min(hi, e0 + (int)blockDim.x)) env_prologue(cfg_of(Bg, e), Bg, e, B.env_index_offset + e, mode);
  }
  UT_SHAKE(1);
  grid.sync();  // every env's ping schedule is in place
  UT_SHAKE(2);
  ph_mark(B, kPhaseWait);
  // ---- 2. particle sets, env by env from the work counter; the next env is
  // claimed at the start of the current one so its first set can be prefetched
  // The claims alternate between two slots: a slot is rewritten two claims
  // later, after barriers every thread has passed since reading it (thread 0
  // writes the next claim right after stage_env, which has no barrier, so one
  // slot would let it overwrite a claim a late warp has not read yet).
  int* claim = reinterpret_cast<int*>(S.bc + kBcClaim);
  int slot = 0;
  if (threadIdx.x == 0) {
    const int e = atomicAdd(B.work, 1);
    claim[0] = e;
    if (FULL && e < n) prefetch_set(B, S, set_off(B, e), B.P);
  }
  ut_bar();
  int e = claim[0];
  while (e < n) {
    // the next claim goes out first: its round trip overlaps the staging loads
    int nxt = 0;
    if (threadIdx.x == 0) nxt = atomicAdd(B.work, 1);
    stage_env(cfg_of(B, e), B, S, rec_of(B, e), e);
    slot ^= 1;
    if (threadIdx.x == 0) claim[slot] = nxt;
    ut_bar();
    const int en = claim[slot];
    const DevConfig& c = *S.cfg;
    if (en < n) prefetch_env(B, en);  // its staging loads hit L2 when its turn comes
    if (FULL) {
      stage_bnd<PPT>(c, S);
      ut_bar();
    }
    const int so = (int)set_off(B, e);
    const int nA = c.A, nT = c.T;
    const int first_next = en < n ? (int)set_off(B, en) : -1;
    for (int a = 0; a < nA; ++a)
      for (int t = 0; t < nT; ++t) {
        const int g = so + a * nT + t;
        const int last = a == nA - 1 && t == nT - 1;
        step_set<PPT, FULL, FULL ? NP / (32 * PPT) : 0>(c, B, S, R, e, g, a, t, tphase, last ? first_next : g + 1);
      }
    ut_bar();  // S.cfg / meas / mlist / claim reused by the next env
    if (threadIdx.x == 0) {  // the env's filter statistics, accumulated in smem per set
      // fire-and-forget reductions (this CTA is the env's only writer): warp 0
      // goes on to the next env's staging without waiting for the loads of +=
      const DevConfig& cg = cfg_of(B, e);
      double* st = B.rec + e + (int64_t)cg.o_stats * B.n_envs;
      atomicAdd(st + 7 * B.n_envs, S.bc[kBcStatUpdates]);
      atomicAdd(st + 8 * B.n_envs, S.bc[kBcStatResamples]);
      atomicAdd(st + 9 * B.n_envs, S.bc[kBcStatExact]);
    }
    e = en;
  }
  ph_mark(B, PH_FILTER);
  UT_SHAKE(3);
  grid.sync();  // every estimate is in place
  UT_SHAKE(4);
  ph_mark(B, kPhaseWait);
  if (blockIdx.x == 0 && threadIdx.x == 0) *B.work = 0;  // for the next launch
  for (int e0 = lo; e0 < hi; e0 += blockDim.x) {
    const int e1 = min(hi, e0 + (int)blockDim.x);
    // ---- 3. reward / done / info, one env per thread; then tokens
    if (B.prev_final_obs) copy_final_rows(Bg, e0, e1);  // ordered before this step's by the barrier below
    {
      const int e = e0 + threadIdx.x;
      if (e < e1) S.flags[threadIdx.x] = env_epilogue(cfg_of(Bg, e), Bg, e) ? kChunkFlagDone : 0;
    }
    ut_bar();
    ph_mark(B, PH_REWARD);
    write_outputs(Bg, e0, e1, S.flags, 0, false);
    // terminal obs of finished envs (VecEnv auto-reset only)
    if (B.auto_reset) write_outputs(Bg, e0, e1, S.flags, kChunkFlagDone, true);
    ph_mark(B, PH_OBSERVE);
    // ---- 4. auto-reset of finished envs (vecenv.cpp:106-112)
    bool any = false;
    for (int i = 0; i < (int)(e1 - e0); ++i) any |= (S.flags[i] & kChunkFlagDone) != 0;
    if (any && B.auto_reset) {
      ut_bar();
      const int e = e0 + threadIdx.x;
      if (e < e1 && (S.flags[threadIdx.x] & kChunkFlagDone)) {
        if (spawn_serial(cfg_of(Bg, e), Bg, e, B.env_index_offset + e))
          S.flags[threadIdx.x] |= kChunkFlagSpawned;
        else
          atomicMax(status, (int)ST_SPAWN_INFEASIBLE);
      }
      ut_bar();
      reinit_chunk<PPT, NP, 1>(Bg, e0, e1);
      write_outputs(Bg, e0, e1, S.flags, kChunkFlagSpawned, false);
      if (e < e1 && (S.flags[threadIdx.x] & kChunkFlagSpawned)) B.step[e] = 0;
    }
    ut_bar();
    ph_mark(B, PH_RESET);
  }
  if (timing && threadIdx.x == 0) {
    const long long* g_ph = ph_slots();
    unsigned long long* out = B.phase_cycles + (size_t)blockIdx.x * kPhaseSlots;
    for (int k = 0; k <= kPhaseWait; ++k) out[k] += (unsigned long long)g_ph[k];
    out[kPhaseWait + 1] += (unsigned long long)(clock64() - g_ph[kPhLast + 1]);
    out[kPhaseWait + 2] += globaltimer_ns() - (unsigned long long)g_ph[kPhLast + 2];
  }
#ifdef UT_SET_PROFILE
  if (threadIdx.x == 0)
    for (int k = 0; k < kSetProfSlots; ++k) atomicAdd(&g_setprof[k], (unsigned long long)g_sp_acc[k]);
#endif
}

// Environment ctor / reset (env.cpp:110-151, 153-233) for every env. When
// `ctor` is set the record starts zeroed and each set's stream is advanced past
// pf::init's 8P draws (tracking.cpp:43-67), whose values spawn overwrites.
template <int PPT, int NP>
__global__ void __launch_bounds__(1024 / PPT, UT_STEP_MIN_BLOCKS) reset_kernel(DevBatch B, int ctor, int32_t* status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Smem S = carve<NP>(smem_raw, B.cfgs[0].sA, B.cfgs[0].sT);
  const DevBatch& Bg = *B.self;
  load_tables(S);  // the re-init's sincos table
  int64_t lo, hi;
  cta_range(B.n_envs, lo, hi);
  for (int64_t e0 = lo; e0 < hi; e0 += blockDim.x) {
    const int64_t e1 = min(hi, e0 + (int64_t)blockDim.x);
    const int64_t e = e0 + threadIdx.x;
    if (e < e1) {
      const DevConfig& c = cfg_of(B, e);
      const Rec rec = rec_of(B, e);
      if (ctor) {
        for (int w = 0; w < c.rec_words; ++w) rec[w] = 0.0;
        for (int a = 0; a < c.A; ++a)
          for (int t = 0; t < c.T; ++t) {
            TRK(K_POS, a * c.sT + t) = 8.0 * (double)c.P;
            TRK(K_MAXSPEED, a * c.sT + t) = 1.0;
          }
        for (int a = 0; a < c.A; ++a) AG(V_RUDDER, a) = 2.0;
        for (int t = 0; t < c.T; ++t) TG(V_RUDDER, t) = 2.0;
      }
      S.flags[threadIdx.x] = 0;
      if (spawn_serial(cfg_of(Bg, e), Bg, e, B.env_index_offset + e))
        S.flags[threadIdx.x] = kChunkFlagSpawned;
      else
        atomicMax(status, (int)ST_SPAWN_INFEASIBLE);
      B.rewards[e] = 0.0;
      B.dones[e] = 0;
      B.step[e] = 0;
    }
    ut_bar();
    reinit_chunk<PPT, NP, 0>(Bg, e0, e1);
    write_outputs(Bg, e0, e1, S.flags, 0, false);
    ut_bar();
  }
}

// VecEnv::refresh_outputs (vecenv.cpp:145-150): one thread per row.
__global__ void tokens_kernel(DevBatch B) {
  const int Am = B.A_max, Rm = B.R_max;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < B.n_envs * Am * Rm; p += stride) {
    const int64_t e = p / (Am * Rm);
    const int q = (int)(p - e * Am * Rm), a = q / Rm, r = q - (q / Rm) * Rm;
    double v[12];
    token_row(cfg_of(B, e), rec_of(B, e), a, r, v);
    const int64_t row = (e * Am + a) * Rm + r;
#pragma unroll
    for (int k = 0; k < 12; ++k) B.obs[(int64_t)k * B.obs_rows + row] = v[k];
  }
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < B.n_envs * Rm; p += stride) {
    const int64_t e = p / Rm;
    const int r = (int)(p - e * Rm);
    double v[12];
    global_row(cfg_of(B, e), rec_of(B, e), r, v);
    const int64_t row = e * Rm + r;
#pragma unroll
    for (int k = 0; k < 12; ++k) B.global[(int64_t)k * B.global_rows + row] = v[k];
  }
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < B.n_envs * Am * 5; p += stride) {
    const int64_t e = p / (Am * 5);
    const int q = (int)(p - e * Am * 5), a = q / 5, k = q - (q / 5) * 5;
    const DevConfig& c = cfg_of(B, e);
    const Rec rec = rec_of(B, e);
    B.masks[e * Am * 5 + q] = (a < c.A && abs(k - (int)AG(V_RUDDER, a)) <= 1) ? 1 : 0;
  }
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < B.n_envs; e += stride) {
    const Rec rec = rec_of(B, e);
    B.step[e] = (int32_t)rec[R_STEP];
  }
}

// Action validation for VecEnv::step (env.cpp:236-248) before anything moves.
__global__ void validate_kernel(DevBatch B) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= B.n_envs) return;
  const DevConfig& c = cfg_of(B, e);
  const Rec rec = rec_of(B, e);
  for (int a = 0; a < c.A; ++a) {
    const int act = B.actions[e * B.A_max + a];
    const int rud = (int)AG(V_RUDDER, a);
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
  const int o_stats = B.cfgs[0].o_stats;
  for (int k = 0; k < kStatCount; ++k) {
    double acc = 0.0;
    double* st = B.rec + (int64_t)(o_stats + k) * B.n_envs;
    for (int64_t e = threadIdx.x; e < B.n_envs; e += blockDim.x) {
      acc = acc + st[e];
      if (reset) st[e] = 0.0;
    }
    const double s = R.sum(acc);
    if (threadIdx.x == 0) out[k] = s;
  }
}

#undef AG
#undef TG
#undef INFO
#undef TRK
#undef STAT

}  // namespace ut
