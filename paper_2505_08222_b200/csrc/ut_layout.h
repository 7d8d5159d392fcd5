// ut_layout.h -- device state-store layout shared by host and device code.
//
// HBM holds three things:
//  1. the particle store, structure-of-arrays: px/py/vx/vy/w each [set][P] fp64,
//     set = set_offset[env] + agent * T + target -- one 8 KB contiguous chunk per
//     set and field at P = 1024 (ParticleSet, tracking.hpp:39-55);
//  2. every other piece of Environment state (env.hpp:44-51, 131-171) as one
//     fp64 array per scalar field, structure-of-arrays ACROSS envs: word w of
//     env e lives at rec[w * n_envs + e], so when thread i of a CTA runs the
//     serial per-env phases of env (base + i) every field access is coalesced.
//     Integer fields are stored as exact fp64 values, like the reference's own
//     state blob (env.cpp:550-593). Field words are laid out for the batch's
//     largest fleet (sA x sT) so mixed fleets share one index space;
//  3. per-step scratch: the ping schedule the prologue hands to the particle
//     phase (horizontal ranges, ping-present and comm-link flags);
//  4. the batch output buffers of VecEnv (vecenv.hpp:51-62), column-major.
#pragma once
#include <stdint.h>

namespace ut {

// record scalar slots
enum : int {
  R_STEP = 0,
  R_EP_SPEED = 1,
  R_ENV_POS = 2,
  R_ENV_HAVE_SPARE = 3,
  R_ENV_SPARE = 4,
  R_BENCH_POS = 5,
  R_EP_RETURN = 6,
  R_LAST_DONE = 7,
  // evaluation accumulators of the running episode (curriculum.cpp:286-325):
  // sum over steps of sum_{a,t} |agent - target|, of sum_t tracking error, and
  // collided | lost<<1 -- not part of the state blob
  R_EV_DIST = 8,
  R_EV_ERR = 9,
  R_EV_FLAGS = 10,
  R_NSCALAR = 11
};
// vehicle fields (agents: first 6; targets: all 8)
enum : int { V_X = 0, V_Y, V_Z, V_HEAD, V_SPEED, V_RUDDER, V_COUNTDOWN, V_CMD };
// AgentInfo fields (env.hpp:19-25)
enum : int { I_X = 0, I_Y, I_Z, I_HEAD, I_AGE, I_VALID, I_NFIELD };
// track fields: TrackEstimate + ever_measured + PF RngStream::State + max_speed
enum : int { K_EX = 0, K_EY, K_SPREAD, K_AGE, K_EVER, K_POS, K_HAVE_SPARE, K_SPARE, K_MAXSPEED,
             K_ESSOK,  // not serialized: 1 when maybe_resample already vetted these weights
             K_NFIELD };
constexpr int K_NBLOB = 9;  // track fields carried by the state blob (env.cpp:578-583)

constexpr int kStatCount = 16;  // ut_env.h UT_N_STATS

// Resolved configuration for one fleet shape (EnvConfig after finalize()).
struct DevConfig {
  int A, T, R, P;
  int horizon, reward_mode, lost_steps, noise_on;
  double dt, agent_speed, tgt_lo, tgt_hi, turn_interval;
  double det_range, comm_range, drop, range_noise, sigma_meas;
  double eps_min, eps_max, d_min, d_safe;
  double min_sep, disc_r, pert_std, depth_min, depth_max;
  double pn, vn, speed_margin, init_radius;
  double inv_P;  // RN(1 / P), the weight after a resample (tracking.cpp:149, 168)
  double head_a, head_b, head_noise, max_turn;
  // record layout (field-word offsets) for the batch strides sA >= A, sT >= T:
  // agent field f of agent a: o_agent + f sA + a; target: o_target + f sT + t;
  // AgentInfo f of (r, s): o_info + f sA^2 + r sA + s; track f of (a, t):
  // o_track + f sA sT + a sT + t.
  int sA, sT;
  int o_agent, o_target, o_miss, o_info, o_track, o_stats, rec_words, _pad;
};

__host__ __device__ inline void layout_config(DevConfig& c, int sA, int sT) {
  c.R = c.A + c.T;
  c.sA = sA;
  c.sT = sT;
  c.o_agent = R_NSCALAR;
  c.o_target = c.o_agent + 6 * sA;
  c.o_miss = c.o_target + 8 * sT;
  c.o_info = c.o_miss + sT;
  c.o_track = c.o_info + I_NFIELD * sA * sA;
  c.o_stats = c.o_track + K_NFIELD * sA * sT;
  c.rec_words = c.o_stats + kStatCount;
}

// Per-batch constant tables (device pointers) passed to every kernel.
struct DevBatch {
  int64_t n_envs;
  int64_t env_index_offset;  // global index of env 0 (RNG key)
  uint64_t seed;
  int n_cfg;
  int A_max, T_max, R_max, P;
  const DevConfig* cfgs;      // [n_cfg]
  const int32_t* cfg_of_env;  // [n_envs] or nullptr (homogeneous)
  const int64_t* set_offset;  // [n_envs] sets, or nullptr: env * A * T
  double* rec;                // [rec_words][n_envs]
  double* sched_r2;           // [n_envs][sA * sT] horizontal ranges this step
  uint8_t* sched_flags;       // [n_envs][sA * sT + sA * sA] ping present | link
  double *px, *py, *vx, *vy, *w;
  int* work;  // the step kernel's env counter for the filter phase (0 between launches)
  // batch outputs
  int64_t obs_rows, global_rows;
  double* obs;
  double* final_obs;
  // double-buffered outputs (ut_vecenv_set_output_buffers(2)): the other set's
  // final_obs / dones, whose rows of the envs that finished at the previous step
  // the step copies into this set (null when single-buffered)
  const double* prev_final_obs;
  const uint8_t* prev_dones;
  double* global;
  double* rewards;
  uint8_t* dones;
  uint8_t* masks;
  double* track_err;
  double* min_dist;
  uint8_t* lost;
  uint8_t* collision;
  int32_t* step;
  const int32_t* actions;
  int32_t* error_env;  // validation: lowest failing env (INT32_MAX if none)
  int32_t* error_info; // [3] agent, action, rudder of that env
  // verification knobs (ut_debug.h): always take the exact sequential update
  // path; printf a per-set trace for one env (-1 = off)
  int32_t force_exact;
  int64_t trace_env;
  // Phase timing (PhaseTimer, env.cpp:18-36): SM cycles per CTA accumulated in
  // [grid][kPhaseSlots] when non-null (kPhaseCount phases, the grid-barrier
  // waits, then the CTA's elapsed SM cycles and globaltimer ns, which convert
  // cycles to ns).
  unsigned long long* phase_cycles;
  // VecEnv auto-reset of finished envs (vecenv.cpp:106-112); 0 = the single
  // Environment semantics (env.cpp:234-504: step never resets, done stays set)
  int32_t auto_reset;
  // Trajectory capture (append_trajectory_rows, trajectory.cpp:13-66) for envs
  // [traj_lo, traj_hi): after every step, before auto-reset, env e writes R_max
  // rows of kTrajFields doubles at traj[((e - traj_lo) * R_max + row) * kTrajFields].
  double* traj;
  int64_t traj_lo, traj_hi;
  // Device copy of this struct, for the out-of-line (cold) device functions, so
  // the kernel's by-value parameter is never address-taken.
  const struct DevBatch* self;
};

// Trajectory row fields (TrajectoryRow, trajectory.hpp:13-21): step, x, y, z,
// heading, has_estimate, est_x, est_y, track_err, reward, collision, is_target.
enum : int { TJ_STEP = 0, TJ_X, TJ_Y, TJ_Z, TJ_HEAD, TJ_HAS_EST, TJ_EST_X, TJ_EST_Y, TJ_ERR, TJ_REWARD,
             TJ_COLLISION, TJ_IS_TARGET, kTrajFields };

// Device phases: the reference's seven StepPhase values (env.hpp:71-80,
// env.cpp:250-279) plus the auto-reset the reference leaves untimed
// (vecenv.cpp:140). The merged range-update pass of a set is split between
// FILTER (its own ping) and COMMS (the fused senders' pings) in proportion.
enum : int { PH_TARGETS = 0, PH_AGENTS, PH_MEASURE, PH_FILTER, PH_COMMS, PH_OBSERVE, PH_REWARD, PH_RESET,
             kPhaseCount };
// per-CTA slots of B.phase_cycles: the phases, the grid-barrier waits, then the
// launch's elapsed SM cycles and globaltimer ns
constexpr int kPhaseWait = kPhaseCount;
constexpr int kPhaseSlots = kPhaseCount + 3;

}  // namespace ut
