/* ut_env.h -- C-ABI drop-in boundary for the batched JaxLrauv environment step
 * (arXiv 2505.08222) on B200 (sm_100a).
 *
 * Every entry point replaces one reference interface of the CPU library `utrack`
 * (paths relative to /root/reference/proj/core). Plain C types only: no torch, no
 * Eigen, no C++ exceptions cross this boundary. Status codes follow the reference's
 * exception -> CLI exit-code mapping (tools/utrack.cpp:384-393):
 *   ContractViolation -> 1, ConfigError -> 2, DataError -> 3 (errors.hpp:10-26);
 * 4 is added for CUDA/runtime failures. The message of the last failure on the
 * calling thread is available from ut_last_error().
 *
 * Threading/ownership (vecenv.hpp:18-23): a ut_vecenv is not reentrant; it owns
 * every device buffer; pointers returned by ut_vecenv_buffers() stay valid until
 * ut_vecenv_destroy(). Calls are synchronous: results are readable on return.
 */
#ifndef UT_ENV_H_
#define UT_ENV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UT_ABI_VERSION 4

enum ut_status {
  UT_OK = 0,
  UT_ERR_CONTRACT = 1, /* ContractViolation (errors.hpp:23-26) */
  UT_ERR_CONFIG = 2,   /* ConfigError (errors.hpp:10-14) */
  UT_ERR_DATA = 3,     /* DataError (errors.hpp:17-21) */
  UT_ERR_RUNTIME = 4   /* CUDA / allocation failure (no reference counterpart) */
};

enum { UT_NUM_ACTIONS = 5, UT_FEATURE_DIM = 12 }; /* env_config.hpp:8, :13 */
enum { UT_REWARD_TRACKING = 0, UT_REWARD_FOLLOW = 1 }; /* env_config.hpp:34 */
enum { UT_POLICY_RANDOM = 0, UT_POLICY_SCRIPTED = 1 }; /* vecenv.hpp:16 */
enum { UT_HEADING_DEFAULT = 0, UT_HEADING_BUCKET = 1 };

/* PfConfig (env_config.hpp:36-42). */
typedef struct ut_pf_config {
  int32_t n_particles;       /* 1024 */
  int32_t _pad0;
  double process_noise_pos;  /* 1.0 m per step */
  double process_noise_vel;  /* 0.05 m/s per step */
  double speed_margin;       /* 1.2 */
  double init_radius;        /* 450 m */
} ut_pf_config;

/* EnvConfig (env_config.hpp:44-93) as a POD. The heading model
 * (kinematics.hpp:34-54) is carried as its resolved bucket for (agent_speed, dt):
 * kind UT_HEADING_DEFAULT resolves it from the shipped default fit
 * (kinematics.cpp:180-186) in ut_config_finalize(); UT_HEADING_BUCKET uses
 * heading_a / heading_b as given. */
typedef struct ut_env_config {
  int32_t n_agents, n_targets, horizon, reward_mode;
  double dt;
  double agent_speed, target_speed_frac, target_speed_frac_max, target_turn_interval;
  double detection_range, comm_range, comm_drop_prob, range_noise_std;
  double eps_min, eps_max, d_min, d_safe;
  double spawn_min_sep, spawn_max_sep, perturbation_std;
  double target_depth_min, target_depth_max;
  int32_t lost_steps;
  int32_t heading_model_kind;
  double heading_a, heading_b, heading_noise_std;
  ut_pf_config pf;
  /* Resolved by ut_config_finalize(): |heading_delta(0.24)| (env.cpp:115-116). */
  double max_turn_per_step;
} ut_env_config;

/* Device views of the batch buffers (vecenv.hpp:51-62). Matrices are
 * column-major like Eigen::MatrixXd: element (row, col) at ptr[col * rows + row].
 *   obs / final_obs : rows ((env * n_agents + agent) * n_rows + row), 12 cols
 *   global_state    : rows (env * n_rows + row), 12 cols
 *   masks           : (env * n_agents + agent) * 5 + action
 *   per-target info : env * n_targets + target                               */
typedef struct ut_buffers {
  int64_t n_envs;
  int32_t n_agents, n_targets, n_rows, n_particles;
  int64_t obs_rows, global_rows;
  double* obs;
  double* final_obs;
  double* global_state;
  double* rewards;
  uint8_t* dones;
  uint8_t* masks;
  double* tracking_error;  /* StepOutput::tracking_error (env.hpp:57) */
  double* min_agent_dist;  /* StepOutput::min_agent_dist (env.hpp:58) */
  uint8_t* target_lost;    /* StepOutput::target_lost (env.hpp:59) */
  uint8_t* collision;      /* StepOutput::collision (env.hpp:56) */
  int32_t* step;           /* WorldState::step per env (env.hpp:50) */
  int32_t* actions;        /* device action staging, n_envs * n_agents */
  /* particle store, structure-of-arrays: field[set * n_particles + k] for
   * set = set_offset[env] + agent * n_targets(env) + target; a homogeneous
   * batch has set_offset == NULL and set = env * n_agents * n_targets + ...
   * (mixed fleets, ut_vecenv_create_mixed, store only their own A_e * T_e sets) */
  double *px, *py, *vx, *vy, *w;
  int64_t total_sets;          /* sets in the store (sum over envs of A_e * T_e) */
  const int64_t* set_offset;   /* device, [n_envs], or NULL when homogeneous */
} ut_buffers;

/* Host destinations for ut_vecenv_copy_outputs(); NULL members are skipped. */
typedef struct ut_host_outputs {
  double* obs;
  double* final_obs;
  double* global_state;
  double* rewards;
  uint8_t* dones;
  uint8_t* masks;
  double* tracking_error;
  double* min_agent_dist;
  uint8_t* target_lost;
  uint8_t* collision;
  int32_t* step;
} ut_host_outputs;

/* Episode statistics accumulated on the device (marl.cpp:288-306 accumulators);
 * the multi-GPU driver all-reduces this vector once per report interval. */
enum {
  UT_STAT_ENV_STEPS = 0,      /* env-steps taken                          */
  UT_STAT_REWARD_SUM,         /* sum of step rewards                      */
  UT_STAT_TRACK_ERR_SUM,      /* sum over env-steps of mean target error  */
  UT_STAT_EPISODES_DONE,      /* completed episodes                       */
  UT_STAT_EPISODE_RETURN_SUM, /* sum of completed-episode returns         */
  UT_STAT_COLLISION_STEPS,    /* env-steps with a collision               */
  UT_STAT_LOST_TARGET_STEPS,  /* (env, target)-steps flagged lost         */
  UT_STAT_PF_UPDATES,         /* particle-filter measurement updates      */
  UT_STAT_PF_RESAMPLES,       /* particle-filter resamples                */
  UT_STAT_PF_EXACT_PATH,      /* sets that took the exact sequential update path */
  /* curriculum::evaluate's Table-2 metrics (curriculum.cpp:267-356) over the
   * completed episodes: per-episode mean agent-target distance and mean tracking
   * error (sums and sums of squares), episodes with a collision / a lost target */
  UT_STAT_EVAL_DIST_SUM,
  UT_STAT_EVAL_DIST_SQ,
  UT_STAT_EVAL_ERR_SUM,
  UT_STAT_EVAL_ERR_SQ,
  UT_STAT_EVAL_COLLIDED_EPISODES,
  UT_STAT_EVAL_LOST_EPISODES,
  UT_N_STATS
};

/* Phases of the step (StepPhase, env.hpp:71-80; PhaseTimer env.cpp:18-36,
 * 250-279) plus the auto-reset, which the reference runs outside its phase
 * timers (vecenv.cpp:140). On the device each CTA times its own share of the
 * grid (SM clock of thread 0, converted to ns), summed over CTAs like the
 * reference sums its envs' timers (vecenv.cpp:160-173). The merged range-update
 * pass of a particle set is split between FILTER (the agent's own ping,
 * env.cpp:356-360) and COMMS (the fused senders' pings, env.cpp:385-392) in
 * proportion; COMMS also holds the comm decisions, maybe_resample and the
 * estimate (env.cpp:365-410). */
enum {
  UT_PHASE_TARGETS = 0, UT_PHASE_AGENTS, UT_PHASE_MEASURE, UT_PHASE_FILTER, UT_PHASE_COMMS,
  UT_PHASE_OBSERVE, UT_PHASE_REWARD, UT_PHASE_RESET, UT_N_PHASES
};

/* BenchmarkReport (vecenv.hpp:87-98), device-timed. */
typedef struct ut_benchmark_report {
  int64_t n_envs;
  int32_t n_agents, n_targets, timed_steps, _pad0;
  double wall_seconds; /* CUDA-event time of the timed steps */
  double sps;          /* env-steps per second, n_envs * steps / seconds (vecenv.cpp:198) */
  double agent_sps;    /* sps * n_agents */
  uint64_t phase_ns[UT_N_PHASES]; /* BenchmarkReport::phase_ns (+ reset), CTA-summed */
  uint64_t total_ns;              /* BenchmarkReport::total_ns: sum of the seven step phases */
} ut_benchmark_report;

typedef struct ut_vecenv ut_vecenv;

/* ---- configuration ---------------------------------------------------- */
/* EnvConfig{} defaults (env_config.hpp:44-80). */
void ut_config_default(ut_env_config* cfg);
/* EnvConfig::finalize (env.cpp:40-65): validates every field (UT_ERR_CONFIG naming
 * the field) and resolves the heading bucket and max turn. */
int ut_config_finalize(ut_env_config* cfg);

/* ---- VecEnv ------------------------------------------------------------- */
/* VecEnv::VecEnv (vecenv.cpp:7-45) = n_envs x Environment::Environment(cfg, seed, i)
 * (env.cpp:110-151). Env i of this shard has GLOBAL index env_index_offset + i,
 * which keys its RNG streams (env.cpp:113-114, 130-133), so a shard of a larger
 * batch is bit-identical to the same envs of the unsharded batch. */
int ut_vecenv_create(const ut_env_config* cfg, int64_t n_envs, uint64_t master_seed,
                     int64_t env_index_offset, int device, ut_vecenv** out);
/* Heterogeneous fleets (no reference counterpart: the reference VecEnv is
 * homogeneous, vecenv.cpp:7-22): env i uses cfgs[cfg_of_env[i]]. Batch buffers are
 * padded to the largest n_agents / n_rows / n_targets (padding rows are zero). */
int ut_vecenv_create_mixed(const ut_env_config* cfgs, int32_t n_cfgs,
                           const int32_t* cfg_of_env, int64_t n_envs, uint64_t master_seed,
                           int64_t env_index_offset, int device, ut_vecenv** out);
void ut_vecenv_destroy(ut_vecenv* v);

/* VecEnv::reset_all (vecenv.cpp:69-77). */
int ut_vecenv_reset_all(ut_vecenv* v);
/* VecEnv::step (vecenv.cpp:79-116): actions row-major n_envs x n_agents, host or
 * device memory. Every action is validated BEFORE any env steps; on a violation
 * nothing is mutated and UT_ERR_CONTRACT names the lowest failing env ("env i: ...").
 * Validation and step are enqueued together (the step kernel is gated on the
 * validation result on the device) and the call returns after ONE wait. */
int ut_vecenv_step(ut_vecenv* v, const int32_t* actions, int actions_on_device);
/* VecEnv::step_policy (vecenv.cpp:118-143), policy UT_POLICY_*. n_steps > 1 runs
 * that many steps back to back with no host round trip in between, as ONE CUDA
 * graph launch of n_steps cooperative step kernels (captured on first use per
 * (policy, n_steps), re-captured after any change to the handle's launch state;
 * single output buffer only; UT_NO_GRAPHS=1 in the environment disables it);
 * the status is checked once at the end. */
int ut_vecenv_step_policy(ut_vecenv* v, int policy, int n_steps);
/* VecEnv::refresh_outputs (vecenv.cpp:145-150). */
int ut_vecenv_refresh_outputs(ut_vecenv* v);

int ut_vecenv_buffers(ut_vecenv* v, ut_buffers* out);
int ut_vecenv_copy_outputs(ut_vecenv* v, const ut_host_outputs* dst);
/* Output double buffering (n = 2; default 1): each step then writes the batch
 * buffers the previous step did not, so the previous step's outputs can be
 * copied out (ut_vecenv_copy_outputs_async) while the next step runs. The
 * pointers of ut_vecenv_buffers() then change with every step (re-query after
 * each), final_obs included: the step copies the terminal rows the previous
 * step wrote into the other set, so either set holds every env's latest terminal
 * observation. Steps and resets wait for an asynchronous copy still reading the
 * set they write. */
int ut_vecenv_set_output_buffers(ut_vecenv* v, int n);
/* Enqueues the D2H copies of the current outputs on `cuda_stream` after the
 * handle's pending work, and returns; synchronize that stream before reading. */
int ut_vecenv_copy_outputs_async(ut_vecenv* v, const ut_host_outputs* dst, void* cuda_stream);
/* Runs subsequent work on a caller-owned cudaStream_t. NULL selects the
 * handle's own (non-blocking) stream; UT_STREAM_LEGACY (the value of
 * cudaStreamLegacy) selects the legacy default stream, which is what a
 * framework's stream handle 0 means (e.g. torch.cuda.current_stream()). */
#define UT_STREAM_LEGACY ((void*)0x1)
int ut_vecenv_set_stream(ut_vecenv* v, void* cuda_stream);
/* Orders the handle's next work after everything enqueued so far on
 * `cuda_stream` (0 = the legacy default stream, as in CUDA): call it before
 * ut_vecenv_step with actions a device policy is still producing, or before a
 * step that will overwrite outputs other kernels are still reading. */
int ut_vecenv_wait_stream(ut_vecenv* v, void* cuda_stream);
int ut_vecenv_synchronize(ut_vecenv* v);
/* Reads (and optionally zeroes) the device statistics vector. */
int ut_vecenv_stats(ut_vecenv* v, double out[UT_N_STATS], int reset);
/* Number of kernels this handle has launched so far. */
int64_t ut_vecenv_launch_count(const ut_vecenv* v);

/* VecEnv::enable_phase_timing / reset_timing / phase_ns (vecenv.hpp:64-67,
 * PhaseTimer env.cpp:18-36) on the device, per UT_PHASE_* (see above): SM
 * cycles, or ns at the SM clock rate the timed launches ran at. */
int ut_vecenv_enable_phase_timing(ut_vecenv* v, int on);
int ut_vecenv_phase_cycles(ut_vecenv* v, uint64_t out[UT_N_PHASES], int reset);
int ut_vecenv_phase_ns(ut_vecenv* v, uint64_t out[UT_N_PHASES], int reset);

/* Auto-reset of finished envs inside step / step_policy (vecenv.cpp:106-112,
 * 140; default on). Off gives the single Environment's semantics
 * (env.cpp:234-504): a finished env keeps its terminal state and stays done
 * until reset; final_obs is not written. */
int ut_vecenv_set_auto_reset(ut_vecenv* v, int on);

/* ---- multi-device VecEnv ------------------------------------------------ */
/* One VecEnv over several GPUs of one box, like the reference's one VecEnv over
 * its worker threads (vecenv.hpp:26-27, sharded by env index at vecenv.cpp:83).
 * Envs shard by contiguous global index range (shard i = envs
 * [n_envs*i/n, n_envs*(i+1)/n)), each shard an ordinary ut_vecenv on
 * device_ids[i] keyed by its global env indices, so the batch is bit-identical to
 * a single-device VecEnv of the same n_envs and seed. Steps run on every device
 * concurrently with no data-path collective; the statistics vector is
 * all-reduced over NCCL (north_star). Homogeneous configs only. */
typedef struct ut_multienv ut_multienv;
enum {
  UT_MULTI_STATS_AUTO = 0, /* NCCL when the device ids are distinct and n_devices > 1, else host */
  UT_MULTI_STATS_NCCL = 1, /* always NCCL (also for one device); device ids must be distinct */
  UT_MULTI_STATS_HOST = 2  /* the shards' vectors summed on the host, in shard order */
};
int ut_multienv_create(const ut_env_config* cfg, int64_t n_envs, uint64_t master_seed, const int32_t* device_ids,
                       int32_t n_devices, int32_t stats_flags, ut_multienv** out);
void ut_multienv_destroy(ut_multienv* m);
int ut_multienv_n_shards(const ut_multienv* m);
/* UT_MULTI_STATS_NCCL or UT_MULTI_STATS_HOST: how ut_multienv_stats reduces. */
int ut_multienv_stats_backend(const ut_multienv* m);
/* Shard i's single-device handle (for its device buffers), its global env range and device. */
int ut_multienv_shard(ut_multienv* m, int32_t i, ut_vecenv** shard, int64_t* env_begin, int64_t* env_end,
                      int32_t* device);
/* The shard holding global env `env`, and its index inside that shard. */
int ut_multienv_locate(ut_multienv* m, int64_t env, ut_vecenv** shard, int64_t* local_env);
int ut_multienv_reset_all(ut_multienv* m);
/* VecEnv::step with host actions, n_envs x n_agents row-major over the WHOLE batch;
 * validated on every device before any env moves (lowest failing GLOBAL env). */
int ut_multienv_step(ut_multienv* m, const int32_t* actions);
int ut_multienv_step_policy(ut_multienv* m, int policy, int n_steps);
int ut_multienv_refresh_outputs(ut_multienv* m);
int ut_multienv_set_auto_reset(ut_multienv* m, int on);
int ut_multienv_synchronize(ut_multienv* m);
/* The whole batch's outputs in the single-handle layout (ut_buffers). */
int ut_multienv_copy_outputs(ut_multienv* m, const ut_host_outputs* dst);
/* Batch statistics, all-reduced over the shards (see UT_MULTI_STATS_*). */
int ut_multienv_stats(ut_multienv* m, double out[UT_N_STATS], int reset);
int ut_multienv_enable_phase_timing(ut_multienv* m, int on);
int ut_multienv_phase_ns(ut_multienv* m, uint64_t out[UT_N_PHASES], int reset);
int64_t ut_multienv_launch_count(const ut_multienv* m);
/* env(i).serialize_state / deserialize_state / world().step by GLOBAL env index. */
int ut_multienv_serialize(ut_multienv* m, int64_t env, double* blob, size_t cap, size_t* len);
int ut_multienv_deserialize(ut_multienv* m, int64_t env, const double* blob, size_t len);
int ut_multienv_world_step(ut_multienv* m, int64_t env, int32_t* step);
/* ncclGetVersion of the NCCL the statistics all-reduce loads (UT_ERR_RUNTIME if none). */
int ut_nccl_version(int* version);

/* ---- per-env state (Environment API) ----------------------------------- */
/* Environment::serialize_state / deserialize_state (env.cpp:550-659), identical
 * blob layout: 5 + 6A + 9T + A*(6A + T*(9 + 5P)) doubles. `len` receives the
 * required length; UT_ERR_DATA if `cap` is too small / the blob is malformed. */
int ut_env_serialize(ut_vecenv* v, int64_t env, double* blob, size_t cap, size_t* len);
int ut_env_deserialize(ut_vecenv* v, int64_t env, const double* blob, size_t len);
/* Batched serialize_state / deserialize_state of envs [env_begin, env_end) (the
 * checkpoint path, marl.cpp:741-805): the blobs back to back, env e's at the sum
 * of the blob lengths before it; packed / unpacked on the device straight from the
 * state store. export: `len` receives the total (blobs may be NULL to query),
 * UT_ERR_DATA if `cap` is too small. import: UT_ERR_DATA unless len is exact. */
int ut_vecenv_export_state(ut_vecenv* v, int64_t env_begin, int64_t env_end, double* blobs, size_t cap,
                           size_t* len);
int ut_vecenv_import_state(ut_vecenv* v, int64_t env_begin, int64_t env_end, const double* blobs, size_t len);
/* Trajectory capture (append_trajectory_rows, trajectory.cpp:13-66; used by
 * curriculum::evaluate and cmd_rollout) for envs [env_begin, env_end) (empty =
 * off): every step, before auto-reset, each captured env records one row per
 * entity -- agents then targets, padded to the batch's rows -- of
 * UT_TRAJ_FIELDS doubles: step (-1 on padding rows), x, y, z, heading,
 * has_estimate, est_x, est_y, track_err, reward, collision, is_target.
 * ut_vecenv_trajectory_rows copies the last step's rows (len = n x rows x fields). */
enum { UT_TRAJ_FIELDS = 12 };
int ut_vecenv_capture_trajectory(ut_vecenv* v, int64_t env_begin, int64_t env_end);
int ut_vecenv_trajectory_rows(ut_vecenv* v, double* rows, size_t cap, size_t* len);
/* world().step (env.hpp:50), read by Trainer::collect_rollout (marl.cpp:211,227). */
int ut_env_world_step(ut_vecenv* v, int64_t env, int32_t* step);

/* ---- benchmark ------------------------------------------------------------ */
/* benchmark_sps (vecenv.cpp:175-202) on the device: warmup + timed step_policy. */
int ut_benchmark_sps(const ut_env_config* cfg, int64_t n_envs, int32_t n_steps, int policy,
                     uint64_t seed, int32_t warmup, int device, ut_benchmark_report* out);

const char* ut_last_error(void);
int ut_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* UT_ENV_H_ */
