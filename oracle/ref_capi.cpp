// ref_capi.cpp -- TEST INFRASTRUCTURE (oracle/_ref only; never linked into the
// product). A thin C wrapper over the REFERENCE's own utrack::VecEnv /
// Environment (compiled unmodified from /root/reference/proj/core/src) so the
// Python tests can drive the reference and the B200 build side by side, and so
// bench.py's `--impl reference` arm can time the reference's benchmark_sps
// (vecenv.cpp:175-202) on the host cores.
#include <cstring>
#include <exception>
#include <memory>
#include <string>

#include "ut_env.h"
#include "utrack/env.hpp"
#include "utrack/errors.hpp"
#include "utrack/vecenv.hpp"

using namespace utrack;

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return UT_OK;
  } catch (const ContractViolation& e) {
    return fail(UT_ERR_CONTRACT, e.what());
  } catch (const ConfigError& e) {
    return fail(UT_ERR_CONFIG, e.what());
  } catch (const DataError& e) {
    return fail(UT_ERR_DATA, e.what());
  } catch (const std::exception& e) {
    return fail(UT_ERR_RUNTIME, e.what());
  }
}

EnvConfig to_ref(const ut_env_config& c) {
  EnvConfig e;
  e.n_agents = c.n_agents;
  e.n_targets = c.n_targets;
  e.horizon = c.horizon;
  e.dt = c.dt;
  e.agent_speed = c.agent_speed;
  e.target_speed_frac = c.target_speed_frac;
  e.target_speed_frac_max = c.target_speed_frac_max;
  e.target_turn_interval = c.target_turn_interval;
  e.detection_range = c.detection_range;
  e.comm_range = c.comm_range;
  e.comm_drop_prob = c.comm_drop_prob;
  e.range_noise_std = c.range_noise_std;
  e.eps_min = c.eps_min;
  e.eps_max = c.eps_max;
  e.d_min = c.d_min;
  e.d_safe = c.d_safe;
  e.reward_mode = c.reward_mode == UT_REWARD_FOLLOW ? RewardMode::kFollow : RewardMode::kTracking;
  e.spawn_min_sep = c.spawn_min_sep;
  e.spawn_max_sep = c.spawn_max_sep;
  e.perturbation_std = c.perturbation_std;
  e.target_depth_min = c.target_depth_min;
  e.target_depth_max = c.target_depth_max;
  e.lost_steps = c.lost_steps;
  e.pf.n_particles = c.pf.n_particles;
  e.pf.process_noise_pos = c.pf.process_noise_pos;
  e.pf.process_noise_vel = c.pf.process_noise_vel;
  e.pf.speed_margin = c.pf.speed_margin;
  e.pf.init_radius = c.pf.init_radius;
  if (c.heading_model_kind == UT_HEADING_BUCKET) {
    e.heading_model = HeadingDeltaModel();
    e.heading_model.set_bucket(c.agent_speed, c.dt, {c.heading_a, c.heading_b});
  } else {
    e.heading_model = default_heading_model();
  }
  e.heading_model.set_noise_std(c.heading_noise_std);
  return e;
}

struct RefVec {
  EnvConfig cfg;
  std::unique_ptr<VecEnv> venv;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// EnvConfig::finalize through the reference, reporting the resolved bucket.
int ref_config_finalize(ut_env_config* c) {
  return guarded([&] {
    EnvConfig e = to_ref(*c);
    e.finalize();
    const LinearCoeffs& b = e.heading_model.bucket(e.agent_speed, e.dt);
    c->heading_a = b.a;
    c->heading_b = b.b;
    c->max_turn_per_step = std::abs(heading_delta(e.heading_model, kMaxRudderAngle, e.agent_speed, e.dt));
  });
}

int ref_vecenv_create(const ut_env_config* c, int64_t n_envs, uint64_t seed, int workers, void** out) {
  return guarded([&] {
    auto r = std::make_unique<RefVec>();
    r->cfg = to_ref(*c);
    r->venv = std::make_unique<VecEnv>(r->cfg, static_cast<int>(n_envs), seed, workers);
    *out = r.release();
  });
}

void ref_vecenv_destroy(void* h) { delete static_cast<RefVec*>(h); }

int ref_vecenv_reset_all(void* h) {
  return guarded([&] { static_cast<RefVec*>(h)->venv->reset_all(); });
}

int ref_vecenv_step(void* h, const int32_t* actions) {
  return guarded([&] {
    VecEnv& v = *static_cast<RefVec*>(h)->venv;
    const std::size_t n = static_cast<std::size_t>(v.n_envs()) * v.n_agents();
    static_assert(sizeof(int) == sizeof(int32_t));
    v.step(std::span<const int>(reinterpret_cast<const int*>(actions), n));
  });
}

int ref_vecenv_step_policy(void* h, int policy, int n_steps) {
  return guarded([&] {
    VecEnv& v = *static_cast<RefVec*>(h)->venv;
    for (int i = 0; i < n_steps; ++i)
      v.step_policy(policy == UT_POLICY_SCRIPTED ? BenchmarkPolicy::kScripted : BenchmarkPolicy::kRandom);
  });
}

int ref_vecenv_refresh_outputs(void* h) {
  return guarded([&] { static_cast<RefVec*>(h)->venv->refresh_outputs(); });
}

int ref_vecenv_copy_outputs(void* h, const ut_host_outputs* d) {
  return guarded([&] {
    VecEnv& v = *static_cast<RefVec*>(h)->venv;
    const int n = v.n_envs();
    const int nt = v.config().n_targets;
    auto copy_mat = [](double* dst, const Eigen::MatrixXd& m) {
      if (dst) std::memcpy(dst, m.data(), sizeof(double) * static_cast<std::size_t>(m.size()));
    };
    copy_mat(d->obs, v.obs_stack());
    copy_mat(d->final_obs, v.final_obs_stack());
    copy_mat(d->global_state, v.global_stack());
    if (d->rewards) std::memcpy(d->rewards, v.rewards().data(), sizeof(double) * n);
    if (d->dones) std::memcpy(d->dones, v.dones().data(), static_cast<std::size_t>(n));
    if (d->masks) std::memcpy(d->masks, v.masks().data(), v.masks().size());
    for (int i = 0; i < n; ++i) {
      const StepOutput& o = v.infos()[static_cast<std::size_t>(i)];
      for (int t = 0; t < nt; ++t) {
        const std::size_t k = static_cast<std::size_t>(i) * nt + t;
        if (d->tracking_error) d->tracking_error[k] = o.tracking_error[static_cast<std::size_t>(t)];
        if (d->min_agent_dist) d->min_agent_dist[k] = o.min_agent_dist[static_cast<std::size_t>(t)];
        if (d->target_lost) d->target_lost[k] = o.target_lost[static_cast<std::size_t>(t)];
      }
      if (d->collision) d->collision[i] = o.collision ? 1 : 0;
      if (d->step) d->step[i] = v.env(i).world().step;
    }
  });
}

int ref_env_serialize(void* h, int64_t env, double* blob, size_t cap, size_t* len) {
  return guarded([&] {
    const std::vector<double> b = static_cast<RefVec*>(h)->venv->env(static_cast<int>(env)).serialize_state();
    *len = b.size();
    if (blob == nullptr) return;
    if (cap < b.size()) throw DataError("serialize: buffer too small");
    std::memcpy(blob, b.data(), sizeof(double) * b.size());
  });
}

int ref_env_deserialize(void* h, int64_t env, const double* blob, size_t len) {
  return guarded([&] {
    static_cast<RefVec*>(h)->venv->env(static_cast<int>(env)).deserialize_state(std::span<const double>(blob, len));
  });
}

// Environment::action_mask after an out-of-band state change (used by the
// oracle-restatement tests to drive identical random actions).
int ref_env_world_step(void* h, int64_t env, int32_t* step) {
  return guarded([&] { *step = static_cast<RefVec*>(h)->venv->env(static_cast<int>(env)).world().step; });
}

// A single reference Environment (env.hpp:91-171): no auto-reset, done stays set.
struct RefEnv {
  EnvConfig cfg;
  std::unique_ptr<Environment> env;
};

int ref_env_create(const ut_env_config* c, uint64_t seed, int64_t env_index, void** out) {
  return guarded([&] {
    auto r = std::make_unique<RefEnv>();
    r->cfg = to_ref(*c);
    r->env = std::make_unique<Environment>(r->cfg, seed, static_cast<int>(env_index));
    *out = r.release();
  });
}

void ref_env_destroy(void* h) { delete static_cast<RefEnv*>(h); }

int ref_env_reset(void* h) {
  return guarded([&] { static_cast<RefEnv*>(h)->env->reset(); });
}

// Environment::step; reward / done / collision of the StepOutput (env.hpp:53-60).
int ref_env_step(void* h, const int32_t* actions, double* reward, int32_t* done, int32_t* collision) {
  return guarded([&] {
    Environment& e = *static_cast<RefEnv*>(h)->env;
    const StepOutput& o =
        e.step(std::span<const int>(reinterpret_cast<const int*>(actions), static_cast<std::size_t>(e.config().n_agents)));
    *reward = o.reward;
    *done = o.done ? 1 : 0;
    *collision = o.collision ? 1 : 0;
  });
}

int ref_env_serialize_one(void* h, double* blob, size_t cap, size_t* len) {
  return guarded([&] {
    const std::vector<double> b = static_cast<RefEnv*>(h)->env->serialize_state();
    *len = b.size();
    if (blob == nullptr) return;
    if (cap < b.size()) throw DataError("serialize: buffer too small");
    std::memcpy(blob, b.data(), sizeof(double) * b.size());
  });
}

// Environment::observation(a) (env.hpp:109-110): R x 12, row-major here.
int ref_env_observation(void* h, int32_t agent, double* out) {
  return guarded([&] {
    const Eigen::MatrixXd& m = static_cast<RefEnv*>(h)->env->observation(agent);
    for (int r = 0; r < m.rows(); ++r)
      for (int k = 0; k < m.cols(); ++k) out[r * m.cols() + k] = m(r, k);
  });
}

// benchmark_sps (vecenv.cpp:175-202): SPS plus the seven phase sums.
int ref_benchmark_sps(const ut_env_config* c, int64_t n_envs, int32_t n_steps, int policy, uint64_t seed,
                      int32_t workers, int32_t warmup, double* sps, double* wall_seconds,
                      int32_t* workers_used, uint64_t* phase_ns /* [7] */, uint64_t* total_ns) {
  return guarded([&] {
    const BenchmarkReport rep = benchmark_sps(
        to_ref(*c), static_cast<int>(n_envs), n_steps,
        policy == UT_POLICY_SCRIPTED ? BenchmarkPolicy::kScripted : BenchmarkPolicy::kRandom, seed, workers,
        warmup);
    *sps = rep.sps;
    *wall_seconds = rep.wall_seconds;
    *workers_used = rep.workers;
    for (int p = 0; p < static_cast<int>(StepPhase::kCount); ++p) phase_ns[p] = rep.phase_ns[static_cast<std::size_t>(p)];
    *total_ns = rep.total_ns;
  });
}

// Raw Philox block and key derivation (rng.hpp:30-38, 116-131) for unit tests.
void ref_philox_block(uint64_t key, uint64_t stream, uint64_t block, uint32_t out[4]) {
  RngStream(key, stream).block_at(block, out);
}
uint64_t ref_derive_key(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  return RngStream::derive_key(a, b, c, d);
}

}  // extern "C"
