// ut_vecenv.hpp -- header-only C++17 facade over the C-ABI (ut_env.h) with the
// reference's utrack::VecEnv surface (core/include/utrack/vecenv.hpp:26-104) and
// error classes (errors.hpp:10-26), so reference-side code can switch by changing
// an include and a namespace alias:
//
//   #include "ut_vecenv.hpp"
//   namespace ut = utrack_b200;
//   ut::VecEnv venv(cfg, n_envs, seed);          // was utrack::VecEnv
//   venv.step(actions);                            // std::span / vector of int
//   const auto& r = venv.rewards();                // host mirrors, refreshed lazily
//
// Host accessors (obs_stack, rewards, ...) copy the device batch buffers into
// host mirrors on first use after a step, exactly the data the reference exposes.
// Device pointers (for a GPU policy; no D2H) come from device_buffers().
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "ut_env.h"

namespace utrack_b200 {

// errors.hpp:10-26 (same bases, same meaning)
class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};
class DataError : public std::runtime_error {
 public:
  explicit DataError(const std::string& w) : std::runtime_error(w) {}
};
class ContractViolation : public std::logic_error {
 public:
  explicit ContractViolation(const std::string& w) : std::logic_error(w) {}
};
class DeviceError : public std::runtime_error {
 public:
  explicit DeviceError(const std::string& w) : std::runtime_error(w) {}
};

inline void check(int rc) {
  if (rc == UT_OK) return;
  const std::string msg = ut_last_error();
  switch (rc) {
    case UT_ERR_CONTRACT: throw ContractViolation(msg);
    case UT_ERR_CONFIG: throw ConfigError(msg);
    case UT_ERR_DATA: throw DataError(msg);
    default: throw DeviceError(msg);
  }
}

using EnvConfig = ut_env_config;
enum class BenchmarkPolicy { kRandom = UT_POLICY_RANDOM, kScripted = UT_POLICY_SCRIPTED };

// EnvConfig{} (env_config.hpp:44-80)
inline EnvConfig default_config() {
  EnvConfig c;
  ut_config_default(&c);
  return c;
}

// Column-major host matrix view (Eigen::MatrixXd storage order).
struct ColMajor {
  std::vector<double> data;
  int64_t rows = 0, cols = 0;
  double operator()(int64_t r, int64_t c) const { return data[c * rows + r]; }
};

// StepOutput (env.hpp:53-60)
struct StepOutput {
  double reward = 0.0;
  bool done = false;
  bool collision = false;
  std::vector<double> tracking_error, min_agent_dist;
  std::vector<uint8_t> target_lost;
};

namespace detail {
// Host mirrors of the batch buffers (vecenv.hpp:51-62), filled by one
// ut_host_outputs copy (single- or multi-device).
struct HostMirror {
  ColMajor obs, global, final_obs;
  std::vector<double> rewards;
  std::vector<uint8_t> dones, masks;
  std::vector<StepOutput> infos;

  template <class Copy>
  void fill(int64_t E, int64_t A, int64_t T, int64_t R, Copy&& copy) {
    obs = {std::vector<double>(E * A * R * UT_FEATURE_DIM), E * A * R, UT_FEATURE_DIM};
    final_obs = {std::vector<double>(E * A * R * UT_FEATURE_DIM), E * A * R, UT_FEATURE_DIM};
    global = {std::vector<double>(E * R * UT_FEATURE_DIM), E * R, UT_FEATURE_DIM};
    rewards.assign(E, 0.0);
    dones.assign(E, 0);
    masks.assign(E * A * UT_NUM_ACTIONS, 0);
    std::vector<double> err(E * T), dist(E * T);
    std::vector<uint8_t> lost(E * T), coll(E);
    ut_host_outputs o{obs.data.data(), final_obs.data.data(), global.data.data(), rewards.data(),
                      dones.data(),    masks.data(),          err.data(),         dist.data(),
                      lost.data(),     coll.data(),           nullptr};
    check(copy(&o));
    infos.resize(E);
    for (int64_t e = 0; e < E; ++e) {
      StepOutput& s = infos[e];
      s.reward = rewards[e];
      s.done = dones[e] != 0;
      s.collision = coll[e] != 0;
      s.tracking_error.assign(err.begin() + e * T, err.begin() + (e + 1) * T);
      s.min_agent_dist.assign(dist.begin() + e * T, dist.begin() + (e + 1) * T);
      s.target_lost.assign(lost.begin() + e * T, lost.begin() + (e + 1) * T);
    }
  }
};
}  // namespace detail

class VecEnv {
 public:
  // VecEnv(cfg, n_envs, master_seed, workers) (vecenv.hpp:26-27); `workers` has
  // no meaning on the device and is ignored; `device` selects the GPU.
  VecEnv(const EnvConfig& cfg, int n_envs, std::uint64_t master_seed, int workers = 0, int device = 0,
         int64_t env_index_offset = 0)
      : n_envs_(n_envs) {
    (void)workers;
    check(ut_vecenv_create(&cfg, n_envs, master_seed, env_index_offset, device, &h_));
    check(ut_vecenv_buffers(h_, &buf_));
    dirty_ = true;
  }
  ~VecEnv() {
    if (h_) ut_vecenv_destroy(h_);
  }
  VecEnv(const VecEnv&) = delete;
  VecEnv& operator=(const VecEnv&) = delete;

  int n_envs() const { return n_envs_; }
  int n_agents() const { return buf_.n_agents; }
  int n_rows() const { return buf_.n_rows; }

  void reset_all() { check(ut_vecenv_reset_all(h_)), dirty_ = true; }
  // actions: n_envs x n_agents, row-major (vecenv.cpp:79-93)
  void step(const int* actions, size_t n) {
    if (n != static_cast<size_t>(n_envs_) * static_cast<size_t>(buf_.n_agents))
      throw ContractViolation("vecenv step: wrong action count");
    check(ut_vecenv_step(h_, reinterpret_cast<const int32_t*>(actions), 0));
    dirty_ = true;
  }
  template <class Span>
  void step(const Span& actions) {
    step(actions.data(), actions.size());
  }
  void step_policy(BenchmarkPolicy p) { check(ut_vecenv_step_policy(h_, static_cast<int>(p), 1)), dirty_ = true; }
  void refresh_outputs() { check(ut_vecenv_refresh_outputs(h_)), dirty_ = true; }

  const ColMajor& obs_stack() { return pull(), m_.obs; }
  const ColMajor& global_stack() { return pull(), m_.global; }
  const ColMajor& final_obs_stack() { return pull(), m_.final_obs; }
  const std::vector<double>& rewards() { return pull(), m_.rewards; }
  const std::vector<uint8_t>& dones() { return pull(), m_.dones; }
  const std::vector<uint8_t>& masks() { return pull(), m_.masks; }
  const std::vector<StepOutput>& infos() { return pull(), m_.infos; }

  // env(i) surface used by the trainer: world().step, serialize/deserialize
  int32_t world_step(int64_t env) const {
    int32_t s = 0;
    check(ut_env_world_step(h_, env, &s));
    return s;
  }
  std::vector<double> serialize_state(int64_t env) const {
    size_t len = 0;
    ut_env_serialize(h_, env, nullptr, 0, &len);
    std::vector<double> blob(len);
    check(ut_env_serialize(h_, env, blob.data(), blob.size(), &len));
    return blob;
  }
  void deserialize_state(int64_t env, const std::vector<double>& blob) {
    check(ut_env_deserialize(h_, env, blob.data(), blob.size()));
    dirty_ = true;
  }

  // batched serialize / deserialize of envs [begin, end), blobs back to back (checkpoints)
  std::vector<double> export_state(int64_t begin, int64_t end) const {
    size_t len = 0;
    check(ut_vecenv_export_state(h_, begin, end, nullptr, 0, &len));
    std::vector<double> blobs(len);
    check(ut_vecenv_export_state(h_, begin, end, blobs.data(), blobs.size(), &len));
    return blobs;
  }
  void import_state(int64_t begin, int64_t end, const std::vector<double>& blobs) {
    check(ut_vecenv_import_state(h_, begin, end, blobs.data(), blobs.size()));
    dirty_ = true;
  }

  const ut_buffers& device_buffers() const { return buf_; }
  ut_vecenv* handle() const { return h_; }

 private:
  void pull() {
    if (!dirty_) return;
    m_.fill(n_envs_, buf_.n_agents, buf_.n_targets, buf_.n_rows,
            [&](const ut_host_outputs* o) { return ut_vecenv_copy_outputs(h_, o); });
    dirty_ = false;
  }

  ut_vecenv* h_ = nullptr;
  int n_envs_;
  ut_buffers buf_{};
  bool dirty_ = true;
  detail::HostMirror m_;
};


// One VecEnv over several GPUs (ut_multienv_*): the reference's VecEnv surface
// (vecenv.hpp:26-104) with the envs sharded by index range over `devices`
// instead of worker threads; bit-identical to VecEnv(cfg, n_envs, seed) on one
// device. stats() is the batch total, all-reduced over NCCL.
class MultiVecEnv {
 public:
  MultiVecEnv(const EnvConfig& cfg, int n_envs, std::uint64_t master_seed, const std::vector<int>& devices,
              int stats_flags = UT_MULTI_STATS_AUTO)
      : n_envs_(n_envs), A_(cfg.n_agents), T_(cfg.n_targets) {
    std::vector<int32_t> d(devices.begin(), devices.end());
    check(ut_multienv_create(&cfg, n_envs, master_seed, d.data(), static_cast<int32_t>(d.size()), stats_flags, &h_));
  }
  ~MultiVecEnv() {
    if (h_) ut_multienv_destroy(h_);
  }
  MultiVecEnv(const MultiVecEnv&) = delete;
  MultiVecEnv& operator=(const MultiVecEnv&) = delete;

  int n_envs() const { return n_envs_; }
  int n_agents() const { return A_; }
  int n_rows() const { return A_ + T_; }
  int n_shards() const { return ut_multienv_n_shards(h_); }
  bool nccl_stats() const { return ut_multienv_stats_backend(h_) == UT_MULTI_STATS_NCCL; }

  void reset_all() { check(ut_multienv_reset_all(h_)), dirty_ = true; }
  void step(const int* actions, size_t n) {
    if (n != static_cast<size_t>(n_envs_) * static_cast<size_t>(A_))
      throw ContractViolation("vecenv step: wrong action count");
    check(ut_multienv_step(h_, reinterpret_cast<const int32_t*>(actions)));
    dirty_ = true;
  }
  template <class Span>
  void step(const Span& actions) {
    step(actions.data(), actions.size());
  }
  void step_policy(BenchmarkPolicy p, int n_steps = 1) {
    check(ut_multienv_step_policy(h_, static_cast<int>(p), n_steps)), dirty_ = true;
  }
  void refresh_outputs() { check(ut_multienv_refresh_outputs(h_)), dirty_ = true; }

  const ColMajor& obs_stack() { return pull(), m_.obs; }
  const ColMajor& global_stack() { return pull(), m_.global; }
  const ColMajor& final_obs_stack() { return pull(), m_.final_obs; }
  const std::vector<double>& rewards() { return pull(), m_.rewards; }
  const std::vector<uint8_t>& dones() { return pull(), m_.dones; }
  const std::vector<uint8_t>& masks() { return pull(), m_.masks; }
  const std::vector<StepOutput>& infos() { return pull(), m_.infos; }

  int32_t world_step(int64_t env) const {
    int32_t s = 0;
    check(ut_multienv_world_step(h_, env, &s));
    return s;
  }
  std::vector<double> serialize_state(int64_t env) const {
    size_t len = 0;
    check(ut_multienv_serialize(h_, env, nullptr, 0, &len));
    std::vector<double> blob(len);
    check(ut_multienv_serialize(h_, env, blob.data(), blob.size(), &len));
    return blob;
  }
  void deserialize_state(int64_t env, const std::vector<double>& blob) {
    check(ut_multienv_deserialize(h_, env, blob.data(), blob.size()));
    dirty_ = true;
  }
  // episode statistics (UT_STAT_*), the batch totals
  std::vector<double> stats(bool reset = false) {
    std::vector<double> s(UT_N_STATS);
    check(ut_multienv_stats(h_, s.data(), reset ? 1 : 0));
    return s;
  }
  // shard i's device buffers and its global env range
  ut_buffers device_buffers(int shard, int64_t* env_begin = nullptr, int64_t* env_end = nullptr) const {
    ut_vecenv* v = nullptr;
    check(ut_multienv_shard(h_, shard, &v, env_begin, env_end, nullptr));
    ut_buffers b{};
    check(ut_vecenv_buffers(v, &b));
    return b;
  }
  ut_multienv* handle() const { return h_; }

 private:
  void pull() {
    if (!dirty_) return;
    m_.fill(n_envs_, A_, T_, A_ + T_, [&](const ut_host_outputs* o) { return ut_multienv_copy_outputs(h_, o); });
    dirty_ = false;
  }

  ut_multienv* h_ = nullptr;
  int n_envs_, A_, T_;
  bool dirty_ = true;
  detail::HostMirror m_;
};

// benchmark_sps (vecenv.hpp:102-104), device-timed
inline ut_benchmark_report benchmark_sps(const EnvConfig& cfg, int n_envs, int n_steps, BenchmarkPolicy policy,
                                         std::uint64_t seed, int warmup = 16, int device = 0) {
  ut_benchmark_report r{};
  check(ut_benchmark_sps(&cfg, n_envs, n_steps, static_cast<int>(policy), seed, warmup, device, &r));
  return r;
}

}  // namespace utrack_b200
