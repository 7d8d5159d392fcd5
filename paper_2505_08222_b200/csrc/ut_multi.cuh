// ut_multi.cuh -- the multi-device VecEnv handle (include/ut_env.h, ut_multienv_*).
// Included at the end of ut_capi.cu: it is host code over the single-device
// handle's internals.
//
// The reference VecEnv is one object over all envs (vecenv.hpp:26-27), sharded
// over its worker threads by env index (vecenv.cpp:83 parallel_for). Here it is
// one object over n_devices GPUs: envs shard by contiguous global index range,
// shard i is an ordinary ut_vecenv on device_ids[i] with env_index_offset = its
// first global env (so the RNG streams are the unsharded batch's), each shard
// steps on its own device's stream with no data-path collective, and every
// device's work is enqueued before the handle waits on any of them. The only
// exchange is the statistics vector: ncclAllReduce over the shards' device
// copies (one communicator per device, ncclCommInitAll), after which every device
// holds the batch totals (BASELINE north_star: NCCL only for the episode-return /
// tracking-error statistics).
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": the one torch has already
// loaded, else the system's), so the library has no link-time NCCL dependency.
// NCCL cannot put two ranks of one communicator on the same device; a handle
// listing a device twice (a 1-GPU test of the sharding) sums the shards'
// vectors on the host in shard order instead (UT_MULTI_STATS_HOST).
#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
};

const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.why = std::string("dlopen(libnccl.so.2) failed: ") + (e ? e : "?");
      return a;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) all = false;
    };
    sym(a.comm_init_all, "ncclCommInitAll");
    sym(a.comm_destroy, "ncclCommDestroy");
    sym(a.all_reduce, "ncclAllReduce");
    sym(a.group_start, "ncclGroupStart");
    sym(a.group_end, "ncclGroupEnd");
    sym(a.error_string, "ncclGetErrorString");
    sym(a.get_version, "ncclGetVersion");
    a.ok = all;
    if (!all) a.why = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

#define UT_NCCL(api, call)                                                                              \
  do {                                                                                                  \
    ncclResult_t r_ = (call);                                                                           \
    if (r_ != ncclSuccess) return fail(UT_ERR_RUNTIME, "%s failed: %s", #call, (api).error_string(r_)); \
  } while (0)

}  // namespace

struct ut_multienv {
  std::vector<ut_vecenv*> shards;
  std::vector<int64_t> begin;  // n_shards + 1 global env boundaries
  std::vector<int> devices;
  int64_t n_envs = 0;
  int A = 0, T = 0, R = 0;
  int stats_backend = UT_MULTI_STATS_HOST;
  std::vector<ncclComm_t> comms;
  std::vector<double*> d_stats;  // per shard, UT_N_STATS doubles on its device

  ~ut_multienv() {
    const NcclApi& api = nccl_api();
    for (size_t i = 0; i < shards.size(); ++i) {
      DeviceGuard dg(devices[i]);
      if (i < d_stats.size() && d_stats[i]) cudaFree(d_stats[i]);
      if (i < comms.size() && comms[i] && api.ok) api.comm_destroy(comms[i]);
      ut_vecenv_destroy(shards[i]);
    }
  }
};

namespace {

// Runs f(shard, i) over every shard on its own device; stops at the first failure.
template <class F>
int each_shard(ut_multienv* m, F&& f) {
  for (size_t i = 0; i < m->shards.size(); ++i) {
    DeviceGuard dg(m->devices[i]);
    const int rc = f(m->shards[i], i);
    if (rc) return rc;
  }
  return UT_OK;
}

// Enqueue `enq` on every device, then wait for and check every device; the first
// failure in shard order wins (each later shard is still waited on).
template <class Enq>
int each_shard_then_status(ut_multienv* m, const char* what, Enq&& enq) {
  int rc = each_shard(m, [&](ut_vecenv* v, size_t i) -> int {
    int r;
    if ((r = enq(v, i))) return r;
    return v->enqueue_status();
  });
  int first = rc;
  for (size_t i = 0; i < m->shards.size(); ++i) {
    DeviceGuard dg(m->devices[i]);
    const int r = m->shards[i]->finish_status(what);
    if (r && !first) first = r;
  }
  return first;
}

}  // namespace

extern "C" {

int ut_multienv_create(const ut_env_config* cfg, int64_t n_envs, uint64_t master_seed, const int32_t* device_ids,
                       int32_t n_devices, int32_t flags, ut_multienv** out) {
  *out = nullptr;
  if (n_devices < 1 || !device_ids) return fail(UT_ERR_CONFIG, "multienv: n_devices must be >= 1");
  if (n_envs < n_devices) return fail(UT_ERR_CONFIG, "multienv: n_envs (%lld) < n_devices (%d)", (long long)n_envs, n_devices);
  ut_multienv* m = new ut_multienv();
  m->n_envs = n_envs;
  m->devices.assign(device_ids, device_ids + n_devices);
  // contiguous shards, sizes differing by at most one (sharding.shard_range)
  m->begin.resize((size_t)n_devices + 1);
  for (int i = 0; i <= n_devices; ++i) m->begin[(size_t)i] = n_envs * i / n_devices;
  int rc = UT_OK;
  for (int i = 0; i < n_devices && !rc; ++i) {
    ut_vecenv* v = nullptr;
    rc = ut_vecenv_create(cfg, m->begin[(size_t)i + 1] - m->begin[(size_t)i], master_seed, m->begin[(size_t)i],
                          m->devices[(size_t)i], &v);
    if (!rc) m->shards.push_back(v);
  }
  if (!rc) {
    ut_vecenv* v0 = m->shards[0];
    m->A = v0->A_max, m->T = v0->T_max, m->R = v0->R_max;
  }
  bool distinct = true;
  for (int i = 0; i < n_devices; ++i)
    for (int j = 0; j < i; ++j) distinct = distinct && device_ids[i] != device_ids[j];
  const bool want_nccl = flags == UT_MULTI_STATS_NCCL || (flags == UT_MULTI_STATS_AUTO && distinct && n_devices > 1);
  if (!rc && flags == UT_MULTI_STATS_NCCL && !distinct)
    rc = fail(UT_ERR_CONFIG, "multienv: NCCL statistics need distinct device ids (NCCL allows one rank per device)");
  if (!rc && want_nccl) {
    const NcclApi& api = nccl_api();
    if (!api.ok) {
      rc = fail(UT_ERR_RUNTIME, "multienv: %s", api.why.c_str());
    } else {
      m->comms.assign((size_t)n_devices, nullptr);
      const ncclResult_t r = api.comm_init_all(m->comms.data(), n_devices, m->devices.data());
      if (r != ncclSuccess) {
        m->comms.assign((size_t)n_devices, nullptr);
        rc = fail(UT_ERR_RUNTIME, "multienv: ncclCommInitAll failed: %s", api.error_string(r));
      } else {
        m->stats_backend = UT_MULTI_STATS_NCCL;
      }
    }
  }
  if (!rc) {
    m->d_stats.assign((size_t)n_devices, nullptr);
    rc = each_shard(m, [&](ut_vecenv*, size_t i) -> int {
      UT_CUDA(cudaMalloc((void**)&m->d_stats[i], sizeof(double) * UT_N_STATS));
      return UT_OK;
    });
  }
  if (rc) {
    delete m;
    return rc;
  }
  *out = m;
  return UT_OK;
}

void ut_multienv_destroy(ut_multienv* m) { delete m; }

int ut_multienv_n_shards(const ut_multienv* m) { return (int)m->shards.size(); }

int ut_multienv_stats_backend(const ut_multienv* m) { return m->stats_backend; }

int ut_multienv_shard(ut_multienv* m, int32_t i, ut_vecenv** shard, int64_t* env_begin, int64_t* env_end,
                      int32_t* device) {
  if (i < 0 || (size_t)i >= m->shards.size())
    return fail(UT_ERR_CONTRACT, "multienv: shard %d outside [0, %zu)", i, m->shards.size());
  if (shard) *shard = m->shards[(size_t)i];
  if (env_begin) *env_begin = m->begin[(size_t)i];
  if (env_end) *env_end = m->begin[(size_t)i + 1];
  if (device) *device = m->devices[(size_t)i];
  return UT_OK;
}

int ut_multienv_locate(ut_multienv* m, int64_t env, ut_vecenv** shard, int64_t* local_env) {
  if (env < 0 || env >= m->n_envs)
    return fail(UT_ERR_CONTRACT, "multienv: env %lld outside [0, %lld)", (long long)env, (long long)m->n_envs);
  const size_t i = (size_t)(std::upper_bound(m->begin.begin(), m->begin.end(), env) - m->begin.begin()) - 1;
  *shard = m->shards[i];
  *local_env = env - m->begin[i];
  return UT_OK;
}

int ut_multienv_reset_all(ut_multienv* m) {
  return each_shard_then_status(m, "reset_all", [](ut_vecenv* v, size_t) -> int {
    int rc;
    if ((rc = v->reset_status())) return rc;
    return v->launch_reset(0);
  });
}

int ut_multienv_step(ut_multienv* m, const int32_t* actions) {
  // validate every shard (all devices in flight), then report the lowest failing
  // global env before anything moves (the single handle's semantics)
  int rc = each_shard(m, [&](ut_vecenv* v, size_t i) -> int { return enqueue_validate(v, actions + m->begin[i] * m->A, 0); });
  if (rc) return rc;
  for (size_t i = 0; i < m->shards.size(); ++i) {
    DeviceGuard dg(m->devices[i]);
    if ((rc = validate_result(m->shards[i], m->begin[i]))) return rc;
  }
  return each_shard_then_status(m, "step", [](ut_vecenv* v, size_t) -> int { return v->launch_step(MODE_EXTERNAL); });
}

int ut_multienv_step_policy(ut_multienv* m, int policy, int n_steps) {
  if (policy != UT_POLICY_RANDOM && policy != UT_POLICY_SCRIPTED)
    return fail(UT_ERR_CONTRACT, "step_policy: unknown policy %d", policy);
  const int mode = policy == UT_POLICY_RANDOM ? MODE_RANDOM : MODE_SCRIPTED;
  return each_shard_then_status(m, "step_policy", [&](ut_vecenv* v, size_t) -> int {
    int rc;
    if ((rc = v->reset_status())) return rc;
    return v->enqueue_policy_steps(mode, n_steps);
  });
}

int ut_multienv_refresh_outputs(ut_multienv* m) {
  return each_shard(m, [](ut_vecenv* v, size_t) -> int { return ut_vecenv_refresh_outputs(v); });
}

int ut_multienv_set_auto_reset(ut_multienv* m, int on) {
  return each_shard(m, [&](ut_vecenv* v, size_t) -> int { return ut_vecenv_set_auto_reset(v, on); });
}

int ut_multienv_synchronize(ut_multienv* m) {
  return each_shard(m, [](ut_vecenv* v, size_t) -> int { return ut_vecenv_synchronize(v); });
}

// The whole batch in the reference's layout (vecenv.hpp:51-62): per-env arrays
// are shard-contiguous; the column-major matrices take one 2-D copy per shard
// (each column's shard rows land at the shard's row offset). Every device's copies
// are enqueued before the handle waits.
int ut_multienv_copy_outputs(ut_multienv* m, const ut_host_outputs* d) {
  const int64_t A = m->A, T = m->T, R = m->R, E = m->n_envs;
  const int64_t obs_rows = E * A * R, glob_rows = E * R;
  int rc = each_shard(m, [&](ut_vecenv* v, size_t i) -> int {
    const DevBatch& B = v->B;
    const int64_t b = m->begin[i], n = v->n_envs;
    cudaStream_t s = v->stream;
    auto cp = [&](void* dst, size_t dst_off, const void* src, size_t bytes) -> cudaError_t {
      if (!dst) return cudaSuccess;
      return cudaMemcpyAsync(static_cast<char*>(dst) + dst_off, src, bytes, cudaMemcpyDeviceToHost, s);
    };
    auto cp_cols = [&](double* dst, int64_t rows_total, int64_t row0, const double* src, int64_t rows) -> cudaError_t {
      if (!dst) return cudaSuccess;
      return cudaMemcpy2DAsync(dst + row0, sizeof(double) * rows_total, src, sizeof(double) * rows,
                               sizeof(double) * rows, UT_FEATURE_DIM, cudaMemcpyDeviceToHost, s);
    };
    UT_CUDA(cp_cols(d->obs, obs_rows, b * A * R, B.obs, n * A * R));
    UT_CUDA(cp_cols(d->final_obs, obs_rows, b * A * R, B.final_obs, n * A * R));
    UT_CUDA(cp_cols(d->global_state, glob_rows, b * R, B.global, n * R));
    UT_CUDA(cp(d->rewards, sizeof(double) * b, B.rewards, sizeof(double) * n));
    UT_CUDA(cp(d->dones, (size_t)b, B.dones, (size_t)n));
    UT_CUDA(cp(d->masks, (size_t)(b * A * 5), B.masks, (size_t)(n * A * 5)));
    UT_CUDA(cp(d->tracking_error, sizeof(double) * b * T, B.track_err, sizeof(double) * n * T));
    UT_CUDA(cp(d->min_agent_dist, sizeof(double) * b * T, B.min_dist, sizeof(double) * n * T));
    UT_CUDA(cp(d->target_lost, (size_t)(b * T), B.lost, (size_t)(n * T)));
    UT_CUDA(cp(d->collision, (size_t)b, B.collision, (size_t)n));
    UT_CUDA(cp(d->step, sizeof(int32_t) * b, B.step, sizeof(int32_t) * n));
    return UT_OK;
  });
  if (rc) return rc;
  return ut_multienv_synchronize(m);
}

// Each shard reduces its statistics into its device vector; the vectors are then
// all-reduced over NCCL (every device ends with the batch totals, and shard 0's
// copy is returned), or summed on the host in shard order (UT_MULTI_STATS_HOST).
int ut_multienv_stats(ut_multienv* m, double out[UT_N_STATS], int reset) {
  int rc = each_shard(m, [&](ut_vecenv* v, size_t i) -> int {
    stats_kernel<<<1, 256, 0, v->stream>>>(v->B, m->d_stats[i], reset);
    ++v->launches;
    UT_CUDA(cudaGetLastError());
    return UT_OK;
  });
  if (rc) return rc;
  if (m->stats_backend == UT_MULTI_STATS_NCCL) {
    const NcclApi& api = nccl_api();
    UT_NCCL(api, api.group_start());
    for (size_t i = 0; i < m->shards.size(); ++i) {
      DeviceGuard dg(m->devices[i]);
      const ncclResult_t r =
          api.all_reduce(m->d_stats[i], m->d_stats[i], UT_N_STATS, ncclFloat64, ncclSum, m->comms[i], m->shards[i]->stream);
      if (r != ncclSuccess) {
        api.group_end();
        return fail(UT_ERR_RUNTIME, "ncclAllReduce failed: %s", api.error_string(r));
      }
    }
    UT_NCCL(api, api.group_end());
    DeviceGuard dg(m->devices[0]);
    UT_CUDA(cudaMemcpyAsync(out, m->d_stats[0], sizeof(double) * UT_N_STATS, cudaMemcpyDeviceToHost,
                            m->shards[0]->stream));
    return ut_multienv_synchronize(m);
  }
  for (int k = 0; k < UT_N_STATS; ++k) out[k] = 0.0;
  return each_shard(m, [&](ut_vecenv* v, size_t i) -> int {
    double h[UT_N_STATS];
    UT_CUDA(cudaMemcpyAsync(h, m->d_stats[i], sizeof h, cudaMemcpyDeviceToHost, v->stream));
    UT_CUDA(cudaStreamSynchronize(v->stream));
    for (int k = 0; k < UT_N_STATS; ++k) out[k] += h[k];
    return UT_OK;
  });
}

int ut_multienv_enable_phase_timing(ut_multienv* m, int on) {
  return each_shard(m, [&](ut_vecenv* v, size_t) -> int { return ut_vecenv_enable_phase_timing(v, on); });
}

// BenchmarkReport::phase_ns over the whole batch: the shards' CTA-summed
// phase times added (the reference adds every env's timers, vecenv.cpp:160-173).
int ut_multienv_phase_ns(ut_multienv* m, uint64_t out[UT_N_PHASES], int reset) {
  for (int k = 0; k < UT_N_PHASES; ++k) out[k] = 0;
  return each_shard(m, [&](ut_vecenv* v, size_t) -> int {
    uint64_t p[UT_N_PHASES];
    const int rc = ut_vecenv_phase_ns(v, p, reset);
    for (int k = 0; k < UT_N_PHASES; ++k) out[k] += p[k];
    return rc;
  });
}

int64_t ut_multienv_launch_count(const ut_multienv* m) {
  int64_t n = 0;
  for (const ut_vecenv* v : m->shards) n += v->launches;
  return n;
}

int ut_multienv_serialize(ut_multienv* m, int64_t env, double* blob, size_t cap, size_t* len) {
  ut_vecenv* v;
  int64_t e;
  int rc;
  if ((rc = ut_multienv_locate(m, env, &v, &e))) return rc;
  return ut_env_serialize(v, e, blob, cap, len);
}

int ut_multienv_deserialize(ut_multienv* m, int64_t env, const double* blob, size_t len) {
  ut_vecenv* v;
  int64_t e;
  int rc;
  if ((rc = ut_multienv_locate(m, env, &v, &e))) return rc;
  return ut_env_deserialize(v, e, blob, len);
}

int ut_multienv_world_step(ut_multienv* m, int64_t env, int32_t* step) {
  ut_vecenv* v;
  int64_t e;
  int rc;
  if ((rc = ut_multienv_locate(m, env, &v, &e))) return rc;
  return ut_env_world_step(v, e, step);
}

int ut_nccl_version(int* version) {
  const NcclApi& api = nccl_api();
  if (!api.ok) return fail(UT_ERR_RUNTIME, "%s", api.why.c_str());
  UT_NCCL(api, api.get_version(version));
  return UT_OK;
}

}  // extern "C"
