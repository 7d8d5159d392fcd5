// ut_capi.cu -- host side of the C-ABI (include/ut_env.h): device memory, launch
// configuration and the reference's VecEnv/Environment semantics around the
// fused step kernel. No CPU fallback: every state transition runs on the GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "ut_env.h"
#include "ut_kernels.cuh"
#include "ut_blob.cuh"

using namespace ut;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

// Scoped current device: every entry point runs on the handle's device and
// leaves the calling thread's current device as it found it.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

#define UT_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t err_ = (call);                                                            \
    if (err_ != cudaSuccess)                                                              \
      return fail(UT_ERR_RUNTIME, "%s failed: %s", #call, cudaGetErrorString(err_));      \
  } while (0)

// ------------------------------------------------------------ config ---
// Default heading bucket: OLS over the shipped synthetic calibration rows of
// (speed, dt) (kinematics.cpp:58-111 fit, :131-154 synth, :119 oracle, :180-186).
// Compiled with -ffp-contract=off like the oracle, so (a, b) are bit-identical.
bool default_bucket(double speed, double dt, double* a_out, double* b_out) {
  static const double speeds[] = {0.5, 0.75, 1.0, 1.25, 1.5, 2.0};
  static const double dts[] = {10.0, 15.0, 30.0, 60.0};
  if (std::find(std::begin(speeds), std::end(speeds), speed) == std::end(speeds)) return false;
  if (std::find(std::begin(dts), std::end(dts), dt) == std::end(dts)) return false;
  constexpr int kRows = 201;
  constexpr double kMax = 0.24, kGain = 0.15;
  double sx = 0.0, sy = 0.0, sxx = 0.0, sxy = 0.0;
  for (int i = 0; i < kRows; ++i) {
    const double t = static_cast<double>(i) / (kRows - 1);
    const double gamma = -kMax + 2.0 * kMax * t;
    const double dpsi = kGain * speed * dt * std::tan(gamma) + 0.0;
    sx += gamma;
    sy += dpsi;
    sxx += gamma * gamma;
    sxy += gamma * dpsi;
  }
  const double n = kRows;
  const double denom = n * sxx - sx * sx;
  *a_out = (n * sxy - sx * sy) / denom;
  *b_out = (sy - *a_out * sx) / n;
  return true;
}

DevConfig to_dev(const ut_env_config& c, int sA, int sT) {
  DevConfig d{};
  d.A = c.n_agents;
  d.T = c.n_targets;
  d.P = c.pf.n_particles;
  d.horizon = c.horizon;
  d.reward_mode = c.reward_mode;
  d.lost_steps = c.lost_steps;
  d.noise_on = (c.pf.process_noise_pos > 0.0 || c.pf.process_noise_vel > 0.0) ? 1 : 0;
  d.dt = c.dt;
  d.agent_speed = c.agent_speed;
  d.tgt_lo = c.agent_speed * c.target_speed_frac;  // env_config.hpp:85-88
  d.tgt_hi = c.agent_speed * std::max(c.target_speed_frac, c.target_speed_frac_max);
  d.turn_interval = c.target_turn_interval;
  d.det_range = c.detection_range;
  d.comm_range = c.comm_range;
  d.drop = c.comm_drop_prob;
  d.range_noise = c.range_noise_std;
  d.sigma_meas = std::max(c.range_noise_std, 0.1);  // env.cpp:340
  d.eps_min = c.eps_min;
  d.eps_max = c.eps_max;
  d.d_min = c.d_min;
  d.d_safe = c.d_safe;
  d.min_sep = c.spawn_min_sep;
  d.disc_r = c.spawn_max_sep / 2.0;
  d.pert_std = c.perturbation_std;
  d.depth_min = c.target_depth_min;
  d.depth_max = c.target_depth_max;
  d.pn = c.pf.process_noise_pos;
  d.vn = c.pf.process_noise_vel;
  d.speed_margin = c.pf.speed_margin;
  d.init_radius = c.pf.init_radius;
  d.inv_P = 1.0 / (double)c.pf.n_particles;
  d.head_a = c.heading_a;
  d.head_b = c.heading_b;
  d.head_noise = c.heading_noise_std;
  d.max_turn = c.max_turn_per_step;
  layout_config(d, sA, sT);
  return d;
}

#ifndef UT_PPT
#define UT_PPT 4
#endif
constexpr int kPPT = UT_PPT;          // particles per thread
constexpr int kMaxParticles = 1024;  // 1024 / kPPT threads x kPPT particles per CTA

int threads_for(int P) {
  int nt = (P + kPPT - 1) / kPPT;
  nt = (nt + 31) / 32 * 32;
  return std::max(32, nt);
}

}  // namespace

struct ut_vecenv {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  int64_t n_envs = 0;
  int64_t offset = 0;
  uint64_t seed = 0;
  std::vector<ut_env_config> cfgs;
  std::vector<DevConfig> dcfgs;
  std::vector<int32_t> cfg_of_env;  // empty: homogeneous
  std::vector<int64_t> set_off;
  int64_t total_sets = 0;
  int A_max = 0, T_max = 0, R_max = 0, P = 0, rec_words = 0;
  int nt = 0, grid = 0, grid_max = 0;
  size_t smem = 0;
  DevBatch B{};
  std::vector<void*> allocs;
  int32_t* d_status = nullptr;  // [0] status, [1] error_env
  int32_t* h_status = nullptr;  // pinned
  unsigned long long* phase_buf = nullptr;
  int64_t launches = 0;

  ~ut_vecenv() {
    if (stream) cudaStreamSynchronize(stream);
    for (cudaEvent_t ev : {copy_done[0], copy_done[1], step_done, order_ev})
      if (ev) cudaEventDestroy(ev);
    for (void* p : allocs) cudaFree(p);
    if (h_status) cudaFreeHost(h_status);
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (own_stream) cudaStreamDestroy(own_stream);
  }

  template <class T>
  int alloc(T** out, size_t count) {
    void* p = nullptr;
    const cudaError_t err = cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(T));
    if (err != cudaSuccess)
      return fail(UT_ERR_RUNTIME, "cudaMalloc(%zu bytes) failed: %s", count * sizeof(T), cudaGetErrorString(err));
    allocs.push_back(p);
    *out = static_cast<T*>(p);
    return UT_OK;
  }

  const DevConfig& cfg(int64_t e) const { return dcfgs[cfg_of_env.empty() ? 0 : cfg_of_env[(size_t)e]]; }
  int64_t set_at(int64_t e) const { return set_off[(size_t)e]; }

  // One env's record column <-> host vector (rec[w * n_envs + e]).
  int get_rec(int64_t e, std::vector<double>& out) {
    out.resize((size_t)rec_words);
    UT_CUDA(cudaStreamSynchronize(stream));
    UT_CUDA(cudaMemcpy2D(out.data(), sizeof(double), B.rec + e, sizeof(double) * n_envs, sizeof(double), rec_words,
                         cudaMemcpyDeviceToHost));
    return UT_OK;
  }
  int put_rec(int64_t e, const std::vector<double>& in) {
    UT_CUDA(cudaStreamSynchronize(stream));
    UT_CUDA(cudaMemcpy2D(B.rec + e, sizeof(double) * n_envs, in.data(), sizeof(double), sizeof(double), rec_words,
                         cudaMemcpyHostToDevice));
    return UT_OK;
  }

  int check_status(const char* what) {
    int rc;
    if ((rc = enqueue_status())) return rc;
    return finish_status(what);
  }
  // The two halves of check_status, so a multi-device handle can have every
  // device's work in flight before it waits on any of them.
  int enqueue_status() {
    UT_CUDA(cudaMemcpyAsync(h_status, d_status, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
    return UT_OK;
  }
  int finish_status(const char* what) {
    UT_CUDA(cudaStreamSynchronize(stream));
    UT_CUDA(cudaGetLastError());
    if (h_status[0] == ST_SPAWN_INFEASIBLE) {
      const ut_env_config& c = cfgs[0];
      return fail(UT_ERR_CONFIG, "%s: spawn infeasible after 1000 attempts: %d entities with separation in [%g, %g] m",
                  what, c.n_agents + c.n_targets, c.spawn_min_sep, c.spawn_max_sep);
    }
    return UT_OK;
  }

  int reset_status() {
    const int32_t init[2] = {0, INT_MAX};
    UT_CUDA(cudaMemcpyAsync(d_status, init, sizeof init, cudaMemcpyHostToDevice, stream));
    return UT_OK;
  }

  DevBatch* d_self = nullptr;  // device copy of B for the kernels' cold paths
  bool full = false;           // P == nt * kPPT: TMA-prefetched register-tile path

  // Publishes B to its device copy; call after any change to B.
  int sync_batch() {
    ++batch_version;  // B is a kernel parameter: captured step graphs are stale now
    B.self = d_self;
    UT_CUDA(cudaMemcpyAsync(d_self, &B, sizeof(DevBatch), cudaMemcpyHostToDevice, stream));
    return UT_OK;
  }

  int np = 1024;              // particle capacity of the step kernel instance
  size_t smem_reset = 0;      // the reset kernel always uses the 1024 layout

  int nt_reset = 0;

  // Output double buffering (ut_vecenv_set_output_buffers): every step writes the
  // set the previous step did not, after any asynchronous copy still reading it
  // (ut_vecenv_copy_outputs_async) has finished. final_obs is double-buffered
  // too: a step only writes the rows of finished envs, so the set it writes is
  // first brought up to date from the previous one.
  struct OutSet {
    double *obs = nullptr, *final_obs = nullptr, *global = nullptr, *rewards = nullptr, *track_err = nullptr,
           *min_dist = nullptr;
    uint8_t *dones = nullptr, *masks = nullptr, *lost = nullptr, *collision = nullptr;
    int32_t* step = nullptr;
  };
  OutSet out[2];
  int n_out = 1, cur = 0;
  cudaEvent_t copy_done[2] = {nullptr, nullptr};
  cudaEvent_t step_done = nullptr;
  cudaEvent_t order_ev = nullptr;  // ut_vecenv_wait_stream

  void bind_outputs(int k) {
    const OutSet& o = out[k];
    B.obs = o.obs, B.final_obs = o.final_obs, B.global = o.global, B.rewards = o.rewards, B.track_err = o.track_err;
    B.min_dist = o.min_dist, B.dones = o.dones, B.masks = o.masks, B.lost = o.lost;
    B.collision = o.collision, B.step = o.step;
    B.prev_final_obs = n_out == 2 ? out[k ^ 1].final_obs : nullptr;
    B.prev_dones = n_out == 2 ? out[k ^ 1].dones : nullptr;
  }
  // before a kernel writes the output set k
  int wait_outputs(int k) {
    if (copy_done[k]) UT_CUDA(cudaStreamWaitEvent(stream, copy_done[k], 0));
    return UT_OK;
  }

  // Multi-step step_policy as one CUDA graph of n cooperative step launches
  // (launch-bound small batches such as C1: one graph launch instead of n
  // kernel launches). The graph is captured on a private stream, launched on the
  // handle's stream (which may be the legacy default stream, where capture is
  // not allowed), and re-captured whenever B, the grid or (mode, n) change.
  uint64_t batch_version = 0;
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  int graph_mode = -1, graph_n = 0, graph_grid = 0;
  uint64_t graph_version = 0;
  bool graphs_off = getenv("UT_NO_GRAPHS") != nullptr;

  int launch_kernel(int mode, cudaStream_t s) {
    void (*kern)(DevBatch, int, int32_t*) = nullptr;
    if (full && np == 1024)
      kern = step_kernel<kPPT, 1024, true>;
    else if (full && np == 512)
      kern = step_kernel<kPPT, 512, true>;
    else if (full && np == 256)
      kern = step_kernel<kPPT, 256, true>;
    else
      kern = step_kernel<kPPT, 1024, false>;
    // cooperative: the kernel's phases are separated by grid-wide barriers
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)grid);
    lc.blockDim = dim3((unsigned)nt);
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    UT_CUDA(cudaLaunchKernelEx(&lc, kern, B, mode, d_status));
    UT_CUDA(cudaGetLastError());
    return UT_OK;
  }

  // n_steps policy steps; true in *used when they went out as one graph launch
  int launch_steps_graph(int mode, int n_steps, bool* used) {
    *used = false;
    if (graphs_off || n_out != 1 || n_steps < 2) return UT_OK;
    if (!graph_exec || graph_mode != mode || graph_n != n_steps || graph_grid != grid ||
        graph_version != batch_version) {
      if (graph_exec) cudaGraphExecDestroy(graph_exec);
      graph_exec = nullptr;
      if (!cap_stream) UT_CUDA(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
      UT_CUDA(cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeThreadLocal));
      int rc = UT_OK;
      for (int i = 0; i < n_steps && !rc; ++i) rc = launch_kernel(mode, cap_stream);
      cudaGraph_t g = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(cap_stream, &g);
      if (rc || ce != cudaSuccess || !g) {
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        graphs_off = true;  // capture unsupported here: plain launches from now on
        return UT_OK;
      }
      const cudaError_t ie = cudaGraphInstantiate(&graph_exec, g, 0);
      cudaGraphDestroy(g);
      if (ie != cudaSuccess) {
        cudaGetLastError();
        graph_exec = nullptr;
        graphs_off = true;
        return UT_OK;
      }
      graph_mode = mode, graph_n = n_steps, graph_grid = grid, graph_version = batch_version;
    }
    int rc;
    if ((rc = wait_outputs(cur))) return rc;
    UT_CUDA(cudaGraphLaunch(graph_exec, stream));
    launches += n_steps;
    *used = true;
    return UT_OK;
  }

  // n_steps policy steps back to back: one graph launch, else n kernel launches
  int enqueue_policy_steps(int mode, int n_steps) {
    bool graphed = false;
    int rc;
    if ((rc = launch_steps_graph(mode, n_steps, &graphed))) return rc;
    for (int i = 0; i < n_steps && !graphed; ++i)
      if ((rc = launch_step(mode))) return rc;
    return UT_OK;
  }

  int launch_step(int mode) {
    int rc;
    if (n_out == 2) {
      const int t = cur ^ 1;
      if ((rc = wait_outputs(t))) return rc;
      bind_outputs(t);  // the kernel brings set t's final_obs up to date (copy_final_rows)
      cur = t;
      if ((rc = sync_batch())) return rc;
    } else if ((rc = wait_outputs(cur))) {
      return rc;
    }
    if ((rc = launch_kernel(mode, stream))) return rc;
    ++launches;
    return UT_OK;
  }
  int launch_reset(int ctor) {
    int rc;
    if ((rc = wait_outputs(cur))) return rc;
    reset_kernel<kPPT, 1024><<<(unsigned)grid, nt_reset, smem_reset, stream>>>(B, ctor, d_status);
    ++launches;
    UT_CUDA(cudaGetLastError());
    return UT_OK;
  }
};

namespace {

int build(ut_vecenv* v, const ut_env_config* cfgs, int n_cfg, const int32_t* cfg_of_env, int64_t n_envs,
          uint64_t seed, int64_t offset, int device) {
  if (n_envs < 1) return fail(UT_ERR_CONFIG, "vecenv: n_envs must be >= 1");
  v->device = device;
  v->n_envs = n_envs;
  v->offset = offset;
  v->seed = seed;
  for (int i = 0; i < n_cfg; ++i) {
    ut_env_config c = cfgs[i];
    const int rc = ut_config_finalize(&c);
    if (rc) return rc;
    if (c.pf.n_particles > kMaxParticles)
      return fail(UT_ERR_CONFIG, "env.pf.n_particles must be <= %d on this device build", kMaxParticles);
    if (c.n_agents + c.n_targets > kMaxEntities)
      return fail(UT_ERR_CONFIG, "env.n_agents + env.n_targets must be <= %d on this device build", kMaxEntities);
    if (i > 0 && c.pf.n_particles != cfgs[0].pf.n_particles)
      return fail(UT_ERR_CONFIG, "mixed fleets must share env.pf.n_particles");
    v->cfgs.push_back(c);
    v->A_max = std::max(v->A_max, c.n_agents);
    v->T_max = std::max(v->T_max, c.n_targets);
    v->R_max = std::max(v->R_max, c.n_agents + c.n_targets);
  }
  for (const ut_env_config& c : v->cfgs) v->dcfgs.push_back(to_dev(c, v->A_max, v->T_max));
  v->rec_words = v->dcfgs[0].rec_words;
  if (cfg_of_env) {
    v->cfg_of_env.assign(cfg_of_env, cfg_of_env + n_envs);
    for (int32_t k : v->cfg_of_env)
      if (k < 0 || k >= n_cfg) return fail(UT_ERR_CONFIG, "cfg_of_env index %d out of range", k);
  }
  v->P = v->dcfgs[0].P;
  v->set_off.resize((size_t)n_envs);
  for (int64_t e = 0; e < n_envs; ++e) {
    const DevConfig& d = v->cfg(e);
    v->set_off[(size_t)e] = v->total_sets;
    v->total_sets += (int64_t)d.A * d.T;
  }
  // the step kernel indexes envs and particle sets in 32 bits
  if (v->total_sets >= ((int64_t)1 << 31) - 1)
    return fail(UT_ERR_CONFIG, "n_envs x agents x targets = %lld particle sets per device (max 2^31 - 2)",
                (long long)v->total_sets);

  DeviceGuard dg(device);
  UT_CUDA(cudaStreamCreateWithFlags(&v->own_stream, cudaStreamNonBlocking));
  v->stream = v->own_stream;
  UT_CUDA(cudaMallocHost(&v->h_status, 2 * sizeof(int32_t)));

  DevBatch& B = v->B;
  B.n_envs = n_envs;
  B.env_index_offset = offset;
  B.seed = seed;
  B.n_cfg = n_cfg;
  B.A_max = v->A_max;
  B.T_max = v->T_max;
  B.R_max = v->R_max;
  B.P = v->P;
  const int64_t P = v->P, Am = v->A_max, Rm = v->R_max, Tm = v->T_max;
  B.obs_rows = n_envs * Am * Rm;
  B.global_rows = n_envs * Rm;
  int rc;
  DevConfig* dc;
  if ((rc = v->alloc(&dc, v->dcfgs.size()))) return rc;
  UT_CUDA(cudaMemcpy(dc, v->dcfgs.data(), sizeof(DevConfig) * v->dcfgs.size(), cudaMemcpyHostToDevice));
  B.cfgs = dc;
  if (!v->cfg_of_env.empty()) {
    int32_t* ce;
    int64_t* so;
    if ((rc = v->alloc(&ce, (size_t)n_envs))) return rc;
    if ((rc = v->alloc(&so, (size_t)n_envs))) return rc;
    UT_CUDA(cudaMemcpy(ce, v->cfg_of_env.data(), sizeof(int32_t) * n_envs, cudaMemcpyHostToDevice));
    UT_CUDA(cudaMemcpy(so, v->set_off.data(), sizeof(int64_t) * n_envs, cudaMemcpyHostToDevice));
    B.cfg_of_env = ce;
    B.set_offset = so;
  }
  const size_t np = (size_t)(v->total_sets * P);
  if ((rc = v->alloc(&B.rec, (size_t)v->rec_words * (size_t)n_envs))) return rc;
  if ((rc = v->alloc(&B.sched_r2, (size_t)(n_envs * Am * Tm)))) return rc;
  if ((rc = v->alloc(&B.sched_flags, (size_t)(n_envs * (Am * Tm + Am * Am))))) return rc;
  if ((rc = v->alloc(&B.px, np))) return rc;
  if ((rc = v->alloc(&B.py, np))) return rc;
  if ((rc = v->alloc(&B.vx, np))) return rc;
  if ((rc = v->alloc(&B.vy, np))) return rc;
  if ((rc = v->alloc(&B.w, np))) return rc;
  if ((rc = v->alloc(&B.obs, (size_t)(12 * B.obs_rows)))) return rc;
  if ((rc = v->alloc(&B.final_obs, (size_t)(12 * B.obs_rows)))) return rc;
  if ((rc = v->alloc(&B.global, (size_t)(12 * B.global_rows)))) return rc;
  if ((rc = v->alloc(&B.rewards, (size_t)n_envs))) return rc;
  if ((rc = v->alloc(&B.dones, (size_t)n_envs))) return rc;
  if ((rc = v->alloc(&B.masks, (size_t)(n_envs * Am * 5)))) return rc;
  if ((rc = v->alloc(&B.track_err, (size_t)(n_envs * Tm)))) return rc;
  if ((rc = v->alloc(&B.min_dist, (size_t)(n_envs * Tm)))) return rc;
  if ((rc = v->alloc(&B.lost, (size_t)(n_envs * Tm)))) return rc;
  if ((rc = v->alloc(&B.collision, (size_t)n_envs))) return rc;
  if ((rc = v->alloc(&B.step, (size_t)n_envs))) return rc;
  v->out[0] = {B.obs, B.final_obs, B.global, B.rewards, B.track_err, B.min_dist,
               B.dones, B.masks, B.lost, B.collision, B.step};
  int32_t* acts;
  if ((rc = v->alloc(&acts, (size_t)(n_envs * Am)))) return rc;
  B.actions = acts;
  if ((rc = v->alloc(&v->d_status, 2))) return rc;
  B.error_env = v->d_status + 1;
  B.error_info = nullptr;
  B.force_exact = 0;
  B.trace_env = -1;
  B.traj = nullptr;
  B.traj_lo = B.traj_hi = 0;
  B.phase_cycles = nullptr;
  B.auto_reset = 1;
  // VecEnv ctor zero-fills every batch buffer (vecenv.cpp:26-38)
  UT_CUDA(cudaMemsetAsync(B.final_obs, 0, sizeof(double) * 12 * B.obs_rows, v->stream));
  UT_CUDA(cudaMemsetAsync(B.track_err, 0, sizeof(double) * n_envs * Tm, v->stream));
  UT_CUDA(cudaMemsetAsync(B.min_dist, 0, sizeof(double) * n_envs * Tm, v->stream));
  UT_CUDA(cudaMemsetAsync(B.lost, 0, n_envs * Tm, v->stream));
  UT_CUDA(cudaMemsetAsync(B.collision, 0, n_envs, v->stream));
  UT_CUDA(cudaMemsetAsync(acts, 0, sizeof(int32_t) * n_envs * Am, v->stream));
  UT_CUDA(cudaMemsetAsync(B.sched_flags, 0, n_envs * (Am * Tm + Am * Am), v->stream));

  v->nt = v->nt_reset = threads_for(v->P);
  int max_optin = 0, sms = 0;
  UT_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  UT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  // FULL instances: P == nt * PPT with a compile-time particle capacity
  // FULL instances also assume particle noise (every config of the batch has it):
  // noise-free configs (test scenarios) take the generic instance
  bool all_noise = true;
  for (const DevConfig& d : v->dcfgs) all_noise = all_noise && d.noise_on != 0;
  v->full = (v->P == v->nt * kPPT) && (v->P == 1024 || v->P == 512 || v->P == 256) && all_noise;
  v->np = v->full ? v->P : 1024;
  const void* fn = nullptr;
  if (v->np == 1024 && v->full) {
    fn = (const void*)step_kernel<kPPT, 1024, true>;
    v->smem = smem_bytes<1024>(v->A_max, v->T_max, v->nt);
  } else if (v->np == 512) {
    fn = (const void*)step_kernel<kPPT, 512, true>;
    v->smem = smem_bytes<512>(v->A_max, v->T_max, v->nt);
  } else if (v->np == 256) {
    fn = (const void*)step_kernel<kPPT, 256, true>;
    v->smem = smem_bytes<256>(v->A_max, v->T_max, v->nt);
  } else {
    fn = (const void*)step_kernel<kPPT, 1024, false>;
    v->smem = smem_bytes<1024>(v->A_max, v->T_max, v->nt);
  }
  v->smem_reset = smem_bytes<1024>(v->A_max, v->T_max, v->nt_reset);
  if ((int)v->smem_reset > max_optin)
    return fail(UT_ERR_CONFIG, "configuration needs %zu B of shared memory per CTA (max %d)", v->smem_reset, max_optin);
  UT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v->smem));
  UT_CUDA(cudaFuncSetAttribute((const void*)reset_kernel<kPPT, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)v->smem_reset));
  // persistent cooperative grid: every resident CTA slot (the step kernel's
  // phases are separated by grid barriers, so all CTAs must be co-resident)
  int per_sm = 0;
  UT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, v->nt, v->smem));
  if (per_sm < 1) return fail(UT_ERR_RUNTIME, "step kernel cannot be resident with %zu B shared memory", v->smem);
  // debug knob (occupancy experiments): cap resident CTAs per SM
  if (const char* cap = getenv("UT_DEBUG_CTAS_PER_SM")) per_sm = std::max(1, std::min(per_sm, atoi(cap)));
  v->grid = (int)std::min<int64_t>(n_envs, (int64_t)per_sm * sms);
  v->grid_max = v->grid;
  if ((rc = v->alloc(&B.work, 1))) return rc;
  UT_CUDA(cudaMemsetAsync(B.work, 0, sizeof(int), v->stream));
  if ((rc = v->alloc(&v->d_self, 1))) return rc;
  if ((rc = v->sync_batch())) return rc;

  // Environment ctors: pf::init draws, then spawn (env.cpp:110-151)
  if ((rc = v->reset_status())) return rc;
  if ((rc = v->launch_reset(1))) return rc;
  return v->check_status("vecenv ctor");
}

int finish_create(ut_vecenv* v, int rc, ut_vecenv** out) {
  if (rc) {
    const std::string msg = g_err;
    delete v;
    g_err = msg;
    return rc;
  }
  *out = v;
  return UT_OK;
}

}  // namespace

extern "C" {

int ut_abi_version(void) { return UT_ABI_VERSION; }
const char* ut_last_error(void) { return g_err.c_str(); }

void ut_config_default(ut_env_config* c) {
  std::memset(c, 0, sizeof *c);
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

int ut_config_finalize(ut_env_config* c) {
  if (c->heading_noise_std < 0.0) return fail(UT_ERR_CONFIG, "heading model noise_std must be >= 0");
  if (c->n_agents < 1) return fail(UT_ERR_CONFIG, "env.n_agents must be >= 1");
  if (c->n_targets < 1) return fail(UT_ERR_CONFIG, "env.n_targets must be >= 1");
  if (c->horizon < 1) return fail(UT_ERR_CONFIG, "env.horizon must be >= 1");
  if (!(c->dt > 0.0)) return fail(UT_ERR_CONFIG, "env.dt must be > 0");
  if (!(c->agent_speed > 0.0)) return fail(UT_ERR_CONFIG, "env.agent_speed must be > 0");
  if (c->target_speed_frac < 0.0) return fail(UT_ERR_CONFIG, "env.target_speed_frac must be >= 0");
  if (c->target_turn_interval < 1.0) return fail(UT_ERR_CONFIG, "env.target_turn_interval must be >= 1 step");
  if (c->eps_min >= c->eps_max) return fail(UT_ERR_CONFIG, "env.eps_min must be < env.eps_max");
  if (c->spawn_min_sep >= c->spawn_max_sep)
    return fail(UT_ERR_CONFIG, "env.spawn_min_sep must be < env.spawn_max_sep");
  if (c->comm_drop_prob < 0.0 || c->comm_drop_prob > 1.0)
    return fail(UT_ERR_CONFIG, "env.comm_drop_prob must be in [0, 1]");
  if (c->range_noise_std < 0.0) return fail(UT_ERR_CONFIG, "env.range_noise_std must be >= 0");
  if (c->target_depth_min < 0.0 || c->target_depth_max < c->target_depth_min)
    return fail(UT_ERR_CONFIG, "env.target_depth band must satisfy 0 <= min <= max");
  if (c->lost_steps < 1) return fail(UT_ERR_CONFIG, "env.lost_steps must be >= 1");
  if (c->pf.n_particles < 1) return fail(UT_ERR_CONFIG, "env.pf.n_particles must be >= 1");
  if (!(c->pf.init_radius > 0.0)) return fail(UT_ERR_CONFIG, "env.pf.init_radius must be > 0");
  if (c->heading_model_kind == UT_HEADING_DEFAULT) {
    double a, b;
    if (!default_bucket(c->agent_speed, c->dt, &a, &b))
      return fail(UT_ERR_CONFIG, "heading model has no bucket for (speed=%g m/s, dt=%g s)", c->agent_speed, c->dt);
    c->heading_a = a;
    c->heading_b = b;
  } else if (c->heading_model_kind != UT_HEADING_BUCKET) {
    return fail(UT_ERR_CONFIG, "env.heading_model_kind must be 0 (default) or 1 (bucket)");
  }
  c->max_turn_per_step = std::fabs(c->heading_a * 0.24 + c->heading_b);  // env.cpp:115-116
  return UT_OK;
}

int ut_vecenv_create(const ut_env_config* cfg, int64_t n_envs, uint64_t master_seed, int64_t env_index_offset,
                     int device, ut_vecenv** out) {
  *out = nullptr;
  auto* v = new ut_vecenv();
  return finish_create(v, build(v, cfg, 1, nullptr, n_envs, master_seed, env_index_offset, device), out);
}

int ut_vecenv_create_mixed(const ut_env_config* cfgs, int32_t n_cfgs, const int32_t* cfg_of_env, int64_t n_envs,
                           uint64_t master_seed, int64_t env_index_offset, int device, ut_vecenv** out) {
  *out = nullptr;
  if (n_cfgs < 1 || !cfg_of_env) return fail(UT_ERR_CONFIG, "mixed vecenv needs >= 1 config and a cfg_of_env map");
  auto* v = new ut_vecenv();
  return finish_create(v, build(v, cfgs, n_cfgs, cfg_of_env, n_envs, master_seed, env_index_offset, device), out);
}

void ut_vecenv_destroy(ut_vecenv* v) {
  if (!v) return;
  DeviceGuard dg(v->device);
  delete v;
}

int ut_vecenv_reset_all(ut_vecenv* v) {
  DeviceGuard dg(v->device);
  int rc;
  if ((rc = v->reset_status()) || (rc = v->launch_reset(0))) return rc;
  return v->check_status("reset_all");
}

namespace {
// First half of VecEnv::step (vecenv.cpp:79-93): stage the actions and validate
// every env's actions on the device; nothing is mutated. The result is read by
// validate_result() once the stream has reached it.
int enqueue_validate(ut_vecenv* v, const int32_t* actions, int actions_on_device, bool with_status = true) {
  const size_t n = (size_t)(v->n_envs * v->A_max);
  UT_CUDA(cudaMemcpyAsync(const_cast<int32_t*>(v->B.actions), actions, n * sizeof(int32_t),
                          actions_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, v->stream));
  int rc;
  if ((rc = v->reset_status())) return rc;
  const int tpb = 256;
  validate_kernel<<<(unsigned)((v->n_envs + tpb - 1) / tpb), tpb, 0, v->stream>>>(v->B);
  ++v->launches;
  UT_CUDA(cudaGetLastError());
  return with_status ? v->enqueue_status() : UT_OK;
}

// UT_ERR_CONTRACT for the lowest env whose action failed validation, its index
// shown as `shown_base + e` (the global index for a shard of a multi-device
// handle); message format of env.cpp:241-246 prefixed like vecenv.cpp:88-93.
int validate_error(ut_vecenv* v, int64_t e, int64_t shown_base) {
  const long long shown = (long long)(shown_base + e);
  std::vector<int32_t> acts((size_t)v->A_max);
  UT_CUDA(cudaMemcpy(acts.data(), v->B.actions + e * v->A_max, sizeof(int32_t) * v->A_max, cudaMemcpyDeviceToHost));
  std::vector<double> rec;
  int rc;
  if ((rc = v->get_rec(e, rec))) return rc;
  const DevConfig& d = v->cfg(e);
  for (int a = 0; a < d.A; ++a) {
    const int act = acts[(size_t)a], r = (int)rec[(size_t)(d.o_agent + V_RUDDER * d.sA + a)];
    if (act < 0 || act >= UT_NUM_ACTIONS || std::abs(act - r) > 1)
      return fail(UT_ERR_CONTRACT, "env %lld: step: invalid action %d for agent %d at rudder index %d", shown, act, a,
                  r);
  }
  return fail(UT_ERR_CONTRACT, "env %lld: step: invalid action", shown);
}
int validate_result(ut_vecenv* v, int64_t shown_base) {
  UT_CUDA(cudaStreamSynchronize(v->stream));
  if (v->h_status[1] == INT_MAX) return UT_OK;
  return validate_error(v, v->h_status[1], shown_base);
}
}  // namespace

int ut_vecenv_step(ut_vecenv* v, const int32_t* actions, int actions_on_device) {
  DeviceGuard dg(v->device);
  // The step kernel itself is gated on the validation result (it returns before
  // touching anything when an action failed), so validation and step go out
  // together and the host waits once: no round trip between them, whose status
  // copy would also queue behind a caller's asynchronous output copies still
  // draining from the previous step.
  int rc;
  if ((rc = enqueue_validate(v, actions, actions_on_device, false))) return rc;
  const int prev_cur = v->cur;
  if ((rc = v->launch_step(MODE_EXTERNAL)) || (rc = v->enqueue_status())) return rc;
  UT_CUDA(cudaStreamSynchronize(v->stream));
  if (v->h_status[1] != INT_MAX) {  // nothing moved: undo the output-set switch
    if (v->cur != prev_cur) {
      v->cur = prev_cur;
      v->bind_outputs(prev_cur);
      if ((rc = v->sync_batch())) return rc;
    }
    return validate_error(v, v->h_status[1], 0);
  }
  return v->finish_status("step");
}

int ut_vecenv_step_policy(ut_vecenv* v, int policy, int n_steps) {
  DeviceGuard dg(v->device);
  if (policy != UT_POLICY_RANDOM && policy != UT_POLICY_SCRIPTED)
    return fail(UT_ERR_CONTRACT, "step_policy: unknown policy %d", policy);
  int rc;
  if ((rc = v->reset_status())) return rc;
  if ((rc = v->enqueue_policy_steps(policy == UT_POLICY_RANDOM ? MODE_RANDOM : MODE_SCRIPTED, n_steps))) return rc;
  return v->check_status("step_policy");
}

int ut_vecenv_refresh_outputs(ut_vecenv* v) {
  DeviceGuard dg(v->device);
  int sms = 0, rc;
  UT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, v->device));
  if ((rc = v->wait_outputs(v->cur))) return rc;
  tokens_kernel<<<(unsigned)(sms * 8), 256, 0, v->stream>>>(v->B);
  ++v->launches;
  UT_CUDA(cudaGetLastError());
  UT_CUDA(cudaStreamSynchronize(v->stream));
  return UT_OK;
}

int ut_vecenv_set_output_buffers(ut_vecenv* v, int n) {
  DeviceGuard dg(v->device);
  if (n != 1 && n != 2) return fail(UT_ERR_CONTRACT, "set_output_buffers: n must be 1 or 2");
  if (n == v->n_out) return UT_OK;
  UT_CUDA(cudaStreamSynchronize(v->stream));
  for (cudaEvent_t ev : {v->copy_done[0], v->copy_done[1]})
    if (ev) UT_CUDA(cudaEventSynchronize(ev));
  if (n == 2 && !v->out[1].obs) {
    const int64_t E = v->n_envs, Am = v->A_max, Tm = v->T_max;
    ut_vecenv::OutSet& o = v->out[1];
    int rc;
    if ((rc = v->alloc(&o.obs, (size_t)(12 * v->B.obs_rows))) || (rc = v->alloc(&o.final_obs, (size_t)(12 * v->B.obs_rows))) ||
        (rc = v->alloc(&o.global, (size_t)(12 * v->B.global_rows))) ||
        (rc = v->alloc(&o.rewards, (size_t)E)) || (rc = v->alloc(&o.dones, (size_t)E)) ||
        (rc = v->alloc(&o.masks, (size_t)(E * Am * 5))) || (rc = v->alloc(&o.track_err, (size_t)(E * Tm))) ||
        (rc = v->alloc(&o.min_dist, (size_t)(E * Tm))) || (rc = v->alloc(&o.lost, (size_t)(E * Tm))) ||
        (rc = v->alloc(&o.collision, (size_t)E)) || (rc = v->alloc(&o.step, (size_t)E)))
      return rc;
    UT_CUDA(cudaMemsetAsync(o.dones, 0, (size_t)E, v->stream));
  }
  if (n == 2) {  // both sets start with every terminal row so far (copy_final_rows keeps them so)
    const ut_vecenv::OutSet &a = v->out[v->cur], &b = v->out[v->cur ^ 1];
    UT_CUDA(cudaMemcpyAsync(b.final_obs, a.final_obs, sizeof(double) * 12 * v->B.obs_rows, cudaMemcpyDeviceToDevice,
                            v->stream));
    UT_CUDA(cudaMemcpyAsync(b.dones, a.dones, (size_t)v->n_envs, cudaMemcpyDeviceToDevice, v->stream));
  }
  if (n == 1 && v->cur == 1) {  // keep the current outputs in set 0
    const ut_vecenv::OutSet &a = v->out[0], &b = v->out[1];
    const int64_t E = v->n_envs, Am = v->A_max, Tm = v->T_max;
    auto cp = [&](void* d, const void* s2, size_t bytes) { return cudaMemcpyAsync(d, s2, bytes, cudaMemcpyDeviceToDevice, v->stream); };
    UT_CUDA(cp(a.obs, b.obs, sizeof(double) * 12 * v->B.obs_rows));
    UT_CUDA(cp(a.final_obs, b.final_obs, sizeof(double) * 12 * v->B.obs_rows));
    UT_CUDA(cp(a.global, b.global, sizeof(double) * 12 * v->B.global_rows));
    UT_CUDA(cp(a.rewards, b.rewards, sizeof(double) * E));
    UT_CUDA(cp(a.dones, b.dones, (size_t)E));
    UT_CUDA(cp(a.masks, b.masks, (size_t)(E * Am * 5)));
    UT_CUDA(cp(a.track_err, b.track_err, sizeof(double) * E * Tm));
    UT_CUDA(cp(a.min_dist, b.min_dist, sizeof(double) * E * Tm));
    UT_CUDA(cp(a.lost, b.lost, (size_t)(E * Tm)));
    UT_CUDA(cp(a.collision, b.collision, (size_t)E));
    UT_CUDA(cp(a.step, b.step, sizeof(int32_t) * E));
    v->cur = 0;
    v->bind_outputs(0);
    int rc;
    if ((rc = v->sync_batch())) return rc;
    UT_CUDA(cudaStreamSynchronize(v->stream));
  }
  v->n_out = n;
  v->bind_outputs(v->cur);  // the other set's final_obs / dones (or none)
  return v->sync_batch();
}

int ut_vecenv_copy_outputs_async(ut_vecenv* v, const ut_host_outputs* d, void* cuda_stream) {
  DeviceGuard dg(v->device);
  cudaStream_t cs = static_cast<cudaStream_t>(cuda_stream);
  if (!v->step_done) UT_CUDA(cudaEventCreateWithFlags(&v->step_done, cudaEventDisableTiming));
  cudaEvent_t& done = v->copy_done[v->cur];
  if (!done) UT_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  UT_CUDA(cudaEventRecord(v->step_done, v->stream));
  UT_CUDA(cudaStreamWaitEvent(cs, v->step_done, 0));
  const DevBatch& B = v->B;
  const int64_t n = v->n_envs, Am = v->A_max, Tm = v->T_max;
  auto cp = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
    if (!dst) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, cs);
  };
  UT_CUDA(cp(d->obs, B.obs, sizeof(double) * 12 * B.obs_rows));
  UT_CUDA(cp(d->final_obs, B.final_obs, sizeof(double) * 12 * B.obs_rows));
  UT_CUDA(cp(d->global_state, B.global, sizeof(double) * 12 * B.global_rows));
  UT_CUDA(cp(d->rewards, B.rewards, sizeof(double) * n));
  UT_CUDA(cp(d->dones, B.dones, (size_t)n));
  UT_CUDA(cp(d->masks, B.masks, (size_t)(n * Am * 5)));
  UT_CUDA(cp(d->tracking_error, B.track_err, sizeof(double) * n * Tm));
  UT_CUDA(cp(d->min_agent_dist, B.min_dist, sizeof(double) * n * Tm));
  UT_CUDA(cp(d->target_lost, B.lost, (size_t)(n * Tm)));
  UT_CUDA(cp(d->collision, B.collision, (size_t)n));
  UT_CUDA(cp(d->step, B.step, sizeof(int32_t) * n));
  UT_CUDA(cudaEventRecord(done, cs));
  return UT_OK;
}

int ut_vecenv_capture_trajectory(ut_vecenv* v, int64_t env_begin, int64_t env_end) {
  DeviceGuard dg(v->device);
  if (env_begin < 0 || env_end > v->n_envs || env_begin > env_end)
    return fail(UT_ERR_CONTRACT, "capture_trajectory: env range [%lld, %lld) outside [0, %lld)",
                (long long)env_begin, (long long)env_end, (long long)v->n_envs);
  UT_CUDA(cudaStreamSynchronize(v->stream));
  if (v->B.traj) {
    cudaFree(v->B.traj);
    v->allocs.erase(std::remove(v->allocs.begin(), v->allocs.end(), (void*)v->B.traj), v->allocs.end());
    v->B.traj = nullptr;
  }
  v->B.traj_lo = env_begin;
  v->B.traj_hi = env_end;
  if (env_end > env_begin) {
    int rc;
    if ((rc = v->alloc(&v->B.traj, (size_t)((env_end - env_begin) * v->R_max * kTrajFields)))) return rc;
    UT_CUDA(cudaMemset(v->B.traj, 0, sizeof(double) * (env_end - env_begin) * v->R_max * kTrajFields));
  }
  return v->sync_batch();
}

int ut_vecenv_trajectory_rows(ut_vecenv* v, double* rows, size_t cap, size_t* len) {
  DeviceGuard dg(v->device);
  const size_t need = (size_t)((v->B.traj_hi - v->B.traj_lo) * v->R_max * kTrajFields);
  *len = need;
  if (!rows) return UT_OK;
  if (cap < need) return fail(UT_ERR_DATA, "trajectory_rows: buffer of %zu doubles too small (need %zu)", cap, need);
  if (need == 0) return UT_OK;
  UT_CUDA(cudaStreamSynchronize(v->stream));
  UT_CUDA(cudaMemcpy(rows, v->B.traj, need * sizeof(double), cudaMemcpyDeviceToHost));
  return UT_OK;
}

int ut_vecenv_buffers(ut_vecenv* v, ut_buffers* o) {
  DeviceGuard dg(v->device);
  const DevBatch& B = v->B;
  o->n_envs = v->n_envs;
  o->n_agents = v->A_max;
  o->n_targets = v->T_max;
  o->n_rows = v->R_max;
  o->n_particles = v->P;
  o->obs_rows = B.obs_rows;
  o->global_rows = B.global_rows;
  o->obs = B.obs;
  o->final_obs = B.final_obs;
  o->global_state = B.global;
  o->rewards = B.rewards;
  o->dones = B.dones;
  o->masks = B.masks;
  o->tracking_error = B.track_err;
  o->min_agent_dist = B.min_dist;
  o->target_lost = B.lost;
  o->collision = B.collision;
  o->step = B.step;
  o->actions = const_cast<int32_t*>(B.actions);
  o->px = B.px;
  o->py = B.py;
  o->vx = B.vx;
  o->vy = B.vy;
  o->w = B.w;
  o->total_sets = v->total_sets;
  o->set_offset = B.set_offset;
  return UT_OK;
}

int ut_vecenv_copy_outputs(ut_vecenv* v, const ut_host_outputs* d) {
  DeviceGuard dg(v->device);
  const DevBatch& B = v->B;
  const int64_t n = v->n_envs, Am = v->A_max, Tm = v->T_max;
  auto cp = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
    if (!dst) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, v->stream);
  };
  UT_CUDA(cp(d->obs, B.obs, sizeof(double) * 12 * B.obs_rows));
  UT_CUDA(cp(d->final_obs, B.final_obs, sizeof(double) * 12 * B.obs_rows));
  UT_CUDA(cp(d->global_state, B.global, sizeof(double) * 12 * B.global_rows));
  UT_CUDA(cp(d->rewards, B.rewards, sizeof(double) * n));
  UT_CUDA(cp(d->dones, B.dones, (size_t)n));
  UT_CUDA(cp(d->masks, B.masks, (size_t)(n * Am * 5)));
  UT_CUDA(cp(d->tracking_error, B.track_err, sizeof(double) * n * Tm));
  UT_CUDA(cp(d->min_agent_dist, B.min_dist, sizeof(double) * n * Tm));
  UT_CUDA(cp(d->target_lost, B.lost, (size_t)(n * Tm)));
  UT_CUDA(cp(d->collision, B.collision, (size_t)n));
  UT_CUDA(cp(d->step, B.step, sizeof(int32_t) * n));
  UT_CUDA(cudaStreamSynchronize(v->stream));
  return UT_OK;
}

int ut_vecenv_set_stream(ut_vecenv* v, void* s) {
  DeviceGuard dg(v->device);
  UT_CUDA(cudaStreamSynchronize(v->stream));
  // NULL: the handle's own stream; UT_STREAM_LEGACY (== cudaStreamLegacy): the
  // legacy default stream; anything else: a caller-owned cudaStream_t
  v->stream = s ? static_cast<cudaStream_t>(s) : v->own_stream;
  return UT_OK;
}

int ut_vecenv_wait_stream(ut_vecenv* v, void* s) {
  DeviceGuard dg(v->device);
  if (!v->order_ev) UT_CUDA(cudaEventCreateWithFlags(&v->order_ev, cudaEventDisableTiming));
  const cudaStream_t cs = s ? static_cast<cudaStream_t>(s) : cudaStreamLegacy;
  if (cs == v->stream) return UT_OK;
  UT_CUDA(cudaEventRecord(v->order_ev, cs));
  UT_CUDA(cudaStreamWaitEvent(v->stream, v->order_ev, 0));
  return UT_OK;
}

int ut_vecenv_synchronize(ut_vecenv* v) {
  DeviceGuard dg(v->device);
  UT_CUDA(cudaStreamSynchronize(v->stream));
  return UT_OK;
}

int ut_vecenv_stats(ut_vecenv* v, double out[UT_N_STATS], int reset) {
  DeviceGuard dg(v->device);
  double* d;
  UT_CUDA(cudaMallocAsync((void**)&d, sizeof(double) * UT_N_STATS, v->stream));
  stats_kernel<<<1, 256, 0, v->stream>>>(v->B, d, reset);
  ++v->launches;
  UT_CUDA(cudaGetLastError());
  UT_CUDA(cudaMemcpyAsync(out, d, sizeof(double) * UT_N_STATS, cudaMemcpyDeviceToHost, v->stream));
  UT_CUDA(cudaFreeAsync(d, v->stream));
  UT_CUDA(cudaStreamSynchronize(v->stream));
  return UT_OK;
}

int64_t ut_vecenv_launch_count(const ut_vecenv* v) { return v->launches; }

int ut_vecenv_enable_phase_timing(ut_vecenv* v, int on) {
  DeviceGuard dg(v->device);
  UT_CUDA(cudaStreamSynchronize(v->stream));
  if (on && !v->phase_buf) {
    int rc;
    if ((rc = v->alloc(&v->phase_buf, (size_t)v->grid_max * kPhaseSlots))) return rc;
    UT_CUDA(cudaMemset(v->phase_buf, 0, sizeof(unsigned long long) * v->grid_max * kPhaseSlots));
  }
  v->B.phase_cycles = on ? v->phase_buf : nullptr;
  return v->sync_batch();
}

// Per-CTA phase cycles summed over the grid (each CTA steps a contiguous env
// range, so this is the device analogue of the per-env phase sums), and the
// same converted to ns with the SM-clock rate the CTAs saw (elapsed globaltimer
// ns over elapsed cycles of every timed launch).
namespace {
int phase_sums(ut_vecenv* v, uint64_t cyc[UT_N_PHASES], double* ns_per_cycle, int reset) {
  for (int k = 0; k < UT_N_PHASES; ++k) cyc[k] = 0;
  *ns_per_cycle = 0.0;
  if (!v->phase_buf) return UT_OK;
  UT_CUDA(cudaStreamSynchronize(v->stream));
  std::vector<unsigned long long> h((size_t)v->grid_max * kPhaseSlots);
  UT_CUDA(cudaMemcpy(h.data(), v->phase_buf, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost));
  double c = 0.0, t = 0.0;
  for (int b = 0; b < v->grid_max; ++b) {
    const unsigned long long* r = h.data() + (size_t)b * kPhaseSlots;
    for (int k = 0; k < kPhaseCount; ++k) cyc[k] += r[k];
    c += (double)r[kPhaseWait + 1];
    t += (double)r[kPhaseWait + 2];
  }
  *ns_per_cycle = c > 0.0 ? t / c : 0.0;
  if (reset) UT_CUDA(cudaMemset(v->phase_buf, 0, sizeof(unsigned long long) * h.size()));
  return UT_OK;
}
}  // namespace

int ut_vecenv_phase_cycles(ut_vecenv* v, uint64_t out[UT_N_PHASES], int reset) {
  DeviceGuard dg(v->device);
  double r;
  return phase_sums(v, out, &r, reset);
}

int ut_vecenv_phase_ns(ut_vecenv* v, uint64_t out[UT_N_PHASES], int reset) {
  DeviceGuard dg(v->device);
  double r;
  uint64_t cyc[UT_N_PHASES];
  const int rc = phase_sums(v, cyc, &r, reset);
  for (int k = 0; k < UT_N_PHASES; ++k) out[k] = (uint64_t)std::llround((double)cyc[k] * r);
  return rc;
}

int ut_vecenv_set_auto_reset(ut_vecenv* v, int on) {
  DeviceGuard dg(v->device);
  UT_CUDA(cudaStreamSynchronize(v->stream));
  v->B.auto_reset = on ? 1 : 0;
  return v->sync_batch();
}

// Environment::serialize_state (env.cpp:550-593)
int ut_env_serialize(ut_vecenv* v, int64_t e, double* blob, size_t cap, size_t* len) {
  DeviceGuard dg(v->device);
  if (e < 0 || e >= v->n_envs) return fail(UT_ERR_CONTRACT, "serialize: env %lld out of range", (long long)e);
  const DevConfig& d = v->cfg(e);
  const int A = d.A, T = d.T, P = d.P, sA = d.sA, sT = d.sT, AA = sA * sA, AT = sA * sT;
  const size_t need = (size_t)(5 + 6 * A + 9 * T + A * (6 * A + T * (9 + 5 * P)));
  *len = need;
  if (!blob) return UT_OK;
  if (cap < need) return fail(UT_ERR_DATA, "serialize: buffer of %zu doubles too small (need %zu)", cap, need);
  std::vector<double> rec;
  int rc;
  if ((rc = v->get_rec(e, rec))) return rc;
  const size_t nset = (size_t)A * T * P;
  std::vector<double> f[5];
  double* src[5] = {v->B.px, v->B.py, v->B.vx, v->B.vy, v->B.w};
  for (int k = 0; k < 5; ++k) {
    f[k].resize(nset);
    UT_CUDA(cudaMemcpy(f[k].data(), src[k] + (size_t)v->set_at(e) * P, sizeof(double) * nset, cudaMemcpyDeviceToHost));
  }
  const double* ag = rec.data() + d.o_agent;
  const double* tg = rec.data() + d.o_target;
  const double* info = rec.data() + d.o_info;
  const double* trk = rec.data() + d.o_track;
  size_t i = 0;
  blob[i++] = rec[R_STEP];
  blob[i++] = rec[R_EP_SPEED];
  blob[i++] = rec[R_ENV_POS];
  blob[i++] = rec[R_ENV_HAVE_SPARE];
  blob[i++] = rec[R_ENV_SPARE];
  for (int a = 0; a < A; ++a)
    for (int fl = 0; fl < 6; ++fl) blob[i++] = ag[fl * sA + a];
  for (int t = 0; t < T; ++t)
    for (int fl = 0; fl < 8; ++fl) blob[i++] = tg[fl * sT + t];
  for (int t = 0; t < T; ++t) blob[i++] = rec[(size_t)d.o_miss + t];
  for (int a = 0; a < A; ++a) {
    for (int j = 0; j < A; ++j)
      for (int fl = 0; fl < I_NFIELD; ++fl) blob[i++] = info[fl * AA + a * sA + j];
    for (int t = 0; t < T; ++t) {
      for (int fl = 0; fl < K_NBLOB; ++fl) blob[i++] = trk[fl * AT + a * sT + t];
      const size_t ps = (size_t)(a * T + t);
      for (int k = 0; k < 5; ++k) {
        std::memcpy(blob + i, f[k].data() + ps * P, sizeof(double) * P);
        i += (size_t)P;
      }
    }
  }
  return UT_OK;
}

// Environment::deserialize_state (env.cpp:595-659). Like the reference, the batch
// buffers are refreshed only by ut_vecenv_refresh_outputs().
int ut_env_deserialize(ut_vecenv* v, int64_t e, const double* blob, size_t len) {
  DeviceGuard dg(v->device);
  if (e < 0 || e >= v->n_envs) return fail(UT_ERR_CONTRACT, "deserialize: env %lld out of range", (long long)e);
  const DevConfig& d = v->cfg(e);
  const int A = d.A, T = d.T, P = d.P, sA = d.sA, sT = d.sT, AA = sA * sA, AT = sA * sT;
  const size_t need = (size_t)(5 + 6 * A + 9 * T + A * (6 * A + T * (9 + 5 * P)));
  if (len < need) return fail(UT_ERR_DATA, "environment state blob truncated");
  if (len > need) return fail(UT_ERR_DATA, "environment state blob has trailing data");
  std::vector<double> rec;
  int rc;
  if ((rc = v->get_rec(e, rec))) return rc;
  double* ag = rec.data() + d.o_agent;
  double* tg = rec.data() + d.o_target;
  double* info = rec.data() + d.o_info;
  double* trk = rec.data() + d.o_track;
  const size_t nset = (size_t)A * T * P;
  std::vector<double> f[5];
  for (auto& x : f) x.resize(nset);
  size_t i = 0;
  // integer fields go through the same (int) truncation as the reference
  auto as_int = [](double x) { return (double)(int)x; };
  rec[R_STEP] = as_int(blob[i++]);
  rec[R_EP_SPEED] = blob[i++];
  rec[R_ENV_POS] = (double)(uint64_t)blob[i++];
  rec[R_ENV_HAVE_SPARE] = blob[i++] != 0.0 ? 1.0 : 0.0;
  rec[R_ENV_SPARE] = blob[i++];
  for (int a = 0; a < A; ++a)
    for (int fl = 0; fl < 6; ++fl) {
      const double x = blob[i++];
      ag[fl * sA + a] = fl == V_RUDDER ? as_int(x) : x;
    }
  for (int t = 0; t < T; ++t)
    for (int fl = 0; fl < 8; ++fl) {
      const double x = blob[i++];
      tg[fl * sT + t] = (fl == V_RUDDER || fl == V_COUNTDOWN) ? as_int(x) : x;
    }
  for (int t = 0; t < T; ++t) rec[(size_t)d.o_miss + t] = as_int(blob[i++]);
  for (int a = 0; a < A; ++a) {
    for (int j = 0; j < A; ++j)
      for (int fl = 0; fl < I_NFIELD; ++fl) {
        const double x = blob[i++];
        double& dst = info[fl * AA + a * sA + j];
        dst = fl == I_AGE ? as_int(x) : fl == I_VALID ? (x != 0.0 ? 1.0 : 0.0) : x;
      }
    for (int t = 0; t < T; ++t) {
      const int ti = a * sT + t;
      for (int fl = 0; fl < K_NBLOB; ++fl) {
        const double x = blob[i++];
        double& dst = trk[fl * AT + ti];
        dst = fl == K_AGE ? as_int(x)
              : (fl == K_EVER || fl == K_HAVE_SPARE) ? (x != 0.0 ? 1.0 : 0.0)
              : fl == K_POS ? (double)(uint64_t)x
                            : x;
      }
      trk[K_ESSOK * AT + ti] = 0.0;  // injected weights have not been vetted
      const size_t ps = (size_t)(a * T + t);
      for (int k = 0; k < 5; ++k) {
        std::memcpy(f[k].data() + ps * P, blob + i, sizeof(double) * P);
        i += (size_t)P;
      }
    }
  }
  if ((rc = v->put_rec(e, rec))) return rc;
  double* dst[5] = {v->B.px, v->B.py, v->B.vx, v->B.vy, v->B.w};
  for (int k = 0; k < 5; ++k)
    UT_CUDA(cudaMemcpy(dst[k] + (size_t)v->set_at(e) * P, f[k].data(), sizeof(double) * nset, cudaMemcpyHostToDevice));
  return UT_OK;
}

// Batched serialize / deserialize of envs [e_begin, e_end): blobs back to back
// (env e's at the sum of the lengths before it), packed on the device one CTA
// per env and moved in staging batches of <= kBlobStaging bytes.
namespace {
constexpr size_t kBlobStaging = size_t(256) << 20;

int blob_batches(ut_vecenv* v, int64_t e_begin, int64_t e_end, bool do_export, double* host_out,
                 const double* host_in) {
  int sms = 0;
  UT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, v->device));
  UT_CUDA(cudaStreamSynchronize(v->stream));
  std::vector<int64_t> off;
  size_t host_pos = 0;
  double* stage = nullptr;
  int64_t* d_off = nullptr;
  size_t stage_cap = 0, off_cap = 0;
  int rc = UT_OK;
  for (int64_t b = e_begin; b < e_end && rc == UT_OK;) {
    off.assign(1, 0);
    int64_t e = b;
    while (e < e_end) {
      const DevConfig& d = v->cfg(e);
      const int64_t l = blob_len(d.A, d.T, d.P);
      if (e > b && (size_t)(off.back() + l) * sizeof(double) > kBlobStaging) break;
      off.push_back(off.back() + l);
      ++e;
    }
    const int64_t n = e - b;
    const size_t words = (size_t)off.back();
    if (words > stage_cap) {
      cudaFree(stage);
      stage = nullptr;
      if (cudaMalloc(&stage, words * sizeof(double)) != cudaSuccess) {
        rc = fail(UT_ERR_RUNTIME, "state export/import: cannot allocate %zu bytes of staging", words * 8);
        break;
      }
      stage_cap = words;
    }
    if ((size_t)n + 1 > off_cap) {
      cudaFree(d_off);
      d_off = nullptr;
      if (cudaMalloc(&d_off, (n + 1) * sizeof(int64_t)) != cudaSuccess) {
        rc = fail(UT_ERR_RUNTIME, "state export/import: cannot allocate offsets");
        break;
      }
      off_cap = (size_t)n + 1;
    }
    cudaError_t err = cudaMemcpyAsync(d_off, off.data(), (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, v->stream);
    const unsigned grid = (unsigned)std::min<int64_t>(n, (int64_t)sms * 8);
    if (err == cudaSuccess && do_export) {
      pack_blobs_kernel<<<grid, 256, 0, v->stream>>>(v->B, b, n, d_off, stage);
      err = cudaGetLastError();
      if (err == cudaSuccess)
        err = cudaMemcpyAsync(host_out + host_pos, stage, words * sizeof(double), cudaMemcpyDeviceToHost, v->stream);
    } else if (err == cudaSuccess) {
      err = cudaMemcpyAsync(stage, host_in + host_pos, words * sizeof(double), cudaMemcpyHostToDevice, v->stream);
      if (err == cudaSuccess) {
        unpack_blobs_kernel<<<grid, 256, 0, v->stream>>>(v->B, b, n, d_off, stage);
        err = cudaGetLastError();
      }
    }
    v->launches += 1;
    if (err == cudaSuccess) err = cudaStreamSynchronize(v->stream);
    if (err != cudaSuccess) rc = fail(UT_ERR_RUNTIME, "state export/import: %s", cudaGetErrorString(err));
    host_pos += words;
    b = e;
  }
  cudaFree(stage);
  cudaFree(d_off);
  return rc;
}

int blob_range(ut_vecenv* v, int64_t e_begin, int64_t e_end, size_t* total, const char* what) {
  if (e_begin < 0 || e_end > v->n_envs || e_begin > e_end)
    return fail(UT_ERR_CONTRACT, "%s: env range [%lld, %lld) outside [0, %lld)", what, (long long)e_begin,
                (long long)e_end, (long long)v->n_envs);
  size_t t = 0;
  for (int64_t e = e_begin; e < e_end; ++e) {
    const DevConfig& d = v->cfg(e);
    t += (size_t)blob_len(d.A, d.T, d.P);
  }
  *total = t;
  return UT_OK;
}
}  // namespace

int ut_vecenv_export_state(ut_vecenv* v, int64_t e_begin, int64_t e_end, double* blobs, size_t cap, size_t* len) {
  DeviceGuard dg(v->device);
  size_t total = 0;
  int rc = blob_range(v, e_begin, e_end, &total, "export_state");
  if (rc) return rc;
  *len = total;
  if (!blobs) return UT_OK;
  if (cap < total) return fail(UT_ERR_DATA, "export_state: buffer of %zu doubles too small (need %zu)", cap, total);
  return blob_batches(v, e_begin, e_end, true, blobs, nullptr);
}

int ut_vecenv_import_state(ut_vecenv* v, int64_t e_begin, int64_t e_end, const double* blobs, size_t len) {
  DeviceGuard dg(v->device);
  size_t total = 0;
  int rc = blob_range(v, e_begin, e_end, &total, "import_state");
  if (rc) return rc;
  if (len < total) return fail(UT_ERR_DATA, "environment state blobs truncated");
  if (len > total) return fail(UT_ERR_DATA, "environment state blobs have trailing data");
  return blob_batches(v, e_begin, e_end, false, nullptr, blobs);
}

int ut_env_world_step(ut_vecenv* v, int64_t e, int32_t* step) {
  DeviceGuard dg(v->device);
  if (e < 0 || e >= v->n_envs) return fail(UT_ERR_CONTRACT, "world_step: env %lld out of range", (long long)e);
  double s = 0.0;
  UT_CUDA(cudaStreamSynchronize(v->stream));
  UT_CUDA(cudaMemcpy(&s, v->B.rec + (int64_t)R_STEP * v->n_envs + e, sizeof(double), cudaMemcpyDeviceToHost));
  *step = (int32_t)s;
  return UT_OK;
}

// benchmark_sps (vecenv.cpp:175-202): warmup, then CUDA-event-timed steps with
// phase timing on (the reference times its phases in the same run).
int ut_benchmark_sps(const ut_env_config* cfg, int64_t n_envs, int32_t n_steps, int policy, uint64_t seed,
                     int32_t warmup, int device, ut_benchmark_report* out) {
  ut_vecenv* v = nullptr;
  int rc = ut_vecenv_create(cfg, n_envs, seed, 0, device, &v);
  if (rc) return rc;
  DeviceGuard dg(device);
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  rc = ut_vecenv_step_policy(v, policy, warmup);
  if (!rc) rc = ut_vecenv_enable_phase_timing(v, 1);
  if (!rc) {
    uint64_t scratch[UT_N_PHASES];
    rc = ut_vecenv_phase_cycles(v, scratch, 1);
  }
  if (!rc) {
    cudaEventRecord(t0, v->stream);
    rc = ut_vecenv_step_policy(v, policy, n_steps);
    cudaEventRecord(t1, v->stream);
    cudaEventSynchronize(t1);
  }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  if (!rc) {
    out->n_envs = n_envs;
    out->n_agents = v->A_max;
    out->n_targets = v->T_max;
    out->timed_steps = n_steps;
    out->wall_seconds = ms / 1e3;
    out->sps = (double)n_envs * n_steps / out->wall_seconds;
    out->agent_sps = out->sps * v->A_max;
    rc = ut_vecenv_phase_ns(v, out->phase_ns, 0);
    out->total_ns = 0;
    for (int k = 0; k < UT_PHASE_RESET; ++k) out->total_ns += out->phase_ns[k];
  }
  ut_vecenv_destroy(v);
  return rc;
}

}  // extern "C"

// ------------------------------------------------------------ ut_debug.h ---
namespace {
// Grid quantity q: 0 log(u1), 1 cos(2pi_f u2), 2 sin(2pi_f u2), 3 the Box-Muller
// radius sqrt(-2 log u1), over all 2^24 values the 24-bit draws can produce.
__global__ void cr_grid_kernel(int q, float* out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (1u << 24)) return;
  const float two_pi_f = 2.0f * 3.14159265358979323846f;
  if (q == 0 || q == 3) {
    const float l = cr_logf((float)(i + 1u) * 0x1.0p-24f);
    out[i] = q == 0 ? l : __fsqrt_rn(-2.0f * l);
  } else {
    float s, c;
    cr_sincosf(__fmul_rn(two_pi_f, (float)i * 0x1.0p-24f), &s, &c);
    out[i] = q == 1 ? c : s;
  }
}
// The production (table-driven) path: the same functions box_muller_fast is
// built from, falling back exactly like the step kernel does.
__global__ void cr_grid_fast_kernel(int q, float* out) {
  __shared__ double2 tl[128], ts[64 * 8];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) tl[i] = make_double2(kLogTab[2 * i], kLogTab[2 * i + 1]);
  for (int i = threadIdx.x; i < 64 * 8; i += blockDim.x)
    ts[i] = make_double2(kSinCosTab[2 * (i >> 3)], kSinCosTab[2 * (i >> 3) + 1]);
  __syncthreads();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (1u << 24)) return;
  const float two_pi_f = 2.0f * 3.14159265358979323846f;
  if (q == 0 || q == 3) {
    const float l = cr_logf_fast((float)(i + 1u) * 0x1.0p-24f, tl);
    out[i] = q == 0 ? l : sqrt_rn_f(-2.0f * l);
  } else {
    float s, c;
    cr_sincosf_fast(__fmul_rn(two_pi_f, (float)i * 0x1.0p-24f), &s, &c, ts);
    out[i] = q == 1 ? c : s;
  }
}
// Random operands over the clamp's domain: sqrt of x = 0 and of log-uniform
// x in [2^-960, 2^200]; a / b with log-uniform a in [2^-20, 2^20], b >= a.
__global__ void ieee_check_kernel(int kind, uint64_t seed, int64_t n, unsigned long long* bad) {
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 r = philox(seed, 0x69656565ull, (uint64_t)i);
    const double u = ((double)(((uint64_t)r.y << 32 | r.x) >> 11)) * 0x1.0p-53;
    const double v = ((double)(((uint64_t)r.w << 32 | r.z) >> 11)) * 0x1.0p-53;
    if (kind == 0) {
      const double x = i == 0 ? 0.0 : exp2(-960.0 + 1160.0 * u) * (1.0 + v);
      const double a = sqrt_rn_clamp(x), b = __dsqrt_rn(x);
      local += __double_as_longlong(a) != __double_as_longlong(b);
    } else if (kind == 4) {
      // the particle-weight exp (exp_neg, table in global memory here) against
      // libm exp over [-760, 0]: results more than 1 ulp off
      const double* tab = kExp2Tab;
      const double x = -760.0 * u;
      const long long a = __double_as_longlong(exp_neg<1>(x, tab)), b = __double_as_longlong(exp(x));
      local += (a - b > 1 || b - a > 1);
    } else if (kind == 2 || kind == 3) {
      // the likelihood distance sqrt (sqrt_dist) against IEEE over squared
      // distances in [2^-60, (40 km)^2] (2: results more than 1 ulp off; 3: any
      // difference); x = 0 is NaN by design (the step's exact path takes it)
      const double x = exp2(-60.0 + 91.0 * u) * (1.0 + v);
      const long long a = __double_as_longlong(sqrt_dist(x)), b = __double_as_longlong(__dsqrt_rn(x));
      local += kind == 3 ? a != b : (a - b > 1 || b - a > 1);
    } else {
      const double a = exp2(-20.0 + 40.0 * u);
      const double b = a * (1.0 + 1e6 * v);
      const double q = div_rn_clamp(a, b), w = __ddiv_rn(a, b);
      local += __double_as_longlong(q) != __double_as_longlong(w);
    }
  }
  if (local) atomicAdd(bad, local);
}
__global__ void philox_kernel(uint64_t key, uint64_t stream, uint64_t block0, int n, uint4* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = philox(key, stream, block0 + (uint64_t)i);
}
__global__ void derive_key_kernel(uint64_t a, uint64_t b, uint64_t c, uint64_t d, uint64_t* out) {
  *out = derive_key(a, b, c, d);
}
// FP64 issue peak: 8 independent DFMA chains per thread (the denominator of the
// step kernel's fp64 roofline).
__global__ void __launch_bounds__(256) fp64_peak_kernel(int iters, double seed, double* sink) {
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed + 1e-9 * (double)threadIdx.x + (double)j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], 0.9999999, 1e-7);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s = s + a[j];
  if (s == 12345.0) *sink = s;
}
}  // namespace

#include "ut_debug.h"

extern "C" {
int ut_debug_set_knobs(ut_vecenv* v, int force_exact, int64_t trace_env) {
  DeviceGuard dg(v->device);
  v->B.force_exact = force_exact;
  v->B.trace_env = trace_env;
  return v->sync_batch();
}
int ut_debug_set_grid(ut_vecenv* v, int32_t ctas) {
  DeviceGuard dg(v->device);
  if (ctas < 0 || ctas > v->grid_max)
    return fail(UT_ERR_CONTRACT, "set_grid: %d CTAs outside [1, %d] (0 = the default)", ctas, v->grid_max);
  UT_CUDA(cudaStreamSynchronize(v->stream));
  v->grid = ctas ? ctas : v->grid_max;
  return UT_OK;
}
int ut_debug_instance(ut_vecenv* v, int32_t* full, int32_t* np) {
  DeviceGuard dg(v->device);
  *full = v->full ? 1 : 0;
  *np = v->np;
  return UT_OK;
}
int ut_debug_cta_cycles(ut_vecenv* v, uint64_t* out, int64_t cap, int64_t* n) {
  DeviceGuard dg(v->device);
  *n = v->phase_buf ? (int64_t)v->grid : 0;
  if (!v->phase_buf || !out) return UT_OK;
  if (cap < *n) return fail(UT_ERR_CONTRACT, "cta_cycles: room for %lld CTAs, need %lld", (long long)cap, (long long)*n);
  UT_CUDA(cudaStreamSynchronize(v->stream));
  std::vector<unsigned long long> h((size_t)v->grid * kPhaseSlots);
  UT_CUDA(cudaMemcpy(h.data(), v->phase_buf, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost));
  for (int64_t b = 0; b < *n; ++b) {  // busy cycles: every phase, not the grid-barrier waits
    uint64_t t = 0;
    for (int k = 0; k < kPhaseCount; ++k) t += h[(size_t)b * kPhaseSlots + k];
    out[b] = t;
  }
  return UT_OK;
}
int ut_debug_abi_sizes(int64_t out[4]) {
  out[0] = sizeof(ut_env_config);
  out[1] = sizeof(ut_buffers);
  out[2] = sizeof(ut_host_outputs);
  out[3] = sizeof(ut_benchmark_report);
  return UT_OK;
}
int ut_debug_cr_grid(int kind, int device, float* host_out) {
  UT_CUDA(cudaSetDevice(device));
  float* d = nullptr;
  const size_t n = (size_t)1 << 24;
  UT_CUDA(cudaMalloc(&d, n * sizeof(float)));
  if (kind < 0 || kind > 7) return fail(UT_ERR_CONTRACT, "cr_grid: kind must be 0..7");
  if (kind < 4)
    cr_grid_kernel<<<(unsigned)(n / 256), 256>>>(kind, d);
  else
    cr_grid_fast_kernel<<<(unsigned)(n / 256), 256>>>(kind - 4, d);
  cudaError_t err = cudaMemcpy(host_out, d, n * sizeof(float), cudaMemcpyDeviceToHost);
  cudaFree(d);
  UT_CUDA(err);
  return UT_OK;
}
int ut_debug_ieee_check(int kind, uint64_t seed, int64_t n, int device, uint64_t* mismatches) {
  UT_CUDA(cudaSetDevice(device));
  unsigned long long* d = nullptr;
  UT_CUDA(cudaMalloc(&d, sizeof(unsigned long long)));
  UT_CUDA(cudaMemset(d, 0, sizeof(unsigned long long)));
  ieee_check_kernel<<<1184, 256>>>(kind, seed, n, d);
  unsigned long long h = 0;
  cudaError_t err = cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(d);
  UT_CUDA(err);
  *mismatches = h;
  return UT_OK;
}
int ut_debug_philox(uint64_t key, uint64_t stream, uint64_t block0, int32_t n, int device, uint32_t* host_out) {
  UT_CUDA(cudaSetDevice(device));
  uint4* d = nullptr;
  UT_CUDA(cudaMalloc(&d, (size_t)n * sizeof(uint4)));
  philox_kernel<<<(unsigned)((n + 255) / 256), 256>>>(key, stream, block0, n, d);
  cudaError_t err = cudaMemcpy(host_out, d, (size_t)n * sizeof(uint4), cudaMemcpyDeviceToHost);
  cudaFree(d);
  UT_CUDA(err);
  return UT_OK;
}
int ut_debug_fp64_peak(int device, double* dfma_per_s) {
  UT_CUDA(cudaSetDevice(device));
  int sms = 0;
  UT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  double* d = nullptr;
  UT_CUDA(cudaMalloc(&d, sizeof(double)));
  cudaEvent_t e0, e1;
  UT_CUDA(cudaEventCreate(&e0));
  UT_CUDA(cudaEventCreate(&e1));
  const int blocks = sms * 8, iters = 1 << 14;
  fp64_peak_kernel<<<blocks, 256>>>(64, 1.0, d);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    fp64_peak_kernel<<<blocks, 256>>>(iters, 1.0, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  UT_CUDA(err);
  *dfma_per_s = (double)blocks * 256.0 * (double)iters * 8.0 / (best * 1e-3);
  return UT_OK;
}
int ut_debug_set_profile(int device, uint64_t* out, int reset) {
  UT_CUDA(cudaSetDevice(device));
#ifdef UT_SET_PROFILE
  UT_CUDA(cudaDeviceSynchronize());
  UT_CUDA(cudaMemcpyFromSymbol(out, g_setprof, sizeof(uint64_t) * kSetProfSlots));
  if (reset) {
    static const unsigned long long zero[kSetProfSlots] = {};
    UT_CUDA(cudaMemcpyToSymbol(g_setprof, zero, sizeof(zero)));
  }
#else
  for (int k = 0; k < kSetProfSlots; ++k) out[k] = 0;
  (void)reset;
#endif
  return UT_OK;
}
int ut_debug_derive_key(uint64_t a, uint64_t b, uint64_t c, uint64_t dd, int device, uint64_t* out) {
  UT_CUDA(cudaSetDevice(device));
  uint64_t* d = nullptr;
  UT_CUDA(cudaMalloc(&d, sizeof(uint64_t)));
  derive_key_kernel<<<1, 1>>>(a, b, c, dd, d);
  cudaError_t err = cudaMemcpy(out, d, sizeof(uint64_t), cudaMemcpyDeviceToHost);
  cudaFree(d);
  UT_CUDA(err);
  return UT_OK;
}
}  // extern "C"

// ------------------------------------------------- multi-device handle ---
#include "ut_multi.cuh"
