// Exercises include/ut_vecenv.hpp the way reference-side C++ would use
// utrack::VecEnv (test_vecenv.cpp style). Prints one JSON line.
#include <cstdio>
#include <vector>

#include "ut_vecenv.hpp"

namespace ut = utrack_b200;

int main() {
  try {
    ut::EnvConfig cfg = ut::default_config();
    cfg.n_agents = 2;
    cfg.n_targets = 2;
    cfg.pf.n_particles = 64;
    cfg.horizon = 3;
    ut::VecEnv venv(cfg, 4, 7);
    std::vector<int> acts(static_cast<size_t>(venv.n_envs() * venv.n_agents()), 2);  // hold course
    venv.step(acts);
    venv.step_policy(ut::BenchmarkPolicy::kRandom);
    venv.step(acts);
    double rsum = 0.0;
    for (double r : venv.rewards()) rsum += r;
    int done = 0;
    for (auto d : venv.dones()) done += d;
    // the same batch through the multi-device handle (two shards on device 0)
    ut::MultiVecEnv multi(cfg, 4, 7, {0, 0});
    multi.step(acts);
    multi.step_policy(ut::BenchmarkPolicy::kRandom);
    multi.step(acts);
    int multi_same = multi.n_shards() == 2 && multi.rewards() == venv.rewards() && multi.dones() == venv.dones() &&
                     multi.obs_stack().data == venv.obs_stack().data && multi.masks() == venv.masks();
    for (int e = 0; e < venv.n_envs(); ++e)
      multi_same = multi_same && multi.serialize_state(e) == venv.serialize_state(e) &&
                   multi.world_step(e) == venv.world_step(e);
    const std::vector<double> all = venv.export_state(0, venv.n_envs());
    venv.import_state(0, venv.n_envs(), all);
    std::printf("{\"ok\": 1, \"reward_sum\": %.17g, \"dones\": %d, \"obs00\": %.17g, \"step0\": %d, \"blob\": %zu, "
                "\"all\": %zu, \"multi_same\": %d}\n",
                rsum, done, venv.obs_stack()(0, 0), venv.world_step(0), venv.serialize_state(0).size(), all.size(),
                multi_same);
  } catch (const ut::DeviceError& e) {
    std::printf("{\"ok\": 0, \"error\": \"DeviceError\"}\n");
  } catch (const std::exception& e) {
    std::printf("{\"ok\": 0, \"error\": \"%s\"}\n", e.what());
    return 1;
  }
  return 0;
}
