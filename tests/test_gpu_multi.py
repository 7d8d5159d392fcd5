"""GPU: the multi-device VecEnv handle (ut_multienv_*, include/ut_env.h).

The reference's VecEnv is one object over all envs, sharded by env index over
its workers (vecenv.hpp:26-27, vecenv.cpp:83), and its own gate for sharding is
partition invariance (test_vecenv.cpp:126-143). Here the shards are devices:
on this one-GPU box the handle lists device 0 several times (a legal handle whose
statistics are summed on the host) and once with NCCL forced on (one-rank
communicator: the NCCL path of the statistics all-reduce runs). The batch must
be bit-identical to a single-device VecEnv of the same size and seed.
"""
import numpy as np
import pytest

from oracle_bindings import default_config, random_legal_actions
from test_gpu_parity import _to_py

pytestmark = pytest.mark.gpu

INT_STATS = ("env_steps", "episodes_done", "collision_steps", "lost_target_steps", "pf_updates",
             "pf_resamples", "pf_exact_path", "eval_collided_episodes", "eval_lost_episodes")


def _pair(n_envs, devices, stats, **kw):
    from paper_2505_08222_b200.vecenv import MultiVecEnv, VecEnv
    cfg = _to_py(default_config(**kw))
    return VecEnv(cfg, n_envs, 11), MultiVecEnv(cfg, n_envs, 11, devices=devices, stats=stats)


def _same_batch(one, multi, n_envs):
    a, b = one.host_outputs(), multi.host_outputs()
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    for e in range(n_envs):
        assert np.array_equal(one.serialize_state(e), multi.serialize_state(e)), e
        assert one.world_step(e) == multi.world_step(e)


def _same_stats(one, multi):
    from paper_2505_08222_b200._abi import STAT_NAMES
    s1, s2 = one.stats(), multi.stats()
    for k, name in enumerate(STAT_NAMES):
        if name in INT_STATS:
            assert s1[k] == s2[k], name
        else:  # shard partial sums added in another order
            assert abs(s1[k] - s2[k]) <= 1e-12 * max(abs(s1[k]), 1.0), name


@pytest.mark.parametrize("n_shards", [2, 3])
def test_shards_on_one_device_equal_the_whole_batch(cuda_device, n_shards):
    kw = dict(n_agents=3, n_targets=2, horizon=6, pf_n_particles=1024)
    n = 37
    one, multi = _pair(n, [0] * n_shards, "auto", **kw)
    assert multi.n_shards() == n_shards and multi.stats_backend() == "host"
    bounds = [multi.shard_range(i)[:2] for i in range(n_shards)]
    assert bounds[0][0] == 0 and bounds[-1][1] == n
    assert all(bounds[i][1] == bounds[i + 1][0] for i in range(n_shards - 1))
    _same_batch(one, multi, n)
    rng = np.random.default_rng(3)
    for s in range(8):  # crosses an auto-reset at step 6
        if s % 2:
            one.step_policy("random")
            multi.step_policy("random")
        else:
            acts = random_legal_actions(one.host_outputs(["masks"])["masks"], rng).reshape(n, 3)
            one.step(acts)
            multi.step(acts)
        _same_batch(one, multi, n)
    _same_stats(one, multi)
    one.reset_all()
    multi.reset_all()
    _same_batch(one, multi, n)


def test_nccl_statistics_all_reduce(cuda_device):
    from paper_2505_08222_b200 import _abi, _native
    lib = _native.lib()
    _abi.declare_product(lib)
    import ctypes as C
    ver = C.c_int()
    assert lib.ut_nccl_version(C.byref(ver)) == 0 and ver.value >= 21800
    kw = dict(n_agents=2, n_targets=2, horizon=5, pf_n_particles=256)
    one, multi = _pair(20, [0], "nccl", **kw)
    assert multi.stats_backend() == "nccl"
    one.step_policy("random", 7)
    multi.step_policy("random", 7)
    _same_batch(one, multi, 20)
    s1, s2 = one.stats(), multi.stats()
    assert np.array_equal(s1, s2)  # one rank: the all-reduce is exact
    assert s1[0] == 140
    multi.stats(reset=True)
    assert np.all(multi.stats() == 0)


def test_invalid_action_names_the_global_env_and_moves_nothing(cuda_device):
    from paper_2505_08222_b200.vecenv import ContractViolation
    kw = dict(n_agents=2, n_targets=1, horizon=9, pf_n_particles=64)
    one, multi = _pair(10, [0, 0], "host", **kw)
    before = [multi.serialize_state(e) for e in range(10)]
    acts = np.full((10, 2), 2, np.int32)
    acts[7, 1] = 4  # env 7 is in the second shard [5, 10)
    acts[8, 0] = 9
    with pytest.raises(ContractViolation, match=r"^env 7: step: invalid action 4 for agent 1"):
        multi.step(acts)
    for e in range(10):
        assert np.array_equal(before[e], multi.serialize_state(e))


def test_phase_timing_sums_the_shards(cuda_device):
    kw = dict(n_agents=2, n_targets=2, horizon=50, pf_n_particles=1024)
    _, multi = _pair(64, [0, 0], "host", **kw)
    multi.enable_phase_timing(True)
    multi.step_policy("random", 3)
    ns = multi.phase_ns()
    assert ns["filter"] > 0 and ns["comms"] > 0 and ns["targets"] > 0
    assert multi.launch_count() >= 6
