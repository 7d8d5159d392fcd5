"""GPU tests of the boundary's semantics beyond the step itself: the single
Environment (no auto-reset, env.cpp:234-504) against the reference's own
Environment, stream ordering of device-resident actions, the ragged particle
view of mixed fleets, double-buffered terminal observations, and the
per-phase timing (PhaseTimer, env.cpp:18-36)."""
import numpy as np
import pytest

from oracle_bindings import Oracle, RefEnvironment, default_config, random_legal_actions, ref_available
from parity import TIGHT_RTOL, Report, compare_blobs, compare_outputs
from test_gpu_parity import _to_py

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_environment_does_not_auto_reset_like_reference(cuda_device):
    """Environment::step never resets (env.cpp:234-504): past the horizon the
    env keeps stepping with done set until reset() (curriculum.cpp:289 calls it
    explicitly); checked against the reference's own Environment."""
    from paper_2505_08222_b200.vecenv import ContractViolation, Environment
    cfg = default_config(n_agents=2, n_targets=2, pf_n_particles=128, horizon=4)
    ref = RefEnvironment(cfg, 9, env_index=3)
    env = Environment(_to_py(cfg), 9, env_index=3)
    rng = np.random.default_rng(5)
    rep = Report()

    def acts():
        return np.array([rng.choice(np.flatnonzero(env.action_mask(a))) for a in range(2)], np.int32)

    for s in range(7):  # terminal at step 4, then 3 more steps with done set
        a = acts()
        want = ref.step(a)
        got = env.step(a)
        assert got["done"] == want["done"] == (s + 1 >= 4)
        assert got["collision"] == want["collision"]
        assert abs(got["reward"] - want["reward"]) <= TIGHT_RTOL * max(abs(want["reward"]), 1e-6)
        compare_blobs(env.serialize_state(), ref.serialize(), 2, 2, 128, rep, tag=f"s{s}")
        assert env.world_step() == s + 1
        for ag in range(2):
            np.testing.assert_allclose(env.observation(ag), ref.observation(ag), rtol=1e-9, atol=1e-12)
    ref.reset()
    env.reset()
    compare_blobs(env.serialize_state(), ref.serialize(), 2, 2, 128, rep, tag="reset")
    for s in range(3):
        a = acts()
        ref.step(a)
        env.step(a)
        compare_blobs(env.serialize_state(), ref.serialize(), 2, 2, 128, rep, tag=f"r{s}")
    assert not rep.int_mismatch and rep.worst() <= TIGHT_RTOL, rep
    with pytest.raises(ContractViolation, match=r"^step: invalid action 9 for agent 0"):
        env.step([9, 2])


def test_device_actions_are_ordered_after_their_producer(cuda_device):
    """Actions written by a torch kernel that is still queued behind a long one
    on torch's stream must be what the step reads (ut_vecenv_wait_stream)."""
    import torch
    from paper_2505_08222_b200.vecenv import VecEnv
    cfg = default_config(n_agents=2, n_targets=1, pf_n_particles=64, horizon=50)
    n = 64
    ora = Oracle(cfg, n, 4)
    gpu = VecEnv(_to_py(cfg), n, 4)
    rng = np.random.default_rng(0)
    dev = torch.empty((n, 2), dtype=torch.int32, device="cuda")
    rep = Report()
    for s in range(4):
        acts = random_legal_actions(ora.outputs()["masks"], rng).reshape(n, 2)
        dev.fill_(9)  # invalid: a stale read raises ContractViolation
        torch.cuda.synchronize()
        torch.cuda._sleep(200_000_000)  # ~0.1 s of GPU time ahead of the producer
        dev.copy_(torch.from_numpy(acts).pin_memory(), non_blocking=True)
        gpu.step(dev)
        ora.step(acts)
        compare_outputs(gpu.host_outputs(), ora.outputs(), rep, tag=f"s{s}")
        assert not rep.int_mismatch, rep
    assert rep.worst() <= TIGHT_RTOL, rep


def test_particle_view_of_mixed_fleet_is_ragged(cuda_device):
    """ut_buffers.total_sets / set_offset: the particle view covers exactly the
    sum of A_e * T_e sets and env e's set (a, t) is row set_offset(e) + a T_e + t."""
    from paper_2505_08222_b200.vecenv import VecEnv
    shapes = [(1, 2), (3, 1), (2, 2)]
    cfgs = [default_config(n_agents=a, n_targets=t, pf_n_particles=64) for a, t in shapes]
    fleet = [0, 1, 2, 1, 0]
    gpu = VecEnv([_to_py(c) for c in cfgs], len(fleet), 8, fleet=fleet)
    gpu.step_policy("random", 2)
    pf = gpu.particles()
    assert pf["px"].shape == (sum(shapes[f][0] * shapes[f][1] for f in fleet), 64)
    px = pf["px"].cpu().numpy()
    for e, f in enumerate(fleet):
        A, T = shapes[f]
        blob = gpu.serialize_state(e)
        base = 5 + 6 * A + 9 * T
        for a in range(A):
            for t in range(T):
                off = base + a * (6 * A + T * (9 + 5 * 64)) + 6 * A + t * (9 + 5 * 64) + 9
                np.testing.assert_array_equal(px[gpu.set_offset(e) + a * T + t], blob[off:off + 64])


def test_final_obs_double_buffered(cuda_device):
    """horizon 1: every env finishes every step; with two output sets each
    step's final_obs (terminal observations) arrives intact through the async
    copy while the next step runs (final_obs was shared)."""
    import torch
    cfg = default_config(n_agents=2, n_targets=2, pf_n_particles=64, horizon=1)
    from paper_2505_08222_b200.vecenv import VecEnv
    n = 8
    ora = Oracle(cfg, n, 12)
    gpu = VecEnv(_to_py(cfg), n, 12)
    gpu.set_output_buffers(2)
    side = torch.cuda.Stream()
    pending = None
    for s in range(6):
        ora.step_policy(1)
        gpu.step_policy("random", 1)
        if pending is not None:
            side.synchronize()
            host, want = pending
            np.testing.assert_allclose(host["final_obs"].numpy(), want, rtol=1e-9, atol=1e-12)
        want = ora.outputs()["final_obs"].copy()
        host = {"final_obs": torch.empty(want.shape, dtype=torch.float64, pin_memory=True)}
        gpu.copy_outputs_async(host, side.cuda_stream)
        pending = (host, want)
    side.synchronize()
    np.testing.assert_allclose(pending[0]["final_obs"].numpy(), pending[1], rtol=1e-9, atol=1e-12)


def test_phase_timing_covers_the_reference_phases(cuda_device):
    """The seven StepPhase sums (env.cpp:250-279) plus reset, in ns."""
    from paper_2505_08222_b200.vecenv import EnvConfig, PfConfig, VecEnv, benchmark_sps
    cfg = EnvConfig(n_agents=3, n_targets=2, horizon=3, spawn_max_sep=400.0, pf=PfConfig(n_particles=1024))
    v = VecEnv(cfg, 512, 1)
    v.enable_phase_timing(True)
    v.phase_ns(reset=True)
    v.step_policy("random", 6)  # two auto-resets
    ns = v.phase_ns()
    cyc = v.phase_cycles()
    assert set(ns) == {"targets", "agents", "measure", "filter", "comms", "observe", "reward", "reset"}
    assert all(ns[k] > 0 for k in ns), ns
    assert ns["filter"] + ns["comms"] > ns["targets"] + ns["agents"] + ns["measure"], ns
    ratio = sum(ns.values()) / sum(cyc.values())
    assert 0.3 < ratio < 1.5, ratio  # ns per SM cycle: 1 / (0.67 .. 3.3 GHz)
    rep = benchmark_sps(cfg, 256, 4, warmup=2)
    assert rep["phase_ns"]["filter"] > 0 and rep["total_ns"] == sum(
        rep["phase_ns"][k] for k in ("targets", "agents", "measure", "filter", "comms", "observe", "reward"))


def test_multi_step_graph_equals_single_launches(cuda_device):
    """step_policy(n > 1) goes out as one CUDA graph of n cooperative launches
    (re-captured after a change to the launch state): the same batch as n
    single-step calls, across an auto-reset and an output-buffer switch."""
    from paper_2505_08222_b200.vecenv import VecEnv
    from test_gpu_parity import _to_py
    cfg = _to_py(default_config(n_agents=2, n_targets=2, pf_n_particles=1024, horizon=4))
    a, b = VecEnv(cfg, 33, 4), VecEnv(cfg, 33, 4)
    for policy, n in (("random", 3), ("scripted", 5), ("random", 3)):
        n0 = a.launch_count()
        a.step_policy(policy, n)
        assert a.launch_count() - n0 == n
        for _ in range(n):
            b.step_policy(policy, 1)
        assert np.array_equal(a.export_state(), b.export_state())
        ha, hb = a.host_outputs(), b.host_outputs()
        assert all(np.array_equal(ha[k], hb[k]) for k in ha)
    a.enable_phase_timing(True)  # changes the kernel parameters: the graph is re-captured
    b.enable_phase_timing(True)
    a.step_policy("random", 3)
    for _ in range(3):
        b.step_policy("random", 1)
    assert np.array_equal(a.export_state(), b.export_state())


def test_final_obs_rows_persist_across_buffer_sets(cuda_device):
    """Double-buffered outputs keep the single buffer's final_obs semantics: the
    terminal rows of an episode stay in final_obs through the following steps
    of either output set (the step copies the other set's rows of the envs that
    finished at the previous step), also across a switch from one to two sets."""
    from paper_2505_08222_b200.vecenv import VecEnv
    from test_gpu_parity import _to_py
    cfg = default_config(n_agents=2, n_targets=2, pf_n_particles=64, horizon=3)
    n = 6
    ora = Oracle(cfg, n, 31)
    gpu = VecEnv(_to_py(cfg), n, 31)
    for s in range(11):
        if s == 4:
            gpu.set_output_buffers(2)  # right after the terminal step 3
        ora.step_policy(1)
        gpu.step_policy("random", 1)
        got, want = gpu.host_outputs(["final_obs"])["final_obs"], ora.outputs()["final_obs"]
        np.testing.assert_allclose(got, want, rtol=1e-9, atol=1e-12, err_msg=f"step {s}")
        if s == 8:  # the zero-copy device view of the current set
            np.testing.assert_allclose(gpu.final_obs_stack().cpu().numpy().T, want, rtol=1e-9, atol=1e-12)


def test_invalid_action_with_double_buffered_outputs_moves_nothing(cuda_device):
    """The step kernel is gated on the validation result on the device (one host
    wait per step): an invalid action leaves the state, the current output set and
    the next valid step exactly as if the bad call had never been made, also with
    two output sets (the switch to the other set is undone)."""
    from paper_2505_08222_b200.vecenv import ContractViolation, VecEnv
    cfg = _to_py(default_config(n_agents=2, n_targets=2, pf_n_particles=1024, horizon=5))
    a, b = VecEnv(cfg, 6, 11), VecEnv(cfg, 6, 11)
    a.set_output_buffers(2)
    b.set_output_buffers(2)
    rng = np.random.default_rng(3)
    for s in range(7):  # crosses an auto-reset
        acts = random_legal_actions(a.host_outputs(["masks"])["masks"], rng).reshape(6, 2)
        if s in (2, 5):
            bad = acts.copy()
            bad[4, 1] = 7
            before = a.export_state()
            out_before = a.host_outputs()
            with pytest.raises(ContractViolation, match=r"^env 4: step: invalid action 7 for agent 1"):
                a.step(bad)
            assert np.array_equal(before, a.export_state())
            out_after = a.host_outputs()
            assert all(np.array_equal(out_before[k], out_after[k]) for k in out_before)
        a.step(acts)
        b.step(acts)
        assert np.array_equal(a.export_state(), b.export_state())
        ha, hb = a.host_outputs(), b.host_outputs()
        assert all(np.array_equal(ha[k], hb[k]) for k in ha)
