"""GPU parity: the B200 step (through the C-ABI) against the CPU oracle.

Bar (BASELINE north_star): integer state bit-exact; floating
point within NORTH_STAR_RTOL = 1e-5 relative per step -- and, in practice, within
TIGHT_RTOL = 1e-9 (element-wise particle math is bit-identical; only reduction
order and fp64 libm ulps differ).
"""
import ctypes as C

import numpy as np
import pytest

from oracle_bindings import (Oracle, RefVecEnv, default_config, oracle_lib, random_legal_actions,
                             ref_available)
from parity import NORTH_STAR_RTOL, TIGHT_RTOL, Report, compare_blobs, compare_outputs

pytestmark = pytest.mark.gpu


def _product():
    from paper_2505_08222_b200 import _abi, _native
    lib = _native.lib()
    _abi.declare_debug(lib)
    return lib


def make_pair(cfg_kw, n_envs, seed, offset=0):
    from paper_2505_08222_b200.vecenv import VecEnv
    cfg = default_config(**cfg_kw)
    ora = Oracle(cfg, n_envs, seed, offset)
    gpu = VecEnv(_to_py(cfg), n_envs, seed, env_index_offset=offset)
    return cfg, ora, gpu


def _to_py(c):
    from paper_2505_08222_b200.vecenv import EnvConfig, PfConfig
    kw = {f: getattr(c, f) for f in (
        "n_agents", "n_targets", "horizon", "dt", "agent_speed", "target_speed_frac", "target_speed_frac_max",
        "target_turn_interval", "detection_range", "comm_range", "comm_drop_prob", "range_noise_std", "eps_min",
        "eps_max", "d_min", "d_safe", "spawn_min_sep", "spawn_max_sep", "perturbation_std", "target_depth_min",
        "target_depth_max", "lost_steps", "heading_noise_std")}
    kw["reward_mode"] = "follow" if c.reward_mode == 1 else "tracking"
    kw["pf"] = PfConfig(c.pf.n_particles, c.pf.process_noise_pos, c.pf.process_noise_vel, c.pf.speed_margin,
                        c.pf.init_radius)
    if c.heading_model_kind == 1:
        kw["heading_bucket"] = (c.heading_a, c.heading_b)
    return EnvConfig(**kw)


def check_state(ora, gpu, rep, tag, outputs=True, skip=()):
    A, T, P = ora.A, ora.T, ora.P
    for e in range(ora.n_envs):
        compare_blobs(gpu.serialize_state(e), ora.serialize(e), A, T, P, rep, tag=f"{tag}/env{e}")
    if outputs:
        compare_outputs(gpu.host_outputs(), ora.outputs(), rep, tag=tag, skip=skip)
    return rep


CONFIGS = {
    "c1_1v1_slow": dict(n_agents=1, n_targets=1, target_speed_frac=0.3, horizon=128, pf_n_particles=1024),
    "small_2v1_p64": dict(n_agents=2, n_targets=1, horizon=6, pf_n_particles=64, target_speed_frac=0.4),
    "c2_2v2": dict(n_agents=2, n_targets=2, horizon=25, pf_n_particles=256),
    "c3_5v5_fast": dict(n_agents=5, n_targets=5, target_speed_frac=0.6, d_min=100.0, spawn_max_sep=400.0,
                        horizon=12, pf_n_particles=1024),
    "c5_heavy_p512": dict(n_agents=3, n_targets=2, comm_drop_prob=0.0, detection_range=1e9, comm_range=1e9,
                          target_speed_frac=0.5, target_speed_frac_max=0.8, horizon=9, pf_n_particles=512),
    "odd_p33_follow": dict(n_agents=2, n_targets=3, pf_n_particles=33, reward_mode=1, perturbation_std=0.05,
                           spawn_max_sep=400.0, horizon=7),
    "quiet_p64": dict(n_agents=2, n_targets=2, comm_drop_prob=0.0, range_noise_std=0.0, target_speed_frac=0.0,
                      heading_noise_std=0.0, pf_n_particles=64, horizon=10),
}


@pytest.mark.parametrize("name", list(CONFIGS))
def test_ctor_matches_oracle(cuda_device, name):
    cfg, ora, gpu = make_pair(CONFIGS[name], 3, 42)
    rep = check_state(ora, gpu, Report(), "ctor", skip=("final_obs",))
    assert not rep.int_mismatch, rep
    assert rep.worst() <= TIGHT_RTOL, rep


@pytest.mark.parametrize("name", list(CONFIGS))
def test_step_external_actions(cuda_device, name):
    cfg, ora, gpu = make_pair(CONFIGS[name], 3, 7)
    rng = np.random.default_rng(1)
    rep = Report()
    steps = 30 if cfg.pf.n_particles <= 256 else 15
    for s in range(steps):
        acts = random_legal_actions(ora.outputs()["masks"], rng)
        ora.step(acts)
        gpu.step(acts)
        check_state(ora, gpu, rep, f"step{s}")
        assert not rep.int_mismatch, rep
    assert rep.worst() <= TIGHT_RTOL, rep


@pytest.mark.parametrize("name", ["small_2v1_p64", "c2_2v2", "c5_heavy_p512"])
def test_step_policy_random(cuda_device, name):
    cfg, ora, gpu = make_pair(CONFIGS[name], 4, 99)
    rep = Report()
    for s in range(20):
        ora.step_policy(1)
        gpu.step_policy("random", 1)
        check_state(ora, gpu, rep, f"pol{s}")
        assert not rep.int_mismatch, rep
    assert rep.worst() <= TIGHT_RTOL, rep


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_scripted_policy_vs_reference(cuda_device):
    from paper_2505_08222_b200.vecenv import VecEnv
    cfg = default_config(n_agents=2, n_targets=2, pf_n_particles=128, horizon=9)
    ref = RefVecEnv(cfg, 3, 5)
    gpu = VecEnv(_to_py(cfg), 3, 5)
    rep = Report()
    for s in range(20):
        ref._check(ref.lib.ref_vecenv_step_policy(ref.h, 1, 1))
        gpu.step_policy("scripted", 1)
        for e in range(3):
            compare_blobs(gpu.serialize_state(e), ref.serialize(e), ref.A, ref.T, ref.P, rep, tag=f"s{s}e{e}")
        assert not rep.int_mismatch, rep
    assert rep.worst() <= TIGHT_RTOL, rep


def test_state_injection_from_reference_blobs(cuda_device):
    """Per-step parity from injected state (Appendix C level 2)."""
    from paper_2505_08222_b200.vecenv import VecEnv
    cfg = default_config(**CONFIGS["c2_2v2"])
    ora = Oracle(cfg, 2, 11)
    gpu = VecEnv(_to_py(cfg), 2, 11)
    rng = np.random.default_rng(3)
    rep = Report()
    for s in range(60):
        acts = random_legal_actions(ora.outputs()["masks"], rng)
        if s in (0, 1, 17, 24, 25, 40):
            for e in range(2):
                gpu.deserialize_state(e, ora.serialize(e))
            gpu.refresh_outputs()
        ora.step(acts)
        gpu.step(acts)
        check_state(ora, gpu, rep, f"inj{s}")
        assert not rep.int_mismatch, rep
    assert rep.worst() <= TIGHT_RTOL, rep


def test_long_free_running_integer_state(cuda_device):
    """1100 free-running steps across auto-resets (Appendix C level 3)."""
    cfg, ora, gpu = make_pair(dict(n_agents=2, n_targets=2, horizon=1000, pf_n_particles=128), 2, 2024)
    rep = Report()
    for chunk in range(11):
        ora.step_policy(100)
        gpu.step_policy("random", 100)
        check_state(ora, gpu, rep, f"t{(chunk + 1) * 100}")
        assert not rep.int_mismatch, rep
    assert rep.worst() <= NORTH_STAR_RTOL, rep


def test_shards_equal_whole_batch(cuda_device):
    """Any partitioning of envs over devices/shards gives identical bits (level 4)."""
    from paper_2505_08222_b200.vecenv import VecEnv
    cfg = _to_py(default_config(n_agents=2, n_targets=2, pf_n_particles=256, horizon=8))
    whole = VecEnv(cfg, 6, 77)
    parts = [VecEnv(cfg, 2, 77, env_index_offset=2 * i) for i in range(3)]
    for _ in range(12):
        whole.step_policy("random", 1)
        for p in parts:
            p.step_policy("random", 1)
    for e in range(6):
        assert np.array_equal(whole.serialize_state(e), parts[e // 2].serialize_state(e % 2))


def test_mixed_fleet_matches_single_env_oracles(cuda_device):
    from paper_2505_08222_b200.vecenv import VecEnv
    kws = [dict(n_agents=1, n_targets=1), dict(n_agents=2, n_targets=3, spawn_max_sep=400.0),
           dict(n_agents=3, n_targets=2, spawn_max_sep=400.0)]
    kws = [dict(k, pf_n_particles=128, horizon=7) for k in kws]
    cfgs = [default_config(**k) for k in kws]
    fleet = [0, 1, 2, 1, 0, 2]
    gpu = VecEnv([_to_py(c) for c in cfgs], len(fleet), 3, fleet=fleet)
    oras = [Oracle(cfgs[f], 1, 3, env_index_offset=e) for e, f in enumerate(fleet)]
    rep = Report()
    for s in range(10):
        gpu.step_policy("random", 1)
        for o in oras:
            o.step_policy(1)
        for e, o in enumerate(oras):
            compare_blobs(gpu.serialize_state(e), o.serialize(0), o.A, o.T, o.P, rep, tag=f"m{s}e{e}")
        assert not rep.int_mismatch, rep
    assert rep.worst() <= TIGHT_RTOL, rep


def test_invalid_action_is_contract_violation_and_steps_nothing(cuda_device):
    from paper_2505_08222_b200.vecenv import ContractViolation
    cfg, ora, gpu = make_pair(CONFIGS["small_2v1_p64"], 3, 1)
    before = [gpu.serialize_state(e) for e in range(3)]
    acts = np.full((3, 2), 2, np.int32)
    acts[1, 1] = 0  # rudder 2 -> 0 jumps two notches (test_env.cpp:176-185)
    with pytest.raises(ContractViolation, match=r"env 1: step: invalid action 0 for agent 1 at rudder index 2"):
        gpu.step(acts)
    for e in range(3):
        assert np.array_equal(before[e], gpu.serialize_state(e))
    with pytest.raises(ContractViolation):
        gpu.step(np.full((3, 2), 5, np.int32))


def test_infeasible_spawn_is_config_error(cuda_device):
    from paper_2505_08222_b200.vecenv import ConfigError, EnvConfig, VecEnv
    with pytest.raises(ConfigError, match="spawn infeasible"):
        VecEnv(EnvConfig(n_agents=5, n_targets=5, spawn_min_sep=95.0, spawn_max_sep=100.0), 2, 1)


def test_serialize_roundtrip_and_errors(cuda_device):
    from paper_2505_08222_b200.vecenv import DataError, EnvConfig, VecEnv
    v = VecEnv(EnvConfig(n_agents=2, n_targets=1), 2, 4)
    v.step_policy("random", 5)
    b = v.serialize_state(1)
    v.deserialize_state(0, b)
    assert np.array_equal(v.serialize_state(0), b)
    with pytest.raises(DataError, match="truncated"):
        v.deserialize_state(0, b[:-1])
    with pytest.raises(DataError, match="trailing"):
        v.deserialize_state(0, np.concatenate([b, [0.0]]))


def test_auto_reset_surfaces_final_obs(cuda_device):
    """test_vecenv.cpp:114-124 on the device."""
    from paper_2505_08222_b200.vecenv import EnvConfig, PfConfig, VecEnv
    v = VecEnv(EnvConfig(n_agents=2, n_targets=1, horizon=3, pf=PfConfig(n_particles=64)), 2, 5)
    rng = np.random.default_rng(2)
    for _ in range(3):
        v.step(random_legal_actions(v.host_outputs(["masks"])["masks"], rng))
    o = v.host_outputs()
    assert o["dones"][0] == 1 and o["step"][0] == 0
    assert not np.array_equal(o["final_obs"], o["obs"])


def test_device_stats_match_oracle(cuda_device):
    cfg, ora, gpu = make_pair(dict(n_agents=2, n_targets=2, horizon=10, pf_n_particles=128), 5, 8)
    ora.step_policy(25)
    gpu.step_policy("random", 25)
    a, b = gpu.stats(), ora.stats()
    # all but slot 9 (device-only: sets that took the exact update path); slots
    # 10.. are curriculum::evaluate's accumulators
    keep = np.arange(a.size) != 9
    assert np.allclose(a[keep], b[keep], rtol=1e-12, atol=1e-12), (a, b)
    assert b[3] == 10 and b[10] > 0 and b[12] > 0
    m = gpu.eval_metrics()
    assert m["episodes"] == 10 and 0 <= m["collision_pct"] <= 100 and m["dist_std"] >= 0


def test_cr_math_exhaustive_on_device(cuda_device):
    """Device fp32 noise math == oracle (correctly rounded log/cos/sin, IEEE sqrt)
    on every value the 24-bit draws can produce: 4 x 2^24 grid points."""
    lib = _product()
    o = oracle_lib()
    want = np.empty(1 << 24, np.float32)
    got = np.empty(1 << 24, np.float32)
    for kind in range(4):  # log, cos, sin, Box-Muller radius sqrt(-2 log u1)
        o.uto_cr_grid(kind, want.ctypes.data)
        # kind: fp64-libm reference path; kind + 4: the table-driven production path
        for dev_kind in (kind, kind + 4):
            assert lib.ut_debug_cr_grid(dev_kind, 0, got.ctypes.data) == 0
            bad = np.flatnonzero(got.view(np.uint32) != want.view(np.uint32))
            assert bad.size == 0, (dev_kind, bad[:10])


def test_philox_and_keys_on_device(cuda_device):
    lib = _product()
    o = oracle_lib()
    rng = np.random.default_rng(0)
    for _ in range(20):
        key, stream, b0 = (int(x) for x in rng.integers(0, 2**63, 3, dtype=np.uint64))
        n = 1000
        got = np.empty(4 * n, np.uint32)
        assert lib.ut_debug_philox(key, stream, b0, n, 0, got.ctypes.data) == 0
        want = np.empty(4, np.uint32)
        for i in (0, 1, 517, n - 1):
            o.uto_philox_block(key, stream, b0 + i, want.ctypes.data_as(C.POINTER(C.c_uint32)))
            assert np.array_equal(got[4 * i:4 * i + 4], want)
        out = C.c_uint64()
        a, b, c, d = (int(x) for x in rng.integers(0, 2**63, 4, dtype=np.uint64))
        assert lib.ut_debug_derive_key(a, b, c, d, 0, C.byref(out)) == 0
        assert out.value == o.uto_derive_key(a, b, c, d)


@pytest.mark.parametrize("kind", [0, 1], ids=["sqrt", "div"])
def test_speed_clamp_arithmetic_is_ieee(cuda_device, kind):
    """The branch-free fp64 sqrt / division of the speed clamp == IEEE on 2^28
    random operands of its domain (the particle state must stay bit-exact)."""
    lib = _product()
    bad = C.c_uint64(1)
    assert lib.ut_debug_ieee_check(kind, 12345, 1 << 28, 0, C.byref(bad)) == 0
    assert bad.value == 0


def test_likelihood_distance_sqrt_within_one_ulp(cuda_device):
    """The likelihood distance sqrt (sqrt_dist: rsqrt seed, one Goldschmidt step,
    residual correction) is within 1 ulp of IEEE on 2^28 squared distances; only
    the particle weights use it (weights carry rounding anyway)."""
    lib = _product()
    bad = C.c_uint64(1)
    assert lib.ut_debug_ieee_check(2, 4242, 1 << 28, 0, C.byref(bad)) == 0
    assert bad.value == 0


def test_batched_state_export_import(cuda_device):
    """ut_vecenv_export_state / import_state (checkpoint path) ==
    per-env serialize / deserialize, bit for bit, and an import restores state."""
    from paper_2505_08222_b200.vecenv import DataError
    cfg, ora, gpu = make_pair(CONFIGS["c2_2v2"], 5, 21)
    gpu.step_policy("random", 4)
    blobs = gpu.export_state()
    assert blobs.shape == (5, gpu.serialize_state(0).size)
    for e in range(5):
        assert blobs[e].tobytes() == gpu.serialize_state(e).tobytes()
    part = gpu.export_state(1, 4)
    assert part.tobytes() == blobs[1:4].tobytes()
    # import the oracle's state into envs 1..3 and compare with per-env injection
    ora.step_policy(2)
    src = np.stack([ora.serialize(e) for e in range(1, 4)])
    gpu.import_state(src, 1, 4)
    for i, e in enumerate(range(1, 4)):
        assert gpu.serialize_state(e).tobytes() == src[i].tobytes()
    with pytest.raises(DataError):
        gpu.import_state(src[:, :-1], 1, 4)


def test_batched_state_export_mixed_fleet(cuda_device):
    from paper_2505_08222_b200.vecenv import VecEnv
    cfgs = [_to_py(default_config(n_agents=1, n_targets=2, pf_n_particles=64)),
            _to_py(default_config(n_agents=3, n_targets=1, pf_n_particles=64))]
    fleet = [0, 1, 1, 0, 1]
    gpu = VecEnv(cfgs, len(fleet), 5, fleet=fleet)
    gpu.step_policy("random", 3)
    flat = gpu.export_state()
    want = np.concatenate([gpu.serialize_state(e) for e in range(len(fleet))])
    assert flat.tobytes() == want.tobytes()
    gpu.import_state(flat)
    assert gpu.export_state().tobytes() == want.tobytes()


def test_output_double_buffering_and_async_copies(cuda_device):
    """set_output_buffers(2) + copy_outputs_async: every step's outputs arrive
    intact while the next step writes the other buffer set."""
    import torch
    cfg, ora, gpu = make_pair(CONFIGS["c2_2v2"], 6, 31)
    gpu.set_output_buffers(2)
    side = torch.cuda.Stream()
    rng = np.random.default_rng(4)
    names = ["obs", "global_state", "rewards", "dones", "masks", "tracking_error", "step"]
    pending = None
    for s in range(8):
        acts = random_legal_actions(ora.outputs()["masks"], rng)
        ora.step(acts)
        gpu.step(acts)
        if pending is not None:  # the previous step's async copy, read after this step ran
            side.synchronize()
            host, want = pending
            for k in names:
                np.testing.assert_allclose(host[k].numpy(), want[k], rtol=TIGHT_RTOL, atol=1e-12, err_msg=k)
        want = {k: v.copy() for k, v in ora.outputs().items()}
        host = {k: torch.empty(want[k].shape, dtype=torch.from_numpy(want[k]).dtype, pin_memory=True)
                for k in names}
        gpu.copy_outputs_async(host, side.cuda_stream)
        pending = (host, want)
        rep = check_state(ora, gpu, Report(), f"db{s}", outputs=False)
        assert rep.ok(TIGHT_RTOL), rep
    side.synchronize()
    gpu.set_output_buffers(1)
    compare_outputs(gpu.host_outputs(), ora.outputs(), rep := Report(), tag="single")
    assert rep.ok(TIGHT_RTOL), rep


def test_trajectory_capture_matches_state(cuda_device, tmp_path):
    """ut_vecenv_capture_trajectory == append_trajectory_rows (trajectory.cpp:13-66)
    computed from the oracle's state after each step; the terminal step is
    captured before the auto-reset; CSV in the reference layout."""
    from paper_2505_08222_b200.trajectory import HEADER, write_trajectory_csv
    A, T, P = 2, 3, 64
    kw = dict(n_agents=A, n_targets=T, pf_n_particles=P, horizon=5, spawn_max_sep=400.0)
    cfg, ora, gpu = make_pair(kw, 4, 17)
    gpu.capture_trajectory(1, 3)
    rng = np.random.default_rng(2)
    steps = []
    for s in range(5):
        acts = random_legal_actions(ora.outputs()["masks"], rng)
        ora.step(acts)
        gpu.step(acts)
        rows = gpu.trajectory_rows()
        assert rows.shape == (2, A + T, 12)
        steps.append(rows[0].copy())
        out = gpu.host_outputs()
        for i, e in enumerate((1, 2)):
            assert np.all(rows[i, :, 0] == s + 1)
            np.testing.assert_array_equal(rows[i, :, 9], out["rewards"][e])
            np.testing.assert_array_equal(rows[i, A:, 8], out["tracking_error"][e * T:(e + 1) * T])
            if s == 4:
                continue  # terminal step: the state has been reset since
            b = ora.serialize(e)
            base = lambda a: 5 + 6 * A + 9 * T + a * (6 * A + T * (9 + 5 * P))
            for a in range(A):
                np.testing.assert_allclose(rows[i, a, 1:5], b[5 + 6 * a:5 + 6 * a + 4], rtol=TIGHT_RTOL, atol=1e-12)
            for t in range(T):
                tv = b[5 + 6 * A + 8 * t:5 + 6 * A + 8 * t + 4]
                np.testing.assert_allclose(rows[i, A + t, 1:5], tv, rtol=TIGHT_RTOL, atol=1e-12)
                ests = [b[base(a) + 6 * A + t * (9 + 5 * P):][:2] for a in range(A)]
                errs = [np.sqrt((ex - tv[0]) ** 2 + (ey - tv[1]) ** 2) for ex, ey in ests]
                best = int(np.argmin(errs))
                np.testing.assert_allclose(rows[i, A + t, 6:8], ests[best], rtol=TIGHT_RTOL, atol=1e-12)
                assert rows[i, A + t, 5] == 1 and rows[i, A + t, 11] == 1
    path = tmp_path / "traj" / "episode_0001.csv"
    write_trajectory_csv(str(path), steps)
    lines = path.read_text().splitlines()
    assert lines[0] == HEADER and len(lines) == 1 + 5 * (A + T)
    assert all(len(ln.split(",")) == 12 for ln in lines)
    assert lines[1].startswith("1,agent_0,agent,") and lines[A + 1].startswith("1,target_0,target,")
    gpu.capture_trajectory(0, 0)
    assert gpu.trajectory_rows().size == 0


def test_c3_at_scale_against_oracle(cuda_device):
    """C3 (5 agents vs 5 fast targets, P = 1024) on 96 envs for 16 steps: every
    output each step and every state word at the end against the oracle."""
    cfg, ora, gpu = make_pair(dict(CONFIGS["c3_5v5_fast"], horizon=128), 96, 7)
    rep = Report()
    for s in range(16):
        ora.step_policy(1)
        gpu.step_policy("random", 1)
        compare_outputs(gpu.host_outputs(), ora.outputs(), rep, tag=f"s{s}")
    check_state(ora, gpu, rep, "final", outputs=False)
    assert rep.ok(TIGHT_RTOL), rep
