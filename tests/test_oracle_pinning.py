"""CPU: pin the oracle (oracle/ut_oracle.c, the plain-C restatement) to the
reference itself.

Three independent anchors:
  1. the reference's own VecEnv/Environment compiled from /root/reference
     against the Eigen shim (oracle/_ref/libutrack_ref.so) -- the restatement
     must be BIT-identical to it on every output and every state-blob word;
  2. the reference's own test suites (test_rng/kinematics/tracking/env/vecenv
     .cpp) built against the doctest shim -- every case passes except five that
     fail for reasons inside the reference;
  3. published known-answer vectors (Random123 Philox4x32-10) and the closed
     forms quoted by the reference tests.
The committed golden fixtures (tests/golden/, made by make_golden.py from
oracle/_ref) keep anchor 1 checkable where /root/reference is absent.
"""
import ctypes as C
import pathlib
import subprocess

import numpy as np
import pytest

from oracle_bindings import (ROOT, Oracle, OracleError, RefVecEnv, default_config, oracle_lib,
                             random_legal_actions, ref_available, ref_lib)

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")

# Small CPU-sized versions of the parity configs (tests/test_gpu_parity.py).
CONFIGS = {
    "c1_1v1_slow": dict(n_agents=1, n_targets=1, target_speed_frac=0.3, horizon=128, pf_n_particles=256),
    "c2_2v2_reset": dict(n_agents=2, n_targets=2, horizon=5, pf_n_particles=128),
    "c3_5v5_fast": dict(n_agents=5, n_targets=5, target_speed_frac=0.6, d_min=100.0, spawn_max_sep=400.0,
                        horizon=12, pf_n_particles=96),
    "c5_heavy": dict(n_agents=3, n_targets=2, comm_drop_prob=0.0, detection_range=1e9, comm_range=1e9,
                     target_speed_frac=0.5, target_speed_frac_max=0.8, horizon=9, pf_n_particles=64),
    "odd_p33_follow": dict(n_agents=2, n_targets=3, pf_n_particles=33, reward_mode=1, perturbation_std=0.05,
                           spawn_max_sep=400.0, horizon=7),
    "quiet": dict(n_agents=2, n_targets=2, comm_drop_prob=0.0, range_noise_std=0.0, target_speed_frac=0.0,
                  heading_noise_std=0.0, pf_n_particles=64, horizon=10),
}


def _bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


# VecEnv::step_policy (vecenv.cpp:117-142) refreshes only rewards, dones and
# masks; the reference leaves obs/global/final_obs/infos stale, so after a
# policy step only those three (and the full state) are compared.
POLICY_KEYS = ("rewards", "dones", "masks")


def _assert_same(ora, ref, tag, keys=None):
    oa, ra = ora.outputs(), ref.outputs()
    for k in keys or oa:
        assert _bits_equal(oa[k], ra[k]), f"{tag}: output {k} differs"
    for e in range(ora.n_envs):
        assert _bits_equal(ora.serialize(e), ref.serialize(e)), f"{tag}: state blob of env {e} differs"


# ------------------------------------------------------------------ anchor 3 --
RANDOM123_KAT = [  # (key, stream, block) -> Philox4x32-10 output, Random123 kat_vectors
    ((0, 0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((2**64 - 1, 2**64 - 1, 2**64 - 1), (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x299f31d0a4093822, 0x0370734413198a2e, 0x85a308d3243f6a88), (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
]


@pytest.mark.parametrize("case", range(len(RANDOM123_KAT)))
def test_philox_known_answers(case):
    (key, stream, block), want = RANDOM123_KAT[case]
    out = (C.c_uint32 * 4)()
    oracle_lib().uto_philox_block(key, stream, block, out)
    assert tuple(out) == want
    if ref_available():
        ref_lib().ref_philox_block(key, stream, block, out)
        assert tuple(out) == want


@needs_ref
def test_derive_key_matches_reference():
    rng = np.random.default_rng(5)
    for _ in range(200):
        a, b, c, d = (int(x) for x in rng.integers(0, 2**63, 4, dtype=np.int64))
        assert oracle_lib().uto_derive_key(a, b, c, d) == ref_lib().ref_derive_key(a, b, c, d)


def test_closed_forms():
    """test_env.cpp:36-56 closed forms through the public Python mirror (host-only)."""
    from paper_2505_08222_b200.vecenv import rudder_angle, valid_actions
    assert [rudder_angle(i) for i in range(5)] == pytest.approx([-0.24, -0.12, 0.0, 0.12, 0.24], abs=1e-15)
    assert list(valid_actions(0)) == [1, 1, 0, 0, 0]
    assert list(valid_actions(2)) == [0, 1, 1, 1, 0]
    assert list(valid_actions(4)) == [0, 0, 0, 1, 1]


def test_cr_math_check():
    """The oracle's fp32 log/cos/sin are correctly rounded on the whole noise grid
    (every u1/u2 the 24-bit draws can produce)."""
    exe = ROOT / "oracle" / "_build" / "cr_math_check"
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300, check=True).stdout
    assert '"log_mismatch": 0' in out and '"cos_mismatch": 0' in out and '"sin_mismatch": 0' in out


# ------------------------------------------------------------------ anchor 1 --
@needs_ref
@pytest.mark.parametrize("name", list(CONFIGS))
def test_restatement_bit_identical_to_reference(name):
    cfg = default_config(**CONFIGS[name])
    n_envs, seed = 3, 42
    ora, ref = Oracle(cfg, n_envs, seed), RefVecEnv(cfg, n_envs, seed, workers=1)
    _assert_same(ora, ref, f"{name}/ctor")
    rng = np.random.default_rng(1)
    for s in range(14):
        acts = random_legal_actions(ora.outputs()["masks"], rng)
        ora.step(acts)
        ref.step(acts)
        _assert_same(ora, ref, f"{name}/step{s}")
    for s in range(6):
        ora.step_policy(1)
        ref.step_policy(1)
        _assert_same(ora, ref, f"{name}/policy{s}", POLICY_KEYS)


@needs_ref
def test_reference_worker_count_invariance():
    """vecenv.hpp:18-23: bit-identical for any worker count (the oracle is serial)."""
    cfg = default_config(**CONFIGS["c2_2v2_reset"])
    ora, ref = Oracle(cfg, 8, 7), RefVecEnv(cfg, 8, 7, workers=4)
    for _ in range(8):
        ora.step_policy(1)
        ref.step_policy(1)
    _assert_same(ora, ref, "workers=4", POLICY_KEYS)


@needs_ref
def test_env_index_offset_is_global_keying():
    """A shard created with env_index_offset k equals envs [k, k+n) of the whole batch."""
    cfg = default_config(**CONFIGS["c2_2v2_reset"])
    whole = RefVecEnv(cfg, 6, 3)
    part = Oracle(cfg, 2, 3, env_index_offset=4)
    for e in range(2):
        assert _bits_equal(part.serialize(e), whole.serialize(4 + e))


@needs_ref
def test_state_injection_roundtrip_matches_reference():
    cfg = default_config(**CONFIGS["c5_heavy"])
    ora, ref = Oracle(cfg, 2, 9), RefVecEnv(cfg, 2, 9)
    for _ in range(3):
        ref.step_policy(1)
    for e in range(2):
        ora.deserialize(e, ref.serialize(e))
    ora.refresh_outputs()
    ref.refresh_outputs()
    # refresh_outputs (vecenv.cpp:145-150) re-gathers observations and masks only
    _assert_same(ora, ref, "injected", ("obs", "global_state", "masks"))
    acts = random_legal_actions(ora.outputs()["masks"], np.random.default_rng(3))
    ora.step(acts)
    ref.step(acts)
    _assert_same(ora, ref, "injected+1")


# ---------------------------------------------------------- error behaviour --
@needs_ref
def test_invalid_action_error_matches_reference():
    cfg = default_config(**CONFIGS["c2_2v2_reset"])
    ora, ref = Oracle(cfg, 3, 1), RefVecEnv(cfg, 3, 1)
    acts = random_legal_actions(ora.outputs()["masks"], np.random.default_rng(0))
    acts[2 * 2 + 1] = 7  # env 2, agent 1: out of range
    with pytest.raises(OracleError) as eo:
        ora.step(acts)
    with pytest.raises(OracleError) as er:
        ref.step(acts)
    assert eo.value.code == er.value.code == 1
    assert str(eo.value).split("] ", 1)[1].startswith("env 2: ")
    assert str(er.value).split("] ", 1)[1].startswith("env 2: ")


@needs_ref
def test_infeasible_spawn_is_config_error_in_both():
    cfg = default_config(n_agents=4, n_targets=4, spawn_min_sep=300.0, spawn_max_sep=310.0, pf_n_particles=16)
    with pytest.raises(OracleError) as eo:
        Oracle(cfg, 1, 0)
    with pytest.raises(OracleError) as er:
        RefVecEnv(cfg, 1, 0)
    assert eo.value.code == er.value.code == 2


@needs_ref
def test_truncated_blob_is_data_error_in_both():
    cfg = default_config(**CONFIGS["quiet"])
    ora, ref = Oracle(cfg, 1, 0), RefVecEnv(cfg, 1, 0)
    blob = ora.serialize(0)[:-3]
    for impl in (ora, ref):
        with pytest.raises(OracleError) as ei:
            impl.deserialize(0, blob)
        assert ei.value.code == 3


@needs_ref
@pytest.mark.parametrize("field,value", [("n_agents", 0), ("n_targets", 0), ("dt", 0.0), ("pf_n_particles", 0),
                                         ("comm_drop_prob", 1.5), ("horizon", 0)])
def test_config_errors_name_the_field(field, value):
    cfg = default_config(**{field: value})
    rc_o = oracle_lib().uto_config_finalize(C.byref(cfg))
    msg_o = oracle_lib().uto_last_error().decode()
    cfg = default_config(**{field: value})
    rc_r = ref_lib().ref_config_finalize(C.byref(cfg))
    msg_r = ref_lib().ref_last_error().decode()
    assert rc_o == rc_r == 2
    assert msg_o == msg_r


@needs_ref
def test_finalize_resolves_heading_model_like_reference():
    """Default heading model: the reference's OLS fit (kinematics.cpp:58-111) -> (a, b)."""
    a, b = default_config(), default_config()
    assert oracle_lib().uto_config_finalize(C.byref(a)) == 0
    assert ref_lib().ref_config_finalize(C.byref(b)) == 0
    assert bytes(a) == bytes(b)


# ------------------------------------------------------------------ anchor 2 --
# The five reference cases that fail in every build we can make here, and why
# (DESIGN.md "Oracle"): three are defects in the tests themselves, two are
# statistical thresholds of the reference PF.
KNOWN_REFERENCE_FAILURES = {
    "test_kinematics": {"zero speed still rotates", "displacement magnitude is exactly speed*dt"},
    "test_tracking": {"noiseless convergence: under 2 m for 95 percent of seeds",
                      "trilateration agrees with the particle-filter limit"},
    "test_env": {"detection threshold is 450 m on the true 3D distance"},
    "test_rng": set(),
    "test_vecenv": set(),
}


@needs_ref
@pytest.mark.parametrize("suite", sorted(KNOWN_REFERENCE_FAILURES))
def test_reference_suite(suite):
    exe = ROOT / "oracle" / "_ref" / suite
    if not exe.exists():
        pytest.skip(f"{exe} not built")
    p = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    failed = {ln.split("FAILED: ", 1)[1].strip() for ln in p.stdout.splitlines() + p.stderr.splitlines()
              if "[doctest-shim] FAILED: " in ln}
    assert failed == KNOWN_REFERENCE_FAILURES[suite], p.stdout[-2000:]


# ------------------------------------------------------------ golden files --
GOLDEN = sorted((ROOT / "tests" / "golden").glob("*.npz"))


@pytest.mark.parametrize("path", GOLDEN, ids=[p.stem for p in GOLDEN])
def test_oracle_matches_golden(path):
    """Fixtures recorded from oracle/_ref by tests/golden/make_golden.py."""
    from golden.make_golden import replay
    g = np.load(path)
    got = replay(lambda cfg, n, seed: Oracle(cfg, n, seed), g)
    for k in g.files:
        if k.startswith("out_") or k.startswith("blob_"):
            assert _bits_equal(got[k], g[k]), f"{path.stem}: {k}"
