"""GPU parity at the benchmark shapes: every device path the benchmarks run is
compared with the CPU oracle (VERDICT r01 "next" item 1).

* C4 mixed fleets through the FULL (TMA, P = 1024) step instance, fleets up to
  8 x 8, one of them estimator-heavy so a set applies kMaxMerged = 8 updates.
* C5 at its real shape: 5 v 5, drop 0, ranges 1e9, P = 1024 -> 5 updates per set.
* the exact sequential update path forced on C3 (ut_debug_set_knobs).
* a 1000-step free-running C3 run (horizon 128, so ~7 auto-resets) with the
  first-divergence step and the maximum relative difference of every field.

Integer state bit-exact; floating point within TIGHT_RTOL = 1e-9 relative per
step (tests/parity.py: per-field floors, weights held to 1e-12 / P), and the
north-star 1e-5 bound over the 1000-step run.
"""
import ctypes as C
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from oracle_bindings import Oracle, default_config
from parity import (NORTH_STAR_RTOL, TIGHT_RTOL, Report, compare_blobs, compare_outputs, blob_floors,
                    blob_spec, output_floor, rel_err, INT_OUTPUTS, FLOAT_OUTPUTS)
from test_gpu_parity import _to_py

pytestmark = pytest.mark.gpu

C3 = dict(n_agents=5, n_targets=5, target_speed_frac=0.6, d_min=100.0, spawn_max_sep=400.0, horizon=128,
          pf_n_particles=1024)
HEAVY = dict(comm_drop_prob=0.0, detection_range=1e9, comm_range=1e9)


def _debug_lib():
    from paper_2505_08222_b200 import _abi, _native
    lib = _native.lib()
    _abi.declare_debug(lib)
    return lib


def _instance(gpu):
    full, np_ = C.c_int32(), C.c_int32()
    assert _debug_lib().ut_debug_instance(gpu._h, C.byref(full), C.byref(np_)) == 0
    return full.value, np_.value


class ShardedOracle:
    """The C restatement over [0, n) in `k` shards stepped on host threads (ctypes
    releases the GIL); every stream is keyed by the global env index, so the
    shards together are the whole batch."""

    def __init__(self, cfg, n_envs, seed, k=4):
        k = max(1, min(k, n_envs))
        base, extra = divmod(n_envs, k)
        self.parts, lo = [], 0
        for i in range(k):
            hi = lo + base + (1 if i < extra else 0)
            self.parts.append((Oracle(cfg, hi - lo, seed, env_index_offset=lo), lo, hi))
            lo = hi
        self.pool = ThreadPoolExecutor(k)
        self.A, self.T, self.P, self.n_envs = cfg.n_agents, cfg.n_targets, cfg.pf.n_particles, n_envs

    def step_policy(self, n=1):
        list(self.pool.map(lambda p: p[0].step_policy(n), self.parts))

    def outputs(self):
        outs = [p[0].outputs() for p in self.parts]
        return {k: np.concatenate([o[k] for o in outs], axis=outs[0][k].ndim - 1) for k in outs[0]}

    def serialize(self, e):
        for o, lo, hi in self.parts:
            if lo <= e < hi:
                return o.serialize(e - lo)
        raise IndexError(e)

    def stats(self):
        return sum(p[0].stats() for p in self.parts)

    def close(self):
        self.pool.shutdown()
        for p in self.parts:
            p[0].close()


def _mix_shapes():
    # (A, T, heavy): 8x8 heavy -> own + 7 fused updates = kMaxMerged per set
    return [(8, 8, True), (8, 8, False), (1, 1, False), (3, 5, False), (5, 3, False), (2, 7, False),
            (7, 2, False), (4, 4, False), (1, 8, False), (8, 1, True), (6, 6, False), (5, 5, True)]


def test_c4_mixed_fleets_through_full_instance(cuda_device):
    """C4: per-env fleets 1..8 x 1..8 (spawn_max_sep 600) in ONE batch on the
    FULL P = 1024 instance (ragged set offsets, 8x8 padding), across an
    auto-reset, each env against a standalone oracle Environment."""
    from paper_2505_08222_b200.vecenv import VecEnv
    shapes = _mix_shapes()
    cfgs = [default_config(n_agents=a, n_targets=t, spawn_max_sep=600.0, horizon=6, pf_n_particles=1024,
                           **(HEAVY if h else {})) for a, t, h in shapes]
    fleet = list(range(len(shapes)))
    seed = 13
    gpu = VecEnv([_to_py(c) for c in cfgs], len(fleet), seed, fleet=fleet)
    assert _instance(gpu) == (1, 1024)
    oras = [Oracle(cfgs[f], 1, seed, env_index_offset=e) for e, f in enumerate(fleet)]
    pool = ThreadPoolExecutor(6)
    rep = Report()
    for s in range(8):  # horizon 6: steps 7-8 run after the auto-reset
        gpu.step_policy("random", 1)
        list(pool.map(lambda o: o.step_policy(1), oras))
        out = gpu.host_outputs(["rewards", "dones", "step"])
        for e, o in enumerate(oras):
            compare_blobs(gpu.serialize_state(e), o.serialize(0), o.A, o.T, o.P, rep, tag=f"m{s}e{e}")
            w = o.outputs()
            assert out["dones"][e] == w["dones"][0] and out["step"][e] == w["step"][0], (s, e)
            r = rel_err(out["rewards"][e], w["rewards"][0])
            rep.max_rel["out.rewards"] = max(rep.max_rel.get("out.rewards", 0.0), float(r))
        assert not rep.int_mismatch, rep
    pool.shutdown()
    want = sum(o.stats() for o in oras)
    got = gpu.stats()
    assert got[7] == want[7] and got[8] == want[8], (got[7:9], want[7:9])  # updates, resamples
    assert rep.worst() <= TIGHT_RTOL, rep


def test_kmaxmerged_update_count_on_heavy_8x8(cuda_device):
    """Every set of an estimator-heavy 8 x 8 fleet applies own + 7 fused updates
    = kMaxMerged = 8 per step on the merged path (no exact fallback needed)."""
    from paper_2505_08222_b200.vecenv import VecEnv
    cfg = default_config(n_agents=8, n_targets=8, spawn_max_sep=600.0, pf_n_particles=1024, **HEAVY)
    gpu = VecEnv(_to_py(cfg), 4, 3)
    assert _instance(gpu) == (1, 1024)
    gpu.step_policy("random", 3)
    st = gpu.stats()
    assert st[7] == 4 * 64 * 3 * 8, st[7]


def test_c5_real_shape(cuda_device):
    """C5: 5 v 5 estimator-heavy (drop 0, ranges 1e9, P = 1024): 5 updates per
    set per step; 64 envs, every output each step, every state word at the end."""
    from paper_2505_08222_b200.vecenv import VecEnv
    cfg = default_config(**C3, **HEAVY)
    n, steps = 64, 6
    ora = ShardedOracle(cfg, n, 5)
    gpu = VecEnv(_to_py(cfg), n, 5)
    assert _instance(gpu) == (1, 1024)
    rep = Report()
    for s in range(steps):
        ora.step_policy(1)
        gpu.step_policy("random", 1)
        compare_outputs(gpu.host_outputs(), ora.outputs(), rep, tag=f"s{s}", skip=("final_obs",))
        assert not rep.int_mismatch, rep
    for e in range(n):
        compare_blobs(gpu.serialize_state(e), ora.serialize(e), 5, 5, 1024, rep, tag=f"e{e}")
    st = gpu.stats()
    assert st[7] == n * 25 * steps * 5, st[7] / (n * 25 * steps)
    np.testing.assert_array_equal(st[7:9], ora.stats()[7:9])
    ora.close()
    assert rep.ok(TIGHT_RTOL), rep


def test_forced_exact_update_path_c3(cuda_device):
    """The exact sequential update (tracking.cpp:119-143 once per measurement)
    forced on every set of C3 with P = 1024 -- the fallback the merged pass
    takes when an underflow could matter (the C5 bench takes it ~70k times)."""
    from paper_2505_08222_b200.vecenv import VecEnv
    cfg = default_config(**C3)
    n = 32
    ora = ShardedOracle(cfg, n, 21)
    gpu = VecEnv(_to_py(cfg), n, 21)
    assert _debug_lib().ut_debug_set_knobs(gpu._h, 1, -1) == 0
    rep = Report()
    for s in range(8):
        ora.step_policy(1)
        gpu.step_policy("random", 1)
        compare_outputs(gpu.host_outputs(), ora.outputs(), rep, tag=f"x{s}", skip=("final_obs",))
        assert not rep.int_mismatch, rep
    for e in range(n):
        compare_blobs(gpu.serialize_state(e), ora.serialize(e), 5, 5, 1024, rep, tag=f"e{e}")
    st = gpu.stats()
    # every set with at least one update took the exact path
    assert st[9] > 0 and st[7] >= st[9]
    np.testing.assert_array_equal(st[7:9], ora.stats()[7:9])
    ora.close()
    assert rep.ok(TIGHT_RTOL), rep


# ---------------------------------------------------------------- drift ----
# env-stream integer state: bit-exact over the whole run (SURVEY App. C level 3)
ENV_INT_GROUPS = ("step", "env_rng_pos", "env_rng_have_spare", "agent.rudder", "target.rudder",
                  "target.countdown", "target.miss_streak", "info.age", "info.valid", "track.age",
                  "track.ever", "pf.rng_have_spare")
# kinematic floats: depend only on the env stream (bit-exact in practice)
KIN_GROUPS = ("episode_target_speed", "env_rng_spare", "agent.x", "agent.y", "agent.z", "agent.heading",
              "agent.speed", "target.x", "target.y", "target.z", "target.heading", "target.speed",
              "target.cmd_heading", "info.x", "info.y", "info.z", "info.heading")


def test_c3_drift_1000_steps(cuda_device):
    """C3 (5 v 5 fast, P = 1024) free-running for 1000 steps (~7 auto-resets)
    against the oracle: env-stream integer state and every integer output
    bit-exact at every step; every float within the north-star 1e-5 bound at
    every step; the first step at which each field leaves the 1e-9 tight bound
    (the PF-derived ones can only do so after a resample index flip) reported."""
    from paper_2505_08222_b200.vecenv import VecEnv
    cfg = default_config(**C3)
    n, steps, blob_every = 16, 1000, 25
    ora = ShardedOracle(cfg, n, 2505)
    gpu = VecEnv(_to_py(cfg), n, 2505)
    names, ints = blob_spec(5, 5, 1024)
    fl = ~ints
    floors = blob_floors(names[fl], 1024)
    first_div, max_rel, int_bad = {}, {}, []
    pf_pos_first = None
    for s in range(1, steps + 1):
        ora.step_policy(1)
        gpu.step_policy("random", 1)
        got, want = gpu.host_outputs(), ora.outputs()
        for k in INT_OUTPUTS:
            if not np.array_equal(got[k], want[k]):
                int_bad.append((s, k))
        for k in FLOAT_OUTPUTS:
            r = float(rel_err(got[k], want[k], output_floor(k, want[k])).max()) if got[k].size else 0.0
            g = "out." + k
            max_rel[g] = max(max_rel.get(g, 0.0), r)
            if r > TIGHT_RTOL and g not in first_div:
                first_div[g] = s
        if s % blob_every == 0 or s == steps:
            for e in range(n):
                a, b = gpu.serialize_state(e), ora.serialize(e)
                diff_int = ints & (a != b)
                for g in np.unique(names[diff_int]):
                    if g == "pf.rng_pos":
                        pf_pos_first = pf_pos_first or s  # resample decisions (PF floats)
                    else:
                        int_bad.append((s, e, str(g)))
                r = rel_err(a[fl], b[fl], floors)
                for g in np.unique(names[fl]):
                    v = float(r[names[fl] == g].max())
                    max_rel[g] = max(max_rel.get(g, 0.0), v)
                    if v > TIGHT_RTOL and g not in first_div:
                        first_div[g] = s
        assert not int_bad, int_bad[:10]
    report = {"config": "c3 5v5 fast P=1024", "envs": n, "steps": steps, "blob_every": blob_every,
              "episodes_done": float(gpu.stats()[3]), "max_rel": max_rel, "first_step_above_1e-9": first_div,
              "first_pf_rng_pos_divergence": pf_pos_first}
    print(json.dumps(report, indent=1, sort_keys=True))
    out = os.environ.get("UT_PARITY_REPORT_DIR")
    if out:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, "c3_drift_1000.json"), "w") as f:
            json.dump(report, f, indent=1, sort_keys=True)
    ora.close()
    assert report["episodes_done"] == n * (steps // 128)
    for g in KIN_GROUPS:
        assert max_rel.get(g, 0.0) <= TIGHT_RTOL, (g, max_rel.get(g))
    worst = max(max_rel.values())
    assert worst <= NORTH_STAR_RTOL, report
