"""Workload of the race gate (tests/test_gpu_race_shake.py): the FULL P = 1024
step instance through the C-ABI only (no torch in the process) on

* "c3":  a 5v5 fast-target batch (the headline shape), and
* "c4":  a mixed 1..8 x 1..8 fleet with estimator-heavy envs (ragged set offsets,
         up to kMaxMerged = 8 merged updates per set),

each run as: ctor, external-action and policy steps across two auto-resets, one
step on the forced exact update path, refresh, reset_all and one more step. The
result is every env's state blob, every output buffer and the statistics.

    python tests/race_workload.py OUT.npz GRID [GRID ...]

writes one result set per grid size (ut_debug_set_grid; 0 = default grid) with
whatever library UT_LIBRARY selects (the race-shaker build in the gate)."""
import ctypes as C
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2505_08222_b200 import _abi, _native  # noqa: E402
from paper_2505_08222_b200.vecenv import EnvConfig, PfConfig, VecEnv  # noqa: E402

VERBOSE = False
HEAVY = dict(comm_drop_prob=0.0, detection_range=1e9, comm_range=1e9)
MIX = [(8, 8, True), (1, 1, False), (3, 5, False), (5, 3, False), (8, 1, True), (2, 7, False), (5, 5, True),
       (4, 4, False)]


def _dbg():
    lib = _native.lib()
    _abi.declare_debug(lib)
    return lib


def make(kind):
    if kind == "c3":
        cfg = EnvConfig(n_agents=5, n_targets=5, horizon=3, target_speed_frac=0.6, d_min=100.0,
                        spawn_max_sep=400.0, pf=PfConfig(n_particles=1024))  # bench.py CONFIGS["c3"]
        return VecEnv(cfg, 24, 5)
    cfgs = [EnvConfig(n_agents=a, n_targets=t, horizon=3, spawn_max_sep=600.0, pf=PfConfig(n_particles=1024),
                      **(HEAVY if h else {})) for a, t, h in MIX]
    fleet = [i % len(MIX) for i in range(12)]
    return VecEnv(cfgs, len(fleet), 9, fleet=fleet)


def run(kind, grid):
    lib = _dbg()
    v = make(kind)
    full, np_ = C.c_int32(), C.c_int32()
    assert lib.ut_debug_instance(v._h, C.byref(full), C.byref(np_)) == 0 and full.value == 1, "not FULL"
    assert lib.ut_debug_set_grid(v._h, grid) == 0, lib.ut_last_error()
    rng = np.random.default_rng(1)
    out = {}
    for s in range(7):  # horizon 3: steps 3 and 6 auto-reset every env
        if s == 4:
            assert lib.ut_debug_set_knobs(v._h, 1, -1) == 0  # exact sequential update path
        if s % 2:
            v.step_policy("random")
        else:
            m = v.host_outputs(["masks"])["masks"].reshape(-1, 5).astype(bool)
            acts = np.array([rng.choice(np.flatnonzero(r)) if r.any() else 2 for r in m], np.int32)
            v.step(acts.reshape(v.n_envs(), v.n_agents()))
        if s == 4:
            assert lib.ut_debug_set_knobs(v._h, 0, -1) == 0
        out[f"s{s}_blobs"] = v.export_state()
        if VERBOSE:
            print(f"{kind} grid {grid} step {s} ok", flush=True)
    v.refresh_outputs()
    for k, a in v.host_outputs().items():
        out[f"out_{k}"] = a
    out["stats"] = v.stats()
    v.reset_all()
    v.step_policy("scripted")
    out["after_reset_blobs"] = v.export_state()
    v.close()
    return out


def main():
    global VERBOSE
    args = [a for a in sys.argv[1:] if a != "-v"]
    VERBOSE = len(args) != len(sys.argv) - 1
    path, grids = args[0], [int(g) for g in args[1:]]
    res = {}
    for kind in ("c3", "c4"):
        for g in grids:
            for k, a in run(kind, g).items():
                res[f"{kind}/g{g}/{k}"] = a
    np.savez(path, **res)
    print("race workload ok", _native.LIB_PATH.name, grids)


if __name__ == "__main__":
    main()
