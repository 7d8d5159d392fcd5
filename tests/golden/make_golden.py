"""TEST INFRASTRUCTURE: record golden vectors from the reference itself.

Run here (where /root/reference exists and oracle/_ref is built):

    python tests/golden/make_golden.py

For each case it drives the reference VecEnv (oracle/_ref/libutrack_ref.so,
built from /root/reference/proj sources by oracle/Makefile) through a ctor and
a fixed sequence of legal actions and stores, bit for bit, the batch outputs
after every step and every env's final state blob. tests/test_oracle_pinning.py
replays the same inputs through the oracle and requires identical bytes, so the
restatement stays pinned to the reference where /root/reference is absent.
"""
import json
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parents[1]))

CASES = {
    "c1_1v1_slow_p64": (dict(n_agents=1, n_targets=1, target_speed_frac=0.3, horizon=128, pf_n_particles=64), 2, 0),
    "c2_2v2_reset_p32": (dict(n_agents=2, n_targets=2, horizon=4, pf_n_particles=32), 2, 42),
    "c3_5v5_fast_p16": (dict(n_agents=5, n_targets=5, target_speed_frac=0.6, d_min=100.0, spawn_max_sep=400.0,
                             horizon=128, pf_n_particles=16), 1, 42),
    "c5_heavy_p32": (dict(n_agents=3, n_targets=2, comm_drop_prob=0.0, detection_range=1e9, comm_range=1e9,
                          target_speed_frac=0.5, horizon=128, pf_n_particles=32), 2, 7),
    "follow_p33": (dict(n_agents=2, n_targets=3, pf_n_particles=33, reward_mode=1, perturbation_std=0.05,
                        spawn_max_sep=400.0, horizon=5), 1, 3),
}
N_STEPS = 8
KEEP = ("obs", "global_state", "rewards", "dones", "masks", "tracking_error", "min_agent_dist", "target_lost",
        "collision", "step", "final_obs")


def replay(factory, g):
    """Drive `factory(cfg, n_envs, seed)` with the recorded inputs; return the
    same keys the fixture holds."""
    from oracle_bindings import default_config
    kw = json.loads(str(g["config_json"]))
    n_envs, seed = int(g["n_envs"]), int(g["seed"])
    env = factory(default_config(**kw), n_envs, seed)
    out = {}

    def grab(tag):
        o = env.outputs()
        for k in KEEP:
            out[f"out_{tag}_{k}"] = o[k]

    grab("ctor")
    for s, acts in enumerate(g["actions"]):
        env.step(acts)
        grab(f"s{s}")
    for e in range(n_envs):
        out[f"blob_{e}"] = env.serialize(e)
    return out


def record(name, kw, n_envs, seed):
    from oracle_bindings import RefVecEnv, default_config, random_legal_actions
    ref = RefVecEnv(default_config(**kw), n_envs, seed)
    rng = np.random.default_rng(seed + 1)
    actions = []
    for _ in range(N_STEPS):
        a = random_legal_actions(ref.outputs()["masks"], rng)
        actions.append(a)
        ref.step(a)
    ref.close()
    g = {"config_json": np.array(json.dumps(kw)), "n_envs": np.array(n_envs), "seed": np.array(seed),
         "actions": np.array(actions, np.int32)}
    g.update(replay(lambda cfg, n, s: RefVecEnv(cfg, n, s), g))
    np.savez_compressed(HERE / f"{name}.npz", **g)
    return sum(v.nbytes for v in g.values())


if __name__ == "__main__":
    for name, (kw, n, seed) in CASES.items():
        print(name, record(name, kw, n, seed), "bytes")
