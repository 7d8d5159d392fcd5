"""CPU: the evaluation metrics accumulated by the step follow
curriculum::evaluate (curriculum.cpp:267-356): per step, the sum over targets of
the tracking error and the sum over agent-target pairs of the 2D distance; per
episode, their means over the horizon, whether any step collided / lost a target.
Checked on the oracle against a direct computation from the step outputs and the
state blobs; the device is checked against the oracle in test_gpu_parity.py."""
import math

import numpy as np

from oracle_bindings import Oracle, default_config

H = 6
CFG = dict(n_agents=2, n_targets=3, horizon=H, pf_n_particles=32, spawn_max_sep=400.0, d_safe=150.0)


def positions(blob, A, T):
    ag = [(blob[5 + 6 * a], blob[5 + 6 * a + 1]) for a in range(A)]
    tg = [(blob[5 + 6 * A + 8 * t], blob[5 + 6 * A + 8 * t + 1]) for t in range(T)]
    return ag, tg


def test_eval_accumulators_follow_curriculum_evaluate():
    n, A, T = 4, CFG["n_agents"], CFG["n_targets"]
    ora = Oracle(default_config(**CFG), n, 3)
    want = np.zeros((n, 2))
    flags = np.zeros(n, int)
    for step in range(H - 1):
        ora.step_policy(1)
        out = ora.outputs()
        for e in range(n):
            ag, tg = positions(ora.serialize(e), A, T)
            want[e, 1] += sum(out["tracking_error"][e * T:(e + 1) * T])
            want[e, 0] += sum(math.hypot(a[0] - t[0], a[1] - t[1]) for a in ag for t in tg)
            flags[e] |= int(out["collision"][e]) | (2 if out["target_lost"][e * T:(e + 1) * T].any() else 0)
    for e in range(n):
        d, err, fl = ora.eval_acc(e)
        np.testing.assert_allclose([d, err], want[e], rtol=1e-13)
        assert int(fl) == flags[e]
    # the H-th step closes every episode: the stats fold the per-episode means
    ora.step_policy(1)
    st = dict(zip(__import__("paper_2505_08222_b200._abi", fromlist=["x"]).STAT_NAMES, ora.stats()))
    assert st["episodes_done"] == n
    out = ora.outputs()
    for e in range(n):
        flags[e] |= int(out["collision"][e]) | (2 if out["target_lost"][e * T:(e + 1) * T].any() else 0)
        assert ora.eval_acc(e) == (0.0, 0.0, 0.0)  # reset with the new episode
    assert st["eval_collided_episodes"] == sum(f & 1 for f in flags)
    assert st["eval_lost_episodes"] == sum(1 for f in flags if f & 2)
    err_lo = sum(want[:, 1]) / (H * T)  # the last step only adds
    assert st["eval_err_sum"] >= err_lo - 1e-9
    assert st["eval_dist_sq"] >= st["eval_dist_sum"] ** 2 / n - 1e-6  # Cauchy-Schwarz
