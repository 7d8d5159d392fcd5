"""CPU: bench.py's contract pieces that do not need a GPU -- the algorithmic
byte count behind the roofline and the reference arm, which times
the reference's own CPU step (oracle/_ref) on this host."""
import json
import subprocess
import sys

import pytest

from oracle_bindings import ROOT, ref_available

sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def test_algorithmic_bytes_match_survey():
    """0.083 MB (C1), 0.330 MB (C2), 2.059 MB (C3) per env-step."""
    for name, A, T, want in (("c1", 1, 1, 0.083e6), ("c2", 2, 2, 0.330e6), ("c3", 5, 5, 2.059e6)):
        got = bench.algorithmic_bytes_per_env_step(A, T, 1024, bench.rec_words_for(A, T))
        assert abs(got - want) / want < 0.02, (name, got)


def test_particle_bytes_dominate():
    A = T = 5
    total = bench.algorithmic_bytes_per_env_step(A, T, 1024, bench.rec_words_for(A, T))
    assert 80 * 1024 * A * T / total > 0.95


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_reference_arm_prints_one_json_line():
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["unit"] == "agent-env steps/s"


@pytest.mark.parametrize("cfg,gpus,scaling,total", [("c3", 2, "strong", 65536), ("c5", 2, "weak", 262144)])
def test_gpus_flag_spawns_one_rank_per_gpu(cfg, gpus, scaling, total):
    """`bench.py --gpus N` outside torchrun re-launches itself as N ranks
    (torch.distributed.run on 127.0.0.1); the ranks shard the envs by contiguous
    global index range (C3 strong: 65,536 in total; C5 weak: 131,072 each) and
    all-reduce over the process group (gloo without a GPU)."""
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(gpus), "--config", cfg, "--dry-run"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == gpus and d["scaling"] == scaling and d["total_envs"] == total
    assert d["envs_sum"] == total and d["max_rank"] == gpus and d["backend"] == "gloo"
    r = d["ranges"]
    assert r[0][0] == 0 and r[-1][1] == total and all(a[1] == b[0] for a, b in zip(r, r[1:]))


@pytest.mark.parametrize("native", [True, False])
def test_e2e_host_policy_draws_legal_actions(native, monkeypatch):
    """The e2e leg's host policy (tools/host_policy.c, or its numpy twin): a legal
    action for every agent with one, 0 for agents without, about uniform over the
    legal ones, and a fresh draw every call."""
    import numpy as np
    n = 20000
    if not native:
        monkeypatch.setattr(bench, "ROOT", ROOT / "no-such-dir")
    elif not (ROOT / "tools" / "_lib" / "libhost_policy.so").exists():
        pytest.skip("tools/_lib/libhost_policy.so not built")
    acts = np.zeros(n, np.int32)
    fn, name = bench.make_host_policy(acts, n, 0)
    assert ("host_policy.c" in name) == native
    rng = np.random.default_rng(1)
    masks = (rng.random((n, 5)) < 0.6).astype(np.uint8)
    masks[:100] = 0  # no legal action (padding agents of a mixed fleet)
    fn(masks.reshape(-1))
    first = acts.copy()
    none = masks.sum(axis=1) == 0
    assert np.all(first[none] == 0)
    assert (masks[np.arange(n), first] == 1)[~none].all()
    only2 = np.flatnonzero((masks == [0, 0, 1, 0, 0]).all(axis=1))
    assert np.all(first[only2] == 2)
    both = np.flatnonzero((masks == [1, 1, 0, 0, 0]).all(axis=1))
    assert 0.35 < np.mean(first[both] == 1) < 0.65
    fn(masks.reshape(-1))
    assert not np.array_equal(first, acts)
