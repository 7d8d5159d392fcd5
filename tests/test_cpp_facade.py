"""The header-only C++ facade (include/ut_vecenv.hpp) compiles against the C-ABI,
links the product library and behaves: DeviceError without a GPU; on a B200 the
same numbers as the Python mirror of the same calls."""
import json
import subprocess

import pytest

from oracle_bindings import ROOT

LIB = ROOT / "paper_2505_08222_b200" / "_lib"


def _build(tmp_path):
    exe = tmp_path / "facade_check"
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cpp" / "facade_check.cpp"), "-L", str(LIB), "-lutrack_b200",
                    f"-Wl,-rpath,{LIB}", "-o", str(exe)], check=True, capture_output=True, text=True)
    return exe


def _run(exe):
    p = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    return p.returncode, json.loads(p.stdout.strip().splitlines()[-1])


def test_facade_compiles_and_fails_loudly_without_gpu(tmp_path):
    import torch
    exe = _build(tmp_path)
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu variant")
    rc, d = _run(exe)
    assert rc == 0 and d == {"ok": 0, "error": "DeviceError"}


@pytest.mark.gpu
def test_facade_matches_python_mirror(tmp_path, cuda_device):
    import numpy as np
    from paper_2505_08222_b200.vecenv import EnvConfig, PfConfig, VecEnv
    rc, d = _run(_build(tmp_path))
    assert rc == 0 and d["ok"] == 1, d
    v = VecEnv(EnvConfig(n_agents=2, n_targets=2, horizon=3, pf=PfConfig(n_particles=64)), 4, 7)
    acts = np.full(8, 2, np.int32)
    v.step(acts)
    v.step_policy("random")
    v.step(acts)
    h = v.host_outputs()
    assert d["reward_sum"] == float(np.sum(h["rewards"]))
    assert d["dones"] == int(np.sum(h["dones"]))
    assert d["obs00"] == float(h["obs"][0, 0])
    assert d["step0"] == v.world_step(0)
    assert d["blob"] == v.serialize_state(0).size
    assert d["all"] == 4 * d["blob"]
    assert d["multi_same"] == 1  # ut::MultiVecEnv over two shards == ut::VecEnv
