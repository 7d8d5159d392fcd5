import os
import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU check")
    # Build the oracle libraries if they are missing and the sources are here.
    oracle_so = ROOT / "oracle" / "_build" / "libut_oracle.so"
    ref_so = ROOT / "oracle" / "_ref" / "libutrack_ref.so"
    if not oracle_so.exists() or (not ref_so.exists() and pathlib.Path("/root/reference/proj").exists()):
        target = "all" if pathlib.Path("/root/reference/proj").exists() else "restatement"
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "-j8", target], check=False)


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda_device():
    if not gpu_available():
        pytest.skip("no CUDA device")
    return 0
