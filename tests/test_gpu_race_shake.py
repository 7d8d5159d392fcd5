"""The race gate of SURVEY §5, in place of compute-sanitizer (closed on this GPU
pool: runs under it left GPUs needing a reset).

The reference's own gate is worker-count invariance (test_vecenv.cpp:126-143):
any partition of the envs over threads gives the same batch. The device
analogue, checked bit for bit on the FULL P = 1024 step kernel (tests/
race_workload.py: a 5v5 batch and a mixed 1..8 x 1..8 heavy fleet, two
auto-resets, the forced exact update path, reset_all):

1. grid-size invariance -- 1, 3, 7 CTAs and the default persistent grid change
   every CTA's static env range (prologue / outputs / resets) and the dynamic
   set schedule of the filter phase;
2. schedule invariance -- the race-shaker build (UT_RACE_SHAKE, ut_device.cuh)
   stalls random warps and single lanes for up to ~4 us around every CTA
   barrier, TMA completion wait, prefetch issue and grid barrier, so warps meet
   the rotating reduction buffers, the TMA-refilled set buffer and the resample
   staging in orders the normal schedule never produces. A missing barrier, a
   write-after-read hazard or a warp-synchronous assumption changes the result.
"""
import os
import pathlib
import subprocess
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests"))
pytestmark = pytest.mark.gpu

GRIDS = [0, 1, 3, 7]


def _run(tmp_path, name, library, grids):
    out = tmp_path / f"{name}.npz"
    env = dict(os.environ)
    if library:
        env["UT_LIBRARY"] = str(library)
    p = subprocess.run([sys.executable, str(ROOT / "tests" / "race_workload.py"), str(out), *map(str, grids)],
                       capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    return dict(np.load(out))


def _same(a, b, ga, gb, what):
    keys = sorted(k.split("/", 2)[2] for k in a if k.split("/")[1] == f"g{ga}")
    assert keys
    for kind in ("c3", "c4"):
        for k in keys:
            x, y = a[f"{kind}/g{ga}/{k}"], b[f"{kind}/g{gb}/{k}"]
            assert x.shape == y.shape and np.array_equal(x.view(np.uint8), y.view(np.uint8)), \
                f"{what}: {kind} {k} differs (grid {ga} vs {gb})"


@pytest.fixture(scope="module")
def baseline(tmp_path_factory, cuda_device):
    return _run(tmp_path_factory.mktemp("race"), "product", None, GRIDS)


def test_grid_size_invariance(baseline):
    for g in GRIDS[1:]:
        _same(baseline, baseline, 0, g, "product build")


def test_race_shaker_schedules_are_invariant(baseline, tmp_path):
    from paper_2505_08222_b200.build import variant_path
    lib = variant_path("ut_race_shake")
    assert lib.exists(), "build() makes the race-shaker variant"
    for rep in range(2):  # the stalls are seeded from the SM clock: every run differs
        shaken = _run(tmp_path, f"shake{rep}", lib, [0, 3])
        for g in (0, 3):
            _same(baseline, shaken, 0, g, f"race shaker run {rep}")
