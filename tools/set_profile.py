"""Wall-clock split of the particle-set loop (thread 0 of each CTA, SM clock),
from a build with -DUT_SET_PROFILE (tools/build_variant.py setprof -DUT_SET_PROFILE):

  UT_LIBRARY=paper_2505_08222_b200/_lib/variants/setprof.so python tools/set_profile.py [--steps 10]
"""
import ctypes as C
import sys
import pathlib

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2505_08222_b200 import _native  # noqa: E402
from paper_2505_08222_b200.vecenv import VecEnv  # noqa: E402

SLOTS = ["noise + setup", "TMA wait", "load + predict", "likelihood stages", "stage barrier + shift + exp",
         "weight sums (barrier)", "normalise / ESS / exact", "resample", "store", "estimate", "track record",
         "unused"]


def main():
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 10
    cfg = bench.make_cfg("c3")
    v = VecEnv(cfg, 65536, master_seed=0)
    lib = _native.lib()
    lib.ut_debug_set_profile.argtypes = [C.c_int, C.POINTER(C.c_uint64), C.c_int]
    out = (C.c_uint64 * 12)()
    v.step_policy("random", 3)
    v.synchronize()
    assert lib.ut_debug_set_profile(0, out, 1) == 0
    v.step_policy("random", steps)
    v.synchronize()
    assert lib.ut_debug_set_profile(0, out, 1) == 0
    tot = float(sum(out[:11])) or 1.0
    for k in range(11):
        print(f"{SLOTS[k]:32s} {100 * out[k] / tot:5.1f} %")


if __name__ == "__main__":
    main()
