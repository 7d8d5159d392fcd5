"""Build the sm_100a CUDA library in-tree (paper_2505_08222_b200/_lib/libutrack_b200.so).

nvcc cross-compiles without a GPU. Flags: --fmad=false keeps every fp64/fp32
expression one-rounding-per-operation (parity with the oracle, which is built
with -ffp-contract=off); host code likewise gets -ffp-contract=off.
"""
import os
import pathlib
import shutil
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "libutrack_b200.so"
# Test-only builds of the same sources (tests/test_gpu_race_shake.py): the race
# shaker (ut_device.cuh, UT_RACE_SHAKE). Never loaded by the product path.
VARIANTS = {"ut_race_shake": ["-DUT_RACE_SHAKE=0x5eed"]}
VARIANT_DIR = LIB_DIR / "variants"
SOURCES = [CSRC / "ut_capi.cu"]
DEPS = SOURCES + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [ROOT / "include" / "ut_env.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-Xptxas", "-v",
    "-I", str(ROOT / "include"),
    "-shared",
]


def nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and pathlib.Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date(path):
    if not path.exists():
        return False
    t = path.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in DEPS)


def variant_path(name):
    return VARIANT_DIR / f"{name}.so"


def build_native(force=False, verbose=False):
    """The product library and the test variants, compiled concurrently."""
    LIB_DIR.mkdir(exist_ok=True)
    VARIANT_DIR.mkdir(exist_ok=True)
    jobs = []
    if force or not up_to_date(LIB):
        jobs.append((LIB, []))
    for name, defines in VARIANTS.items():
        if force or not up_to_date(variant_path(name)):
            jobs.append((variant_path(name), defines))
    procs = []
    for out, defines in jobs:
        tmp = out.with_suffix(".so.tmp")
        cmd = [nvcc(), *NVCC_FLAGS, *defines, "-o", str(tmp), *map(str, SOURCES)]
        procs.append((out, tmp, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    for out, tmp, proc in procs:
        so, se = proc.communicate()
        if proc.returncode != 0:
            sys.stderr.write(so + se)
            raise RuntimeError(f"nvcc failed for {out.name}")
        if out == LIB:
            (LIB_DIR / "ptxas.log").write_text(so + se)
            if verbose:
                sys.stdout.write(se)
        os.replace(tmp, out)
    return LIB


if __name__ == "__main__":
    build_native(force="--force" in sys.argv, verbose=True)
    print(LIB)
