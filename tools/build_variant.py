"""Build the CUDA library as it is at a git revision (or the working tree) into
paper_2505_08222_b200/_lib/variants/<name>.so, for A/B timing with tools/ab.py
(UT_LIBRARY selects the library at load time).

  python tools/build_variant.py NAME [REV] [-DMACRO=VALUE ...]
"""
import pathlib
import shutil
import subprocess
import sys
import tempfile

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2505_08222_b200.build import NVCC_FLAGS, nvcc  # noqa: E402


def main():
    name = sys.argv[1]
    rev = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("-D") else None
    defines = [a for a in sys.argv[2:] if a.startswith("-D")]
    out = ROOT / "paper_2505_08222_b200" / "_lib" / "variants" / f"{name}.so"
    out.parent.mkdir(parents=True, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        tmp = pathlib.Path(tmp)
        if rev:
            for d in ("paper_2505_08222_b200/csrc", "include"):
                (tmp / d).mkdir(parents=True)
                files = subprocess.run(["git", "ls-tree", "--name-only", f"{rev}:{d}"], cwd=ROOT, check=True,
                                       capture_output=True, text=True).stdout.split()
                for f in files:
                    blob = subprocess.run(["git", "show", f"{rev}:{d}/{f}"], cwd=ROOT, check=True,
                                          capture_output=True).stdout
                    (tmp / d / f).write_bytes(blob)
        else:
            shutil.copytree(ROOT / "paper_2505_08222_b200" / "csrc", tmp / "paper_2505_08222_b200" / "csrc")
            shutil.copytree(ROOT / "include", tmp / "include")
        flags = [f if f != str(ROOT / "include") else str(tmp / "include") for f in NVCC_FLAGS]
        cmd = [nvcc(), *flags, *defines, "-o", str(out), str(tmp / "paper_2505_08222_b200" / "csrc" / "ut_capi.cu")]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
            sys.exit(1)
        lines = r.stdout.splitlines() + r.stderr.splitlines()
        for i, ln in enumerate(lines):  # the FULL P = 1024 step kernel's registers / spills
            if "Function properties for _ZN2ut11step_kernelILi4ELi1024ELb1" in ln:
                print("  ", " | ".join(x.strip() for x in lines[i + 1:i + 3]))
                break
    print(out)


if __name__ == "__main__":
    main()
