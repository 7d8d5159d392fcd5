"""Per-region instruction table of the step kernel from an ncu capture.

ncu's source page gives per-SASS-instruction counters (warp / thread instructions
executed, stall samples); nvdisasm -gi of the same build gives each
instruction's inlined source chain. Joining the two by instruction offset
attributes every executed instruction to a region of the particle-set loop
(the first ut_kernels.cuh line of the chain that falls in a region) and to the
innermost helper (ut_device.cuh function).

  python tools/sass_regions.py REPORT.ncu-rep [LIB.so] [--kernel step_kernelILi4ELi1024ELb1] [--per N]

--per: divide thread instructions by N (e.g. particle-steps of the launch).
"""
import argparse
import csv
import io
import pathlib
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

ROOT = pathlib.Path(__file__).resolve().parents[1]
KERN = ROOT / "paper_2505_08222_b200" / "csrc" / "ut_kernels.cuh"
DEV = ROOT / "paper_2505_08222_b200" / "csrc" / "ut_device.cuh"


def region_table():
    """(name, first line, last line) of ut_kernels.cuh, located by marker text so
    the table follows edits of the file."""
    lines = KERN.read_text().splitlines()

    def find(pat, start=0):
        for i in range(start, len(lines)):
            if pat in lines[i]:
                return i + 1
        raise KeyError(pat)

    s0 = find("__device__ void step_set(")
    marks = [
        ("set: setup + Philox blocks", s0),
        ("set: noise window + Box-Muller", find("// ---- pf::predict (tracking.cpp:94-117): the normals first", s0)),
        ("set: TMA wait + loads", find("const int nm = S.mcount[ti];", s0)),
        ("set: predict + speed clamp", find("s.px[j] = s.px[j] + s.vx[j] * c.dt;", s0) - 3),
        ("set: likelihood stages", find("// ---- range updates: own ping", s0)),
        ("set: shift + weights + ESS", find("double shift = 0.0;  // sum_j s'_j", s0)),
        ("set: weight sums + resample scan", find("// e, its running sums (the resample scan's thread part) and squares", s0)),
        ("set: resample (merged update)", find("// pf::maybe_resample's resample on the scan above", s0)),
        ("set: exact sequential path", find("if (exact && nm > 0) {", s0)),
        ("set: maybe_resample (no update / injected state)", find("// ---- pf::maybe_resample", s0)),
        ("set: store to HBM", find("// ---- the set back to HBM", s0)),
        ("set: estimate + track record", find("// ---- estimate (env.cpp:403-407)", s0)),
    ]
    end = next(i + 1 for i in range(s0, len(lines)) if lines[i] == "}")  # step_set's closing brace
    regs = []
    for i, (name, a) in enumerate(marks):
        b = marks[i + 1][1] - 1 if i + 1 < len(marks) else end
        regs.append((name, a, b))
    funcs = [
        ("pf_update_seq (exact path)", find("__device__ __noinline__ int pf_update_seq("), None),
        ("pf_estimate", find("__device__ __forceinline__ double3 pf_estimate("), None),
        ("pf_resample", find("__device__ void pf_resample("), None),
        ("resample_stage / resample_select", find("__device__ __forceinline__ void resample_stage("), None),
        ("stage_env", find("__device__ __forceinline__ void stage_env("), None),
        ("stage_bnd (boundary Philox blocks)", find("void stage_bnd("), None),
        ("prefetch_env", find("void prefetch_env("), None),
        ("reinit (auto-reset PF)", find("__device__ __forceinline__ void reinit_particle("), None),
        ("step_kernel body", find("__global__ void __launch_bounds__(1024 / PPT, UT_STEP_MIN_BLOCKS) step_kernel("), None),
        ("env_prologue", find("__device__ __noinline__ void env_prologue("), None),
        ("env_epilogue", find("__device__ __noinline__ bool env_epilogue("), None),
        ("spawn_serial", find("__device__ __noinline__ bool spawn_serial("), None),
        ("outputs", find("// ----------------------------------------------------------- outputs ---"), None),
    ]
    # function spans: up to the next listed function start
    starts = sorted((a, n) for n, a, _ in funcs)
    fspans = []
    for i, (a, n) in enumerate(starts):
        b = starts[i + 1][0] - 1 if i + 1 < len(starts) else len(lines)
        fspans.append((n, a, b))
    return regs, fspans


def device_funcs():
    """(name, first line) of ut_device.cuh functions, for the innermost helper."""
    out = []
    for i, ln in enumerate(DEV.read_text().splitlines()):
        m = re.search(r"__device__[^(]*?\b([a-zA-Z_0-9]+)\s*\(", ln)
        if m:
            out.append((i + 1, m.group(1)))
        m = re.match(r"struct (\w+)", ln)
        if m:
            out.append((i + 1, m.group(1)))
    return out


def disasm(lib, kernel):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", str(lib)], cwd=d, check=True, capture_output=True)
        cub = next(pathlib.Path(d).glob("*.cubin"))
        txt = subprocess.run(["nvdisasm", "-c", "-gi", str(cub)], check=True, capture_output=True, text=True).stdout
    sec = None
    insts = []  # (offset, opcode text, chain [(file, line), ...] innermost first)
    chain, pending = [], False
    loc_re = re.compile(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?')
    for ln in txt.splitlines():
        if ln.startswith(".text."):
            sec = ln[6:].rstrip(":")
            continue
        if sec is None or kernel not in sec:
            continue
        m = loc_re.search(ln)
        if m:
            if not pending:
                chain = []
                pending = True
            chain.append((pathlib.Path(m.group(1)).name, int(m.group(2))))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            pending = False
            insts.append((int(m.group(1), 16), m.group(2).strip(), list(chain)))
    return insts


def ncu_sass(report, kernel):
    out = subprocess.run(["ncu", "-i", str(report), "--page", "source", "--csv", "--print-source", "sass"],
                         check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    data = [dict(zip(hdr, r)) for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
    base = int(data[0]["Address"], 16)
    for d in data:
        d["off"] = int(d["Address"], 16) - base
    return data


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("lib", nargs="?", default=str(ROOT / "paper_2505_08222_b200" / "_lib" / "libutrack_b200.so"))
    ap.add_argument("--kernel", default="step_kernelILi4ELi1024ELb1")
    ap.add_argument("--per", type=float, default=None)
    ap.add_argument("--top", type=int, default=0, help="also list the N hottest source lines")
    a = ap.parse_args()
    insts = disasm(a.lib, a.kernel)
    rows = ncu_sass(a.report, a.kernel)
    by_off = {o: (op, ch) for o, op, ch in insts}
    mism = sum(1 for r in rows if r["off"] in by_off and
               by_off[r["off"]][0].split()[0] not in r["Source"])
    if len(rows) != len(insts) or mism:
        sys.exit(f"the library does not match the capture: {len(rows)} vs {len(insts)} instructions, "
                 f"{mism} opcode mismatches")
    regs, fspans = region_table()
    dfuncs = device_funcs()

    def region(chain):
        for f, line in chain:
            if f != KERN.name:
                continue
            for n, lo, hi in regs:
                if lo <= line <= hi:
                    return n
        for f, line in chain:
            if f != KERN.name:
                continue
            for n, lo, hi in fspans:
                if lo <= line <= hi:
                    return n
        return "other"

    def helper(chain):
        if chain and chain[0][0] == DEV.name:
            line = chain[0][1]
            name = None
            for l0, n in dfuncs:
                if l0 <= line:
                    name = n
            return name or "ut_device"
        return "-"

    agg = defaultdict(lambda: [0, 0, 0])  # warp inst, thread inst, stall samples
    sub = defaultdict(lambda: [0, 0, 0])
    lines_hot = defaultdict(lambda: [0, 0])
    tot = [0, 0, 0]
    for r in rows:
        op, ch = by_off[r["off"]]
        wi = int(r["Instructions Executed"] or 0)
        ti = int(r["Thread Instructions Executed"] or 0)
        ss = int(r["Warp Stall Sampling (All Samples)"] or 0)
        rg = region(ch)
        for acc in (agg[rg], sub[(rg, helper(ch))], tot):
            acc[0] += wi
            acc[1] += ti
            acc[2] += ss
        if ch:
            lines_hot[ch[0]][0] += ti
            lines_hot[ch[0]][1] += ss
    per = a.per
    print(f"| region | warp inst % | thread inst % | thread inst / unit | stall samples % |")
    print("|---|---|---|---|---|")
    for rg, (wi, ti, ss) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        pu = f"{ti / per:.1f}" if per else "-"
        print(f"| {rg} | {100 * wi / tot[0]:.1f} | {100 * ti / tot[1]:.1f} | {pu} | {100 * ss / max(tot[2], 1):.1f} |")
    pu = f"{tot[1] / per:.1f}" if per else "-"
    print(f"| **total** | 100 | 100 | {pu} | 100 |")
    print()
    print("| region / innermost helper | thread inst % | thread inst / unit |")
    print("|---|---|---|")
    for (rg, h), (wi, ti, ss) in sorted(sub.items(), key=lambda kv: -kv[1][1])[:40]:
        pu = f"{ti / per:.1f}" if per else "-"
        print(f"| {rg} / {h} | {100 * ti / tot[1]:.1f} | {pu} |")
    if a.top:
        print()
        print("| source line (innermost) | thread inst % | stall samples % |")
        print("|---|---|---|")
        for (f, line), (ti, ss) in sorted(lines_hot.items(), key=lambda kv: -kv[1][0])[:a.top]:
            print(f"| {f}:{line} | {100 * ti / tot[1]:.1f} | {100 * ss / max(tot[2], 1):.1f} |")


if __name__ == "__main__":
    main()
