"""A/B timing of library variants on one box (CUDA events, C3 unless --config):

  python tools/ab.py [--config c3] [--envs N] [--steps K] [--reps R] lib1.so lib2.so ...

Each variant runs in its own process (UT_LIBRARY selects it; "default" = the
in-tree product library); the list is repeated R times, interleaved, so clock
drift shows up as spread, not as a bias. Per run: ms per step over K steps
after warm-up, ms of reset_all (every env re-spawned: the auto-reset burst),
and the pf statistics of the timed steps.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, json, torch
sys.path.insert(0, ROOT)
import bench
from paper_2505_08222_b200.vecenv import VecEnv
cfgname, steps, warm, envs = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
cfg = bench.make_cfg(cfgname)
v = VecEnv(cfg, envs, master_seed=0, device=0)
s = torch.cuda.current_stream(); v.set_stream(s.cuda_stream)
v.step_policy("random", warm); torch.cuda.synchronize()
st0 = v.stats()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(s); v.step_policy("random", steps); b.record(s); torch.cuda.synchronize()
ms = a.elapsed_time(b) / steps
st = v.stats() - st0
a.record(s); v.reset_all(); b.record(s); torch.cuda.synchronize()
rms = a.elapsed_time(b)
print(json.dumps({"ms": round(ms, 3), "reset_ms": round(rms, 3), "updates": float(st[7]),
                  "resamples": float(st[8]), "exact": float(st[9])}))
'''.replace("ROOT", repr(ROOT))

if __name__ == "__main__":
    args = sys.argv[1:]
    cfg, steps, warm, envs, reps = "c3", 10, 3, 65536, 2
    libs = []
    i = 0
    while i < len(args):
        if args[i] in ("--config", "--envs", "--steps", "--reps"):
            k, val = args[i][2:], args[i + 1]
            if k == "config":
                cfg = val
            elif k == "envs":
                envs = int(val)
            elif k == "steps":
                steps = int(val)
            else:
                reps = int(val)
            i += 2
            continue
        libs.append(args[i])
        i += 1
    for rep in range(reps):
        for lib in libs:
            env = dict(os.environ)
            name = lib
            if "@" in lib:  # lib@VAR=VALUE,VAR2=VALUE2
                lib, extra = lib.split("@", 1)
                for kv in extra.split(","):
                    k, val = kv.split("=", 1)
                    env[k] = val
            if lib != "default":
                env["UT_LIBRARY"] = os.path.abspath(lib)
            r = subprocess.run([sys.executable, "-c", CHILD, cfg, str(steps), str(warm), str(envs)], env=env,
                               capture_output=True, text=True)
            out = r.stdout.strip().splitlines()
            print(name, rep, out[-1] if out else r.stderr[-2000:], flush=True)
