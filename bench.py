#!/usr/bin/env python3
"""Throughput of the batched JaxLrauv environment step on B200.

Metric (BASELINE.json): agent-env steps/sec on the 5-agent / 5-fast-target
workload (65,536 envs, P = 1024, fp64 particle filters),
random legal actions from the device bench stream (vecenv.cpp:118-135).

Multi-GPU: one process per GPU. Under torchrun the ranks come from the
environment; `--gpus N` without WORLD_SIZE re-launches itself under
torch.distributed.run with N processes. Envs shard by global index range and
each GPU steps its shard independently (no data-path collective); the episode
statistics are all-reduced once over NCCL after the run (NCCL_DEBUG=INFO).
C3 (and C1/C2) scale strongly -- 65,536 envs in total, 8,192 per GPU at N = 8
(SURVEY §8e); C4/C5 weakly (their per-GPU shard is fixed by HBM capacity).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]
                  [--scaling strong|weak] [--dry-run]
"""
import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # SURVEY §8d synthetic inputs; everything else takes the EnvConfig defaults
    "c1": dict(desc="1 agent vs 1 slow target", n_agents=1, n_targets=1, target_speed_frac=0.3,
               horizon=128, envs=1024),
    "c2": dict(desc="2 agents vs 2 targets, 1000-step episodes", n_agents=2, n_targets=2, horizon=1000,
               envs=16384),
    "c3": dict(desc="5 agents vs 5 fast targets (paper headline)", n_agents=5, n_targets=5,
               target_speed_frac=0.6, d_min=100.0, spawn_max_sep=400.0, horizon=128, envs=65536),
    "c5": dict(desc="5v5 estimator-heavy (every pair pinged, every link up)", n_agents=5, n_targets=5,
               target_speed_frac=0.6, d_min=100.0, spawn_max_sep=400.0, horizon=128,
               comm_drop_prob=0.0, detection_range=1e9, comm_range=1e9, envs=131072),
    # per-env fleet (A_i, T_i) ~ U{1..8}^2 keyed by derive_key(seed, "mix", i),
    # padded to 8 x 8 in the batch buffers, ragged particle storage. 262,144 envs need
    # ~218 GB of particles, so one GPU runs 65,536 (the 8-GPU run holds the full mix).
    "c4": dict(desc="curriculum mix: 1-8 agents x 1-8 targets per env (padded 8x8, ragged particles)",
               n_agents=8, n_targets=8, spawn_max_sep=600.0, horizon=128, envs=65536, mix=True),
}
MIX_TAG = 0x6d6978  # "mix"
# C3 is the strong-scaling workload (67 GB fits one GPU); C5 needs
# 135 GB per GPU even at N = 8 and C4 ~218 GB ragged, so they scale weakly.
DEFAULT_SCALING = {"c1": "strong", "c2": "strong", "c3": "strong", "c4": "weak", "c5": "weak"}


def mix_fleet(lo, hi, seed=0):
    """(A_i, T_i) for global envs [lo, hi): the low 6 bits of derive_key(seed, "mix", i)
    (rng.hpp:30-38) as two 3-bit fields."""
    def splitmix(x):
        x = (x + 0x9e3779b97f4a7c15) & (2**64 - 1)
        x = ((x ^ (x >> 30)) * 0xbf58476d1ce4e5b9) & (2**64 - 1)
        x = ((x ^ (x >> 27)) * 0x94d049bb133111eb) & (2**64 - 1)
        return x ^ (x >> 31)

    def derive(a, b, c, d=0):
        h = 0x9e3779b97f4a7c15
        for v in (a, b, c, d):
            h ^= splitmix((v + h) & (2**64 - 1))
            h = ((h << 23) | (h >> 41)) & (2**64 - 1)
        return splitmix(h)
    out = []
    for i in range(lo, hi):
        h = derive(seed, MIX_TAG, i)
        out.append((1 + (h & 7), 1 + ((h >> 3) & 7)))
    return out


def make_cfg(name, particles=1024, n_agents=None, n_targets=None):
    from paper_2505_08222_b200.vecenv import EnvConfig, PfConfig
    kw = {k: v for k, v in CONFIGS[name].items() if k not in ("desc", "envs", "mix")}
    if n_agents is not None:
        kw.update(n_agents=n_agents, n_targets=n_targets)
    return EnvConfig(**kw, pf=PfConfig(n_particles=particles))


def oracle_cfg(name, particles=1024):
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_bindings import default_config
    kw = {k: v for k, v in CONFIGS[name].items() if k not in ("desc", "envs")}
    return default_config(**kw, pf_n_particles=particles)


def make_host_policy(acts_np, n_ag, rank):
    """The e2e leg's host policy: a uniform legal action per agent from its
    returned 5-byte mask (the device random policy's rule, vecenv.cpp:125-134).
    tools/host_policy.c (OpenMP, built by __graft_entry__.build()) when present,
    else the same rule vectorised in numpy. Padding agents of mixed fleets have no
    legal action and get 0 (ignored by the step). Returns (fn(masks_u8), name)."""
    import ctypes as C
    so = ROOT / "tools" / "_lib" / "libhost_policy.so"
    if so.exists():
        lib = C.CDLL(str(so))
        lib.host_policy.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64), C.c_int]
        lib.host_policy.restype = None
        counter = C.c_uint64(0)
        seed = 0x5eed0000 + rank
        out = acts_np.ctypes.data
        # the node's cores split over the ranks on it
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", os.environ.get("WORLD_SIZE", "1")))
        n_threads = max(1, (os.cpu_count() or 1) // max(1, local_world))

        def fn(masks):
            lib.host_policy(masks.ctypes.data, n_ag, out, seed, C.byref(counter), n_threads)
        return fn, f"tools/host_policy.c (OpenMP, {n_threads} threads)"
    import numpy as np
    rng = np.random.default_rng(rank)
    kth = np.zeros((32, 5), np.int32)
    n_legal = np.zeros(32, np.float32)
    for code in range(32):
        bits = [b for b in range(5) if (code >> b) & 1]
        n_legal[code] = len(bits)
        kth[code, :len(bits)] = bits
    kth_flat = kth.reshape(-1)
    u = np.empty(n_ag, np.float32)
    code = np.empty(n_ag, np.uint8)
    tmp = np.empty(n_ag, np.uint8)
    flat = np.empty(n_ag, np.int64)

    def fn(masks):
        mv = masks.reshape(-1, 5)
        np.bitwise_or(mv[:, 0], np.left_shift(mv[:, 1], 1, out=tmp), out=code)
        for b in (2, 3, 4):
            np.bitwise_or(code, np.left_shift(mv[:, b], b, out=tmp), out=code)
        rng.random(out=u, dtype=np.float32)
        np.multiply(u, n_legal.take(code), out=u)
        flat[:] = u                      # floor (u * #legal) < #legal
        np.add(flat, code.astype(np.int64) * 5, out=flat)
        kth_flat.take(flat, out=acts_np)
    return fn, "numpy (tools/_lib/libhost_policy.so not built)"



def algorithmic_bytes_per_env_step(A, T, P, rec_words):
    """read + write of the whole state once per step (80 B per
    particle), the env record (read + write), and the step's outputs."""
    R = A + T
    pf = 80 * P * A * T
    rec = 16 * rec_words
    outs = 8 * 12 * A * R + 8 * 12 * R + 8 + 1 + 5 * A + T * (8 + 8 + 1) + 1 + 4
    return pf + rec + outs


def rec_words_for(A, T):
    """Words of one env record (csrc/ut_layout.h layout_config)."""
    o_track = 11 + 6 * A + 8 * T + T + 6 * A * A
    return o_track + 10 * A * T + 16


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = pathlib.Path(f"/tmp/ut_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.gpu)], stdout=self.fh, stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None
            return self
        # nvidia-smi takes ~0.1-0.5 s to produce its first line: wait for it, so
        # even a sub-second timed region is sampled (the first sample is pre-load)
        t0 = time.time()
        while time.time() - t0 < 3.0 and self.proc.poll() is None:
            if self.path.stat().st_size > 0:
                break
            time.sleep(0.02)
        self.skip = sum(1 for _ in self.path.open()) if self.path.exists() else 0
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.path.read_text().splitlines()
        skip = getattr(self, "skip", 0)
        if len(lines) > skip:  # samples taken before the timed region started are dropped
            lines = lines[skip:]
        for line in lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def workload_config(name, per_gpu, total, particles, scaling):
    """The `config` object both arms print (same workload, same keys)."""
    c = CONFIGS[name]
    A, T = c["n_agents"], c["n_targets"]
    gb = algorithmic_bytes_per_env_step(A, T, particles, rec_words_for(A, T)) * per_gpu / 1e9
    return {"workload": f"{name}: {c['desc']}", "envs_per_gpu": per_gpu, "total_envs": total,
            "particles": particles, "agents": A, "targets": T, "horizon": c["horizon"], "scaling": scaling,
            "policy": "random legal (bench stream, vecenv.cpp:125-134)",
            "l2": f"inputs larger than L2 ({gb:.1f} GB touched per step per GPU)"}


def shard_plan(name, world, rank, args):
    """(scaling, per-GPU envs nominal, total envs, this rank's [lo, hi))."""
    from paper_2505_08222_b200.sharding import shard_range
    scaling = args.scaling or DEFAULT_SCALING[name]
    if scaling == "strong":
        total = args.total_envs or CONFIGS[name]["envs"]
        per_gpu = -(-total // world)
    else:
        per_gpu = args.envs_per_gpu or CONFIGS[name]["envs"]
        total = per_gpu * world
    lo, hi = shard_range(total, rank, world)
    return scaling, per_gpu, total, lo, hi


def measured_counts(name, per_gpu, particles):
    """ncu counters per step-kernel launch of the same workload (profiles/traffic.json,
    from `ncu --metrics ...` captures): DRAM bytes, fp64 thread instructions."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return {}
    return json.loads(p.read_text()).get(f"{name}:{per_gpu}:{particles}", {})


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def fp64_peak_per_s(device):
    """Measured thread-level DFMA issue rate of this device (ut_debug_fp64_peak)."""
    import ctypes as C
    from paper_2505_08222_b200 import _native, _abi
    lib = _native.lib()
    _abi.declare_debug(lib)
    out = C.c_double()
    if lib.ut_debug_fp64_peak(device, C.byref(out)) != 0:
        return None
    return out.value


REF_BUILD = ("reference sources compiled unmodified by oracle/Makefile: -O3 -std=gnu++20 -march=x86-64-v3 "
             "-ffp-contract=off (reference: -march=native, contraction on); Eigen 3.4 is absent here, so a "
             "shim supplies it with correctly rounded fp32 log/sin/cos through libm and sequential reductions "
             "(Eigen: SIMD polynomials) -- a slower CPU path than a real-Eigen -march=native build")


def cpu_baseline(cfg_name, particles, budget_s=12.0):
    """The reference's own benchmark_sps (vecenv.cpp:175-202), compiled from its
    sources into oracle/_ref, on this host's cores over a bounded sample."""
    import ctypes as C
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_bindings as ob
    cfg = oracle_cfg(cfg_name, particles)
    cores = ob.env_cpu_count()
    A = CONFIGS[cfg_name]["n_agents"]
    n_envs = max(32 * cores, 64)
    if ob.ref_available():
        lib = ob.ref_lib()
        kind = "reference"

        def run(steps, warm):
            sps, wall, wk, tot = C.c_double(), C.c_double(), C.c_int32(), C.c_uint64()
            ph = (C.c_uint64 * 7)()
            rc = lib.ref_benchmark_sps(C.byref(cfg), n_envs, steps, 0, 0, cores, warm, C.byref(sps), C.byref(wall),
                                       C.byref(wk), ph, C.byref(tot))
            if rc:
                raise RuntimeError(lib.ref_last_error().decode())
            return sps.value, wall.value, wk.value, list(ph)
    else:
        kind = "port"
        cores = 1
        n_envs = 16

        def run(steps, warm):
            o = ob.Oracle(cfg, n_envs, 0)
            o.step_policy(warm)
            t0 = time.perf_counter()
            o.step_policy(steps)
            wall = time.perf_counter() - t0
            o.close()
            return n_envs * steps / wall, wall, 1, []
    sps, wall, wk, ph = run(1, 1)  # probe
    steps = int(max(2, min(64, budget_s / max(wall, 1e-3))))
    sps, wall, wk, ph = run(steps, 2)
    names = ["targets", "agents", "measure", "filter", "comms", "observe", "reward"]
    out = {"value": sps * A, "unit": "agent-env steps/s", "cores": wk, "kind": kind,
           "sample": f"{n_envs} envs x {steps} steps of {cfg_name} (P={particles}), "
                     f"benchmark_sps(kRandom) after 2 warmup steps, {wall:.1f} s wall",
           "timed_envs": n_envs, "timed_steps": steps, "env_sps": sps,
           "build": REF_BUILD if kind == "reference" else "oracle/ut_oracle.c restatement, 1 thread"}
    if ph:
        tot = float(sum(ph)) or 1.0
        out["phase_ns"] = dict(zip(names, ph))
        out["phase_ns_per_env_step"] = {k: v / (n_envs * steps) for k, v in zip(names, ph)}
        out["phase_share"] = {k: v / tot for k, v in zip(names, ph)}
    return out


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    base = cpu_baseline(args.config, args.particles, budget_s=max(5.0, 2.0 * (args.steps + args.warmup)))
    scaling = args.scaling or DEFAULT_SCALING[args.config]
    world = max(1, args.gpus)
    if scaling == "strong":
        total = args.total_envs or CONFIGS[args.config]["envs"]
        per_gpu = -(-total // world)
    else:
        per_gpu = args.envs_per_gpu or CONFIGS[args.config]["envs"]
        total = per_gpu * world
    config = workload_config(args.config, per_gpu, total, args.particles, scaling)
    config["timed_envs"] = base["timed_envs"]
    config["note"] = (f"the CPU reference timed {base['timed_envs']} envs (host RAM: ~2.9 MB per 5v5 env), "
                      "not the full batch; SPS is flat in n_envs once n_envs >> cores (SPEC.md:426)")
    line = {
        "metric": metric_name(args.config),
        "value": base["value"], "unit": "agent-env steps/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config, "cpu_baseline": base,
        "e2e": {"value": base["value"], "unit": "agent-env steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def metric_name(name):
    return "agent-env steps/sec (5v5 fast targets)" if name == "c3" else f"agent-env steps/sec ({name})"


def free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(n):
    """`--gpus N` outside torchrun: re-launch this script as N ranks, exactly like
    the driver does (torch.distributed.run, rendezvous on 127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", str(pathlib.Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd, cwd=str(ROOT))


def dry_run(args):
    """The multi-rank plumbing without stepping: process group (NCCL on GPUs, gloo
    without), shard ranges, a MAX and a SUM all-reduce; rank 0 prints one line."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    use_cuda = torch.cuda.is_available()
    if world > 1:
        if use_cuda:
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl" if use_cuda else "gloo")
    scaling, per_gpu, total, lo, hi = shard_plan(args.config, world, rank, args)
    dev = "cuda" if use_cuda else "cpu"
    rng = torch.tensor([float(lo), float(hi)], dtype=torch.float64, device=dev)
    ranges = [torch.zeros_like(rng) for _ in range(world)]
    cnt = torch.tensor([float(hi - lo)], dtype=torch.float64, device=dev)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_gather(ranges, rng)
        dist.all_reduce(cnt)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    else:
        ranges = [rng]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "scaling": scaling, "total_envs": total,
                          "envs_per_gpu": per_gpu, "backend": dist.get_backend() if world > 1 else None,
                          "ranges": [[int(a), int(b)] for a, b in (r.tolist() for r in ranges)],
                          "envs_sum": int(cnt.item()), "max_rank": int(t.item())}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--scaling", default=None, choices=["strong", "weak"],
                    help="strong: --total-envs over all GPUs; weak: --envs-per-gpu on each (default per config)")
    ap.add_argument("--envs-per-gpu", type=int, default=None)
    ap.add_argument("--total-envs", type=int, default=None)
    ap.add_argument("--particles", type=int, default=1024)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-episode", action="store_true", help="skip the full-horizon / reset-step timing")
    ap.add_argument("--dry-run", action="store_true", help="rank plumbing only (no stepping)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.dry_run:
        return dry_run(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2505_08222_b200.vecenv import VecEnv
    from paper_2505_08222_b200._abi import STAT_NAMES

    cfg = make_cfg(args.config, args.particles)
    A, T, P = cfg.n_agents, cfg.n_targets, cfg.pf.n_particles
    scaling, per_gpu, total, lo, hi = shard_plan(args.config, world, rank, args)
    if CONFIGS[args.config].get("mix"):
        fleets = mix_fleet(lo, hi)
        shapes = [(a, t) for a in range(1, 9) for t in range(1, 9)]
        cfgs = [make_cfg(args.config, args.particles, a, t) for a, t in shapes]
        venv = VecEnv(cfgs, hi - lo, master_seed=0, env_index_offset=lo, device=local,
                      fleet=[shapes.index(f) for f in fleets])
        agents_local = sum(a for a, _ in fleets)
        pf_bytes_local = sum(80 * P * a * t for a, t in fleets)
    else:
        venv = VecEnv(cfg, hi - lo, master_seed=0, env_index_offset=lo, device=local)
        agents_local = (hi - lo) * A
        pf_bytes_local = (hi - lo) * 80 * P * A * T
    stream = torch.cuda.current_stream()
    venv.set_stream(stream.cuda_stream)  # the legacy default stream: the events below bracket the kernels

    venv.step_policy("random", args.warmup)
    torch.cuda.synchronize()
    # settle (untimed, on top of the W warm-up steps): a fresh box has shown a
    # first timed window ~50 % slower than every later one; step until two
    # consecutive single-step times agree within 3 % (at most 8 more steps)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prev, settle_steps = None, 0
    while settle_steps < 8:
        start.record(stream)
        venv.step_policy("random", 1)
        end.record(stream)
        torch.cuda.synchronize()
        settle_steps += 1
        t_one = start.elapsed_time(end)
        if prev is not None and abs(t_one - prev) <= 0.03 * prev:
            break
        prev = t_one
    # windows of exactly K steps; short ones are repeated until ~1 s has been
    # timed so the clock sampler (200 ms period) sees the load (median window);
    # each repeat starts at the same episode step (reset + the same warm-up)
    windows = max(1, min(5000, int(1000.0 / max(prev or t_one, 1e-3) / max(1, args.steps)) + 1))
    if world > 1:
        t_w = torch.tensor([windows], dtype=torch.int64, device="cuda")
        dist.all_reduce(t_w, op=dist.ReduceOp.MAX)
        windows = int(t_w.item())
    times, launches_timed, upd_sum = [], 0, 0.0
    i_upd = STAT_NAMES.index("pf_updates")
    with ClockSampler(local) as clocks:
        for w in range(windows):
            if w > 0:
                # every window starts at the episode step the first one did: the
                # step cost falls as the episode goes on (pings and resamples thin
                # out), so later windows would not time the same workload
                venv.reset_all()
                venv.step_policy("random", args.warmup + settle_steps)
            upd0 = float(venv.stats()[i_upd])
            launches0 = venv.launch_count()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            start.record(stream)
            venv.step_policy("random", args.steps)
            end.record(stream)
            torch.cuda.synchronize()
            times.append(start.elapsed_time(end))
            launches_timed += venv.launch_count() - launches0
            upd_sum += float(venv.stats()[i_upd]) - upd0
    gpu_launches = launches_timed // windows
    upd_timed = upd_sum / windows
    ms = statistics.median(times)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    secs = ms_max / 1e3
    env_steps = total * args.steps
    ag = torch.tensor([float(agents_local)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ag)
    agents_total = float(ag.item())  # = total * A for a homogeneous fleet
    value = agents_total * args.steps / secs

    # ---- one full horizon (auto-reset included: every env finishes once), then
    # the reset step alone, with the device phase timers on around it
    episode = None
    if not args.no_episode:
        horizon = CONFIGS[args.config]["horizon"]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        start.record(stream)
        venv.step_policy("random", horizon)
        end.record(stream)
        torch.cuda.synchronize()
        ep_ms = torch.tensor([start.elapsed_time(end)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(ep_ms, op=dist.ReduceOp.MAX)
        ep_ms = float(ep_ms.item())
        # align to the step before the (aligned) auto-reset
        k = venv.world_step(0)
        if k < horizon - 2:
            venv.step_policy("random", horizon - 2 - k)
        elif k == horizon - 1:
            venv.step_policy("random", horizon - 1)
        venv.enable_phase_timing(True)
        venv.phase_ns(reset=True)
        step_ms, phases = [], []
        for _ in range(3):  # before, reset, after
            torch.cuda.synchronize()
            start.record(stream)
            venv.step_policy("random", 1)
            end.record(stream)
            torch.cuda.synchronize()
            step_ms.append(start.elapsed_time(end))
            phases.append(venv.phase_ns(reset=True))
        venv.enable_phase_timing(False)
        names7 = ("targets", "agents", "measure", "filter", "comms", "observe", "reward")
        n_loc = hi - lo
        plain = {k: (phases[0][k] + phases[2][k]) / 2.0 for k in names7}
        tot7 = sum(plain.values()) or 1.0
        episode = {
            "steps": horizon, "ms": ep_ms, "ms_per_step": ep_ms / horizon,
            "value": agents_total * horizon / (ep_ms / 1e3),
            "reset_step_ms": step_ms[1], "step_ms_before_after_reset": [step_ms[0], step_ms[2]],
            "reset_over_step": step_ms[1] / (0.5 * (step_ms[0] + step_ms[2])),
            "note": "one horizon of steps timed as one window: every env auto-resets once inside it "
                    "(vecenv.cpp:140); `value` above is the K-step window the driver asks for",
            "phase_ns_per_env_step": {k: v / n_loc for k, v in plain.items()},
            "phase_share": {k: v / tot7 for k, v in plain.items()},
            "reset_ns_per_env": phases[1]["reset"] / n_loc,
            "phase_timer": "SM clock of thread 0 per CTA, CTA-summed, ns at the measured clock "
                           "(UT_PHASE_*, ut_env.h); shares comparable to cpu_baseline.phase_share",
        }

    # episode statistics: the one NCCL collective (north_star)
    st = torch.tensor(venv.stats(), dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(st)
    st = st.cpu().numpy()

    # ---- e2e through the public API with host buffers (pinned), copies timed.
    # The step cost depends on the episode step (pings and resamples thin out as
    # the targets run), so the e2e steps start where the timed window started:
    # a fresh reset, then the same warm-up and settle steps (untimed).
    # the same K steps from the same episode step as the device-timed window
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else args.steps
    if e2e_steps:
        venv.reset_all()
        venv.step_policy("random", args.warmup + settle_steps)
        torch.cuda.synchronize()
    n_loc = hi - lo
    Am, Rm, Tm = venv.n_agents(), venv.n_rows(), venv.n_targets()
    acts_h = torch.empty((n_loc, Am), dtype=torch.int32, pin_memory=True)
    host = {
        "obs": torch.empty((12, n_loc * Am * Rm), dtype=torch.float64, pin_memory=True),
        "global_state": torch.empty((12, n_loc * Rm), dtype=torch.float64, pin_memory=True),
        "rewards": torch.empty(n_loc, dtype=torch.float64, pin_memory=True),
        "dones": torch.empty(n_loc, dtype=torch.uint8, pin_memory=True),
        "masks": torch.empty(n_loc * Am * 5, dtype=torch.uint8, pin_memory=True),
        "tracking_error": torch.empty(n_loc * Tm, dtype=torch.float64, pin_memory=True),
        "min_agent_dist": torch.empty(n_loc * Tm, dtype=torch.float64, pin_memory=True),
        "target_lost": torch.empty(n_loc * Tm, dtype=torch.uint8, pin_memory=True),
        "collision": torch.empty(n_loc, dtype=torch.uint8, pin_memory=True),
    }
    d2h = sum(v.numel() * v.element_size() for v in host.values())
    h2d = acts_h.numel() * 4
    # Double-buffered outputs: the masks the host policy needs come back right
    # after each step; the rest of that step's outputs is copied on a side stream
    # while the next step runs (ut_vecenv_copy_outputs_async).
    venv.set_output_buffers(2)
    venv.set_stream(None)  # the handle's own non-blocking stream, as a default VecEnv runs
    copy_stream = torch.cuda.Stream()
    rest = {k: v for k, v in host.items() if k != "masks"}
    venv.copy_outputs_into({"masks": host["masks"]})
    acts_np = acts_h.numpy().reshape(-1)
    host_policy, policy_impl = make_host_policy(acts_np, n_loc * Am, rank)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    split = {"host_policy": 0.0, "step_call": 0.0, "masks_d2h": 0.0, "async_enqueue": 0.0}
    for _ in range(e2e_steps):
        ta = time.perf_counter()
        host_policy(host["masks"].numpy())
        tb = time.perf_counter()
        venv.step(acts_h)
        tc = time.perf_counter()
        venv.copy_outputs_into({"masks": host["masks"]})
        td = time.perf_counter()
        venv.copy_outputs_async(rest, copy_stream.cuda_stream)
        te_ = time.perf_counter()
        split["host_policy"] += tb - ta
        split["step_call"] += tc - tb
        split["masks_d2h"] += td - tc
        split["async_enqueue"] += te_ - td
    copy_stream.synchronize()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = agents_total * e2e_steps / float(te.item()) if e2e_steps else None

    peak, peak_kind = measured_peaks()
    # particle bytes of this shard's fleet + record and (padded) outputs per env
    per_env_rest = algorithmic_bytes_per_env_step(A, T, P, rec_words_for(A, T)) - 80 * P * A * T
    bytes_launch = pf_bytes_local + per_env_rest * (hi - lo)
    avg_launch_s = ms / 1e3 / max(1, args.steps)  # this rank's own launches
    achieved = bytes_launch / avg_launch_s / 1e9
    counts = measured_counts(args.config, hi - lo, P)
    fp64_peak = fp64_peak_per_s(local)
    sets_local = pf_bytes_local // (80 * P)
    if counts.get("fp64_thread_inst_per_launch"):
        fp64_launch = float(counts["fp64_thread_inst_per_launch"])
        fp64_src = counts.get("fp64_source", "ncu smsp__sass_thread_inst_executed_op_d{fma,mul,add}_pred_on.sum")
    else:  # SURVEY 8d model: 39 + 55 u fp64 instructions per particle-step
        fp64_launch = P * (39.0 * sets_local + 55.0 * upd_timed / max(1, args.steps))
        fp64_src = "model 39 + 55 u per particle-step (SURVEY 8d): no ncu counts for this workload"
    fp64_achieved = fp64_launch / avg_launch_s

    line = {
        "metric": metric_name(args.config),
        "value": value, "unit": "agent-env steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(workload_config(args.config, per_gpu, total, P, scaling), env_steps_per_s=env_steps / secs,
                       settle_steps=settle_steps, timed_windows=windows,
                       window_ms=[round(x, 4) for x in times]),
        "e2e": {"value": e2e_value, "unit": "agent-env steps/s", "h2d_bytes_per_step": h2d,
                "ms_per_step_split": {k: 1e3 * v / max(1, e2e_steps) for k, v in split.items()},
                "d2h_bytes_per_step": d2h, "steps": e2e_steps, "host_policy": policy_impl,
                "path": "VecEnv.step(host int32 actions from a host policy on the returned masks) + every output "
                        "to pinned host (ut_vecenv_step, ut_vecenv_copy_outputs for the masks, "
                        "ut_vecenv_copy_outputs_async for the rest, overlapping the next step); the e2e "
                        "steps are the timed window's K steps from the same episode step (reset + the same "
                        "warm-up and settle steps), on the handle's own stream"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": counts.get("dram_bytes_per_launch"),
                     "kernel": "step_kernel<4,1024,FULL>", "bytes_per_launch": bytes_launch,
                     "avg_launch_ms": avg_launch_s * 1e3, "peak_source": peak_kind,
                     "components": {
                         "hbm": {"achieved_gbs": achieved, "peak_gbs": peak, "frac": achieved / peak},
                         "fp64": {"achieved_tinstr_s": fp64_achieved / 1e12,
                                  "peak_tinstr_s": fp64_peak / 1e12 if fp64_peak else None,
                                  "frac": fp64_achieved / fp64_peak if fp64_peak else None,
                                  "instr_per_launch": fp64_launch, "source": fp64_src,
                                  "updates_per_set_step": upd_timed / max(1, sets_local * args.steps),
                                  "peak_source": "ut_debug_fp64_peak (8 DFMA chains/thread)"}}},
        "gpu_launches": gpu_launches,
        "clocks": clocks.summary(),
        "stats": {k: float(v) for k, v in zip(STAT_NAMES, st)},
    }
    if episode is not None:
        line["episode"] = episode
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(args.config, P)
        except Exception as exc:  # noqa: BLE001 -- reported, not fatal
            line["cpu_baseline"] = {"value": None, "error": str(exc)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    venv.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
