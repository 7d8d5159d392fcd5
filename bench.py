#!/usr/bin/env python3
"""Throughput of the batched JaxLrauv environment step on B200.

Metric (BASELINE.json): agent-env steps/sec on the 5-agent / 5-fast-target
workload (65,536 envs per GPU, P = 1024, fp64 particle
filters), random legal actions from the device bench stream (vecenv.cpp:118-135).
Multi-GPU (torchrun): envs shard by global index range, each GPU steps its
shard independently (weak scaling, no data-path collective); the episode
statistics are all-reduced once over NCCL after the run.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]
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
        for line in self.path.read_text().splitlines():
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


def workload_config(name, per_gpu, total, particles):
    """The `config` object both arms print (same workload, same keys)."""
    c = CONFIGS[name]
    A, T = c["n_agents"], c["n_targets"]
    gb = algorithmic_bytes_per_env_step(A, T, particles, rec_words_for(A, T)) * per_gpu / 1e9
    return {"workload": f"{name}: {c['desc']}", "envs_per_gpu": per_gpu, "total_envs": total,
            "particles": particles, "agents": A, "targets": T,
            "policy": "random legal (bench stream, vecenv.cpp:125-134)",
            "l2": f"inputs larger than L2 ({gb:.1f} GB touched per step per GPU)"}


def measured_traffic(name, per_gpu, particles):
    """DRAM bytes per step-kernel launch from the committed ncu --set full capture
    of the same workload (profiles/traffic.json), or None."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text()).get(f"{name}:{per_gpu}:{particles}")
    return None if d is None else float(d["dram_bytes_per_launch"])


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
    return {"value": sps * A, "unit": "agent-env steps/s", "cores": wk, "kind": kind,
            "sample": f"{n_envs} envs x {steps} steps of {cfg_name} (P={particles}), "
                      f"benchmark_sps(kRandom) after 2 warmup steps, {wall:.1f} s wall",
            "env_sps": sps, "phase_ns": dict(zip(names, ph)) if ph else None}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    base = cpu_baseline(args.config, args.particles, budget_s=max(5.0, 2.0 * (args.steps + args.warmup)))
    per_gpu = args.envs_per_gpu or CONFIGS[args.config]["envs"]
    line = {
        "metric": "agent-env steps/sec (5v5 fast targets)" if args.config == "c3" else f"agent-env steps/sec ({args.config})",
        "value": base["value"], "unit": "agent-env steps/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.config, per_gpu, per_gpu * args.gpus, args.particles),
        "cpu_baseline": base,
        "e2e": {"value": base["value"], "unit": "agent-env steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--envs-per-gpu", type=int, default=None)
    ap.add_argument("--particles", type=int, default=1024)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--traffic-bytes", type=float, default=None,
                    help="dram bytes per launch from an ncu --set full capture (profiles/)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2505_08222_b200.vecenv import VecEnv
    from paper_2505_08222_b200.sharding import shard_range
    from paper_2505_08222_b200._abi import STAT_NAMES

    cfg = make_cfg(args.config, args.particles)
    A, T, P = cfg.n_agents, cfg.n_targets, cfg.pf.n_particles
    per_gpu = args.envs_per_gpu or CONFIGS[args.config]["envs"]
    total = per_gpu * world
    lo, hi = shard_range(total, rank, world)
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
    venv.set_stream(stream.cuda_stream)

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
    if world > 1:
        dist.barrier()
    launches0 = venv.launch_count()
    upd0 = float(venv.stats()[STAT_NAMES.index("pf_updates")])
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        start.record(stream)
        venv.step_policy("random", args.steps)
        end.record(stream)
        torch.cuda.synchronize()
    gpu_launches = venv.launch_count() - launches0
    upd_timed = float(venv.stats()[STAT_NAMES.index("pf_updates")]) - upd0
    ms = start.elapsed_time(end)
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

    # episode statistics: the one NCCL collective (north_star)
    st = torch.tensor(venv.stats(), dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(st)
    st = st.cpu().numpy()

    # ---- e2e through the public API with host buffers (pinned), copies timed
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else min(args.steps, 10)
    n_loc = hi - lo
    acts_h = torch.empty((n_loc, A), dtype=torch.int32, pin_memory=True)
    host = {
        "obs": torch.empty((12, n_loc * A * (A + T)), dtype=torch.float64, pin_memory=True),
        "global_state": torch.empty((12, n_loc * (A + T)), dtype=torch.float64, pin_memory=True),
        "rewards": torch.empty(n_loc, dtype=torch.float64, pin_memory=True),
        "dones": torch.empty(n_loc, dtype=torch.uint8, pin_memory=True),
        "masks": torch.empty(n_loc * A * 5, dtype=torch.uint8, pin_memory=True),
        "tracking_error": torch.empty(n_loc * T, dtype=torch.float64, pin_memory=True),
        "min_agent_dist": torch.empty(n_loc * T, dtype=torch.float64, pin_memory=True),
        "target_lost": torch.empty(n_loc * T, dtype=torch.uint8, pin_memory=True),
        "collision": torch.empty(n_loc, dtype=torch.uint8, pin_memory=True),
    }
    d2h = sum(v.numel() * v.element_size() for v in host.values())
    h2d = acts_h.numel() * 4
    # Double-buffered outputs: the masks the host policy needs come back right
    # after each step; the rest of that step's outputs is copied on a side stream
    # while the next step runs (ut_vecenv_copy_outputs_async).
    venv.set_output_buffers(2)
    copy_stream = torch.cuda.Stream()
    rest = {k: v for k, v in host.items() if k != "masks"}
    venv.copy_outputs_into({"masks": host["masks"]})
    rng = np.random.default_rng(rank)
    acts_np = acts_h.numpy().reshape(-1)
    # host policy: a uniform legal action per agent from its returned 5-bit mask
    # (lookup of the j-th set bit, j = floor(u * #legal)), vectorised with
    # preallocated buffers and 1-D takes
    kth = np.zeros((32, 5), np.int32)
    n_legal = np.zeros(32, np.float32)
    for code in range(32):
        bits = [b for b in range(5) if (code >> b) & 1]
        n_legal[code] = len(bits)
        kth[code, :len(bits)] = bits
    kth_flat = kth.reshape(-1)
    n_ag = n_loc * A
    u = np.empty(n_ag, np.float32)
    code = np.empty(n_ag, np.uint8)
    tmp = np.empty(n_ag, np.uint8)
    flat = np.empty(n_ag, np.int64)

    def host_policy(mv):
        np.bitwise_or(mv[:, 0], np.left_shift(mv[:, 1], 1, out=tmp), out=code)
        for b in (2, 3, 4):
            np.bitwise_or(code, np.left_shift(mv[:, b], b, out=tmp), out=code)
        rng.random(out=u, dtype=np.float32)
        np.multiply(u, n_legal.take(code), out=u)
        flat[:] = u                      # floor (u * #legal) < #legal
        np.add(flat, code.astype(np.int64) * 5, out=flat)
        kth_flat.take(flat, out=acts_np)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        host_policy(host["masks"].numpy().reshape(-1, 5))
        venv.step(acts_h)
        venv.copy_outputs_into({"masks": host["masks"]})
        venv.copy_outputs_async(rest, copy_stream.cuda_stream)
    copy_stream.synchronize()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = agents_total * e2e_steps / float(te.item())

    peak, peak_kind = measured_peaks()
    # particle bytes of this shard's fleet + record and (padded) outputs per env
    per_env_rest = algorithmic_bytes_per_env_step(A, T, P, rec_words_for(A, T)) - 80 * P * A * T
    bytes_launch = pf_bytes_local + per_env_rest * (hi - lo)
    avg_launch_s = secs / max(1, args.steps)
    achieved = bytes_launch / avg_launch_s / 1e9
    # SURVEY 8d fp64 component: 39 + 55 u algorithmic fp64 instructions per
    # particle per step (u = range updates applied to its set this step, counted
    # by the kernel), against the device's measured DFMA issue rate.
    sets_local = pf_bytes_local // (80 * P)
    fp64_launch = P * (39.0 * sets_local * args.steps + 55.0 * upd_timed) / args.steps
    fp64_peak = fp64_peak_per_s(local)
    fp64_achieved = fp64_launch / avg_launch_s

    line = {
        "metric": "agent-env steps/sec (5v5 fast targets)" if args.config == "c3" else f"agent-env steps/sec ({args.config})",
        "value": value, "unit": "agent-env steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(workload_config(args.config, per_gpu, total, P), env_steps_per_s=env_steps / secs,
                       settle_steps=settle_steps),
        "e2e": {"value": e2e_value, "unit": "agent-env steps/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                "path": "VecEnv.step(host int32 actions from a host policy on the returned masks) + every output to pinned host (ut_vecenv_step, ut_vecenv_copy_outputs for the masks, ut_vecenv_copy_outputs_async for the rest, overlapping the next step)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": args.traffic_bytes if args.traffic_bytes is not None
                     else measured_traffic(args.config, per_gpu, P),
                     "kernel": "step_kernel<4,1024,FULL>", "bytes_per_launch": bytes_launch,
                     "avg_launch_ms": avg_launch_s * 1e3, "peak_source": peak_kind,
                     "components": {
                         "hbm": {"achieved_gbs": achieved, "peak_gbs": peak, "frac": achieved / peak},
                         "fp64": {"achieved_tinstr_s": fp64_achieved / 1e12,
                                  "peak_tinstr_s": fp64_peak / 1e12 if fp64_peak else None,
                                  "frac": fp64_achieved / fp64_peak if fp64_peak else None,
                                  "instr_per_launch": fp64_launch,
                                  "updates_per_set_step": upd_timed / max(1, sets_local * args.steps),
                                  "model": "39 + 55 u fp64 instr per particle-step (SURVEY 8d)",
                                  "peak_source": "ut_debug_fp64_peak (8 DFMA chains/thread)"}}},
        "gpu_launches": gpu_launches,
        "clocks": clocks.summary(),
        "stats": {k: float(v) for k, v in zip(STAT_NAMES, st)},
    }
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
