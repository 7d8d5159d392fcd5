"""Host-side mirror of the reference's C++ environment API, driving the B200
kernels through the C-ABI (include/ut_env.h).

Same names, argument meaning and error behaviour as utrack (paths relative to
/root/reference/proj/core):

* ``EnvConfig`` / ``PfConfig``     env_config.hpp:36-93 (``finalize`` env.cpp:40-65)
* ``VecEnv``                       vecenv.hpp:24-85 / vecenv.cpp
* ``Environment``                  env.hpp:91-171 (one env of a VecEnv shard)
* ``benchmark_sps``                vecenv.cpp:175-202
* ``ConfigError`` / ``DataError`` / ``ContractViolation``  errors.hpp:10-26

Batch views are zero-copy CUDA tensors over the library's device buffers;
``obs_stack()`` etc. have the reference's (rows, 12) shape and column-major
storage (the tensor is the transpose of a contiguous (12, rows) buffer).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import Optional, Sequence

import numpy as np

from . import _abi
from ._native import lib

kNumActions = _abi.UT_NUM_ACTIONS
kFeatureDim = _abi.UT_FEATURE_DIM


class ConfigError(RuntimeError):
    """Invalid or inconsistent configuration (errors.hpp:10-14; exit code 2)."""


class DataError(RuntimeError):
    """Malformed or incompatible data (errors.hpp:17-21; exit code 3)."""


class ContractViolation(ValueError):
    """A caller broke a documented precondition (errors.hpp:23-26; exit code 1)."""


class DeviceError(RuntimeError):
    """CUDA runtime failure (no reference counterpart)."""


_ERRORS = {_abi.UT_ERR_CONTRACT: ContractViolation, _abi.UT_ERR_CONFIG: ConfigError,
           _abi.UT_ERR_DATA: DataError, _abi.UT_ERR_RUNTIME: DeviceError}


def _check(rc):
    if rc != _abi.UT_OK:
        raise _ERRORS.get(rc, DeviceError)(lib().ut_last_error().decode())


@dataclasses.dataclass
class PfConfig:
    n_particles: int = 1024
    process_noise_pos: float = 1.0
    process_noise_vel: float = 0.05
    speed_margin: float = 1.2
    init_radius: float = 450.0


@dataclasses.dataclass
class EnvConfig:
    """EnvConfig (env_config.hpp:44-93). The heading model is the shipped default
    fit unless ``heading_bucket=(a, b)`` gives the (agent_speed, dt) bucket."""
    n_agents: int = 1
    n_targets: int = 1
    horizon: int = 128
    dt: float = 30.0
    agent_speed: float = 1.0
    target_speed_frac: float = 0.3
    target_speed_frac_max: float = 0.0
    target_turn_interval: float = 20.0
    detection_range: float = 450.0
    comm_range: float = 1500.0
    comm_drop_prob: float = 0.1
    range_noise_std: float = 3.0
    eps_min: float = 10.0
    eps_max: float = 50.0
    d_min: float = 50.0
    d_safe: float = 10.0
    reward_mode: str = "tracking"  # or "follow"
    spawn_min_sep: float = 50.0
    spawn_max_sep: float = 200.0
    perturbation_std: float = 0.0
    target_depth_min: float = 10.0
    target_depth_max: float = 60.0
    lost_steps: int = 20
    pf: PfConfig = dataclasses.field(default_factory=PfConfig)
    heading_noise_std: float = 0.02
    heading_bucket: Optional[tuple] = None

    def n_entities(self) -> int:
        return self.n_agents + self.n_targets

    def to_c(self) -> _abi.EnvConfigC:
        c = _abi.EnvConfigC()
        lib().ut_config_default(C.byref(c))
        for f in dataclasses.fields(self):
            if f.name in ("pf", "reward_mode", "heading_bucket"):
                continue
            setattr(c, f.name, getattr(self, f.name))
        if self.reward_mode not in ("tracking", "follow"):
            raise ConfigError("env.reward_mode must be 'tracking' or 'follow'")
        c.reward_mode = _abi.UT_REWARD_FOLLOW if self.reward_mode == "follow" else _abi.UT_REWARD_TRACKING
        for f in dataclasses.fields(self.pf):
            setattr(c.pf, f.name, getattr(self.pf, f.name))
        if self.heading_bucket is not None:
            c.heading_model_kind = _abi.UT_HEADING_BUCKET
            c.heading_a, c.heading_b = map(float, self.heading_bucket)
        return c

    def finalize(self) -> _abi.EnvConfigC:
        """EnvConfig::finalize (env.cpp:40-65): validates and resolves the bucket."""
        c = self.to_c()
        _check(lib().ut_config_finalize(C.byref(c)))
        return c


def rudder_angle(index: int) -> float:
    """env.cpp:67-72."""
    if index < 0 or index >= kNumActions:
        raise ContractViolation(f"rudder index out of range: {index}")
    return -0.24 + 0.12 * index


def valid_actions(rudder_index: int):
    """env.cpp:74-81."""
    if rudder_index < 0 or rudder_index >= kNumActions:
        raise ContractViolation(f"rudder index out of range: {rudder_index}")
    return [abs(i - rudder_index) <= 1 for i in range(kNumActions)]


class _DeviceArray:
    """__cuda_array_interface__ wrapper so torch.as_tensor can view a device buffer."""

    def __init__(self, ptr, shape, typestr, owner):
        self.__cuda_array_interface__ = {
            "shape": tuple(int(s) for s in shape), "typestr": typestr,
            "data": (int(ptr), False), "version": 3, "strides": None, "stream": None,
        }
        self._owner = owner


_POLICIES = {"random": _abi.UT_POLICY_RANDOM, "scripted": _abi.UT_POLICY_SCRIPTED,
             _abi.UT_POLICY_RANDOM: _abi.UT_POLICY_RANDOM, _abi.UT_POLICY_SCRIPTED: _abi.UT_POLICY_SCRIPTED}


class VecEnv:
    """Batched independent environments on one GPU (vecenv.hpp:24-85).

    ``env_index_offset`` makes this object a shard: env i is global env
    ``env_index_offset + i`` (its RNG streams are keyed by the global index), so
    shards of a batch are bit-identical to the same envs of the whole batch.
    """

    def __init__(self, cfg, n_envs: int, master_seed: int, workers: int = 0, *,
                 env_index_offset: int = 0, device: int = 0, fleet: Optional[Sequence[int]] = None):
        self._lib = lib()
        self._h = C.c_void_p()
        if isinstance(cfg, (list, tuple)):
            cfgs = [c.to_c() for c in cfg]
            if fleet is None or len(fleet) != n_envs:
                raise ConfigError("mixed VecEnv needs fleet (config index per env)")
            arr = (_abi.EnvConfigC * len(cfgs))(*cfgs)
            fl = np.ascontiguousarray(fleet, np.int32)
            _check(self._lib.ut_vecenv_create_mixed(arr, len(cfgs), fl.ctypes.data_as(C.POINTER(C.c_int32)),
                                                    n_envs, master_seed, env_index_offset, device,
                                                    C.byref(self._h)))
            self._cfgs = list(cfg)
            self._config = cfg[0]
        else:
            c = cfg.to_c()
            _check(self._lib.ut_vecenv_create(C.byref(c), n_envs, master_seed, env_index_offset, device,
                                              C.byref(self._h)))
            self._cfgs = [cfg]
            self._config = cfg
        self.device = device
        self.master_seed = master_seed
        self.env_index_offset = env_index_offset
        self._b = _abi.Buffers()
        _check(self._lib.ut_vecenv_buffers(self._h, C.byref(self._b)))
        self._views = {}
        self._n_out = 1
        self._set_offsets = None
        if isinstance(cfg, (list, tuple)):  # ragged particle store (ut_buffers.set_offset)
            sizes = np.array([cfg[f].n_agents * cfg[f].n_targets for f in fleet], np.int64)
            self._set_offsets = np.concatenate([[0], np.cumsum(sizes)])

    # -- shape (vecenv.hpp:29-33)
    def n_envs(self) -> int:
        return int(self._b.n_envs)

    def n_agents(self) -> int:
        return int(self._b.n_agents)

    def n_targets(self) -> int:
        return int(self._b.n_targets)

    def n_rows(self) -> int:
        return int(self._b.n_rows)

    def n_particles(self) -> int:
        return int(self._b.n_particles)

    def config(self):
        return self._config

    # -- output buffering (ut_vecenv_set_output_buffers)
    def set_output_buffers(self, n: int):
        """n = 2: each step writes the batch buffers the previous step did not, so
        copy_outputs_async() of one step overlaps the next step's kernel."""
        _check(self._lib.ut_vecenv_set_output_buffers(self._h, n))
        self._n_out = n
        self._sync_buffers()

    def _sync_buffers(self):
        _check(self._lib.ut_vecenv_buffers(self._h, C.byref(self._b)))
        self._views = {k: v for k, v in self._views.items() if k.startswith("pf_")}

    def _after_write(self):
        if self._n_out == 2:
            self._sync_buffers()

    # -- stream ordering
    def _order_after_caller(self):
        """The next device work of this handle runs after everything torch has
        already enqueued on its current stream (a GPU policy producing actions,
        kernels still reading the zero-copy output views)."""
        import sys
        torch = sys.modules.get("torch")
        if torch is not None and torch.cuda.is_available() and torch.cuda.is_initialized():
            s = torch.cuda.current_stream(self.device).cuda_stream
            _check(self._lib.ut_vecenv_wait_stream(self._h, C.c_void_p(s)))

    # -- stepping
    def reset_all(self):
        """vecenv.cpp:69-77."""
        self._order_after_caller()
        _check(self._lib.ut_vecenv_reset_all(self._h))
        self._after_write()

    def step(self, actions):
        """vecenv.cpp:79-116. actions: n_envs x n_agents ints (numpy / list / CPU or
        CUDA tensor). Every action is validated before any env moves."""
        try:
            import torch
            if isinstance(actions, torch.Tensor):
                t = actions.to(torch.int32).contiguous()
                if t.numel() != self.n_envs() * self.n_agents():
                    raise ContractViolation("vecenv step: wrong action count")
                if t.is_cuda:
                    self._order_after_caller()  # the producer of `actions` may still be running
                    _check(self._lib.ut_vecenv_step(self._h, C.c_void_p(t.data_ptr()), 1))
                    self._after_write()
                    return
                actions = t.numpy()
        except ImportError:
            pass
        a = np.ascontiguousarray(actions, dtype=np.int32).reshape(-1)
        if a.size != self.n_envs() * self.n_agents():
            raise ContractViolation("vecenv step: wrong action count")
        self._order_after_caller()
        _check(self._lib.ut_vecenv_step(self._h, C.c_void_p(a.ctypes.data), 0))
        self._after_write()

    def step_policy(self, policy="random", n_steps: int = 1):
        """vecenv.cpp:118-143 (``n_steps`` > 1 runs back-to-back device steps)."""
        if policy not in _POLICIES:
            raise ContractViolation(f"unknown policy {policy!r}")
        self._order_after_caller()
        _check(self._lib.ut_vecenv_step_policy(self._h, _POLICIES[policy], n_steps))
        self._after_write()

    def refresh_outputs(self):
        """vecenv.cpp:145-150."""
        self._order_after_caller()
        _check(self._lib.ut_vecenv_refresh_outputs(self._h))

    # -- zero-copy device views (vecenv.hpp:51-62)
    def _view(self, name, ptr, shape, typestr):
        import torch
        if name not in self._views:
            self._views[name] = torch.as_tensor(_DeviceArray(ptr, shape, typestr, self),
                                                device=f"cuda:{self.device}")
        return self._views[name]

    def obs_stack(self):
        return self._view("obs", self._b.obs, (kFeatureDim, self._b.obs_rows), "<f8").t()

    def final_obs_stack(self):
        return self._view("final_obs", self._b.final_obs, (kFeatureDim, self._b.obs_rows), "<f8").t()

    def global_stack(self):
        return self._view("global", self._b.global_state, (kFeatureDim, self._b.global_rows), "<f8").t()

    def rewards(self):
        return self._view("rewards", self._b.rewards, (self._b.n_envs,), "<f8")

    def dones(self):
        return self._view("dones", self._b.dones, (self._b.n_envs,), "|u1")

    def masks(self):
        return self._view("masks", self._b.masks, (self._b.n_envs * self._b.n_agents * kNumActions,), "|u1")

    def infos(self):
        """StepOutput fields (env.hpp:53-60) as per-env device tensors."""
        n, T = self._b.n_envs, self._b.n_targets
        return {
            "reward": self.rewards(),
            "done": self.dones(),
            "collision": self._view("collision", self._b.collision, (n,), "|u1"),
            "tracking_error": self._view("track_err", self._b.tracking_error, (n, T), "<f8"),
            "min_agent_dist": self._view("min_dist", self._b.min_agent_dist, (n, T), "<f8"),
            "target_lost": self._view("lost", self._b.target_lost, (n, T), "|u1"),
            "step": self._view("step", self._b.step, (n,), "<i4"),
        }

    def particles(self):
        """The SoA particle store: px, py, vx, vy, w each (total_sets, P). Env e's
        set (a, t) is row set_offset(e) + a * T_e + t."""
        P = self._b.n_particles
        n_sets = int(self._b.total_sets)
        return {k: self._view("pf_" + k, getattr(self._b, k), (n_sets, P), "<f8")
                for k in ("px", "py", "vx", "vy", "w")}

    def set_offset(self, env: int) -> int:
        """First particle-set row of env `env` (ragged for mixed fleets)."""
        if self._set_offsets is None:
            return env * self.n_agents() * self.n_targets()
        return int(self._set_offsets[env])

    def host_outputs(self, names=None):
        """Copies the batch buffers to host numpy arrays (one synchronous call)."""
        n, A, T, R = self._b.n_envs, self._b.n_agents, self._b.n_targets, self._b.n_rows
        shapes = {
            "obs": ((kFeatureDim, n * A * R), np.float64), "final_obs": ((kFeatureDim, n * A * R), np.float64),
            "global_state": ((kFeatureDim, n * R), np.float64), "rewards": ((n,), np.float64),
            "dones": ((n,), np.uint8), "masks": ((n * A * kNumActions,), np.uint8),
            "tracking_error": ((n * T,), np.float64), "min_agent_dist": ((n * T,), np.float64),
            "target_lost": ((n * T,), np.uint8), "collision": ((n,), np.uint8), "step": ((n,), np.int32),
        }
        names = list(shapes) if names is None else list(names)
        out = {k: np.empty(*shapes[k]) for k in names}
        ho = _abi.HostOutputs(**{k: v.ctypes.data for k, v in out.items()})
        _check(self._lib.ut_vecenv_copy_outputs(self._h, C.byref(ho)))
        return out

    def copy_outputs_into(self, host: dict):
        """ut_vecenv_copy_outputs into caller-owned (e.g. pinned) host buffers."""
        ho = _abi.HostOutputs(**{k: int(v.data_ptr() if hasattr(v, "data_ptr") else v.ctypes.data)
                                 for k, v in host.items()})
        _check(self._lib.ut_vecenv_copy_outputs(self._h, C.byref(ho)))

    def copy_outputs_async(self, host: dict, stream_ptr: int):
        """ut_vecenv_copy_outputs_async: enqueue the copies on a CUDA stream and
        return (pinned host buffers; synchronize the stream before reading)."""
        ho = _abi.HostOutputs(**{k: int(v.data_ptr() if hasattr(v, "data_ptr") else v.ctypes.data)
                                 for k, v in host.items()})
        _check(self._lib.ut_vecenv_copy_outputs_async(self._h, C.byref(ho), C.c_void_p(stream_ptr)))

    # -- per-env state (env.hpp:130-137)
    def serialize_state(self, env: int) -> np.ndarray:
        n = C.c_size_t()
        _check(self._lib.ut_env_serialize(self._h, env, None, 0, C.byref(n)))
        blob = np.empty(n.value, np.float64)
        _check(self._lib.ut_env_serialize(self._h, env, blob.ctypes.data_as(C.POINTER(C.c_double)), n.value,
                                          C.byref(n)))
        return blob

    def deserialize_state(self, env: int, blob):
        b = np.ascontiguousarray(blob, np.float64)
        _check(self._lib.ut_env_deserialize(self._h, env, b.ctypes.data_as(C.POINTER(C.c_double)), b.size))

    def export_state(self, begin: int = 0, end: Optional[int] = None) -> np.ndarray:
        """serialize_state of envs [begin, end) in one device pass: the blobs back
        to back (shape (n, blob_len) for a homogeneous fleet, flat otherwise)."""
        end = self.n_envs() if end is None else end
        n = C.c_size_t()
        _check(self._lib.ut_vecenv_export_state(self._h, begin, end, None, 0, C.byref(n)))
        out = np.empty(n.value, np.float64)
        _check(self._lib.ut_vecenv_export_state(self._h, begin, end, out.ctypes.data_as(C.POINTER(C.c_double)),
                                                n.value, C.byref(n)))
        if len(self._cfgs) == 1 and end > begin:
            out = out.reshape(end - begin, -1)
        return out

    def import_state(self, blobs, begin: int = 0, end: Optional[int] = None):
        """deserialize_state of envs [begin, end) from blobs back to back."""
        end = self.n_envs() if end is None else end
        b = np.ascontiguousarray(blobs, np.float64).reshape(-1)
        _check(self._lib.ut_vecenv_import_state(self._h, begin, end, b.ctypes.data_as(C.POINTER(C.c_double)),
                                                b.size))

    def capture_trajectory(self, begin: int, end: int):
        """Record append_trajectory_rows (trajectory.cpp:13-66) for envs [begin,
        end) after every step, before auto-reset (empty range: off)."""
        _check(self._lib.ut_vecenv_capture_trajectory(self._h, begin, end))

    def trajectory_rows(self) -> np.ndarray:
        """The last step's captured rows: (n_captured, n_rows, UT_TRAJ_FIELDS)."""
        n = C.c_size_t()
        _check(self._lib.ut_vecenv_trajectory_rows(self._h, None, 0, C.byref(n)))
        out = np.empty(n.value, np.float64)
        _check(self._lib.ut_vecenv_trajectory_rows(self._h, out.ctypes.data_as(C.POINTER(C.c_double)), n.value,
                                                   C.byref(n)))
        return out.reshape(-1, self._b.n_rows, _abi.UT_TRAJ_FIELDS)

    def world_step(self, env: int) -> int:
        s = C.c_int32()
        _check(self._lib.ut_env_world_step(self._h, env, C.byref(s)))
        return s.value

    def eval_metrics(self) -> dict:
        """curriculum::evaluate's Table-2 metrics (curriculum.cpp:267-356) over the
        episodes completed so far, accumulated on the device: mean / population std
        of the per-episode mean agent-target distance and mean tracking error, and
        the percentage of episodes with a collision / a lost target."""
        st = dict(zip(_abi.STAT_NAMES, self.stats()))
        n = st["episodes_done"]
        if n <= 0:
            return {"episodes": 0}

        def mean_std(s, sq):
            mu = s / n
            return mu, float(np.sqrt(max(sq / n - mu * mu, 0.0)))

        dm, ds = mean_std(st["eval_dist_sum"], st["eval_dist_sq"])
        em, es = mean_std(st["eval_err_sum"], st["eval_err_sq"])
        return {"episodes": int(n), "dist_mean": dm, "dist_std": ds, "err_mean": em, "err_std": es,
                "collision_pct": 100.0 * st["eval_collided_episodes"] / n,
                "loss_pct": 100.0 * st["eval_lost_episodes"] / n}

    def stats(self, reset: bool = False) -> np.ndarray:
        out = (C.c_double * _abi.UT_N_STATS)()
        _check(self._lib.ut_vecenv_stats(self._h, out, int(reset)))
        return np.array(out[:])

    PHASES = _abi.PHASE_NAMES

    def enable_phase_timing(self, on: bool = True):
        """VecEnv::enable_phase_timing (vecenv.hpp:64) on the device."""
        _check(self._lib.ut_vecenv_enable_phase_timing(self._h, int(on)))

    def phase_cycles(self, reset: bool = False) -> dict:
        """SM cycles per phase (the reference's seven + reset), CTA-summed."""
        out = (C.c_uint64 * len(self.PHASES))()
        _check(self._lib.ut_vecenv_phase_cycles(self._h, out, int(reset)))
        return dict(zip(self.PHASES, out[:]))

    def phase_ns(self, reset: bool = False) -> dict:
        """VecEnv::phase_ns (vecenv.cpp:160-173): ns per phase, CTA-summed."""
        out = (C.c_uint64 * len(self.PHASES))()
        _check(self._lib.ut_vecenv_phase_ns(self._h, out, int(reset)))
        return dict(zip(self.PHASES, out[:]))

    def set_auto_reset(self, on: bool):
        """Auto-reset of finished envs (vecenv.cpp:106-112); off = Environment semantics."""
        _check(self._lib.ut_vecenv_set_auto_reset(self._h, int(on)))

    def launch_count(self) -> int:
        return int(self._lib.ut_vecenv_launch_count(self._h))

    def set_stream(self, stream_ptr):
        """Run on a caller's CUDA stream; 0 is the legacy default stream (torch's
        default), passed to the library as UT_STREAM_LEGACY; None returns to the
        handle's own non-blocking stream."""
        if stream_ptr is None:
            _check(self._lib.ut_vecenv_set_stream(self._h, None))
            return
        s = stream_ptr if stream_ptr else _abi.UT_STREAM_LEGACY
        _check(self._lib.ut_vecenv_set_stream(self._h, C.c_void_p(s)))

    def synchronize(self):
        _check(self._lib.ut_vecenv_synchronize(self._h))

    def close(self):
        if getattr(self, "_h", None):
            self._views.clear()
            self._lib.ut_vecenv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MultiVecEnv:
    """One VecEnv over several GPUs of one box (ut_multienv_*): the reference's
    single VecEnv over all envs (vecenv.hpp:26-27), sharded by contiguous env index
    range over ``devices`` instead of worker threads (vecenv.cpp:83). Bit-identical
    to ``VecEnv(cfg, n_envs, seed)``; the statistics are all-reduced over NCCL
    (``stats_backend() == "nccl"``), or summed on the host when a device repeats."""

    _BACKENDS = {"auto": _abi.UT_MULTI_STATS_AUTO, "nccl": _abi.UT_MULTI_STATS_NCCL,
                 "host": _abi.UT_MULTI_STATS_HOST}

    def __init__(self, cfg: EnvConfig, n_envs: int, master_seed: int, devices: Sequence[int] = (0,),
                 stats: str = "auto"):
        self._lib = lib()
        self._h = C.c_void_p()
        c = cfg.to_c()
        dev = (C.c_int32 * len(devices))(*devices)
        _check(self._lib.ut_multienv_create(C.byref(c), n_envs, master_seed, dev, len(devices),
                                            self._BACKENDS[stats], C.byref(self._h)))
        self._cfg = cfg
        self._n = n_envs
        self.devices = list(devices)

    def n_envs(self) -> int:
        return self._n

    def n_shards(self) -> int:
        return int(self._lib.ut_multienv_n_shards(self._h))

    def shard_range(self, i: int):
        b, e, d = C.c_int64(), C.c_int64(), C.c_int32()
        _check(self._lib.ut_multienv_shard(self._h, i, None, C.byref(b), C.byref(e), C.byref(d)))
        return int(b.value), int(e.value), int(d.value)

    def stats_backend(self) -> str:
        return "nccl" if self._lib.ut_multienv_stats_backend(self._h) == _abi.UT_MULTI_STATS_NCCL else "host"

    def reset_all(self):
        _check(self._lib.ut_multienv_reset_all(self._h))

    def step(self, actions):
        a = np.ascontiguousarray(np.asarray(actions, np.int32).reshape(-1))
        if a.size != self._n * self._cfg.n_agents:
            raise ContractViolation("vecenv step: wrong action count")
        _check(self._lib.ut_multienv_step(self._h, a.ctypes.data_as(C.c_void_p)))

    def step_policy(self, policy="random", n_steps: int = 1):
        _check(self._lib.ut_multienv_step_policy(self._h, _POLICIES[policy], n_steps))

    def refresh_outputs(self):
        _check(self._lib.ut_multienv_refresh_outputs(self._h))

    def set_auto_reset(self, on: bool):
        _check(self._lib.ut_multienv_set_auto_reset(self._h, int(on)))

    def host_outputs(self, names=None):
        """The whole batch's outputs, laid out like VecEnv.host_outputs()."""
        n, A, T = self._n, self._cfg.n_agents, self._cfg.n_targets
        R = A + T
        shapes = {
            "obs": ((kFeatureDim, n * A * R), np.float64), "final_obs": ((kFeatureDim, n * A * R), np.float64),
            "global_state": ((kFeatureDim, n * R), np.float64), "rewards": ((n,), np.float64),
            "dones": ((n,), np.uint8), "masks": ((n * A * kNumActions,), np.uint8),
            "tracking_error": ((n * T,), np.float64), "min_agent_dist": ((n * T,), np.float64),
            "target_lost": ((n * T,), np.uint8), "collision": ((n,), np.uint8), "step": ((n,), np.int32),
        }
        names = list(shapes) if names is None else list(names)
        out = {k: np.empty(*shapes[k]) for k in names}
        ho = _abi.HostOutputs(**{k: v.ctypes.data for k, v in out.items()})
        _check(self._lib.ut_multienv_copy_outputs(self._h, C.byref(ho)))
        return out

    def stats(self, reset: bool = False) -> np.ndarray:
        out = (C.c_double * _abi.UT_N_STATS)()
        _check(self._lib.ut_multienv_stats(self._h, out, int(reset)))
        return np.array(out[:])

    def enable_phase_timing(self, on: bool = True):
        _check(self._lib.ut_multienv_enable_phase_timing(self._h, int(on)))

    def phase_ns(self, reset: bool = False) -> dict:
        out = (C.c_uint64 * _abi.UT_N_PHASES)()
        _check(self._lib.ut_multienv_phase_ns(self._h, out, int(reset)))
        return dict(zip(_abi.PHASE_NAMES, out[:]))

    def serialize_state(self, env: int) -> np.ndarray:
        n = C.c_size_t()
        _check(self._lib.ut_multienv_serialize(self._h, env, None, 0, C.byref(n)))
        blob = np.empty(n.value, np.float64)
        _check(self._lib.ut_multienv_serialize(self._h, env, blob.ctypes.data_as(C.POINTER(C.c_double)),
                                               blob.size, C.byref(n)))
        return blob

    def deserialize_state(self, env: int, blob):
        b = np.ascontiguousarray(blob, np.float64)
        _check(self._lib.ut_multienv_deserialize(self._h, env, b.ctypes.data_as(C.POINTER(C.c_double)), b.size))

    def world_step(self, env: int) -> int:
        s = C.c_int32()
        _check(self._lib.ut_multienv_world_step(self._h, env, C.byref(s)))
        return int(s.value)

    def launch_count(self) -> int:
        return int(self._lib.ut_multienv_launch_count(self._h))

    def synchronize(self):
        _check(self._lib.ut_multienv_synchronize(self._h))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.ut_multienv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Environment:
    """One environment (env.hpp:91-171): a VecEnv shard holding the single global
    env ``env_index``, so its streams equal ``Environment(cfg, seed, env_index)``.
    Like the reference it never resets on its own (env.cpp:234-504): after the
    terminal step the state stays terminal (done stays set) until ``reset()``."""

    def __init__(self, cfg: EnvConfig, seed: int, env_index: int = 0, device: int = 0):
        self._v = VecEnv(cfg, 1, seed, env_index_offset=env_index, device=device)
        self._v.set_auto_reset(False)
        self._cfg = cfg

    def config(self):
        return self._cfg

    def reset(self):
        """Environment::reset (env.cpp:153-233)."""
        self._v.reset_all()

    def step(self, actions):
        """Environment::step (env.cpp:235-287); invalid actions raise
        ContractViolation("step: invalid action ...") and change nothing."""
        try:
            self._v.step(np.asarray(actions, np.int32).reshape(1, -1))
        except ContractViolation as exc:
            msg = str(exc)
            raise ContractViolation(msg.split(": ", 1)[1] if msg.startswith("env ") else msg) from None
        o = self._v.host_outputs(["rewards", "dones", "collision", "tracking_error", "min_agent_dist",
                                  "target_lost"])
        return {"reward": float(o["rewards"][0]), "done": bool(o["dones"][0]),
                "collision": bool(o["collision"][0]), "tracking_error": o["tracking_error"].tolist(),
                "min_agent_dist": o["min_agent_dist"].tolist(),
                "target_lost": o["target_lost"].tolist()}

    def observation(self, agent: int) -> np.ndarray:
        R = self._v.n_rows()
        obs = self._v.host_outputs(["obs"])["obs"]
        return obs[:, agent * R:(agent + 1) * R].T.copy()

    def global_state(self) -> np.ndarray:
        return self._v.host_outputs(["global_state"])["global_state"].T.copy()

    def action_mask(self, agent: int):
        m = self._v.host_outputs(["masks"])["masks"]
        return [bool(x) for x in m[agent * kNumActions:(agent + 1) * kNumActions]]

    def serialize_state(self):
        return self._v.serialize_state(0)

    def deserialize_state(self, blob):
        self._v.deserialize_state(0, blob)
        self._v.refresh_outputs()

    def world_step(self) -> int:
        return self._v.world_step(0)

    def close(self):
        self._v.close()


def benchmark_sps(cfg: EnvConfig, n_envs: int, n_steps: int, policy="random", seed: int = 0,
                  workers: int = 0, warmup: int = 16, device: int = 0) -> dict:
    """benchmark_sps (vecenv.cpp:175-202) on the device, CUDA-event timed."""
    rep = _abi.BenchmarkReport()
    c = cfg.to_c()
    _check(lib().ut_benchmark_sps(C.byref(c), n_envs, n_steps, _POLICIES[policy], seed, warmup, device,
                                  C.byref(rep)))
    return {"n_envs": rep.n_envs, "n_agents": rep.n_agents, "n_targets": rep.n_targets,
            "timed_steps": rep.timed_steps, "wall_seconds": rep.wall_seconds, "sps": rep.sps,
            "agent_sps": rep.agent_sps, "phase_ns": dict(zip(_abi.PHASE_NAMES, rep.phase_ns[:])),
            "total_ns": rep.total_ns}
