"""TEST INFRASTRUCTURE: ctypes bindings for the oracle libraries.

* ``Oracle``   -- the plain-C restatement, oracle/_build/libut_oracle.so
* ``RefVecEnv`` -- the reference's own VecEnv compiled against the Eigen shim,
  oracle/_ref/libutrack_ref.so (prebuilt here; travels to the GPU box)

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module.
"""
import ctypes as C
import os
import pathlib

import numpy as np

from paper_2505_08222_b200._abi import (EnvConfigC, HostOutputs, UT_FEATURE_DIM,
                                        UT_NUM_ACTIONS, UT_N_STATS)

ROOT = pathlib.Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "_build" / "libut_oracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libutrack_ref.so"


def _load(path):
    if not path.exists():
        raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
    return C.CDLL(str(path))


_oracle_lib = None
_ref_lib = None


def oracle_lib():
    global _oracle_lib
    if _oracle_lib is None:
        lib = _load(ORACLE_SO)
        P, I64, U64 = C.c_void_p, C.c_int64, C.c_uint64
        cfgp = C.POINTER(EnvConfigC)
        lib.uto_config_default.argtypes = [cfgp]
        lib.uto_config_finalize.argtypes = [cfgp]
        lib.uto_create.argtypes = [cfgp, I64, U64, I64, C.POINTER(P)]
        lib.uto_destroy.argtypes = [P]
        lib.uto_destroy.restype = None
        lib.uto_reset_all.argtypes = [P]
        lib.uto_step.argtypes = [P, P]
        lib.uto_step_policy.argtypes = [P, C.c_int, C.c_int]
        lib.uto_refresh_outputs.argtypes = [P]
        lib.uto_copy_outputs.argtypes = [P, C.POINTER(HostOutputs)]
        lib.uto_serialize.argtypes = [P, I64, C.POINTER(C.c_double), C.c_size_t, C.POINTER(C.c_size_t)]
        lib.uto_deserialize.argtypes = [P, I64, C.POINTER(C.c_double), C.c_size_t]
        lib.uto_stats.argtypes = [P, C.POINTER(C.c_double)]
        lib.uto_last_error.restype = C.c_char_p
        lib.uto_philox_block.argtypes = [U64, U64, U64, C.POINTER(C.c_uint32)]
        lib.uto_philox_block.restype = None
        lib.uto_derive_key.argtypes = [U64, U64, U64, U64]
        lib.uto_derive_key.restype = U64
        for f in ("uto_cr_logf", "uto_cr_cosf", "uto_cr_sinf"):
            getattr(lib, f).argtypes = [C.c_float]
            getattr(lib, f).restype = C.c_float
        lib.uto_fill_normals.argtypes = [U64, U64, U64, I64, C.POINTER(C.c_float)]
        lib.uto_fill_normals.restype = None
        lib.uto_eval_acc.argtypes = [P, I64, C.POINTER(C.c_double)]
        lib.uto_cr_grid.argtypes = [C.c_int, C.c_void_p]
        lib.uto_cr_grid.restype = None
        _oracle_lib = lib
    return _oracle_lib


def ref_available():
    return REF_SO.exists()


def ref_lib():
    global _ref_lib
    if _ref_lib is None:
        lib = _load(REF_SO)
        P, I32, I64, U64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
        cfgp = C.POINTER(EnvConfigC)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_config_finalize.argtypes = [cfgp]
        lib.ref_vecenv_create.argtypes = [cfgp, I64, U64, C.c_int, C.POINTER(P)]
        lib.ref_vecenv_destroy.argtypes = [P]
        lib.ref_vecenv_destroy.restype = None
        lib.ref_vecenv_reset_all.argtypes = [P]
        lib.ref_vecenv_step.argtypes = [P, P]
        lib.ref_vecenv_step_policy.argtypes = [P, C.c_int, C.c_int]
        lib.ref_vecenv_refresh_outputs.argtypes = [P]
        lib.ref_vecenv_copy_outputs.argtypes = [P, C.POINTER(HostOutputs)]
        lib.ref_env_serialize.argtypes = [P, I64, C.POINTER(C.c_double), C.c_size_t, C.POINTER(C.c_size_t)]
        lib.ref_env_deserialize.argtypes = [P, I64, C.POINTER(C.c_double), C.c_size_t]
        lib.ref_benchmark_sps.argtypes = [cfgp, I64, I32, C.c_int, U64, I32, I32,
                                          C.POINTER(C.c_double), C.POINTER(C.c_double),
                                          C.POINTER(I32), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        lib.ref_philox_block.argtypes = [U64, U64, U64, C.POINTER(C.c_uint32)]
        lib.ref_philox_block.restype = None
        lib.ref_derive_key.argtypes = [U64, U64, U64, U64]
        lib.ref_derive_key.restype = U64
        lib.ref_env_create.argtypes = [cfgp, U64, I64, C.POINTER(P)]
        lib.ref_env_destroy.argtypes = [P]
        lib.ref_env_destroy.restype = None
        lib.ref_env_reset.argtypes = [P]
        lib.ref_env_step.argtypes = [P, P, C.POINTER(C.c_double), C.POINTER(I32), C.POINTER(I32)]
        lib.ref_env_serialize_one.argtypes = [P, C.POINTER(C.c_double), C.c_size_t, C.POINTER(C.c_size_t)]
        lib.ref_env_observation.argtypes = [P, I32, C.POINTER(C.c_double)]
        _ref_lib = lib
    return _ref_lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def blob_len(A, T, P):
    """env.cpp:550-593 blob length."""
    return 5 + 6 * A + 9 * T + A * (6 * A + T * (9 + 5 * P))


def alloc_outputs(n_envs, A, T):
    R = A + T
    arrs = {
        "obs": np.zeros((UT_FEATURE_DIM, n_envs * A * R), np.float64),
        "final_obs": np.zeros((UT_FEATURE_DIM, n_envs * A * R), np.float64),
        "global_state": np.zeros((UT_FEATURE_DIM, n_envs * R), np.float64),
        "rewards": np.zeros(n_envs, np.float64),
        "dones": np.zeros(n_envs, np.uint8),
        "masks": np.zeros(n_envs * A * UT_NUM_ACTIONS, np.uint8),
        "tracking_error": np.zeros(n_envs * T, np.float64),
        "min_agent_dist": np.zeros(n_envs * T, np.float64),
        "target_lost": np.zeros(n_envs * T, np.uint8),
        "collision": np.zeros(n_envs, np.uint8),
        "step": np.zeros(n_envs, np.int32),
    }
    ho = HostOutputs(**{k: v.ctypes.data for k, v in arrs.items()})
    return arrs, ho


class _Base:
    """Shared VecEnv-like surface for the two CPU implementations."""

    def __init__(self, cfg, n_envs):
        self.cfg = cfg
        self.n_envs = n_envs
        self.A, self.T, self.P = cfg.n_agents, cfg.n_targets, cfg.pf.n_particles

    def outputs(self):
        arrs, ho = alloc_outputs(self.n_envs, self.A, self.T)
        self._check(self._copy(C.byref(ho)))
        return arrs

    def serialize(self, env):
        n = blob_len(self.A, self.T, self.P)
        buf = np.zeros(n, np.float64)
        ln = C.c_size_t()
        self._check(self._ser(env, buf.ctypes.data_as(C.POINTER(C.c_double)), n, C.byref(ln)))
        assert ln.value == n
        return buf

    def deserialize(self, env, blob):
        blob = np.ascontiguousarray(blob, np.float64)
        self._check(self._deser(env, blob.ctypes.data_as(C.POINTER(C.c_double)), blob.size))

    def step(self, actions):
        a = np.ascontiguousarray(actions, np.int32)
        self._check(self._step(a.ctypes.data))


class Oracle(_Base):
    """The plain-C restatement (oracle/ut_oracle.c)."""

    def __init__(self, cfg, n_envs, seed, env_index_offset=0):
        super().__init__(cfg, n_envs)
        self.lib = oracle_lib()
        h = C.c_void_p()
        self._check(self.lib.uto_create(C.byref(cfg), n_envs, seed, env_index_offset, C.byref(h)))
        self.h = h

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.uto_last_error().decode())

    def _copy(self, ho):
        return self.lib.uto_copy_outputs(self.h, ho)

    def _ser(self, *a):
        return self.lib.uto_serialize(self.h, *a)

    def _deser(self, *a):
        return self.lib.uto_deserialize(self.h, *a)

    def _step(self, ptr):
        return self.lib.uto_step(self.h, ptr)

    def step_policy(self, n_steps=1):
        self._check(self.lib.uto_step_policy(self.h, 0, n_steps))

    def reset_all(self):
        self._check(self.lib.uto_reset_all(self.h))

    def refresh_outputs(self):
        self._check(self.lib.uto_refresh_outputs(self.h))

    def stats(self):
        out = (C.c_double * UT_N_STATS)()
        self._check(self.lib.uto_stats(self.h, out))
        return np.array(out[:])

    def eval_acc(self, env):
        out = (C.c_double * 3)()
        self._check(self.lib.uto_eval_acc(self.h, env, out))
        return tuple(out)

    def close(self):
        if getattr(self, "h", None):
            self.lib.uto_destroy(self.h)
            self.h = None

    __del__ = close


class RefVecEnv(_Base):
    """The reference's own utrack::VecEnv (oracle/_ref)."""

    def __init__(self, cfg, n_envs, seed, workers=1):
        super().__init__(cfg, n_envs)
        self.lib = ref_lib()
        h = C.c_void_p()
        self._check(self.lib.ref_vecenv_create(C.byref(cfg), n_envs, seed, workers, C.byref(h)))
        self.h = h

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def _copy(self, ho):
        return self.lib.ref_vecenv_copy_outputs(self.h, ho)

    def _ser(self, *a):
        return self.lib.ref_env_serialize(self.h, *a)

    def _deser(self, *a):
        return self.lib.ref_env_deserialize(self.h, *a)

    def _step(self, ptr):
        return self.lib.ref_vecenv_step(self.h, ptr)

    def step_policy(self, n_steps=1):
        self._check(self.lib.ref_vecenv_step_policy(self.h, 0, n_steps))

    def reset_all(self):
        self._check(self.lib.ref_vecenv_reset_all(self.h))

    def refresh_outputs(self):
        self._check(self.lib.ref_vecenv_refresh_outputs(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.ref_vecenv_destroy(self.h)
            self.h = None

    __del__ = close


class RefEnvironment:
    """The reference's own single utrack::Environment (oracle/_ref): no
    auto-reset (env.cpp:234-504)."""

    def __init__(self, cfg, seed, env_index=0):
        self.lib = ref_lib()
        self.A, self.T, self.P = cfg.n_agents, cfg.n_targets, cfg.pf.n_particles
        h = C.c_void_p()
        self._check(self.lib.ref_env_create(C.byref(cfg), seed, env_index, C.byref(h)))
        self.h = h

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def step(self, actions):
        a = np.ascontiguousarray(actions, np.int32)
        r, d, c = C.c_double(), C.c_int32(), C.c_int32()
        self._check(self.lib.ref_env_step(self.h, a.ctypes.data, C.byref(r), C.byref(d), C.byref(c)))
        return {"reward": r.value, "done": bool(d.value), "collision": bool(c.value)}

    def reset(self):
        self._check(self.lib.ref_env_reset(self.h))

    def serialize(self):
        n = blob_len(self.A, self.T, self.P)
        buf = np.zeros(n, np.float64)
        ln = C.c_size_t()
        self._check(self.lib.ref_env_serialize_one(self.h, buf.ctypes.data_as(C.POINTER(C.c_double)), n,
                                                   C.byref(ln)))
        return buf

    def observation(self, agent):
        out = np.zeros((self.A + self.T, UT_FEATURE_DIM), np.float64)
        self._check(self.lib.ref_env_observation(self.h, agent, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def close(self):
        if getattr(self, "h", None):
            self.lib.ref_env_destroy(self.h)
            self.h = None

    __del__ = close


def default_config(**kw):
    """EnvConfig defaults (env_config.hpp:44-80) with keyword overrides; pf.* via pf_<name>."""
    cfg = EnvConfigC()
    oracle_lib().uto_config_default(C.byref(cfg))
    for k, v in kw.items():
        if k.startswith("pf_"):
            setattr(cfg.pf, k[3:], v)
        else:
            setattr(cfg, k, v)
    return cfg


def random_legal_actions(masks, rng):
    """Uniform legal action per agent from the batch masks (test_vecenv.cpp:15-27 style)."""
    m = masks.reshape(-1, UT_NUM_ACTIONS).astype(bool)
    out = np.empty(m.shape[0], np.int32)
    for i in range(m.shape[0]):
        legal = np.flatnonzero(m[i])
        out[i] = legal[rng.integers(len(legal))]
    return out


def oracle_build_present():
    return ORACLE_SO.exists()


def env_cpu_count():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
