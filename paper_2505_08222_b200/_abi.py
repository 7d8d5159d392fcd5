"""ctypes mirror of include/ut_env.h (the C-ABI drop-in boundary).

Field order and types must match the header exactly; tests/test_abi.py checks the
sizes against the compiled library.
"""
import ctypes as C

UT_OK, UT_ERR_CONTRACT, UT_ERR_CONFIG, UT_ERR_DATA, UT_ERR_RUNTIME = 0, 1, 2, 3, 4
UT_NUM_ACTIONS = 5
UT_TRAJ_FIELDS = 12
UT_FEATURE_DIM = 12
UT_REWARD_TRACKING, UT_REWARD_FOLLOW = 0, 1
UT_POLICY_RANDOM, UT_POLICY_SCRIPTED = 0, 1
UT_HEADING_DEFAULT, UT_HEADING_BUCKET = 0, 1
UT_STREAM_LEGACY = 1  # cudaStreamLegacy
UT_MULTI_STATS_AUTO, UT_MULTI_STATS_NCCL, UT_MULTI_STATS_HOST = 0, 1, 2
# UT_PHASE_* (ut_env.h): the reference's seven StepPhase values, then the auto-reset
PHASE_NAMES = ("targets", "agents", "measure", "filter", "comms", "observe", "reward", "reset")
UT_N_PHASES = len(PHASE_NAMES)

STAT_NAMES = (
    "env_steps", "reward_sum", "track_err_sum", "episodes_done", "episode_return_sum",
    "collision_steps", "lost_target_steps", "pf_updates", "pf_resamples", "pf_exact_path",
    "eval_dist_sum", "eval_dist_sq", "eval_err_sum", "eval_err_sq", "eval_collided_episodes",
    "eval_lost_episodes",
)
UT_ABI_VERSION = 4
UT_N_STATS = len(STAT_NAMES)


class PfConfig(C.Structure):
    """PfConfig (env_config.hpp:36-42)."""
    _fields_ = [
        ("n_particles", C.c_int32), ("_pad0", C.c_int32),
        ("process_noise_pos", C.c_double), ("process_noise_vel", C.c_double),
        ("speed_margin", C.c_double), ("init_radius", C.c_double),
    ]


class EnvConfigC(C.Structure):
    """EnvConfig (env_config.hpp:44-93) as the ABI POD."""
    _fields_ = [
        ("n_agents", C.c_int32), ("n_targets", C.c_int32), ("horizon", C.c_int32),
        ("reward_mode", C.c_int32),
        ("dt", C.c_double),
        ("agent_speed", C.c_double), ("target_speed_frac", C.c_double),
        ("target_speed_frac_max", C.c_double), ("target_turn_interval", C.c_double),
        ("detection_range", C.c_double), ("comm_range", C.c_double),
        ("comm_drop_prob", C.c_double), ("range_noise_std", C.c_double),
        ("eps_min", C.c_double), ("eps_max", C.c_double), ("d_min", C.c_double),
        ("d_safe", C.c_double),
        ("spawn_min_sep", C.c_double), ("spawn_max_sep", C.c_double),
        ("perturbation_std", C.c_double),
        ("target_depth_min", C.c_double), ("target_depth_max", C.c_double),
        ("lost_steps", C.c_int32), ("heading_model_kind", C.c_int32),
        ("heading_a", C.c_double), ("heading_b", C.c_double), ("heading_noise_std", C.c_double),
        ("pf", PfConfig),
        ("max_turn_per_step", C.c_double),
    ]


class Buffers(C.Structure):
    _fields_ = [
        ("n_envs", C.c_int64),
        ("n_agents", C.c_int32), ("n_targets", C.c_int32), ("n_rows", C.c_int32),
        ("n_particles", C.c_int32),
        ("obs_rows", C.c_int64), ("global_rows", C.c_int64),
        ("obs", C.c_void_p), ("final_obs", C.c_void_p), ("global_state", C.c_void_p),
        ("rewards", C.c_void_p), ("dones", C.c_void_p), ("masks", C.c_void_p),
        ("tracking_error", C.c_void_p), ("min_agent_dist", C.c_void_p),
        ("target_lost", C.c_void_p), ("collision", C.c_void_p), ("step", C.c_void_p),
        ("actions", C.c_void_p),
        ("px", C.c_void_p), ("py", C.c_void_p), ("vx", C.c_void_p), ("vy", C.c_void_p),
        ("w", C.c_void_p),
        ("total_sets", C.c_int64), ("set_offset", C.c_void_p),
    ]


class HostOutputs(C.Structure):
    _fields_ = [
        ("obs", C.c_void_p), ("final_obs", C.c_void_p), ("global_state", C.c_void_p),
        ("rewards", C.c_void_p), ("dones", C.c_void_p), ("masks", C.c_void_p),
        ("tracking_error", C.c_void_p), ("min_agent_dist", C.c_void_p),
        ("target_lost", C.c_void_p), ("collision", C.c_void_p), ("step", C.c_void_p),
    ]


class BenchmarkReport(C.Structure):
    _fields_ = [
        ("n_envs", C.c_int64), ("n_agents", C.c_int32), ("n_targets", C.c_int32),
        ("timed_steps", C.c_int32), ("_pad0", C.c_int32),
        ("wall_seconds", C.c_double), ("sps", C.c_double), ("agent_sps", C.c_double),
        ("phase_ns", C.c_uint64 * UT_N_PHASES), ("total_ns", C.c_uint64),
    ]


HOST_OUTPUT_FIELDS = tuple(name for name, _ in HostOutputs._fields_)


def declare_product(lib):
    """Attach argtypes/restype for every entry point declared in ut_env.h."""
    P, I32, I64, U64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
    cfgp = C.POINTER(EnvConfigC)
    sig = {
        "ut_config_default": (None, [cfgp]),
        "ut_config_finalize": (C.c_int, [cfgp]),
        "ut_vecenv_create": (C.c_int, [cfgp, I64, U64, I64, C.c_int, C.POINTER(P)]),
        "ut_vecenv_create_mixed": (C.c_int, [cfgp, I32, C.POINTER(I32), I64, U64, I64, C.c_int,
                                             C.POINTER(P)]),
        "ut_vecenv_destroy": (None, [P]),
        "ut_vecenv_reset_all": (C.c_int, [P]),
        "ut_vecenv_step": (C.c_int, [P, P, C.c_int]),
        "ut_vecenv_step_policy": (C.c_int, [P, C.c_int, C.c_int]),
        "ut_vecenv_refresh_outputs": (C.c_int, [P]),
        "ut_vecenv_buffers": (C.c_int, [P, C.POINTER(Buffers)]),
        "ut_vecenv_copy_outputs": (C.c_int, [P, C.POINTER(HostOutputs)]),
        "ut_vecenv_set_stream": (C.c_int, [P, P]),
        "ut_vecenv_wait_stream": (C.c_int, [P, P]),
        "ut_vecenv_set_auto_reset": (C.c_int, [P, C.c_int]),
        "ut_vecenv_phase_ns": (C.c_int, [P, C.POINTER(C.c_uint64), C.c_int]),
        "ut_vecenv_set_output_buffers": (C.c_int, [P, C.c_int]),
        "ut_vecenv_capture_trajectory": (C.c_int, [P, I64, I64]),
        "ut_vecenv_trajectory_rows": (C.c_int, [P, C.POINTER(C.c_double), C.c_size_t, C.POINTER(C.c_size_t)]),
        "ut_vecenv_copy_outputs_async": (C.c_int, [P, C.POINTER(HostOutputs), P]),
        "ut_vecenv_synchronize": (C.c_int, [P]),
        "ut_vecenv_stats": (C.c_int, [P, C.POINTER(C.c_double), C.c_int]),
        "ut_vecenv_launch_count": (I64, [P]),
        "ut_env_serialize": (C.c_int, [P, I64, C.POINTER(C.c_double), C.c_size_t,
                                       C.POINTER(C.c_size_t)]),
        "ut_env_deserialize": (C.c_int, [P, I64, C.POINTER(C.c_double), C.c_size_t]),
        "ut_env_world_step": (C.c_int, [P, I64, C.POINTER(I32)]),
        "ut_vecenv_export_state": (C.c_int, [P, I64, I64, C.POINTER(C.c_double), C.c_size_t,
                                             C.POINTER(C.c_size_t)]),
        "ut_vecenv_import_state": (C.c_int, [P, I64, I64, C.POINTER(C.c_double), C.c_size_t]),
        "ut_benchmark_sps": (C.c_int, [cfgp, I64, I32, C.c_int, U64, I32, C.c_int,
                                       C.POINTER(BenchmarkReport)]),
        "ut_vecenv_enable_phase_timing": (C.c_int, [P, C.c_int]),
        "ut_vecenv_phase_cycles": (C.c_int, [P, C.POINTER(C.c_uint64), C.c_int]),
        "ut_multienv_create": (C.c_int, [cfgp, I64, U64, C.POINTER(I32), I32, I32, C.POINTER(P)]),
        "ut_multienv_destroy": (None, [P]),
        "ut_multienv_n_shards": (C.c_int, [P]),
        "ut_multienv_stats_backend": (C.c_int, [P]),
        "ut_multienv_shard": (C.c_int, [P, I32, C.POINTER(P), C.POINTER(I64), C.POINTER(I64), C.POINTER(I32)]),
        "ut_multienv_locate": (C.c_int, [P, I64, C.POINTER(P), C.POINTER(I64)]),
        "ut_multienv_reset_all": (C.c_int, [P]),
        "ut_multienv_step": (C.c_int, [P, P]),
        "ut_multienv_step_policy": (C.c_int, [P, C.c_int, C.c_int]),
        "ut_multienv_refresh_outputs": (C.c_int, [P]),
        "ut_multienv_set_auto_reset": (C.c_int, [P, C.c_int]),
        "ut_multienv_synchronize": (C.c_int, [P]),
        "ut_multienv_copy_outputs": (C.c_int, [P, C.POINTER(HostOutputs)]),
        "ut_multienv_stats": (C.c_int, [P, C.POINTER(C.c_double), C.c_int]),
        "ut_multienv_enable_phase_timing": (C.c_int, [P, C.c_int]),
        "ut_multienv_phase_ns": (C.c_int, [P, C.POINTER(C.c_uint64), C.c_int]),
        "ut_multienv_launch_count": (I64, [P]),
        "ut_multienv_serialize": (C.c_int, [P, I64, C.POINTER(C.c_double), C.c_size_t, C.POINTER(C.c_size_t)]),
        "ut_multienv_deserialize": (C.c_int, [P, I64, C.POINTER(C.c_double), C.c_size_t]),
        "ut_multienv_world_step": (C.c_int, [P, I64, C.POINTER(I32)]),
        "ut_nccl_version": (C.c_int, [C.POINTER(C.c_int)]),
        "ut_last_error": (C.c_char_p, []),
        "ut_abi_version": (C.c_int, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def declare_debug(lib):
    """Signatures of include/ut_debug.h."""
    lib.ut_debug_cr_grid.argtypes = [C.c_int, C.c_int, C.c_void_p]
    lib.ut_debug_cr_grid.restype = C.c_int
    lib.ut_debug_philox.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32, C.c_int, C.c_void_p]
    lib.ut_debug_philox.restype = C.c_int
    lib.ut_debug_derive_key.argtypes = [C.c_uint64] * 4 + [C.c_int, C.POINTER(C.c_uint64)]
    lib.ut_debug_derive_key.restype = C.c_int
    lib.ut_debug_fp64_peak.argtypes = [C.c_int, C.POINTER(C.c_double)]
    lib.ut_debug_fp64_peak.restype = C.c_int
    lib.ut_debug_cta_cycles.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.c_int64, C.POINTER(C.c_int64)]
    lib.ut_debug_cta_cycles.restype = C.c_int
    lib.ut_debug_abi_sizes.argtypes = [C.POINTER(C.c_int64)]
    lib.ut_debug_abi_sizes.restype = C.c_int
    lib.ut_debug_ieee_check.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_int, C.POINTER(C.c_uint64)]
    lib.ut_debug_ieee_check.restype = C.c_int
    lib.ut_debug_set_knobs.argtypes = [C.c_void_p, C.c_int, C.c_int64]
    lib.ut_debug_set_knobs.restype = C.c_int
    lib.ut_debug_set_grid.argtypes = [C.c_void_p, C.c_int32]
    lib.ut_debug_set_grid.restype = C.c_int
    lib.ut_debug_instance.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    lib.ut_debug_instance.restype = C.c_int
    return lib


PRODUCT_SYMBOLS = (
    "ut_config_default", "ut_config_finalize", "ut_vecenv_create", "ut_vecenv_create_mixed",
    "ut_vecenv_destroy", "ut_vecenv_reset_all", "ut_vecenv_step", "ut_vecenv_step_policy",
    "ut_vecenv_refresh_outputs", "ut_vecenv_buffers", "ut_vecenv_copy_outputs",
    "ut_vecenv_set_stream", "ut_vecenv_synchronize", "ut_vecenv_stats", "ut_vecenv_launch_count",
    "ut_env_serialize", "ut_env_deserialize", "ut_env_world_step", "ut_benchmark_sps",
    "ut_vecenv_export_state", "ut_vecenv_import_state", "ut_vecenv_set_output_buffers",
    "ut_vecenv_copy_outputs_async", "ut_vecenv_capture_trajectory", "ut_vecenv_trajectory_rows",
    "ut_vecenv_enable_phase_timing", "ut_vecenv_phase_cycles", "ut_vecenv_phase_ns",
    "ut_vecenv_wait_stream", "ut_vecenv_set_auto_reset",
    "ut_multienv_create", "ut_multienv_destroy", "ut_multienv_n_shards", "ut_multienv_stats_backend",
    "ut_multienv_shard", "ut_multienv_locate", "ut_multienv_reset_all", "ut_multienv_step",
    "ut_multienv_step_policy", "ut_multienv_refresh_outputs", "ut_multienv_set_auto_reset",
    "ut_multienv_synchronize", "ut_multienv_copy_outputs", "ut_multienv_stats",
    "ut_multienv_enable_phase_timing", "ut_multienv_phase_ns", "ut_multienv_launch_count",
    "ut_multienv_serialize", "ut_multienv_deserialize", "ut_multienv_world_step", "ut_nccl_version",
    "ut_last_error", "ut_abi_version",
)
