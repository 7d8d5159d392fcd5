"""TEST INFRASTRUCTURE: field-aware comparison of Environment state blobs
(env.cpp:550-593 layout) and batch outputs, implementing SURVEY Appendix C:
integer state bit-exact, floating point within a stated relative tolerance."""
import numpy as np

# North-star bound for floating-point state per step (BASELINE.json north_star).
NORTH_STAR_RTOL = 1e-5
# What the implementation actually achieves per step (element-wise fp64 math is
# bit-identical; sums differ only in reduction order and libm ulps).
TIGHT_RTOL = 1e-9
TIGHT_ATOL = 1e-12


def blob_spec(A, T, P):
    """Per-slot (group name, is_integer) for the state blob."""
    names, ints = [], []

    def add(name, is_int, count=1):
        names.extend([name] * count)
        ints.extend([is_int] * count)

    add("step", True)
    add("episode_target_speed", False)
    add("env_rng_pos", True)
    add("env_rng_have_spare", True)
    add("env_rng_spare", False)
    for _ in range(A):
        for f in ("x", "y", "z", "heading", "speed"):
            add("agent." + f, False)
        add("agent.rudder", True)
    for _ in range(T):
        for f in ("x", "y", "z", "heading", "speed"):
            add("target." + f, False)
        add("target.rudder", True)
        add("target.countdown", True)
        add("target.cmd_heading", False)
    add("target.miss_streak", True, T)
    for _ in range(A):
        for _ in range(A):
            for f in ("x", "y", "z", "heading"):
                add("info." + f, False)
            add("info.age", True)
            add("info.valid", True)
        for _ in range(T):
            add("track.est_x", False)
            add("track.est_y", False)
            add("track.spread", False)
            add("track.age", True)
            add("track.ever", True)
            add("pf.rng_pos", True)
            add("pf.rng_have_spare", True)
            add("pf.rng_spare", False)
            add("pf.max_speed", False)
            for f in ("px", "py", "vx", "vy", "w"):
                add("pf." + f, False, P)
    return np.array(names), np.array(ints, bool)


# Relative comparison with a per-field absolute floor: |a - b| / max(|b|, floor).
# A floor is where a value stops being meaningful relative to its own
# magnitude: the rounding noise of the quantities it is computed from (machine
# epsilon x their magnitude) divided by the tight tolerance. Positions,
# estimates, spreads and distances are built from coordinates of up to ~1 km
# (noise ~1e-13 m), so below 1 mm (1e-3 m) they are held to 1e-12 m absolute and
# above it relatively. The spread is a root-mean-square over P particles of
# differences of such coordinates, so its noise is up to ~P eps |x| ~ 1e-10 m:
# floor 1 cm (a collapsed cloud has spread 0 on one side and ~1e-11 m of
# rounding noise on the other). Headings, speeds, velocities, rewards and
# normals (inputs of order 1) use 1e-6; the token columns scale metres by 1/1000
# (floor 1e-6) and the spread by 1/100 (1e-4); the particle weights (~1/P) use
# 1e-12 / P, so a weight of 1e-300 is held to 1e-21 absolute.
DEFAULT_FLOOR = 1e-6
METRE_FLOOR = 1e-3
SPREAD_FLOOR = 1e-2
METRE_GROUPS = ("agent.x", "agent.y", "agent.z", "target.x", "target.y", "target.z", "info.x", "info.y",
                "info.z", "track.est_x", "track.est_y", "pf.px", "pf.py")
OUTPUT_FLOORS = {"tracking_error": METRE_FLOOR, "min_agent_dist": METRE_FLOOR}
# obs / final_obs columns (env_config.hpp:15-34): dx dy dz sin cos speed self agent
# target valid age spread
OBS_COL_FLOORS = np.array([1e-6] * 11 + [SPREAD_FLOOR / 100])


def weight_floor(P):
    return 1e-12 / max(int(P), 1)


def blob_floors(names, P):
    """Per-slot floors for the float slots `names` of a state blob."""
    f = np.full(names.shape, DEFAULT_FLOOR)
    f[np.isin(names, METRE_GROUPS)] = METRE_FLOOR
    f[names == "track.spread"] = SPREAD_FLOOR
    f[names == "pf.w"] = weight_floor(P)
    return f


def rel_err(a, b, floor=DEFAULT_FLOOR):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    d = np.abs(a - b)
    scale = np.maximum(np.abs(b), floor)
    with np.errstate(invalid="ignore"):
        r = np.where(d == 0, 0.0, d / scale)
    return r


class Report:
    def __init__(self):
        self.int_mismatch = []
        self.max_rel = {}

    def ok(self, rtol):
        return not self.int_mismatch and all(v <= rtol for v in self.max_rel.values())

    def worst(self):
        return max(self.max_rel.values(), default=0.0)

    def __repr__(self):
        top = sorted(self.max_rel.items(), key=lambda kv: -kv[1])[:5]
        return f"Report(int_mismatch={self.int_mismatch[:5]}, worst={top})"


def compare_blobs(got, want, A, T, P, report=None, tag=""):
    names, ints = blob_spec(A, T, P)
    assert got.shape == want.shape == names.shape, (got.shape, want.shape, names.shape)
    rep = report or Report()
    bad = np.flatnonzero(ints & (got != want))
    for i in bad[:20]:
        rep.int_mismatch.append((tag, names[i], int(i), float(got[i]), float(want[i])))
    fl = ~ints
    r = rel_err(got[fl], want[fl], blob_floors(names[fl], P))
    for g in np.unique(names[fl]):
        m = names[fl] == g
        v = float(r[m].max()) if m.any() else 0.0
        rep.max_rel[g] = max(rep.max_rel.get(g, 0.0), v)
    return rep


def output_floor(name, arr):
    if name in ("obs", "final_obs"):
        return OBS_COL_FLOORS.reshape(12, 1) if np.ndim(arr) == 2 else DEFAULT_FLOOR
    return OUTPUT_FLOORS.get(name, DEFAULT_FLOOR)


INT_OUTPUTS = ("dones", "masks", "target_lost", "collision", "step")
FLOAT_OUTPUTS = ("obs", "global_state", "rewards", "tracking_error", "min_agent_dist", "final_obs")


def compare_outputs(got, want, report=None, tag="", skip=()):
    rep = report or Report()
    for k in INT_OUTPUTS:
        if k in got and k in want and k not in skip:
            if not np.array_equal(got[k], want[k]):
                idx = np.flatnonzero(got[k].ravel() != want[k].ravel())
                rep.int_mismatch.append((tag, k, idx[:5].tolist()))
    for k in FLOAT_OUTPUTS:
        if k in got and k in want and k not in skip:
            r = rel_err(got[k], want[k], output_floor(k, want[k]))
            rep.max_rel["out." + k] = max(rep.max_rel.get("out." + k, 0.0), float(r.max()) if r.size else 0.0)
    return rep
