"""Trajectory export (trajectory.cpp:13-93): rows captured on the device by
ut_vecenv_capture_trajectory, written in the reference's CSV layout
(kTrajectoryHeader, trajectory.hpp:23-24; numbers as ostream precision(10))."""
from __future__ import annotations

import os
from typing import Iterable, List

import numpy as np

from . import _abi

HEADER = "step,entity_id,kind,x,y,z,heading,est_x,est_y,track_err,reward,collision"
(TJ_STEP, TJ_X, TJ_Y, TJ_Z, TJ_HEAD, TJ_HAS_EST, TJ_EST_X, TJ_EST_Y, TJ_ERR, TJ_REWARD, TJ_COLLISION,
 TJ_IS_TARGET) = range(_abi.UT_TRAJ_FIELDS)


def _fmt(v: float) -> str:
    return "%.10g" % v


def env_rows(block: np.ndarray) -> List[str]:
    """CSV lines of one env's captured step (block: rows x UT_TRAJ_FIELDS), in
    append_trajectory_rows order: agent_0.., target_0.."""
    lines, na, nt = [], 0, 0
    for r in block:
        if r[TJ_STEP] < 0:  # padding row of a smaller fleet
            continue
        tgt = r[TJ_IS_TARGET] != 0
        eid = f"target_{nt}" if tgt else f"agent_{na}"
        nt, na = (nt + 1, na) if tgt else (nt, na + 1)
        est_x = _fmt(r[TJ_EST_X]) if r[TJ_HAS_EST] else ""
        est_y = _fmt(r[TJ_EST_Y]) if r[TJ_HAS_EST] else ""
        err = _fmt(r[TJ_ERR]) if tgt and np.isfinite(r[TJ_ERR]) else ""
        lines.append(",".join([str(int(r[TJ_STEP])), eid, "target" if tgt else "agent", _fmt(r[TJ_X]),
                               _fmt(r[TJ_Y]), _fmt(r[TJ_Z]), _fmt(r[TJ_HEAD]), est_x, est_y, err,
                               _fmt(r[TJ_REWARD]), str(int(r[TJ_COLLISION]))]))
    return lines


def write_trajectory_csv(path: str, steps: Iterable[np.ndarray]):
    """write_trajectory_csv (trajectory.cpp:79-93) for one env: `steps` are its
    captured blocks, one per step."""
    parent = os.path.dirname(path)
    if parent:
        os.makedirs(parent, exist_ok=True)
    with open(path, "w") as f:
        f.write(HEADER + "\n")
        for block in steps:
            for line in env_rows(block):
                f.write(line + "\n")
