"""Oracle facade: build both engines, evaluate u = u_near + u_far
(/root/reference/pkg/src/perisum/solver.py:18-45).  Test infrastructure only."""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .far_engine import FarPlan, build_far, eval_far
from .near_engine import NearPlan, build_near, eval_near
from .problem import Problem


@dataclass
class OraclePlan:
    near: NearPlan
    far: FarPlan
    build_seconds: float

    def evaluate(self, q):
        return eval_near(self.near, q) + eval_far(self.far, q)          # solver.py:24-25


def build_plan(pb: Problem, src_pos, obs_pos=None, obs_src=None) -> OraclePlan:
    """obs_pos None means observers = sources (same_points).  obs_src (index array)
    marks observers that are a subset of the sources -- the subset-observer oracle."""
    src_pos = np.ascontiguousarray(np.asarray(src_pos, dtype=float))
    if obs_pos is None:
        obs_pos = src_pos
    obs_pos = np.ascontiguousarray(np.asarray(obs_pos, dtype=float))
    t0 = time.perf_counter()
    near = build_near(pb, src_pos, obs_pos, obs_src=obs_src)
    far = build_far(pb, src_pos, obs_pos)
    return OraclePlan(near, far, time.perf_counter() - t0)
