"""Multi-process oracle plan build (test / baseline infrastructure only).

Same algorithm and output as pipeline.build_plan -- the correction-pair
discovery (nearzone.py:303-487) is split into ascending observer ranges that
run in forked worker processes and are concatenated in order, so the pair
lists are identical to the single-process build.  Used by `bench.py --impl
reference` to get the reference CPU plan of C2 built in well under a minute
on a many-core host; evaluation itself stays the reference's single-threaded
numpy path.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from . import near_engine as ne
from .far_engine import build_far
from .lagrange import make_stencil, near_grid
from .pipeline import OraclePlan
from .problem import Problem

_CTX = None


def _work(rng):
    return ne.discover_range(_CTX, rng[0], rng[1])


def build_plan_parallel(pb: Problem, src_pos, workers=None, chunk=2048) -> OraclePlan:
    global _CTX
    src_pos = np.ascontiguousarray(src_pos, dtype=float)
    obs_pos = src_pos
    t0 = time.perf_counter()
    dims = pb.near_dims(len(src_pos))
    grid = near_grid(pb.D, dims)
    h = grid.spacing
    nb = tuple(max(d - 1, 1) for d in dims)
    kdisp, coincident = ne.kernel_table(pb, grid)
    khat = np.fft.fftn(ne.embed(kdisp, dims))
    margin = tuple(1e-9 * max(h[a], 1.0) for a in range(3))
    sst = make_stencil(grid, src_pos, pb.near_order, margin)
    jr_full = ne.correction_radius(pb.er_range_boxes, pb.near_order)
    jr = ne.join_radius(pb, grid, nb, jr_full)
    _CTX = ne.discovery_context(pb, grid, nb, jr, jr_full, sst, sst, src_pos, obs_pos, kdisp,
                                np.arange(len(obs_pos)))
    n = len(obs_pos)
    ranges = [(lo, min(n, lo + chunk)) for lo in range(0, n, chunk)]
    workers = workers or os.cpu_count() or 1
    if workers > 1 and len(ranges) > 1:
        with mp.get_context("fork").Pool(min(workers, len(ranges))) as pool:
            parts = pool.map(_work, ranges, chunksize=1)
    else:
        parts = [_work(r) for r in ranges]
    _CTX = None
    pairs = ne.merge_ranges(parts, n)
    near = ne.NearPlan(pb, grid, sst, sst, kdisp, khat, nb, jr, jr_full, *pairs, coincident)
    far = build_far(pb, src_pos, obs_pos)
    return OraclePlan(near, far, time.perf_counter() - t0)
