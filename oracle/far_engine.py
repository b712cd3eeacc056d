"""Far-zone engine restated from /root/reference/pkg/src/perisum/farzone.py
(test infrastructure only): shifted grids, difference-indexed series kernel
(farzone.py:62-131), evaluation project -> dense grid sum -> interpolate
(farzone.py:134-159)."""
from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

from .lagrange import Grid, Stencil, far_grids, make_stencil
from .lattice_sums import SeriesError, far_kernel
from .problem import Problem


@dataclass
class FarPlan:
    pb: Problem
    sgrid: Grid
    ogrid: Grid
    src: Stencil
    obs: Stencil
    kernel: np.ndarray          # (2n-1 or 1) per axis over grid difference vectors
    kernel_terms: int


def difference_points(sg: Grid, og: Grid):
    """(l_o - l_s) * h + (origin_o - origin_s) per axis, C-order mesh; farzone.py:62-73."""
    axes = []
    for a in range(3):
        n = sg.dims[a]
        shift = og.origin[a] - sg.origin[a]
        axes.append(np.array([shift]) if n == 1 else np.arange(-(n - 1), n) * sg.spacing[a] + shift)
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([m.ravel() for m in mesh], axis=1), tuple(len(x) for x in axes)


def build_far(pb: Problem, src_pos, obs_pos, kernel=None) -> FarPlan:
    """farzone.py:76-131 (build_far_plan, without the blob cache)."""
    if pb.i_d < 1:
        raise ValueError("far-zone engine requires i_d >= 1")
    dims = tuple(pb.far_grid[a] if pb.D[a] > 0.0 else 1 for a in range(3))
    sg, og = far_grids(pb.D, dims)
    if pb.dim == 1 and pb.D[1] == 0.0 and pb.D[2] == 0.0:
        # farzone.py:89-98: cloud on the periodic axis -> source grid moved by h/2 in y
        warnings.warn("source cloud lies exactly on the periodic axis; offsetting the "
                      "source grid transversely", stacklevel=2)
        sg = Grid(sg.dims, (sg.origin[0], sg.spacing[0] / 2.0, sg.origin[2]), sg.spacing)
    pts, shape = difference_points(sg, og)
    terms = 0
    if kernel is None:
        vals, t, conv = far_kernel(pts, pb)
        if not conv.all():
            i = int(np.argmin(conv))
            raise SeriesError("not_converged", f"far kernel series did not converge at {pts[i].tolist()}")
        kernel = vals.reshape(shape)
        terms = int(t.max())
    margins = tuple(sg.spacing[a] if sg.dims[a] > 1 else 0.0 for a in range(3))
    return FarPlan(pb, sg, og, make_stencil(sg, src_pos, pb.far_order, margins),
                   make_stencil(og, obs_pos, pb.far_order, margins), kernel, terms)


def grid_sum(kernel, qg):
    """ug[o] = sum_s K[o - s + (n-1)] qg[s] over all node pairs; farzone.py:134-158."""
    nx, ny, nz = qg.shape
    base = kernel[nx - 1 if nx > 1 else 0:, ny - 1 if ny > 1 else 0:, nz - 1 if nz > 1 else 0:]
    s0, s1, s2 = kernel.strides
    view = np.lib.stride_tricks.as_strided(base, shape=(nx, ny, nz, nx, ny, nz),
                                           strides=(s0, s1, s2, -s0, -s1, -s2), writeable=False)
    return np.einsum("abcdef,def->abc", view, qg)


def eval_far(plan: FarPlan, q):
    """farzone.py:150-159."""
    q = np.asarray(q, dtype=complex)
    if q.shape[0] != plan.src.starts.shape[0]:
        raise ValueError(f"expected {plan.src.starts.shape[0]} amplitudes, got {q.shape[0]}")
    qg = plan.src.project(q).reshape(plan.sgrid.dims)
    return plan.obs.interpolate(grid_sum(plan.kernel, qg).ravel())
