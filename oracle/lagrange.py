"""Uniform grids and tensor-product Lagrange stencils, restated from
/root/reference/pkg/src/perisum/grids.py (test infrastructure only)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .lattice_sums import SeriesError


@dataclass(frozen=True)
class Grid:
    dims: tuple
    origin: tuple
    spacing: tuple

    @property
    def size(self) -> int:
        return int(np.prod(self.dims))


def near_grid(D, dims) -> Grid:
    """Coinciding grid on [0, D_a], spacing D_a/(n_a-1); grids.py:90-107."""
    spc = []
    for a in range(3):
        if D[a] <= 0.0 or dims[a] == 1:
            if D[a] > 0.0:
                raise ValueError(f"near grid needs >= 2 points on active axis {a}")
            spc.append(0.0)
        else:
            spc.append(D[a] / (dims[a] - 1))
    return Grid(tuple(int(d) if D[a] > 0.0 else 1 for a, d in enumerate(dims)),
                (0.0, 0.0, 0.0), tuple(spc))


def far_grids(D, dims):
    """Shifted source/observer pair, spacing D/n, observer origin +spacing/2;
    grids.py:58-87."""
    sd, so, ss, oo = [], [], [], []
    for a in range(3):
        if D[a] <= 0.0:
            sd.append(1), so.append(0.0), ss.append(0.0), oo.append(0.0)
            continue
        if dims[a] < 2:
            raise ValueError(f"far grid needs >= 2 points on active axis {a}")
        h = D[a] / dims[a]
        sd.append(int(dims[a])), so.append(0.0), ss.append(h), oo.append(h / 2.0)
    return Grid(tuple(sd), tuple(so), tuple(ss)), Grid(tuple(sd), tuple(oo), tuple(ss))


def axis_stencil(x, n, origin, h, order, margin):
    """starts (P,) and Lagrange weights (P, order+1) along one axis;
    grids.py:110-140 (start = rint(t - q/2) clipped to [0, n-1-q])."""
    p = x.shape[0]
    if n == 1:
        return np.zeros(p, dtype=np.int64), np.ones((p, 1))
    if order + 1 > n:
        raise ValueError(f"order {order} needs {order + 1} planes, grid has {n}")
    t = (x - origin) / h
    slack = margin / h + 1e-9
    if np.any(t < -slack) or np.any(t > n - 1 + slack):
        raise SeriesError("domain", "point outside grid hull")
    start = np.clip(np.rint(t - order / 2.0).astype(np.int64), 0, n - 1 - order)
    rel = t - start
    nodes = np.arange(order + 1, dtype=float)
    w = np.empty((p, order + 1))
    for j in range(order + 1):
        num = np.ones(p)
        for i in range(order + 1):
            if i != j:
                num = num * (rel - nodes[i])
        w[:, j] = num / np.prod(j - nodes[nodes != j])
    return start, w


@dataclass(frozen=True)
class Stencil:
    """Per-point axis starts/weights and the flattened (index, weight) form;
    grids.py:143-217.  The same data projects (W^T q) and interpolates (W u)."""
    grid: Grid
    starts: np.ndarray          # (P, 3) int64
    axis_w: tuple               # 3 x (P, q_a+1)
    flat_index: np.ndarray      # (P, S) int32, C order x*ny*nz + y*nz + z
    flat_weight: np.ndarray     # (P, S)

    def project(self, values):
        # grids.py:167-181: bincount scatter of w*q (real and imaginary separately)
        v = np.asarray(values)
        contrib = (self.flat_weight * v[:, None]).ravel()
        idx = self.flat_index.ravel()
        n = self.grid.size
        if np.iscomplexobj(contrib):
            return (np.bincount(idx, weights=contrib.real, minlength=n)
                    + 1j * np.bincount(idx, weights=contrib.imag, minlength=n))
        return np.bincount(idx, weights=contrib, minlength=n)

    def interpolate(self, grid_values):
        # grids.py:183-188: u = W u_g
        g = np.asarray(grid_values).ravel()
        return np.einsum("ps,ps->p", self.flat_weight, g[self.flat_index])


def make_stencil(grid: Grid, pts, order, margins) -> Stencil:
    """grids.py:191-217."""
    pts = np.atleast_2d(np.asarray(pts, dtype=float))
    p = pts.shape[0]
    starts = np.empty((p, 3), dtype=np.int64)
    ws = []
    for a in range(3):
        s, w = axis_stencil(pts[:, a], grid.dims[a], grid.origin[a], grid.spacing[a], order, margins[a])
        starts[:, a] = s
        ws.append(w)
    ny, nz = grid.dims[1], grid.dims[2]
    ix = starts[:, 0, None] + np.arange(ws[0].shape[1])
    iy = starts[:, 1, None] + np.arange(ws[1].shape[1])
    iz = starts[:, 2, None] + np.arange(ws[2].shape[1])
    flat = (ix[:, :, None, None] * (ny * nz) + iy[:, None, :, None] * nz + iz[:, None, None, :]).astype(np.int32)
    w3 = ws[0][:, :, None, None] * ws[1][:, None, :, None] * ws[2][:, None, None, :]
    return Stencil(grid, starts, tuple(ws), flat.reshape(p, -1), w3.reshape(p, -1))
