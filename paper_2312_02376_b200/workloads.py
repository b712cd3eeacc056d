"""Seeded synthetic inputs for the five BASELINE.json configurations (C1..C5).

The reference quotes no dataset; every config is synthetic.
Seeds: `np.random.default_rng(c)` for config c.  Draw order: positions, then
the real part of q, then the imaginary part (C5: all real parts of the 64
excitations, then all imaginary parts).  Parameters not named by a config use
the SolverParams defaults of the reference (model.py:173-180): i_d=1, far grid
10^3, far order 3, series_tol 1e-10, er_range_boxes 1.  The config's grid is
`near_grid` and its interpolation order is `near_order`.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

PI = np.pi


@dataclass(frozen=True)
class Workload:
    name: str
    dim: int
    L: tuple
    D: tuple
    k0: complex
    kshift: tuple
    regime: str
    near_grid: tuple
    near_order: int
    n_points: int
    complex_q: bool
    excitations: int = 1
    extra: dict = field(default_factory=dict, compare=False)

    def params(self) -> dict:
        return dict(i_d=1, far_order=3, far_grid=(10, 10, 10), near_order=self.near_order,
                    near_grid=self.near_grid, series_tol=1e-10, er_range_boxes=1)


CONFIGS = {
    1: Workload("C1-3D-NPSP-N4096", 3, (1.0, 1.0, 1.0), (1.0, 1.0, 1.0), 0j, (0j, 0j, 0j),
                "npsp", (32, 32, 32), 3, 4096, False),
    2: Workload("C2-1D-Helmholtz-N65536", 1, (1.0, 1.0, 1.0), (1.0, 1.0, 1.0), complex(PI),
                (complex(0.3 * PI), 0j, 0j), "dynamic", (64, 64, 64), 3, 65536, True),
    3: Workload("C3-2D-NPSP-blobs-N1048576", 2, (1.0, 1.0, 1.0), (1.0, 1.0, 0.5), 0j,
                (0j, 0j, 0j), "npsp", (128, 128, 64), 4, 1048576, False),
    4: Workload("C4-3D-Helmholtz-N8388608", 3, (1.0, 1.0, 1.0), (1.0, 1.0, 1.0), complex(2 * PI),
                (complex(0.2 * PI), complex(0.1 * PI), 0j), "dynamic", (256, 256, 256), 4,
                8388608, True),
    5: Workload("C5-2D-Helmholtz-sweep-N2097152", 2, (1.0, 1.0, 1.0), (1.0, 1.0, 0.25),
                complex(1.5 * PI), (0j, 0j, 0j), "dynamic", (192, 192, 48), 3, 2097152, True,
                excitations=64),
}


def c5_kshift(e: int) -> tuple:
    """kx0_e = (e + 1/2) pi / 64: e*pi/64 hits an exact Wood anomaly at e = 32."""
    return (complex((e + 0.5) * PI / 64.0), 0j, 0j)


def positions(c: int, rng=None, n=None) -> np.ndarray:
    w = CONFIGS[c]
    rng = np.random.default_rng(c) if rng is None else rng
    n = w.n_points if n is None else n
    if c == 3:
        blobs = 64
        per = max(n // blobs, 1)
        centres = rng.uniform(0.0, 1.0, (blobs, 3)) * np.array([1.0, 1.0, 0.5])
        off = rng.normal(0.0, 0.02, (blobs, per, 3))
        p = (centres[:, None, :] + off).reshape(-1, 3)
        p[:, 0] = np.mod(p[:, 0], 1.0)
        p[:, 1] = np.mod(p[:, 1], 1.0)
        t = np.mod(p[:, 2], 1.0)
        p[:, 2] = np.where(t > 0.5, 1.0 - t, t)
        return np.ascontiguousarray(p)
    return np.ascontiguousarray(rng.uniform(0.0, 1.0, (n, 3)) * np.asarray(w.D))


def charges(c: int, n: int, rng) -> np.ndarray:
    w = CONFIGS[c]
    if w.excitations > 1:
        re = rng.standard_normal((w.excitations, n))
        im = rng.standard_normal((w.excitations, n))
        return re + 1j * im
    re = rng.standard_normal(n)
    if not w.complex_q:
        return (re - re.mean()).astype(complex)
    return re + 1j * rng.standard_normal(n)


def make_inputs(c: int, n=None):
    """(positions (N,3) f64, q (N,) or (E,N) complex128) for config c, seeded."""
    rng = np.random.default_rng(c)
    pos = positions(c, rng, n)
    return pos, charges(c, pos.shape[0], rng)
