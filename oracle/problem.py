"""Plain problem description for the oracle (test infrastructure only).

The oracle deliberately does not import the product package: it takes one flat
record with the same meaning as the reference's PeriodicityConfig / TargetBox /
SolverParams triple (/root/reference/pkg/src/perisum/model.py:42-76, 80-88,
166-190).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

REGIMES = ("dynamic", "static-shifted", "npsp")


class Regime:
    DYNAMIC = "dynamic"
    STATIC_SHIFTED = "static-shifted"
    NPSP = "npsp"


@dataclass(frozen=True)
class Problem:
    dim: int                                  # number of periodic axes (x; x,y; x,y,z)
    L: tuple                                  # lattice periods
    D: tuple                                  # target box extent
    k0: complex = 0j
    kshift: tuple = (0j, 0j, 0j)
    regime: str = Regime.NPSP
    i_d: int = 1
    near_order: int = 2
    near_grid: tuple | None = None
    far_order: int = 3
    far_grid: tuple = (10, 10, 10)
    series_tol: float = 1e-10
    er_range_boxes: int = 1
    extras: dict = field(default_factory=dict, compare=False)

    @property
    def periodic(self) -> tuple:
        return tuple(range(self.dim))

    def near_dims(self, n_points: int) -> tuple:
        """Resolved near grid; SolverParams.resolve_near_grid model.py:187-190 and
        auto_near_dims model.py:146-162 (>= 1.15 N nodes, odd count per active axis)."""
        if self.near_grid is not None:
            dims = tuple(int(v) for v in self.near_grid)
        else:
            act = [a for a in range(3) if self.D[a] > 0.0]
            side = max(2, math.ceil((1.15 * max(int(n_points), 1)) ** (1.0 / len(act))))
            side += 1 - side % 2
            dims = tuple(side if a in act else 1 for a in range(3))
        # nearzone.py:198-199: zero-extent axes collapse to one plane
        return tuple(dims[a] if self.D[a] > 0.0 else 1 for a in range(3))


def make_problem(dim, L=(1.0, 1.0, 1.0), D=None, k0=0j, kshift=(0j, 0j, 0j), regime=None,
                 **params) -> Problem:
    """Regime inference as the reference's tests do it (tests/conftest.py:8-17)."""
    if regime is None:
        nophase = k0 == 0 and all(k == 0 for k in kshift)
        regime = Regime.NPSP if nophase else (Regime.STATIC_SHIFTED if k0 == 0 else Regime.DYNAMIC)
    L = tuple(float(v) for v in L)
    D = L if D is None else tuple(float(v) for v in D)
    return Problem(dim=int(dim), L=L, D=D, k0=complex(k0),
                   kshift=tuple(complex(k) for k in kshift), regime=regime, **params)
