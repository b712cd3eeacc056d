"""Golden-case definitions shared by tests/golden/make_golden.py (which runs the
reference in the build container) and the tests that replay them.

Inputs are regenerated from the seed, so only outputs are stored in fixtures.
"""
from __future__ import annotations

import numpy as np

PI = np.pi

# name -> definition.  k0 / kshift are complex; params follow SolverParams names.
SMALL_CASES = {
    "p3_npsp": dict(dim=3, L=(1, 1, 1), D=(1, 1, 1), k0=0, kshift=(0, 0, 0), n=260,
                    params=dict(near_grid=(10, 10, 10), near_order=3, far_grid=(6, 6, 6))),
    "p1_dyn": dict(dim=1, L=(1, 1, 1), D=(1, 1, 1), k0=PI, kshift=(0.3 * PI, 0, 0), n=300,
                   params=dict(near_grid=(10, 10, 10), near_order=3, far_grid=(6, 6, 6))),
    "p2_dyn": dict(dim=2, L=(1, 1, 1), D=(1, 1, 0.5), k0=1.5 * PI, kshift=(0.2, 0, 0), n=240,
                   params=dict(near_grid=(10, 10, 6), near_order=3, far_grid=(6, 6, 6))),
    "p3_dyn": dict(dim=3, L=(1, 1, 1), D=(1, 1, 1), k0=2 * PI, kshift=(0.2 * PI, 0.1 * PI, 0), n=220,
                   params=dict(near_grid=(9, 9, 9), near_order=4, far_grid=(6, 6, 6))),
    "p2_npsp_o4": dict(dim=2, L=(1, 1, 1), D=(1, 1, 0.5), k0=0, kshift=(0, 0, 0), n=240,
                       params=dict(near_grid=(11, 11, 7), near_order=4, far_grid=(6, 6, 6))),
    "p1_npsp": dict(dim=1, L=(1, 1, 1), D=(1, 1, 1), k0=0, kshift=(0, 0, 0), n=200,
                    params=dict(near_grid=(9, 9, 9), near_order=2, far_grid=(5, 5, 5))),
    "p2_static_sep": dict(dim=2, L=(1, 1, 1), D=(1, 1, 0.5), k0=0, kshift=(0.5, 0.3, 0), n=200, m=90,
                          params=dict(near_grid=(9, 9, 6), near_order=3, far_grid=(6, 6, 6))),
    "p3_npsp_DltL_sep": dict(dim=3, L=(1, 1, 1), D=(0.9, 1, 1), k0=0, kshift=(0, 0, 0), n=180, m=70,
                             params=dict(near_grid=(9, 11, 10), near_order=2, far_grid=(6, 6, 6))),
    "p3_dyn_lossy_id2": dict(dim=3, L=(1.2, 1, 1.1), D=(1.2, 1, 1.1), k0=3 - 0.4j,
                             kshift=(0.3, -0.2, 0.1), n=150,
                             params=dict(near_grid=(10, 9, 9), near_order=2, far_grid=(5, 5, 5), i_d=2)),
    "p2_planar_npsp": dict(dim=2, L=(1, 1, 1), D=(1, 1, 0), k0=0, kshift=(0, 0, 0), n=200, z0=0.0,
                           params=dict(near_grid=(12, 12, 1), near_order=3, far_grid=(6, 6, 6))),
    "p1_axis_dyn": dict(dim=1, L=(1, 1, 1), D=(1, 0, 0), k0=PI, kshift=(0.25 * PI, 0, 0), n=120, axis=True,
                        params=dict(near_grid=(24, 1, 1), near_order=3, far_grid=(6, 6, 6))),
    "p3_npsp_auto": dict(dim=3, L=(1, 1, 1), D=(1, 1, 1), k0=0, kshift=(0, 0, 0), n=500,
                         params=dict(near_order=2, far_grid=(6, 6, 6))),
}


def regime_of(case) -> str:
    k0 = complex(case["k0"])
    ks = [complex(k) for k in case["kshift"]]
    if k0 == 0 and all(k == 0 for k in ks):
        return "npsp"
    return "static-shifted" if k0 == 0 else "dynamic"


def case_inputs(name: str):
    """(src positions, q, observer positions or None) for a small case, seeded by
    the case's index in SMALL_CASES."""
    case = SMALL_CASES[name]
    seed = 1000 + list(SMALL_CASES).index(name)
    rng = np.random.default_rng(seed)
    D = np.asarray(case["D"], dtype=float)
    n = case["n"]
    pos = rng.uniform(0.0, 1.0, (n, 3)) * D
    if case.get("axis"):
        pos[:, 1:] = 0.0
    q = rng.standard_normal(n).astype(complex)
    if regime_of(case) == "npsp":
        q -= q.mean()
    else:
        q = q + 1j * rng.standard_normal(n)
    obs = None
    if "m" in case:
        obs = rng.uniform(0.0, 1.0, (case["m"], 3)) * D
    return pos, q, obs
