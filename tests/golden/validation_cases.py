"""Seeded problem descriptions for the host-side validation pin
(tests/golden/make_validation_golden.py, tests/test_problem_cpu.py).

Each case is plain data so that the generator (which imports the reference) and
the test (which imports this repo's `problem` module) build the same problem:
  dim, L, D, k0 (re, im), kshift, regime name, params kwargs,
  src: (n, seed, scale per axis, charge rule), obs: (m, seed, scale, shift)
"""
from __future__ import annotations

import numpy as np

CASES = {
    # clean problems of every regime
    "clean_npsp_1d": dict(dim=1, L=(1, 1, 1), D=(1, 1, 1), k0=(0, 0), kshift=(0, 0, 0), regime="NPSP",
                          params=dict(), src=(12, 1, (1, 1, 1), "neutral"), obs=(5, 2, (1, 1, 1), (0, 0, 0))),
    "clean_dynamic_1d": dict(dim=1, L=(1, 1, 1), D=(1, 1, 1), k0=(1, -1), kshift=(0, 0, 0), regime="DYNAMIC",
                             params=dict(near_grid=(7, 7, 7)), src=(2, 3, (1, 1, 1), "raw"),
                             obs=(1, 4, (1, 1, 1), (0, 0, 0))),
    "clean_shifted_2d": dict(dim=2, L=(2, 2, 1), D=(2, 2, 1), k0=(0, 0), kshift=(0.3, 0.1, 0), regime="STATIC_SHIFTED",
                             params=dict(near_grid=(9, 9, 9)), src=(20, 5, (2, 2, 1), "raw"),
                             obs=(6, 6, (2, 2, 1), (0, 0, 0))),
    "clean_dynamic_3d": dict(dim=3, L=(1, 1, 1), D=(1, 1, 1), k0=(6.2, 0), kshift=(0.6, 0.3, 0), regime="DYNAMIC",
                             params=dict(near_grid=(12, 12, 12), near_order=3), src=(50, 7, (1, 1, 1), "raw"),
                             obs=(50, 7, (1, 1, 1), (0, 0, 0))),
    # one violation each
    "net_charge": dict(dim=1, L=(1, 1, 1), D=(1, 1, 1), k0=(0, 0), kshift=(0, 0, 0), regime="NPSP",
                       params=dict(), src=(9, 8, (1, 1, 1), "raw"), obs=(3, 9, (1, 1, 1), (0, 0, 0))),
    "net_charge_loose_tol": dict(dim=1, L=(1, 1, 1), D=(1, 1, 1), k0=(0, 0), kshift=(0, 0, 0), regime="NPSP",
                                 params=dict(neutrality_rtol=10.0), src=(9, 8, (1, 1, 1), "raw"),
                                 obs=(3, 9, (1, 1, 1), (0, 0, 0))),
    "box_over_period": dict(dim=1, L=(1, 1, 1), D=(2, 1, 1), k0=(0, 0), kshift=(0, 0, 0), regime="NPSP",
                            params=dict(), src=(4, 10, (2, 1, 1), "neutral"), obs=(2, 11, (2, 1, 1), (0, 0, 0))),
    "box_over_period_axis1": dict(dim=2, L=(3, 1, 1), D=(1, 1.5, 1), k0=(0, 0), kshift=(0, 0, 0), regime="NPSP",
                                  params=dict(), src=(4, 10, (1, 1.5, 1), "neutral"),
                                  obs=(2, 11, (1, 1.5, 1), (0, 0, 0))),
    "npsp_with_k0": dict(dim=1, L=(1, 1, 1), D=(1, 1, 1), k0=(1, 0), kshift=(0, 0, 0), regime="NPSP",
                         params=dict(), src=(4, 12, (1, 1, 1), "neutral"), obs=(2, 13, (1, 1, 1), (0, 0, 0))),
    "dynamic_without_k0": dict(dim=1, L=(1, 1, 1), D=(1, 1, 1), k0=(0, 0), kshift=(0, 0, 0), regime="DYNAMIC",
                               params=dict(), src=(4, 12, (1, 1, 1), "neutral"), obs=(2, 13, (1, 1, 1), (0, 0, 0))),
    "shifted_with_k0": dict(dim=2, L=(1, 1, 1), D=(1, 1, 1), k0=(2, 0), kshift=(0.1, 0, 0), regime="STATIC_SHIFTED",
                            params=dict(), src=(4, 12, (1, 1, 1), "raw"), obs=(2, 13, (1, 1, 1), (0, 0, 0))),
    "observer_outside": dict(dim=1, L=(1, 1, 1), D=(1, 1, 1), k0=(0, 0), kshift=(0, 0, 0), regime="NPSP",
                             params=dict(), src=(4, 14, (1, 1, 1), "neutral"), obs=(3, 15, (1, 1, 1), (0.8, 0, 0))),
    "source_outside_two_axes": dict(dim=3, L=(1, 1, 1), D=(1, 1, 1), k0=(3, 0), kshift=(0, 0, 0), regime="DYNAMIC",
                                    params=dict(near_grid=(8, 8, 8)), src=(6, 16, (1.4, 1, 1.7), "raw"),
                                    obs=(3, 17, (1, 1, 1), (0, 0, 0))),
    "id_zero": dict(dim=1, L=(1, 1, 1), D=(1, 1, 1), k0=(0, 0), kshift=(0, 0, 0), regime="NPSP",
                    params=dict(i_d=0), src=(4, 18, (1, 1, 1), "neutral"), obs=(2, 19, (1, 1, 1), (0, 0, 0))),
    "far_order_over_grid": dict(dim=1, L=(1, 1, 1), D=(1, 1, 1), k0=(0, 0), kshift=(0, 0, 0), regime="NPSP",
                                params=dict(far_order=6, far_grid=(6, 6, 6)), src=(4, 18, (1, 1, 1), "neutral"),
                                obs=(2, 19, (1, 1, 1), (0, 0, 0))),
    "near_order_over_grid": dict(dim=1, L=(1, 1, 1), D=(1, 1, 1), k0=(0, 0), kshift=(0, 0, 0), regime="NPSP",
                                 params=dict(near_order=5, near_grid=(4, 9, 9)), src=(4, 18, (1, 1, 1), "neutral"),
                                 obs=(2, 19, (1, 1, 1), (0, 0, 0))),
    "er_range_too_wide": dict(dim=1, L=(1, 1, 1), D=(1, 1, 1), k0=(0, 0), kshift=(0, 0, 0), regime="NPSP",
                              params=dict(near_grid=(3, 9, 9), er_range_boxes=1), src=(4, 20, (1, 1, 1), "neutral"),
                              obs=(2, 21, (1, 1, 1), (0, 0, 0))),
    "series_tol_and_er_boxes": dict(dim=1, L=(1, 1, 1), D=(1, 1, 1), k0=(0, 0), kshift=(0, 0, 0), regime="NPSP",
                                    params=dict(series_tol=0.0, er_range_boxes=0), src=(4, 20, (1, 1, 1), "neutral"),
                                    obs=(2, 21, (1, 1, 1), (0, 0, 0))),
    "empty_sets": dict(dim=1, L=(1, 1, 1), D=(1, 1, 1), k0=(0, 0), kshift=(0, 0, 0), regime="NPSP",
                       params=dict(near_grid=(7, 7, 7)), src=(0, 22, (1, 1, 1), "raw"),
                       obs=(0, 23, (1, 1, 1), (0, 0, 0))),
    "planar_box": dict(dim=2, L=(1, 1, 1), D=(1, 1, 0), k0=(0, 0), kshift=(0, 0, 0), regime="NPSP",
                       params=dict(), src=(30, 24, (1, 1, 0), "neutral"), obs=(5, 25, (1, 1, 0), (0, 0, 0))),
    "flat_periodic_axis": dict(dim=2, L=(1, 1, 1), D=(1, 0, 1), k0=(0, 0), kshift=(0, 0, 0), regime="NPSP",
                               params=dict(), src=(8, 26, (1, 0, 1), "neutral"), obs=(5, 27, (1, 0, 1), (0, 0, 0))),
    # several violations at once: order of the messages is part of the contract
    "many": dict(dim=2, L=(1, 0.5, 1), D=(1.2, 0.9, 1), k0=(1, 0), kshift=(0, 0, 0), regime="NPSP",
                 params=dict(i_d=0, far_order=7, far_grid=(5, 5, 5), near_grid=(3, 3, 3), near_order=4),
                 src=(7, 28, (1.5, 0.9, 1), "raw"), obs=(3, 29, (1.2, 0.9, 1.3), (0, 0, 0))),
}

AUTO_DIMS = [(n, d) for n in (1, 2, 7, 100, 3096, 12175, 53601, 92233, 177973, 1_000_000, 8_388_608)
             for d in ((1.0, 1.0, 1.0), (1.0, 1.0, 0.0), (0.0, 2.0, 0.0))]


def points(n, seed, scale, shift=(0.0, 0.0, 0.0)):
    rng = np.random.default_rng(seed)
    return rng.uniform(0.0, 1.0, (n, 3)) * np.asarray(scale, dtype=float) + np.asarray(shift, dtype=float)


def charges(n, seed, rule):
    rng = np.random.default_rng(seed + 1000)
    q = rng.uniform(-1.0, 1.0, n)
    if rule == "neutral" and n:
        q = q - q.mean()
        q[-1] -= q.sum()
    return q


def build(case, ns):
    """Instantiate the case with the types of namespace `ns` (the reference's
    `perisum.model` or this repo's `problem` module: same names)."""
    c = CASES[case]
    cfg = ns.PeriodicityConfig(dim=ns.Periodicity(c["dim"]), L=c["L"], k0=complex(*c["k0"]), kshift=c["kshift"],
                               regime=getattr(ns.Regime, c["regime"]))
    box = ns.TargetBox(c["D"])
    n, seed, scale, rule = c["src"]
    src = ns.SourcePointSet(points(n, seed, scale), charges(n, seed, rule))
    m, oseed, oscale, shift = c["obs"]
    obs = ns.ObserverPointSet(points(m, oseed, oscale, shift))
    return cfg, box, src, obs, ns.SolverParams(**c["params"])
