"""Randomized parity sweep: 24 seeded problems drawn across the parameter space of
the path (tests/random_problems.py: periodicity, regime, lossy k0, D < L, planar
boxes, orders 1-4, i_d 1-2, separate observers) through the CUDA path (C ABI)
against the pinned CPU oracle.  A draw the oracle refuses (the reference's
NotConverged / Wood / domain errors) has to be refused by the GPU build with the
matching exception class.  Tolerance 1e-10 relative to the potential's scale
(north_star), pair counts equal.  tools/check_random_problems.py runs the oracle
side alone on CPU."""
from __future__ import annotations

import numpy as np
import pytest

import random_problems as rp

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def fp():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2312_02376_b200 as fp
    fp._native.load()
    return fp


@pytest.mark.parametrize("seed", range(rp.N_DRAWS))
def test_random_problem_matches_oracle(fp, seed):
    from oracle.far_engine import eval_far as o_far
    from oracle.lattice_sums import SeriesError
    from oracle.near_engine import eval_near as o_near
    from oracle.pipeline import build_plan as oracle_build
    from oracle.problem import make_problem
    d = rp.draw(seed)
    kinds = {"domain": fp.DomainError, "wood": fp.WoodAnomalyError, "not_converged": fp.NotConvergedError,
             "separation": fp.SeparationError}
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity(d["dim"]), L=d["L"], k0=d["k0"], kshift=d["kshift"],
                               regime=fp.Regime(d["regime"]))
    obs = fp.ObserverPointSet(d["src"] if d["obs"] is None else d["obs"])

    def gpu_build():
        return fp.build_plan(cfg, fp.TargetBox(d["D"]), fp.SourcePointSet(d["src"], d["q"]), obs,
                             fp.SolverParams(**d["params"]))

    pb = make_problem(d["dim"], L=d["L"], D=d["D"], k0=d["k0"], kshift=d["kshift"], regime=d["regime"], **d["params"])
    try:
        op = oracle_build(pb, d["src"], d["obs"])
    except SeriesError as e:
        with pytest.raises(kinds[e.kind]):
            gpu_build()
        return
    plan = gpu_build()
    assert plan.near.native.info.n_pairs == op.near.pair_obs.shape[0]
    on, of = o_near(op.near, d["q"]), o_far(op.far, d["q"])
    gn, gf = fp.eval_near(plan.near, d["q"]), fp.eval_far(plan.far, d["q"])
    scale = float(np.max(np.abs(on + of)))
    assert np.max(np.abs(gn - on)) <= TOL * scale
    assert np.max(np.abs(gf - of)) <= TOL * scale
    u = plan.evaluate(d["q"])
    assert np.max(np.abs(u - (on + of))) <= TOL * scale
    # the fused evaluation equals the sum of its zones to rounding, and repeats bitwise
    assert np.max(np.abs(u - (gn + gf))) <= 1e-13 * scale
    assert np.array_equal(u, plan.evaluate(d["q"]))
