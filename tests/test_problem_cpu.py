"""Host-side domain types and validation against the reference's own output
(`perisum.model`, model.py:41-297).  The golden file holds the messages the
reference's `validate_problem` produced for the seeded problems of
tests/golden/validation_cases.py (tests/golden/make_validation_golden.py);
this repo's `validate_problem` has to give the same messages in the same order,
and `auto_near_dims` the same grid sizes.  No GPU, no native library."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

import validation_cases as vc
from conftest import GOLDEN
from paper_2312_02376_b200 import problem as P

with open(os.path.join(GOLDEN, "validation_golden.json")) as _f:
    GOLD = json.load(_f)


@pytest.mark.parametrize("name", sorted(vc.CASES))
def test_validation_messages_equal_reference(name):
    cfg, box, src, obs, params = vc.build(name, P)
    report = P.validate_problem(cfg, box, src, obs, params)
    assert list(report.messages) == GOLD["messages"][name]
    # report protocol (model.py:194-205): truthy <=> violations, ok() the opposite
    assert bool(report) == bool(GOLD["messages"][name])
    assert report.ok() != bool(report)
    for m in report.messages:
        assert report.contains(m[:12])
    assert not report.contains("no such fragment")


def test_validation_is_pure_and_repeatable():
    cfg, box, src, obs, params = vc.build("many", P)
    pos0, q0 = src.positions.copy(), src.amplitudes.copy()
    first = P.validate_problem(cfg, box, src, obs, params)
    second = P.validate_problem(cfg, box, src, obs, params)
    assert first.messages == second.messages
    assert np.array_equal(src.positions, pos0) and np.array_equal(src.amplitudes, q0)


def test_auto_near_dims_equal_reference():
    for n, d, dims in GOLD["auto_near_dims"]:
        assert list(P.auto_near_dims(n, P.TargetBox(tuple(d)))) == dims, (n, d)


def test_auto_near_dims_rules():
    # an odd, equal node count on every axis with extent, 1 on flat axes, >= 1.15 N nodes
    for n in (5, 640, 70001):
        dims = P.auto_near_dims(n, P.TargetBox((1.0, 2.0, 0.0)))
        assert dims[2] == 1 and dims[0] == dims[1] and dims[0] % 2 == 1
        assert dims[0] * dims[1] >= 1.15 * n
    with pytest.raises(ValueError):
        P.auto_near_dims(10, P.TargetBox((0.0, 0.0, 0.0)))


def test_point_sets_normalise_and_reject_bad_shapes():
    with pytest.raises(ValueError):
        P.SourcePointSet(np.zeros((4, 2)), np.zeros(4))
    with pytest.raises(ValueError):
        P.SourcePointSet(np.zeros((4, 3)), np.zeros(3))
    with pytest.raises(ValueError):
        P.ObserverPointSet(np.zeros((2, 4)))
    empty = P.SourcePointSet(np.zeros((0, 3)), np.zeros(0))
    assert len(empty) == 0 and empty.net_charge() == 0
    one = P.SourcePointSet([0.1, 0.2, 0.3], [2.0])   # a single point given as a flat triple
    assert one.positions.shape == (1, 3) and one.amplitudes.dtype == np.complex128
    s = P.SourcePointSet(np.arange(6.0).reshape(2, 3)[:, ::-1], np.array([1, -1], dtype=np.int32))
    assert s.positions.flags.c_contiguous and s.positions.dtype == np.float64
    assert s.net_charge() == 0
    assert len(P.ObserverPointSet(np.zeros((5, 3)))) == 5


def test_config_and_params_normalise():
    cfg = P.PeriodicityConfig(dim=P.Periodicity.P2D, L=(1, 2, 3), k0=0.0, kshift=(0, 0, 0), regime=P.Regime.NPSP)
    assert cfg.periodic_axes == (0, 1) and cfg.is_static_nophase()
    dyn = P.PeriodicityConfig(dim=P.Periodicity.P3D, L=(1, 1, 1), k0=2.0 - 0.1j, kshift=(0.1, 0, 0),
                              regime=P.Regime.DYNAMIC)
    assert dyn.periodic_axes == (0, 1, 2) and not dyn.is_static_nophase()
    assert cfg.canonical_key() != dyn.canonical_key()
    assert cfg.canonical_key() == P.PeriodicityConfig(dim=P.Periodicity.P2D, L=(1.0, 2.0, 3.0), k0=0j,
                                                      kshift=(0j, 0j, 0j), regime=P.Regime.NPSP).canonical_key()
    prm = P.SolverParams(far_grid=[6, 7, 8], near_grid=np.array([9, 9, 9]))
    assert prm.far_grid == (6, 7, 8) and prm.near_grid == (9, 9, 9)
    assert prm.resolve_near_grid(10**6, P.TargetBox((1, 1, 1))) == (9, 9, 9)
    assert P.SolverParams().resolve_near_grid(3096, P.TargetBox((1, 1, 1))) == (17, 17, 17)
    # reference defaults (model.py:166-190)
    d = P.SolverParams()
    assert (d.i_d, d.far_order, d.far_grid, d.near_order, d.near_grid, d.series_tol, d.er_range_boxes) == \
        (1, 3, (10, 10, 10), 2, None, 1e-10, 1)


def test_potential_field_flags_non_finite():
    assert P.PotentialField([1.0, 2.0 + 1j]).is_finite()
    assert not P.PotentialField([1.0, np.nan]).is_finite()
    assert not P.PotentialField([complex(0.0, np.inf)]).is_finite()
    assert P.PotentialField(np.ones((2, 2))).values.shape == (4,)
