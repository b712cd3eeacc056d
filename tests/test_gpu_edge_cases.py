"""Edge-case inputs of the reference's own near-/far-zone tests, run through the
CUDA path (C ABI) and compared with the pinned CPU oracle on the same input:
single points, two points, points on grid nodes and on the box faces, sources
moved across the periodic boundary, a face-hugging fully corrected cluster,
one-cell clusters (every pair collides in one box), ragged source / observer
counts, zero charges, reciprocity, and the domain errors.

Behaviours follow /root/reference/pkg/tests/test_nearzone.py (self pair,
coinciding observer, boundary relabeling, fully corrected instance, wrapped
pairs, determinism) and test_grids.py (cardinal weights, partition of unity,
degree reproduction, hull check); the inputs and checks here are this repo's.
Tolerance: 1e-10 relative (bit-exact pair sets are pinned in test_gpu_parity)."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def fp():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2312_02376_b200 as fp
    fp._native.load()
    return fp


def _both(fp, dim, src_pos, q, obs_pos=None, L=(1.0, 1.0, 1.0), D=None, k0=0j, kshift=(0, 0, 0), plan_q=None, **params):
    """(gpu near, gpu far, oracle near, oracle far, gpu near plan, oracle plan)"""
    from oracle.far_engine import eval_far as o_far
    from oracle.near_engine import eval_near as o_near
    from oracle.pipeline import build_plan as oracle_build
    from oracle.problem import make_problem
    D = L if D is None else D
    pb = make_problem(dim, L=L, D=D, k0=k0, kshift=kshift, **params)
    src_pos = np.ascontiguousarray(src_pos, dtype=float)
    q = np.asarray(q, dtype=complex)
    op = oracle_build(pb, src_pos, obs_pos)
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity(dim), L=L, k0=k0, kshift=kshift, regime=fp.Regime(pb.regime))
    obs = fp.ObserverPointSet(src_pos if obs_pos is None else obs_pos)
    # plan_q: the amplitudes the facade validates (NPSP neutrality); evaluations take any q
    plan = fp.build_plan(cfg, fp.TargetBox(D), fp.SourcePointSet(src_pos, q if plan_q is None else plan_q), obs,
                         fp.SolverParams(**params))
    return (fp.eval_near(plan.near, q), fp.eval_far(plan.far, q), o_near(op.near, q), o_far(op.far, q), plan, op)


def _close(a, b, scale=None):
    a, b = np.asarray(a), np.asarray(b)
    s = max(float(np.max(np.abs(b))) if scale is None else scale, 1e-300)
    return float(np.max(np.abs(a - b))) / s


def _assert_parity(res, floor=0.0):
    gn, gf, on, of, plan, op = res
    assert plan.near.native.info.n_pairs == op.near.pair_obs.shape[0]
    scale = max(float(np.max(np.abs(on + of))), floor)
    assert _close(gn, on, scale) <= TOL and _close(gf, of, scale) <= TOL
    u0 = plan.evaluate(np.zeros(plan.near.n_sources, dtype=complex))
    assert u0.shape == on.shape and not u0.any()                     # exactly zero for q = 0


def test_single_point_self_pair(fp):
    """One source that is its own observer (test_nearzone.py:106-117): a plan
    of one point builds, the self pair is counted and contributes nothing."""
    pos = np.array([[1.7, 2.2, 1.1]])
    q = np.array([2.0 - 1.0j])
    gn, gf, on, of, plan, op = _both(fp, 1, pos, q, L=(4.0, 4.0, 4.0), near_grid=(7, 7, 7), plan_q=[0.0])
    assert plan.near.same_points and plan.near.n_self_pairs == 1
    assert abs(on[0]) < 1e-13 and abs(gn[0]) < 1e-13
    assert abs(gf[0] - of[0]) <= TOL * max(abs(of[0]), 1e-3)


@pytest.mark.parametrize("dim,k0,ks", [(1, 0j, (0, 0, 0)), (2, 1.5, (0.3, 0.2, 0)), (3, 2.0 - 0.3j, (0.2, 0.1, 0.4))])
def test_two_points(fp, dim, k0, ks):
    pos = np.array([[0.31, 0.42, 0.55], [0.36, 0.47, 0.49]])
    q = np.array([1.0, -1.0], dtype=complex)
    _assert_parity(_both(fp, dim, pos, q, k0=k0, kshift=ks, near_grid=(8, 8, 8), near_order=2, far_grid=(5, 5, 5)))


def test_one_source_many_observers_and_back(fp):
    rng = np.random.default_rng(5)
    many = rng.uniform(0.05, 0.95, (200, 3))
    one = np.array([[0.5, 0.52, 0.47]])
    kw = dict(k0=3.0, kshift=(0.2, 0.0, 0.1), near_grid=(9, 9, 9), near_order=3, far_grid=(6, 6, 6))
    _assert_parity(_both(fp, 3, one, [1.0 + 0.5j], obs_pos=many, **kw))
    q = rng.standard_normal(200) + 1j * rng.standard_normal(200)
    _assert_parity(_both(fp, 3, many, q, obs_pos=one + 1e-3, **kw))


def test_points_on_nodes_and_faces(fp):
    """Points exactly on near-grid nodes (cardinal weights, test_grids.py) and on
    all faces / corners of the box, where stencil starts clip (grids.py:118-121)."""
    n = 9
    ax = np.linspace(0.0, 1.0, n)
    # periodic along x only: the x = 1 face is left out (it is the lattice image of x = 0, see
    # test_domain_errors); y and z carry both faces
    nodes = np.stack(np.meshgrid(ax[:-1:2], ax[::4], ax[::2], indexing="ij"), -1).reshape(-1, 3)
    rng = np.random.default_rng(6)
    q = rng.standard_normal(nodes.shape[0]) + 1j * rng.standard_normal(nodes.shape[0])
    res = _both(fp, 1, nodes, q, k0=2.5, kshift=(0.1, 0, 0), near_grid=(n, n, n), near_order=2, far_grid=(5, 5, 5))
    _assert_parity(res)
    op = res[4].near.proj_op
    for a in range(3):
        w = op.axis_weights[a]
        assert np.all(np.sort(w, axis=1)[:, :-1] == 0.0) and np.all(w.max(axis=1) == 1.0)   # one-hot
        node = np.rint(nodes[:, a] * (n - 1)).astype(int)
        assert np.all(op.axis_starts[:, a] + np.argmax(w, axis=1) == node)


def test_device_stencils_partition_and_reproduce_polynomials(fp):
    """Partition of unity, locality and exactness for polynomials of degree <= order
    (test_grids.py) of the stencils the device computes, for every order."""
    rng = np.random.default_rng(7)
    pos = rng.uniform(0.0, 1.0, (400, 3)) * np.array([1.0, 0.7, 0.4])
    q = rng.standard_normal(400) + 0j
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity.P3D, L=(1, 1, 1), k0=2.0, kshift=(0.1, 0, 0), regime=fp.Regime.DYNAMIC)
    for order, grid in [(1, (6, 7, 8)), (2, (9, 8, 7)), (3, (8, 8, 8)), (4, (10, 9, 8)), (5, (9, 9, 9))]:
        plan = fp.build_plan(cfg, fp.TargetBox((1.0, 0.7, 0.4)), fp.SourcePointSet(pos, q), fp.ObserverPointSet(pos),
                             fp.SolverParams(near_grid=grid, near_order=order, far_grid=(6, 6, 6)))
        for op, g in ((plan.near.proj_op, plan.near.grid), (plan.far.interp_op, plan.far.observer_grid)):
            o = op.order
            for a in range(3):
                w, s = op.axis_weights[a], op.axis_starts[:, a]
                assert w.shape[1] == o + 1 and np.max(np.abs(w.sum(axis=1) - 1.0)) <= 1e-13
                assert s.min() >= 0 and s.max() + o <= g.dims[a] - 1
                x = (s[:, None] + np.arange(o + 1)[None, :]) * g.spacing[a] + g.origin[a]
                inside = (pos[:, a] >= g.origin[a]) & (pos[:, a] <= g.origin[a] + (g.dims[a] - 1) * g.spacing[a])
                # the stencil brackets the point whenever the point lies inside the grid hull
                assert np.all((x[inside, 0] <= pos[inside, a] + 1e-12) & (pos[inside, a] <= x[inside, -1] + 1e-12))
                for deg in range(o + 1):
                    assert np.max(np.abs((w * x**deg).sum(axis=1) - pos[:, a] ** deg)) <= 1e-12
        assert np.max(np.abs(plan.near.proj_op.flat_weight.sum(axis=1) - 1.0)) <= 1e-12   # charge conservation of K1


def test_source_moved_across_the_boundary(fp):
    """A source at x = 0 and its lattice image at x = L with the amplitude rotated by
    the Floquet phase give the same near potential (test_nearzone.py:231-258); a
    strongly decaying wavenumber suppresses the truncation-set difference."""
    L, k0, kx = 1.0, -25j, 0.4
    rng = np.random.default_rng(9)
    obs = rng.uniform(0.1, 0.9, (14, 3))
    rest = rng.uniform(0.15, 0.85, (7, 3))
    amp = np.concatenate([[1.3 - 0.7j], rng.standard_normal(7) + 1j * rng.standard_normal(7)])
    pa = np.vstack([[[0.0, 0.55, 0.48]], rest])
    pb_ = pa.copy()
    pb_[0, 0] = L
    amp_b = amp.copy()
    amp_b[0] *= np.exp(-1j * kx * L)
    kw = dict(k0=k0, kshift=(kx, 0, 0), near_grid=(11, 11, 11))
    ra = _both(fp, 1, pa, amp, obs_pos=obs, **kw)
    rb = _both(fp, 1, pb_, amp_b, obs_pos=obs, **kw)
    _assert_parity(ra)
    _assert_parity(rb)
    assert _close(ra[0], rb[0]) <= 1e-10
    assert ra[4].near.n_wrapped_pairs > 0 or rb[4].near.n_wrapped_pairs > 0


def test_face_hugging_cluster_is_fully_corrected(fp):
    """Every pair is close directly or through one wrapped image, so the near potential
    equals the exact truncated image sum (test_nearzone.py:261-300): checked
    against the oracle AND against explicit sums of the decaying free-space kernel."""
    L, k0 = 1.0, -30j
    rng = np.random.default_rng(11)
    left = rng.uniform(0.0, 0.04, (6, 1))
    right = rng.uniform(0.96, 1.0, (6, 1))
    pos = np.hstack([np.vstack([left, right]), rng.uniform(0.45, 0.55, (12, 2))])
    q = rng.standard_normal(12) + 1j * rng.standard_normal(12)
    res = _both(fp, 1, pos, q, k0=k0, near_grid=(11, 11, 11), near_order=2)
    _assert_parity(res)
    plan = res[4]
    assert plan.near.n_wrapped_pairs > 0
    exact = np.zeros(12, dtype=complex)
    for m in (-1, 0, 1):
        d = pos[:, None, :] - pos[None, :, :] - np.array([m * L, 0.0, 0.0])
        r = np.sqrt((d * d).sum(-1))
        with np.errstate(divide="ignore", invalid="ignore"):
            g = np.where(r > 0, np.exp(-1j * k0 * r) / (4 * np.pi * r), 0.0)
        exact += g @ q
    assert _close(res[0], exact) <= 1e-9


@pytest.mark.parametrize("dim,k0,ks,order", [(3, 0j, (0, 0, 0), 2), (3, 4.0, (0.5, 0.2, 0.1), 4), (2, 0j, (0.2, 0.1, 0), 3)])
def test_all_points_in_one_cell(fp, dim, k0, ks, order):
    """A tight cluster inside one near-grid box: every pair collides in the same
    source box (dense K4 rows, one K1 cell, one observer tile)."""
    rng = np.random.default_rng(12)
    pos = 0.5 + rng.uniform(-0.02, 0.02, (300, 3))
    q = rng.standard_normal(300) + 0j
    q = q - q.mean() if (k0 == 0 and not any(ks)) else q + 1j * rng.standard_normal(300)
    res = _both(fp, dim, pos, q, k0=k0, kshift=ks, near_grid=(10, 10, 10), near_order=order, far_grid=(6, 6, 6))
    _assert_parity(res)
    assert res[4].near.native.info.n_pairs == 300 * 300


def test_reciprocity_of_the_npsp_operator(fp):
    """u = A q with A symmetric for same points and the even NPSP kernel: <p, A q> =
    <q, A p>.  Couples K1/K3 adjointness (test_grids.py transpose identity) with the
    symmetry of the correction coefficients."""
    rng = np.random.default_rng(13)
    pos = rng.uniform(0, 1, (500, 3))
    p, q = rng.standard_normal((2, 500))
    p -= p.mean()
    q -= q.mean()
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity.P3D, L=(1, 1, 1))
    plan = fp.build_plan(cfg, fp.TargetBox((1, 1, 1)), fp.SourcePointSet(pos, q), fp.ObserverPointSet(pos),
                         fp.SolverParams(near_grid=(10, 10, 10), near_order=3))
    a, b = np.vdot(p, fp.eval_near(plan.near, q + 0j)), np.vdot(q, fp.eval_near(plan.near, p + 0j))
    assert abs(a - b) <= 1e-11 * max(abs(a), abs(b))


def test_domain_errors(fp):
    """An observer on top of a distinct source (test_nearzone.py:120-127) and a point
    outside the grid hull (test_grids.py) are refused with the reference's classes."""
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity.P1D, L=(4, 4, 4))
    src = fp.SourcePointSet([[1.0, 1.0, 1.0], [2.0, 2.0, 2.0]], [1.0, -1.0])
    with pytest.raises(fp.DomainError):
        fp.build_near_plan(cfg, fp.TargetBox((4, 4, 4)), src, fp.ObserverPointSet([[2.0, 2.0, 2.0]]),
                           fp.SolverParams(near_grid=(7, 7, 7)))
    # a point on the x = 0 face and one on the x = L face are lattice images of each other:
    # the wrapped copy coincides with a distinct source
    faces = fp.SourcePointSet([[0.0, 2.0, 2.0], [4.0, 2.0, 2.0], [1.0, 3.0, 1.0]], [1.0, -0.5, -0.5])
    with pytest.raises(fp.DomainError):
        fp.build_plan(cfg, fp.TargetBox((4, 4, 4)), faces, fp.ObserverPointSet(faces.positions),
                      fp.SolverParams(near_grid=(7, 7, 7)))
    with pytest.raises((fp.ValidationError, fp.DomainError)):
        fp.build_plan(cfg, fp.TargetBox((4, 4, 4)), src, fp.ObserverPointSet([[4.5, 2.0, 2.0]]),
                      fp.SolverParams(near_grid=(7, 7, 7)))
    with pytest.raises(fp.ValidationError):     # empty sets are a validation error, not a crash
        fp.build_plan(cfg, fp.TargetBox((4, 4, 4)), fp.SourcePointSet(np.zeros((0, 3)), np.zeros(0)),
                      fp.ObserverPointSet(np.zeros((0, 3))), fp.SolverParams(near_grid=(7, 7, 7)))
    plan = fp.build_plan(cfg, fp.TargetBox((4, 4, 4)), src, fp.ObserverPointSet([[3.0, 1.0, 2.5]]),
                         fp.SolverParams(near_grid=(7, 7, 7)))
    with pytest.raises(ValueError):             # ragged charge vector
        plan.evaluate(np.ones(3, dtype=complex))
