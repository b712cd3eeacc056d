"""Drop-in boundary behaviour on the GPU:

* build_near_plan / build_far_plan build only their zone (nearzone.py:194-273,
  farzone.py:76-131) and refuse the other zone's evaluation; their sum equals
  build_plan's evaluation;
* the PIMF kernel cache (farzone.py:103-123): a blob written by the REFERENCE
  is a hit (table and kernel_terms from the blob, potentials equal the
  reference's eval_far), a miss writes the blob, a second build hits, a changed
  tolerance misses;
* a SpectralTransformProvider cannot be plugged in (raises);
* repeated evaluate(tensor) calls with retained outputs update one graph
  executable instead of instantiating a new one per call."""
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN, rel_l2

pytestmark = pytest.mark.gpu

PROBLEM = dict(dim=3, L=(1.0, 1.0, 1.0), D=(1.0, 1.0, 1.0), k0=2.0 * np.pi,
               kshift=(0.2 * np.pi, 0.1 * np.pi, 0.0), far_grid=(6, 6, 6), far_order=3,
               near_grid=(12, 12, 12), near_order=3)


@pytest.fixture(scope="module")
def fp():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2312_02376_b200 as fp
    fp._native.load()
    return fp


def _objects(fp, tol=1e-10):
    g = np.load(os.path.join(GOLDEN, "ref_far_kernel.npz"))
    p = PROBLEM
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity(p["dim"]), L=p["L"], k0=p["k0"], kshift=p["kshift"],
                               regime=fp.Regime.DYNAMIC)
    prm = fp.SolverParams(far_grid=p["far_grid"], far_order=p["far_order"], near_grid=p["near_grid"],
                          near_order=p["near_order"], series_tol=tol)
    return g, cfg, fp.TargetBox(p["D"]), fp.SourcePointSet(g["pos"], g["q"]), fp.ObserverPointSet(g["pos"]), prm


def test_reference_blob_is_a_cache_hit(fp, tmp_path):
    g, cfg, box, src, obs, prm = _objects(fp)
    path = tmp_path / "k.pimf"
    shutil.copy(os.path.join(GOLDEN, "ref_far_kernel.pimf"), path)
    before = path.read_bytes()
    far = fp.build_far_plan(cfg, box, src, obs, prm, cache_path=path)
    assert far.native.kernel_cache_hit
    np.testing.assert_array_equal(far.kernel, g["kernel"])
    assert far.kernel_terms == int(g["kernel_terms"])
    assert path.read_bytes() == before            # a hit does not rewrite the blob
    assert rel_l2(fp.eval_far(far, g["q"]), g["u_far"]) <= 1e-10


def test_cache_miss_writes_then_hits(fp, tmp_path):
    g, cfg, box, src, obs, prm = _objects(fp)
    path = tmp_path / "cache.pimf"
    p1 = fp.build_far_plan(cfg, box, src, obs, prm, cache_path=path)
    assert not p1.native.kernel_cache_hit and path.exists()
    p2 = fp.build_far_plan(cfg, box, src, obs, prm, cache_path=path)
    assert p2.native.kernel_cache_hit
    np.testing.assert_array_equal(p1.kernel, p2.kernel)
    assert p1.kernel_terms == p2.kernel_terms
    np.testing.assert_array_equal(fp.eval_far(p1, g["q"]), fp.eval_far(p2, g["q"]))
    # a different tolerance changes the signature: miss, rebuild, blob rewritten
    g, cfg, box, src, obs, prm8 = _objects(fp, tol=1e-8)
    p3 = fp.build_far_plan(cfg, box, src, obs, prm8, cache_path=path)
    assert not p3.native.kernel_cache_hit
    assert p3.kernel.shape == p1.kernel.shape
    # build_plan's kernel_cache goes through the same path
    plan = fp.build_plan(cfg, box, src, obs, prm8, kernel_cache=path)
    assert plan.native.kernel_cache_hit
    # a corrupt blob is a miss (KernelCacheError swallowed, farzone.py:110-111)
    path.write_bytes(b"XXXX" + path.read_bytes()[4:])
    p4 = fp.build_far_plan(cfg, box, src, obs, prm8, cache_path=path)
    assert not p4.native.kernel_cache_hit and path.read_bytes()[:4] == b"PIMF"


def test_zone_plans_build_one_zone(fp):
    g, cfg, box, src, obs, prm = _objects(fp)
    q = g["q"]
    full = fp.build_plan(cfg, box, src, obs, prm)
    near = fp.build_near_plan(cfg, box, src, obs, prm)
    far = fp.build_far_plan(cfg, box, src, obs, prm)
    nat = fp._native
    assert near.native.info.built_parts == nat.NEAR and far.native.info.built_parts == nat.FAR
    assert far.native.info.n_pairs == 0 and near.native.info.n_pairs == full.native.info.n_pairs
    assert near.native.info.kernel_terms == 0 and far.kernel_terms == full.far.kernel_terms
    assert far.native.info.device_bytes < full.native.info.device_bytes
    assert rel_l2(fp.eval_near(near, q) + fp.eval_far(far, q), full.evaluate(q)) <= 1e-13
    assert rel_l2(fp.eval_far(far, q), g["u_far"]) <= 1e-10
    with pytest.raises(ValueError, match="without the near zone"):
        fp.eval_near(fp.NearZonePlan(far.native), q)
    with pytest.raises(ValueError, match="without the far zone"):
        fp.eval_far(fp.FarZonePlan(near.native), q)


def test_provider_is_refused(fp):
    g, cfg, box, src, obs, prm = _objects(fp)

    class NumpyLikeProvider:
        def forward(self, a):
            return np.fft.fftn(a)

        def inverse(self, a):
            return np.fft.ifftn(a)

    with pytest.raises(TypeError, match="SpectralTransformProvider"):
        fp.build_plan(cfg, box, src, obs, prm, provider=NumpyLikeProvider())
    with pytest.raises(TypeError):
        fp.build_near_plan(cfg, box, src, obs, prm, provider=NumpyLikeProvider())


def test_retained_outputs_update_one_graph(fp):
    import torch
    g, cfg, box, src, obs, prm = _objects(fp)
    plan = fp.build_plan(cfg, box, src, obs, prm)
    qd = torch.from_numpy(g["q"]).cuda()
    outs = [plan.evaluate(qd) for _ in range(100)]       # a fresh output tensor each call
    torch.cuda.synchronize()
    info = plan.native.refresh_info()
    assert info.graph_captures == 100
    assert info.graph_instantiations == 1
    ref = outs[0].cpu().numpy()
    for u in outs[1:]:
        np.testing.assert_array_equal(u.cpu().numpy(), ref)


@pytest.mark.parametrize("name", ["p3_dyn", "p2_static_sep", "p2_planar_npsp", "p1_axis_dyn"])
def test_plan_operand_views(fp, name):
    """NearZonePlan.proj_op / interp_op / kernel_disp / seg_obs / seg_starts / d_er and
    FarZonePlan.proj_op / interp_op (nearzone.py:55-80, farzone.py:32-44) read back from
    the device plan: stencil starts and weights bit-identical to the oracle's
    (grids.py:110-140), flat forms equal, the displacement table to round-off."""
    from cases import SMALL_CASES, case_inputs, regime_of
    from oracle.pipeline import build_plan as oracle_build
    from oracle.problem import make_problem
    case = SMALL_CASES[name]
    pos, q, obs = case_inputs(name)
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity(case["dim"]), L=case["L"], k0=case["k0"],
                               kshift=case["kshift"], regime=fp.Regime(regime_of(case)))
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        plan = fp.build_plan(cfg, fp.TargetBox(case["D"]), fp.SourcePointSet(pos, q),
                             fp.ObserverPointSet(pos if obs is None else obs), fp.SolverParams(**case["params"]))
        ref = oracle_build(make_problem(case["dim"], L=case["L"], D=case["D"], k0=case["k0"],
                                        kshift=case["kshift"], **case["params"]), pos, obs)
    for got, want in ((plan.near.proj_op, ref.near.src), (plan.near.interp_op, ref.near.obs),
                      (plan.far.proj_op, ref.far.src), (plan.far.interp_op, ref.far.obs)):
        np.testing.assert_array_equal(got.axis_starts, want.starts)
        for a in range(3):
            np.testing.assert_array_equal(got.axis_weights[a], want.axis_w[a])
        np.testing.assert_array_equal(got.flat_index, want.flat_index)
        np.testing.assert_array_equal(got.flat_weight, want.flat_weight)
        assert got.n_points == want.starts.shape[0] and got.stencil_size == want.flat_index.shape[1]
    np.testing.assert_array_equal(plan.near.seg_obs, ref.near.seg_obs)
    np.testing.assert_array_equal(plan.near.seg_starts, ref.near.seg_starts)
    assert plan.near.kernel_disp.shape == ref.near.kernel_disp.shape
    assert rel_l2(plan.near.kernel_disp, ref.near.kernel_disp) <= 1e-12
    active = [a for a in range(3) if plan.near.grid.dims[a] > 1]
    assert plan.near.d_er == case["params"].get("er_range_boxes", 1) * max(plan.near.grid.spacing[a] for a in active)
