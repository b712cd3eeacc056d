"""Device brute-force oracle (direct_kernels.cu) through
the C ABI: the reference's own outputs (tests/golden/direct_cases.npz), the
failure records and chunk semantics, the oracle restatement on larger random
instances, and the FFT-PIM accuracy it exists to measure."""
import warnings

import numpy as np
import pytest

from conftest import golden, rel_l2
from oracle.direct import direct as oracle_direct
from oracle.problem import make_problem

pytestmark = pytest.mark.gpu

D = golden("direct_cases.npz")
NAMES = [str(n) for n in D["names"]]
REASON = {"separation": 1, "not converged": 2}


@pytest.fixture(scope="module")
def fp():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2312_02376_b200 as fp
    fp._native.load()
    return fp


def case(name):
    return {k.split("__", 1)[1]: D[k] for k in D.files if k.startswith(name + "__")}


def config(fp, c):
    regime = {"dynamic": fp.Regime.DYNAMIC, "npsp": fp.Regime.NPSP}[str(c["regime"])]
    return fp.PeriodicityConfig(dim=fp.Periodicity(int(c["dim"])), L=tuple(c["L"]), k0=complex(c["k0"]),
                                kshift=tuple(complex(k) for k in c["kshift"]), regime=regime)


@pytest.mark.parametrize("name", NAMES)
def test_direct_matches_reference(fp, name):
    c = case(name)
    src, obs = fp.SourcePointSet(c["src"], c["q"]), fp.ObserverPointSet(c["obs"])
    if str(c["mode"]) == "free":
        u = fp.eval_free_space(complex(c["k0"]), src, obs)
        assert rel_l2(u, c["u"]) <= 1e-13
        return
    pol = fp.TruncationPolicy(float(c["tol"]), int(c["max_terms"]), int(c["consecutive"]))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        cfg = config(fp, c)
    if str(c["mode"]) == "far":
        rep = fp.eval_direct_farzone(cfg, src, obs, int(c["i_d"]), pol)
    else:
        rep = fp.eval_direct(cfg, src, obs, pol)
    assert rel_l2(rep.values, c["u"]) <= 1e-10
    assert rep.worst_terms == int(c["worst"])
    got = np.array([(i, j, REASON[r]) for i, j, r in rep.failures], dtype=np.int64).reshape(-1, 3)
    assert np.array_equal(got, c["failures"])
    assert rep.ok() == (len(c["failures"]) == 0)
    if len(c["failures"]) and (c["failures"][:, 2] == 1).any():
        # a chunk with a separation failure keeps 0 potentials (oracle.py:78-80)
        assert np.all(rep.values[:64] == 0)


@pytest.mark.parametrize("dim,regime,i_d", [(3, "npsp", None), (2, "dynamic", 1), (1, "dynamic", None),
                                            (3, "dynamic", None)])
def test_direct_matches_oracle_random(fp, dim, regime, i_d):
    """Several 64-observer chunks (per-chunk 3D lattice lead ranges) and the
    multi-launch path; against the numpy restatement."""
    rng = np.random.default_rng(31 + dim)
    n, m = (40, 130) if (dim, regime) == (3, "dynamic") else (150, 200)
    src_p = rng.uniform(0, 1, (n, 3))
    obs_p = rng.uniform(0, 1, (m, 3))
    if regime == "npsp":
        q = rng.standard_normal(n)
        q -= q.mean()
        k0, ks = 0.0, (0, 0, 0)
    else:
        q = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        k0, ks = 1.5 * np.pi - 0.4j, (0.2 * np.pi, 0.1 * np.pi, 0)
        if dim == 2:   # |z| differences away from 0 (2D spectral series)
            src_p[:, 2] *= 0.3
            obs_p[:, 2] = 0.6 + 0.4 * obs_p[:, 2]
    tol = 1e-10 if dim < 3 or regime == "npsp" else 1e-8
    pb = make_problem(dim, k0=k0, kshift=ks, regime=regime)
    u_ref, worst, fails = oracle_direct(pb, src_p, q, obs_p, i_d=i_d, tol=tol)
    reg = fp.Regime.NPSP if regime == "npsp" else fp.Regime.DYNAMIC
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        cfg = fp.PeriodicityConfig(dim=fp.Periodicity(dim), L=(1, 1, 1), k0=k0, kshift=ks, regime=reg)
    src, obs = fp.SourcePointSet(src_p, q), fp.ObserverPointSet(obs_p)
    pol = fp.TruncationPolicy(tol=tol)
    rep = fp.eval_direct(cfg, src, obs, pol) if i_d is None else fp.eval_direct_farzone(cfg, src, obs, i_d, pol)
    # 3D spectral series overflow (inf * 0) on long z stacks in the reference's
    # arithmetic as well: the same observers come out NaN
    bad = np.isnan(u_ref)
    assert np.array_equal(np.isnan(rep.values), bad)
    assert rel_l2(rep.values[~bad], u_ref[~bad]) <= 1e-10
    assert rep.worst_terms == worst
    assert len(rep.failures) == len(fails)


def test_free_space_coincident_raises(fp):
    p = np.random.default_rng(0).uniform(size=(5, 3))
    with pytest.raises(ZeroDivisionError):
        fp.eval_free_space(1.0, fp.SourcePointSet(p, np.ones(5)), fp.ObserverPointSet(p))


def test_fftpim_accuracy_against_direct(fp):
    """The error study the oracle exists for (cli.py:275-317): FFT-PIM vs the
    per-pair converged sum on observers separate from the sources."""
    rng = np.random.default_rng(7)
    n = 400
    src_p = rng.uniform(0, 1, (n, 3))
    obs_p = rng.uniform(0.05, 0.95, (120, 3))
    q = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity.P1D, L=(1, 1, 1), k0=np.pi, kshift=(0.3 * np.pi, 0, 0),
                               regime=fp.Regime.DYNAMIC)
    src, obs = fp.SourcePointSet(src_p, q), fp.ObserverPointSet(obs_p)
    ref = fp.eval_direct(cfg, src, obs, fp.TruncationPolicy(tol=1e-12))
    assert ref.ok()
    errs = []
    for order in (2, 4):
        plan = fp.build_plan(cfg, fp.TargetBox((1, 1, 1)), src, obs,
                             fp.SolverParams(near_grid=(16, 16, 16), near_order=order))
        u = plan.evaluate(q)
        errs.append(float(np.max(np.abs(u - ref.values)) / np.max(np.abs(ref.values))))
    assert errs[1] < errs[0] and errs[1] < 1e-3, errs


@pytest.mark.parametrize("key", ["c0", "c1", "c2"])
def test_near_only_id0_plan_matches_reference(fp, key):
    """build_near_plan(i_d = 0) + eval_near on the device against the reference
    (the free-space baseline of the reference's bench, cli.py:343-347); the far
    engine refuses such a plan like the reference (farzone.py:84-85)."""
    g = golden("near_id0.npz")
    c = {k.split("__", 1)[1]: g[k] for k in g.files if k.startswith(key + "__")}
    regime = {"dynamic": fp.Regime.DYNAMIC, "npsp": fp.Regime.NPSP}[str(c["regime"])]
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity(int(c["dim"])), L=(1, 1, 1), k0=complex(c["k0"]),
                               kshift=tuple(complex(k) for k in c["kshift"]), regime=regime)
    prm = fp.SolverParams(i_d=0, near_grid=(10, 10, 10), near_order=3)
    src, obs = fp.SourcePointSet(c["pos"], c["q"]), fp.ObserverPointSet(c["pos"])
    near = fp.build_near_plan(cfg, fp.TargetBox((1, 1, 1)), src, obs, prm)
    assert near.native.info.n_pairs == int(c["n_pairs"])
    assert near.n_wrapped_pairs == 0
    assert tuple(near.join_radius) == tuple(int(v) for v in c["join_radius"])
    assert rel_l2(fp.eval_near(near, c["q"]), c["u"]) <= 1e-10
    with pytest.raises(ValueError):
        near.native.evaluate(c["q"], fp._native.ALL)
    with pytest.raises(fp.ValidationError):
        fp.build_plan(cfg, fp.TargetBox((1, 1, 1)), src, obs, prm)
