"""Batched excitation sweep: one SweepPlan with E phase
shifts along a periodic axis must reproduce E independent plans (each built
with that shift), and the reference's own output where a golden fixture exists
(small cases: the case's shift; C5: excitation 0 on the reference's observer
sample)."""
import warnings

import numpy as np
import pytest

from conftest import golden, rel_l2
from cases import SMALL_CASES, case_inputs, regime_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fp():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2312_02376_b200 as fp
    fp._native.load()
    return fp


def objects(fp, case, pos, q, obs, kshift=None):
    ks = case["kshift"] if kshift is None else kshift
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity(case["dim"]), L=case["L"], k0=case["k0"], kshift=ks,
                               regime=fp.Regime(regime_of(case)))
    return (cfg, fp.TargetBox(case["D"]), fp.SourcePointSet(pos, q),
            fp.ObserverPointSet(pos if obs is None else obs), fp.SolverParams(**case["params"]))


@pytest.mark.parametrize("name,axis", [("p1_dyn", 0), ("p2_dyn", 0), ("p2_dyn", 1), ("p3_dyn", 1),
                                       ("p3_dyn_lossy_id2", 0), ("p2_static_sep", 0)])
def test_sweep_matches_independent_plans(fp, name, axis):
    case = SMALL_CASES[name]
    pos, q, obs = case_inputs(name)
    base = complex(case["kshift"][axis])
    shifts = [base, base + 0.37, base - 0.81, 1.3 + 0.0j, base + 0.05]
    rng = np.random.default_rng(5)
    Q = np.stack([q] + [rng.normal(size=q.shape) + 1j * rng.normal(size=q.shape) for _ in shifts[1:]])
    cfg, box, src, ob, prm = objects(fp, case, pos, q, obs)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        sw = fp.build_sweep_plan(cfg, box, src, ob, prm, axis, shifts)
        U = sw.evaluate(Q)
        for e, k in enumerate(shifts):
            ks = list(case["kshift"])
            ks[axis] = k
            plan = fp.build_plan(*objects(fp, case, pos, q, obs, tuple(ks)))
            assert rel_l2(U[e], plan.evaluate(Q[e])) <= 1e-12, (e, k)
    # excitation 0 carries the case's own shift: the reference's output
    g = golden(f"small_{name}.npz")
    assert rel_l2(U[0], g["u"]) <= 1e-10
    # the pair list is the single-excitation one
    assert sw.info.n_pairs == int(g["n_pairs"])


def test_sweep_errors(fp):
    case = SMALL_CASES["p3_npsp"]
    pos, q, obs = case_inputs("p3_npsp")
    cfg, box, src, ob, prm = objects(fp, case, pos, q, obs)
    with pytest.raises((ValueError, fp.ValidationError)):
        fp.build_sweep_plan(cfg, box, src, ob, prm, 0, [0.1, 0.2])   # NPSP: nothing to sweep
    case = SMALL_CASES["p1_dyn"]
    pos, q, obs = case_inputs("p1_dyn")
    cfg, box, src, ob, prm = objects(fp, case, pos, q, obs)
    with pytest.raises(ValueError):
        fp.build_sweep_plan(cfg, box, src, ob, prm, 1, [0.1])      # y is not periodic in 1D
    with pytest.raises(ValueError):
        fp.build_sweep_plan(cfg, box, src, ob, prm, 0, np.zeros(65))


def test_sweep_c5_subset(fp):
    """C5 at full scale: five excitations in one sweep; excitations 0, 31 and 63
    against the reference's own runs on the seeded observer sample
    (tests/golden/make_subset_golden.py 5 5:31 5:63), two against independent
    plans."""
    from paper_2312_02376_b200.workloads import CONFIGS, c5_kshift, make_inputs
    g = golden("c5_subset.npz")
    w = CONFIGS[5]
    pos, qall = make_inputs(5)
    es = [0, 17, 31, 40, 63]
    Q = np.ascontiguousarray(qall[es])
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity(w.dim), L=w.L, k0=w.k0, kshift=c5_kshift(0),
                               regime=fp.Regime(w.regime))
    sw = fp.build_sweep_plan(cfg, fp.TargetBox(w.D), fp.SourcePointSet(pos, Q[0]), fp.ObserverPointSet(pos),
                             fp.SolverParams(**w.params()), 0, [c5_kshift(e)[0] for e in es])
    U = sw.evaluate(Q)
    sel = g["obs_index"]
    assert rel_l2(U[0][sel], g["u"]) <= 1e-10
    for j, e in ((2, 31), (4, 63)):
        ge = golden(f"c5_subset_e{e}.npz")
        assert int(ge["excitation"]) == e
        assert rel_l2(U[j][ge["obs_index"]], ge["u"]) <= 1e-10
    del sw
    for j in (1, 3):
        cfg_e = fp.PeriodicityConfig(dim=fp.Periodicity(w.dim), L=w.L, k0=w.k0, kshift=c5_kshift(es[j]),
                                     regime=fp.Regime(w.regime))
        plan = fp.build_plan(cfg_e, fp.TargetBox(w.D), fp.SourcePointSet(pos, Q[j]), fp.ObserverPointSet(pos),
                             fp.SolverParams(**w.params()))
        assert rel_l2(U[j], plan.evaluate(Q[j])) <= 1e-12
        del plan


def test_sweep_source_ordered_rows(fp, monkeypatch):
    """Sweep plans with rows in source order (the default for large pair lists;
    the phase components are permuted with the rows): same potentials to 1e-13."""
    name = "p2_dyn"
    case = SMALL_CASES[name]
    pos, q, obs = case_inputs(name)
    shifts = [complex(case["kshift"][0]) + 0.07 * e for e in range(12)]
    rng = np.random.default_rng(12)
    Q = rng.normal(size=(len(shifts), q.size)) + 1j * rng.normal(size=(len(shifts), q.size))
    cfg, box, src, ob, prm = objects(fp, case, pos, q, obs)
    u0 = fp.build_sweep_plan(cfg, box, src, ob, prm, 0, shifts).evaluate(Q)
    monkeypatch.setenv("FFTPIM_K4_SORT", "1")
    sw = fp.build_sweep_plan(cfg, box, src, ob, prm, 0, shifts)
    assert sw.info.pair_rows_source_order == 1
    u1 = sw.evaluate(Q)
    assert rel_l2(u1, u0) <= 1e-13
    np.testing.assert_array_equal(sw.evaluate(Q), u1)


def test_sweep_device_and_host_entries_agree(fp):
    """The device entry (caller stream, tensors) and the host entry (chunked
    uploads overlapping the chains) give bitwise identical potentials, and
    repeated sweeps are bitwise reproducible (fixed-order reductions only)."""
    import torch
    name = "p2_dyn"
    case = SMALL_CASES[name]
    pos, q, obs = case_inputs(name)
    shifts = [complex(case["kshift"][0]) + 0.1 * e for e in range(40)]   # E > 32: two excitations per lane
    rng = np.random.default_rng(9)
    Q = rng.normal(size=(len(shifts), q.size)) + 1j * rng.normal(size=(len(shifts), q.size))
    cfg, box, src, ob, prm = objects(fp, case, pos, q, obs)
    sw = fp.build_sweep_plan(cfg, box, src, ob, prm, 0, shifts)
    u_host = sw.evaluate(Q)
    u_pin = torch.empty(u_host.shape, dtype=torch.complex128).pin_memory()
    q_pin = torch.from_numpy(Q).pin_memory()
    sw.evaluate(q_pin.numpy(), out=u_pin.numpy())
    u_dev = sw.evaluate(torch.from_numpy(Q).cuda()).cpu().numpy()
    assert np.array_equal(u_host, u_dev)
    assert np.array_equal(u_host, u_pin.numpy())
    assert np.array_equal(u_dev, sw.evaluate(torch.from_numpy(Q).cuda()).cpu().numpy())
    with pytest.raises(ValueError):
        sw.evaluate(Q[:3])
