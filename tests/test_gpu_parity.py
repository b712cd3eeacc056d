"""CUDA path vs the reference (golden fixtures made by running it) and vs the
CPU oracle, through the C ABI.  Bar: relative L2 <= 1e-10 in fp64 on the
potentials (BASELINE.json north star), identical correction-pair sets."""
import hashlib

import numpy as np
import pytest

from conftest import golden, rel_l2
from cases import SMALL_CASES, case_inputs, regime_of

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module")
def fp():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2312_02376_b200 as fp
    fp._native.load()
    return fp


def ref_objects(fp, case, pos, q, obs):
    import numpy as np
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity(case["dim"]), L=case["L"], k0=case["k0"],
                               kshift=case["kshift"], regime=fp.Regime(regime_of(case)))
    box = fp.TargetBox(case["D"])
    src = fp.SourcePointSet(pos, q)
    ob = fp.ObserverPointSet(pos if obs is None else obs)
    return cfg, box, src, ob, fp.SolverParams(**case["params"])


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", list(SMALL_CASES))
def test_small_case_parity(fp, name):
    case = SMALL_CASES[name]
    g = golden(f"small_{name}.npz")
    pos, q, obs = case_inputs(name)
    cfg, box, src, ob, prm = ref_objects(fp, case, pos, q, obs)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        plan = fp.build_plan(cfg, box, src, ob, prm)
    near = plan.near
    # identical correction-pair set, order and bookkeeping (nearzone.py:303-487)
    assert near.pair_obs.size == int(g["n_pairs"])
    assert digest(near.pair_obs, near.pair_src, near.pair_code) == str(g["pair_digest"])
    assert near.n_self_pairs == int(g["n_self"]) and near.n_wrapped_pairs == int(g["n_wrap"])
    assert near.coincident_kernel_terms == int(g["coincident_terms"])
    assert tuple(near.grid.dims) == tuple(g["near_dims"])
    assert tuple(near.join_radius) == tuple(g["join_radius"])
    # coefficients
    assert abs(near.pair_coef.sum() - complex(g["coef_sum"])) <= 1e-11 * float(g["coef_abs_sum"])
    # far kernel table (same truncation layer by layer, pgf.py:166-195)
    assert plan.far.kernel_terms == int(g["far_terms"])
    assert rel_l2(plan.far.kernel, g["far_kernel"]) <= 1e-11
    # potentials: full, near-only, far-only
    assert rel_l2(plan.evaluate(q), g["u"]) <= TOL
    assert rel_l2(fp.eval_near(plan.near, q), g["u_near"]) <= TOL
    assert rel_l2(fp.eval_far(plan.far, q), g["u_far"]) <= TOL


@pytest.mark.parametrize("k1,obs,far", [("lines", "pos", "warps"), ("lines_smem", "tile", "win")])
@pytest.mark.parametrize("name", list(SMALL_CASES))
def test_small_case_parity_point_paths(fp, name, k1, obs, far, monkeypatch):
    """The large-N evaluation paths forced on every small case: K1 as a line
    sweep (line_kernels.cu: plan stencil records, or stencils computed from the
    sorted positions) and the observer pass computing its stencils from the
    sorted positions (gathering from global memory, or from shared-memory grid
    tiles), and the far projection on per-chunk windows.  Same potentials as the reference (1e-10) and as the
    default small-N paths (ELL K1, stored-weight observer pass) to 1e-13."""
    case = SMALL_CASES[name]
    g = golden(f"small_{name}.npz")
    pos, q, obs = case_inputs(name)
    cfg, box, src, ob, prm = ref_objects(fp, case, pos, q, obs)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        base = fp.build_plan(cfg, box, src, ob, prm)
        monkeypatch.setenv("FFTPIM_K1", k1)
        monkeypatch.setenv("FFTPIM_OBS", obs)
        monkeypatch.setenv("FFTPIM_FAR", far)
        plan = fp.build_plan(cfg, box, src, ob, prm)
    u = plan.evaluate(q)
    assert rel_l2(u, g["u"]) <= TOL
    assert rel_l2(u, base.evaluate(q)) <= 1e-13
    assert rel_l2(fp.eval_near(plan.near, q), g["u_near"]) <= TOL
    assert rel_l2(fp.eval_far(plan.far, q), g["u_far"]) <= TOL
    np.testing.assert_array_equal(plan.evaluate(q), u)   # bitwise reproducible


@pytest.mark.parametrize("name", list(SMALL_CASES))
def test_source_ordered_pair_rows(fp, name, monkeypatch):
    """Rows stored in source order (the default for large pair lists, K4 gather
    locality): the same (observer, source, image code, coefficient) set as the
    reference-order plan, the same potentials to 1e-13, bitwise reproducible."""
    case = SMALL_CASES[name]
    pos, q, obs = case_inputs(name)
    cfg, box, src, ob, prm = ref_objects(fp, case, pos, q, obs)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        base = fp.build_plan(cfg, box, src, ob, prm)
        monkeypatch.setenv("FFTPIM_K4_SORT", "1")
        plan = fp.build_plan(cfg, box, src, ob, prm)
    assert plan.native.info.pair_rows_source_order == 1 and base.native.info.pair_rows_source_order == 0

    def rows(p):
        n = p.near
        code = n.pair_code.astype(np.int64)
        key = np.lexsort((code[:, 2], code[:, 1], code[:, 0], n.pair_src, n.pair_obs))
        return n.pair_obs[key], n.pair_src[key], n.pair_code[key], n.pair_coef[key]

    for a, b in zip(rows(plan), rows(base)):
        np.testing.assert_array_equal(a, b)
    u = plan.evaluate(q)
    assert rel_l2(u, base.evaluate(q)) <= 1e-13
    np.testing.assert_array_equal(plan.evaluate(q), u)


@pytest.mark.parametrize("name", list(SMALL_CASES))
@pytest.mark.parametrize("sort,kernel", [("1", "bulk"), ("0", "bulk"), ("1", "ldg"), ("0", "ldg")])
def test_run_encoded_pair_stream(fp, name, sort, kernel, monkeypatch):
    """K4 with run-encoded sources (opt-in, FFTPIM_K4_RUNS=1), streamed with bulk
    asynchronous copies into shared memory (cp.async.bulk + mbarrier) or with
    per-thread loads: same pairs, order and arithmetic as the int32-index
    kernel, so the potentials are bit-identical; with rows in discovery order
    (sort = 0) tiles hold more than 64 runs and the overflow-bias path runs.
    A plan that dropped its index array exports the same pairs (decoded runs)."""
    monkeypatch.setenv("FFTPIM_K4_RUNS_KERNEL", kernel)
    case = SMALL_CASES[name]
    pos, q, obs = case_inputs(name)
    cfg, box, src, ob, prm = ref_objects(fp, case, pos, q, obs)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        monkeypatch.setenv("FFTPIM_K4_SORT", sort)
        monkeypatch.setenv("FFTPIM_K4_RUNS", "0")
        base = fp.build_plan(cfg, box, src, ob, prm)
        monkeypatch.setenv("FFTPIM_K4_RUNS", "1")
        monkeypatch.setenv("FFTPIM_K4_DROP_SRC", "1")
        plan = fp.build_plan(cfg, box, src, ob, prm)
    assert base.native.info.k4_runs == -1
    n_pairs = plan.native.info.n_pairs
    if n_pairs == 0:
        assert plan.native.info.k4_runs == -1
        return
    assert 0 < plan.native.info.k4_runs <= n_pairs + 3 * ((n_pairs + 255) // 256)
    u = plan.evaluate(q)
    np.testing.assert_array_equal(u, base.evaluate(q))
    np.testing.assert_array_equal(plan.evaluate(q), u)
    np.testing.assert_array_equal(fp.eval_near(plan.near, q), fp.eval_near(base.near, q))
    for a, b in ((plan.near.pair_obs, base.near.pair_obs), (plan.near.pair_src, base.near.pair_src),
                 (plan.near.pair_coef, base.near.pair_coef)):
        np.testing.assert_array_equal(a, b)
    g = golden(f"small_{name}.npz")
    assert rel_l2(u, g["u"]) <= TOL


def _full(fp, c):
    from paper_2312_02376_b200.workloads import CONFIGS, make_inputs
    w = CONFIGS[c]
    pos, q = make_inputs(c)
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity(w.dim), L=w.L, k0=w.k0, kshift=w.kshift,
                               regime=fp.Regime(w.regime))
    plan = fp.build_plan(cfg, fp.TargetBox(w.D), fp.SourcePointSet(pos, q), fp.ObserverPointSet(pos),
                         fp.SolverParams(**w.params()))
    return plan, q


@pytest.mark.parametrize("c", [1, 2])
def test_baseline_config_parity(fp, c):
    """C1 (3D NPSP, N=4096) and C2 (1D Helmholtz, N=65536) against the reference's
    own output on the seeded inputs."""
    g = golden(f"c{c}_full.npz")
    plan, q = _full(fp, c)
    assert plan.near.pair_obs.size == int(g["n_pairs"])
    assert digest(plan.near.pair_obs, plan.near.pair_src, plan.near.pair_code) == str(g["pair_digest"])
    assert plan.far.kernel_terms == int(g["far_terms"])
    assert rel_l2(plan.far.kernel, g["far_kernel"]) <= 1e-11
    assert rel_l2(plan.evaluate(q), g["u"]) <= TOL


def test_device_path_matches_host_and_is_deterministic(fp):
    import torch
    plan, q = _full(fp, 1)
    u_host = plan.evaluate(q)
    qd = torch.from_numpy(q).cuda()
    u1 = plan.evaluate(qd)
    u2 = plan.evaluate(qd)
    torch.cuda.synchronize()
    assert torch.equal(u1, u2)                      # fixed reduction order: bitwise repeatable
    assert np.array_equal(u1.cpu().numpy(), u_host)


def test_batch_and_linearity(fp):
    plan, q = _full(fp, 2)
    rng = np.random.default_rng(5)
    q2 = rng.standard_normal(q.size) + 1j * rng.standard_normal(q.size)
    ub = plan.evaluate(np.stack([q, q2, 2.0 * q - 3j * q2]))
    assert rel_l2(ub[2], 2.0 * ub[0] - 3j * ub[1]) <= 1e-12
    assert np.array_equal(ub[0], plan.evaluate(q))


@pytest.mark.parametrize("B", [12, 70])
def test_multi_rhs_batch_matches_single_evaluations(fp, B):
    """Batches of >= 8 charge vectors stream the correction pairs once per 64
    right-hand sides (batched K4 + per-vector chains); every row equals the
    single-vector evaluation to rounding, both through the host and device entry."""
    import torch
    plan, q = _full(fp, 2)
    rng = np.random.default_rng(B)
    Q = rng.standard_normal((B, q.size)) + 1j * rng.standard_normal((B, q.size))
    U = plan.evaluate(Q)
    for b in (0, 5, B - 1):
        assert rel_l2(U[b], plan.evaluate(Q[b])) <= 1e-13, b
    Ud = plan.evaluate(torch.from_numpy(Q).cuda()).cpu().numpy()
    assert np.array_equal(U, Ud)
    q_pin = torch.from_numpy(Q).pin_memory()            # host graph with pinned buffers
    u_pin = torch.empty(Q.shape, dtype=torch.complex128).pin_memory()
    plan.native.evaluate(q_pin.numpy(), out=u_pin.numpy())
    assert np.array_equal(U, u_pin.numpy())
    assert np.array_equal(U, plan.evaluate(Q))          # bitwise reproducible
    g = golden("c2_full.npz")
    Q[3] = q
    assert rel_l2(plan.evaluate(Q)[3], g["u"]) <= 1e-10


def test_concurrent_callers_on_one_plan(fp):
    """Two torch streams and two host threads evaluating one plan: the plan's
    evaluation guard orders them (shared work buffers), every result equals
    the sequential one bitwise (SPEC: concurrent evaluate with distinct q)."""
    import threading
    import torch
    plan, q = _full(fp, 2)
    rng = np.random.default_rng(11)
    qs = [rng.standard_normal(q.size) + 1j * rng.standard_normal(q.size) for _ in range(4)]
    ref = [plan.evaluate(x) for x in qs]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    qd = [torch.from_numpy(x).cuda() for x in qs]
    torch.cuda.synchronize()
    outs = []
    for k in range(4):
        with torch.cuda.stream(s1 if k % 2 == 0 else s2):
            outs.append(plan.evaluate(qd[k]))
    torch.cuda.synchronize()
    for k in range(4):
        assert np.array_equal(outs[k].cpu().numpy(), ref[k]), k
    res = {}

    def worker(k):
        for _ in range(3):
            res[k] = plan.evaluate(qs[k])

    th = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    for k in range(4):
        assert np.array_equal(res[k], ref[k]), k


def test_npsp_real_and_complex_charges(fp):
    """NPSP plans gather real charges as 8-byte values in K4 when every
    imaginary part is zero (a per-evaluation device flag); complex charges take
    the full path.  Both agree with linearity, batches mix the two, and the
    complex path of a real q (imag = tiny) stays within rounding of it."""
    plan, q = _full(fp, 1)
    q = np.ascontiguousarray(q.real + 0j)
    rng = np.random.default_rng(8)
    qi = rng.standard_normal(q.size)
    qi -= qi.mean()
    u_re, u_im = plan.evaluate(q), plan.evaluate(qi + 0j)
    u_c = plan.evaluate(q + 1j * qi)
    assert rel_l2(u_c, u_re + 1j * u_im) <= 1e-13
    ub = plan.evaluate(np.stack([q, q + 1j * qi, q]))
    assert np.array_equal(ub[0], u_re) and np.array_equal(ub[2], u_re)
    assert rel_l2(ub[1], u_c) <= 1e-15
    g = golden("c1_full.npz")
    assert rel_l2(u_re, g["u"]) <= 1e-10


def test_oracle_parity_random_cases(fp):
    """Fresh seeded instances (not in the golden set) against the CPU oracle."""
    from oracle.pipeline import build_plan as oracle_build
    from oracle.problem import make_problem
    rng = np.random.default_rng(77)
    for dim, k0, ks, D, grid, order in [
        (3, 0, (0, 0, 0), (1, 1, 1), (8, 8, 8), 3),
        (2, 2.0, (0.4, -0.3, 0), (1, 1, 0.6), (9, 9, 6), 2),
        (1, 1.0 - 0.2j, (0.1, 0, 0), (1, 0.5, 0.5), (10, 6, 6), 4),
    ]:
        n = 180
        pos = rng.uniform(0, 1, (n, 3)) * np.asarray(D)
        q = rng.standard_normal(n) + 0j
        if k0 == 0:
            q -= q.mean()
        else:
            q = q + 1j * rng.standard_normal(n)
        pb = make_problem(dim, D=D, k0=k0, kshift=ks, near_grid=grid, near_order=order, far_grid=(5, 5, 5))
        u_ref = oracle_build(pb, pos).evaluate(q)
        cfg = fp.PeriodicityConfig(dim=fp.Periodicity(dim), L=(1, 1, 1), k0=k0, kshift=ks,
                                   regime=fp.Regime(pb.regime))
        plan = fp.build_plan(cfg, fp.TargetBox(D), fp.SourcePointSet(pos, q), fp.ObserverPointSet(pos),
                             fp.SolverParams(near_grid=grid, near_order=order, far_grid=(5, 5, 5)))
        assert rel_l2(plan.evaluate(q), u_ref) <= TOL


def test_errors_map_to_reference_classes(fp):
    # a distinct source on top of an observer inside the correction region (nearzone.py:410-416)
    pos = np.random.default_rng(3).uniform(0, 1, (50, 3))
    obs = pos[:5].copy()
    q = np.ones(50, dtype=complex)
    q -= q.mean()
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity.P3D, L=(1, 1, 1))
    with pytest.raises(fp.DomainError):
        fp.build_plan(cfg, fp.TargetBox((1, 1, 1)), fp.SourcePointSet(pos, q), fp.ObserverPointSet(obs),
                      fp.SolverParams(near_grid=(8, 8, 8)))
    # exact Rayleigh-Wood anomaly: 2D, k0 = 1.5 pi, kx0 = pi/2 (hard part 5)
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity.P2D, L=(1, 1, 1), k0=1.5 * np.pi,
                               kshift=(np.pi / 2, 0, 0), regime=fp.Regime.DYNAMIC)
    p2 = np.random.default_rng(4).uniform(0, 1, (60, 3)) * np.array([1, 1, 0.25])
    with pytest.raises(fp.WoodAnomalyError):
        fp.build_plan(cfg, fp.TargetBox((1, 1, 0.25)), fp.SourcePointSet(p2, np.ones(60)),
                      fp.ObserverPointSet(p2), fp.SolverParams(near_grid=(8, 8, 4)))


@pytest.mark.parametrize("c", [5, 4, 3])
def test_baseline_config_subset_parity(fp, c):
    """C3/C4/C5 at full scale on the GPU against the reference run on a seeded
    observer sample (tests/golden/make_subset_golden.py)."""
    import os
    from conftest import GOLDEN
    from paper_2312_02376_b200.workloads import CONFIGS, c5_kshift, make_inputs
    path = os.path.join(GOLDEN, f"c{c}_subset.npz")
    if not os.path.exists(path):
        pytest.skip(f"no subset fixture for C{c}")
    g = np.load(path)
    w = CONFIGS[c]
    pos, q = make_inputs(c)
    kshift = w.kshift
    if c == 5:
        q, kshift = q[0], c5_kshift(0)
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity(w.dim), L=w.L, k0=w.k0, kshift=kshift,
                               regime=fp.Regime(w.regime))
    plan = fp.build_plan(cfg, fp.TargetBox(w.D), fp.SourcePointSet(pos, q), fp.ObserverPointSet(pos),
                         fp.SolverParams(**w.params()))
    assert plan.far.kernel_terms == int(g["far_terms"])
    assert rel_l2(plan.far.kernel, g["far_kernel"]) <= 1e-11
    u = plan.evaluate(q)
    assert rel_l2(u[g["obs_index"]], g["u"]) <= TOL
