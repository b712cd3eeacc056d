"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py [--full]

Writes (all committed, all small):
  reference_constants.json  frozen 50-digit values the reference's own tests pin
                            (test_special.py HANKEL2_REFS / BESSELK0_REFS,
                            test_pgf.py spectral/lattice references), read by
                            importing those test modules -- plus the points and
                            configurations they belong to.
  small_<case>.npz          reference outputs for tests/golden/cases.py: potentials
                            u = build_plan(...).evaluate(q), pair-set digests, pair
                            counts, coefficient checksums, far kernel table.
  c1_full.npz / c2_full.npz (with --full) reference potentials at BASELINE configs
                            C1 (N=4096) and C2 (N=65536) on the seeded inputs of
                            paper_2312_02376_b200/workloads.py.

Nothing at run time (GPU box, bench, smoke) reads /root/reference.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

import perisum as P  # noqa: E402  (the reference)

from cases import SMALL_CASES, case_inputs, regime_of  # noqa: E402


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def ref_config(dim, L, k0, kshift, regime):
    return P.PeriodicityConfig(dim=P.Periodicity(dim), L=tuple(L), k0=complex(k0),
                               kshift=tuple(complex(k) for k in kshift), regime=P.Regime(regime))


def constants():
    import test_pgf as TP
    import test_special as TS
    bench_dyn = dict(L=(1.0, 1.0, 1.0), k0=[TP.BENCH_K0.real, TP.BENCH_K0.imag],
                     kshift=[[k.real, k.imag] for k in TP.BENCH_KSHIFT], point=list(TP.BENCH_POINT))
    cz = lambda c: [c.real, c.imag]  # noqa: E731
    out = {
        "hankel2_0": [[cz(z), cz(v)] for z, v in TS.HANKEL2_REFS],
        "bessel_k0": [[cz(z), cz(v)] for z, v in TS.BESSELK0_REFS],
        "series_tol": 1e-12,
        "series": [
            dict(kind="spectral", dim=1, regime="dynamic", value=cz(TP.SPECTRAL_1D_REF), **bench_dyn),
            dict(kind="spectral", dim=2, regime="dynamic", value=cz(TP.SPECTRAL_2D_REF), **bench_dyn),
            dict(kind="spectral", dim=3, regime="dynamic", value=cz(TP.SPECTRAL_3D_REF), **bench_dyn),
            dict(kind="lattice", dim=1, regime="npsp", value=cz(TP.LATTICE_1D_REF), L=(1.0, 1.0, 1.0),
                 k0=[0, 0], kshift=[[0, 0]] * 3, point=list(TP.BENCH_POINT)),
            dict(kind="lattice", dim=2, regime="npsp", value=cz(TP.LATTICE_2D_REF), L=(1.0, 1.0, 1.0),
                 k0=[0, 0], kshift=[[0, 0]] * 3, point=list(TP.BENCH_POINT)),
            dict(kind="lattice", dim=3, regime="npsp", value=cz(TP.LATTICE_3D_REF), L=(1.0, 1.0, 1.0),
                 k0=[0, 0], kshift=[[0, 0]] * 3, point=list(TP.BENCH_POINT)),
            # generic points (test_pgf.py:105-111, :197-200)
            dict(kind="lattice", dim=1, regime="npsp", value=cz(TP.LATTICE_1D_GEN), L=(2.6, 1.0, 1.0),
                 k0=[0, 0], kshift=[[0, 0]] * 3, point=[0.37, 0.21, -0.4]),
            dict(kind="spectral", dim=1, regime="dynamic", value=cz(TP.SPECTRAL_1D_GEN), L=(1.4, 1.0, 1.0),
                 k0=[2.0, -0.7], kshift=[[0.4, 0], [0, 0], [0, 0]], point=[0.3, 0.25, -0.15]),
            dict(kind="spectral", dim=2, regime="dynamic", value=cz(TP.SPECTRAL_2D_GEN), L=(1.2, 0.9, 1.0),
                 k0=[1.1, -0.6], kshift=[[0.3, 0], [-0.2, 0], [0, 0]], point=[0.3, 0.45, 0.35]),
        ],
    }
    with open(os.path.join(HERE, "reference_constants.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote reference_constants.json")


def run_reference(dim, L, D, k0, kshift, regime, params, pos, q, obs=None):
    cfg = ref_config(dim, L, k0, kshift, regime)
    box = P.TargetBox(tuple(D))
    src = P.SourcePointSet(pos, q)
    ob = P.ObserverPointSet(pos if obs is None else obs)
    prm = P.SolverParams(**params)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        t0 = time.perf_counter()
        plan = P.build_plan(cfg, box, src, ob, prm)
        tb = time.perf_counter() - t0
    t0 = time.perf_counter()
    u = plan.evaluate(q)
    te = time.perf_counter() - t0
    n = plan.near
    return dict(
        u=u,
        u_near=P.eval_near(n, q), u_far=P.eval_far(plan.far, q),
        n_pairs=np.int64(n.pair_obs.size), n_self=np.int64(n.n_self_pairs), n_wrap=np.int64(n.n_wrapped_pairs),
        pair_digest=np.array(digest(n.pair_obs, n.pair_src, n.pair_code)),
        pair_src_sum=np.int64(n.pair_src.astype(np.int64).sum()),
        coef_sum=n.pair_coef.sum(), coef_abs_sum=np.abs(n.pair_coef).sum(),
        near_dims=np.array(n.grid.dims), join_radius=np.array(n.join_radius),
        coincident_terms=np.int64(n.coincident_kernel_terms),
        far_kernel=plan.far.kernel, far_terms=np.int64(plan.far.kernel_terms),
        build_seconds=np.float64(tb), eval_seconds=np.float64(te),
    )


def small_cases(only=None):
    for name, case in SMALL_CASES.items():
        if only and name not in only:
            continue
        pos, q, obs = case_inputs(name)
        res = run_reference(case["dim"], case["L"], case["D"], case["k0"], case["kshift"],
                            regime_of(case), case["params"], pos, q, obs)
        np.savez_compressed(os.path.join(HERE, f"small_{name}.npz"), **res)
        print(f"{name}: pairs={int(res['n_pairs'])} terms={int(res['far_terms'])} "
              f"build={float(res['build_seconds']):.1f}s")


def full_cases(which):
    from paper_2312_02376_b200.workloads import CONFIGS, make_inputs
    for c in which:
        w = CONFIGS[c]
        pos, q = make_inputs(c)
        res = run_reference(w.dim, w.L, w.D, w.k0, w.kshift, w.regime, w.params(), pos, q)
        keep = {k: res[k] for k in ("u", "n_pairs", "n_self", "n_wrap", "pair_digest", "pair_src_sum",
                                    "coef_sum", "coef_abs_sum", "far_kernel", "far_terms",
                                    "build_seconds", "eval_seconds", "near_dims", "join_radius")}
        np.savez_compressed(os.path.join(HERE, f"c{c}_full.npz"), **keep)
        print(f"C{c}: pairs={int(res['n_pairs'])} build={float(res['build_seconds']):.1f}s "
              f"eval={float(res['eval_seconds']):.3f}s")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", type=int, nargs="*", default=None, help="BASELINE configs to run in full (1 2)")
    ap.add_argument("--only", nargs="*", default=None)
    ap.add_argument("--skip-small", action="store_true")
    a = ap.parse_args()
    constants()
    if not a.skip_small:
        small_cases(a.only)
    if a.full is not None:
        full_cases(a.full or [1, 2])
