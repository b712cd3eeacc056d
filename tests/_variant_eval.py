"""Subprocess helper for tests/test_gpu_paths.py: build one case under the
current environment (which selects the K1 / FFT variant), evaluate it and
save u; print the plan's path selection as one JSON line.

    python tests/_variant_eval.py <case> <out.npy>
case: c1 | c2 (bench workloads), blobs3d (clustered 3D, crowded cells), or a
tests/golden/cases.py SMALL_CASES name.
"""
import json
import os
import sys
import warnings

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(HERE, "golden"))

import numpy as np  # noqa: E402


def blobs3d():
    rng = np.random.default_rng(77)
    centres = rng.uniform(0.1, 0.9, (8, 3))
    pos = (centres[:, None, :] + rng.normal(0.0, 0.05, (8, 4000, 3))).reshape(-1, 3) % 1.0
    q = rng.normal(size=pos.shape[0]) - 0.0
    q -= q.mean()
    return pos, q.astype(np.complex128)


def main():
    case, out = sys.argv[1], sys.argv[2]
    import paper_2312_02376_b200 as fp
    if case in ("c1", "c2"):
        from paper_2312_02376_b200.workloads import CONFIGS, make_inputs
        c = int(case[1])
        w = CONFIGS[c]
        pos, q = make_inputs(c)
        cfg = fp.PeriodicityConfig(dim=fp.Periodicity(w.dim), L=w.L, k0=w.k0, kshift=w.kshift,
                                   regime=fp.Regime(w.regime))
        box, obs, prm = fp.TargetBox(w.D), pos, fp.SolverParams(**w.params())
    elif case == "blobs3d":
        pos, q = blobs3d()
        cfg = fp.PeriodicityConfig(dim=fp.Periodicity(3), L=(1, 1, 1), k0=0, kshift=(0, 0, 0),
                                   regime=fp.Regime("npsp"))
        box, obs = fp.TargetBox((1, 1, 1)), pos
        prm = fp.SolverParams(near_grid=(20, 20, 20), near_order=3, far_grid=(6, 6, 6))
    elif case == "tri":
        # doubled dims 96, 384, 24: the L = 3 * 2^k register FFTs (96, 384) and a Stockham axis
        rng = np.random.default_rng(31)
        pos = rng.uniform(0.0, 1.0, (3000, 3)) * np.array([1.0, 1.0, 0.25])
        q = rng.standard_normal(3000) + 1j * rng.standard_normal(3000)
        cfg = fp.PeriodicityConfig(dim=fp.Periodicity(2), L=(1, 1, 1), k0=1.5 * np.pi - 0.2j,
                                   kshift=(0.3, 0.1, 0), regime=fp.Regime("dynamic"))
        box, obs = fp.TargetBox((1, 1, 0.25)), pos
        prm = fp.SolverParams(near_grid=(48, 192, 12), near_order=3, far_grid=(6, 6, 4))
    elif case == "g256":
        # 256^3 grid: L = 512 on every axis (z, y forward stages, fused x stage, inverses)
        rng = np.random.default_rng(256)
        pos = rng.uniform(0.0, 1.0, (20000, 3))
        q = rng.standard_normal(20000) + 1j * rng.standard_normal(20000)
        cfg = fp.PeriodicityConfig(dim=fp.Periodicity(3), L=(1, 1, 1), k0=2.0 * np.pi,
                                   kshift=(0.2 * np.pi, 0.1 * np.pi, 0), regime=fp.Regime("dynamic"))
        box, obs = fp.TargetBox((1, 1, 1)), pos
        prm = fp.SolverParams(near_grid=(256, 256, 256), near_order=3, far_grid=(6, 6, 6))
    else:
        from cases import SMALL_CASES, case_inputs, regime_of
        d = SMALL_CASES[case]
        pos, q, obs = case_inputs(case)
        obs = pos if obs is None else obs
        cfg = fp.PeriodicityConfig(dim=fp.Periodicity(d["dim"]), L=d["L"], k0=d["k0"], kshift=d["kshift"],
                                   regime=fp.Regime(regime_of(d)))
        box, prm = fp.TargetBox(d["D"]), fp.SolverParams(**d["params"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        plan = fp.build_plan(cfg, box, fp.SourcePointSet(pos, q), fp.ObserverPointSet(obs), prm)
    u = plan.evaluate(q)
    np.save(out, u)
    info = plan.native.info
    print(json.dumps({"k1_ell": bool(info.k1_operator), "custom_fft": bool(info.custom_fft),
                      "k1_slots": int(info.k1_slots)}))


if __name__ == "__main__":
    main()
