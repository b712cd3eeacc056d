"""Subset-observer golden fixtures for the BASELINE configs whose full reference
plan cannot be built on a host (C3, C4, C5 -- 35-221 GB of correction pairs,
SURVEY.md 8c).

The REFERENCE is run from a temporary copy of /root/reference/pkg/src/perisum
(outside the repo; nothing is committed) with the one-line subset-observer
patch SURVEY.md 8c describes: observers are a seeded sample of the sources and
a pair is a self pair iff obs_to_src[observer] == source and the image code is
zero (nearzone.py:407-409).  On such observers this is bitwise identical to the
full run (measured in the survey at N=3000).  Full-scale sources, grid, FFT and
far kernel are used; only the observer set is sampled.

    python tests/golden/make_subset_golden.py 3 5      # ~10 min each, ~9 GB RAM
    python tests/golden/make_subset_golden.py 4        # ~15 min, ~60 GB RAM
    python tests/golden/make_subset_golden.py 5:31 5:63   # C5 excitations 31 and 63

Writes tests/golden/c<c>_subset.npz (C5 excitation e > 0: c5_subset_e<e>.npz):
observer indices, u at those observers, pair counts and the far kernel table.
"""
from __future__ import annotations

import os
import shutil
import sys
import tempfile
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

SUBSET = {3: 2048, 4: 4096, 5: 4096}

PATCH_FROM = "            selfish = (p_obs == p_src) & (p_code == 0).all(axis=1)"
PATCH_TO = ("            selfish = (_OBS_TO_SRC[p_obs] == p_src) & (p_code == 0).all(axis=1)"
            " if _OBS_TO_SRC is not None else (p_obs == p_src) & (p_code == 0).all(axis=1)")


def patched_reference():
    tmp = tempfile.mkdtemp(prefix="perisum_subset_")
    shutil.copytree("/root/reference/pkg/src/perisum", os.path.join(tmp, "perisum"))
    path = os.path.join(tmp, "perisum", "nearzone.py")
    src = open(path).read()
    assert PATCH_FROM in src, "reference changed: subset patch anchor not found"
    src = src.replace("        if same_points:\n" + PATCH_FROM, "        if same_points or _OBS_TO_SRC is not None:\n" + PATCH_TO)
    src = src.replace("_PAIR_CHUNK = 16384", "_PAIR_CHUNK = 16384\n_OBS_TO_SRC = None")
    open(path, "w").write(src)
    sys.path.insert(0, tmp)
    import perisum
    return perisum, tmp


def main(configs):
    from paper_2312_02376_b200.workloads import CONFIGS, c5_kshift, make_inputs
    P, tmp = patched_reference()
    import perisum.nearzone as NZ
    try:
        for spec in configs:
            c, e = (int(v) for v in spec.split(":")) if ":" in spec else (int(spec), 0)
            w = CONFIGS[c]
            pos, q = make_inputs(c)
            kshift = w.kshift
            if c == 5:
                q = q[e]
                kshift = c5_kshift(e)
            idx = np.sort(np.random.default_rng(100 + c).choice(len(pos), SUBSET[c], replace=False))
            NZ._OBS_TO_SRC = idx
            cfg = P.PeriodicityConfig(dim=P.Periodicity(w.dim), L=w.L, k0=w.k0, kshift=kshift,
                                      regime=P.Regime(w.regime))
            t0 = time.perf_counter()
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                plan = P.build_plan(cfg, P.TargetBox(w.D), P.SourcePointSet(pos, q),
                                    P.ObserverPointSet(pos[idx]), P.SolverParams(**w.params()))
            tb = time.perf_counter() - t0
            t0 = time.perf_counter()
            u = plan.evaluate(q)
            te = time.perf_counter() - t0
            n = plan.near
            name = f"c{c}_subset.npz" if e == 0 else f"c{c}_subset_e{e}.npz"
            np.savez_compressed(os.path.join(HERE, name), obs_index=idx, u=u, excitation=np.int64(e),
                                n_pairs=np.int64(n.pair_obs.size), n_self=np.int64(n.n_self_pairs),
                                n_wrap=np.int64(n.n_wrapped_pairs), far_kernel=plan.far.kernel,
                                far_terms=np.int64(plan.far.kernel_terms), kshift=np.array(kshift),
                                build_seconds=np.float64(tb), eval_seconds=np.float64(te))
            print(f"C{c}: {len(idx)} observers, pairs={n.pair_obs.size}, build {tb:.0f}s, eval {te:.1f}s", flush=True)
    finally:
        NZ._OBS_TO_SRC = None
        shutil.rmtree(tmp, ignore_errors=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["3", "5"])
