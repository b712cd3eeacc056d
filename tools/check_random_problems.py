"""CPU pre-check of tests/random_problems.py: every draw passes this repo's host
validation and builds / evaluates in the oracle (no GPU needed).
    python tools/check_random_problems.py"""
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import random_problems as rp  # noqa: E402
from oracle.pipeline import build_plan  # noqa: E402
from oracle.problem import make_problem  # noqa: E402
from paper_2312_02376_b200 import problem as P  # noqa: E402

for seed in range(rp.N_DRAWS):
    d = rp.draw(seed)
    cfg = P.PeriodicityConfig(dim=P.Periodicity(d["dim"]), L=d["L"], k0=d["k0"], kshift=d["kshift"],
                              regime=P.Regime(d["regime"]))
    obs = d["src"] if d["obs"] is None else d["obs"]
    rep = P.validate_problem(cfg, P.TargetBox(d["D"]), P.SourcePointSet(d["src"], d["q"]), P.ObserverPointSet(obs),
                             P.SolverParams(**d["params"]))
    t0 = time.perf_counter()
    pb = make_problem(d["dim"], L=d["L"], D=d["D"], k0=d["k0"], kshift=d["kshift"], regime=d["regime"], **d["params"])
    try:
        plan = build_plan(pb, d["src"], d["obs"])
        u = plan.evaluate(d["q"])
        status = f"pairs {plan.near.pair_obs.size} |u| {np.abs(u).max():.3g}"
    except Exception as e:  # noqa: BLE001
        status = f"ORACLE {type(e).__name__}: {e}"
    print(seed, d["dim"], d["regime"], d["k0"], d["params"]["near_grid"], "o", d["params"]["near_order"], "id", d["params"]["i_d"],
          "n", len(d["src"]), "m", None if d["obs"] is None else len(d["obs"]), "D", tuple(round(x, 2) for x in d["D"]),
          "valid" if rep.ok() else list(rep.messages), status, f"{time.perf_counter() - t0:.1f}s")
