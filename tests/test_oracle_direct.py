"""The oracle's restatement of the reference's brute-force sums
(oracle/direct.py <- oracle.py:62-123) pinned to the reference's own outputs
(tests/golden/direct_cases.npz, made by tests/golden/make_direct_golden.py)."""
import numpy as np
import pytest

from conftest import golden, rel_l2
from oracle.direct import direct, free_space
from oracle.problem import make_problem

D = golden("direct_cases.npz")
NAMES = [str(n) for n in D["names"]]
REASON = {"separation": 1, "not converged": 2}


def case(name):
    return {k.split("__", 1)[1]: D[k] for k in D.files if k.startswith(name + "__")}


def problem(c):
    return make_problem(int(c["dim"]), L=tuple(c["L"]), k0=complex(c["k0"]), kshift=tuple(c["kshift"]),
                        regime=str(c["regime"]))


@pytest.mark.parametrize("name", NAMES)
def test_oracle_direct_matches_reference(name):
    c = case(name)
    if str(c["mode"]) == "free":
        u = free_space(complex(c["k0"]), c["src"], c["q"], c["obs"])
        assert rel_l2(u, c["u"]) <= 1e-14
        return
    i_d = int(c["i_d"]) if str(c["mode"]) == "far" else None
    u, worst, fails = direct(problem(c), c["src"], c["q"], c["obs"], i_d=i_d, tol=float(c["tol"]),
                             max_terms=int(c["max_terms"]), consecutive=int(c["consecutive"]))
    assert rel_l2(u, c["u"]) <= 1e-13
    assert worst == int(c["worst"])
    got = np.array([(i, j, REASON[r]) for i, j, r in fails], dtype=np.int64).reshape(-1, 3)
    assert np.array_equal(got, c["failures"])


def test_free_space_coincident_raises():
    p = np.random.default_rng(0).uniform(size=(5, 3))
    with pytest.raises(ZeroDivisionError):
        free_space(1.0, p, np.ones(5), p)


@pytest.mark.parametrize("key", ["c0", "c1", "c2"])
def test_oracle_near_only_id0_matches_reference(key):
    """build_near_plan with i_d = 0 (cli.py:343-347 free-space baseline): no
    wrapped copies, unclipped join radius, free-space near kernel."""
    from oracle.near_engine import build_near, eval_near
    g = golden("near_id0.npz")
    c = {k.split("__", 1)[1]: g[k] for k in g.files if k.startswith(key + "__")}
    pb = make_problem(int(c["dim"]), k0=complex(c["k0"]), kshift=tuple(c["kshift"]), regime=str(c["regime"]),
                      i_d=0, near_grid=(10, 10, 10), near_order=3)
    plan = build_near(pb, c["pos"], c["pos"])
    assert plan.pair_obs.size == int(c["n_pairs"])
    assert rel_l2(eval_near(plan, c["q"]), c["u"]) <= 1e-12
