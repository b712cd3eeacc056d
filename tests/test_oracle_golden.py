"""Pin the CPU oracle against the reference: its own frozen 50-digit values
and outputs of the reference itself (tests/golden, made by make_golden.py).
CPU only."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden, rel_l2
from cases import SMALL_CASES, case_inputs, regime_of
from oracle import bessel, lattice_sums
from oracle.pipeline import build_plan
from oracle.problem import make_problem

CONST = json.load(open(os.path.join(GOLDEN, "reference_constants.json")))


def cz(p):
    return complex(p[0], p[1])


@pytest.mark.parametrize("z,ref", [(cz(a), cz(b)) for a, b in CONST["hankel2_0"]])
def test_hankel2_frozen(z, ref):
    assert abs(bessel.h0(np.array([z]))[0] - ref) <= 1e-12 * abs(ref)


@pytest.mark.parametrize("w,ref", [(cz(a), cz(b)) for a, b in CONST["bessel_k0"]])
def test_k0_frozen(w, ref):
    assert abs(bessel.k0(np.array([w]))[0] - ref) <= 1e-12 * abs(ref)


def test_sqrt_branch():
    z = np.array([-4 + 0j, -4 - 0j, 4 + 0j, 1j, -1j, -3 + 4j, -3 - 4j])
    w = bessel.csqrt_lower(z)
    assert np.all(w.imag <= 0.0)
    assert np.allclose(w * w, z, rtol=1e-15, atol=0)


@pytest.mark.parametrize("case", CONST["series"], ids=lambda c: f"{c['kind']}{c['dim']}")
def test_series_frozen(case):
    pb = make_problem(case["dim"], L=case["L"], k0=cz(case["k0"]), kshift=[cz(k) for k in case["kshift"]],
                      regime=case["regime"])
    fn = lattice_sums.lattice if case["kind"] == "lattice" else lattice_sums.spectral
    vals, terms, conv = fn(np.array([case["point"]]), pb, CONST["series_tol"])
    ref = cz(case["value"])
    assert conv[0]
    assert abs(vals[0] - ref) <= 1e-11 * abs(ref)


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def problem_for(case):
    return make_problem(case["dim"], L=case["L"], D=case["D"], k0=case["k0"], kshift=case["kshift"],
                        regime=regime_of(case), **case["params"])


@pytest.mark.parametrize("name", list(SMALL_CASES))
def test_oracle_matches_reference_small(name):
    """Oracle == reference on every small golden case: same pair set (digest),
    same counts, far kernel and potentials to roundoff (observed: bitwise)."""
    case = SMALL_CASES[name]
    g = golden(f"small_{name}.npz")
    pos, q, obs = case_inputs(name)
    with pytest.warns(UserWarning) if case.get("axis") else _null():
        plan = build_plan(problem_for(case), pos, obs)
    nz = plan.near
    assert nz.pair_obs.size == int(g["n_pairs"])
    assert _digest(nz.pair_obs, nz.pair_src, nz.pair_code) == str(g["pair_digest"])
    assert nz.n_self == int(g["n_self"]) and nz.n_wrap == int(g["n_wrap"])
    assert nz.coincident_terms == int(g["coincident_terms"])
    assert plan.far.kernel_terms == int(g["far_terms"])
    assert rel_l2(plan.far.kernel, g["far_kernel"]) <= 1e-14
    assert rel_l2(plan.evaluate(q), g["u"]) <= 1e-13


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


@pytest.mark.slow
def test_oracle_matches_reference_c1():
    from paper_2312_02376_b200.workloads import CONFIGS, make_inputs
    w = CONFIGS[1]
    pos, q = make_inputs(1)
    pb = make_problem(w.dim, L=w.L, D=w.D, k0=w.k0, kshift=w.kshift, regime=w.regime, **w.params())
    plan = build_plan(pb, pos)
    g = golden("c1_full.npz")
    assert plan.near.pair_obs.size == int(g["n_pairs"])
    assert _digest(plan.near.pair_obs, plan.near.pair_src, plan.near.pair_code) == str(g["pair_digest"])
    assert rel_l2(plan.evaluate(q), g["u"]) <= 1e-13
