"""CPU oracle for the FFT-PIM potential evaluation -- TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the reference algorithm of
`perisum.solver.SolvePlan.evaluate` (/root/reference/pkg/src/perisum/solver.py:24-25)
and everything that produces its operands (`build_plan`, solver.py:35-45).
Each function cites the reference file:line it follows.

It exists only as the *checker*: `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it.  The
product path (`paper_2312_02376_b200`) never imports it and fails loudly when
its CUDA library is missing.

Parity pinning: the oracle is checked (tests/test_oracle_golden.py) against
  * the reference's own frozen 50-digit special-function and lattice/spectral
    values (copied into tests/golden/reference_constants.json by
    tests/golden/make_golden.py, which imports the reference test modules), and
  * outputs of the reference itself run in the build container on seeded
    inputs (plan operands and potentials, tests/golden/*.npz, same script).
"""
from .problem import Problem, Regime, make_problem
from .pipeline import OraclePlan, build_plan

__all__ = ["Problem", "Regime", "make_problem", "OraclePlan", "build_plan"]
