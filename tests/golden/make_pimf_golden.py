"""PIMF far-kernel blob written by the REFERENCE (farzone.py:166-212), for the
kernel-cache parity tests (tests/test_pimf_cpu.py, tests/test_gpu_boundary.py).

Run in the build container (where /root/reference exists):
    python tests/golden/make_pimf_golden.py

Writes (committed, small):
  ref_far_kernel.pimf   build_far_plan(..., cache_path=...) of a 3D dynamic problem
                        with a phase shift (far grid 6^3, order 3): the blob the
                        reference's cache miss writes
  ref_far_kernel.npz    its inputs (positions, charges, problem) and the
                        reference's eval_far output, kernel_terms and signature
Nothing at run time reads /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

PROBLEM = dict(dim=3, L=(1.0, 1.0, 1.0), D=(1.0, 1.0, 1.0), k0=2.0 * np.pi, kshift=(0.2 * np.pi, 0.1 * np.pi, 0.0),
               far_grid=(6, 6, 6), far_order=3, near_grid=(12, 12, 12), near_order=3, n=500, seed=4242)


def main():
    from perisum.farzone import _kernel_signature, build_far_plan, eval_far
    from perisum.model import (ObserverPointSet, PeriodicityConfig, Periodicity, Regime, SolverParams,
                               SourcePointSet, TargetBox)
    p = PROBLEM
    rng = np.random.default_rng(p["seed"])
    pos = rng.uniform(0.0, 1.0, (p["n"], 3))
    q = rng.standard_normal(p["n"]) + 1j * rng.standard_normal(p["n"])
    cfg = PeriodicityConfig(dim=Periodicity(p["dim"]), L=p["L"], k0=p["k0"], kshift=p["kshift"],
                            regime=Regime.DYNAMIC)
    box = TargetBox(p["D"])
    params = SolverParams(far_grid=p["far_grid"], far_order=p["far_order"], near_grid=p["near_grid"],
                          near_order=p["near_order"])
    blob = os.path.join(HERE, "ref_far_kernel.pimf")
    if os.path.exists(blob):
        os.remove(blob)
    plan = build_far_plan(cfg, box, SourcePointSet(pos, q), ObserverPointSet(pos), params, cache_path=blob)
    u_far = eval_far(plan, q)
    sig = _kernel_signature(cfg, box, p["far_grid"], params.i_d, params.series_tol)
    np.savez(os.path.join(HERE, "ref_far_kernel.npz"), pos=pos, q=q, u_far=u_far,
             kernel_terms=np.int64(plan.kernel_terms), signature=np.uint64(sig),
             kernel=plan.kernel)
    print(f"wrote {blob}: {os.path.getsize(blob)} bytes, kernel_terms {plan.kernel_terms}, signature {sig}")


if __name__ == "__main__":
    main()
