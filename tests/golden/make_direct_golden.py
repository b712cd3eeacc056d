"""Golden fixtures for the device brute-force oracle, made
by running the REFERENCE's eval_direct / eval_direct_farzone / eval_free_space
(/root/reference/pkg/src/perisum/oracle.py:92-123) on small seeded inputs.

Run in the build container (where /root/reference exists):
    python tests/golden/make_direct_golden.py

Also writes tests/golden/near_id0.npz: build_near_plan with i_d = 0 (the
near-zone-only plan the reference's bench uses as its free-space baseline,
cli.py:343-347) and eval_near on small seeded 1D/2D/3D problems.

Writes tests/golden/direct_cases.npz: per case the inputs (positions, charges,
configuration, policy) and the reference's values, worst_terms and failure
records (observer, source, 1 = separation | 2 = not converged).  Nothing at run
time reads /root/reference.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import perisum as P  # noqa: E402  (the reference)
from perisum.oracle import eval_direct, eval_direct_farzone, eval_free_space  # noqa: E402
from perisum.pgf import TruncationPolicy  # noqa: E402

REASON = {"separation": 1, "not converged": 2}

# name: (dim, L, k0, kshift, regime, mode, i_d, n_src, n_obs, policy (tol, max_terms, consecutive), layout)
CASES = {
    "p1_dyn": (1, (1.0, 1.0, 1.0), np.pi, (0.3 * np.pi, 0, 0), "dynamic", "direct", 0, 24, 70, None, "box"),
    "p1_dyn_far": (1, (1.0, 1.0, 1.0), np.pi, (0.3 * np.pi, 0, 0), "dynamic", "far", 1, 24, 70, None, "box"),
    "p2_dyn": (2, (1.0, 1.0, 1.0), 1.5 * np.pi, (0.2 * np.pi, 0.1 * np.pi, 0), "dynamic", "direct", 0, 20, 70,
               None, "slab"),
    "p2_dyn_far_id2": (2, (1.0, 1.2, 1.0), 1.5 * np.pi, (0.2 * np.pi, 0, 0), "dynamic", "far", 2, 20, 40, None,
                       "slab"),
    "p3_dyn": (3, (1.0, 1.0, 1.0), 2.0 * np.pi - 0.3j, (0.2 * np.pi, 0.1 * np.pi, 0), "dynamic", "direct", 0, 10,
               20, (1e-8, 1_000_000, 3), "box"),
    "p1_npsp": (1, (1.0, 1.0, 1.0), 0.0, (0, 0, 0), "npsp", "direct", 0, 30, 70, None, "box"),
    "p2_npsp_sep": (2, (1.0, 1.0, 1.0), 0.0, (0, 0, 0), "npsp", "direct", 0, 30, 70, None, "sep"),
    "p3_npsp": (3, (1.0, 1.0, 1.0), 0.0, (0, 0, 0), "npsp", "direct", 0, 20, 70, None, "box"),
    "p3_npsp_far": (3, (1.0, 1.0, 1.0), 0.0, (0, 0, 0), "npsp", "far", 1, 20, 40, None, "box"),
    "p2_dyn_nc": (2, (1.0, 1.0, 1.0), 1.5 * np.pi, (0.2 * np.pi, 0.1 * np.pi, 0), "dynamic", "direct", 0, 12, 70,
                  (1e-10, 5, 3), "slab"),
    "free": (0, (1.0, 1.0, 1.0), 2.0 + 0.1j, (0, 0, 0), "dynamic", "free", 0, 30, 50, None, "box"),
}


def inputs(name, spec, seed):
    dim, L, k0, ks, regime, mode, i_d, n, m, pol, layout = spec
    rng = np.random.default_rng(seed)
    src = rng.uniform(0.0, 1.0, (n, 3))
    obs = rng.uniform(0.0, 1.0, (m, 3))
    if layout == "slab":          # keep |z| differences away from 0 (spectral series in 2D/3D)
        src[:, 2] *= 0.3
        obs[:, 2] = 0.6 + 0.4 * obs[:, 2]
    if layout == "sep":           # observer 5 on source 3's transverse lattice line (y + L_y, same z)
        obs[5] = (0.77, src[3, 1], src[3, 2])
    q = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    if regime == "npsp":
        q = rng.standard_normal(n)
        q = q - q.mean()
    return src, obs, q


def main():
    out = {}
    for c, (name, spec) in enumerate(CASES.items()):
        dim, L, k0, ks, regime, mode, i_d, n, m, pol, layout = spec
        src, obs, q = inputs(name, spec, 100 + c)
        t0 = time.perf_counter()
        S, O = P.SourcePointSet(src, q), P.ObserverPointSet(obs)
        if mode == "free":
            vals, worst, fails = eval_free_space(complex(k0), S, O), 0, ()
        else:
            cfg = P.PeriodicityConfig(dim=P.Periodicity(dim), L=tuple(L), k0=complex(k0),
                                      kshift=tuple(complex(k) for k in ks), regime=P.Regime(regime))
            policy = TruncationPolicy(*pol) if pol else TruncationPolicy()
            rep = eval_direct(cfg, S, O, policy) if mode == "direct" else eval_direct_farzone(cfg, S, O, i_d, policy)
            vals, worst, fails = rep.values, rep.worst_terms, rep.failures
        f = np.array([(i, j, REASON[r]) for i, j, r in fails], dtype=np.int64).reshape(-1, 3)
        print(f"{name}: {time.perf_counter() - t0:.1f}s worst={worst} failures={len(f)} |u|={np.linalg.norm(vals):.3e}")
        pol = pol or (1e-10, 1_000_000, 3)
        for k, v in dict(src=src, obs=obs, q=q, u=vals, worst=worst, failures=f, dim=dim, L=np.array(L),
                         k0=complex(k0), kshift=np.array(ks, dtype=complex), regime=regime, mode=mode, i_d=i_d,
                         tol=pol[0], max_terms=pol[1], consecutive=pol[2]).items():
            out[f"{name}__{k}"] = v
    np.savez_compressed(os.path.join(HERE, "direct_cases.npz"), names=np.array(list(CASES)), **out)


def near_id0():
    from perisum.nearzone import build_near_plan, eval_near
    out = {}
    for c, (dim, regime, k0, ks) in enumerate([(1, "npsp", 0.0, (0, 0, 0)), (2, "dynamic", np.pi, (0.3 * np.pi, 0, 0)),
                                               (3, "dynamic", 2.0, (0.1, 0.2, 0.0))]):
        rng = np.random.default_rng(300 + c)
        n = 300
        pos = rng.uniform(0.0, 1.0, (n, 3))
        q = rng.standard_normal(n) + (0j if regime == "npsp" else 1j * rng.standard_normal(n))
        if regime == "npsp":
            q = q - q.mean()
        cfg = P.PeriodicityConfig(dim=P.Periodicity(dim), L=(1.0, 1.0, 1.0), k0=complex(k0),
                                  kshift=tuple(complex(k) for k in ks), regime=P.Regime(regime))
        params = P.SolverParams(i_d=0, near_grid=(10, 10, 10), near_order=3)
        plan = build_near_plan(cfg, P.TargetBox((1.0, 1.0, 1.0)), P.SourcePointSet(pos, q), P.ObserverPointSet(pos),
                               params)
        u = eval_near(plan, q)
        key = f"c{c}"
        out.update({f"{key}__pos": pos, f"{key}__q": q, f"{key}__u": u, f"{key}__dim": dim, f"{key}__regime": regime,
                    f"{key}__k0": complex(k0), f"{key}__kshift": np.array(ks, dtype=complex),
                    f"{key}__n_pairs": int(plan.pair_obs.size), f"{key}__n_wrapped": int(plan.n_wrapped_pairs),
                    f"{key}__join_radius": np.array(plan.join_radius)})
        print(f"near i_d=0 {key}: pairs={plan.pair_obs.size} wrapped={plan.n_wrapped_pairs} jr={plan.join_radius}")
    np.savez_compressed(os.path.join(HERE, "near_id0.npz"), **out)


if __name__ == "__main__":
    main()
    near_id0()
