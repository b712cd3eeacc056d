"""Seeded random small problems across the whole parameter space of the path
(periodicity 1D/2D/3D, the three regimes, lossy wavenumbers, D < L, planar boxes,
orders 1-4, i_d 1-2, separate observer sets) for the randomized GPU-vs-oracle
parity sweep (tests/test_gpu_random.py) and its CPU pre-check
(tests/test_oracle_golden.py imports nothing from here; tools/check_random_problems.py
runs the oracle alone over every draw)."""
from __future__ import annotations

import numpy as np

N_DRAWS = 24


def draw(seed: int) -> dict:
    """One problem: plain data (dim, L, D, k0, kshift, params, src, q, obs or None)."""
    rng = np.random.default_rng(7000 + seed)
    for _ in range(100):
        dim = int(rng.integers(1, 4))
        regime = ("npsp", "static-shifted", "dynamic", "dynamic-lossy")[int(rng.integers(0, 4))]
        L = tuple(float(v) for v in np.round(rng.uniform(0.8, 1.6, 3), 3))
        frac = np.where(rng.random(3) < 0.5, 1.0, np.round(rng.uniform(0.55, 0.95, 3), 3))
        D = [L[a] * float(frac[a]) for a in range(3)]
        planar = dim <= 2 and rng.random() < 0.25
        if planar:
            D[2] = 0.0
        D = tuple(D)
        grid = tuple(int(rng.integers(6, 12)) if D[a] > 0 else 1 for a in range(3))
        order = int(rng.integers(1, 5))
        i_d = 2 if rng.random() < 0.2 else 1
        far_grid = tuple(int(rng.integers(5, 8)) for _ in range(3))
        far_order = int(rng.integers(2, 4))
        ks = [0.0, 0.0, 0.0]
        k0 = 0j
        if regime != "npsp":
            for a in range(dim):
                ks[a] = float(np.round(rng.uniform(-0.9, 0.9), 3))
            if not any(ks):
                ks[0] = 0.37
        if regime == "dynamic":
            k0 = complex(float(np.round(rng.uniform(0.6, 3.0), 3)))
        elif regime == "dynamic-lossy":
            k0 = complex(float(np.round(rng.uniform(0.6, 3.0), 3)), -float(np.round(rng.uniform(0.05, 0.6), 3)))
        n = int(rng.integers(40, 260))
        src = rng.uniform(0.0, 1.0, (n, 3)) * np.asarray(D)
        q = rng.standard_normal(n) + 0j
        if regime == "npsp":
            q -= q.mean()
            q[-1] -= q.sum()
        else:
            q = q + 1j * rng.standard_normal(n)
        obs = None
        if rng.random() < 0.35:
            m = int(rng.integers(1, 120))
            obs = rng.uniform(0.02, 0.98, (m, 3)) * np.asarray(D)
        min_active = min(grid[a] for a in range(3) if D[a] > 0)
        if order + 1 > min_active:
            continue
        # 2 D_ER < L on periodic axes (model.py:288-296)
        if any(grid[a] > 1 and 2.0 * D[a] / (grid[a] - 1) >= L[a] for a in range(dim)):
            continue
        if any(D[a] <= 0.0 for a in range(dim)):
            continue
        return dict(seed=seed, dim=dim, L=L, D=D, k0=k0, kshift=tuple(ks), regime=regime.split("-lossy")[0],
                    params=dict(near_grid=grid, near_order=order, far_grid=far_grid, far_order=far_order, i_d=i_d),
                    src=src, q=q, obs=obs)
    raise RuntimeError(f"no admissible draw for seed {seed}")
