"""Brute-force periodic sums, restated from
/root/reference/pkg/src/perisum/oracle.py (test infrastructure only: the
checker for the device direct evaluator, never on a product path).

  direct        eval_direct / eval_direct_farzone          oracle.py:62-111
  free_space    eval_free_space                            oracle.py:114-123

Observers go in chunks of 64 (oracle.py:20); a chunk with a separation
failure (oracle.py:35-59) is skipped (potentials 0, only those failures
reported), otherwise its non-converged pairs are reported.  Failures are
(observer, source, "separation" | "not converged") in the reference's order.
"""
from __future__ import annotations

import numpy as np

from .lattice_sums import image_sum, lattice, spectral
from .problem import Problem, Regime

CHUNK = 64


def _failures(pb: Problem, diffs, rows, conv=None):
    """oracle.py:35-59."""
    floor = 1e-12 * max(pb.L[a] for a in pb.periodic)
    if pb.dim == 1:
        bad = np.hypot(diffs[:, :, 1], diffs[:, :, 2]) <= floor
    elif pb.regime == Regime.NPSP:
        ly, lz = pb.L[1], pb.L[2]
        ry = np.abs(np.remainder(diffs[:, :, 1] + ly / 2, ly) - ly / 2)
        rz = np.abs(diffs[:, :, 2]) if pb.dim == 2 else np.abs(np.remainder(diffs[:, :, 2] + lz / 2, lz) - lz / 2)
        bad = np.hypot(ry, rz) <= floor
    else:
        bad = np.zeros(diffs.shape[:2], dtype=bool)
    out = [(int(rows[i]), int(j), "separation") for i, j in zip(*np.nonzero(bad))]
    if conv is not None:
        nc = ~conv & ~bad
        out += [(int(rows[i]), int(j), "not converged") for i, j in zip(*np.nonzero(nc))]
    return out, bad


def direct(pb: Problem, src_pos, q, obs_pos, i_d=None, tol=1e-10, max_terms=1_000_000, consecutive=3):
    """u_m = sum_n G(r_m - r_n) q_n; G = total (i_d None) or total minus the
    |i| <= i_d images (eval_direct_farzone).  Returns (u, worst_terms, failures)."""
    src_pos = np.asarray(src_pos, dtype=float)
    obs_pos = np.asarray(obs_pos, dtype=float)
    q = np.asarray(q, dtype=complex)
    n, m = len(src_pos), len(obs_pos)
    series = lattice if pb.regime == Regime.NPSP else spectral
    u = np.zeros(m, dtype=complex)
    worst, fails = 0, []
    for i0 in range(0, m, CHUNK):
        rows = np.arange(i0, min(i0 + CHUNK, m))
        diffs = obs_pos[rows, None, :] - src_pos[None, :, :]
        f, bad = _failures(pb, diffs, rows)
        if f:
            fails += f
            continue
        flat = diffs.reshape(-1, 3)
        vals, terms, conv = series(flat, pb, tol, max_terms=max_terms, consecutive=consecutive)
        if i_d is not None:
            vals = vals - image_sum(flat, pb, i_d)
        f, _ = _failures(pb, diffs, rows, conv.reshape(len(rows), n))
        fails += f
        worst = max(worst, int(terms.max()) if terms.size else 0)
        u[rows] = vals.reshape(len(rows), n) @ q
    return u, worst, fails


def free_space(k0, src_pos, q, obs_pos):
    """oracle.py:114-123."""
    src_pos = np.asarray(src_pos, dtype=float)
    obs_pos = np.asarray(obs_pos, dtype=float)
    u = np.zeros(len(obs_pos), dtype=complex)
    for i0 in range(0, len(obs_pos), CHUNK):
        sl = slice(i0, min(i0 + CHUNK, len(obs_pos)))
        d = obs_pos[sl, None, :] - src_pos[None, :, :]
        r = np.sqrt(np.einsum("mnk,mnk->mn", d, d))
        if np.any(r == 0.0):
            raise ZeroDivisionError("observer coincides with a source")
        u[sl] = (np.exp(-1j * k0 * r) / (4.0 * np.pi * r)) @ np.asarray(q, dtype=complex)
    return u
