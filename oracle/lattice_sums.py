"""Periodic Green's function series, restated from
/root/reference/pkg/src/perisum/pgf.py (test infrastructure only).

  image_sum   phase-weighted free-space images |i_a| <= h        pgf.py:114-154
  drive       per-point adaptive layer truncation                  pgf.py:166-195
  spectral    Floquet series (dynamic / static-shifted)            pgf.py:202-295
  lattice     log + K0 series (neutral, no phase)                  pgf.py:317-425
  far_kernel  total minus the |i| <= i_d images                    pgf.py:450-462
"""
from __future__ import annotations

import itertools

import numpy as np

from .bessel import csqrt_lower, h0, k0
from .problem import Problem, Regime

FOUR_PI = 4.0 * np.pi
MAX_LAYERS = 200_000
CONSECUTIVE_SMALL = 3
MAX_TERMS = 1_000_000


class SeriesError(Exception):
    """Raised with a kind in {"domain", "wood", "not_converged", "separation"}."""

    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = kind


def sep_tol(pb: Problem) -> float:
    return 1e-13 * max(max(pb.L[a] for a in pb.periodic), 1.0)          # pgf.py:93-94


def wood_threshold(pb: Problem) -> float:
    return 1e-8 * 2.0 * np.pi / max(pb.L[a] for a in pb.periodic)       # pgf.py:88-90


def image_table(pb: Problem, h):
    """Image index triples in itertools.product order (x slowest), their offsets
    i*L and phases exp(-j i.(kshift*L)); pgf.py:114-123."""
    half = [int(h) if a in pb.periodic else 0 for a in range(3)]
    idx = np.array(list(itertools.product(*[range(-v, v + 1) for v in half])), dtype=float)
    kl = np.asarray(pb.kshift) * np.asarray(pb.L)
    return idx * np.asarray(pb.L), np.exp(-1j * (idx @ kl))


def image_sum(points, pb: Problem, h, drop=False, tol=None):
    """sum_i phase_i e^{-j k0 r_i}/(4 pi r_i), r_i = |p - i L|; pgf.py:126-154.
    drop=True zeroes coincident terms (r <= tol) instead of raising."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    tol = sep_tol(pb) if tol is None else tol
    offs, phs = image_table(pb, h)
    acc = np.zeros(pts.shape[0], dtype=complex)
    with np.errstate(under="ignore", divide="ignore", invalid="ignore"):
        for off, ph in zip(offs, phs):
            d = pts - off
            r = np.sqrt(np.einsum("ij,ij->i", d, d))
            bad = r <= tol
            if bad.any():
                if not drop:
                    raise SeriesError("domain", f"image {off.tolist()} coincides with a point")
                rr = np.where(bad, 1.0, r)
                acc += np.where(bad, 0.0, ph * np.exp(-1j * pb.k0 * rr) / (FOUR_PI * rr))
            else:
                acc += ph * np.exp(-1j * pb.k0 * r) / (FOUR_PI * r)
    return acc


def drive(points, tol, lead, layer, first, max_terms=MAX_TERMS, consecutive=CONSECUTIVE_SMALL):
    """pgf.py:166-195: every point keeps adding layers until `consecutive` layers
    in a row satisfy |layer| <= tol*max(|total|, 1e-300), or max_terms is reached
    (TruncationPolicy, pgf.py:40-58)."""
    n = points.shape[0]
    total = np.zeros(n, dtype=complex)
    terms = np.zeros(n, dtype=np.int64)
    quiet = np.zeros(n, dtype=np.int32)
    done = np.zeros(n, dtype=bool)
    if lead is not None:
        total += lead(points)
        terms += 1
    live = np.arange(n)
    s = first
    while live.size and s < MAX_LAYERS:
        v, c = layer(points[live], s)
        total[live] += v
        terms[live] += c
        small = np.abs(v) <= tol * np.maximum(np.abs(total[live]), 1e-300)
        quiet[live] = np.where(small, quiet[live] + 1, 0)
        fin = quiet[live] >= consecutive
        done[live[fin]] = True
        live = live[~fin & (terms[live] < max_terms)]
        s += 1
    return total, terms, done


def shell(s: int):
    """(m, n) index order of square shell s; pgf.py:202-212."""
    if s == 0:
        return np.zeros(1, dtype=int), np.zeros(1, dtype=int)
    top = np.arange(-s, s + 1)
    side = np.arange(-s + 1, s)
    ms = np.concatenate([np.repeat(top, 2), np.tile([s, -s], side.size)])
    ns = np.concatenate([np.tile([s, -s], top.size), np.repeat(side, 2)])
    return ms, ns


def spectral(points, pb: Problem, tol, **policy):
    """Floquet series; pgf.py:215-295."""
    if pb.regime == Regime.NPSP:
        raise SeriesError("domain", "spectral series diverges for NPSP")
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    wood = wood_threshold(pb)
    kx0, ky0, kz0 = pb.kshift
    lx, ly, lz = pb.L

    def kx(m):
        return kx0 + 2.0 * np.pi * np.asarray(m) / lx

    def ky(n):
        return ky0 + 2.0 * np.pi * np.asarray(n) / ly

    if pb.dim == 1:
        if np.any(np.hypot(pts[:, 1], pts[:, 2]) <= sep_tol(pb)):
            raise SeriesError("separation", "1D spectral series needs rho > 0")

        def layer1(p, s):
            rho = np.hypot(p[:, 1], p[:, 2])
            acc = np.zeros(p.shape[0], dtype=complex)
            ms = (0,) if s == 0 else (s, -s)
            for m in ms:
                km = complex(kx(m))
                kr = complex(csqrt_lower(pb.k0 ** 2 - km ** 2))
                if abs(kr) < wood:
                    raise SeriesError("wood", f"|k_rho(m={m})| below threshold")
                acc += np.exp(-1j * km * p[:, 0]) * h0(kr * rho) / (4j * lx)
            return acc, len(ms)

        return drive(pts, tol, None, layer1, 0, **policy)

    three = pb.dim == 3

    def layer23(p, s):
        ms, ns = shell(s)
        kxs, kys = kx(ms), ky(ns)
        kz = csqrt_lower(pb.k0 ** 2 - kxs ** 2 - kys ** 2)
        if np.any(np.abs(kz) < wood):
            raise SeriesError("wood", f"|k_z| below threshold in shell {s}")
        x, y, z = p[:, 0], p[:, 1], p[:, 2]
        if three:
            ea = np.exp(-1j * (kz - kz0) * lz)
            eb = np.exp(-1j * (kz + kz0) * lz)
            if np.any(np.maximum(np.abs(ea), np.abs(eb)) > 1.0 + 1e-12):
                raise SeriesError("not_converged", "z image stack diverges")
            if np.any(np.minimum(np.abs(1.0 - ea), np.abs(1.0 - eb)) < 1e-8):
                raise SeriesError("wood", f"resonant z stack in shell {s}")
            ca, cb = ea / (1.0 - ea), eb / (1.0 - eb)
        acc = np.zeros(p.shape[0], dtype=complex)
        with np.errstate(under="ignore"):
            for j0 in range(0, kxs.size, 64):
                sl = slice(j0, j0 + 64)
                a = kxs[sl][:, None]
                b = kys[sl][:, None]
                c = kz[sl][:, None]
                f = np.exp(-1j * c * np.abs(z))
                if three:
                    f = f + ca[sl][:, None] * np.exp(-1j * c * z) + cb[sl][:, None] * np.exp(1j * c * z)
                acc += (np.exp(-1j * (a * x + b * y)) * f / (2j * c * lx * ly)).sum(axis=0)
        return acc, kxs.size

    return drive(pts, tol, None, layer23, 0, **policy)


def _log_trig(y, a, ly):
    # pgf.py:317-325: ln(1 - 2 e^{-2 pi a/ly} cos(2 pi y/ly) + e^{-4 pi a/ly})
    with np.errstate(under="ignore"):
        e = np.exp(-2.0 * np.pi * a / ly)
    arg = 1.0 - 2.0 * e * np.cos(2.0 * np.pi * y / ly) + e * e
    if np.any(arg <= 0.0):
        raise SeriesError("domain", "lattice log argument vanished")
    return np.log(arg)


def lattice(points, pb: Problem, tol, **policy):
    """NPSP lattice series; pgf.py:328-425.  Note the 3D lead's z-image range and
    the layers' (n, k) ranges come from the extrema over the *whole* call."""
    if pb.regime != Regime.NPSP:
        raise SeriesError("domain", "lattice series is NPSP-only")
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    lx, ly, lz = pb.L
    cut = float(np.log(1.0 / tol) + 8.0)                                 # pgf.py:56-58
    sep = sep_tol(pb)

    def modulate(acc, p, m):
        return (acc * (np.cos(2.0 * m * np.pi * p[:, 0] / lx) / (np.pi * lx))).astype(complex)

    if pb.dim == 1:
        def lead1(p):
            rho = np.hypot(p[:, 1], p[:, 2])
            if np.any(rho <= sep):
                raise SeriesError("separation", "1D lattice series needs rho > 0")
            return -np.log(rho) / (2.0 * np.pi * lx)

        def layer1(p, m):
            arg = 2.0 * m * np.pi * np.hypot(p[:, 1], p[:, 2]) / lx
            v = np.zeros(p.shape[0])
            ok = arg <= cut
            if ok.any():
                v[ok] = k0(arg[ok])
            return modulate(v, p, m), 1

        return drive(pts, tol, lead1, layer1, 1, **policy)

    if pb.dim == 2:
        def lead2(p):
            az = np.abs(p[:, 2])
            return (-az / (2.0 * lx * ly) - _log_trig(p[:, 1], az, ly) / (4.0 * np.pi * lx)).astype(complex)

        def layer2(p, m):
            y, z = p[:, 1], p[:, 2]
            smax = cut * lx / (2.0 * np.pi * m)
            acc = np.zeros(p.shape[0])
            cnt = np.zeros(p.shape[0], dtype=np.int64)
            for n in range(int(np.floor((-smax - y.max()) / ly)), int(np.ceil((smax - y.min()) / ly)) + 1):
                s2 = (n * ly + y) ** 2 + z * z
                if np.any(s2 <= sep * sep):
                    raise SeriesError("domain", "lattice K0 argument vanished")
                arg = 2.0 * m * np.pi * np.sqrt(s2) / lx
                ok = arg <= cut
                if ok.any():
                    acc[ok] += k0(arg[ok])
                    cnt[ok] += 1
            return modulate(acc, p, m), np.maximum(cnt, 1)

        return drive(pts, tol, lead2, layer2, 1, **policy)

    def lead3(p):
        y, z = p[:, 1], p[:, 2]
        az = np.abs(z)
        v = (z * z - az * lz) / (2.0 * lx * ly * lz)
        reach = cut * ly / (2.0 * np.pi)
        for kk in range(int(np.floor((-reach - z.max()) / lz)), int(np.ceil((reach - z.min()) / lz)) + 1):
            v = v - _log_trig(y, np.abs(kk * lz + z), ly) / (4.0 * np.pi * lx)
        return v.astype(complex)

    def layer3(p, m):
        y, z = p[:, 1], p[:, 2]
        smax = cut * lx / (2.0 * np.pi * m)
        acc = np.zeros(p.shape[0])
        cnt = np.zeros(p.shape[0], dtype=np.int64)
        krange = range(int(np.floor((-smax - z.max()) / lz)), int(np.ceil((smax - z.min()) / lz)) + 1)
        for n in range(int(np.floor((-smax - y.max()) / ly)), int(np.ceil((smax - y.min()) / ly)) + 1):
            uy = (n * ly + y) ** 2
            for kk in krange:
                s2 = uy + (kk * lz + z) ** 2
                if np.any(s2 <= sep * sep):
                    raise SeriesError("domain", "lattice K0 argument vanished")
                arg = 2.0 * m * np.pi * np.sqrt(s2) / lx
                ok = arg <= cut
                if ok.any():
                    acc[ok] += k0(arg[ok])
                    cnt[ok] += 1
        return modulate(acc, p, m), np.maximum(cnt, 1)

    return drive(pts, tol, lead3, layer3, 1, **policy)


def far_kernel(points, pb: Problem):
    """G_far = G_total - images(|i| <= i_d); pgf.py:450-462."""
    total = lattice if pb.regime == Regime.NPSP else spectral
    vals, terms, conv = total(points, pb, pb.series_tol)
    return vals - image_sum(points, pb, pb.i_d), terms, conv
