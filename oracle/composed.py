"""Composed CPU time of one reference evaluation at full scale -- BASELINE
INFRASTRUCTURE ONLY (bench.py's `cpu_baseline` leg and `--impl reference` arm).

C3/C4/C5 cannot run the reference's `SolvePlan.evaluate` (solver.py:24-25) on a
host: their plans hold 35-221 GB of correction pairs and take 10-60 min to build
(SURVEY.md 8c).  SURVEY.md 8d prescribes a *composed* time instead: every stage
of `eval_near` + `eval_far` (nearzone.py:490-525, farzone.py:150-159) is run with
the oracle's own numpy code on a bounded sample of the same workload and scaled
to the full size, single-threaded like the reference's eval loops:

  K1  project   (grids.py:167-181)  np.bincount of S sampled sources' w*q into the
                                    full near grid; t = t(empty bincount of the grid)
                                    + (t(S) - t(empty)) * N / S
  K2  FFT conv  (nearzone.py:500-504) each of the three forward and three inverse
                                    axis passes of the full padded buffer timed on a
                                    1/F slice of the other axes (same strides), x F;
                                    spectrum product, zero fill + corner copy and the
                                    cropped ravel likewise
  K3  interpolate (grids.py:183-188) S sampled observers, x N / S
  K4  corrections (nearzone.py:506-524) the oracle's chunked take/multiply/reduceat on
                                    the pair lists of a sample of observers (found by
                                    the reference's discovery rule, nearzone.py:374-396;
                                    coefficient VALUES are random -- the apply's cost
                                    does not depend on them), x P / P_sample
  K5  far project + grid sum + interpolate (farzone.py:156-159): project and
                                    interpolate on the S sample, x N / S; grid sum full
  + the final u_near + u_far add (solver.py:25), x N / S

P is the exact pair count when the caller knows it (the GPU plan), else the
sample's pairs per observer x M.  Everything that is plan build (stencils, pair
discovery, far kernel, kernel_hat) stays outside the timed regions.
"""
from __future__ import annotations

import time

import numpy as np

from . import near_engine as ne
from .far_engine import grid_sum
from .lagrange import far_grids, make_stencil, near_grid
from .problem import Problem


def _best(fn, reps=1):
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


def discover_pairs(pb: Problem, grid, src_pos, obs_idx):
    """(pair_obs local, pair_src) of the observers src_pos[obs_idx] (observers =
    sources), sorted stably by observer with the reference's db-major discovery
    order inside an observer (nearzone.py:303-396, 465-478).  Coefficients are not
    computed (plan build)."""
    dims, h = grid.dims, grid.spacing
    nb = tuple(max(d - 1, 1) for d in dims)
    jr_full = ne.correction_radius(pb.er_range_boxes, pb.near_order)
    jr = ne.join_radius(pb, grid, nb, jr_full)
    pad = tuple(r + 1 for r in jr)
    aug_pos, aug_orig, _ = ne.wrapped_sources(pb, grid, pad, src_pos)
    mp = max(pad) if any(p > 0 for p in pad) else 0
    ext = tuple(nb[a] + 2 * mp if dims[a] > 1 else 1 for a in range(3))
    sbox = ne.box_index(aug_pos, grid, nb, mp)
    skey = (sbox[:, 0] * ext[1] + sbox[:, 1]) * ext[2] + sbox[:, 2]
    order = np.argsort(skey, kind="stable").astype(np.int64)
    counts = np.bincount(skey[order], minlength=ext[0] * ext[1] * ext[2])
    first = np.concatenate([[0], np.cumsum(counts)])
    obs_pos = src_pos[obs_idx]
    obox = ne.box_index(obs_pos, grid, nb, mp)
    inv_h = np.array([1.0 / h[a] if dims[a] > 1 else 0.0 for a in range(3)])
    r2_keep = float(jr_full) ** 2 + 1e-9
    offsets = [(a, b, c) for a in (range(-jr[0], jr[0] + 1) if dims[0] > 1 else (0,))
               for b in (range(-jr[1], jr[1] + 1) if dims[1] > 1 else (0,))
               for c in (range(-jr[2], jr[2] + 1) if dims[2] > 1 else (0,))]
    chunk = np.arange(obs_idx.size, dtype=np.int64)
    po, ps = [], []
    for db in offsets:
        tb = obox + np.asarray(db, dtype=np.int64)
        ok = np.all((tb >= 0) & (tb < np.asarray(ext)), axis=1)
        if not ok.any():
            continue
        key = (tb[ok, 0] * ext[1] + tb[ok, 1]) * ext[2] + tb[ok, 2]
        cnt = counts[key]
        nz = cnt > 0
        if not nz.any():
            continue
        om, key, cnt = chunk[ok][nz], key[nz], cnt[nz]
        p_obs = np.repeat(om, cnt)
        local = np.arange(int(cnt.sum())) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        p_aug = order[np.repeat(first[key], cnt) + local]
        d = obs_pos[p_obs] - aug_pos[p_aug]
        keep = np.einsum("ij,ij->i", d * inv_h, d * inv_h) <= r2_keep
        po.append(p_obs[keep])
        ps.append(aug_orig[p_aug[keep]])
    if not po:
        return np.zeros(0, np.int64), np.zeros(0, np.int32)
    p_obs, p_src = np.concatenate(po), np.concatenate(ps)
    srt = np.argsort(p_obs, kind="stable")
    return p_obs[srt], p_src[srt].astype(np.int32)


class ComposedSampler:
    """Holds the sampled operands of one workload; `measure()` times one composed
    evaluation and returns (seconds, per-stage seconds)."""

    def __init__(self, pb: Problem, pos, q, n_pairs=None, n_sample=1 << 18, pair_target=6_000_000,
                 obs_max=16384, fft_slices=16, seed=12345):
        t0 = time.perf_counter()
        pos = np.ascontiguousarray(np.asarray(pos, dtype=float))
        self.N = N = pos.shape[0]
        self.q = np.asarray(q, dtype=complex)
        rng = np.random.default_rng(seed)
        dims = pb.near_dims(N)
        grid = near_grid(pb.D, dims)
        self.dims = dims
        S = min(N, n_sample)
        self.S = S
        idx = np.arange(S)                      # caller order is already a random sample
        margin = tuple(1e-9 * max(grid.spacing[a], 1.0) for a in range(3))
        self.near_st = make_stencil(grid, pos[idx], pb.near_order, margin)
        self.qs = self.q[idx]
        self.ng = grid.size
        self.ug = rng.standard_normal(grid.size) + 1j * rng.standard_normal(grid.size)
        fdims = tuple(pb.far_grid[a] if pb.D[a] > 0.0 else 1 for a in range(3))
        sg, og = far_grids(pb.D, fdims)
        fm = tuple(sg.spacing[a] if sg.dims[a] > 1 else 0.0 for a in range(3))
        self.far_src = make_stencil(sg, pos[idx], pb.far_order, fm)
        self.far_obs = make_stencil(og, pos[idx], pb.far_order, fm)
        self.far_dims = sg.dims
        kd = tuple(2 * n - 1 if n > 1 else 1 for n in sg.dims)
        self.far_kernel = rng.standard_normal(kd) + 1j * rng.standard_normal(kd)
        # padded FFT buffers at full size (the axis passes are timed on slices)
        self.mdims = tuple(2 * d if d > 1 else 1 for d in dims)
        self.buf = np.zeros(self.mdims, dtype=complex)
        self.buf[:dims[0], :dims[1], :dims[2]] = (rng.standard_normal(dims) + 0j)
        self.khat = np.full(self.mdims, 1.0 + 0.5j)
        self.F = fft_slices
        # K4 sample: grow the observer sample until it holds ~pair_target pairs
        n_obs = 0
        po, ps = [np.zeros(0, np.int64)], [np.zeros(0, np.int32)]
        step = 256
        while n_obs < min(obs_max, N):
            oi = np.arange(n_obs, min(n_obs + step, N, obs_max))
            a, b = discover_pairs(pb, grid, pos, oi)
            po.append(a + n_obs)
            ps.append(b)
            n_obs = oi[-1] + 1
            if sum(x.size for x in ps) >= pair_target:
                break
            step = min(step * 2, 4096)
        p_obs = np.concatenate(po)
        self.pair_src = np.concatenate(ps)
        self.n_obs = n_obs
        self.p_sample = self.pair_src.size
        self.pair_coef = rng.standard_normal(self.p_sample) + 1j * rng.standard_normal(self.p_sample)
        cnt = np.bincount(p_obs, minlength=n_obs)
        self.seg_obs = np.nonzero(cnt)[0]
        self.seg_starts = (np.cumsum(cnt) - cnt)[self.seg_obs]
        self.pairs_exact = n_pairs is not None
        self.P = int(n_pairs) if n_pairs is not None else int(round(self.p_sample / n_obs * N))
        self.setup_seconds = time.perf_counter() - t0

    # -- stages ---------------------------------------------------------------
    def _k1(self):
        st = self.near_st
        empty = _best(lambda: np.bincount(np.zeros(0, np.int64), minlength=self.ng) +
                      1j * np.bincount(np.zeros(0, np.int64), minlength=self.ng))
        t = _best(lambda: st.project(self.qs))
        return empty + max(t - empty, 0.0) * self.N / self.S

    def _fft(self):
        m, F = self.mdims, self.F
        total = 0.0
        for fn in (np.fft.fft, np.fft.ifft):
            for ax in range(3):
                other = [a for a in range(3) if a != ax and m[a] > 1]
                if m[ax] == 1:
                    continue
                cut = other[0] if other else None
                sl = [slice(None)] * 3
                frac = 1.0
                if cut is not None:
                    k = max(1, m[cut] // F)
                    sl[cut] = slice(0, k)
                    frac = k / m[cut]
                view = self.buf[tuple(sl)]
                total += _best(lambda: fn(view, axis=ax)) / frac
        # spectrum product, zero fill + corner copy, cropped ravel (1/F of each)
        k0 = max(1, m[0] // F)
        total += _best(lambda: self.buf[:k0] * self.khat[:k0]) * m[0] / k0
        d = self.dims
        kx = max(1, d[0] // F)
        sub = self.buf[:kx, :d[1], :d[2]]

        def fill():
            b = np.zeros((max(1, m[0] // F),) + tuple(m[1:]), dtype=complex)
            b[:kx, :d[1], :d[2]] = sub
        total += _best(fill) * F
        total += _best(lambda: np.ravel(self.buf[:kx, :d[1], :d[2]])) * d[0] / kx
        return total

    def _k3(self):
        return _best(lambda: self.near_st.interpolate(self.ug)) * self.N / self.S

    def _k4(self):
        u = np.zeros(self.n_obs, dtype=complex)
        plan = _K4View(self.pair_src, self.pair_coef, self.seg_obs, self.seg_starts)
        t = _best(lambda: ne.apply_corrections(plan, self.q, u))
        return t * self.P / max(self.p_sample, 1)

    def _far(self):
        tp = _best(lambda: self.far_src.project(self.qs)) * self.N / self.S
        qg = self.far_src.project(self.qs).reshape(self.far_dims)
        ts = _best(lambda: grid_sum(self.far_kernel, qg))
        ug = grid_sum(self.far_kernel, qg).ravel()
        ti = _best(lambda: self.far_obs.interpolate(ug)) * self.N / self.S
        return tp + ts + ti

    def _add(self):
        a = self.qs
        return _best(lambda: a + a) * self.N / self.S

    def measure(self):
        st = {"near_project": self._k1(), "fft_conv": self._fft(), "interpolate": self._k3(),
              "corrections": self._k4(), "far": self._far(), "sum": self._add()}
        return float(sum(st.values())), st

    def describe(self) -> str:
        return (f"composed (SURVEY.md 8d): oracle numpy stages timed on a bounded sample and scaled -- "
                f"K1/K3/far on {self.S} of {self.N} points, FFT axis passes on 1/{self.F} slices of the full "
                f"{'x'.join(map(str, self.mdims))} buffer, K4 on the {self.p_sample} pairs of {self.n_obs} "
                f"observers x {self.P / max(self.p_sample, 1):.0f} "
                f"({'exact' if self.pairs_exact else 'estimated'} P = {self.P}); single-threaded numpy")


class _K4View:
    """The four NearPlan fields apply_corrections reads."""

    def __init__(self, pair_src, pair_coef, seg_obs, seg_starts):
        self.pair_src, self.pair_coef, self.seg_obs, self.seg_starts = pair_src, pair_coef, seg_obs, seg_starts
        self.pair_obs = pair_src   # only .size is read
