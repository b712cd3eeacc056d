"""Near-zone engine restated from /root/reference/pkg/src/perisum/nearzone.py
(test infrastructure only): kernel table + circulant embedding + FFT
(nearzone.py:212-235), stencils (:237-239), correction radius (:245-256,
:290-300), correction pairs and coefficients (:303-487), evaluation (:490-525).

Extension used only for the subset-observer oracle: observers
may be given as an index subset of the sources (`obs_src`), which makes the
self-pair rule `obs_src[m] == n` instead of `m == n`.  With obs_src = arange(N)
this is exactly the reference's same_points behaviour.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

from .lagrange import Grid, Stencil, make_stencil, near_grid
from .lattice_sums import SeriesError, image_sum, image_table
from .problem import Problem

MATVEC_CHUNK = 1 << 22
TAP_CHUNK = 16384


@dataclass
class NearPlan:
    pb: Problem
    grid: Grid
    src: Stencil
    obs: Stencil
    kernel_disp: np.ndarray
    kernel_hat: np.ndarray
    nb: tuple
    jr: tuple
    jr_full: int
    pair_obs: np.ndarray
    pair_src: np.ndarray
    pair_code: np.ndarray
    pair_coef: np.ndarray
    seg_obs: np.ndarray
    seg_starts: np.ndarray
    n_self: int
    n_wrap: int
    coincident_terms: int


def correction_radius(er_range_boxes: int, order: int) -> int:
    return er_range_boxes + order + 2                                   # nearzone.py:290-300


def embed(kernel_disp, dims):
    """Zero-padded circulant embedding on doubled axes; nearzone.py:127-147.
    Non-negative displacements land at [0, n-1], negative ones at [n+1, 2n-1]."""
    out = np.zeros(tuple(2 * d if d > 1 else 1 for d in dims), dtype=complex)
    per_axis = []
    for a, n in enumerate(dims):
        if n == 1:
            per_axis.append([(slice(0, 1), slice(0, 1))])
        else:
            per_axis.append([(slice(0, n), slice(n - 1, 2 * n - 1)),
                             (slice(n + 1, 2 * n), slice(0, n - 1))])
    for combo in itertools.product(*per_axis):
        out[tuple(c[0] for c in combo)] = kernel_disp[tuple(c[1] for c in combo)]
    return out


def sing_tol(pb: Problem) -> float:
    return 1e-12 * max(max(pb.L), max(pb.D), 1.0)                       # nearzone.py:213


def box_index(pts, grid: Grid, nb, pad):
    """Padded per-axis box ids floor(x/h) clipped to [-pad, nb-1+pad], + pad;
    nearzone.py:181-191 (degenerate axes are forced to 0 by the caller)."""
    out = np.zeros((pts.shape[0], 3), dtype=np.int64)
    for a in range(3):
        if grid.dims[a] == 1:
            continue
        out[:, a] = np.clip(np.floor(pts[:, a] / grid.spacing[a]).astype(np.int64), -pad, nb[a] - 1 + pad) + pad
    return out


def correlate(wo, ws):
    """C[u], u = a - b + (w-1), accumulated a-major then b; nearzone.py:150-157."""
    p, w = wo.shape
    c = np.zeros((p, 2 * w - 1))
    for a in range(w):
        for b in range(w):
            c[:, a - b + w - 1] += wo[:, a] * ws[:, b]
    return c


def gather_taps(table, base, d0, cx, cy, cz):
    """G_grid = sum_uvw Cx Cy Cz T[d0 - base + (u,v,w)]; nearzone.py:160-178."""
    p = d0.shape[0]
    out = np.empty(p, dtype=complex)
    ux, uy, uz = cx.shape[1], cy.shape[1], cz.shape[1]
    for i0 in range(0, p, TAP_CHUNK):
        sl = slice(i0, min(p, i0 + TAP_CHUNK))
        ix = (d0[sl, 0] - base[0])[:, None, None, None] + np.arange(ux)[None, :, None, None]
        iy = (d0[sl, 1] - base[1])[:, None, None, None] + np.arange(uy)[None, None, :, None]
        iz = (d0[sl, 2] - base[2])[:, None, None, None] + np.arange(uz)[None, None, None, :]
        out[sl] = np.einsum("pu,pv,pw,puvw->p", cx[sl], cy[sl], cz[sl], table[ix, iy, iz])
    return out


def kernel_table(pb: Problem, grid: Grid):
    """G_near on every grid displacement (2n-1 per active axis), coincident image
    terms dropped, centre zeroed; nearzone.py:215-233."""
    dims, h = grid.dims, grid.spacing
    axes = [np.zeros(1) if dims[a] == 1 else np.arange(-(dims[a] - 1), dims[a]) * h[a] for a in range(3)]
    mesh = np.meshgrid(*axes, indexing="ij")
    pts = np.stack([m.ravel() for m in mesh], axis=1)
    tab = image_sum(pts, pb, pb.i_d, drop=True, tol=sing_tol(pb)).reshape(tuple(len(x) for x in axes))
    tab[tuple(dims[a] - 1 if dims[a] > 1 else 0 for a in range(3))] = 0.0
    offs, _ = image_table(pb, pb.i_d)
    tol = sing_tol(pb)
    coincident = sum(int(np.count_nonzero(np.einsum("ij,ij->i", pts - o, pts - o) <= tol * tol)) for o in offs)
    return tab, coincident


def join_radius(pb: Problem, grid: Grid, nb, jr_full):
    """Per-axis box radius; nearzone.py:245-256."""
    jr = []
    for a in range(3):
        if grid.dims[a] == 1:
            jr.append(0)
            continue
        r = jr_full
        if pb.i_d >= 1 and a in pb.periodic:
            per_period = int(np.floor(pb.L[a] / grid.spacing[a] + 1e-9))
            r = min(r, max((per_period - 1) // 2, 1))
        jr.append(min(r, nb[a]))
    return tuple(jr)


def build_near(pb: Problem, src_pos, obs_pos, obs_src=None, fft=np.fft.fftn) -> NearPlan:
    """nearzone.py:194-273 (build_near_plan)."""
    dims = pb.near_dims(max(len(src_pos), len(obs_pos)))
    grid = near_grid(pb.D, dims)
    h = grid.spacing
    nb = tuple(max(d - 1, 1) for d in dims)
    if pb.i_d >= 1:
        for a in pb.periodic:
            if dims[a] > 1 and 2.0 * pb.er_range_boxes * h[a] >= pb.L[a]:
                raise ValueError(f"error-correction range on axis {a} must satisfy 2*D_ER < L")
    kdisp, coincident = kernel_table(pb, grid)
    khat = fft(embed(kdisp, dims))
    margin = tuple(1e-9 * max(h[a], 1.0) for a in range(3))
    sst = make_stencil(grid, src_pos, pb.near_order, margin)
    ost = make_stencil(grid, obs_pos, pb.near_order, margin)
    if obs_src is None:
        same = src_pos is obs_pos or (src_pos.shape == obs_pos.shape and np.array_equal(src_pos, obs_pos))
        obs_src = np.arange(len(obs_pos)) if same else None
    jr_full = correction_radius(pb.er_range_boxes, pb.near_order)
    jr = join_radius(pb, grid, nb, jr_full)
    pairs = corrections(pb, grid, nb, jr, jr_full, sst, ost, src_pos, obs_pos, kdisp, obs_src)
    return NearPlan(pb, grid, sst, ost, kdisp, khat, nb, jr, jr_full, *pairs, coincident)


def wrapped_sources(pb: Problem, grid: Grid, pad, src_pos):
    """Originals plus shifted copies (src + c*L) near periodic faces, code-major in
    itertools.product order; nearzone.py:310-339."""
    n = src_pos.shape[0]
    pos, orig, code = [src_pos], [np.arange(n, dtype=np.int64)], [np.zeros((n, 3), dtype=np.int8)]
    if pb.i_d >= 1:
        choices = [(-1, 0, 1) if (a in pb.periodic and grid.dims[a] > 1) else (0,) for a in range(3)]
        for c in itertools.product(*choices):
            if c == (0, 0, 0):
                continue
            keep = np.ones(n, dtype=bool)
            for a in range(3):
                if c[a] < 0:
                    keep &= src_pos[:, a] >= pb.L[a] - pad[a] * grid.spacing[a]
                elif c[a] > 0:
                    keep &= src_pos[:, a] <= pb.D[a] - pb.L[a] + pad[a] * grid.spacing[a]
            if keep.any():
                sel = np.nonzero(keep)[0]
                pos.append(src_pos[sel] + np.asarray(c, dtype=float) * np.asarray(pb.L))
                orig.append(sel.astype(np.int64))
                code.append(np.tile(np.asarray(c, dtype=np.int8), (sel.size, 1)))
    return np.concatenate(pos), np.concatenate(orig), np.concatenate(code)


def discovery_context(pb, grid, nb, jr, jr_full, sst, ost, src_pos, obs_pos, kdisp, obs_src):
    """Everything pair discovery needs, shared by all observer ranges
    (nearzone.py:305-372): wrapped copies, box buckets, offsets, tolerances."""
    dims, h = grid.dims, grid.spacing
    pad = tuple(r + 1 for r in jr)
    aug_pos, aug_orig, aug_code = wrapped_sources(pb, grid, pad, src_pos)
    mp = max(pad) if any(p > 0 for p in pad) else 0
    ext = tuple(nb[a] + 2 * mp if dims[a] > 1 else 1 for a in range(3))
    sbox = box_index(aug_pos, grid, nb, mp)
    skey = (sbox[:, 0] * ext[1] + sbox[:, 1]) * ext[2] + sbox[:, 2]
    order = np.argsort(skey, kind="stable").astype(np.int64)
    counts = np.bincount(skey[order], minlength=ext[0] * ext[1] * ext[2])
    return dict(
        pb=pb, dims=dims, h=h, sst=sst, ost=ost, obs_pos=obs_pos, kdisp=kdisp, obs_src=obs_src,
        aug_pos=aug_pos, aug_orig=aug_orig, aug_code=aug_code, ext=ext, order=order, counts=counts,
        first=np.concatenate([[0], np.cumsum(counts)]), obox=box_index(obs_pos, grid, nb, mp),
        offsets=list(itertools.product(*[range(-jr[a], jr[a] + 1) if dims[a] > 1 else (0,) for a in range(3)])),
        r2_keep=float(jr_full) ** 2 + 1e-9,
        inv_h=np.array([1.0 / h[a] if dims[a] > 1 else 0.0 for a in range(3)]),
        phase_k=np.asarray(pb.kshift) * np.asarray(pb.L),
        widths=tuple(ost.axis_w[a].shape[1] for a in range(3)),
        main_base=tuple(-(dims[a] - 1) if dims[a] > 1 else 0 for a in range(3)),
        stol=sing_tol(pb))


def corrections(pb, grid, nb, jr, jr_full, sst, ost, src_pos, obs_pos, kdisp, obs_src,
                obs_chunk=1 << 16):
    """Pair discovery + coefficients; nearzone.py:303-487.  Processed in observer
    chunks: within a chunk the box offsets run db-major (as in the reference), then
    a stable sort by observer; chunks are ascending, so the global order equals the
    reference's single stable argsort."""
    ctx = discovery_context(pb, grid, nb, jr, jr_full, sst, ost, src_pos, obs_pos, kdisp, obs_src)
    n_obs = obs_pos.shape[0]
    parts = [discover_range(ctx, c0, min(n_obs, c0 + obs_chunk)) for c0 in range(0, n_obs, obs_chunk)]
    return merge_ranges(parts, n_obs)


def merge_ranges(parts, n_obs):
    """Concatenate ascending observer ranges and derive the reduceat segments."""
    parts = [p for p in parts if p[0].size]
    n_self = sum(p[4] for p in parts)
    n_wrap = sum(p[5] for p in parts)
    if parts:
        p_obs = np.concatenate([p[0] for p in parts])
        p_src = np.concatenate([p[1] for p in parts])
        p_code = np.concatenate([p[2] for p in parts])
        coef = np.concatenate([p[3] for p in parts])
        cnt = np.bincount(p_obs, minlength=n_obs)
        seg_obs = np.nonzero(cnt)[0]
        seg_starts = (np.cumsum(cnt) - cnt)[seg_obs]
    else:
        p_obs = np.zeros(0, np.int32)
        p_src = np.zeros(0, np.int32)
        p_code = np.zeros((0, 3), np.int8)
        coef = np.zeros(0, complex)
        seg_obs = np.zeros(0, np.int64)
        seg_starts = np.zeros(0, np.int64)
    return p_obs, p_src, p_code, coef, seg_obs, seg_starts, n_self, n_wrap


def discover_range(ctx, lo, hi):
    """Pairs of observers [lo, hi): (obs, src, code, coef, n_self, n_wrap), sorted
    by observer, db-major discovery order inside an observer (nearzone.py:374-478)."""
    pb, h, sst, ost, obs_pos = ctx["pb"], ctx["h"], ctx["sst"], ctx["ost"], ctx["obs_pos"]
    kdisp, obs_src, aug_pos = ctx["kdisp"], ctx["obs_src"], ctx["aug_pos"]
    aug_orig, aug_code, ext, order = ctx["aug_orig"], ctx["aug_code"], ctx["ext"], ctx["order"]
    counts, first, obox, r2_keep = ctx["counts"], ctx["first"], ctx["obox"], ctx["r2_keep"]
    inv_h, phase_k, widths, main_base, stol = (ctx["inv_h"], ctx["phase_k"], ctx["widths"],
                                               ctx["main_base"], ctx["stol"])
    n_self = n_wrap = 0
    offsets = ctx["offsets"]
    chunk = np.arange(lo, hi, dtype=np.int64)
    part = {k: [] for k in ("obs", "src", "code", "coef")}
    for db in offsets:
        tb = obox[chunk] + np.asarray(db, dtype=np.int64)
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
        if not keep.any():
            continue
        p_obs, p_aug, d = p_obs[keep], p_aug[keep], d[keep]
        p_src, p_code = aug_orig[p_aug], aug_code[p_aug]
        is_self = np.zeros(p_obs.shape[0], dtype=bool)
        if obs_src is not None:
            is_self = (obs_src[p_obs] == p_src) & np.all(p_code == 0, axis=1)
        clash = (np.einsum("ij,ij->i", d, d) <= stol * stol) & ~is_self
        if clash.any():
            i = int(np.argmax(clash))
            raise SeriesError("domain", f"observer {int(p_obs[i])} coincides with distinct source "
                                        f"{int(p_src[i])} (code {p_code[i].tolist()})")
        direct = np.zeros(p_obs.shape[0], dtype=complex)
        if (~is_self).any():
            direct[~is_self] = image_sum(d[~is_self], pb, pb.i_d, tol=stol)   # nearzone.py:418-421
        d0 = ost.starts[p_obs] - sst.starts[p_src] - (np.asarray(widths) - 1)  # nearzone.py:423-427
        cor = [correlate(ost.axis_w[a][p_obs], sst.axis_w[a][p_src]) for a in range(3)]
        cid = (p_code[:, 0].astype(np.int64) + 1) * 9 + (p_code[:, 1].astype(np.int64) + 1) * 3 + (p_code[:, 2] + 1)
        ggrid = np.empty(p_obs.shape[0], dtype=complex)
        for cf in np.unique(cid):                                          # nearzone.py:433-454
            sel = np.nonzero(cid == cf)[0]
            cv = (int(cf // 9) - 1, int((cf % 9) // 3) - 1, int(cf % 3) - 1)
            if cv == (0, 0, 0):
                tab, base = kdisp, main_base
            else:
                shift = np.asarray(cv, dtype=float) * np.asarray(pb.L)
                lo = [int(d0[sel, a].min()) for a in range(3)]
                hi = [int(d0[sel, a].max()) + 2 * (widths[a] - 1) for a in range(3)]
                ax = [np.arange(lo[a], hi[a] + 1) * h[a] - shift[a] for a in range(3)]
                mesh = np.meshgrid(*ax, indexing="ij")
                tp = np.stack([m.ravel() for m in mesh], axis=1)
                tab = image_sum(tp, pb, pb.i_d, drop=True, tol=stol).reshape(tuple(len(x) for x in ax))
                base = tuple(lo)
            ggrid[sel] = gather_taps(tab, base, d0[sel], cor[0][sel], cor[1][sel], cor[2][sel])
        coef = np.exp(-1j * (p_code @ phase_k)) * (direct - ggrid)        # nearzone.py:456-457
        n_self += int(np.count_nonzero(is_self))
        n_wrap += int(np.count_nonzero(np.any(p_code != 0, axis=1)))
        part["obs"].append(p_obs.astype(np.int32))
        part["src"].append(p_src.astype(np.int32))
        part["code"].append(p_code)
        part["coef"].append(coef)
    if not part["obs"]:
        return (np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros((0, 3), np.int8),
                np.zeros(0, complex), 0, 0)
    po = np.concatenate(part["obs"])
    srt = np.argsort(po, kind="stable")
    return (po[srt], np.concatenate(part["src"])[srt], np.concatenate(part["code"])[srt],
            np.concatenate(part["coef"])[srt], n_self, n_wrap)


def apply_corrections(plan: NearPlan, q, u):
    """u[m] += sum_pairs coef * q[src], chunked at segment boundaries;
    nearzone.py:506-524."""
    npairs = plan.pair_obs.size
    if not npairs:
        return u
    segs = plan.seg_starts
    buf = np.empty(min(npairs, MATVEC_CHUNK), dtype=complex)
    s0 = 0
    while s0 < segs.size:
        p0 = int(segs[s0])
        s1 = max(int(np.searchsorted(segs, p0 + MATVEC_CHUNK, side="left")), s0 + 1)
        p1 = int(segs[s1]) if s1 < segs.size else npairs
        blk = buf[:p1 - p0] if p1 - p0 <= buf.size else np.empty(p1 - p0, dtype=complex)
        np.take(q, plan.pair_src[p0:p1], out=blk)
        blk *= plan.pair_coef[p0:p1]
        u[plan.seg_obs[s0:s1]] += np.add.reduceat(blk, segs[s0:s1] - p0)
        s0 = s1
    return u


def eval_near(plan: NearPlan, q, ifft=np.fft.ifftn, fft=np.fft.fftn):
    """project -> zero-padded FFT convolution -> interpolate -> correct;
    nearzone.py:490-525."""
    q = np.asarray(q, dtype=complex)
    if q.shape[0] != plan.src.starts.shape[0]:
        raise ValueError(f"expected {plan.src.starts.shape[0]} amplitudes, got {q.shape[0]}")
    dims = plan.grid.dims
    buf = np.zeros(plan.kernel_hat.shape, dtype=complex)
    buf[:dims[0], :dims[1], :dims[2]] = plan.src.project(q).reshape(dims)
    ug = ifft(fft(buf) * plan.kernel_hat)[:dims[0], :dims[1], :dims[2]]
    u = plan.obs.interpolate(ug.ravel())
    return apply_corrections(plan, q, u)
