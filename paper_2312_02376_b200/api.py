"""The drop-in facade: the reference's entry points on the B200 path.

  build_plan / SolvePlan.evaluate / solve      solver.py:18-55
  build_near_plan / eval_near                  nearzone.py:194-197, 490-525
  build_far_plan / eval_far                    farzone.py:76-131, 150-159
  save_far_kernel / load_far_kernel (PIMF)     farzone.py:166-212

Every plan operand is built and kept on the GPU by libfftpim.so; these
classes only hold the opaque handle plus the summary attributes the reference
CLI reads (cli.py:232-236).  `evaluate` accepts numpy arrays (host path, the
reference's calling convention) or CUDA tensors (device path, stream ordered on
torch's current stream).
"""
from __future__ import annotations

import ctypes as C
import hashlib
import struct
import time
import warnings
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .exceptions import KernelCacheError, ValidationError
from .problem import (REGIME_CODE, ObserverPointSet, PeriodicityConfig, PotentialField, Regime,
                      SolverParams, SourcePointSet, TargetBox, validate_problem)

__all__ = ["UniformGrid", "NativePlan", "NearZonePlan", "FarZonePlan", "SolvePlan", "SolveResult",
           "build_plan", "solve", "build_near_plan", "eval_near", "build_far_plan", "eval_far",
           "save_far_kernel", "load_far_kernel"]


@dataclass(frozen=True)
class UniformGrid:
    """Geometry-only view of a grid (grids.py:25-56)."""
    dims: tuple
    origin: tuple
    spacing: tuple

    @property
    def size(self) -> int:
        return int(np.prod(self.dims))


def _same_points(src: SourcePointSet, obs: ObserverPointSet) -> bool:
    # nearzone.py:241-243
    return src.positions is obs.positions or (
        src.positions.shape == obs.positions.shape and np.array_equal(src.positions, obs.positions))


def problem_struct(cfg: PeriodicityConfig, box: TargetBox, src: SourcePointSet, obs: ObserverPointSet,
                   params: SolverParams, device: int | None = None, parts: int = nat.ALL, far_kernel=None,
                   far_kernel_terms: int = 0):
    """FftpimProblem for the C ABI; returns (struct, same_points, arrays to keep alive).
    `parts` selects the zones to build (build_near_plan / build_far_plan build one,
    nearzone.py:194-273, farzone.py:76-131); `far_kernel` is a far-kernel table read
    from a PIMF blob, used instead of tabulating the series (farzone.py:103-112)."""
    same = _same_points(src, obs)
    pr = nat.Problem()
    pr.dim = cfg.dim.value
    pr.regime = REGIME_CODE[cfg.regime]
    for a in range(3):
        pr.L[a] = cfg.L[a]
        pr.D[a] = box.D[a]
        pr.kshift[a][0] = cfg.kshift[a].real
        pr.kshift[a][1] = cfg.kshift[a].imag
        pr.far_grid[a] = params.far_grid[a]
    pr.k0[0], pr.k0[1] = cfg.k0.real, cfg.k0.imag
    pr.i_d = params.i_d
    pr.near_order = params.near_order
    dims = params.resolve_near_grid(max(len(src), len(obs)), box)
    for a in range(3):
        pr.near_grid[a] = int(dims[a])
    pr.far_order = params.far_order
    pr.series_tol = params.series_tol
    pr.er_range_boxes = params.er_range_boxes
    sp = np.ascontiguousarray(src.positions, dtype=np.float64)
    op = sp if same else np.ascontiguousarray(obs.positions, dtype=np.float64)
    pr.n_src, pr.n_obs = len(src), len(obs)
    pr.src_pos = sp.ctypes.data
    pr.obs_pos = None if same else op.ctypes.data
    pr.same_points = int(same)
    pr.device = _default_device() if device is None else int(device)
    pr.parts = int(parts)
    keep = [sp, op]
    if far_kernel is not None:
        fk = np.ascontiguousarray(far_kernel, dtype=np.complex128)
        keep.append(fk)
        pr.far_kernel = fk.ctypes.data
        pr.far_kernel_terms = int(far_kernel_terms)
    return pr, same, tuple(keep)


class NativePlan:
    """Owns one libfftpim plan (device memory lives until this object dies)."""

    def __init__(self, cfg: PeriodicityConfig, box: TargetBox, src: SourcePointSet,
                 obs: ObserverPointSet, params: SolverParams, device: int | None = None,
                 parts: int = nat.ALL, far_kernel=None, far_kernel_terms: int = 0):
        lib = nat.load()
        self.cfg, self.box, self.params = cfg, box, params
        pr, same, keep = problem_struct(cfg, box, src, obs, params, device, parts, far_kernel, far_kernel_terms)
        self._src_pos, self._obs_pos = keep[0], keep[1]
        self.device = pr.device
        handle = C.c_void_p()
        self._lib = lib
        self._h = None
        nat.check(lib.fftpim_plan_create(C.byref(pr), C.byref(handle)))
        del keep
        self._h = handle
        info = nat.Info()
        nat.check(lib.fftpim_plan_info(self._h, C.byref(info)))
        self.info = info
        self.same_points = same
        self.n_sources, self.n_observers = int(info.n_src), int(info.n_obs)
        if info.on_axis_offset:
            warnings.warn("source cloud lies exactly on the periodic axis; offsetting the source grid "
                          "transversely by half a grid spacing in y (kernel evaluated at that offset)",
                          stacklevel=3)

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._lib is not None:
            self._lib.fftpim_plan_destroy(self._h)
            self._h = None

    # ---------------------------------------------------------------- evaluation
    def evaluate(self, q, parts: int = nat.ALL, out=None):
        """u for one charge vector (N,) or a batch (B, N).  numpy in -> numpy out
        (host path; `out` may be a preallocated, e.g. pinned, complex128 array);
        CUDA tensor in -> CUDA tensor out (device path)."""
        if _is_cuda_tensor(q):
            return self._evaluate_device(q, parts)
        qa = np.ascontiguousarray(np.asarray(q, dtype=np.complex128))
        batch = 1 if qa.ndim == 1 else qa.shape[0]
        if qa.shape[-1] != self.n_sources:
            raise ValueError(f"expected {self.n_sources} amplitudes, got {qa.shape[-1]}")
        shape = (self.n_observers,) if qa.ndim == 1 else (batch, self.n_observers)
        if out is None:
            out = np.empty(shape, dtype=np.complex128)
        elif out.shape != shape or out.dtype != np.complex128 or not out.flags.c_contiguous:
            raise ValueError(f"out must be a C-contiguous complex128 array of shape {shape}")
        nat.check(self._lib.fftpim_plan_evaluate_host(self._h, qa.ctypes.data, out.ctypes.data, batch, parts))
        return out

    def _evaluate_device(self, q, parts):
        import torch
        if q.dtype != torch.complex128:
            q = q.to(torch.complex128)
        q = q.contiguous()
        if q.shape[-1] != self.n_sources:
            raise ValueError(f"expected {self.n_sources} amplitudes, got {q.shape[-1]}")
        batch = 1 if q.dim() == 1 else q.shape[0]
        u = torch.empty((batch, self.n_observers), dtype=torch.complex128, device=q.device)
        stream = torch.cuda.current_stream(q.device).cuda_stream
        nat.check(self._lib.fftpim_plan_evaluate(self._h, q.data_ptr(), u.data_ptr(), batch, parts, stream))
        return u[0] if q.dim() == 1 else u

    def evaluate_into(self, q_ptr: int, u_ptr: int, batch: int = 1, parts: int = nat.ALL, stream: int = 0):
        """Raw device-pointer entry (bench / FFI users)."""
        nat.check(self._lib.fftpim_plan_evaluate(self._h, q_ptr, u_ptr, batch, parts, stream))

    def profile(self, q_ptr: int, u_ptr: int, parts: int = nat.ALL, stream: int = 0) -> dict:
        """Per-stage device milliseconds of one evaluation (CUDA events between stages)."""
        ms = (C.c_double * nat.N_STAGES)()
        nat.check(self._lib.fftpim_plan_profile(self._h, q_ptr, u_ptr, parts, stream, ms))
        return dict(zip(nat.STAGES, list(ms)))

    # ---------------------------------------------------------------- operands
    def export(self, which: int) -> np.ndarray:
        p = int(self.info.n_pairs)
        if which in (nat.PAIR_OBS, nat.PAIR_SRC):
            out = np.empty(p, dtype=np.int32)
        elif which == nat.PAIR_CODE:
            out = np.empty((p, 3), dtype=np.int8)
        elif which == nat.PAIR_COEF:
            out = np.empty(p, dtype=np.complex128)
        elif which == nat.FAR_KERNEL:
            out = np.empty(tuple(2 * d - 1 if d > 1 else 1 for d in self.info.far_dims), dtype=np.complex128)
        elif which == nat.KERNEL_HAT:
            out = np.empty(tuple(self.info.fft_dims), dtype=np.complex128)
        elif nat.NEAR_SRC_START <= which <= nat.FAR_OBS_W:
            k = which - nat.NEAR_SRC_START
            n = self.n_observers if k & 2 else self.n_sources
            width = (self.params.far_order if k >= 4 else self.params.near_order) + 1
            out = np.empty((n, 3, width), dtype=np.float64) if k & 1 else np.empty((n, 3), dtype=np.int32)
        else:
            raise ValueError(f"unknown operand {which}")
        nat.check(self._lib.fftpim_plan_export(self._h, which, out.ctypes.data, out.nbytes))
        return out

    def refresh_info(self):
        """Re-read the plan summary (graph capture counters change with use)."""
        nat.check(self._lib.fftpim_plan_info(self._h, C.byref(self.info)))
        return self.info

    def set_far_kernel(self, kernel: np.ndarray):
        k = np.ascontiguousarray(kernel, dtype=np.complex128)
        nat.check(self._lib.fftpim_plan_set_far_kernel(self._h, k.ctypes.data, k.size))


def _default_device() -> int:
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # noqa: BLE001 - torch is optional for the host path
        pass
    return 0


def _is_cuda_tensor(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


class _LazyPairs:
    def __init__(self, plan: NativePlan, which):
        self._plan, self._which, self._arr = plan, which, None

    def get(self):
        if self._arr is None:
            self._arr = self._plan.export(self._which)
        return self._arr


@dataclass(frozen=True)
class SparseInterpOperator:
    """Stencil data of one point set on one grid (grids.py:143-165 field names), read
    back from the device plan.  A view for inspection and parity checks: projection
    and interpolation themselves run inside `plan.evaluate` on the GPU."""
    grid: UniformGrid
    order: int
    role: str                          # "project" or "interpolate"
    axis_starts: np.ndarray            # (P, 3) int64
    axis_weights: tuple                # (P, q_a + 1) each; (P, 1) ones on single-plane axes

    @property
    def n_points(self) -> int:
        return self.axis_starts.shape[0]

    @property
    def stencil_size(self) -> int:
        return int(np.prod([w.shape[1] for w in self.axis_weights]))

    def _offsets(self):
        return [self.axis_starts[:, a][:, None] + np.arange(self.axis_weights[a].shape[1])[None, :]
                for a in range(3)]

    @property
    def flat_index(self) -> np.ndarray:
        """(P, S) C-order node indices of every stencil tap (grids.py:200-206)."""
        ox, oy, oz = self._offsets()
        _, gy, gz = self.grid.dims
        flat = ox[:, :, None, None] * (gy * gz) + oy[:, None, :, None] * gz + oz[:, None, None, :]
        return flat.astype(np.int32).reshape(self.n_points, -1)

    @property
    def flat_weight(self) -> np.ndarray:
        """(P, S) tensor-product weights (grids.py:207-210)."""
        wx, wy, wz = self.axis_weights
        w3 = wx[:, :, None, None] * wy[:, None, :, None] * wz[:, None, None, :]
        return w3.reshape(self.n_points, -1)


def _operator_view(native, grid, order, role, which_start, which_w) -> SparseInterpOperator:
    starts = native.export(which_start).astype(np.int64)
    w = native.export(which_w)
    weights = tuple(np.ascontiguousarray(w[:, a, :1] if grid.dims[a] == 1 else w[:, a, :]) for a in range(3))
    return SparseInterpOperator(grid, order, role, starts, weights)


class NearZonePlan:
    """Near-zone view of a native plan (nearzone.py:55-124 field names)."""

    def __init__(self, native: NativePlan):
        self.native = native
        info = native.info
        self.cfg, self.box = native.cfg, native.box
        self.i_d = native.params.i_d
        self.order = native.params.near_order
        self.er_range_boxes = native.params.er_range_boxes
        dims = tuple(int(v) for v in info.near_dims)
        self.grid = UniformGrid(dims, (0.0, 0.0, 0.0),
                                tuple(self.box.D[a] / (dims[a] - 1) if dims[a] > 1 else 0.0 for a in range(3)))
        self.box_counts = tuple(max(d - 1, 1) for d in dims)
        self.join_radius = tuple(int(v) for v in info.join_radius)
        self.same_points = native.same_points
        self.n_self_pairs = int(info.n_self_pairs)
        self.n_wrapped_pairs = int(info.n_wrapped_pairs)
        self.coincident_kernel_terms = int(info.coincident_kernel_terms)
        self._lazy = {k: _LazyPairs(native, k) for k in (nat.PAIR_OBS, nat.PAIR_SRC, nat.PAIR_CODE,
                                                          nat.PAIR_COEF, nat.KERNEL_HAT)}
        self._ops = {}

    n_sources = property(lambda self: self.native.n_sources)
    n_observers = property(lambda self: self.native.n_observers)
    pair_obs = property(lambda self: self._lazy[nat.PAIR_OBS].get())
    pair_src = property(lambda self: self._lazy[nat.PAIR_SRC].get())
    pair_code = property(lambda self: self._lazy[nat.PAIR_CODE].get())
    pair_coef = property(lambda self: self._lazy[nat.PAIR_COEF].get())
    kernel_hat = property(lambda self: self._lazy[nat.KERNEL_HAT].get())

    @property
    def d_er(self) -> float:
        """Error-correction range (nearzone.py:204)."""
        active = [a for a in range(3) if self.grid.dims[a] > 1]
        return self.er_range_boxes * max(self.grid.spacing[a] for a in active)

    @property
    def proj_op(self) -> SparseInterpOperator:
        if "proj" not in self._ops:
            self._ops["proj"] = _operator_view(self.native, self.grid, self.order, "project",
                                               nat.NEAR_SRC_START, nat.NEAR_SRC_W)
        return self._ops["proj"]

    @property
    def interp_op(self) -> SparseInterpOperator:
        if "interp" not in self._ops:
            self._ops["interp"] = _operator_view(self.native, self.grid, self.order, "interpolate",
                                                 nat.NEAR_OBS_START, nat.NEAR_OBS_W)
        return self._ops["interp"]

    @property
    def seg_obs(self) -> np.ndarray:
        """Observers owning at least one pair (nearzone.py:470-476)."""
        cnt = np.bincount(self.pair_obs, minlength=self.n_observers)
        return np.nonzero(cnt)[0]

    @property
    def seg_starts(self) -> np.ndarray:
        """reduceat segment starts into the pair arrays (nearzone.py:470-476)."""
        cnt = np.bincount(self.pair_obs, minlength=self.n_observers)
        ends = np.cumsum(cnt)
        return (ends - cnt)[np.nonzero(cnt)[0]]

    @property
    def kernel_disp(self) -> np.ndarray:
        """Raw displacement table (2Nx-1, 2Ny-1, 2Nz-1) (nearzone.py:212-227), recovered from
        the device's kernel_hat by undoing the circulant embedding (nearzone.py:127-147)."""
        dims = self.grid.dims
        c = np.fft.ifftn(self.kernel_hat)
        out = np.zeros(tuple(2 * d - 1 if d > 1 else 1 for d in dims), dtype=complex)
        import itertools
        for neg in itertools.product(*[(0, 1) if d > 1 else (0,) for d in dims]):
            sl_c, sl_k = [], []
            for axis, ng in enumerate(neg):
                n = dims[axis]
                if n == 1:
                    sl_c.append(slice(0, 1)); sl_k.append(slice(0, 1))
                elif not ng:
                    sl_c.append(slice(0, n)); sl_k.append(slice(n - 1, 2 * n - 1))
                else:
                    sl_c.append(slice(n + 1, 2 * n)); sl_k.append(slice(0, n - 1))
            out[tuple(sl_k)] = c[tuple(sl_c)]
        return out


class FarZonePlan:
    """Far-zone view of a native plan (farzone.py:32-52 field names)."""

    def __init__(self, native: NativePlan):
        self.native = native
        info = native.info
        self.cfg, self.box = native.cfg, native.box
        self.i_d = native.params.i_d
        self.order = native.params.far_order
        self.series_tol = native.params.series_tol
        dims = tuple(int(v) for v in info.far_dims)
        h = tuple(self.box.D[a] / dims[a] if self.box.D[a] > 0.0 else 0.0 for a in range(3))
        sy = h[0] / 2.0 if info.on_axis_offset else 0.0
        self.source_grid = UniformGrid(dims, (0.0, sy, 0.0), h)
        self.observer_grid = UniformGrid(dims, tuple(v / 2.0 for v in h), h)
        self.kernel_terms = int(info.kernel_terms)
        self._kernel = None
        self._ops = {}

    n_sources = property(lambda self: self.native.n_sources)
    n_observers = property(lambda self: self.native.n_observers)

    @property
    def kernel(self) -> np.ndarray:
        if self._kernel is None:
            self._kernel = self.native.export(nat.FAR_KERNEL)
        return self._kernel

    @property
    def proj_op(self) -> SparseInterpOperator:
        if "proj" not in self._ops:
            self._ops["proj"] = _operator_view(self.native, self.source_grid, self.order, "project",
                                               nat.FAR_SRC_START, nat.FAR_SRC_W)
        return self._ops["proj"]

    @property
    def interp_op(self) -> SparseInterpOperator:
        if "interp" not in self._ops:
            self._ops["interp"] = _operator_view(self.native, self.observer_grid, self.order, "interpolate",
                                                 nat.FAR_OBS_START, nat.FAR_OBS_W)
        return self._ops["interp"]


@dataclass(frozen=True)
class SolvePlan:
    near: NearZonePlan
    far: FarZonePlan
    build_seconds: float

    @property
    def native(self) -> NativePlan:
        return self.near.native

    def evaluate(self, q):
        """u = eval_near + eval_far (solver.py:24-25), fused on the GPU."""
        return self.native.evaluate(q, nat.ALL)


@dataclass(frozen=True)
class SolveResult:
    field: PotentialField
    plan: SolvePlan
    eval_seconds: float


def _validated_native(cfg, box, src, obs, params, device=None, parts=nat.ALL, kernel_cache=None) -> NativePlan:
    params = params or SolverParams()
    report = validate_problem(cfg, box, src, obs, params)
    if report:
        raise ValidationError(report)
    if kernel_cache is None or not (parts & nat.FAR):
        return NativePlan(cfg, box, src, obs, params, device, parts)
    return _native_with_kernel_cache(cfg, box, src, obs, params, device, parts, kernel_cache)


def _check_provider(provider):
    """The reference threads a SpectralTransformProvider (nearzone.py:29-48) into
    the near-zone FFT; the B200 plan runs its pruned column FFTs on the device and
    has no host transform to replace -- refuse rather than silently ignore it."""
    if provider is not None:
        raise TypeError("the B200 plan transforms on the device: a SpectralTransformProvider "
                        f"({type(provider).__name__}) cannot be plugged in; pass provider=None")


def build_plan(cfg: PeriodicityConfig, box: TargetBox, src: SourcePointSet, obs: ObserverPointSet,
               params: SolverParams | None = None, provider=None, kernel_cache=None,
               device: int | None = None) -> SolvePlan:
    """solver.py:35-45.  `kernel_cache`: PIMF far-kernel blob path (a hit skips the
    far series, a miss tabulates and writes it, farzone.py:103-123).  `provider` must
    be None (see _check_provider)."""
    _check_provider(provider)
    t0 = time.perf_counter()
    native = _validated_native(cfg, box, src, obs, params, device, nat.ALL, kernel_cache)
    return SolvePlan(NearZonePlan(native), FarZonePlan(native), time.perf_counter() - t0)


def solve(cfg, box, src, obs, params=None, provider=None, kernel_cache=None) -> SolveResult:
    """solver.py:48-55."""
    plan = build_plan(cfg, box, src, obs, params, provider, kernel_cache)
    t0 = time.perf_counter()
    u = plan.evaluate(src.amplitudes)
    return SolveResult(PotentialField(u), plan, time.perf_counter() - t0)


def build_near_plan(cfg, box, src, obs, params, provider=None) -> NearZonePlan:
    """nearzone.py:194-197 signature; builds the near zone only (no far series,
    no far buffers).  Validation follows the facade's rules; i_d = 0 builds a
    near-zone-only plan (free-space near kernel, no wrapped copies,
    nearzone.py:205-212, :314), as the reference's bench baseline does
    (cli.py:343-347); the far-zone and D_ER rules only apply for i_d >= 1."""
    _check_provider(provider)
    params = params or SolverParams()
    if params.i_d != 0:
        return NearZonePlan(_validated_native(cfg, box, src, obs, params, parts=nat.NEAR))
    report = validate_problem(cfg, box, src, obs, params)
    rest = tuple(m for m in report.messages if "i_d must be" not in m and "error-correction range" not in m)
    if rest:
        raise ValidationError(type(report)(rest))
    return NearZonePlan(NativePlan(cfg, box, src, obs, params, parts=nat.NEAR))


def eval_near(plan: NearZonePlan, q, provider=None):
    """nearzone.py:490-525: project, FFT convolve, interpolate, correct."""
    _check_provider(provider)
    return plan.native.evaluate(q, nat.NEAR)


def build_far_plan(cfg, box, src, obs, params, cache_path=None) -> FarZonePlan:
    """farzone.py:76-131: the far zone only (no correction pairs, no near FFT
    operands); `cache_path` is the PIMF kernel blob (hit: table and kernel_terms
    from the blob, no series; miss: tabulate and save)."""
    if params is not None and params.i_d < 1:
        raise ValueError("far-zone engine requires i_d >= 1")
    return FarZonePlan(_validated_native(cfg, box, src, obs, params, parts=nat.FAR, kernel_cache=cache_path))


def eval_far(plan: FarZonePlan, q):
    """farzone.py:150-159: project, dense grid sum, interpolate."""
    return plan.native.evaluate(q, nat.FAR)


# ---------------------------------------------------------------- PIMF blob (farzone.py:166-212)
_BLOB_MAGIC = b"PIMF"
_BLOB_VERSION = 1
_HEADER_FMT = "<4sI3IIQQ"


def _kernel_signature(cfg: PeriodicityConfig, box: TargetBox, dims, i_d: int, tol: float) -> int:
    txt = f"{cfg.canonical_key()}|D={box.D!r}|dims={tuple(dims)!r}|i_d={int(i_d)}|tol={tol!r}"
    return int.from_bytes(hashlib.sha256(txt.encode()).digest()[:8], "little")


def save_blob(path, kernel, grid_dims, regime: Regime, signature: int, kernel_terms: int):
    head = struct.pack(_HEADER_FMT, _BLOB_MAGIC, _BLOB_VERSION, *(int(d) for d in kernel.shape),
                       REGIME_CODE[regime], signature, kernel_terms).ljust(64, b"\0")
    with open(path, "wb") as f:
        f.write(head)
        f.write(np.ascontiguousarray(kernel, dtype=np.complex128).tobytes())


def save_far_kernel(plan: FarZonePlan, path):
    dims = plan.source_grid.dims
    sig = _kernel_signature(plan.cfg, plan.box, dims, plan.i_d, plan.series_tol)
    save_blob(path, plan.kernel, dims, plan.cfg.regime, sig, plan.kernel_terms)


def load_far_kernel(path, expect_dims=None, expect_regime=None, expect_signature=None):
    with open(path, "rb") as f:
        head = f.read(64)
        if len(head) < 64:
            raise KernelCacheError("kernel blob truncated (short header)")
        magic, version, d0, d1, d2, code, sig, terms = struct.unpack(
            _HEADER_FMT, head[:struct.calcsize(_HEADER_FMT)])
        if magic != _BLOB_MAGIC:
            raise KernelCacheError(f"bad magic {magic!r}")
        if version != _BLOB_VERSION:
            raise KernelCacheError(f"unsupported blob version {version}")
        if expect_regime is not None and code != REGIME_CODE[expect_regime]:
            raise KernelCacheError("kernel blob regime mismatch")
        if expect_signature is not None and sig != expect_signature:
            raise KernelCacheError("kernel blob signature mismatch")
        shape = (d0, d1, d2)
        if expect_dims is not None:
            want = tuple(2 * d - 1 if d > 1 else 1 for d in expect_dims)
            if shape != want:
                raise KernelCacheError(f"kernel table shape {shape} != expected {want}")
        payload = f.read()
    arr = np.frombuffer(payload, dtype=np.complex128)
    if arr.size != d0 * d1 * d2:
        raise KernelCacheError(f"kernel blob payload has {arr.size} entries, expected {d0 * d1 * d2}")
    return arr.reshape(shape).copy(), int(terms)


def _far_dims(params: SolverParams, box: TargetBox):
    return tuple(params.far_grid[a] if box.D[a] > 0.0 else 1 for a in range(3))


def _native_with_kernel_cache(cfg, box, src, obs, params, device, parts, path) -> NativePlan:
    """farzone.py:103-123: a blob matching this problem (dims, regime, signature)
    supplies the far kernel and kernel_terms and the series is skipped; on a miss
    (no file, or any KernelCacheError) the plan tabulates the kernel and the blob
    is (re)written."""
    dims = _far_dims(params, box)
    sig = _kernel_signature(cfg, box, dims, params.i_d, params.series_tol)
    try:
        kernel, terms = load_far_kernel(path, expect_dims=dims, expect_regime=cfg.regime, expect_signature=sig)
    except (FileNotFoundError, KernelCacheError):
        kernel, terms = None, 0
    native = NativePlan(cfg, box, src, obs, params, device, parts, far_kernel=kernel, far_kernel_terms=terms)
    native.kernel_cache_hit = kernel is not None
    if kernel is None:
        save_far_kernel(FarZonePlan(native), path)
    return native
