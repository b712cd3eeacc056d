"""Batched excitation sweep (BASELINE config C5).

The reference evaluates a sweep of Floquet phase shifts as independent plans,
one `build_plan(...)` + `evaluate(q_e)` per excitation (solver.py:24-45).  For
shifts that differ only along one periodic axis the B200 build shares the
geometry, stencils, projection operator and correction-pair list across the
excitations: every pair coefficient (nearzone.py:405-457) is linear in the
image phases exp(-j i_a k_a L_a) (pgf.py:114-123), so the plan stores 2 i_d + 1
phase components per pair and one batched precorrection pass serves all
excitations (`sweep_kernels.cu`); kernel_hat and the far kernel are tabulated
per excitation.  `SweepPlan.evaluate(Q)[e]` equals
`build_plan(cfg_e, ...).evaluate(Q[e])` with `cfg_e.kshift[axis] = shifts[e]`.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import replace

import numpy as np

from . import _native as nat
from .api import problem_struct
from .exceptions import ValidationError
from .problem import ObserverPointSet, PeriodicityConfig, SolverParams, SourcePointSet, TargetBox, validate_problem

MAX_EXCITATIONS = 64


class SweepPlan:
    """One geometry, E <= 64 excitations with shifts along `axis`."""

    def __init__(self, cfg: PeriodicityConfig, box: TargetBox, src: SourcePointSet, obs: ObserverPointSet,
                 params: SolverParams, axis: int, shifts, device: int | None = None):
        lib = nat.load()
        shifts = np.asarray(shifts, dtype=np.complex128).ravel()
        if not 1 <= shifts.size <= MAX_EXCITATIONS:
            raise ValueError(f"a sweep plan holds 1..{MAX_EXCITATIONS} excitations, got {shifts.size}")
        pr, same, keep = problem_struct(cfg, box, src, obs, params, device)
        self._keep = keep
        k = np.ascontiguousarray(np.stack([shifts.real, shifts.imag], axis=1))
        handle = C.c_void_p()
        self._lib, self._h = lib, None
        t0 = time.perf_counter()
        nat.check(lib.fftpim_sweep_create(C.byref(pr), int(axis), int(shifts.size), k.ctypes.data, C.byref(handle)))
        self._h = handle
        self.build_seconds = time.perf_counter() - t0
        info = nat.Info()
        nat.check(lib.fftpim_plan_info(self._h, C.byref(info)))
        self.info = info
        self.axis, self.shifts, self.device = int(axis), shifts, pr.device
        self.n_excitations = int(shifts.size)
        self.n_sources, self.n_observers = int(info.n_src), int(info.n_obs)

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._lib is not None:
            self._lib.fftpim_plan_destroy(self._h)
            self._h = None

    def evaluate_into(self, q_ptr: int, u_ptr: int, stream: int = 0):
        """Raw device pointers: q (E, N) and u (E, M) complex128."""
        nat.check(self._lib.fftpim_sweep_evaluate(self._h, q_ptr, u_ptr, stream))

    def profile(self, q_ptr: int, u_ptr: int, stream: int = 0) -> dict:
        """Device ms: the batched precorrection alone, and one whole sweep
        evaluation (the per-excitation chains overlap the precorrection)."""
        ms = (C.c_double * 2)()
        nat.check(self._lib.fftpim_sweep_profile(self._h, q_ptr, u_ptr, stream, ms))
        return {"corr_sweep": ms[0], "sweep_total": ms[1]}

    def evaluate(self, Q, out=None):
        """U[e] = potential of excitation e.  CUDA tensor in -> CUDA tensor out
        (stream ordered on the current stream); host array in -> host array out
        through fftpim_sweep_evaluate_host (uploads overlap the per-excitation
        chains; pinned buffers, e.g. from torch's pin_memory(), transfer fastest).
        `out`: optional host array (E, M) complex128 to write into."""
        import torch
        shape = (self.n_excitations, self.n_sources)
        if isinstance(Q, torch.Tensor) and Q.is_cuda:
            if tuple(Q.shape) != shape:
                raise ValueError(f"expected charges of shape {shape}, got {tuple(Q.shape)}")
            dev = torch.device("cuda", self.device)
            qd = Q.to(dev, dtype=torch.complex128).contiguous()
            u = torch.empty((self.n_excitations, self.n_observers), dtype=torch.complex128, device=dev)
            self.evaluate_into(qd.data_ptr(), u.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
            return u
        if isinstance(Q, torch.Tensor):
            Q = Q.numpy()
        q = np.asarray(Q)
        if q.shape != shape:
            raise ValueError(f"expected charges of shape {shape}, got {q.shape}")
        if q.dtype != np.complex128 or not q.flags.c_contiguous:
            q = np.ascontiguousarray(q, dtype=np.complex128)
        if out is None:
            out = np.empty((self.n_excitations, self.n_observers), dtype=np.complex128)
        elif out.shape != (self.n_excitations, self.n_observers) or out.dtype != np.complex128 \
                or not out.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous complex128 array of shape (E, M)")
        nat.check(self._lib.fftpim_sweep_evaluate_host(self._h, q.ctypes.data, out.ctypes.data))
        return out


def build_sweep_plan(cfg: PeriodicityConfig, box: TargetBox, src: SourcePointSet, obs: ObserverPointSet,
                     params: SolverParams | None, axis: int, shifts, device: int | None = None) -> SweepPlan:
    """Validate every excitation's configuration like build_plan, then build one sweep plan."""
    params = params or SolverParams()
    for k in np.asarray(shifts, dtype=np.complex128).ravel():
        ks = list(cfg.kshift)
        ks[axis] = complex(k)
        report = validate_problem(replace(cfg, kshift=tuple(ks)), box, src, obs, params)
        if report:
            raise ValidationError(report)
    return SweepPlan(cfg, box, src, obs, params, axis, shifts, device)
