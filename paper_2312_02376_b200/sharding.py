"""Multi-GPU decompositions of the evaluation.

* `SlabGroup` -- C4-style slab decomposition of ONE problem over `world`
  shards (one per GPU, NCCL over NVLink inside libfftpim: all-to-all FFT
  transposes, far-grid all-reduce, interpolation halo), or all shards emulated
  in one process on one GPU (`nccl_id=None`) to check the decomposition.
* `excitation_shard` -- C5-style sharding of independent excitations (each its
  own Floquet shift and plan): round-robin, no collective in the loop.
* `slab_planes` / `fft_columns` restate the C library's partition arithmetic
  (fftpim.cu, build / setup_fft_pipeline_shard) for the host-side tests.

The reference has no counterpart (single-process numpy).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from .api import _is_cuda_tensor, problem_struct
from .exceptions import ValidationError
from .problem import ObserverPointSet, PeriodicityConfig, SolverParams, SourcePointSet, TargetBox, validate_problem

__all__ = ["SlabGroup", "nccl_unique_id", "slab_planes", "fft_columns", "excitation_shard"]


def slab_planes(n0: int, world: int) -> list:
    """Shard r owns near-grid x-planes [X_r, X_{r+1}), X_r = floor(r*n0/world)."""
    return [r * n0 // world for r in range(world + 1)]


def fft_columns(n1: int, n2: int, world: int) -> list:
    """Shard r transforms the (ky, kz) columns [C_r, C_{r+1}) of the doubled (2n1, 2n2) plane."""
    c = (2 * n1) * (2 * n2)
    return [r * c // world for r in range(world + 1)]


def excitation_shard(n_excitations: int, world: int, rank: int) -> list:
    """Excitations handled by `rank` (round-robin; C5: 64 over 1/2/4/8 GPUs)."""
    return list(range(rank, n_excitations, world))


def nccl_unique_id() -> bytes:
    lib = nat.load()
    buf = C.create_string_buffer(128)
    nat.check(lib.fftpim_nccl_unique_id(buf, 128))
    return buf.raw


class SlabGroup:
    """Slab-decomposed plan.  nccl_id=None: emulate all shards on this device."""

    def __init__(self, cfg: PeriodicityConfig, box: TargetBox, src: SourcePointSet, obs: ObserverPointSet,
                 params: SolverParams, world: int, rank: int = 0, nccl_id: bytes | None = None,
                 device: int | None = None):
        lib = nat.load()
        params = params or SolverParams()
        report = validate_problem(cfg, box, src, obs, params)
        if report:
            raise ValidationError(report)
        pr, same, self._keep = problem_struct(cfg, box, src, obs, params, device)
        if not same:
            raise ValueError("slab-decomposed plans need observers == sources")
        self._lib, self._h = lib, None
        self.world, self.rank, self.device = world, rank, pr.device
        self.n_sources, self.n_observers = int(pr.n_src), int(pr.n_obs)
        h = C.c_void_p()
        idbuf = None if nccl_id is None else C.create_string_buffer(nccl_id, 128)
        nat.check(lib.fftpim_group_create(C.byref(pr), world, rank, idbuf, C.byref(h)))
        self._h = h
        self.shards = 1 if nccl_id is not None else world
        self.infos = []
        for k in range(self.shards):
            info = nat.Info()
            nat.check(lib.fftpim_group_info(self._h, k, C.byref(info)))
            self.infos.append(info)

    def __del__(self):
        if getattr(self, "_h", None) is not None:
            self._lib.fftpim_group_destroy(self._h)
            self._h = None

    def evaluate_into(self, q_ptr: int, u_ptr: int, stream: int = 0):
        nat.check(self._lib.fftpim_group_evaluate(self._h, q_ptr, u_ptr, stream))

    def evaluate(self, q):
        """u for the observers this process's shard(s) own (all of them when
        emulating); other entries of the returned array are zero."""
        import torch
        if _is_cuda_tensor(q):
            qd = q.to(torch.complex128).contiguous()
        else:
            qd = torch.from_numpy(np.ascontiguousarray(np.asarray(q, dtype=np.complex128))).to(f"cuda:{self.device}")
        u = torch.zeros(self.n_observers, dtype=torch.complex128, device=qd.device)
        self.evaluate_into(qd.data_ptr(), u.data_ptr(), torch.cuda.current_stream(qd.device).cuda_stream)
        return u if _is_cuda_tensor(q) else u.cpu().numpy()
