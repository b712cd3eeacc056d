"""Brute-force periodic superposition on the GPU: the reference's accuracy
oracle, same entry points as
/root/reference/pkg/src/perisum/oracle.py:

  eval_direct(cfg, src, obs, policy)              oracle.py:92-97
  eval_direct_farzone(cfg, src, obs, i_d, policy) oracle.py:100-111
  eval_free_space(k0, src, obs)                   oracle.py:114-123

Each (observer, source) pair gets its own converged series (the reference's
adaptive layer driver, pgf.py:166-195) in `direct_kernels.cu`; observers are
walked in chunks of 64 with the reference's failure semantics (a chunk with a
separation failure stays at 0 and reports only those).  O(N*M) work: the tool
for accuracy studies (cli.py:275-317), not an evaluation path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .exceptions import DomainError
from .problem import REGIME_CODE, ObserverPointSet, PeriodicityConfig, SourcePointSet

__all__ = ["TruncationPolicy", "OracleReport", "eval_direct", "eval_direct_farzone", "eval_free_space"]

_REASON = {1: "separation", 2: "not converged"}


@dataclass(frozen=True)
class TruncationPolicy:
    """Adaptive truncation (pgf.py:40-58): stop after `consecutive_small`
    layers each contributing less than `tol` relative to the running sum."""
    tol: float = 1e-10
    max_terms: int = 1_000_000
    consecutive_small: int = 3

    def __post_init__(self):
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.max_terms < 1:
            raise ValueError("max_terms must be >= 1")

    @property
    def inner_cutoff(self) -> float:
        return float(np.log(1.0 / self.tol) + 8.0)


@dataclass(frozen=True)
class OracleReport:
    values: np.ndarray
    worst_terms: int
    failures: tuple          # (observer index, source index, reason)

    def ok(self) -> bool:
        return not self.failures


def _problem(cfg: PeriodicityConfig | None, k0: complex, src: SourcePointSet, obs: ObserverPointSet,
             i_d: int, device: int | None):
    pr = nat.Problem()
    if cfg is not None:
        pr.dim = cfg.dim.value
        pr.regime = REGIME_CODE[cfg.regime]
        for a in range(3):
            pr.L[a] = cfg.L[a]
            pr.kshift[a][0] = complex(cfg.kshift[a]).real
            pr.kshift[a][1] = complex(cfg.kshift[a]).imag
        k0 = cfg.k0
    k0 = complex(k0)
    pr.k0[0], pr.k0[1] = k0.real, k0.imag
    pr.i_d = int(i_d)
    sp = np.ascontiguousarray(src.positions, dtype=np.float64).reshape(-1, 3)
    op = np.ascontiguousarray(obs.positions, dtype=np.float64).reshape(-1, 3)
    pr.n_src, pr.n_obs = len(sp), len(op)
    pr.src_pos = sp.ctypes.data
    pr.obs_pos = op.ctypes.data
    if device is None:
        import torch
        device = torch.cuda.current_device()
    pr.device = int(device)
    return pr, (sp, op)


def _run(pr, keep, mode: int, policy: TruncationPolicy, q: np.ndarray, n_obs: int):
    lib = nat.load()
    q = np.ascontiguousarray(q, dtype=np.complex128).ravel()
    u = np.zeros(n_obs, dtype=np.complex128)
    rep = nat.DirectReport()
    cap = 4096
    while True:
        fails = np.zeros((cap, 3), dtype=np.int64)
        nat.check(lib.fftpim_direct_evaluate(C.byref(pr), mode, float(policy.tol), int(policy.max_terms),
                                             int(policy.consecutive_small), q.ctypes.data, u.ctypes.data,
                                             fails.ctypes.data, cap, C.byref(rep)))
        if rep.n_failures <= cap:
            break
        cap = int(rep.n_failures)   # rare: run again with room for every record
    del keep
    failures = tuple((int(i), int(j), _REASON[int(r)]) for i, j, r in fails[:rep.n_failures])
    return u, int(rep.worst_terms), failures


def eval_direct(cfg: PeriodicityConfig, src: SourcePointSet, obs: ObserverPointSet,
                policy: TruncationPolicy | None = None, device: int | None = None) -> OracleReport:
    """u(r_m) = sum_n G_p(r_m - r_n) q_n with per-pair converged series (oracle.py:92-97)."""
    policy = policy or TruncationPolicy()
    pr, keep = _problem(cfg, 0, src, obs, 0, device)
    u, worst, failures = _run(pr, keep, 0, policy, src.amplitudes, len(obs))
    return OracleReport(values=u, worst_terms=worst, failures=failures)


def eval_direct_farzone(cfg: PeriodicityConfig, src: SourcePointSet, obs: ObserverPointSet, i_d: int,
                        policy: TruncationPolicy | None = None, device: int | None = None) -> OracleReport:
    """Same sum with the far kernel (total minus |i| <= i_d images), oracle.py:100-111."""
    policy = policy or TruncationPolicy()
    pr, keep = _problem(cfg, 0, src, obs, i_d, device)
    u, worst, failures = _run(pr, keep, 1, policy, src.amplitudes, len(obs))
    return OracleReport(values=u, worst_terms=worst, failures=failures)


def eval_free_space(k0: complex, src: SourcePointSet, obs: ObserverPointSet, device: int | None = None) -> np.ndarray:
    """Plain free-space superposition (oracle.py:114-123); ZeroDivisionError when
    an observer coincides with a source."""
    pr, keep = _problem(None, k0, src, obs, 0, device)
    try:
        u, _, _ = _run(pr, keep, 2, TruncationPolicy(), src.amplitudes, len(obs))
    except DomainError as e:
        raise ZeroDivisionError("observer coincides with a source") from e
    return u
