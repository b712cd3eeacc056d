"""ctypes binding of the C ABI in include/fftpim.h (libfftpim.so, built in-tree
by `__graft_entry__.build()` / `make -C paper_2312_02376_b200/csrc`).

There is no CPU fallback: if the library cannot be loaded every entry point
raises NativeLibraryError.
"""
from __future__ import annotations

import ctypes as C
import os

from .exceptions import (DomainError, KernelCacheError, NativeLibraryError, NotConvergedError,
                         PerisumError, SeparationError, WoodAnomalyError)

LIB_PATH = os.environ.get("FFTPIM_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                                                          "libfftpim.so")

OK, VALIDATION, DOMAIN, WOOD, NOT_CONVERGED, SEPARATION, KERNEL_CACHE, CUDA, VALUE = range(9)
NEAR, FAR, ALL = 1, 2, 3
PAIR_OBS, PAIR_SRC, PAIR_CODE, PAIR_COEF, FAR_KERNEL, KERNEL_HAT = 1, 2, 3, 4, 5, 6
(NEAR_SRC_START, NEAR_SRC_W, NEAR_OBS_START, NEAR_OBS_W,
 FAR_SRC_START, FAR_SRC_W, FAR_OBS_START, FAR_OBS_W) = range(7, 15)


class Problem(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("regime", C.c_int32),
        ("L", C.c_double * 3), ("D", C.c_double * 3),
        ("k0", C.c_double * 2), ("kshift", (C.c_double * 2) * 3),
        ("i_d", C.c_int32), ("near_order", C.c_int32), ("near_grid", C.c_int32 * 3),
        ("far_order", C.c_int32), ("far_grid", C.c_int32 * 3),
        ("series_tol", C.c_double), ("er_range_boxes", C.c_int32),
        ("n_src", C.c_int64), ("n_obs", C.c_int64),
        ("src_pos", C.c_void_p), ("obs_pos", C.c_void_p),
        ("same_points", C.c_int32), ("device", C.c_int32),
        ("parts", C.c_int32), ("reserved_", C.c_int32),
        ("far_kernel", C.c_void_p), ("far_kernel_terms", C.c_int64),
    ]


class Info(C.Structure):
    _fields_ = [
        ("near_dims", C.c_int32 * 3), ("fft_dims", C.c_int32 * 3), ("far_dims", C.c_int32 * 3),
        ("join_radius", C.c_int32 * 3), ("jr_full", C.c_int32), ("on_axis_offset", C.c_int32),
        ("n_src", C.c_int64), ("n_obs", C.c_int64), ("n_pairs", C.c_int64),
        ("n_self_pairs", C.c_int64), ("n_wrapped_pairs", C.c_int64),
        ("coincident_kernel_terms", C.c_int64), ("kernel_terms", C.c_int64),
        ("device_bytes", C.c_int64), ("build_seconds", C.c_double),
        ("real_coefficients", C.c_int32), ("k1_operator", C.c_int32), ("custom_fft", C.c_int32),
        ("k1_slots", C.c_int64),
        ("built_parts", C.c_int32), ("reserved_", C.c_int32),
        ("graph_captures", C.c_int64), ("graph_instantiations", C.c_int64),
        ("k4_wide_groups", C.c_int64),
        ("pair_rows_source_order", C.c_int32), ("reserved2_", C.c_int32),
        ("k4_runs", C.c_int64),
    ]


class DirectReport(C.Structure):
    _fields_ = [("worst_terms", C.c_int64), ("n_failures", C.c_int64), ("n_skipped_chunks", C.c_int64)]


EXPORTED = ("fftpim_plan_create", "fftpim_plan_evaluate", "fftpim_plan_evaluate_host",
            "fftpim_plan_info", "fftpim_plan_export", "fftpim_plan_set_far_kernel",
            "fftpim_plan_destroy", "fftpim_last_error", "fftpim_launch_count", "fftpim_plan_profile",
            "fftpim_nccl_unique_id", "fftpim_group_create", "fftpim_group_evaluate", "fftpim_group_info",
            "fftpim_group_destroy", "fftpim_sweep_create", "fftpim_sweep_evaluate", "fftpim_sweep_info",
            "fftpim_sweep_profile", "fftpim_sweep_evaluate_host", "fftpim_direct_evaluate")
N_STAGES = 9
STAGES = ("permute_q", "far_project", "far_sum", "near_project", "fft_forward", "spectrum_mul",
          "fft_inverse", "corr_matvec", "observers")

_lib = None
_load_error = None


def load(path: str = LIB_PATH):
    """Load libfftpim.so once; raise NativeLibraryError (no fallback) on failure."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        _load_error = f"{path} not found: run __graft_entry__.build() (make -C paper_2312_02376_b200/csrc)"
        raise NativeLibraryError(_load_error)
    try:
        lib = C.CDLL(path)
    except OSError as exc:
        _load_error = str(exc)
        raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
    vp = C.c_void_p
    lib.fftpim_plan_create.argtypes = [C.POINTER(Problem), C.POINTER(vp)]
    lib.fftpim_plan_evaluate.argtypes = [vp, vp, vp, C.c_int64, C.c_int32, vp]
    lib.fftpim_plan_evaluate_host.argtypes = [vp, vp, vp, C.c_int64, C.c_int32]
    lib.fftpim_plan_info.argtypes = [vp, C.POINTER(Info)]
    lib.fftpim_plan_export.argtypes = [vp, C.c_int32, vp, C.c_int64]
    lib.fftpim_plan_set_far_kernel.argtypes = [vp, vp, C.c_int64]
    lib.fftpim_plan_profile.argtypes = [vp, vp, vp, C.c_int32, vp, C.POINTER(C.c_double)]
    lib.fftpim_plan_destroy.argtypes = [vp]
    lib.fftpim_plan_destroy.restype = None
    lib.fftpim_nccl_unique_id.argtypes = [vp, C.c_int64]
    lib.fftpim_group_create.argtypes = [C.POINTER(Problem), C.c_int32, C.c_int32, vp, C.POINTER(vp)]
    lib.fftpim_group_evaluate.argtypes = [vp, vp, vp, vp]
    lib.fftpim_group_info.argtypes = [vp, C.c_int32, C.POINTER(Info)]
    lib.fftpim_group_destroy.argtypes = [vp]
    lib.fftpim_group_destroy.restype = None
    lib.fftpim_sweep_create.argtypes = [C.POINTER(Problem), C.c_int32, C.c_int32, vp, C.POINTER(vp)]
    lib.fftpim_sweep_evaluate.argtypes = [vp, vp, vp, vp]
    lib.fftpim_sweep_info.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    lib.fftpim_sweep_profile.argtypes = [vp, vp, vp, vp, C.POINTER(C.c_double)]
    lib.fftpim_sweep_evaluate_host.argtypes = [vp, vp, vp]
    lib.fftpim_direct_evaluate.argtypes = [C.POINTER(Problem), C.c_int32, C.c_double, C.c_int64, C.c_int32,
                                           vp, vp, vp, C.c_int64, C.POINTER(DirectReport)]
    for name in ("fftpim_nccl_unique_id", "fftpim_group_create", "fftpim_group_evaluate", "fftpim_group_info",
                 "fftpim_sweep_create", "fftpim_sweep_evaluate", "fftpim_sweep_info", "fftpim_sweep_profile",
                 "fftpim_sweep_evaluate_host", "fftpim_direct_evaluate"):
        getattr(lib, name).restype = C.c_int
    lib.fftpim_last_error.restype = C.c_char_p
    lib.fftpim_launch_count.restype = C.c_int64
    for name in ("fftpim_plan_create", "fftpim_plan_evaluate", "fftpim_plan_evaluate_host",
                 "fftpim_plan_info", "fftpim_plan_export", "fftpim_plan_set_far_kernel", "fftpim_plan_profile"):
        getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib


_ERRORS = {DOMAIN: DomainError, WOOD: WoodAnomalyError, NOT_CONVERGED: NotConvergedError,
           SEPARATION: SeparationError, KERNEL_CACHE: KernelCacheError, VALUE: ValueError,
           CUDA: NativeLibraryError}


def check(status: int):
    """Map a C status onto the reference's exception classes (errors.py:4-37)."""
    if status == OK:
        return
    msg = _lib.fftpim_last_error().decode(errors="replace")
    raise _ERRORS.get(status, PerisumError)(msg)


def launch_count() -> int:
    return int(load().fftpim_launch_count())
