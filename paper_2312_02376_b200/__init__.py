"""B200-native FFT-PIM potential evaluation (drop-in for `perisum`'s hot path).

Same entry points as the reference (/root/reference/pkg/src/perisum/__init__.py):
problem setup with PeriodicityConfig / TargetBox / SourcePointSet /
ObserverPointSet / SolverParams, then `build_plan(...).evaluate(q)`.  Plan
build and evaluation run in hand-written sm_100a kernels (libfftpim.so);
there is no CPU fallback.
"""
from .api import (FarZonePlan, NativePlan, NearZonePlan, SolvePlan, SolveResult, UniformGrid,
                  build_far_plan, build_near_plan, build_plan, eval_far, eval_near, load_far_kernel,
                  save_far_kernel, solve)
from .exceptions import (DomainError, KernelCacheError, NativeLibraryError, NotConvergedError,
                         PerisumError, SeparationError, ValidationError, WoodAnomalyError)
from .direct import OracleReport, TruncationPolicy, eval_direct, eval_direct_farzone, eval_free_space
from .sweep import SweepPlan, build_sweep_plan
from .problem import (ObserverPointSet, Periodicity, PeriodicityConfig, PotentialField, Regime,
                      SolverParams, SourcePointSet, TargetBox, ValidationReport, auto_near_dims,
                      validate_problem)

__version__ = "0.1.0"

__all__ = [
    "FarZonePlan", "NativePlan", "NearZonePlan", "SolvePlan", "SolveResult", "UniformGrid",
    "build_far_plan", "build_near_plan", "build_plan", "eval_far", "eval_near", "load_far_kernel",
    "save_far_kernel", "solve", "DomainError", "KernelCacheError", "NativeLibraryError",
    "NotConvergedError", "PerisumError", "SeparationError", "ValidationError", "WoodAnomalyError",
    "ObserverPointSet", "Periodicity", "PeriodicityConfig", "PotentialField", "Regime",
    "SolverParams", "SourcePointSet", "TargetBox", "ValidationReport", "auto_near_dims",
    "validate_problem", "SweepPlan", "build_sweep_plan", "OracleReport", "TruncationPolicy", "eval_direct",
    "eval_direct_farzone", "eval_free_space",
]
