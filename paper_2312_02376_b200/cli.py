"""Command-line driver on the B200 path: the reference's
`perisum solve | error-study | bench` (/root/reference/pkg/src/perisum/cli.py)
with the same problem-file keys, CSV layouts, output columns and exit codes,
evaluating through libfftpim.so instead of numpy.

    python -m paper_2312_02376_b200 solve problem.txt [--output u.csv]
    python -m paper_2312_02376_b200 error-study problem.txt --orders 1,3,6
    python -m paper_2312_02376_b200 bench --sizes 10000,20000 --dim 3

Exit codes (cli.py:192-237): 0 ok, 1 validation, 2 kernel-series failure
(Wood anomaly / not converged / separation), 3 file I/O.  The reference's
`convergence` (a per-point series trace) and `gen-coax` (a mesh generator)
are host-side utilities off the evaluation path and are not part of this
build.
"""
from __future__ import annotations

import argparse
import io
import sys
import time
from dataclasses import dataclass, fields, replace

import numpy as np

from .api import build_near_plan, build_plan, eval_near
from .direct import TruncationPolicy, eval_direct
from .exceptions import NotConvergedError, PerisumError, SeparationError, ValidationError, WoodAnomalyError
from .problem import (ObserverPointSet, Periodicity, PeriodicityConfig, Regime, SolverParams, SourcePointSet,
                      TargetBox, validate_problem)

__all__ = ["ProblemFile", "main", "read_sources_csv", "read_observers_csv", "write_sources_csv",
           "write_observers_csv", "write_potentials_csv"]

NUM = "%.17g"   # full double precision in every CSV (cli.py:29)
REGIME_NAMES = {"dynamic": Regime.DYNAMIC, "static-shifted": Regime.STATIC_SHIFTED, "npsp": Regime.NPSP}
SERIES_ERRORS = (WoodAnomalyError, NotConvergedError, SeparationError)


@dataclass
class ProblemFile:
    """Plain-text `key = value` problem description (cli.py:35-114); unknown
    keys are errors, '#' starts a comment."""
    dim: int = 1
    Lx: float = 1.0
    Ly: float = 1.0
    Lz: float = 1.0
    k0_re: float = 0.0
    k0_im: float = 0.0
    kx0_re: float = 0.0
    kx0_im: float = 0.0
    ky0_re: float = 0.0
    ky0_im: float = 0.0
    kz0_re: float = 0.0
    kz0_im: float = 0.0
    regime: str = "npsp"
    Dx: float = 1.0
    Dy: float = 1.0
    Dz: float = 1.0
    i_d: int = 1
    far_order: int = 3
    far_grid: str = "10,10,10"
    near_order: int = 2
    near_grid: str = "auto"
    series_tol: float = 1e-10
    er_range_boxes: int = 1
    sources_path: str = ""
    observers_path: str = ""
    output_path: str = ""

    @classmethod
    def load(cls, path) -> "ProblemFile":
        kinds = {f.name: f.type for f in fields(cls)}
        cast = {"int": int, int: int, "float": float, float: float}
        got = {}
        with open(path) as fh:
            for no, line in enumerate(fh, 1):
                text = line.split("#", 1)[0].strip()
                if not text:
                    continue
                key, sep, val = text.partition("=")
                if not sep:
                    bits = text.split(None, 1)
                    if len(bits) != 2:
                        raise ValueError(f"{path}:{no}: expected 'key = value'")
                    key, val = bits
                key, val = key.strip(), val.strip()
                if key not in kinds:
                    raise ValueError(f"{path}:{no}: unknown key '{key}'")
                got[key] = cast.get(kinds[key], str)(val)
        return cls(**got)

    def config(self) -> PeriodicityConfig:
        return PeriodicityConfig(dim=Periodicity(self.dim), L=(self.Lx, self.Ly, self.Lz),
                                 k0=complex(self.k0_re, self.k0_im),
                                 kshift=(complex(self.kx0_re, self.kx0_im), complex(self.ky0_re, self.ky0_im),
                                         complex(self.kz0_re, self.kz0_im)),
                                 regime=REGIME_NAMES[self.regime])

    def box(self) -> TargetBox:
        return TargetBox((self.Dx, self.Dy, self.Dz))

    def params(self) -> SolverParams:
        near = None if self.near_grid.strip().lower() == "auto" else int_triple(self.near_grid)
        return SolverParams(i_d=self.i_d, far_order=self.far_order, far_grid=int_triple(self.far_grid),
                            near_order=self.near_order, near_grid=near, series_tol=self.series_tol,
                            er_range_boxes=self.er_range_boxes)


def int_triple(text) -> tuple:
    vals = [int(v) for v in str(text).replace(",", " ").split()]
    if len(vals) == 1:
        vals *= 3
    if len(vals) != 3:
        raise ValueError(f"expected 1 or 3 integers, got {text!r}")
    return tuple(vals)


# ---------------------------------------------------------------- CSV (cli.py:133-180)
def _table(path, header: tuple) -> np.ndarray:
    with open(path) as fh:
        first = fh.readline().strip()
        if tuple(c.strip() for c in first.split(",")) != header:
            raise ValueError(f"{path}: expected header {','.join(header)}, got {first!r}")
        body = fh.read().strip()
    if not body:
        return np.zeros((0, len(header)))
    data = np.loadtxt(io.StringIO(body), delimiter=",", ndmin=2)
    if data.shape[1] != len(header):
        raise ValueError(f"{path}: expected {len(header)} columns")
    return data


def read_sources_csv(path) -> SourcePointSet:
    t = _table(path, ("x", "y", "z", "q_re", "q_im"))
    return SourcePointSet(t[:, :3], t[:, 3] + 1j * t[:, 4])


def read_observers_csv(path) -> ObserverPointSet:
    return ObserverPointSet(_table(path, ("x", "y", "z")))


def _rows(fh, header, cols):
    fh.write(header + "\n")
    for row in zip(*cols):
        fh.write(",".join(NUM % v for v in row) + "\n")


def write_sources_csv(path, src: SourcePointSet) -> None:
    p, a = src.positions, src.amplitudes
    with open(path, "w", newline="\n") as fh:
        _rows(fh, "x,y,z,q_re,q_im", (p[:, 0], p[:, 1], p[:, 2], a.real, a.imag))


def write_observers_csv(path, obs: ObserverPointSet) -> None:
    p = obs.positions
    with open(path, "w", newline="\n") as fh:
        _rows(fh, "x,y,z", (p[:, 0], p[:, 1], p[:, 2]))


def write_potentials_csv(stream, positions: np.ndarray, values: np.ndarray) -> None:
    _rows(stream, "x,y,z,u_re,u_im",
          (positions[:, 0], positions[:, 1], positions[:, 2], values.real, values.imag))


class _Out:
    """stdout for '' or '-', else a file (LF line ends)."""

    def __init__(self, path):
        self.path = path

    def __enter__(self):
        self.fh = sys.stdout if not self.path or self.path == "-" else open(self.path, "w", newline="\n")
        return self.fh

    def __exit__(self, *exc):
        if self.fh is not sys.stdout:
            self.fh.close()


def _problem(args) -> ProblemFile:
    pf = ProblemFile.load(args.problem) if getattr(args, "problem", None) else ProblemFile()
    upd = {f.name: getattr(args, f.name) for f in fields(ProblemFile) if getattr(args, f.name, None) is not None}
    return replace(pf, **upd) if upd else pf


def _points(pf: ProblemFile):
    return read_sources_csv(pf.sources_path), read_observers_csv(pf.observers_path)


# ---------------------------------------------------------------- commands
def cmd_solve(args) -> int:
    """cli.py:192-237 on the B200 plan."""
    pf = _problem(args)
    try:
        src, obs = _points(pf)
    except (OSError, ValueError) as e:
        print(f"error: cannot read point sets: {e}" if isinstance(e, OSError) else f"error: {e}", file=sys.stderr)
        return 3
    cfg, box, params = pf.config(), pf.box(), pf.params()
    report = validate_problem(cfg, box, src, obs, params)
    if report:
        for m in report.messages:
            print(f"validation: {m}", file=sys.stderr)
        return 1
    try:
        t0 = time.perf_counter()
        plan = build_plan(cfg, box, src, obs, params, kernel_cache=args.kernel_cache)
        t1 = time.perf_counter()
        u = plan.evaluate(src.amplitudes)
        t2 = time.perf_counter()
    except SERIES_ERRORS as e:
        print(f"kernel series failure: {e}", file=sys.stderr)
        return 2
    except ValidationError as e:
        print(f"validation: {e}", file=sys.stderr)
        return 1
    try:
        with _Out(pf.output_path or args.output) as fh:
            write_potentials_csv(fh, obs.positions, u)
    except OSError as e:
        print(f"error: cannot write output: {e}", file=sys.stderr)
        return 3
    print(f"N={len(src)} M={len(obs)} near_grid={plan.near.grid.dims} far_grid={plan.far.source_grid.dims} "
          f"build={(t1 - t0) * 1e3:.1f}ms eval={(t2 - t1) * 1e3:.1f}ms far_series_terms={plan.far.kernel_terms} "
          f"corrections={plan.native.info.n_pairs}", file=sys.stderr)
    return 0


def cmd_error_study(args) -> int:
    """cli.py:275-317: max relative error of FFT-PIM against the per-pair
    converged sum (device brute force, direct_kernels.cu) over far orders, far
    grids and i_d."""
    pf = _problem(args)
    try:
        src, obs = _points(pf)
    except (OSError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 3
    if len(src) > args.oracle_cap:
        print(f"error: N={len(src)} exceeds the oracle cap {args.oracle_cap}", file=sys.stderr)
        return 1
    cfg, box = pf.config(), pf.box()
    try:
        ref = eval_direct(cfg, src, obs, TruncationPolicy(tol=pf.series_tol * 1e-2))
        if not ref.ok():
            print(f"oracle failures on {len(ref.failures)} pairs (first: {ref.failures[0]})", file=sys.stderr)
            return 2
        scale = float(np.max(np.abs(ref.values)))
        with _Out(args.output) as fh:
            fh.write("order,grid,i_d,max_rel_error\n")
            for i_d in (int(v) for v in args.id_values.split(",")):
                for grid in (int(v) for v in args.grids.split(",")):
                    for order in (int(v) for v in args.orders.split(",")):
                        prm = replace(pf.params(), far_order=order, far_grid=(grid, grid, grid), i_d=i_d)
                        u = build_plan(cfg, box, src, obs, prm).evaluate(src.amplitudes)
                        err = float(np.max(np.abs(u - ref.values))) / scale
                        fh.write(f"{order},{grid},{i_d},{NUM % err}\n")
    except SERIES_ERRORS as e:
        print(f"kernel series failure: {e}", file=sys.stderr)
        return 2
    return 0


def _best(fn, repeats: int) -> float:
    fn()   # warm-up (cli.py:360-366)
    best = float("inf")
    for _ in range(max(1, repeats)):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


def cmd_bench(args) -> int:
    """cli.py:320-357: build and evaluation time per N, and the periodic
    overhead against a free-space (i_d = 0) near-zone-only plan."""
    d = args.box_size
    cfg = PeriodicityConfig(Periodicity(args.dim), (d + args.gap,) * 3)
    box = TargetBox((d, d, d))
    rng = np.random.default_rng(args.seed)
    with _Out(args.output) as fh:
        fh.write("N,build_ms,eval_ms,periodic_overhead_ratio,build_overhead_ratio\n")
        for n in (int(v) for v in args.sizes.split(",")):
            pos = rng.uniform(0.0, d, (n, 3))
            q = rng.uniform(-1.0, 1.0, n)
            q -= q.mean()
            src, obs = SourcePointSet(pos, q), ObserverPointSet(pos)
            t0 = time.perf_counter()
            plan = build_plan(cfg, box, src, obs, SolverParams())
            build_p = time.perf_counter() - t0
            eval_p = _best(lambda: plan.evaluate(q), args.repeats)
            del plan
            t0 = time.perf_counter()
            near0 = build_near_plan(cfg, box, src, obs, SolverParams(i_d=0))
            build_f = time.perf_counter() - t0
            eval_f = _best(lambda: eval_near(near0, q), args.repeats)
            del near0
            fh.write(f"{n},{build_p * 1e3:.3f},{eval_p * 1e3:.3f},{eval_p / eval_f:.4f},{build_p / build_f:.4f}\n")
            fh.flush()
    return 0


def _problem_flags(p: argparse.ArgumentParser) -> None:
    for f in fields(ProblemFile):
        typ = {"int": int, int: int, "float": float, float: float}.get(f.type, str)
        p.add_argument(f"--{f.name}", type=typ, default=None)


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2312_02376_b200", description="FFT-PIM periodic potentials on B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("solve", help="evaluate potentials for a problem file")
    p.add_argument("problem", nargs="?")
    p.add_argument("--output", default="")
    p.add_argument("--kernel-cache", default=None, help="PIMF far-kernel blob (read if valid, else written)")
    _problem_flags(p)
    p.set_defaults(fn=cmd_solve)
    p = sub.add_parser("error-study", help="FFT-PIM error against the brute-force periodic sum")
    p.add_argument("problem", nargs="?")
    p.add_argument("--orders", default="1,3,6")
    p.add_argument("--grids", default="10")
    p.add_argument("--id-values", default="1")
    p.add_argument("--oracle-cap", type=int, default=20000)
    p.add_argument("--output", default="")
    _problem_flags(p)
    p.set_defaults(fn=cmd_error_study)
    p = sub.add_parser("bench", help="timing sweep over problem sizes")
    p.add_argument("--sizes", default="10000,20000,40000,80000")
    p.add_argument("--dim", type=int, default=3)
    p.add_argument("--box-size", type=float, default=100.0)
    p.add_argument("--gap", type=float, default=1.0)
    p.add_argument("--repeats", type=int, default=3)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--output", default="")
    p.set_defaults(fn=cmd_bench)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except PerisumError as e:   # cli.py:469-478
        print(f"error: {e}", file=sys.stderr)
        return 2
    except OSError as e:
        print(f"error: {e}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
