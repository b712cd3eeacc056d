"""FFT-PIM potential-evaluation benchmark (BASELINE.json metric: source=observer
points/sec per evaluation, HBM-roofline fraction, relative L2 error).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl b200|reference]

A step is one SolvePlan.evaluate (solver.py:24-25) of the config's charge
vector, inputs resident in HBM.  Default workload: configs[3] = C4 (3D-periodic
Helmholtz with phase shift, N = 8,388,608, 256^3 grid, order 4) -- the largest
BASELINE config that fits one B200 (122 GB of correction pairs).  At N > 1 C4 is
slab-decomposed over the ranks (NCCL all-to-all FFT transposes, "scaling":
"strong"); C5 shards its 64 excitations; C1/C2/C3 run replicas ("weak").
`--gpus N` without torchrun re-launches itself under torch.distributed.run.

`--impl reference` times the reference algorithm on the host CPU (the numpy
oracle port; the reference is pure Python/numpy): C1/C2 a full evaluation of the
oracle plan per step; C3/C4/C5 (plans of 35-221 GB that no host builds in
minutes) the composed time of SURVEY.md 8d per step (oracle/composed.py: every
eval stage timed on a bounded sample and scaled to the full size).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_2312_02376_b200.workloads import CONFIGS, c5_kshift, make_inputs  # noqa: E402

METRIC = "source=observer points/sec per FFT-PIM potential eval"
UNIT = "points/s"
HBM_FALLBACK = 6650.0


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def measured_peak():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return HBM_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms (B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if "Active" in s[2 + i]
                          and "Not" not in s[2 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def problem_objects(fp, c, e=0):
    """Config c; for C5 (64 excitations, each its own Floquet shift) excitation e."""
    w = CONFIGS[c]
    pos, q = make_inputs(c)
    kshift = w.kshift
    if w.excitations > 1:
        q, kshift = q[e], c5_kshift(e)
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity(w.dim), L=w.L, k0=w.k0, kshift=kshift,
                               regime=fp.Regime(w.regime))
    return w, pos, q, cfg, fp.TargetBox(w.D), fp.SolverParams(**w.params())


def stage_bytes(w, info, n_far):
    """Algorithmic bytes per evaluation stage.
    q, u and grid values are complex128 (16 B); coefficients 8 B (NPSP) or 16 B."""
    N = M = w.n_points
    ng = int(np.prod(info.near_dims))
    nfft = int(np.prod(info.fft_dims))
    P = int(info.n_pairs)
    sc = 8 if info.real_coefficients else 16
    n0, n1, n2 = (int(v) for v in info.near_dims)
    L0, L1, L2 = (int(v) for v in info.fft_dims)
    a1, a2 = n0 * n1 * L2, n0 * L1 * L2
    fold = 1.0
    for ax in (1, 2):   # G_near is even along an axis without a phase shift (fftpim.cu: fold_y / fold_z)
        if info.near_dims[ax] > 1 and (ax >= w.dim or w.kshift[ax] == 0):
            fold *= 0.5
    return {
        "permute_q": 16 * N + 4 * N + 16 * N,
        "far_project": N * (24 + 16) + 16 * n_far,
        # positions + q read, the n^3 grid written once (the pruned FFT never stores the padding)
        "near_project": N * (24 + 16) + 16 * ng,
        # pruned column stages (K2): the zero padding is never stored.  z: n^3 -> n0 n1 L2,
        # y: -> n0 L1 L2; fused x stage in place on n0 L1 L2 plus the spectrum, read at its folded
        # columns (half per even axis); the inverse mirrors the forward stages
        "fft_forward": 16 * (ng + 2 * a1 + a2),
        "spectrum_mul": 16 * 2 * a2 + int(16 * nfft * fold),
        "fft_inverse": 16 * (ng + 2 * a1 + a2),
        # K4: coefficient + int32 source index per pair, q gathered once, row sums out
        "corr_matvec": P * (sc + 4) + 16 * N + 16 * M,
        # K3 + K5c + fix-up: observer stencil, grid reads, row sums, u written once
        "observers": M * 24 + 16 * ng + 8 * M + 16 * M + 16 * M,
    }


def workload_config(w) -> dict:
    """The `config` dict both arms print (identical keys and values)."""
    cfg = {"workload": w.name, "N": w.n_points, "near_grid": list(w.near_grid), "near_order": w.near_order,
           "regime": w.regime,
           "l2": "inputs larger than L2 (no flush): the correction-pair stream alone is "
                 "0.23 GB (C2) to 122 GB (C4) per evaluation"}
    if w.excitations > 1:
        cfg["excitations"] = w.excitations
    return cfg


def oracle_problem(w, e=0):
    from oracle.problem import make_problem
    kshift = c5_kshift(e) if w.excitations > 1 else w.kshift
    return make_problem(w.dim, L=w.L, D=w.D, k0=w.k0, kshift=kshift, regime=w.regime, **w.params())


def composed_cpu_baseline(w, pos, q, n_pairs=None, reps=3):
    """SURVEY.md 8d composed CPU time of one full evaluation (oracle/composed.py):
    the oracle's numpy eval stages timed on a bounded sample and scaled; best of
    `reps` (cli.py:360-366)."""
    from oracle.composed import ComposedSampler
    s = ComposedSampler(oracle_problem(w), pos, q, n_pairs=n_pairs)
    runs = [s.measure() for _ in range(reps)]
    best, stages = min(runs, key=lambda r: r[0])
    return {"value": w.n_points / best, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": s.describe() + f"; best of {reps}; host nproc={os.cpu_count()}",
            "seconds_per_eval": best, "stages_s": stages, "setup_seconds": s.setup_seconds}


def cpu_baseline_from_plan(w, plan, pos, q, budget_s=20.0):
    """Time the oracle's evaluation (the reference algorithm: eval_near + eval_far,
    nearzone.py:490-525 + farzone.py:150-159) on this host's CPU with the plan
    operands exported from the GPU plan (identical pair lists -- tests pin that)."""
    from oracle import far_engine as fe
    from oracle import near_engine as ne
    from oracle.lagrange import far_grids, make_stencil, near_grid
    from oracle.problem import make_problem
    pb = make_problem(w.dim, L=w.L, D=w.D, k0=w.k0, kshift=w.kshift, regime=w.regime, **w.params())
    nat = plan.native
    dims = tuple(int(v) for v in nat.info.near_dims)
    grid = near_grid(pb.D, dims)
    margin = tuple(1e-9 * max(grid.spacing[a], 1.0) for a in range(3))
    st = make_stencil(grid, pos, pb.near_order, margin)
    p_obs = plan.near.pair_obs
    cnt = np.bincount(p_obs, minlength=len(pos))
    seg_obs = np.nonzero(cnt)[0]
    seg_starts = (np.cumsum(cnt) - cnt)[seg_obs]
    near = ne.NearPlan(pb, grid, st, st, None, plan.near.kernel_hat, None, None, None, p_obs,
                       plan.near.pair_src, plan.near.pair_code, plan.near.pair_coef, seg_obs, seg_starts, 0, 0, 0)
    fdims = tuple(pb.far_grid[a] if pb.D[a] > 0.0 else 1 for a in range(3))
    sg, og = far_grids(pb.D, fdims)
    fm = tuple(sg.spacing[a] if sg.dims[a] > 1 else 0.0 for a in range(3))
    far = fe.FarPlan(pb, sg, og, make_stencil(sg, pos, pb.far_order, fm), make_stencil(og, pos, pb.far_order, fm),
                     plan.far.kernel, plan.far.kernel_terms)
    times, u = [], None
    t_start = time.perf_counter()
    while len(times) < 5 and (len(times) < 2 or time.perf_counter() - t_start < budget_s):
        t0 = time.perf_counter()
        u = ne.eval_near(near, q) + fe.eval_far(far, q)
        times.append(time.perf_counter() - t0)
    best = min(times)
    return {"value": w.n_points / best, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{len(times)} full {w.name} evaluations (N={w.n_points}) of the numpy oracle "
                      f"(reference algorithm, single-threaded numpy eval loops; host nproc={os.cpu_count()}), "
                      f"plan operands exported from the GPU plan; best of {len(times)} (cli.py:360-366)",
            "seconds_per_eval": best}, u


def run_b200(args):
    import torch
    import torch.distributed as dist
    import paper_2312_02376_b200 as fp
    from paper_2312_02376_b200 import _native as nat

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # C5: excitations sharded over ranks (rank r evaluates excitation r); others replicas
    w, pos, q, cfg, box, prm = problem_objects(fp, args.config, e=rank if args.config == 5 else 0)
    t0 = time.perf_counter()
    plan = fp.build_plan(cfg, box, fp.SourcePointSet(pos, q), fp.ObserverPointSet(pos), prm, device=local)
    build_s = time.perf_counter() - t0
    info = plan.native.info
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    q_dev = torch.from_numpy(q).to(f"cuda:{local}")
    u_dev = torch.empty(w.n_points, dtype=torch.complex128, device=f"cuda:{local}")
    nplan = plan.native

    def step():
        nplan.evaluate_into(q_dev.data_ptr(), u_dev.data_ptr(), 1, nat.ALL, sptr)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = nat.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = (nat.launch_count() - launches0) // args.steps
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * w.n_points / (ms_max * 1e-3)

    # per-stage device times (events between stages, same stream), averaged
    prof = {k: 0.0 for k in nat.STAGES}
    reps = 10
    for _ in range(reps):
        for k, v in nplan.profile(q_dev.data_ptr(), u_dev.data_ptr(), nat.ALL, sptr).items():
            prof[k] += v / reps
    nbytes = stage_bytes(w, info, int(np.prod(info.far_dims)))
    own = {k: v for k, v in prof.items() if not k.startswith("fft_") and k in nbytes}
    dom = max(own, key=own.get)
    peak, peak_kind = measured_peak()
    achieved = nbytes[dom] / (prof[dom] * 1e-3) / 1e9
    traffic = None
    summ = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(summ):
        try:
            traffic = json.load(open(summ)).get(f"C{args.config}", {}).get(dom)
        except Exception:  # noqa: BLE001
            traffic = None

    # end to end through the public API with host buffers (pinned), H2D + D2H inside
    q_pin = torch.from_numpy(q).pin_memory()
    u_pin = torch.empty(w.n_points, dtype=torch.complex128).pin_memory()
    q_host, u_host = q_pin.numpy(), u_pin.numpy()
    for _ in range(2):
        plan.native.evaluate(q_host, out=u_host)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        plan.native.evaluate(q_host, out=u_host)
    e2e_s = (time.perf_counter() - t0) / args.steps
    te = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * w.n_points / float(te.item())
    # the stock drop-in call: plan.evaluate(q_numpy) with pageable buffers and a
    # fresh output array per call (what a reference user writes, solver.py:24-25)
    n_pg = max(2, min(args.steps, 10))
    plan.evaluate(q)
    t0 = time.perf_counter()
    for _ in range(n_pg):
        plan.evaluate(q)
    e2e_pageable = world * w.n_points / ((time.perf_counter() - t0) / n_pg)

    # parity of this very run against the reference's own output (C1/C2 full,
    # C3/C4/C5 on the reference's seeded observer sample)
    rel, rel_basis = None, None
    gpath = os.path.join(REPO, "tests", "golden", f"c{args.config}_full.npz")
    spath = os.path.join(REPO, "tests", "golden", f"c{args.config}_subset.npz")
    got = u_dev.cpu().numpy()
    if os.path.exists(gpath):
        ref = np.load(gpath)["u"]
        rel, rel_basis = float(np.linalg.norm(got - ref) / np.linalg.norm(ref)), "all observers"
    elif os.path.exists(spath):
        g = np.load(spath)
        ref, idx = g["u"], g["obs_index"]
        rel = float(np.linalg.norm(got[idx] - ref) / np.linalg.norm(ref))
        rel_basis = f"{len(idx)} seeded observers (reference subset run)"

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if int(info.n_pairs) < 10**8:     # C1/C2: full oracle evaluations
            cpu, u_cpu = cpu_baseline_from_plan(w, plan, pos, q)
            if rel is None:
                rel = float(np.linalg.norm(u_dev.cpu().numpy() - u_cpu) / np.linalg.norm(u_cpu))
        else:                             # C3/C4/C5: composed
            cpu = composed_cpu_baseline(w, pos, q, n_pairs=int(info.n_pairs))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "complex128/f64", "data": "synthetic (seeded, workloads.py)",
            "config": workload_config(w), "pairs": int(info.n_pairs), "parallelism": f"replicas x{world}",
            "rel_l2_vs_reference": rel, "rel_l2_basis": rel_basis,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind, "traffic": traffic,
                         "algorithmic_bytes": nbytes[dom], "kernel_ms": prof[dom]},
            "stages_ms": prof,
            "schedule": ("one CUDA graph: near chain (high-priority stream) | K4 (low priority, capped grid) | "
                         "far chain, split observer pass" if int(info.n_pairs) <= 500_000_000 else
                         "chains in order (K4 uses the whole chip)"),
            "stage_gbs": {k: nbytes[k] / (prof[k] * 1e-3) / 1e9 for k in nbytes if prof.get(k, 0) > 0},
            # SURVEY.md 8d "end to end": every stage's algorithmic bytes over the whole step time
            "roofline_whole_evaluation": {"algorithmic_bytes": int(sum(nbytes.values())),
                                          "achieved": sum(nbytes.values()) / (ms_max * 1e-3) / 1e9, "unit": "GB/s",
                                          "frac": sum(nbytes.values()) / (ms_max * 1e-3) / 1e9 / peak},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 16 * w.n_points,
                    "d2h_bytes_per_step": 16 * w.n_points, "buffers": "pinned host (evaluate(q, out=u))"},
            "e2e_pageable": {"value": e2e_pageable, "unit": UNIT, "calls": n_pg,
                             "buffers": "pageable numpy, fresh output per call (plan.evaluate(q))"},
            "gpu_launches": int(launches),
            "build_seconds": build_s, "plan_device_bytes": int(info.device_bytes),
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_slab(args):
    """C4 partitioned over the ranks: near-grid x-slabs, NCCL all-to-all FFT
    transposes, far-grid all-reduce, halo.  Total work fixed:
    'scaling': 'strong'."""
    import torch
    import torch.distributed as dist
    import paper_2312_02376_b200 as fp
    from paper_2312_02376_b200 import _native as nat
    from paper_2312_02376_b200.sharding import SlabGroup, nccl_unique_id

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w, pos, q, cfg, box, prm = problem_objects(fp, args.config)
    blob = [nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(blob, src=0)
    t0 = time.perf_counter()
    grp = SlabGroup(cfg, box, fp.SourcePointSet(pos, q), fp.ObserverPointSet(pos), prm, world=world, rank=rank,
                    nccl_id=blob[0], device=local)
    build_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    q_dev = torch.from_numpy(q).to(f"cuda:{local}")
    u_dev = torch.zeros(w.n_points, dtype=torch.complex128, device=f"cuda:{local}")

    def step():
        grp.evaluate_into(q_dev.data_ptr(), u_dev.data_ptr(), stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = nat.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = (nat.launch_count() - launches0) // args.steps
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=f"cuda:{local}")
    # e2e: every rank uploads the (replicated) charges from pinned host memory,
    # evaluates its slab and downloads the potential buffer (its own observers)
    q_pin = torch.from_numpy(q).pin_memory()
    u_pin = torch.empty(w.n_points, dtype=torch.complex128).pin_memory()
    q_e2e = torch.empty_like(q_dev)
    u_e2e = torch.zeros_like(u_dev)

    def e2e_step():
        q_e2e.copy_(q_pin, non_blocking=True)
        grp.evaluate_into(q_e2e.data_ptr(), u_e2e.data_ptr(), stream.cuda_stream)
        u_pin.copy_(u_e2e, non_blocking=True)
        stream.synchronize()

    e2e_step()
    if world > 1:
        dist.barrier()
    te0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    te = torch.tensor([(time.perf_counter() - te0) / args.steps], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        dist.all_reduce(u_dev)   # each rank holds only its own observers
    ms = float(t.item())
    rel, basis = None, None
    spath = os.path.join(REPO, "tests", "golden", f"c{args.config}_subset.npz")
    if rank == 0 and os.path.exists(spath):
        g = np.load(spath)
        got = u_dev.cpu().numpy()[g["obs_index"]]
        rel = float(np.linalg.norm(got - g["u"]) / np.linalg.norm(g["u"]))
        basis = f"{len(g['obs_index'])} seeded observers (reference subset run)"
    pairs = torch.tensor([sum(int(i.n_pairs) for i in grp.infos)], dtype=torch.int64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(pairs)
    if rank == 0:
        P = int(pairs.item())
        peak, peak_kind = measured_peak()
        print(json.dumps({
            "metric": METRIC, "value": w.n_points / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "complex128/f64", "data": "synthetic (seeded, workloads.py)",
            "config": workload_config(w), "pairs": P, "parallelism": f"slab x{world} (NCCL all-to-all)",
            "rel_l2_vs_reference": rel, "rel_l2_basis": basis,
            "roofline": {"bound": "hbm", "kernel": "whole evaluation (correction stream dominated)",
                         "achieved": P * 20 / (ms * 1e-3) / 1e9 / world, "peak": peak, "unit": "GB/s",
                         "frac": P * 20 / (ms * 1e-3) / 1e9 / world / peak, "peak_kind": peak_kind, "traffic": None},
            "e2e": {"value": w.n_points / float(te.item()), "unit": UNIT, "h2d_bytes_per_step": 16 * w.n_points,
                    "d2h_bytes_per_step": 16 * w.n_points},
            "gpu_launches": int(launches), "build_seconds": build_s, "clocks": clocks.summary(),
            "cpu_baseline": None}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_sweep(args):
    """C5: the 64-excitation sweep.  Excitations are sharded over the ranks
    (sharding.excitation_shard); each rank holds one SweepPlan (shared geometry and pair
    list, phase-factorised coefficients, batched precorrection) and evaluates its
    block; no collective in the loop.  Total work fixed: 'scaling': 'strong'."""
    import torch
    import torch.distributed as dist
    import paper_2312_02376_b200 as fp
    from paper_2312_02376_b200 import _native as nat

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = CONFIGS[args.config]
    pos, qall = make_inputs(args.config)
    from paper_2312_02376_b200.sharding import excitation_shard
    E = w.excitations
    es = excitation_shard(E, world, rank)
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity(w.dim), L=w.L, k0=w.k0, kshift=c5_kshift(es[0]),
                               regime=fp.Regime(w.regime))
    t0 = time.perf_counter()
    sw = fp.build_sweep_plan(cfg, fp.TargetBox(w.D), fp.SourcePointSet(pos, qall[es[0]]), fp.ObserverPointSet(pos),
                             fp.SolverParams(**w.params()), 0, [c5_kshift(e)[0] for e in es], device=local)
    build_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    q_host = np.ascontiguousarray(qall[es])
    q_dev = torch.from_numpy(q_host).to(f"cuda:{local}")
    u_dev = torch.empty((len(es), w.n_points), dtype=torch.complex128, device=f"cuda:{local}")

    def step():
        sw.evaluate_into(q_dev.data_ptr(), u_dev.data_ptr(), stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = nat.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = (nat.launch_count() - launches0) // args.steps
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    prof = sw.profile(q_dev.data_ptr(), u_dev.data_ptr(), stream.cuda_stream)
    # e2e: the public API with host buffers (H2D of all charge vectors, D2H of all potentials)
    q_pin = torch.from_numpy(q_host).pin_memory()
    u_pin = torch.empty((len(es), w.n_points), dtype=torch.complex128).pin_memory()
    sw.evaluate(q_pin.numpy(), out=u_pin.numpy())
    if world > 1:
        dist.barrier()
    te0 = time.perf_counter()
    for _ in range(max(1, min(args.steps, 3))):
        sw.evaluate(q_pin.numpy(), out=u_pin.numpy())
    te = torch.tensor([(time.perf_counter() - te0) / max(1, min(args.steps, 3))], dtype=torch.float64,
                      device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = composed_cpu_baseline(w, pos, qall[es[0]], n_pairs=int(sw.info.n_pairs))
        cpu["sample"] = "per excitation (the sweep's unit): " + cpu["sample"]
    rel, basis = None, None
    spath = os.path.join(REPO, "tests", "golden", f"c{args.config}_subset.npz")
    if rank == 0 and os.path.exists(spath):
        g = np.load(spath)
        got = u_dev[0].cpu().numpy()[g["obs_index"]]
        rel = float(np.linalg.norm(got - g["u"]) / np.linalg.norm(g["u"]))
        basis = f"excitation 0 on {len(g['obs_index'])} seeded observers (reference subset run)"
    if rank == 0:
        P = int(sw.info.n_pairs)
        nc = 2 * w.params()["i_d"] + 1
        peak, peak_kind = measured_peak()
        k4_bytes = P * (16 * nc + 4) + 2 * 16 * w.n_points * len(es) + 16 * w.n_points * len(es)
        achieved = k4_bytes / (prof["corr_sweep"] * 1e-3) / 1e9
        k4_flops = 8.0 * nc * P * len(es) + 8.0 * (nc + 2) * w.n_points * len(es)
        print(json.dumps({
            "metric": METRIC, "value": E * w.n_points / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "complex128/f64",
            "data": "synthetic (seeded, workloads.py)",
            "config": workload_config(w), "pairs": P,
            "parallelism": f"excitation shards x{world} (sweep plans: phase-factorised pairs)",
            "step": f"one sweep evaluation of {len(es)} excitations per rank "
                    f"(coefficient components {P * 16 * nc / 1e9:.0f} GB streamed)",
            "rel_l2_vs_reference": rel, "rel_l2_basis": basis,
            "roofline": {"bound": "hbm", "kernel": "corr_sweep (batched precorrection)", "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak, "peak_kind": peak_kind,
                         "traffic": None, "algorithmic_bytes": k4_bytes, "kernel_ms": prof["corr_sweep"],
                         "fp64_tflops": k4_flops / (prof["corr_sweep"] * 1e-3) / 1e12},
            "stages_ms": prof,
            "schedule": "batched precorrection (FP64-bound) on a low-priority stream, per-excitation "
                        "chains on a high-priority stream, then one K4-sum pass",
            "e2e": {"value": E * w.n_points / float(te.item()), "unit": UNIT,
                    "h2d_bytes_per_step": 16 * w.n_points * len(es), "d2h_bytes_per_step": 16 * w.n_points * len(es)},
            "gpu_launches": int(launches), "build_seconds": build_s, "clocks": clocks.summary(),
            "cpu_baseline": cpu}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_batch(args):
    """Multi-RHS: one plan, B charge vectors per step (B >= 8 streams the pairs once
    per 64 vectors, DESIGN.md 6b').  Row 0 is the config's own charge vector (its
    parity against the reference is reported), rows 1.. are seeded N(0,1)."""
    import torch
    import torch.distributed as dist
    import paper_2312_02376_b200 as fp
    from paper_2312_02376_b200 import _native as nat

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B = args.batch
    w, pos, q, cfg, box, prm = problem_objects(fp, args.config, e=0)
    t0 = time.perf_counter()
    plan = fp.build_plan(cfg, box, fp.SourcePointSet(pos, q), fp.ObserverPointSet(pos), prm, device=local)
    build_s = time.perf_counter() - t0
    info = plan.native.info
    rng = np.random.default_rng(1000 + args.config)
    Q = rng.standard_normal((B, w.n_points)) + 1j * rng.standard_normal((B, w.n_points))
    Q[0] = q
    Q = np.ascontiguousarray(Q)
    stream = torch.cuda.current_stream()
    q_dev = torch.from_numpy(Q).to(f"cuda:{local}")
    u_dev = torch.empty((B, w.n_points), dtype=torch.complex128, device=f"cuda:{local}")

    def step():
        plan.native.evaluate_into(q_dev.data_ptr(), u_dev.data_ptr(), B, nat.ALL, stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = nat.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = (nat.launch_count() - launches0) // args.steps
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    q_pin = torch.from_numpy(Q).pin_memory()
    u_pin = torch.empty((B, w.n_points), dtype=torch.complex128).pin_memory()
    for _ in range(2):
        plan.native.evaluate(q_pin.numpy(), out=u_pin.numpy())
    te0 = time.perf_counter()
    n_e2e = max(1, min(args.steps, 5))
    for _ in range(n_e2e):
        plan.native.evaluate(q_pin.numpy(), out=u_pin.numpy())
    te = torch.tensor([(time.perf_counter() - te0) / n_e2e], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    rel, basis = None, None
    got = u_dev[0].cpu().numpy()
    for name, key in ((f"c{args.config}_full.npz", None), (f"c{args.config}_subset.npz", "obs_index")):
        p = os.path.join(REPO, "tests", "golden", name)
        if os.path.exists(p) and rel is None:
            g = np.load(p)
            idx = g[key] if key else slice(None)
            rel = float(np.linalg.norm(got[idx] - g["u"]) / np.linalg.norm(g["u"]))
            basis = "row 0, " + ("all observers" if key is None else f"{len(g[key])} seeded observers")
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": world * B * w.n_points / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "complex128/f64",
            "data": "synthetic (seeded, workloads.py; rows 1.. seeded N(0,1))",
            "config": dict(workload_config(w), batch=B), "pairs": int(info.n_pairs),
            "parallelism": f"replicas x{world}", "step": f"one evaluate call with {B} charge vectors (multi-RHS)",
            "rel_l2_vs_reference": rel, "rel_l2_basis": basis,
            "e2e": {"value": world * B * w.n_points / float(te.item()), "unit": UNIT,
                    "h2d_bytes_per_step": 16 * B * w.n_points, "d2h_bytes_per_step": 16 * B * w.n_points},
            "gpu_launches": int(launches), "build_seconds": build_s, "clocks": clocks.summary(),
            "cpu_baseline": None}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def arm_scaling(config: int, world: int) -> str:
    """C4 at N > 1 is one partitioned problem (slabs) and C5 shards one fixed sweep:
    total work fixed ("strong"); replicas otherwise ("weak")."""
    return "strong" if (config == 4 and world > 1) or config == 5 else "weak"


def run_reference(args):
    """Reference algorithm on the host CPU (numpy oracle port; the reference itself
    is Python and is not shipped to the GPU box).  Rank 0 alone runs; other ranks
    exit without work.  C1/C2: each step one full evaluation of the oracle plan
    (built once, multi-process).  C3/C4/C5: each step one composed evaluation
    (oracle/composed.py); C5 counts its 64 excitations per step, each
    costing one per-excitation evaluation (same geometry and pair count)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w = CONFIGS[args.config]
    pos, q = make_inputs(args.config)
    if w.excitations > 1:
        q = q[0]
    extra = {}
    if args.config in (1, 2):
        from oracle.parallel import build_plan_parallel
        t0 = time.perf_counter()
        plan = build_plan_parallel(oracle_problem(w), pos)
        build_s = time.perf_counter() - t0
        for _ in range(args.warmup):
            plan.evaluate(q)
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            plan.evaluate(q)
            times.append(time.perf_counter() - t0)
        sample = (f"each step = one full {w.name} evaluation by the numpy oracle (reference algorithm; its eval "
                  f"loops are single-threaded numpy); plan built once by the oracle over {os.cpu_count()} "
                  f"processes in {build_s:.1f} s")
        extra["pairs"] = int(plan.near.pair_obs.size)
    else:
        from oracle.composed import ComposedSampler
        t0 = time.perf_counter()
        s = ComposedSampler(oracle_problem(w), pos, q)
        build_s = time.perf_counter() - t0
        for _ in range(args.warmup):
            s.measure()
        times, stages = [], []
        for _ in range(args.steps):
            sec, st = s.measure()
            times.append(sec * w.excitations)
            stages.append(st)
        sample = (f"each step = " + (f"{w.excitations} x " if w.excitations > 1 else "") +
                  "one " + s.describe() + f"; sampled operands prepared once in {build_s:.1f} s")
        extra["pairs_estimated"] = s.P
        extra["stages_s_median"] = {k: float(np.median([x[k] for x in stages])) for k in stages[0]}
    sec = float(np.median(times))
    value = w.excitations * w.n_points / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": arm_scaling(args.config, world), "vs_baseline": None, "dtype": "complex128/f64",
        "data": "synthetic (seeded, workloads.py)",
        "config": workload_config(w),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "build_seconds": build_s,
    }
    line.update(extra)
    print(json.dumps(line))


def relaunch_distributed(args) -> int:
    """`--gpus N` outside torchrun: run this script under torch.distributed.run with
    N ranks on this node (the driver's own launch line)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # defaults: sub-millisecond single evaluations (C1, C2) time 200 steps after 20
    # warm-up steps (a 20-step window is a few ms, dominated by clock ramp and
    # first-replay effects); everything else 20 after 5
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--slab", action="store_true", help="slab-decomposed group (NCCL) even on one GPU")
    ap.add_argument("--batch", type=int, default=1,
                    help="multi-RHS: B charge vectors per evaluate call on one plan (C1-C4; C5 uses --per-excitation)")
    ap.add_argument("--per-excitation", action="store_true",
                    help="C5: one ordinary plan per excitation (rank r evaluates excitation r) instead of the sweep")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args))
    short = args.impl == "b200" and args.config in (1, 2) and args.batch == 1 and not args.slab
    if args.steps is None:
        args.steps = 200 if short else 20
    if args.warmup is None:
        args.warmup = 20 if short else 5
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.slab or (args.config == 4 and int(os.environ.get("WORLD_SIZE", 1)) > 1):
        run_slab(args)
    elif args.batch > 1:
        run_batch(args)
    elif args.config == 5 and not args.per_excitation:
        run_sweep(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
