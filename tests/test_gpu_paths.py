"""Equivalence of the alternative device paths a plan can select (same inputs,
same plan geometry):

* K1: the plan-time sliced-ELL operator vs the computed (gather / tiled /
  tap-major / line-sweep) projections -- the ELL rows keep the gather order and
  weight expression, so the potentials agree to rounding of the exact-zero
  padding; the line sweep sums in another fixed order (1e-13);
* K2: the register-resident column FFTs (incl. L = 512 as 8 x 8 x 8 and as
  32 x 16) vs the shared-memory Stockham stages vs cuFFT;
* the host entry with pinned buffers (one graph: upload, evaluation,
  download) vs pageable buffers vs the device entry;
* misaligned device buffers are rejected with FFTPIM_VALUE.
Each variant is selected by the environment variable the library reads at
plan build / first launch, in a fresh process (tests/_variant_eval.py)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
RUNNER = os.path.join(HERE, "_variant_eval.py")


def run_variant(case, env_extra, tmp_path, tag):
    out = tmp_path / f"{case}_{tag}.npy"
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, RUNNER, case, str(out)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    info = json.loads(r.stdout.strip().splitlines()[-1])
    return np.load(out), info


@pytest.mark.parametrize("case", ["c1", "c2", "blobs3d", "p2_planar_npsp", "p1_axis_dyn"])
def test_k1_ell_matches_computed_projection(case, tmp_path):
    u_ell, i_ell = run_variant(case, {"FFTPIM_K1": "ell"}, tmp_path, "ell")
    u_gat, i_gat = run_variant(case, {"FFTPIM_K1": "gather"}, tmp_path, "gather")
    assert i_ell["k1_ell"] and not i_gat["k1_ell"]
    assert rel_l2(u_ell, u_gat) <= 1e-14
    # line sweep with in-kernel stencils (line_kernels.cu): same weights, another
    # fixed summation order
    u_lin, i_lin = run_variant(case, {"FFTPIM_K1": "lines"}, tmp_path, "lines")
    assert not i_lin["k1_ell"]
    assert rel_l2(u_lin, u_gat) <= 1e-13
    if case in ("c1", "blobs3d"):
        u_tap, i_tap = run_variant(case, {"FFTPIM_K1": "taps"}, tmp_path, "taps")
        assert rel_l2(u_ell, u_tap) <= 1e-13


@pytest.mark.parametrize("case", ["c1", "c2", "blobs3d", "tri", "g256"])
def test_register_fft_matches_stockham_and_cufft(case, tmp_path):
    u_reg, _ = run_variant(case, {}, tmp_path, "reg")
    if case == "g256":   # L = 512: the 8 x 8 x 8 kernel and in-place E = 32 DFTs vs the default
        u_e32, _ = run_variant(case, {"FFTPIM_FFT_R8": "1"}, tmp_path, "r8")
        assert rel_l2(u_reg, u_e32) <= 1e-13
        u_ip, _ = run_variant(case, {"FFTPIM_FFT_IP": "1"}, tmp_path, "ip")
        assert rel_l2(u_reg, u_ip) <= 1e-13
    u_smem, _ = run_variant(case, {"FFTPIM_FFT_REG": "0"}, tmp_path, "smem")
    if case == "tri":   # the radix-3 register kernels alone switched off
        u_r3, _ = run_variant(case, {"FFTPIM_FFT_REG3": "0"}, tmp_path, "noreg3")
        assert rel_l2(u_reg, u_r3) <= 1e-13
    u_cufft, i_cufft = run_variant(case, {"FFTPIM_FFT": "cufft"}, tmp_path, "cufft")
    assert not i_cufft["custom_fft"]
    assert rel_l2(u_reg, u_smem) <= 1e-13
    assert rel_l2(u_reg, u_cufft) <= 1e-13


@pytest.mark.parametrize("case", ["c1", "c2", "blobs3d"])
def test_k4_16bit_offsets_bitwise(case, tmp_path):
    """K4 with 16-bit source offsets per 32-pair group (int32 for wide groups):
    same pairs, order and arithmetic as the int32 stream -> identical bits."""
    u16, _ = run_variant(case, {"FFTPIM_K4_C16": "1"}, tmp_path, "c16")
    u32, _ = run_variant(case, {"FFTPIM_K4_C16": "0"}, tmp_path, "c32")
    np.testing.assert_array_equal(u16, u32)


@pytest.mark.parametrize("case", ["c2", "blobs3d", "p2_planar_npsp", "p1_axis_dyn", "p3_dyn"])
def test_far_windows_from_the_plan_bitwise(case, tmp_path):
    """Windowed far projection variants.  k_far_project_win2 (plan-time chunk windows,
    staged batches split into runs by ballot) against k_far_project_win (windows
    recomputed, every point tested): same chunks, runs and summation order ->
    identical bits.  k_far_project_win4 (order-3 stencils, four points per warp
    step, group sums added in a fixed shuffle order; opt-in, measured slower) agrees to
    rounding and is bitwise reproducible; all within rounding of the
    stored-weight projection."""
    u2, _ = run_variant(case, {"FFTPIM_FAR": "win", "FFTPIM_FAR_WIN2": "1"}, tmp_path, "win2")
    u1, _ = run_variant(case, {"FFTPIM_FAR": "win"}, tmp_path, "win1")
    u4, _ = run_variant(case, {"FFTPIM_FAR": "win", "FFTPIM_FAR_WIN4": "1"}, tmp_path, "win4")
    u4b, _ = run_variant(case, {"FFTPIM_FAR": "win", "FFTPIM_FAR_WIN4": "1"}, tmp_path, "win4b")
    uw, _ = run_variant(case, {"FFTPIM_FAR": "warps"}, tmp_path, "warps")
    np.testing.assert_array_equal(u2, u1)
    np.testing.assert_array_equal(u4, u4b)
    assert rel_l2(u4, u1) <= 1e-13
    assert rel_l2(u2, uw) <= 1e-13


def test_pageable_host_entry_staged():
    """Pageable caller buffers above 8 MiB go through the plan's pinned staging in
    chunks (host threads copying beside the DMA): bitwise equal to the device
    entry and to pinned buffers."""
    import torch
    import paper_2312_02376_b200 as fp
    rng = np.random.default_rng(300)
    n = 300_000
    pos = rng.uniform(0.0, 1.0, (n, 3))
    q = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity(3), L=(1, 1, 1), k0=2.0 * np.pi,
                               kshift=(0.2 * np.pi, 0.1 * np.pi, 0), regime=fp.Regime("dynamic"))
    plan = fp.build_plan(cfg, fp.TargetBox((1, 1, 1)), fp.SourcePointSet(pos, q), fp.ObserverPointSet(pos),
                         fp.SolverParams(near_grid=(64, 64, 64), near_order=3, far_grid=(6, 6, 6)))
    u_page = plan.evaluate(q)                                     # pageable in, fresh pageable out
    u_page2 = plan.evaluate(q[::-1].copy()[::-1].copy())          # another pageable buffer
    u_dev = plan.evaluate(torch.from_numpy(q).cuda()).cpu().numpy()
    q_pin = torch.from_numpy(q).pin_memory()
    u_pin = torch.empty(n, dtype=torch.complex128).pin_memory()
    plan.native.evaluate(q_pin.numpy(), out=u_pin.numpy())
    np.testing.assert_array_equal(u_page, u_dev)
    np.testing.assert_array_equal(u_page2, u_dev)
    np.testing.assert_array_equal(u_pin.numpy(), u_dev)


def test_host_entries_and_alignment():
    import torch
    import paper_2312_02376_b200 as fp
    from paper_2312_02376_b200 import _native as nat
    from paper_2312_02376_b200.workloads import CONFIGS, make_inputs
    w = CONFIGS[1]
    pos, q = make_inputs(1)
    cfg = fp.PeriodicityConfig(dim=fp.Periodicity(w.dim), L=w.L, k0=w.k0, kshift=w.kshift,
                               regime=fp.Regime(w.regime))
    plan = fp.build_plan(cfg, fp.TargetBox(w.D), fp.SourcePointSet(pos, q), fp.ObserverPointSet(pos),
                         fp.SolverParams(**w.params()))
    nplan = plan.native
    q = q.astype(np.complex128)
    u_page = nplan.evaluate(q)
    q_pin = torch.from_numpy(q).pin_memory()
    u_pin = torch.empty(q.shape[0], dtype=torch.complex128).pin_memory()
    for _ in range(3):   # capture, then replays
        nplan.evaluate(q_pin.numpy(), out=u_pin.numpy())
    u_dev = nplan.evaluate(torch.from_numpy(q).cuda()).cpu().numpy()
    # the pinned host graph's K1 indexes the caller-order charges, the device
    # path's the sorted ones: same rows, same summation order -> bitwise equal
    np.testing.assert_array_equal(u_pin.numpy(), u_page)
    np.testing.assert_array_equal(u_dev, u_page)
    # a new pinned output buffer re-captures the host graph
    u_pin2 = torch.empty_like(u_pin).pin_memory()
    nplan.evaluate(q_pin.numpy(), out=u_pin2.numpy())
    np.testing.assert_array_equal(u_pin2.numpy(), u_page)
    # misaligned device pointers
    buf = torch.zeros(2 * q.shape[0] + 2, dtype=torch.float64, device="cuda")
    good = torch.zeros(2 * q.shape[0], dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match="16-byte aligned"):
        nplan.evaluate_into(buf.data_ptr() + 8, good.data_ptr(), 1, nat.ALL, 0)
