"""PIMF far-kernel blob I/O (farzone.py:166-212) without a GPU: the reference's
own round-trip and header-error checks (test_farzone.py:114-135) on our
save/load, and a blob WRITTEN BY THE REFERENCE (tests/golden/make_pimf_golden.py)
read back bit for bit, with the cache signature our builder computes equal to
the one the reference stored -- so a reference-written cache is a hit for us."""
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN

from paper_2312_02376_b200 import KernelCacheError, PeriodicityConfig, Periodicity, Regime, TargetBox
from paper_2312_02376_b200.api import _kernel_signature, load_far_kernel, save_blob

PROBLEM = dict(dim=3, L=(1.0, 1.0, 1.0), D=(1.0, 1.0, 1.0), k0=2.0 * np.pi,
               kshift=(0.2 * np.pi, 0.1 * np.pi, 0.0), far_grid=(6, 6, 6))


def test_reference_blob_reads_bitwise():
    g = np.load(os.path.join(GOLDEN, "ref_far_kernel.npz"))
    kernel, terms = load_far_kernel(os.path.join(GOLDEN, "ref_far_kernel.pimf"), expect_dims=(6, 6, 6),
                                    expect_regime=Regime.DYNAMIC)
    assert kernel.shape == (11, 11, 11)
    np.testing.assert_array_equal(kernel, g["kernel"])
    assert terms == int(g["kernel_terms"])


def test_signature_matches_reference():
    """farzone.py:55-59 + model.py:70-76: same canonical key -> same signature."""
    g = np.load(os.path.join(GOLDEN, "ref_far_kernel.npz"))
    p = PROBLEM
    cfg = PeriodicityConfig(dim=Periodicity(p["dim"]), L=p["L"], k0=p["k0"], kshift=p["kshift"],
                            regime=Regime.DYNAMIC)
    assert _kernel_signature(cfg, TargetBox(p["D"]), p["far_grid"], 1, 1e-10) == int(g["signature"])
    # the signature check of the loader accepts it
    load_far_kernel(os.path.join(GOLDEN, "ref_far_kernel.pimf"), expect_signature=int(g["signature"]))
    with pytest.raises(KernelCacheError):
        load_far_kernel(os.path.join(GOLDEN, "ref_far_kernel.pimf"), expect_signature=int(g["signature"]) ^ 1)


def test_blob_roundtrip_and_header_errors(tmp_path):
    rng = np.random.default_rng(5)
    kernel = rng.standard_normal((11, 11, 11)) + 1j * rng.standard_normal((11, 11, 11))
    path = tmp_path / "kernel.pimf"
    save_blob(path, kernel, (6, 6, 6), Regime.NPSP, 1234, 77)
    loaded, terms = load_far_kernel(path, expect_dims=(6, 6, 6), expect_regime=Regime.NPSP, expect_signature=1234)
    np.testing.assert_array_equal(loaded, kernel)
    assert terms == 77
    raw = path.read_bytes()
    assert raw[:4] == b"PIMF" and len(raw) == 64 + kernel.size * 16
    with pytest.raises(KernelCacheError):
        load_far_kernel(path, expect_dims=(7, 7, 7))
    with pytest.raises(KernelCacheError):
        load_far_kernel(path, expect_regime=Regime.DYNAMIC)
    bad = tmp_path / "bad.pimf"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(KernelCacheError, match="bad magic"):
        load_far_kernel(bad)
    short = tmp_path / "short.pimf"
    short.write_bytes(raw[:40])
    with pytest.raises(KernelCacheError, match="truncated"):
        load_far_kernel(short)
    cut = tmp_path / "cut.pimf"
    cut.write_bytes(raw[:-16])
    with pytest.raises(KernelCacheError, match="payload"):
        load_far_kernel(cut)
    with pytest.raises(FileNotFoundError):
        load_far_kernel(tmp_path / "missing.pimf")
    shutil.copy(path, tmp_path / "copy.pimf")
    assert load_far_kernel(tmp_path / "copy.pimf")[1] == 77
