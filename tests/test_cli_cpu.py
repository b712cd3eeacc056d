"""CLI host logic (no GPU): problem files, CSV round trips, the potentials
format and the entry point -- the reference's tests/test_cli.py:48-84, 189-194
on paper_2312_02376_b200.cli."""
import io
import subprocess
import sys

import numpy as np
import pytest

from conftest import REPO
from paper_2312_02376_b200.cli import (ProblemFile, read_observers_csv, read_sources_csv, write_observers_csv,
                                       write_potentials_csv, write_sources_csv)
from paper_2312_02376_b200.problem import ObserverPointSet, SourcePointSet


def test_problem_file_defaults_and_unknown_key(tmp_path):
    p = tmp_path / "p.txt"
    p.write_text("dim = 2\nLx = 3.5\n# comment\nregime = dynamic\nk0_re 1.0\n")
    prob = ProblemFile.load(p)
    assert prob.dim == 2 and prob.Lx == 3.5 and prob.Ly == 1.0 and prob.k0_re == 1.0
    assert prob.far_order == 3 and prob.series_tol == 1e-10
    assert prob.params().near_grid is None and prob.params().far_grid == (10, 10, 10)
    assert prob.config().k0 == 1.0
    bad = tmp_path / "bad.txt"
    bad.write_text("dim = 1\nnosuchkey = 5\n")
    with pytest.raises(ValueError, match="unknown key"):
        ProblemFile.load(bad)


def test_csv_roundtrip_bit_exact(tmp_path, rng):
    pos = rng.uniform(-1, 1, (37, 3)) * 10.0 ** rng.integers(-12, 12, (37, 3))
    q = rng.normal(size=37) * 1e-7 + 1j * rng.normal(size=37) * 1e3
    path = tmp_path / "s.csv"
    write_sources_csv(path, SourcePointSet(pos, q))
    back = read_sources_csv(path)
    assert np.array_equal(back.positions, pos) and np.array_equal(back.amplitudes, q)
    path2 = tmp_path / "o.csv"
    write_observers_csv(path2, ObserverPointSet(pos))
    assert np.array_equal(read_observers_csv(path2).positions, pos)
    bad = tmp_path / "b.csv"
    bad.write_text("x,y\n1,2\n")
    with pytest.raises(ValueError, match="expected header"):
        read_observers_csv(bad)


def test_potentials_csv_format():
    buf = io.StringIO()
    write_potentials_csv(buf, np.array([[0.1, 0.2, 0.3]]), np.array([1.5 - 2.5j]))
    lines = buf.getvalue().split("\n")
    assert lines[0] == "x,y,z,u_re,u_im"
    assert lines[1] == "0.10000000000000001,0.20000000000000001,0.29999999999999999,1.5,-2.5"


def test_console_entry_point():
    r = subprocess.run([sys.executable, "-m", "paper_2312_02376_b200", "--help"], capture_output=True, text=True,
                       cwd=REPO)
    assert r.returncode == 0
    assert "solve" in r.stdout and "error-study" in r.stdout and "bench" in r.stdout
