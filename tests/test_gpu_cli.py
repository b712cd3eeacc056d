"""The CLI on the B200 path: the reference's
tests/test_cli.py:86-187 scenarios through paper_2312_02376_b200.cli, plus the
solve output checked against the oracle."""
import numpy as np
import pytest

from conftest import rel_l2
from paper_2312_02376_b200.cli import main, write_observers_csv, write_sources_csv
from paper_2312_02376_b200.problem import ObserverPointSet, SourcePointSet

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def gpu():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"


def cloud(tmp_path, rng, n=60, m=8, box=5.0):
    pos = rng.uniform(0, box, (n, 3))
    q = rng.uniform(-1, 1, n)
    q -= q.mean()
    rows = []
    while len(rows) < m:
        cand = rng.uniform(0.3, box - 0.3, (6 * m, 3))
        d = cand[:, None, :] - pos[None, :, :]
        ok = (np.hypot(d[:, :, 1], d[:, :, 2]).min(axis=1) > 0.15) & \
             (np.sqrt(np.einsum("mnk,mnk->mn", d, d)).min(axis=1) > 0.25)
        rows.extend(cand[ok][: m - len(rows)])
    sp, op = tmp_path / "src.csv", tmp_path / "obs.csv"
    write_sources_csv(sp, SourcePointSet(pos, q))
    write_observers_csv(op, ObserverPointSet(np.asarray(rows)))
    return pos, q, np.asarray(rows), sp, op


def problem_text(sp, op, out, box=5.0, extra=""):
    return (f"dim = 1\nLx = {box}\nLy = {box}\nLz = {box}\nregime = npsp\nDx = {box}\nDy = {box}\nDz = {box}\n"
            f"near_grid = 9,9,9\nfar_grid = 6\nsources_path = {sp}\nobservers_path = {op}\noutput_path = {out}\n"
            + extra)


def test_solve_matches_oracle_and_is_permutation_invariant(tmp_path, rng):
    from oracle.pipeline import build_plan as oracle_build
    from oracle.problem import make_problem
    pos, q, obs, sp, op = cloud(tmp_path, rng)
    out1 = tmp_path / "u1.csv"
    (tmp_path / "p1.txt").write_text(problem_text(sp, op, out1))
    assert main(["solve", str(tmp_path / "p1.txt")]) == 0
    u1 = np.loadtxt(out1, delimiter=",", skiprows=1)
    assert np.array_equal(u1[:, :3], obs)
    pb = make_problem(1, L=(5, 5, 5), near_grid=(9, 9, 9), far_grid=(6, 6, 6), near_order=2)
    ref = oracle_build(pb, pos, obs).evaluate(q)
    assert rel_l2(u1[:, 3] + 1j * u1[:, 4], ref) <= 1e-10
    perm = rng.permutation(len(q))
    write_sources_csv(sp, SourcePointSet(pos[perm], q[perm]))
    out2 = tmp_path / "u2.csv"
    (tmp_path / "p2.txt").write_text(problem_text(sp, op, out2))
    assert main(["solve", str(tmp_path / "p2.txt")]) == 0
    u2 = np.loadtxt(out2, delimiter=",", skiprows=1)
    scale = np.abs(u1[:, 3] + 1j * u1[:, 4]).max()
    assert np.max(np.abs(u1 - u2)) <= 1e-14 * max(scale, 1.0)


def test_solve_exit_codes(tmp_path, rng):
    pos, q, obs, sp, op = cloud(tmp_path, rng, n=10, m=3)
    empty = tmp_path / "empty.csv"
    empty.write_text("x,y,z,q_re,q_im\n")
    (tmp_path / "v.txt").write_text(problem_text(empty, op, tmp_path / "u.csv"))
    assert main(["solve", str(tmp_path / "v.txt")]) == 1
    (tmp_path / "io.txt").write_text(problem_text(tmp_path / "missing.csv", tmp_path / "missing2.csv", ""))
    assert main(["solve", str(tmp_path / "io.txt")]) == 3
    pos, q, obs, sp, op = cloud(tmp_path, rng, n=10, m=3, box=1.0)
    (tmp_path / "a.txt").write_text(
        f"dim = 2\nLx = 1\nLy = 1\nLz = 1\nregime = dynamic\nk0_re = {2 * np.pi}\nkx0_re = 0\n"
        f"Dx = 1\nDy = 1\nDz = 1\nnear_grid = 7,7,7\nfar_grid = 5\nfar_order = 2\n"
        f"sources_path = {sp}\nobservers_path = {op}\n")
    assert main(["solve", str(tmp_path / "a.txt")]) == 2   # Wood anomaly


def test_error_study_runs_and_trends(tmp_path, rng):
    pos, q, obs, sp, op = cloud(tmp_path, rng, n=120, m=10)
    (tmp_path / "p.txt").write_text(problem_text(sp, op, ""))
    out = tmp_path / "study.csv"
    assert main(["error-study", str(tmp_path / "p.txt"), "--orders", "1,3", "--grids", "6", "--id-values", "1",
                 "--output", str(out)]) == 0
    rows = out.read_text().strip().split("\n")
    assert rows[0] == "order,grid,i_d,max_rel_error" and len(rows) == 3
    errs = {int(r.split(",")[0]): float(r.split(",")[3]) for r in rows[1:]}
    assert errs[3] < 0.05 and errs[1] < 0.5
    assert main(["error-study", str(tmp_path / "p.txt"), "--oracle-cap", "10"]) == 1


def test_bench_smoke(tmp_path):
    out = tmp_path / "bench.csv"
    assert main(["bench", "--sizes", "400,800", "--dim", "1", "--box-size", "10", "--repeats", "1",
                 "--output", str(out)]) == 0
    rows = out.read_text().strip().split("\n")
    assert rows[0].startswith("N,build_ms,eval_ms,periodic_overhead_ratio") and len(rows) == 3
