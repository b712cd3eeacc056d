"""Host logic of the brute-force oracle facade (no GPU): the truncation policy
mirrors pgf.py:40-58 and the report mirrors oracle.py:23-29."""
import numpy as np
import pytest

from paper_2312_02376_b200.direct import OracleReport, TruncationPolicy


def test_truncation_policy_validation_and_cutoff():
    p = TruncationPolicy()
    assert (p.tol, p.max_terms, p.consecutive_small) == (1e-10, 1_000_000, 3)
    assert p.inner_cutoff == pytest.approx(np.log(1e10) + 8.0)
    with pytest.raises(ValueError):
        TruncationPolicy(tol=0.0)
    with pytest.raises(ValueError):
        TruncationPolicy(max_terms=0)


def test_oracle_report_ok():
    assert OracleReport(np.zeros(2), 5, ()).ok()
    assert not OracleReport(np.zeros(2), 5, ((0, 1, "separation"),)).ok()
