"""bench.py --report: the per-(k, l) accounting rows (host logic, no GPU)."""
import numpy as np

from paper_2306_15049_b200.pipeline import StepOut, report_rows


def test_report_rows_per_shift_and_overhead():
    M = 4
    o = StepOut(1, np.array([5, 0, 7, 2]), np.array([7, 1, 9, 4]), np.zeros(M, int), np.full(M, 1e-9),
                np.array([9, 9, 8, 9]), 40, 2, np.ones(M), np.ones(M), 123, np.array([1, 1, 0, 1]), None)
    rows = report_rows([o], np.logspace(-3, 0, M))
    assert len(rows) == M + 1
    assert [r["l"] for r in rows] == [1, 2, 3, 4, -1]
    assert rows[2]["iters"] == 7 and rows[2]["applies_A"] == 9 == rows[2]["applies_E"]
    assert rows[-1]["applies_A"] == 123 and rows[0]["lstar"] == 3 and rows[0]["nc"] == 40
    assert sum(r["applies_A"] for r in rows) == int(o.applies.sum()) + o.overhead_applies
