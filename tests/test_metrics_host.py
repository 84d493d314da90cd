"""Host-side metrics of the paper harness: error_report and TimingStats
(restating the checks of the reference's pkg/tests/test_metrics.py:17-70
on this package's metrics.py / harness.py; no GPU needed)."""

import dataclasses

import numpy as np
import pytest

from paper_1710_05781_b200.harness import TimingStats
from paper_1710_05781_b200.metrics import ErrorReport, error_report


def test_error_report_hand_values():
    r = error_report([1.1, 2.0, 3.0], [1.0, 2.0, 3.0])
    assert r.max_relative == pytest.approx(0.1)
    assert r.avg_relative == pytest.approx(0.1 / 6.0)
    assert r.excluded_targets == 0


def test_error_report_near_zero_reference_excluded_from_max():
    # below 1e-12 max|E_direct| a reference value is left out of the max
    # ratio (and counted) but still feeds the sums of the average
    r = error_report([1.0, 1e-8], [1.0, 1e-20])
    assert r.excluded_targets == 1
    assert r.max_relative == 0.0
    assert r.avg_relative == pytest.approx(1e-8)


def test_error_report_scale_invariance_and_zero_error():
    rng = np.random.default_rng(0)
    ref = rng.normal(size=50)
    approx = ref + rng.normal(scale=1e-9, size=50)
    a, b = error_report(approx, ref), error_report(approx * 1e9, ref * 1e9)
    assert a.max_relative == pytest.approx(b.max_relative, rel=1e-12)
    assert a.avg_relative == pytest.approx(b.avg_relative, rel=1e-12)
    assert a.excluded_targets == b.excluded_targets
    v = np.linspace(-2, 2, 9)
    z = error_report(v, v)
    assert z.max_relative == 0.0 and z.avg_relative == 0.0


@pytest.mark.parametrize("tree_vals,direct_vals",
                         [([1.0], [1.0, 2.0]), ([], []), ([1.0, 2.0], [0.0, 0.0])])
def test_error_report_rejects(tree_vals, direct_vals):
    with pytest.raises(ValueError):
        error_report(tree_vals, direct_vals)


def test_error_report_is_frozen():
    r = ErrorReport(0.0, 0.0, 0)
    with pytest.raises(dataclasses.FrozenInstanceError):
        r.max_relative = 1.0


def test_timing_stats_of_and_ordering():
    s = TimingStats.of([0.001, 0.002, 0.003])
    assert (s.min_ms, s.max_ms, s.avg_ms) == (pytest.approx(1.0), pytest.approx(3.0),
                                              pytest.approx(2.0))
    with pytest.raises(ValueError):
        TimingStats(max_ms=1.0, min_ms=2.0, avg_ms=1.5)
