"""The drop-in surface (no GPU needed): every public name of the reference
package exists here, and the host-side records validate like the
reference's."""

import pytest

# disctree/__init__.py:45-80 (the reference's __all__), copied as data so the
# check runs where the reference is absent
REFERENCE_ALL = (
    "BenchRecord", "Charge", "ChargeSystem", "DensitySpec", "DepthScanRecord", "DiscKernel",
    "ErrorReport", "EvalConfig", "FieldResult", "ImageSpec", "PChoice", "TimingStats", "Tree",
    "TreeNode", "TruncationBound", "bench", "bound_value", "build", "choose_p", "contour_max",
    "depth_scan", "error_report", "evaluate_all", "evaluate_direct", "evaluate_point",
    "from_density", "from_particles", "phi", "phi_derivatives", "random_instance",
    "sign_term_all", "single_cell_errors", "truncation_bound", "well_separated", "with_images",
)


def test_reference_names_exported():
    import paper_1710_05781_b200 as dt

    missing = [n for n in REFERENCE_ALL if not hasattr(dt, n) or n not in dt.__all__]
    assert not missing, missing


def test_timing_stats_validation():
    """metrics.py:41-58: min <= avg <= max is enforced."""
    from paper_1710_05781_b200 import TimingStats

    s = TimingStats.of([0.002, 0.001, 0.003])
    assert (s.min_ms, s.max_ms) == (1.0, 3.0) and abs(s.avg_ms - 2.0) < 1e-12
    with pytest.raises(ValueError, match="min <= avg <= max"):
        TimingStats(max_ms=1.0, min_ms=2.0, avg_ms=1.5)
    with pytest.raises(ValueError):
        TimingStats(max_ms=3.0, min_ms=1.0, avg_ms=4.0)


def test_records_match_reference_fields():
    """BenchRecord / DepthScanRecord carry the reference's fields and derived
    properties (metrics.py:61-88)."""
    import dataclasses

    from paper_1710_05781_b200 import BenchRecord, DepthScanRecord, TimingStats

    assert [f.name for f in dataclasses.fields(BenchRecord)] == [
        "n", "repeats", "tree_build", "tree_eval", "direct_eval"]
    assert [f.name for f in dataclasses.fields(DepthScanRecord)] == [
        "leaf_capacity", "depth", "mean_leaf_occupancy", "build_ms", "eval_ms"]
    t = TimingStats(2.0, 1.0, 1.5)
    r = BenchRecord(10, 3, t, t, t)
    assert r.tree_total_avg_ms == 3.0
    assert DepthScanRecord(8, 5, 7.5, 1.25, 2.5).total_ms == 3.75
