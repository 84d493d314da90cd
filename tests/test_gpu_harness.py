"""Paper-table harness on the GPU (SURVEY.md §8(f) "next" #3): the sweeps run
and agree with the reference's semantics (single-cell errors match the CPU
oracle's moments; records carry the reference's fields)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1710_05781_b200 as pkg

    return pkg


def test_bench_and_depth_scan(dt):
    from paper_1710_05781_b200 import harness as H

    k = dt.DiscKernel(0.1)
    cfg = dt.EvalConfig(p=10, leaf_capacity=40)
    recs = H.bench([10_000, 50_000], 2, k, cfg)
    assert [r.n for r in recs] == [10_000, 50_000]
    for r in recs:
        assert 0 < r.tree_build.min_ms <= r.tree_build.avg_ms <= r.tree_build.max_ms
        assert r.tree_total_avg_ms > 0 and r.direct_eval.avg_ms > 0
    scan = H.depth_scan(50_000, k, cfg, [781, 98, 13])
    assert [s.leaf_capacity for s in scan] == [781, 98, 13]
    assert scan[0].depth < scan[1].depth < scan[2].depth
    assert all(s.mean_leaf_occupancy <= s.leaf_capacity for s in scan)


def test_single_cell_errors_decrease_and_match_oracle(dt):
    from oracle import oracle as O
    from paper_1710_05781_b200 import harness as H
    from paper_1710_05781_b200.kernel import phi_derivatives
    from paper_1710_05781_b200.metrics import random_instance

    k = dt.DiscKernel(0.1)
    ps = [5, 10, 15, 20]
    errs = H.single_cell_errors(2000, k, 2.0, ps)
    vals = [e for _, e in errs]
    assert vals[0] > vals[-1] and all(v < 1e-2 for v in vals)
    # the same numbers from the oracle's direct moments of the one-leaf root
    xs, qs = random_instance(2000, (0, 2000), interval=(-0.5, 0.5)).numpy()
    t = O.build(xs, qs, 20, 2000, False)
    d = phi_derivatives(k, float(t.center[0]), 2.0, 20)
    exact = float(np.sum(qs * (xs - 2.0) / np.sqrt((xs - 2.0) ** 2 + 0.01)))
    for (p, e), p2 in zip(errs, ps):
        want = abs(float(d[: p2 + 1] @ t.moments[0, : p2 + 1]) - exact) / abs(exact)
        assert e == pytest.approx(want, rel=1e-6, abs=1e-15)
