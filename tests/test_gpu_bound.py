"""On-GPU a-posteriori truncation-bound audit (SURVEY.md §8(f) "next" #4).

The reference checks the paper's bound node by node on a 2000-charge case
(test_tree.py:216-250).  Here the traversal accumulates, per target, the
bound of every accepted far node at the order it used (exact contour
supremum, kernel.py:147-150) and the field error against the fp64 direct sum
is checked to stay below it at full size."""

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


def _audit(dt, xs, qs, targets, r_d, p, adaptive, tol, leaf=64, n_check=2048):
    from paper_1710_05781_b200.tree import evaluate_with_bound

    system = dt.from_sorted(xs, qs)
    kernel = dt.DiscKernel(r_d)
    cfg = dt.EvalConfig(p=p, leaf_capacity=leaf, adaptive=adaptive, tolerance=tol)
    tree = dt.build(system, kernel, cfg)
    ys = torch.from_numpy(np.ascontiguousarray(targets)).cuda()
    vals, bounds = evaluate_with_bound(tree, kernel, cfg, system, ys)
    plain = dt.evaluate_all(tree, kernel, cfg, system, ys).values
    assert torch.equal(vals, plain), "the audit must not change the field"
    idx = np.unique(np.linspace(0, len(targets) - 1, n_check).astype(np.int64))
    direct = dt.evaluate_direct(system, kernel, targets[idx]).values
    err = np.abs(vals.cpu().numpy()[idx] - direct)
    b = bounds.cpu().numpy()[idx]
    scale = float(np.abs(qs).sum())
    assert np.all(err <= b + 1e-13 * scale), float(np.max(err - b) / scale)
    assert np.all(b >= 0) and np.isfinite(b).all()
    return err, b, scale


def test_bound_reference_case(dt):
    """test_tree.py:216-250's instance shape: r_d 0.1, p = 10, leaf 25."""
    from paper_1710_05781_b200 import metrics

    system = metrics.random_instance(2000, seed=12)
    xs, qs = system.numpy()
    t = np.sort(np.random.default_rng(13).uniform(-0.1, 1.1, 512))
    err, b, scale = _audit(dt, xs, qs, t, 0.1, 10, False, 1e-10, leaf=25, n_check=512)
    assert b.max() > 0


@pytest.mark.parametrize("r_d,tol", [(0.01, 1e-10), (1e-3, 1e-8)])
def test_bound_cfg1(dt, r_d, tol):
    from paper_1710_05781_b200 import workloads as W

    w = W.cfg1(cells=1 << 18)
    _audit(dt, w.xs, w.qs, w.targets, r_d, 8, True, tol)


@pytest.mark.slow
def test_bound_cfg2_full(dt):
    from paper_1710_05781_b200 import workloads as W

    w = W.cfg2()
    err, b, scale = _audit(dt, w.xs, w.qs, w.targets, w.r_d, w.p, True, w.tolerance,
                           n_check=1024)
    # the adaptive orders keep the whole bound near the requested tolerance
    assert b.max() <= 1e-8 * scale
