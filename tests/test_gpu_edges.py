"""Edge cases of the public API on the GPU paths added for speed: unaligned
pair views, host/device target kinds at the pipeline threshold, far-away and
non-finite targets, empty systems for the assembly helpers."""

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


def test_unaligned_pair_view(dt):
    rng = np.random.default_rng(1)
    pairs = torch.from_numpy(np.column_stack([rng.uniform(0, 1, 1001), rng.normal(size=1001)]))
    dev = pairs.cuda()
    view = dev.view(-1)[1:-1].view(-1, 2)  # 8-byte offset: (q0, x1), (q1, x2), ...
    assert view.data_ptr() % 16 == 8
    s = dt.from_particles(view)
    want = dt.from_particles(view.cpu().numpy())
    assert torch.equal(s.xs, want.xs) and torch.equal(s.qs, want.qs)


def test_targets_far_outside_and_at_sources(dt):
    rng = np.random.default_rng(2)
    x = np.sort(rng.uniform(-1, 1, 3000))
    q = rng.normal(size=3000)
    s = dt.from_sorted(x, q)
    k = dt.DiscKernel(0.01)
    cfg = dt.EvalConfig(p=12, leaf_capacity=16, adaptive=True, tolerance=1e-10)
    tree = dt.build(s, k, cfg)
    t = np.concatenate([[-1e6, -50.0, -1.0 - 1e-12], x[::7], [x[-1], 1.0 + 1e-9, 3.5, 1e5]])
    got = dt.evaluate_all(tree, k, cfg, s, t).values
    ref = dt.evaluate_direct(s, k, t).values
    assert np.max(np.abs(got - ref)) <= 1e-10 * np.abs(q).sum()


@pytest.mark.parametrize("n", [(1 << 20) - 1, 1 << 20])
def test_pipeline_threshold_paths_agree(dt, n):
    """Just below / at the host-pipeline threshold: pinned, pageable and
    device targets give identical values."""
    from paper_1710_05781_b200 import workloads as W

    w = W.cfg1(cells=1 << 18)
    s = dt.from_sorted(w.xs, w.qs)
    k = dt.DiscKernel(w.r_d)
    cfg = dt.EvalConfig(p=8, leaf_capacity=64, adaptive=True, tolerance=1e-10)
    tree = dt.build(s, k, cfg)
    t = np.sort(np.random.default_rng(3).uniform(-1.1, 1.1, n))
    dev = dt.evaluate_all(tree, k, cfg, s, torch.from_numpy(t).cuda()).values.cpu().numpy()
    host = dt.evaluate_all(tree, k, cfg, s, t).values
    pinned = dt.evaluate_all(tree, k, cfg, s, torch.from_numpy(t).pin_memory()).values.numpy()
    np.testing.assert_array_equal(host, dev)
    np.testing.assert_array_equal(pinned, dev)


def test_non_finite_targets_rejected_everywhere(dt):
    s = dt.from_particles([(0.1, 1.0), (0.4, -2.0), (0.9, 0.5)])
    k = dt.DiscKernel(0.05)
    cfg = dt.EvalConfig(p=6, leaf_capacity=1)
    tree = dt.build(s, k, cfg)
    for bad in (np.nan, np.inf, -np.inf):
        t = np.array([0.2, bad, 0.7])
        with pytest.raises(ValueError):
            dt.evaluate_all(tree, k, cfg, s, t)
        with pytest.raises(ValueError):
            dt.evaluate_all(tree, k, cfg, s, torch.from_numpy(t).cuda())
        with pytest.raises(ValueError):
            dt.evaluate_direct(s, k, t)


def test_assembly_edges(dt):
    empty = dt.from_particles([])
    im = dt.with_images(empty, dt.ImageSpec(gap_length=1.0))
    assert len(im) == 0
    one = dt.from_density(dt.DensitySpec(domain=(0.0, 2.0), cells=1, values=[3.0],
                                         quadrature_order=1, eps0=1.0))
    # one node at the cell middle with q = (w/2) sigma dx / (2 eps0) = 1 * 3 * 2 / 2
    assert one.xs.tolist() == [1.0] and one.qs.tolist() == [3.0]


@pytest.mark.parametrize("kind", ["cluster", "geometric", "duplicates"])
def test_deep_trees_bit_exact(dt, kind):
    """Trees far deeper than the precomputed dyadic levels, whose deep levels
    run in one block with the shared-memory split samples: node arrays
    bit-identical to the oracle's build."""
    from oracle import oracle as O

    rng = np.random.default_rng(11)
    if kind == "cluster":  # a dense clump 1e-9 wide inside a uniform background
        x = np.concatenate([rng.uniform(-1, 1, 60000), 0.3 + 1e-9 * rng.uniform(0, 1, 60000)])
    elif kind == "geometric":  # spacing shrinking geometrically toward 0.3
        x = 0.3 + np.concatenate([-(1.0 - 0.9998 ** np.arange(40000)),
                                  1.0 - 0.9997 ** np.arange(40000)]) * 0.5
    else:  # long runs of identical positions (depth hits the cap)
        x = np.repeat(rng.uniform(-1, 1, 300), 400)
    x = np.sort(x)
    q = rng.normal(size=len(x))
    system = dt.from_sorted(x, q)
    cfg = dt.EvalConfig(p=8, leaf_capacity=16)
    tree = dt.build(system, dt.DiscKernel(0.01), cfg)
    assert tree.depth > 16
    host = tree.numpy()
    ot = O.build_structure(x, 16)
    for f in ("lo", "hi", "center", "half", "level", "start", "end", "left", "right"):
        np.testing.assert_array_equal(host[f], getattr(ot, f), err_msg=f)


def test_sign_terms_tile_aligned_sorted_runs(dt):
    """Targets made of sorted runs whose length is a multiple of the sign
    kernel's 2048-target tile: each tile is sorted on its own but the next
    tile starts lower, so its bracket must not bound this tile's search
    (dt_sign_terms, charges.py:183-187 semantics for any target order)."""
    from oracle import oracle as O

    rng = np.random.default_rng(21)
    x = np.sort(rng.uniform(-1, 1, 5000))
    q = rng.normal(size=5000)
    s = dt.from_sorted(x, q)
    g = np.sort(rng.uniform(-1.2, 1.2, 4096))
    t = np.concatenate([g, g, g[::-1][:2048], g])
    from paper_1710_05781_b200.charges import _sign_terms

    got = _sign_terms(s, torch.from_numpy(t).cuda()).cpu().numpy()
    pre = O.prefix(q)
    want = O.sign_terms(x, pre, float(pre[-1]), t)
    assert np.max(np.abs(got - want)) <= 1e-13 * np.abs(q).sum()
    # and through the field paths, against the oracle's tree and direct sums
    k = dt.DiscKernel(0.01)
    cfg = dt.EvalConfig(p=8, leaf_capacity=32)
    tree = dt.build(s, k, cfg)
    f = dt.evaluate_all(tree, k, cfg, s, t).values
    fw, _ = O.evaluate_tree(x, q, 0.01, 8, cfg.theta, 32, False, 1e-9, t)
    assert np.max(np.abs(f - fw)) <= 1e-12 * np.abs(q).sum()
    d = dt.evaluate_direct(s, k, t).values
    assert np.max(np.abs(d - O.evaluate_direct(x, q, 0.01, t))) <= 1e-13 * np.abs(q).sum()


def test_capacity_overflow_rebuild(dt):
    """Clusters of leaf_capacity + 1 coincident sources split down to the
    depth limit, so the tree needs far more nodes than the initial capacity
    estimate: build() detects the overflow after the moments were already
    enqueued (they return at once on an overflowed tree), rebuilds with a
    larger capacity, and the result matches the oracle's structure and the
    direct sum."""
    from oracle import oracle as O
    from paper_1710_05781_b200.tree import initial_node_capacity

    rng = np.random.default_rng(11)
    m, lc = 100, 64
    centers = np.sort(rng.uniform(-1, 1, m))
    x = np.repeat(centers, lc + 1)
    q = rng.normal(size=x.size)
    s = dt.from_sorted(x, q)
    k = dt.DiscKernel(0.01)
    cfg = dt.EvalConfig(p=10, leaf_capacity=lc)
    tree = dt.build(s, k, cfg)
    assert len(tree) > initial_node_capacity(x.size, lc)  # the first build overflowed
    ref = O.build_structure(x, lc)
    for f in O.NODE_FIELDS:
        np.testing.assert_array_equal(getattr(tree, f).cpu().numpy(), getattr(ref, f), err_msg=f)
    assert np.isfinite(tree.meval.cpu().numpy()).all()
    t = np.sort(rng.uniform(-1.1, 1.1, 2000))
    got = dt.evaluate_all(tree, k, cfg, s, t).values
    want = dt.evaluate_direct(s, k, t).values
    assert np.max(np.abs(got - want)) <= 1e-8 * np.abs(q).sum()
