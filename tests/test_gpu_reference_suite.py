"""The behaviours the reference's own unit tests pin for the evaluation path
(pkg/tests/test_charges.py, test_tree.py, test_direct.py), checked on the
GPU path through the public API.  Each test names the reference test it
restates; the checks are the same properties at the same tolerances, with
brute-force numpy sums as the checker (exact-count semantics of the sign
term, tree invariants, moment definitions, traversal accuracy, determinism).

Property tests draw inputs with hypothesis like the reference does
(test_charges.py:76-85, 223-236).
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
hypothesis = pytest.importorskip("hypothesis")
from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

finite = st.floats(min_value=-1e3, max_value=1e3, allow_nan=False, allow_infinity=False)


@pytest.fixture(scope="module")
def dt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1710_05781_b200 as pkg

    return pkg


def _pkg():
    # the hypothesis tests take no fixtures (function-scoped fixtures are not
    # reset between examples)
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1710_05781_b200 as pkg

    return pkg


def _np(v):
    return v.cpu().numpy() if isinstance(v, torch.Tensor) else np.asarray(v)


def _sign_brute(xs, qs, ys):
    """e(y) = sum_{x < y} q - sum_{x >= y} q, one target at a time."""
    return np.array([qs[xs < y].sum() - qs[xs >= y].sum() for y in ys])


def _phi_brute(xs, qs, r_d, y):
    d = xs - y
    return float(np.sum(qs * d / np.sqrt(d * d + r_d * r_d)))


# -- charges: from_particles and the sign term (test_charges.py:34-236) --------


def test_from_particles_order_prefix_total(dt):
    """test_sorts_by_position, test_prefix_and_total, test_len_getitem_iter,
    test_empty_input (test_charges.py:35-65)."""
    s = dt.from_particles([(0.5, 1.0), (-1.0, 2.0), (0.0, 3.0)])
    np.testing.assert_array_equal(_np(s.xs), [-1.0, 0.0, 0.5])
    np.testing.assert_array_equal(_np(s.qs), [2.0, 3.0, 1.0])
    s = dt.from_particles([(0.0, 1.0), (1.0, 2.0), (2.0, -0.5)])
    np.testing.assert_array_equal(_np(s.prefix), [1.0, 3.0, 2.5])
    assert s.total == 2.5
    s = dt.from_particles([(0.0, 1.0), (2.0, -1.0)])
    assert len(s) == 2
    assert s[1] == dt.Charge(2.0, -1.0)
    assert list(s) == [dt.Charge(0.0, 1.0), dt.Charge(2.0, -1.0)]
    e = dt.from_particles([])
    assert len(e) == 0 and e.total == 0.0


@pytest.mark.parametrize("bad", [[(0.0, math.nan)], [(math.inf, 1.0)], [(0.0, 1.0, 2.0)]])
def test_from_particles_rejects(dt, bad):
    """test_rejects_nonfinite, test_rejects_wrong_shape (test_charges.py:66-74)."""
    with pytest.raises(ValueError):
        dt.from_particles(bad)


@given(st.lists(st.tuples(finite, finite), min_size=1, max_size=60))
@settings(max_examples=60, deadline=None)
def test_from_particles_invariants_any_input(pairs):
    """test_invariants_hold_for_any_input (test_charges.py:76-85): sorted,
    a stable permutation of the input, prefix = running sum, total = last
    prefix.  The prefix is a parallel scan here (dt_prefix_scan), so it is
    checked to round-off of the running sum of |q| rather than bitwise."""
    dt = _pkg()
    s = dt.from_particles(pairs)
    xs, qs, pre = _np(s.xs), _np(s.qs), _np(s.prefix)
    assert np.all(np.diff(xs) >= 0)
    order = np.argsort(np.array([x for x, _ in pairs]), kind="stable")
    np.testing.assert_array_equal(xs, np.array([pairs[i][0] for i in order]))
    np.testing.assert_array_equal(qs, np.array([pairs[i][1] for i in order]))
    bound = 1e-15 * len(qs) * np.cumsum(np.abs(qs)) + 1e-300
    assert np.all(np.abs(pre - np.cumsum(qs)) <= bound)
    assert s.total == pre[-1]


def test_sign_term_hand_and_boundary(dt):
    """test_hand_case, test_charge_exactly_at_target_counts_minus,
    test_outside_support (test_charges.py:190-227)."""
    s = dt.from_particles([(0.0, 1.0), (1.0, 2.0), (2.0, 4.0)])
    np.testing.assert_array_equal(_np(dt.sign_term_all(s, [0.5, 1.5])), [-5.0, -1.0])
    # a charge at the target counts on the minus side; one ulp above it plus
    s1 = dt.from_particles([(1.0, 3.0)])
    np.testing.assert_array_equal(_np(dt.sign_term_all(s1, [1.0])), [-3.0])
    np.testing.assert_array_equal(_np(dt.sign_term_all(s1, [np.nextafter(1.0, 2.0)])), [3.0])
    np.testing.assert_array_equal(_np(dt.sign_term_all(s1, [1.0 + 1e-12])), [3.0])
    s2 = dt.from_particles([(0.0, 1.0), (1.0, 2.0)])
    np.testing.assert_array_equal(_np(dt.sign_term_all(s2, [-5.0, 5.0])), [-3.0, 3.0])


def test_sign_term_rejects(dt):
    """test_rejects_unsorted_targets, test_rejects_bad_shape
    (test_charges.py:210-218)."""
    s = dt.from_particles([(0.0, 1.0)])
    with pytest.raises(ValueError):
        dt.sign_term_all(s, [1.0, 0.5])
    with pytest.raises(ValueError):
        dt.sign_term_all(s, [[0.5]])


def test_sign_term_duplicates_brute(dt):
    """test_matches_brute_force_with_duplicates (test_charges.py:200-208):
    positions rounded to 0.01 so runs of equal x straddle targets that sit
    exactly on sources."""
    rng = np.random.default_rng(5)
    xs = np.round(rng.uniform(0, 1, 200), 2)
    qs = rng.uniform(-1, 1, 200)
    s = dt.from_particles(np.column_stack([xs, qs]))
    ys = np.sort(np.concatenate([rng.uniform(0, 1, 50), xs[:10]]))
    got = _np(dt.sign_term_all(s, ys))
    np.testing.assert_allclose(got, _sign_brute(xs, qs, ys), rtol=1e-12, atol=1e-12)


@given(st.lists(st.tuples(finite, finite), min_size=1, max_size=40),
       st.lists(finite, min_size=1, max_size=20))
@settings(max_examples=60, deadline=None)
def test_sign_term_any_input(pairs, raw):
    """test_matches_brute_force_for_any_input (test_charges.py:223-236)."""
    dt = _pkg()
    s = dt.from_particles(pairs)
    ys = np.sort(np.asarray(raw, dtype=np.float64))
    got = _np(dt.sign_term_all(s, ys))
    xs, qs = _np(s.xs), _np(s.qs)
    scale = float(np.abs(qs).sum()) or 1.0
    np.testing.assert_allclose(got, _sign_brute(xs, qs, ys), rtol=0, atol=1e-9 * scale)


# -- tree build (test_tree.py:50-136) ----------------------------------------


def _leaves(tree):
    h = tree.numpy()
    leaf = (h["left"] < 0) & (h["right"] < 0)  # a node may have one child
    return h, leaf


def test_leaves_partition_sources(dt):
    """test_leaves_partition_sources (test_tree.py:51-61)."""
    s = dt.random_instance(777, seed=1)
    tree = dt.build(s, dt.DiscKernel(0.1), dt.EvalConfig(leaf_capacity=16))
    h, leaf = _leaves(tree)
    rng_ = sorted(zip(h["start"][leaf], h["end"][leaf]))
    assert rng_[0][0] == 0 and rng_[-1][1] == 777
    assert all(a[1] == b[0] for a, b in zip(rng_, rng_[1:]))
    assert np.all(h["end"][leaf] - h["start"][leaf] <= 16)
    assert tree.leaf_count == int(leaf.sum())
    # the TreeNode view agrees with the arrays
    view = [tree.node(i) for i in range(len(tree)) if tree.node(i).is_leaf]
    assert sorted(v.source_range for v in view) == [tuple(map(int, r)) for r in rng_]


@pytest.mark.parametrize("n,cap,seed", [(300, 10, 2), (5000, 7, 12)])
def test_children_bisect_parent(dt, n, cap, seed):
    """test_children_split_parent_interval_and_range (test_tree.py:63-78):
    children halve the parent's interval at its exact midpoint, split its
    source range, sit one level down."""
    s = dt.random_instance(n, seed=seed)
    tree = dt.build(s, dt.DiscKernel(0.1), dt.EvalConfig(leaf_capacity=cap))
    for i in range(len(tree)):
        node = tree.node(i)
        kids = node.children
        if not kids:
            continue
        assert sum(k.source_count for k in kids) == node.source_count
        lo, hi = node.interval
        mid = 0.5 * (lo + hi)
        for k in kids:
            assert k.interval in ((lo, mid), (mid, hi))
            assert k.level == node.level + 1


def test_sources_strictly_inside_root(dt):
    """test_all_sources_inside_root_interval (test_tree.py:80-85)."""
    s = dt.random_instance(100, seed=3)
    tree = dt.build(s, dt.DiscKernel(0.1), dt.EvalConfig())
    lo, hi = tree.root.interval
    xs = _np(s.xs)
    assert np.all(xs > lo) and np.all(xs < hi)


def test_depth_matches_capacity(dt):
    """test_depth_matches_capacity (test_tree.py:87-91): 1e5 uniform sources,
    40 per leaf, depth 12 or 13."""
    s = dt.random_instance(100_000, seed=0)
    tree = dt.build(s, dt.DiscKernel(0.1), dt.EvalConfig(leaf_capacity=40))
    assert tree.depth in (12, 13)


def test_coincident_positions_terminate(dt):
    """test_single_charge_tree, test_coincident_positions_terminate
    (test_tree.py:93-104)."""
    tree = dt.build(dt.from_particles([(0.5, 1.0)] * 10), dt.DiscKernel(0.1),
                    dt.EvalConfig(leaf_capacity=2))
    assert tree.depth <= 60 and tree.leaf_count >= 1
    # the bisection keeps only non-empty children: a chain down to the
    # depth cap ending in one leaf that holds all ten sources
    h, leaf = _leaves(tree)
    assert tree.leaf_count == int(leaf.sum()) == 1
    assert int((h["end"][leaf] - h["start"][leaf]).sum()) == 10


def test_moments_hand_case_and_definition(dt):
    """test_moments_hand_case, test_moments_match_definition,
    test_adaptive_raises_moment_order (test_tree.py:110-136)."""
    tree = dt.build(dt.from_particles([(-1.0, 1.0), (1.0, 1.0)]), dt.DiscKernel(0.1),
                    dt.EvalConfig(p=4, leaf_capacity=10))
    np.testing.assert_allclose(tree.root.moments, [2.0, 0.0, 1.0, 0.0, 1.0 / 12.0],
                               rtol=1e-9, atol=1e-9)
    s = dt.random_instance(500, seed=4)
    tree = dt.build(s, dt.DiscKernel(0.1), dt.EvalConfig(p=6, leaf_capacity=20))
    xs, qs = _np(s.xs), _np(s.qs)
    m = _np(tree.moments)
    h = tree.numpy()
    for i in range(len(tree)):
        t = xs[h["start"][i]:h["end"][i]] - h["center"][i]
        q = qs[h["start"][i]:h["end"][i]]
        for k in range(7):
            want = np.sum(q * t**k) / math.factorial(k)
            assert m[i, k] == pytest.approx(want, rel=1e-12, abs=1e-14), (i, k)
    tree = dt.build(dt.random_instance(50, seed=5), dt.DiscKernel(0.1),
                    dt.EvalConfig(p=4, adaptive=True))
    assert tree.moment_order == 30 and tuple(tree.moments.shape[1:]) == (31,)


def test_well_separated_boundary(dt):
    """test_boundary_inclusive, test_target_at_center_never_separated
    (test_tree.py:139-152)."""
    s = dt.from_particles([(0.0, 1.0), (1.0, 1.0)])
    root = dt.build(s, dt.DiscKernel(0.1), dt.EvalConfig(leaf_capacity=10)).root
    r, c = root.half_width, root.center
    assert dt.well_separated(root, c + 3.0 * r, 1.0 / 3.0)
    assert not dt.well_separated(root, c + 2.9 * r, 1.0 / 3.0)
    root = dt.build(s, dt.DiscKernel(0.1), dt.EvalConfig()).root
    assert not dt.well_separated(root, root.center, 0.999)


# -- single-target traversal (test_tree.py:154-214) ---------------------------


def test_point_high_order_brute(dt):
    """test_matches_brute_force_high_order (test_tree.py:162-172)."""
    k = dt.DiscKernel(0.1)
    cfg = dt.EvalConfig(p=20, leaf_capacity=8)
    s = dt.random_instance(400, seed=6)
    tree = dt.build(s, k, cfg)
    xs, qs = _np(s.xs), _np(s.qs)
    scale = float(np.abs(qs).sum())
    for y in np.random.default_rng(7).uniform(-0.2, 1.2, 40):
        got = dt.evaluate_point(tree, k, cfg, float(y))
        assert got == pytest.approx(_phi_brute(xs, qs, 0.1, float(y)), abs=1e-11 * scale)


def test_point_exterior_and_translation(dt):
    """test_exterior_target, test_translation_invariance (test_tree.py:174-195)."""
    k = dt.DiscKernel(0.1)
    cfg = dt.EvalConfig(p=16)
    s = dt.random_instance(1000, seed=8, interval=(-0.5, 0.5))
    tree = dt.build(s, k, cfg)
    want = _phi_brute(_np(s.xs), _np(s.qs), 0.1, 1.0)
    assert dt.evaluate_point(tree, k, cfg, 1.0) == pytest.approx(want, rel=1e-10)

    cfg = dt.EvalConfig(p=12, leaf_capacity=10)
    rng = np.random.default_rng(9)
    xs, qs = rng.uniform(0, 1, 250), rng.uniform(-1, 1, 250)
    t1 = dt.build(dt.from_particles(np.column_stack([xs, qs])), k, cfg)
    t2 = dt.build(dt.from_particles(np.column_stack([xs + 10.0, qs])), k, cfg)
    for y in (1.7, 0.31):
        a = dt.evaluate_point(t1, k, cfg, y)
        b = dt.evaluate_point(t2, k, cfg, y + 10.0)
        assert a == pytest.approx(b, rel=1e-12, abs=1e-12)


def test_point_order_and_adaptive_tolerance(dt):
    """test_requires_sufficient_moment_order, test_adaptive_meets_tolerance
    (test_tree.py:197-214)."""
    k = dt.DiscKernel(0.1)
    tree = dt.build(dt.random_instance(100, seed=10), k, dt.EvalConfig(p=5))
    with pytest.raises(ValueError):
        dt.evaluate_point(tree, k, dt.EvalConfig(p=10), 0.5)
    cfg = dt.EvalConfig(adaptive=True, tolerance=1e-10, leaf_capacity=10)
    s = dt.random_instance(800, seed=11)
    tree = dt.build(s, k, cfg)
    xs, qs = _np(s.xs), _np(s.qs)
    scale = float(np.abs(qs).sum())
    for y in (0.123, 0.77, 1.5):
        got = dt.evaluate_point(tree, k, cfg, y)
        assert abs(got - _phi_brute(xs, qs, 0.1, y)) <= 1e-10 * scale


# -- all targets (test_tree.py:253-330) --------------------------------------


def test_all_equals_sign_plus_point(dt):
    """test_matches_point_twin (test_tree.py:254-267): evaluate_all is the
    sign term plus the single-target traversal.  Both run the same GPU
    traversal here, so the sum agrees to one rounding of the addition."""
    k = dt.DiscKernel(0.1)
    cfg = dt.EvalConfig(p=8, leaf_capacity=12)
    s = dt.random_instance(300, seed=14)
    tree = dt.build(s, k, cfg)
    ys = np.sort(np.random.default_rng(15).uniform(0, 1, 64))
    res = dt.evaluate_all(tree, k, cfg, s, ys)
    e = _np(dt.sign_term_all(s, ys))
    twin = np.array([dt.evaluate_point(tree, k, cfg, float(y)) for y in ys])
    np.testing.assert_allclose(res.values, e + twin, rtol=1e-10, atol=1e-12)


def test_all_thread_count_invariance(dt):
    """test_thread_count_invariance (test_tree.py:269-278): the threads
    argument is accepted and never changes a bit."""
    k = dt.DiscKernel(0.1)
    cfg = dt.EvalConfig()
    s = dt.random_instance(2000, seed=16)
    tree = dt.build(s, k, cfg)
    ys = _np(s.xs).copy()
    base = dt.evaluate_all(tree, k, cfg, s, ys, threads=1).values
    for threads in (2, 5, None):
        np.testing.assert_array_equal(base, dt.evaluate_all(tree, k, cfg, s, ys,
                                                            threads=threads).values)


def test_all_close_to_direct(dt):
    """test_close_to_direct (test_tree.py:280-290): p = 20 on 3000 self
    targets, relative L1 error below 1e-11."""
    k = dt.DiscKernel(0.1)
    cfg = dt.EvalConfig(p=20)
    s = dt.random_instance(3000, seed=17)
    tree = dt.build(s, k, cfg)
    ys = _np(s.xs).copy()
    res = dt.evaluate_all(tree, k, cfg, s, ys).values
    ref = dt.evaluate_direct(s, k, ys).values
    assert np.sum(np.abs(res - ref)) / np.sum(np.abs(ref)) < 1e-11


def test_all_empty_targets_and_build_time(dt):
    """test_empty_targets, test_records_build_time (test_tree.py:292-309)."""
    k = dt.DiscKernel(0.1)
    cfg = dt.EvalConfig()
    tree = dt.build(dt.random_instance(10, seed=18), k, cfg)
    assert dt.evaluate_all(tree, k, cfg, tree.system, []).values.shape == (0,)
    tree = dt.build(dt.random_instance(100, seed=19), k, cfg)
    res = dt.evaluate_all(tree, k, cfg, tree.system, [0.5])
    assert res.method == "tree"
    assert res.build_time == tree.build_seconds > 0.0


# -- direct sums (test_direct.py:100-150) -------------------------------------


def test_direct_determinism(dt):
    """test_thread_invariance_distinct_targets, ..._self_targets,
    test_repeat_call_bitwise_identical (test_direct.py:101-123)."""
    k = dt.DiscKernel(0.1)
    s = dt.random_instance(3000, seed=25)
    ys = np.random.default_rng(26).uniform(0, 1, 500)
    base = dt.evaluate_direct(s, k, ys, threads=1).values
    for threads in (2, 7, None):
        np.testing.assert_array_equal(base, dt.evaluate_direct(s, k, ys, threads=threads).values)
    xs = _np(s.xs).copy()
    base = dt.evaluate_direct(s, k, xs, threads=1).values
    for threads in (2, 7, None):
        np.testing.assert_array_equal(base, dt.evaluate_direct(s, k, xs, threads=threads).values)
    np.testing.assert_array_equal(base, dt.evaluate_direct(s, k, xs).values)


def test_direct_compensated(dt):
    """test_close_to_plain, test_close_to_symmetric_path,
    test_compensated_thread_invariance (test_direct.py:127-150)."""
    k = dt.DiscKernel(0.1)
    s = dt.random_instance(2000, seed=29)
    ys = np.random.default_rng(30).uniform(0, 1, 100)
    scale = float(np.abs(_np(s.qs)).sum())
    plain = dt.evaluate_direct(s, k, ys).values
    kahan = dt.evaluate_direct(s, k, ys, compensated=True).values
    assert np.max(np.abs(plain - kahan)) <= 1e-13 * scale
    s = dt.random_instance(2000, seed=31)
    xs = _np(s.xs).copy()
    sym = dt.evaluate_direct(s, k, xs).values
    kahan = dt.evaluate_direct(s, k, xs, compensated=True).values
    assert np.max(np.abs(sym - kahan)) <= 1e-13 * float(np.abs(_np(s.qs)).sum())
    s = dt.random_instance(1000, seed=32)
    ys = _np(s.xs)[::2].copy()
    a = dt.evaluate_direct(s, k, ys, compensated=True, threads=1).values
    b = dt.evaluate_direct(s, k, ys, compensated=True, threads=3).values
    np.testing.assert_array_equal(a, b)


def test_random_instance_reproducible_and_in_interval(dt):
    """TestRandomInstance (test_metrics.py:73-86): same seed, same charges;
    positions inside the interval and sorted, strengths non-negative."""
    a, b = dt.random_instance(100, seed=5), dt.random_instance(100, seed=5)
    np.testing.assert_array_equal(_np(a.xs), _np(b.xs))
    np.testing.assert_array_equal(_np(a.qs), _np(b.qs))
    s = dt.random_instance(200, seed=6, interval=(2.0, 3.0))
    xs, qs = _np(s.xs), _np(s.qs)
    assert np.all(xs >= 2.0) and np.all(xs <= 3.0)
    assert np.all(np.diff(xs) >= 0) and np.all(qs >= 0)
