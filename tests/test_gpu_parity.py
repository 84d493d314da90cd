"""GPU parity: the sm_100a path against the golden fixtures (produced by the
live reference) and against the CPU oracle.  Needs a B200."""

import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, TREE_CASES, load_case

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1710_05781_b200 as pkg

    return pkg


def _system(dt, g):
    return dt.from_particles(np.column_stack([g["xs"], g["qs"]]))


def _config(dt, g):
    return dt.EvalConfig(p=int(g["p"]), theta=float(g["theta"]),
                         leaf_capacity=int(g["leaf_capacity"]), adaptive=bool(g["adaptive"]),
                         tolerance=float(g["tolerance"]))


@pytest.mark.parametrize("name", TREE_CASES)
def test_structure_bit_exact(dt, name):
    g = load_case(name)
    system = _system(dt, g)
    np.testing.assert_array_equal(system.xs.cpu().numpy(), g["xs"])
    tree = dt.build(system, dt.DiscKernel(float(g["r_d"])), _config(dt, g))
    host = tree.numpy()
    for f in ("lo", "hi", "center", "half", "level", "start", "end", "left", "right"):
        np.testing.assert_array_equal(host[f], g[f], err_msg=f)
    assert tree.depth == int(g["depth"])
    assert tree.leaf_count == int(g["leaf_count"])
    assert tree.moment_order == int(g["moment_order"])


@pytest.mark.parametrize("name", TREE_CASES)
def test_moments(dt, name):
    from test_oracle_golden import moment_scale

    g = load_case(name)
    tree = dt.build(_system(dt, g), dt.DiscKernel(float(g["r_d"])), _config(dt, g))
    m = tree.moments.cpu().numpy()
    scale = moment_scale(g)
    # M2M accumulates round-off along a node's ancestry (about depth * order
    # ulps of the natural scale); the reference sums every node directly.
    tol = 1e-13 * max(1.0, int(g["depth"]) / 6.0)
    ratio = np.abs(m - g["moments"]) / (scale + 1e-300)
    assert np.all(np.abs(m - g["moments"]) <= tol * scale + 1e-300), float(ratio.max())


@pytest.mark.parametrize("name", TREE_CASES)
def test_tree_field_vs_reference(dt, name):
    """north_star: fields within 1e-12 of the reference's tree output.

    Full field E = e + phi: max |dE| <= 1e-12 sum|q| (the normalisation of
    the reference's own tests, test_tree.py:168-172).  The kernel-sum part
    phi (the reference's tree_phi_sum seam output) additionally meets
    avg_relative <= 1e-12 (metrics.error_report).  The e term rests on the
    reference's sequential np.cumsum, whose own drift dominates E when E is
    a small difference of O(sum|q|) terms; it is checked in test_sign_terms.
    """
    from paper_1710_05781_b200.tree import tree_phi_sum

    g = load_case(name)
    system = _system(dt, g)
    kernel = dt.DiscKernel(float(g["r_d"]))
    cfg = _config(dt, g)
    tree = dt.build(system, kernel, cfg)
    res = dt.evaluate_all(tree, kernel, cfg, system, g["targets"])
    assert isinstance(res.values, np.ndarray) and res.method == "tree"
    scale = np.abs(g["qs"]).sum()
    assert np.max(np.abs(res.values - g["E_tree"])) <= 1e-12 * scale
    ys = torch.from_numpy(g["targets"]).cuda()
    phi = torch.zeros_like(ys)
    tree_phi_sum(tree, kernel, cfg, ys, phi, accumulate=False)
    phi = phi.cpu().numpy()
    dphi = np.abs(phi - g["phi_tree"])
    assert dphi.max() <= 1e-13 * scale
    if np.abs(g["phi_tree"]).sum() > 0:
        assert dt.error_report(phi, g["phi_tree"]).avg_relative <= 1e-12


@pytest.mark.parametrize("name", TREE_CASES)
def test_interaction_lists_vs_oracle(dt, name):
    """Per-target interaction lists (far node ids with p_use, near leaves, DFS
    order) hash-identical to the oracle's replica of _kernels.py:199-264."""
    from oracle import oracle as O
    from paper_1710_05781_b200 import _lib
    from paper_1710_05781_b200.tree import tree_phi_sum

    g = load_case(name)
    system = _system(dt, g)
    kernel = dt.DiscKernel(float(g["r_d"]))
    cfg = _config(dt, g)
    tree = dt.build(system, kernel, cfg)
    t = np.sort(g["targets"])
    ys = torch.from_numpy(t).cuda()
    out = torch.zeros_like(ys)
    T = len(t)
    bufs = {k: torch.zeros(T, dtype=torch.int64, device="cuda")
            for k in ("hash", "near_pairs", "n_far", "sum_p", "n_p0", "n_exact")}
    st = _lib.EvalStats(*[bufs[k].data_ptr() for k in
                          ("hash", "near_pairs", "n_far", "sum_p", "n_p0", "n_exact")])
    tree_phi_sum(tree, kernel, cfg, ys, out, accumulate=False, stats=st)
    otree = O.build(g["xs"], g["qs"], cfg.p, cfg.leaf_capacity, cfg.adaptive)
    _, ost = O.tree_phi_sum(otree, g["xs"], g["qs"], kernel.r_d ** 2, cfg.theta, cfg.p,
                            cfg.adaptive, O.tol_share(cfg.tolerance, otree.depth), t,
                            instrument=True)
    np.testing.assert_array_equal(bufs["near_pairs"].cpu().numpy(), ost.near_pairs)
    np.testing.assert_array_equal(bufs["n_far"].cpu().numpy(), ost.n_far)
    np.testing.assert_array_equal(bufs["sum_p"].cpu().numpy(), ost.sum_p)
    np.testing.assert_array_equal(bufs["hash"].cpu().numpy().view(np.uint64), ost.hash)


def test_pchoice_golden(dt):
    """Adaptive orders equal the compiled reference's on the golden samples,
    in both selection modes."""
    from paper_1710_05781_b200 import _lib
    from paper_1710_05781_b200.tree import contour_tables

    with np.load(os.path.join(GOLDEN, "pchoice.npz")) as z:
        d = {k: z[k] for k in z.files}
    cos_t, sin_t = contour_tables(torch.device("cuda"))
    L = _lib.load()
    groups = {}
    for i, key in enumerate(zip(d["rd2"], d["tol"], d["p_cap"])):
        groups.setdefault(key, []).append(i)
    for mode in (_lib.DT_PSEL_FAST, _lib.DT_PSEL_EXACT):
        for (rd2, tol, cap), idx in groups.items():
            idx = np.array(idx)
            R = torch.from_numpy(d["big_r"][idx]).cuda()
            H = torch.from_numpy(d["h"][idx]).cuda()
            p_out = torch.empty(len(idx), dtype=torch.int64, device="cuda")
            _lib.check(L.dt_choose_p_batch(_lib.ptr(R), _lib.ptr(H), len(idx), float(rd2),
                                           float(tol), int(cap), _lib.ptr(cos_t),
                                           _lib.ptr(sin_t), 64, mode, _lib.ptr(p_out), None,
                                           _lib.stream_handle()), "choose_p")
            np.testing.assert_array_equal(p_out.cpu().numpy(), d["p_use"][idx])


def test_pchoice_random_vs_oracle(dt):
    """2e5 random (R, h) pairs at the configs' radii/tolerances: the fast tier
    and its fallbacks reproduce the exact replica bit for bit."""
    from oracle import oracle as O
    from paper_1710_05781_b200 import _lib
    from paper_1710_05781_b200.tree import contour_tables

    rng = np.random.default_rng(11)
    cos_t, sin_t = contour_tables(torch.device("cuda"))
    L = _lib.load()
    for rd in (0.01, 0.005, 1e-4, 0.1):
        for tol in (1e-10 / 42.0, 1e-12 / 63.0, 1e-8 / 60.0):
            n = 12500
            R = 10.0 ** rng.uniform(-9.0, 0.4, n)
            H = R * rng.uniform(0.0, 1.0 / 3.0, n)
            Rt, Ht = torch.from_numpy(R).cuda(), torch.from_numpy(H).cuda()
            p_out = torch.empty(n, dtype=torch.int64, device="cuda")
            tier = torch.empty(n, dtype=torch.int32, device="cuda")
            _lib.check(L.dt_choose_p_batch(_lib.ptr(Rt), _lib.ptr(Ht), n, rd * rd, tol, 30,
                                           _lib.ptr(cos_t), _lib.ptr(sin_t), 64,
                                           _lib.DT_PSEL_FAST, _lib.ptr(p_out), _lib.ptr(tier),
                                           _lib.stream_handle()), "choose_p")
            want = np.array([O.choose_p(a, b, rd * rd, tol, 30) for a, b in zip(R, H)])
            got = p_out.cpu().numpy()
            bad = np.nonzero(got != want)[0]
            assert len(bad) == 0, (rd, tol, R[bad[:3]], H[bad[:3]], got[bad[:3]], want[bad[:3]])
            assert (tier.cpu().numpy() > 0).mean() < 0.05


@pytest.mark.parametrize("name", [n for n in TREE_CASES if "phi_kahan" in load_case(n)])
def test_direct_vs_reference(dt, name):
    from paper_1710_05781_b200 import _lib
    from paper_1710_05781_b200.direct import phi_sum_direct

    g = load_case(name)
    system = _system(dt, g)
    kernel = dt.DiscKernel(float(g["r_d"]))
    scale = np.abs(g["qs"]).sum()
    res = dt.evaluate_direct(system, kernel, g["targets"])
    assert np.max(np.abs(res.values - g["E_direct"])) <= 1e-12 * scale
    ys = torch.from_numpy(g["targets"]).cuda()

    def phi(mode):
        out = torch.zeros_like(ys)
        phi_sum_direct(system.xs, system.qs, ys, kernel.r_d ** 2, out, mode, accumulate=False)
        return out.cpu().numpy()

    assert np.max(np.abs(phi(_lib.DT_DIRECT_FP64) - g["phi_plain"])) <= 1e-13 * scale
    # Kahan: bit-identical to the reference's phi_sum_kahan
    np.testing.assert_array_equal(phi(_lib.DT_DIRECT_KAHAN), g["phi_kahan"])
    assert np.max(np.abs(phi(_lib.DT_DIRECT_FP32) - g["phi_plain"])) <= 1e-5 * scale


@pytest.mark.parametrize("name", TREE_CASES)
def test_sign_terms(dt, name):
    g = load_case(name)
    system = _system(dt, g)
    e = dt.charges._sign_terms(system, torch.from_numpy(g["targets"]).cuda()).cpu().numpy()
    scale = max(np.abs(g["qs"]).sum(), 1e-300)
    assert np.max(np.abs(e - g["sign"])) <= 1e-13 * scale
    assert abs(system.total - float(g["total"])) <= 1e-13 * scale


def test_permutation_and_repeat_invariance(dt):
    g = load_case("cfg1s")
    system = _system(dt, g)
    kernel = dt.DiscKernel(float(g["r_d"]))
    cfg = _config(dt, g)
    tree = dt.build(system, kernel, cfg)
    t = g["targets"]
    base = dt.evaluate_all(tree, kernel, cfg, system, t).values
    again = dt.evaluate_all(tree, kernel, cfg, system, t, threads=None).values
    np.testing.assert_array_equal(base, again)
    perm = np.random.default_rng(3).permutation(len(t))
    shuffled = dt.evaluate_all(tree, kernel, cfg, system, t[perm]).values
    np.testing.assert_array_equal(shuffled, base[perm])
    # torch in -> torch out, same values
    tv = dt.evaluate_all(tree, kernel, cfg, system, torch.from_numpy(t).cuda()).values
    assert isinstance(tv, torch.Tensor) and tv.is_cuda
    np.testing.assert_array_equal(tv.cpu().numpy(), base)


def test_reference_hand_values(dt):
    """test_direct.py:37-59 hand cases and test_tree.py edge cases."""
    k = dt.DiscKernel(0.1)
    s = dt.from_particles([(0.0, 1.0)])
    r = dt.evaluate_direct(s, k, [0.5])
    assert r.values[0] == pytest.approx(1.0 - 0.5 / math.sqrt(0.26), rel=1e-15)
    assert r.method == "direct" and r.build_time == 0.0
    s = dt.from_particles([(0.3, 2.5)])
    assert dt.evaluate_direct(s, k, [0.3]).values[0] == -2.5
    s = dt.from_particles([(0.25, 0.7), (0.75, 0.7)])
    assert dt.evaluate_direct(s, k, [0.5]).values[0] == 0.0
    assert dt.evaluate_direct(dt.from_particles([]), k, [0.5]).values[0] == 0.0
    assert dt.evaluate_direct(s, k, []).values.shape == (0,)
    with pytest.raises(ValueError):
        dt.evaluate_direct(s, k, [np.nan])
    with pytest.raises(ValueError):
        dt.build(dt.from_particles([]), k, dt.EvalConfig())
    tree = dt.build(dt.from_particles([(0.2, 1.0)]), k, dt.EvalConfig())
    assert len(tree) == 1 and tree.root.is_leaf and tree.root.half_width > 0
    got = dt.evaluate_point(tree, k, dt.EvalConfig(), 0.9)
    assert got == pytest.approx(dt.phi(k, 0.2, 0.9), rel=1e-15)
    with pytest.raises(ValueError):
        dt.evaluate_all(tree, k, dt.EvalConfig(p=11), tree.system, [0.5])
    res = dt.evaluate_all(tree, k, dt.EvalConfig(), tree.system, [])
    assert res.values.shape == (0,)


def test_sign_term_api(dt):
    s = dt.from_particles([(0.0, 1.0), (1.0, 2.0), (2.0, 4.0)])
    np.testing.assert_array_equal(dt.sign_term_all(s, [0.5, 1.5]), [-5.0, -1.0])
    s1 = dt.from_particles([(1.0, 3.0)])
    np.testing.assert_array_equal(dt.sign_term_all(s1, [1.0]), [-3.0])
    np.testing.assert_array_equal(dt.sign_term_all(s1, [1.0 + 1e-12]), [3.0])
    with pytest.raises(ValueError):
        dt.sign_term_all(s1, [1.0, 0.5])
    sd = dt.from_particles([(1.0, 10.0), (1.0, 20.0), (0.0, 5.0)])
    np.testing.assert_array_equal(sd.qs.cpu().numpy(), [5.0, 10.0, 20.0])


def test_direct_matches_mpmath(dt):
    """test_direct.py:61-80 (50-digit oracle), rel 1e-13."""
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.dps = 50
    rng = np.random.default_rng(21)
    xs, qs = rng.uniform(0, 1, 40), rng.uniform(-1, 1, 40)
    s = dt.from_particles(np.column_stack([xs, qs]))
    k = dt.DiscKernel(0.05)
    targets = np.array([-0.3, 0.0, 0.25, 0.5, 0.8, 1.0, 1.4])
    got = dt.evaluate_direct(s, k, targets).values
    for v, y in zip(got, targets):
        tot = below = acc = mpmath.mpf(0)
        for x, q in zip(xs, qs):
            tot += mpmath.mpf(q)
            if x < y:
                below += mpmath.mpf(q)
            dd = mpmath.mpf(x) - mpmath.mpf(y)
            acc += mpmath.mpf(q) * dd / mpmath.sqrt(dd * dd + mpmath.mpf(0.05) ** 2)
        assert v == pytest.approx(float(2 * below - tot + acc), rel=1e-13, abs=1e-13)


def test_seam_mirror_entry(dt):
    """dt_tree_phi_sum takes the reference seam's SoA arrays and moments
    (_kernels.py:164-186) and matches the packed path."""
    from paper_1710_05781_b200 import _lib
    from paper_1710_05781_b200.tree import contour_tables, tree_phi_sum

    g = load_case("cfg2s")
    system = _system(dt, g)
    kernel = dt.DiscKernel(float(g["r_d"]))
    cfg = _config(dt, g)
    tree = dt.build(system, kernel, cfg)
    ys = torch.from_numpy(g["targets"]).cuda()
    want = torch.zeros_like(ys)
    tree_phi_sum(tree, kernel, cfg, ys, want, accumulate=False)
    got = torch.zeros_like(ys)
    L = _lib.load()
    stride = tree.moment_order + 1
    ws_bytes = L.dt_tree_eval_workspace(len(tree), len(system), stride)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    c, s = contour_tables(ys.device)
    p = _lib.ptr
    _lib.check(L.dt_tree_phi_sum(
        p(tree.center), p(tree.half), p(tree.start), p(tree.end), p(tree.left), p(tree.right),
        p(tree.moments), stride, len(tree), p(system.xs), p(system.qs), len(system),
        kernel.r_d ** 2, cfg.theta, cfg.p, 1, cfg.tolerance / (3.0 * tree.depth),
        tree.moment_order, p(c), p(s), 64, p(ys), p(got), 0, ys.numel(), 0, p(ws), ws_bytes,
        _lib.stream_handle()), "dt_tree_phi_sum")
    scale = np.abs(g["qs"]).sum()
    assert float((got - want).abs().max()) <= 1e-14 * scale
    assert np.max(np.abs(got.cpu().numpy() - g["phi_tree"])) <= 1e-13 * scale


def test_sharded_evaluation_is_partition_invariant(dt):
    """Contiguous target slices per rank (parallel.shard_bounds) give a
    bit-identical field for any world size (the GPU analogue of the
    reference's thread-count invariance, test_tree.py:269-278)."""
    from paper_1710_05781_b200.parallel import gpu_slice_evaluator, shard_bounds

    g = load_case("cfg2s")
    system = _system(dt, g)
    kernel = dt.DiscKernel(float(g["r_d"]))
    cfg = _config(dt, g)
    tree = dt.build(system, kernel, cfg)
    ys = torch.from_numpy(g["targets"]).cuda()
    base = dt.evaluate_all(tree, kernel, cfg, system, ys).values
    run = gpu_slice_evaluator(tree, kernel, cfg, system, ys)
    for world in (2, 3, 8):
        parts = [run(*shard_bounds(ys.numel(), world, r)) for r in range(world)]
        assert torch.equal(torch.cat(parts), base)


@pytest.mark.parametrize("p,adaptive,tol", [(40, False, 1e-10), (45, True, 1e-14),
                                             (64, False, 1e-10), (100, False, 1e-10),
                                             (127, False, 1e-10)])
def test_high_order_paths(dt, p, adaptive, tol):
    """Moment orders above 31: the warp-per-leaf dataflow upward pass and the
    wide (rolled) far-field loop.  Interaction lists hash-identical to the
    oracle, moments and field within the usual tolerances."""
    from oracle import oracle as O
    from paper_1710_05781_b200 import _lib
    from paper_1710_05781_b200.tree import tree_phi_sum

    g = load_case("rand_default")
    xs, qs = g["xs"], g["qs"]
    system = dt.from_sorted(xs, qs)
    r_d = 0.05
    kernel = dt.DiscKernel(r_d)
    cfg = dt.EvalConfig(p=p, leaf_capacity=16, adaptive=adaptive, tolerance=tol)
    tree = dt.build(system, kernel, cfg)
    assert tree.moment_order == p
    otree = O.build(xs, qs, p, 16, adaptive)
    m, om = tree.moments.cpu().numpy(), otree.moments
    # relative to each row's scale sum|q| r^k / k!
    r = np.maximum(np.abs(otree.hi - otree.center), np.abs(otree.center - otree.lo))
    from math import factorial
    scale = np.array([[np.abs(qs[s:e]).sum() * rk ** k / factorial(k) for k in range(p + 1)]
                      for s, e, rk in zip(otree.start, otree.end, r)])
    assert np.max(np.abs(m - om) / np.maximum(scale, 1e-300)) <= 1e-12
    t = np.sort(np.random.default_rng(4).uniform(xs[0] - 0.1, xs[-1] + 0.1, 3000))
    ys = torch.from_numpy(t).cuda()
    out = torch.zeros_like(ys)
    names = ("hash", "near_pairs", "n_far", "sum_p", "n_p0", "n_exact")
    bufs = {k: torch.zeros(len(t), dtype=torch.int64, device="cuda") for k in names}
    st = _lib.EvalStats(*[bufs[k].data_ptr() for k in names])
    tree_phi_sum(tree, kernel, cfg, ys, out, accumulate=False, stats=st)
    otree.moments = m  # same moments: the difference is the far-field arithmetic only
    phi_o, ost = O.tree_phi_sum(otree, xs, qs, r_d ** 2, cfg.theta, p, adaptive,
                                O.tol_share(tol, otree.depth), t, instrument=True)
    np.testing.assert_array_equal(bufs["hash"].cpu().numpy().view(np.uint64), ost.hash)
    np.testing.assert_array_equal(bufs["sum_p"].cpu().numpy(), ost.sum_p)
    assert bufs["sum_p"].sum().item() > 0
    got = out.cpu().numpy()
    assert np.isfinite(got).all()
    if np.isfinite(phi_o).all():
        assert np.max(np.abs(got - phi_o)) <= 1e-12 * np.abs(qs).sum()
    else:
        # the reference's four-term recurrence overflows (k!/rho^k) at the
        # top orders; the scaled three-term one does not: check against the
        # direct sum instead (the truncation error is negligible at p = 127)
        d = t[:, None] - xs[None, :]
        phi_d = (qs[None, :] * (xs[None, :] - t[:, None]) / np.sqrt(d * d + r_d ** 2)).sum(1)
        assert np.max(np.abs(got - phi_d)) <= 1e-11 * np.abs(qs).sum()


@pytest.mark.parametrize("case", ["cfg2s", "rand_adaptive", "cfg1s", "graded_2e20"])
def test_order_tables_vs_exact_replica(dt, case):
    """The traversal's adaptive orders through the per-level breakpoint
    tables (DT_PSEL_FAST) equal the exact replica's (DT_PSEL_EXACT, all 64
    samples for every pair): per-target interaction hashes and order sums."""
    from paper_1710_05781_b200 import _lib
    from paper_1710_05781_b200 import workloads as W
    from paper_1710_05781_b200.tree import tree_phi_sum

    if case == "graded_2e20":
        w = W.cfg2(cells=1 << 18)
        system = dt.from_sorted(w.xs, w.qs)
        kernel = dt.DiscKernel(w.r_d)
        cfg = dt.EvalConfig(p=w.p, theta=w.theta, leaf_capacity=w.leaf_capacity,
                            adaptive=True, tolerance=w.tolerance)
        ys = torch.from_numpy(w.targets[::7].copy()).cuda()
    else:
        g = load_case(case)
        system = _system(dt, g)
        kernel = dt.DiscKernel(float(g["r_d"]))
        cfg = dt.EvalConfig(p=int(g["p"]), theta=float(g["theta"]),
                            leaf_capacity=int(g["leaf_capacity"]), adaptive=True,
                            tolerance=float(g["tolerance"]) if bool(g["adaptive"]) else 1e-10)
        ys = torch.from_numpy(np.sort(g["targets"])).cuda()
    tree = dt.build(system, kernel, cfg)
    res = {}
    for mode in (_lib.DT_PSEL_FAST, _lib.DT_PSEL_EXACT):
        names = ("hash", "near_pairs", "n_far", "sum_p", "n_p0", "n_exact")
        bufs = {k: torch.zeros(len(ys), dtype=torch.int64, device="cuda") for k in names}
        st = _lib.EvalStats(*[bufs[k].data_ptr() for k in names])
        out = torch.zeros_like(ys)
        tree_phi_sum(tree, kernel, cfg, ys, out, accumulate=False, stats=st, psel_mode=mode)
        res[mode] = {k: v.cpu().numpy() for k, v in bufs.items()}
    f, e = res[_lib.DT_PSEL_FAST], res[_lib.DT_PSEL_EXACT]
    np.testing.assert_array_equal(f["hash"], e["hash"])
    np.testing.assert_array_equal(f["sum_p"], e["sum_p"])
    assert f["sum_p"].sum() > 0


@pytest.mark.parametrize("r_d", [1e-4, 5e-3, 1e-1])
@pytest.mark.parametrize("tol", [1e-4, 1e-8, 1e-12])
def test_order_tables_geometry_sweep(dt, r_d, tol):
    """Adaptive orders through the tables (breakpoint bins, and the interval
    bins of the low-order regime R << r_d on deep levels) equal the exact
    replica's over a sweep of r_d and tolerance on a graded mesh (depth ~24):
    per-target interaction hashes, order sums and counts of order-0 pairs."""
    from paper_1710_05781_b200 import _lib
    from paper_1710_05781_b200 import workloads as W
    from paper_1710_05781_b200.tree import tree_phi_sum

    w = W.cfg2(cells=1 << 16)
    system = dt.from_sorted(w.xs, w.qs)
    kernel = dt.DiscKernel(r_d)
    cfg = dt.EvalConfig(p=8, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=tol)
    ys = torch.from_numpy(w.targets[::5].copy()).cuda()
    tree = dt.build(system, kernel, cfg)
    res = {}
    for mode in (_lib.DT_PSEL_FAST, _lib.DT_PSEL_EXACT):
        names = ("hash", "near_pairs", "n_far", "sum_p", "n_p0", "n_exact")
        bufs = {k: torch.zeros(len(ys), dtype=torch.int64, device="cuda") for k in names}
        st = _lib.EvalStats(*[bufs[k].data_ptr() for k in names])
        out = torch.zeros_like(ys)
        tree_phi_sum(tree, kernel, cfg, ys, out, accumulate=False, stats=st, psel_mode=mode)
        res[mode] = {k: v.cpu().numpy() for k, v in bufs.items()}
    f, e = res[_lib.DT_PSEL_FAST], res[_lib.DT_PSEL_EXACT]
    np.testing.assert_array_equal(f["hash"], e["hash"])
    np.testing.assert_array_equal(f["sum_p"], e["sum_p"])
    np.testing.assert_array_equal(f["n_p0"], e["n_p0"])
    assert f["n_far"].sum() > 0
