"""GPU tests of the public-API host paths (pinned / numpy targets streamed in
chunks, one-pass input validation)."""

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


@pytest.fixture(scope="module")
def case(dt):
    from paper_1710_05781_b200 import workloads as W

    w = W.cfg1(cells=1 << 18)  # 2^20 sources and targets
    system = dt.from_sorted(w.xs, w.qs)
    kernel = dt.DiscKernel(w.r_d)
    cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True,
                        tolerance=w.tolerance)
    tree = dt.build(system, kernel, cfg)
    want = dt.evaluate_all(tree, kernel, cfg, system, torch.from_numpy(w.targets).cuda())
    return w, system, kernel, cfg, tree, want.values.cpu().numpy()


@pytest.mark.parametrize("chunk", [1 << 17, 1 << 21])
@pytest.mark.parametrize("kind", ["pinned", "cpu", "numpy"])
def test_pipelined_host_targets_bit_identical(dt, case, monkeypatch, chunk, kind):
    from paper_1710_05781_b200 import tree as T

    w, system, kernel, cfg, tree, want = case
    monkeypatch.setattr(T, "PIPELINE_CHUNK", chunk)
    t = w.targets.copy()
    arg = {"pinned": torch.from_numpy(t).pin_memory(), "cpu": torch.from_numpy(t),
           "numpy": t}[kind]
    res = dt.evaluate_all(tree, kernel, cfg, system, arg)
    got = res.values if kind == "numpy" else res.values.numpy()
    assert isinstance(res.values, np.ndarray) == (kind == "numpy")
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("pinned", [False, True])
def test_host_paths_reject_non_finite(dt, case, pinned):
    w, system, kernel, cfg, tree, _ = case
    t = w.targets.copy()
    t[len(t) // 2] = np.nan
    t[7] = np.inf
    arg = torch.from_numpy(t).pin_memory() if pinned else t
    with pytest.raises(ValueError, match="finite"):
        dt.evaluate_all(tree, kernel, cfg, system, arg)


def test_field_packed_abi_device_and_host(dt, case):
    """dt_tree_field_packed on device and on pinned host buffers equals
    sign term + traversal (bit for bit)."""
    from paper_1710_05781_b200 import _lib
    from paper_1710_05781_b200.tree import _tol_share, contour_tables

    w, system, kernel, cfg, tree, want = case
    L, p = _lib.load(), _lib.ptr
    cos_t, sin_t = contour_tables(system.xs.device)
    ws = torch.empty(_lib.DT_EVAL_COUNTER_BYTES, dtype=torch.uint8, device="cuda")
    for where in ("cuda", "pinned"):
        ys = torch.from_numpy(w.targets.copy())
        ys = ys.cuda() if where == "cuda" else ys.pin_memory()
        out = torch.full_like(ys, float("nan"))
        if where == "pinned":
            out = out.pin_memory()
        flags = torch.zeros(2, dtype=torch.int64, device="cuda")
        rc = L.dt_tree_field_packed(
            p(tree.packed), len(tree), p(tree.meval), tree.meval.shape[1], p(tree.xq),
            p(system.xs), p(system.prefix), len(system), kernel.r_d ** 2, float(cfg.theta),
            int(cfg.p), 1, _tol_share(tree, cfg), int(tree.moment_order), p(cos_t), p(sin_t),
            cos_t.numel(), ys.data_ptr(), out.data_ptr(), 3, len(ys) - 5, p(flags), p(ws),
            ws.numel(), None)
        assert rc == 0
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        np.testing.assert_array_equal(got[3:-5], want[3:-5])
        assert np.isnan(got[:3]).all() and np.isnan(got[-5:]).all()
        assert flags.tolist() == [0, 0]
    # with the bracket workspace, sorted and shuffled targets alike
    big = torch.empty(int(L.dt_tree_field_workspace(len(w.targets))), dtype=torch.uint8,
                      device="cuda")
    perm = np.random.default_rng(8).permutation(len(w.targets))
    for order in (np.arange(len(w.targets)), perm):
        ys = torch.from_numpy(w.targets[order].copy()).cuda()
        out = torch.full_like(ys, float("nan"))
        rc = L.dt_tree_field_packed(
            p(tree.packed), len(tree), p(tree.meval), tree.meval.shape[1], p(tree.xq),
            p(system.xs), p(system.prefix), len(system), kernel.r_d ** 2, float(cfg.theta),
            int(cfg.p), 1, _tol_share(tree, cfg), int(tree.moment_order), p(cos_t), p(sin_t),
            cos_t.numel(), ys.data_ptr(), out.data_ptr(), 0, len(ys), None, p(big), big.numel(),
            None)
        assert rc == 0
        np.testing.assert_array_equal(out.cpu().numpy(), want[order])
    # pageable host memory is refused before any device work
    ys = torch.from_numpy(w.targets.copy())
    out = torch.empty_like(ys)
    rc = L.dt_tree_field_packed(
        p(tree.packed), len(tree), p(tree.meval), tree.meval.shape[1], p(tree.xq), p(system.xs),
        p(system.prefix), len(system), kernel.r_d ** 2, float(cfg.theta), int(cfg.p), 1,
        _tol_share(tree, cfg), int(tree.moment_order), p(cos_t), p(sin_t), cos_t.numel(),
        ys.data_ptr(), out.data_ptr(), 0, len(ys), None, p(ws), ws.numel(), None)
    assert rc == -1 and b"pinned" in L.dt_last_error()
    # misaligned node records (32-byte loads) and moment rows are refused
    ys = torch.from_numpy(w.targets.copy()).cuda()
    out = torch.empty_like(ys)
    for shift_nodes, shift_m in ((16, 0), (0, 8)):
        rc = L.dt_tree_field_packed(
            tree.packed.data_ptr() + shift_nodes, len(tree), tree.meval.data_ptr() + shift_m,
            tree.meval.shape[1], p(tree.xq), p(system.xs), p(system.prefix), len(system),
            kernel.r_d ** 2, float(cfg.theta), int(cfg.p), 1, _tol_share(tree, cfg),
            int(tree.moment_order), p(cos_t), p(sin_t), cos_t.numel(), ys.data_ptr(),
            out.data_ptr(), 0, len(ys), None, p(ws), ws.numel(), None)
        assert rc == -1 and b"aligned" in L.dt_last_error()
    rc = L.dt_tree_field_packed(
        p(tree.packed), len(tree), p(tree.meval), tree.meval.shape[1] - 1, p(tree.xq),
        p(system.xs), p(system.prefix), len(system), kernel.r_d ** 2, float(cfg.theta),
        int(cfg.p), 1, _tol_share(tree, cfg), int(tree.moment_order), p(cos_t), p(sin_t),
        cos_t.numel(), ys.data_ptr(), out.data_ptr(), 0, len(ys), None, p(ws), ws.numel(), None)
    assert rc == -1 and b"even" in L.dt_last_error()


def test_unsorted_host_targets_take_the_sorting_path(dt, case):
    w, system, kernel, cfg, tree, want = case
    perm = np.random.default_rng(5).permutation(len(w.targets))
    got = dt.evaluate_all(tree, kernel, cfg, system, w.targets[perm]).values
    np.testing.assert_array_equal(got, want[perm])


def test_from_particles_validation_and_sort(dt):
    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, 5000)
    q = rng.normal(size=5000)
    s = dt.from_particles(np.column_stack([x, q]))
    order = np.argsort(x, kind="stable")
    np.testing.assert_array_equal(s.xs.cpu().numpy(), x[order])
    np.testing.assert_array_equal(s.qs.cpu().numpy(), q[order])
    for bad in (np.inf, -np.inf, np.nan):
        y = x.copy()
        y[77] = bad
        with pytest.raises(ValueError, match="finite"):
            dt.from_particles(np.column_stack([y, q]))
        r = q.copy()
        r[4999] = bad
        with pytest.raises(ValueError, match="finite"):
            dt.from_particles(np.column_stack([x, r]))
    # already sorted input: no sort, same arrays
    s2 = dt.from_particles(torch.from_numpy(np.column_stack([x[order], q[order]])).cuda())
    assert torch.equal(s2.xs, s.xs) and torch.equal(s2.qs, s.qs)


def test_check_values_counts(dt):
    from paper_1710_05781_b200.charges import check_values

    v = torch.tensor([0.0, 1.0, 1.0, 0.5, float("inf"), 2.0, float("nan"), 3.0],
                     dtype=torch.float64, device="cuda")
    bad, desc = check_values(v).tolist()
    assert bad == 2
    assert desc == 2  # 1.0 -> 0.5 and inf -> 2.0 (comparisons with NaN are false)


def test_pipeline_fused_sign_matches_separate():
    """The device pipeline with the sign term fused into the traversal
    (dt_tree_field_device) gives the same field bit for bit as the separate
    sign-term kernel + accumulate."""
    import paper_1710_05781_b200 as dt
    from paper_1710_05781_b200 import workloads as W
    from paper_1710_05781_b200.pipeline import TreePipeline

    w = W.cfg2(cells=1 << 14)
    k = dt.DiscKernel(w.r_d)
    cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=1e-10)
    xs, qs, ys = (torch.from_numpy(a).cuda() for a in (w.xs, w.qs, w.targets))
    outs = []
    for fused in (False, True):
        pipe = TreePipeline.planned(xs, ys.numel(), k, cfg, fused_sign=fused)
        out = torch.full_like(ys, float("nan"))
        pipe.step(xs, qs, ys, out)
        pipe.check()
        outs.append(out)
    assert torch.equal(outs[0], outs[1])
