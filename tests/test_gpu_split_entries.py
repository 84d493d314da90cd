"""The two-launch forms of the C ABI give the one-launch results bit for bit:
dt_eval_prepare + dt_tree_eval_device_prepared against dt_tree_eval_device,
and dt_sign_bracket + dt_sign_terms_bracketed against dt_sign_terms (the
device pipeline runs the first halves on another stream)."""

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


@pytest.mark.parametrize("cells,adaptive", [(1 << 12, True), (1 << 14, True), (1 << 12, False)])
def test_eval_prepare_split(dt, cells, adaptive):
    from paper_1710_05781_b200 import _lib
    from paper_1710_05781_b200 import workloads as W
    from paper_1710_05781_b200.tree import contour_tables

    w = W.cfg2(cells=cells)
    system = dt.from_sorted(w.xs, w.qs)
    kernel = dt.DiscKernel(w.r_d)
    cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=adaptive,
                        tolerance=w.tolerance)
    tree = dt.build(system, kernel, cfg)
    ys = torch.from_numpy(w.targets).cuda()
    cos_t, sin_t = contour_tables(ys.device)
    L = _lib.load()
    p = _lib.ptr
    cap = tree.packed.numel() // 32
    outs = []
    for split in (False, True):
        ws = torch.empty(_lib.DT_EVAL_COUNTER_BYTES, dtype=torch.uint8, device="cuda")
        out = torch.full_like(ys, 1.0)  # accumulate = 1: out + phi
        args = (p(tree.packed), p(tree.meta), cap, p(tree.meval), tree.meval.shape[1], p(tree.xq),
                len(system), w.r_d * w.r_d, float(cfg.theta), int(cfg.p), int(adaptive),
                float(cfg.tolerance), tree.moment_order, p(cos_t), p(sin_t), cos_t.numel(),
                p(ys), p(out), 0, ys.numel(), 1, p(ws), ws.numel(), _lib.stream_handle())
        if split:
            _lib.check(L.dt_eval_prepare(*args), "dt_eval_prepare")
            _lib.check(L.dt_tree_eval_device_prepared(*args), "dt_tree_eval_device_prepared")
        else:
            _lib.check(L.dt_tree_eval_device(*args), "dt_tree_eval_device")
        outs.append(out)
    torch.cuda.synchronize()
    assert torch.isfinite(outs[0]).all()
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("n,T,shuffle", [(5000, 7000, False), (70001, 3000, True), (300, 0, False),
                                         (0, 50, False)])
def test_sign_bracket_split(dt, n, T, shuffle):
    from paper_1710_05781_b200 import _lib
    from paper_1710_05781_b200.charges import prefix_sum

    rng = np.random.default_rng(n + T)
    xs = torch.from_numpy(np.sort(rng.uniform(-1, 1, n))).cuda()
    qs = torch.from_numpy(rng.normal(size=n)).cuda()
    y = np.sort(rng.uniform(-1.2, 1.2, T))
    if shuffle:
        y = rng.permutation(y)
    ys = torch.from_numpy(y).cuda()
    pre = prefix_sum(qs) if n else torch.empty(0, dtype=torch.float64, device="cuda")
    L = _lib.load()
    p = _lib.ptr
    sb = int(L.dt_sign_terms_workspace(T))
    outs = []
    for split in (False, True):
        ws = torch.empty(max(sb, 8), dtype=torch.uint8, device="cuda")
        e = torch.full_like(ys, float("nan"))
        if split:
            _lib.check(L.dt_sign_bracket(p(xs), n, p(ys), T, p(ws), sb, _lib.stream_handle()),
                       "dt_sign_bracket")
            _lib.check(L.dt_sign_terms_bracketed(p(xs), p(pre), n, p(ys), p(e), T, p(ws), sb,
                                                 _lib.stream_handle()), "dt_sign_terms_bracketed")
        else:
            _lib.check(L.dt_sign_terms(p(xs), p(pre), n, p(ys), p(e), T, p(ws), sb,
                                       _lib.stream_handle()), "dt_sign_terms")
        outs.append(e)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    if T:
        assert torch.isfinite(outs[0]).all()
