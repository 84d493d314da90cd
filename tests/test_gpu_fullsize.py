"""Full-size GPU parity (BASELINE configs at their stated sizes).

The CPU oracle finishes a full build in seconds, so the tree structure is
compared bit for bit at full size; fields, interaction lists and orders are
compared on strided target samples (the oracle's adaptive traversal costs
~0.1 ms per target per thread).  Size-independent properties: tree vs
direct within the adaptive tolerance.
"""

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1710_05781_b200 as pkg

    return pkg


def _check_config(dt, w, n_sample=4096, direct_sample=512):
    from oracle import oracle as O
    from paper_1710_05781_b200 import _lib
    from paper_1710_05781_b200.tree import tree_phi_sum

    system = dt.from_sorted(w.xs, w.qs)
    kernel = dt.DiscKernel(w.r_d)
    cfg = dt.EvalConfig(p=w.p, theta=w.theta, leaf_capacity=w.leaf_capacity,
                        adaptive=w.adaptive, tolerance=w.tolerance)
    tree = dt.build(system, kernel, cfg)
    # (b) structure bit-exact at full size
    ot = O.build_structure(w.xs, w.leaf_capacity)
    host = tree.numpy()
    for f in O.NODE_FIELDS:
        np.testing.assert_array_equal(host[f], getattr(ot, f), err_msg=f)
    assert tree.depth == ot.depth and tree.leaf_count == ot.leaf_count
    # (d)+(e) full evaluation on the GPU, sample checked against the oracle
    ys = torch.from_numpy(w.targets).cuda()
    full = dt.evaluate_all(tree, kernel, cfg, system, ys).values
    T = ys.numel()
    idx = np.unique(np.linspace(0, T - 1, n_sample).astype(np.int64))
    t = w.targets[idx]
    ot.moment_order = tree.moment_order
    ot.moments = tree.moments.cpu().numpy()  # oracle traversal over the GPU moments
    phi_o, st = O.tree_phi_sum(ot, w.xs, w.qs, w.r_d**2, w.theta, w.p, w.adaptive,
                               O.tol_share(w.tolerance, ot.depth), t, instrument=True)
    pre = O.prefix(w.qs)
    e_o = O.sign_terms(w.xs, pre, float(pre[-1]), t)
    scale = float(np.abs(w.qs).sum())
    got = full[torch.from_numpy(idx).cuda()].cpu().numpy()
    assert np.max(np.abs(got - (e_o + phi_o))) <= 1e-12 * scale
    # interaction lists + orders identical on the sample
    ts = torch.from_numpy(t).cuda()
    names = ("hash", "near_pairs", "n_far", "sum_p", "n_p0", "n_exact")
    bufs = {k: torch.zeros(len(t), dtype=torch.int64, device="cuda") for k in names}
    stats = _lib.EvalStats(*[bufs[k].data_ptr() for k in names])
    tree_phi_sum(tree, kernel, cfg, ts, torch.zeros_like(ts), accumulate=False, stats=stats)
    np.testing.assert_array_equal(bufs["hash"].cpu().numpy().view(np.uint64), st.hash)
    np.testing.assert_array_equal(bufs["sum_p"].cpu().numpy(), st.sum_p)
    # tree vs direct within the adaptive tolerance (test_tree.py:204-213)
    didx = idx[:: max(1, len(idx) // direct_sample)]
    dres = dt.evaluate_direct(system, kernel, w.targets[didx]).values
    err = np.abs(full[torch.from_numpy(didx).cuda()].cpu().numpy() - dres)
    if w.adaptive:
        assert err.max() <= w.tolerance * scale
    return tree, full


def test_cfg1_full(dt):
    from paper_1710_05781_b200 import workloads as W

    _check_config(dt, W.cfg1())


def test_cfg2_full(dt):
    from paper_1710_05781_b200 import workloads as W

    tree, _ = _check_config(dt, W.cfg2(), n_sample=8192)
    assert tree.depth >= 28


def test_cfg3_full(dt):
    from paper_1710_05781_b200 import workloads as W

    _check_config(dt, W.cfg3(r_d=1e-2, tolerance=1e-8), n_sample=2048, direct_sample=64)


@pytest.mark.parametrize("r_d,tol", [(1e-4, 1e-12), (1e-1, 1e-8)])
def test_cfg3_geometry_sweep_reduced(dt, r_d, tol):
    """configs[3]'s r_d / tolerance sweep at 2^23 sources, 2^22 targets."""
    from paper_1710_05781_b200 import workloads as W

    _check_config(dt, W.cfg3(r_d=r_d, tolerance=tol, cells=1 << 21, n_targets=1 << 22),
                  n_sample=2048, direct_sample=64)


def test_cfg4_direct_full(dt):
    """configs[4]: 2^20 x 2^20 direct sums, fp64 and fp32-eval variants."""
    from oracle import oracle as O
    from paper_1710_05781_b200 import workloads as W

    w = W.cfg4()
    system = dt.from_sorted(w.xs, w.qs)
    kernel = dt.DiscKernel(w.r_d)
    ys = torch.from_numpy(w.targets).cuda()
    e64 = dt.evaluate_direct(system, kernel, ys).values
    e32 = dt.evaluate_direct(system, kernel, ys, precision="fp32").values
    idx = np.linspace(0, len(w.targets) - 1, 256).astype(np.int64)
    want = O.evaluate_direct(w.xs, w.qs, w.r_d, w.targets[idx])
    scale = float(np.abs(w.qs).sum())
    sel = torch.from_numpy(idx).cuda()
    assert np.max(np.abs(e64[sel].cpu().numpy() - want)) <= 1e-13 * scale
    assert np.max(np.abs(e32[sel].cpu().numpy() - want)) <= 1e-6 * scale
