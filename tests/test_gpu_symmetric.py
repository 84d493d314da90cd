"""targets == sources direct sums, each pair once (dt_phi_sum_symmetric,
mirror of _kernels.phi_sum_symmetric, _kernels.py:107-142): against the plain
GPU kernel and the C oracle, across band boundaries (2048 rows per band),
determinism and accumulate mode.  n = 70001 and 100003 span 3 and 4 column
chunks of 32768 (several row partials per target, the combine's chunk loop)."""
import numpy as np
import pytest
import torch

import paper_1710_05781_b200 as dt

pytestmark = pytest.mark.gpu


def _instance(n, seed):
    rng = np.random.default_rng(seed)
    xs = np.sort(rng.uniform(-1.0, 1.0, n))
    if n > 10:
        xs[n // 3: n // 3 + 4] = xs[n // 3]  # coincident sources (d = 0 pairs)
    qs = rng.uniform(-1e-3, 1e-3, n) + 2e-4
    return xs, qs


@pytest.mark.parametrize("n", [1, 2, 100, 2047, 2048, 2049, 4096, 5000, 20011, 70001, 100003])
def test_symmetric_matches_plain_and_oracle(n):
    from oracle import oracle as O
    from paper_1710_05781_b200.direct import phi_sum_direct, phi_sum_symmetric

    xs, qs = _instance(n, n)
    rd2 = 0.01 ** 2
    x, q = torch.from_numpy(xs).cuda(), torch.from_numpy(qs).cuda()
    sym = torch.zeros(n, dtype=torch.float64, device="cuda")
    assert phi_sum_symmetric(x, q, rd2, sym, accumulate=False)
    plain = torch.zeros_like(sym)
    phi_sum_direct(x, q, x, rd2, plain)
    scale = float(np.abs(qs).sum())
    got = sym.cpu().numpy()
    assert np.isfinite(got).all()
    assert np.max(np.abs(got - plain.cpu().numpy())) <= 1e-13 * scale
    # the oracle's full field minus its sign term is the kernel sum
    idx = np.unique(np.linspace(0, n - 1, min(n, 64)).astype(np.int64))
    want = O.evaluate_direct(xs, qs, 0.01, xs[idx])
    sys = dt.from_sorted(xs, qs)
    e = dt.sign_term_all(sys, torch.from_numpy(xs[idx]).cuda())
    e = e.cpu().numpy() if hasattr(e, "cpu") else np.asarray(e)
    assert np.max(np.abs(got[idx] + e - want)) <= 1e-13 * scale
    # bitwise deterministic; accumulate adds onto out
    again = torch.ones_like(sym)
    assert phi_sum_symmetric(x, q, rd2, again, accumulate=True)
    np.testing.assert_array_equal(again.cpu().numpy() - 1.0, (sym + 1.0).cpu().numpy() - 1.0)
    again2 = torch.zeros_like(sym)
    phi_sum_symmetric(x, q, rd2, again2, accumulate=False)
    np.testing.assert_array_equal(again2.cpu().numpy(), got)


def test_evaluate_direct_dispatches_symmetric():
    """evaluate_direct on targets == sources (direct.py:80) takes the symmetric
    path and agrees with the same call on a copy offset by nothing but object
    identity (plain path on distinct but equal targets is also symmetric), and
    with the plain kernel on a permutation of the targets."""
    xs, qs = _instance(6000, 7)
    sys = dt.from_sorted(xs, qs)
    k = dt.DiscKernel(0.005)
    a = dt.evaluate_direct(sys, k, xs).values
    perm = np.random.default_rng(1).permutation(len(xs))
    b = dt.evaluate_direct(sys, k, xs[perm]).values  # not equal to xs: plain kernel
    scale = float(np.abs(qs).sum())
    assert np.max(np.abs(np.asarray(a)[perm] - np.asarray(b))) <= 1e-13 * scale
