"""The device stable sort (dt_sort_stable, csrc/dt_sort.cu) against numpy's
np.argsort(kind="stable") (charges.py:127 from_particles): permutations
identical on random, duplicate-heavy, signed-zero, subnormal, huge and
presorted keys across tile boundaries; from_particles on unsorted pairs
against the oracle's stable sort."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _cases():
    rng = np.random.default_rng(7)
    yield "one", np.array([3.5])
    yield "two", np.array([1.0, -1.0])
    for n in (4095, 4096, 4097, 100003, (1 << 20) + 7):
        yield f"normal{n}", rng.normal(size=n) * 10.0 ** rng.integers(-5, 5, n)
    d = np.repeat(rng.uniform(-1, 1, 1000), 57)
    yield "duplicates", rng.permutation(d)
    z = np.zeros(30000)
    z[rng.random(30000) < 0.5] = -0.0
    z[::7] = 1e-310  # subnormals
    z[::11] = -5e-324
    yield "zeros_subnormal", z
    yield "huge", rng.choice([-1.7e308, 1.7e308, 0.0, 1.0, -1.0, 2.2e-308], 50000)
    yield "sorted", np.sort(rng.uniform(0, 1, 200000))
    yield "reversed", np.sort(rng.uniform(0, 1, 200000))[::-1].copy()


@pytest.mark.parametrize("name,v", list(_cases()), ids=lambda x: x if isinstance(x, str) else "")
def test_stable_sort_matches_numpy(name, v):
    from paper_1710_05781_b200.charges import sort_stable

    dv = torch.from_numpy(v).cuda()
    pay = torch.from_numpy(np.arange(len(v), dtype=np.float64) * 0.5).cuda()
    s, perm, p = sort_stable(dv, pay)
    want = np.argsort(v, kind="stable")
    np.testing.assert_array_equal(perm.cpu().numpy(), want)
    got = s.cpu().numpy()
    assert np.array_equal(got.view(np.uint64), v[want].view(np.uint64))  # exact bits
    np.testing.assert_array_equal(p.cpu().numpy(), want * 0.5)


def test_from_particles_unsorted_matches_oracle():
    import paper_1710_05781_b200 as dt
    from oracle import oracle as O  # noqa: F401  (the oracle's sort is numpy's)

    rng = np.random.default_rng(3)
    x = np.round(rng.uniform(-1, 1, 300000), 4)  # many exact duplicates
    q = rng.normal(size=len(x))
    s = dt.from_particles(np.column_stack([x, q]))
    order = np.argsort(x, kind="stable")
    np.testing.assert_array_equal(s.xs.cpu().numpy(), x[order])
    np.testing.assert_array_equal(s.qs.cpu().numpy(), q[order])


def test_permute_round_trip():
    from paper_1710_05781_b200.charges import permute

    rng = np.random.default_rng(5)
    v = torch.from_numpy(rng.normal(size=12345)).cuda()
    perm = torch.from_numpy(rng.permutation(12345)).cuda()
    g = permute(v, perm)
    np.testing.assert_array_equal(g.cpu().numpy(), v.cpu().numpy()[perm.cpu().numpy()])
    back = permute(g, perm, scatter=True)
    assert torch.equal(back, v)
