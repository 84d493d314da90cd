"""Pin the CPU oracle (oracle/) against the live reference's fixtures.

The fixtures in tests/golden/ were produced by the reference itself
(tests/golden/make_golden.py).  These tests run without a GPU.
"""

import numpy as np
import pytest

from conftest import TREE_CASES, load_case
from oracle import oracle as O

# /root/reference/pkg/tests/test_kernel.py:22-46 (50-digit frozen values)
PHI_03_07_RD01 = -0.97014250014533189408
DERIVS_RD01_XC0_Y1 = [
    -0.99503719020998913567, 0.0098518533684157340165, 0.029262930797274457475,
    0.11560306324863869834, 0.56942375877452992929, 3.3571959210308800877,
    23.032658337377190754, 180.12148628695314528, 1580.4501921883089336,
]
DERIVS_RD13_XC04_YM08 = [
    0.67828010273306578454, 0.30518992907850936525, -0.35101717082512259262,
    0.3803620567780215527, -0.12361147295028763635, -1.3963025379575772582,
    6.8363798248712214313, -18.459085124433179007, 1.3154315162870905525,
]


@pytest.mark.parametrize("name", TREE_CASES)
def test_structure_bit_exact(name):
    g = load_case(name)
    t = O.build_structure(g["xs"], int(g["leaf_capacity"]))
    for f in O.NODE_FIELDS:
        np.testing.assert_array_equal(getattr(t, f), g[f], err_msg=f)
    assert t.depth == int(g["depth"])
    assert t.leaf_count == int(g["leaf_count"])


def moment_scale(g) -> np.ndarray:
    """sum|q| r^k / k! per node: the natural size of m_k."""
    from math import factorial

    order = int(g["moment_order"])
    absq = np.abs(g["qs"])
    node_q = np.array([absq[s:e].sum() for s, e in zip(g["start"], g["end"])])
    # cluster radius: max |x_j - c| (can exceed the half-width by rounding
    # on intervals a few ulps wide)
    h = np.array([
        max(hh, float(np.max(np.abs(g["xs"][s:e] - c)))) if e > s else hh
        for s, e, c, hh in zip(g["start"], g["end"], g["center"], g["half"])
    ])
    k = np.arange(order + 1)
    fact = np.array([float(factorial(int(i))) for i in k])
    return node_q[:, None] * h[:, None] ** k[None, :] / fact[None, :]


@pytest.mark.parametrize("name", TREE_CASES)
def test_moments(name):
    g = load_case(name)
    t = O.build_structure(g["xs"], int(g["leaf_capacity"]))
    m = O.moments(g["xs"], g["qs"], t, int(g["moment_order"]))
    scale = moment_scale(g)
    assert np.all(np.abs(m - g["moments"]) <= 1e-13 * scale + 1e-300)


@pytest.mark.parametrize("name", TREE_CASES)
def test_sign_terms_bit_exact(name):
    g = load_case(name)
    pre = O.prefix(g["qs"])
    np.testing.assert_array_equal(pre, g["prefix"])
    e = O.sign_terms(g["xs"], pre, float(pre[-1]), g["targets"])
    np.testing.assert_array_equal(e, g["sign"])


@pytest.mark.parametrize("name", TREE_CASES)
def test_tree_field(name):
    g = load_case(name)
    E, _ = O.evaluate_tree(
        g["xs"], g["qs"], float(g["r_d"]), int(g["p"]), float(g["theta"]),
        int(g["leaf_capacity"]), bool(g["adaptive"]), float(g["tolerance"]), g["targets"],
    )
    scale = np.abs(g["qs"]).sum()
    assert np.max(np.abs(E - g["E_tree"])) <= 1e-13 * scale


@pytest.mark.parametrize("name", [n for n in TREE_CASES if "phi_tree" in load_case(n)])
def test_tree_phi_seam(name):
    """Oracle kernel-sum part vs the reference's tree_phi_sum output."""
    g = load_case(name)
    tree = O.build(g["xs"], g["qs"], int(g["p"]), int(g["leaf_capacity"]), bool(g["adaptive"]))
    phi = O.tree_phi_sum(tree, g["xs"], g["qs"], float(g["r_d"]) ** 2, float(g["theta"]),
                         int(g["p"]), bool(g["adaptive"]),
                         O.tol_share(float(g["tolerance"]), tree.depth), g["targets"])
    scale = np.abs(g["qs"]).sum()
    assert np.max(np.abs(phi - g["phi_tree"])) <= 1e-13 * scale
    if "phi_kahan" in g:
        rd2 = float(g["r_d"]) ** 2
        np.testing.assert_array_equal(O.phi_sum_kahan(g["xs"], g["qs"], g["targets"], rd2),
                                      g["phi_kahan"])
        plain = O.phi_sum_plain(g["xs"], g["qs"], g["targets"], rd2)
        assert np.max(np.abs(plain - g["phi_plain"])) <= 1e-13 * scale


@pytest.mark.parametrize("name", [n for n in TREE_CASES if "E_direct" in load_case(n)])
def test_direct_field(name):
    g = load_case(name)
    scale = np.abs(g["qs"]).sum()
    E = O.evaluate_direct(g["xs"], g["qs"], float(g["r_d"]), g["targets"])
    assert np.max(np.abs(E - g["E_direct"])) <= 1e-13 * scale
    K = O.evaluate_direct(g["xs"], g["qs"], float(g["r_d"]), g["targets"], compensated=True)
    np.testing.assert_array_equal(K, g["E_kahan"])


def test_pchoice_bit_exact():
    import os

    from conftest import GOLDEN

    with np.load(os.path.join(GOLDEN, "pchoice.npz")) as z:
        R, h, rd2, tol, cap, want = (z[k] for k in ("big_r", "h", "rd2", "tol", "p_cap", "p_use"))
    got = np.array([
        O.choose_p(float(a), float(b), float(c), float(d), int(e))
        for a, b, c, d, e in zip(R, h, rd2, tol, cap)
    ])
    mismatch = np.nonzero(got != want)[0]
    assert len(mismatch) == 0, f"{len(mismatch)} mismatches, first {mismatch[:5]}"
    assert len(np.unique(want)) > 20


def test_derivative_golden_vectors():
    d = O.phi_derivatives(0.0 - 1.0, 0.1 * 0.1, 8)
    np.testing.assert_allclose(d, DERIVS_RD01_XC0_Y1, rtol=5e-13)
    d = O.phi_derivatives(0.4 - (-0.8), 1.3 * 1.3, 8)
    np.testing.assert_allclose(d, DERIVS_RD13_XC04_YM08, rtol=5e-13)
    assert O.phi_derivatives(0.3 - 0.7, 0.01, 0)[0] == pytest.approx(PHI_03_07_RD01, rel=1e-15)


def test_interaction_stats_consistent():
    g = load_case("cfg1s")
    E, tree, st = O.evaluate_tree(
        g["xs"], g["qs"], float(g["r_d"]), int(g["p"]), float(g["theta"]),
        int(g["leaf_capacity"]), True, float(g["tolerance"]), g["targets"], instrument=True,
    )
    # every source is reached exactly once per target: near pairs + far-covered sources
    assert np.all(st.near_pairs > 0)
    assert np.all(st.n_far > 0)
    assert np.all(st.sum_p <= 30 * st.n_far)
    assert np.all(st.flops() > 0)
    # deterministic hashes
    _, _, st2 = O.evaluate_tree(
        g["xs"], g["qs"], float(g["r_d"]), int(g["p"]), float(g["theta"]),
        int(g["leaf_capacity"]), True, float(g["tolerance"]), g["targets"], tree=tree,
        instrument=True,
    )
    np.testing.assert_array_equal(st.hash, st2.hash)
