"""Charge assembly on the device (SURVEY.md §8(f) "next" #2) against golden
fixtures made by the live reference (tests/golden/make_assembly.py):
from_density and with_images positions and strengths bit for bit."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

torch = pytest.importorskip("torch")


def _golden():
    with np.load(os.path.join(GOLDEN, "assembly.npz")) as z:
        return {k: z[k] for k in z.files}


def test_assembly_fixture_is_consistent():
    g = _golden()
    for name in g["density_cases"]:
        a, b, cells, order, _ = g[f"{name}_spec"]
        xs = g[f"{name}_xs"]
        assert len(xs) == int(cells) * int(order)
        assert np.all(np.diff(xs) >= 0) and a < xs[0] and xs[-1] < b
    for name in g["image_cases"]:
        assert np.all(np.diff(g[f"{name}_xs"]) >= 0)


@pytest.fixture(scope="module")
def dt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1710_05781_b200 as pkg

    return pkg


@pytest.mark.gpu
def test_from_density_bit_identical(dt):
    g = _golden()
    for name in g["density_cases"]:
        a, b, cells, order, eps0 = g[f"{name}_spec"]
        spec = dt.DensitySpec(domain=(a, b), cells=int(cells), values=g[f"{name}_values"],
                              quadrature_order=int(order), eps0=eps0)
        s = dt.from_density(spec)
        np.testing.assert_array_equal(s.xs.cpu().numpy(), g[f"{name}_xs"], err_msg=str(name))
        np.testing.assert_array_equal(s.qs.cpu().numpy(), g[f"{name}_qs"], err_msg=str(name))


@pytest.mark.gpu
def test_with_images_bit_identical(dt):
    g = _golden()
    system = dt.from_particles(g["images_pairs"])
    for name in g["image_cases"]:
        gap, lower, rl, ru = g[f"{name}_spec"]
        spec = dt.ImageSpec(gap_length=gap, lower_electrode=lower, reflect_lower=bool(rl),
                            reflect_upper=bool(ru))
        s = dt.with_images(system, spec)
        np.testing.assert_array_equal(s.xs.cpu().numpy(), g[f"{name}_xs"], err_msg=str(name))
        np.testing.assert_array_equal(s.qs.cpu().numpy(), g[f"{name}_qs"], err_msg=str(name))


@pytest.mark.gpu
def test_assembly_reference_hand_cases(dt):
    """test_charges.py:87-182 cases."""
    import math

    eps0 = 8.8541878128e-12
    s = dt.from_density(dt.DensitySpec(domain=(0.0, 1.0), cells=4, values=[2.0 * eps0] * 4,
                                       quadrature_order=3))
    assert len(s) == 12 and s.total == pytest.approx(1.0, rel=1e-12)
    s = dt.from_density(dt.DensitySpec(domain=(0.0, 1.0), cells=1, values=[1.0],
                                       quadrature_order=2, eps0=0.5))
    r3 = 1.0 / (2.0 * math.sqrt(3.0))
    np.testing.assert_allclose(s.xs.cpu().numpy(), [0.5 - r3, 0.5 + r3], rtol=1e-14)
    with pytest.raises(ValueError):
        dt.DensitySpec(domain=(1.0, 0.0), cells=1, values=[1.0], quadrature_order=2)
    with pytest.raises(ValueError):
        dt.DensitySpec(domain=(0.0, 1.0), cells=3, values=[1.0], quadrature_order=2)
    with pytest.raises(ValueError):
        dt.from_density(dt.DensitySpec(domain=(0.0, 1.0), cells=1, values=[1.0],
                                       quadrature_order=17))
    base = dt.from_particles([(0.3, 1.0), (0.9, 2.0)])
    im = dt.with_images(base, dt.ImageSpec(gap_length=1.0))
    np.testing.assert_allclose(im.xs.cpu().numpy(), [-0.9, -0.3, 0.3, 0.9, 1.1, 1.7])
    np.testing.assert_allclose(im.qs.cpu().numpy(), [-2.0, -1.0, 1.0, 2.0, -2.0, -1.0])
    assert len(dt.with_images(dt.from_particles([(1.0, 1.0)]),
                              dt.ImageSpec(gap_length=1.0, reflect_upper=False))) == 1
    on_plane = dt.with_images(dt.from_particles([(0.0, 1.0)]),
                              dt.ImageSpec(gap_length=1.0, reflect_upper=False))
    assert len(on_plane) == 2 and on_plane.total == 0.0
    with pytest.raises(ValueError):
        dt.ImageSpec(gap_length=0.0)
