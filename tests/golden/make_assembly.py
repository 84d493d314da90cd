"""Golden fixtures for device charge assembly, from the LIVE reference.

Run in the build container (the reference is absent on the GPU box):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_assembly.py

Calls disctree.from_density / with_images (charges.py:135-180) on seeded
specs and stores the inputs with the reference's xs and qs in
tests/golden/assembly.npz.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import disctree as dt  # noqa: E402


def main():
    rng = np.random.default_rng(31)
    out = {}
    eps0 = 8.8541878128e-12
    dens = [
        ("d_const", (0.0, 1.0), 4, [2.0 * eps0] * 4, 3, eps0),
        ("d_order2", (0.0, 1.0), 1, [1.0], 2, 0.5),
        ("d_linear", (0.0, 1.0), 5, list(np.linspace(0.0, 1.0, 6)), 2, 0.5),
        ("d_rand_cells", (-2.0, 3.0), 777, list(rng.normal(size=777)), 5, eps0),
        ("d_rand_edges", (-1.3, 2.9), 1001, list(rng.normal(size=1002)), 7, 8.854e-12),
        ("d_big", (-1.0, 1.0), 1 << 13, list(rng.uniform(0, 1e-3, (1 << 13) + 1)), 4, 8.854e-12),
    ]
    for order in range(1, 17):
        dens.append((f"d_o{order}", (0.1, 0.7), 13, list(rng.normal(size=14)), order, 1.0))
    names = []
    for name, dom, cells, values, order, e0 in dens:
        spec = dt.DensitySpec(domain=dom, cells=cells, values=values, quadrature_order=order,
                              eps0=e0)
        s = dt.from_density(spec)
        out[f"{name}_spec"] = np.array([dom[0], dom[1], cells, order, e0])
        out[f"{name}_values"] = np.asarray(values, dtype=np.float64)
        out[f"{name}_xs"] = s.xs
        out[f"{name}_qs"] = s.qs
        names.append(name)
    out["density_cases"] = np.array(names)
    pairs = np.column_stack([np.concatenate([rng.uniform(-0.5, 2.5, 600), [0.0, 1.0, 2.0]]),
                             rng.normal(size=603)])
    imgs = [
        ("i_both", 1.0, 0.0, True, True),
        ("i_lower", 1.0, 0.0, True, False),
        ("i_upper_offset", 1.0, 1.0, False, True),
        ("i_wide", 2.5, -0.25, True, True),
        ("i_narrow", 0.3, 0.2, True, True),
    ]
    names = []
    system = dt.from_particles(pairs)
    out["images_pairs"] = pairs
    for name, gap, lower, rl, ru in imgs:
        spec = dt.ImageSpec(gap_length=gap, lower_electrode=lower, reflect_lower=rl,
                            reflect_upper=ru)
        s = dt.with_images(system, spec)
        out[f"{name}_spec"] = np.array([gap, lower, float(rl), float(ru)])
        out[f"{name}_xs"] = s.xs
        out[f"{name}_qs"] = s.qs
        names.append(name)
    out["image_cases"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "assembly.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
