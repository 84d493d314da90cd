"""Generate golden fixtures from the LIVE reference (`disctree`).

Run in the build container only (the reference is not present on the GPU
box):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py

It imports the reference from /root/reference/pkg/src, runs its own public
API (from_particles, build, evaluate_all, evaluate_direct, sign_term_all)
on seeded instances and writes compressed .npz fixtures next to this file.
The adaptive truncation orders chosen by the compiled kernel
(_kernels.tree_phi_sum, lines 212-231) are extracted through the kernel
itself: a one-node tree whose moment row is m_k = 1/Phi^(k)(c, y) makes the
far-field sum equal p_use + 1.
"""

from __future__ import annotations

import os
import platform
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import disctree as dt  # noqa: E402
from disctree import _kernels  # noqa: E402

from paper_1710_05781_b200 import workloads as W  # noqa: E402

NODE_FIELDS = ("lo", "hi", "center", "half", "level", "start", "end", "left", "right")


def _meta() -> dict:
    import numba

    cpu = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    cpu = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {
        "numpy": np.__version__,
        "numba": numba.__version__,
        "python": platform.python_version(),
        "cpu": cpu,
    }


def tree_case(name, pairs, r_d, config: dt.EvalConfig, targets, direct=True):
    system = dt.from_particles(pairs)
    kernel = dt.DiscKernel(r_d)
    tree = dt.build(system, kernel, config)
    res = dt.evaluate_all(tree, kernel, config, system, targets, threads=1)
    out = {
        "xs": system.xs,
        "qs": system.qs,
        "prefix": system.prefix,
        "total": np.float64(system.total),
        "targets": np.asarray(targets, dtype=np.float64),
        "r_d": np.float64(r_d),
        "p": np.int64(config.p),
        "theta": np.float64(config.theta),
        "leaf_capacity": np.int64(config.leaf_capacity),
        "adaptive": np.bool_(config.adaptive),
        "tolerance": np.float64(config.tolerance),
        "depth": np.int64(tree.depth),
        "leaf_count": np.int64(tree.leaf_count),
        "moment_order": np.int64(tree.moment_order),
        "moments": tree.moments,
        "E_tree": res.values,
        "sign": dt.charges._sign_terms(system, np.asarray(targets, dtype=np.float64)),
    }
    for f in NODE_FIELDS:
        out[f] = getattr(tree, f)
    # kernel-sum parts straight from the reference's numba seams (the e term
    # is compared separately: it rests on the sequential np.cumsum)
    t = np.ascontiguousarray(targets, dtype=np.float64)
    rd2 = kernel.r_d * kernel.r_d
    if len(t):
        angles = np.linspace(0.0, 2.0 * np.pi, 64, endpoint=False)
        phi = np.empty_like(t)
        _kernels.tree_phi_sum(
            tree.center, tree.half, tree.start, tree.end, tree.left, tree.right, tree.moments,
            tree.system.xs, tree.system.qs, rd2, config.theta, config.p, config.adaptive,
            config.tolerance / (3.0 * max(tree.depth, 1)), tree.moment_order, np.cos(angles),
            np.sin(angles), t, phi, 0, len(t),
        )
        out["phi_tree"] = phi
        if direct:
            plain = np.empty_like(t)
            _kernels.phi_sum_plain(system.xs, system.qs, t, rd2, plain, 0, len(t))
            kahan = np.empty_like(t)
            _kernels.phi_sum_kahan(system.xs, system.qs, t, rd2, kahan, 0, len(t))
            out["phi_plain"] = plain
            out["phi_kahan"] = kahan
    if direct:
        out["E_direct"] = dt.evaluate_direct(system, kernel, targets, threads=1).values
        out["E_kahan"] = dt.evaluate_direct(system, kernel, targets, compensated=True).values
    np.savez_compressed(os.path.join(HERE, f"tree_{name}.npz"), **out)
    print(f"{name}: N={len(system)} nodes={len(tree)} depth={tree.depth} T={len(targets)}")


def p_use_from_kernel(c, h, y, rd, theta, tol_share, p_cap, cos_tab, sin_tab) -> int:
    """Run the compiled tree_phi_sum on a one-node tree and decode p_use."""
    kernel = dt.DiscKernel(rd)
    derivs = dt.phi_derivatives(kernel, c, y, p_cap)
    if not np.all(np.isfinite(1.0 / derivs)) or np.any(derivs == 0.0):
        return -1
    moments = (1.0 / derivs)[None, :].copy()
    out = np.empty(1)
    _kernels.tree_phi_sum(
        np.array([c]), np.array([h]), np.array([0], np.int64), np.array([1], np.int64),
        np.array([-1], np.int64), np.array([-1], np.int64), moments,
        np.array([0.0]), np.array([0.0]), rd * rd, theta, 0, True, tol_share, p_cap,
        cos_tab, sin_tab, np.array([y]), out, 0, 1,
    )
    v = out[0] - 1.0
    k = int(round(v))
    if abs(v - k) > 1e-6:
        return -1
    return k


def pchoice_case():
    rng = np.random.default_rng(2024)
    angles = np.linspace(0.0, 2.0 * np.pi, 64, endpoint=False)
    cos_tab, sin_tab = np.cos(angles), np.sin(angles)
    rows = []
    for rd in (0.1, 0.01, 0.005, 1e-4):
        for tol in (1e-6, 1e-8 / 30.0, 1e-10 / 42.0, 1e-10 / 84.0, 1e-12 / 63.0):
            n = 400
            big_r = 10.0 ** rng.uniform(-8.0, 0.5, n)
            ratio = rng.uniform(0.0, 0.995, n)
            ratio[:20] = 1.0 / 3.0
            sign = rng.choice([-1.0, 1.0], n)
            centers = rng.uniform(-1.0, 1.0, n)
            for c, R, q, sg in zip(centers, big_r, ratio, sign):
                h = q * R
                y = c - sg * R
                Rk = abs(c - y)
                if not Rk > 0.0 or h > 0.999 * Rk:
                    continue
                pu = p_use_from_kernel(c, h, y, rd, 0.999, tol, 30, cos_tab, sin_tab)
                if pu < 0:
                    continue
                rows.append((Rk, h, rd * rd, tol, 30, pu))
    arr = np.array(rows)
    np.savez_compressed(
        os.path.join(HERE, "pchoice.npz"),
        big_r=arr[:, 0], h=arr[:, 1], rd2=arr[:, 2], tol=arr[:, 3],
        p_cap=arr[:, 4].astype(np.int64), p_use=arr[:, 5].astype(np.int64),
    )
    print(f"pchoice: {len(arr)} samples, p range {arr[:, 5].min():.0f}..{arr[:, 5].max():.0f}")


def main():
    _kernels.warm_up()
    # configs[0]: N=16384 uniform GL, fixed p=8, leaf 64, r_d=0.01
    w = W.cfg0()
    tree_case("cfg0", np.column_stack([w.xs, w.qs]), w.r_d,
              dt.EvalConfig(p=8, leaf_capacity=64), w.targets)
    # configs[1] scaled to N=16384: adaptive tol 1e-10
    tree_case("cfg1s", np.column_stack([w.xs, w.qs]), w.r_d,
              dt.EvalConfig(p=8, leaf_capacity=64, adaptive=True, tolerance=1e-10),
              w.targets, direct=False)
    # configs[2] scaled to N=16384: graded streamer mesh, r_d=0.005, adaptive
    x, q, _ = W.graded_streamer(4096)
    tree_case("cfg2s", np.column_stack([x, q]), 0.005,
              dt.EvalConfig(p=8, leaf_capacity=64, adaptive=True, tolerance=1e-10), x)
    # configs[3] flavour: separate sorted random targets, r_d=1e-4, tol 1e-12
    x, q = W.uniform_gaussian(2048)
    t = np.sort(np.random.default_rng(1).uniform(0.0, 1.0, 4096))
    tree_case("cfg3s", np.column_stack([x, q]), 1e-4,
              dt.EvalConfig(p=8, leaf_capacity=64, adaptive=True, tolerance=1e-12), t)
    # reference test shapes (test_tree.py): random instances, unsorted targets
    tree_case("rand_default", W.random_instance(2000, 16), 0.1, dt.EvalConfig(),
              W.random_instance(2000, 16)[:, 0])
    tree_case("rand_adaptive", W.random_instance(800, 11), 0.1,
              dt.EvalConfig(adaptive=True, tolerance=1e-10, leaf_capacity=10),
              np.random.default_rng(7).uniform(-0.2, 1.2, 300))
    tree_case("rand_p20", W.random_instance(3000, 17), 0.1, dt.EvalConfig(p=20),
              W.random_instance(3000, 17)[:, 0])
    # duplicates (test_charges.py:189-196 style) and coincident points
    rng = np.random.default_rng(5)
    xd = np.round(rng.uniform(0, 1, 600), 2)
    qd = rng.uniform(-1, 1, 600)
    td = np.concatenate([rng.uniform(0, 1, 50), xd[:40]])
    tree_case("duplicates", np.column_stack([xd, qd]), 0.05,
              dt.EvalConfig(p=12, leaf_capacity=4), td)
    tree_case("coincident", [(0.5, 1.0)] * 10 + [(0.25, -2.0), (0.75, 3.0)], 0.1,
              dt.EvalConfig(p=6, leaf_capacity=2), np.array([0.1, 0.25, 0.5, 0.6, 0.75, 2.0]))
    tree_case("leafcap1", W.random_instance(300, 3), 0.1, dt.EvalConfig(p=10, leaf_capacity=1),
              W.random_instance(300, 3)[:, 0])
    tree_case("single", [(0.2, 1.0)], 0.1, dt.EvalConfig(), np.array([0.9, 0.2, -1.0]))
    tree_case("shifted", np.column_stack([np.linspace(1e3, 1e3 + 1.0, 700),
                                          np.random.default_rng(9).uniform(-1, 1, 700)]),
              0.02, dt.EvalConfig(p=9, leaf_capacity=16, adaptive=True, tolerance=1e-9),
              np.linspace(1e3 - 0.5, 1e3 + 1.5, 257))
    pchoice_case()
    np.savez(os.path.join(HERE, "meta.npz"), **{k: np.str_(v) for k, v in _meta().items()})


if __name__ == "__main__":
    main()
