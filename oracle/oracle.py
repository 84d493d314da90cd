"""ctypes front end of the CPU oracle (oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py (cpu_baseline leg and ``--impl reference``), never by the product
package.  Each wrapper names the reference routine it restates.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int64)
_U = C.POINTER(C.c_uint64)

MAX_DEPTH = 60  # tree.py:32
CONTOUR_SAMPLES = 64  # kernel.py:18
P_MAX = 30  # kernel.py:19


class _Tree(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int64),
        ("capacity", C.c_int64),
        ("lo", _D),
        ("hi", _D),
        ("center", _D),
        ("half", _D),
        ("level", _I),
        ("start", _I),
        ("end", _I),
        ("left", _I),
        ("right", _I),
        ("depth", C.c_int64),
        ("leaf_count", C.c_int64),
    ]


def build_library() -> str:
    """Compile liboracle.so with oracle/Makefile (no-op when up to date)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build_library()
        L = C.CDLL(_SO)
        L.or_prefix.argtypes = [_D, C.c_int64, _D]
        L.or_sign_terms.argtypes = [_D, _D, C.c_double, C.c_int64, _D, C.c_int64, _D]
        L.or_build.argtypes = [_D, C.c_int64, C.c_int64, C.c_int64, C.POINTER(_Tree)]
        L.or_build.restype = C.c_int
        L.or_tree_free.argtypes = [C.POINTER(_Tree)]
        L.or_moments.argtypes = [_D, _D, C.c_int64, _D, _I, _I, C.c_int64, _D]
        L.or_moments_cascade.argtypes = L.or_moments.argtypes
        L.or_adaptive_value.argtypes = [C.c_double, C.c_double, C.c_double, _D, _D, C.c_int64, _D]
        L.or_adaptive_value.restype = C.c_double
        L.or_choose_p.argtypes = [
            C.c_double, C.c_double, C.c_double, C.c_double, C.c_int64, _D, _D, C.c_int64,
        ]
        L.or_choose_p.restype = C.c_int64
        L.or_phi_derivatives.argtypes = [C.c_double, C.c_double, C.c_int64, _D]
        L.or_tree_phi_sum.argtypes = [
            _D, _D, _I, _I, _I, _I, _D, C.c_int64, _D, _D, C.c_double, C.c_double, C.c_int64,
            C.c_int, C.c_double, C.c_int64, _D, _D, C.c_int64, _D, _D, C.c_int64, C.c_int64,
            _U, _I, _I, _I, _I,
        ]
        L.or_phi_sum_plain.argtypes = [_D, _D, C.c_int64, _D, C.c_double, _D, C.c_int64, C.c_int64]
        L.or_phi_sum_kahan.argtypes = L.or_phi_sum_plain.argtypes
        L.or_num_threads.restype = C.c_int
        L.or_set_num_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def _d(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _i(a: np.ndarray):
    return a.ctypes.data_as(_I)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def set_threads(n: int) -> None:
    lib().or_set_num_threads(int(n))


def num_threads() -> int:
    return int(lib().or_num_threads())


# ---------------------------------------------------------------- (a)
def prefix(qs) -> np.ndarray:
    """charges.py:130 (sequential cumsum)."""
    qs = _f64(qs)
    out = np.empty_like(qs)
    lib().or_prefix(_d(qs), len(qs), _d(out))
    return out


def sign_terms(xs, pre, total: float, ys) -> np.ndarray:
    """charges.py:183-187."""
    xs, pre, ys = _f64(xs), _f64(pre), _f64(ys)
    out = np.empty_like(ys)
    lib().or_sign_terms(_d(xs), _d(pre), float(total), len(xs), _d(ys), len(ys), _d(out))
    return out


# ---------------------------------------------------------------- (b) + (c)
@dataclass
class OracleTree:
    lo: np.ndarray
    hi: np.ndarray
    center: np.ndarray
    half: np.ndarray
    level: np.ndarray
    start: np.ndarray
    end: np.ndarray
    left: np.ndarray
    right: np.ndarray
    depth: int
    leaf_count: int
    moments: np.ndarray | None = None
    moment_order: int = -1

    def __len__(self) -> int:
        return len(self.lo)


NODE_FIELDS = ("lo", "hi", "center", "half", "level", "start", "end", "left", "right")


def build_structure(xs, leaf_capacity: int, max_depth: int = MAX_DEPTH) -> OracleTree:
    """tree.py:156-222 (bit-exact node arrays, depth, leaf_count)."""
    xs = _f64(xs)
    t = _Tree()
    rc = lib().or_build(_d(xs), len(xs), int(leaf_capacity), int(max_depth), C.byref(t))
    if rc == -2:
        raise ValueError("cannot build a tree over an empty charge system")
    if rc != 0:
        raise MemoryError("oracle build failed")
    n = t.n_nodes
    try:
        arrs = {}
        for f in NODE_FIELDS:
            ptr = getattr(t, f)
            dt = np.float64 if f in ("lo", "hi", "center", "half") else np.int64
            arrs[f] = np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt, copy=True)
        return OracleTree(depth=int(t.depth), leaf_count=int(t.leaf_count), **arrs)
    finally:
        lib().or_tree_free(C.byref(t))


def moments(xs, qs, tree: OracleTree, order: int) -> np.ndarray:
    """tree.py:224-238 (direct per-node moments)."""
    xs, qs = _f64(xs), _f64(qs)
    out = np.empty((len(tree), order + 1))
    lib().or_moments(
        _d(xs), _d(qs), len(tree), _d(tree.center), _i(tree.start), _i(tree.end), int(order),
        _d(out),
    )
    return out


def moments_cascade(xs, qs, tree: OracleTree, order: int) -> np.ndarray:
    """The reference's per-source terms (tree.py:235-237) with cascade
    summation: a more accurate yardstick than its sequential sums."""
    xs, qs = _f64(xs), _f64(qs)
    out = np.empty((len(tree), order + 1))
    lib().or_moments_cascade(
        _d(xs), _d(qs), len(tree), _d(tree.center), _i(tree.start), _i(tree.end), int(order),
        _d(out),
    )
    return out


def moment_order(p: int, adaptive: bool) -> int:
    """tree.py:224-226."""
    return max(p, P_MAX) if adaptive else p


def build(xs, qs, p: int, leaf_capacity: int, adaptive: bool) -> OracleTree:
    tree = build_structure(xs, leaf_capacity)
    tree.moment_order = moment_order(p, adaptive)
    tree.moments = moments(xs, qs, tree, tree.moment_order)
    return tree


# ---------------------------------------------------------------- (d) + (e)
def contour_tables(samples: int = CONTOUR_SAMPLES):
    """tree.py:342: host numpy cos/sin of linspace(0, 2pi, 64, endpoint=False)."""
    angles = np.linspace(0.0, 2.0 * np.pi, samples, endpoint=False)
    return np.cos(angles), np.sin(angles)


def tol_share(tolerance: float, depth: int) -> float:
    """tree.py:268-270."""
    return tolerance / (3.0 * max(depth, 1))


def adaptive_value(big_r: float, h: float, rd2: float) -> tuple[float, float]:
    c, s = contour_tables()
    m = C.c_double()
    v = lib().or_adaptive_value(big_r, h, rd2, _d(c), _d(s), len(c), C.byref(m))
    return float(v), float(m.value)


def choose_p(big_r: float, h: float, rd2: float, tol: float, p_cap: int) -> int:
    """_kernels.py:212-231 (bit-exact replica of the compiled decision)."""
    c, s = contour_tables()
    return int(lib().or_choose_p(big_r, h, rd2, tol, int(p_cap), _d(c), _d(s), len(c)))


def phi_derivatives(d: float, rd2: float, p: int) -> np.ndarray:
    out = np.empty(p + 1)
    lib().or_phi_derivatives(float(d), float(rd2), int(p), _d(out))
    return out


@dataclass
class TraversalStats:
    hash: np.ndarray
    near_pairs: np.ndarray
    n_far: np.ndarray
    sum_p: np.ndarray
    n_p0: np.ndarray

    def flops(self) -> np.ndarray:
        """W(y) = 14*near_pairs + sum_far F_far(p),
        F_far(p) = 20 + 11p (p >= 1), 14 (p = 0)."""
        return (
            14 * self.near_pairs
            + 20 * (self.n_far - self.n_p0)
            + 11 * self.sum_p
            + 14 * self.n_p0
        )


def tree_phi_sum(tree: OracleTree, xs, qs, rd2: float, theta: float, p: int, adaptive: bool,
                 tol: float, ys, instrument: bool = False):
    """_kernels.py:163-266 over all targets; returns phi_part (and stats)."""
    xs, qs, ys = _f64(xs), _f64(qs), _f64(ys)
    c, s = contour_tables()
    out = np.empty_like(ys)
    T = len(ys)
    if instrument:
        st = TraversalStats(
            np.zeros(T, np.uint64), np.zeros(T, np.int64), np.zeros(T, np.int64),
            np.zeros(T, np.int64), np.zeros(T, np.int64),
        )
        ptrs = (
            st.hash.ctypes.data_as(_U), _i(st.near_pairs), _i(st.n_far), _i(st.sum_p),
            _i(st.n_p0),
        )
    else:
        st = None
        ptrs = (None, None, None, None, None)
    mom = np.ascontiguousarray(tree.moments)
    lib().or_tree_phi_sum(
        _d(tree.center), _d(tree.half), _i(tree.start), _i(tree.end), _i(tree.left),
        _i(tree.right), _d(mom), mom.shape[1], _d(xs), _d(qs), float(rd2), float(theta), int(p),
        int(bool(adaptive)), float(tol), int(tree.moment_order), _d(c), _d(s), len(c), _d(ys),
        _d(out), 0, T, *ptrs,
    )
    return (out, st) if instrument else out


# ---------------------------------------------------------------- (f)
def phi_sum_plain(xs, qs, ys, rd2: float) -> np.ndarray:
    """_kernels.py:49-59."""
    xs, qs, ys = _f64(xs), _f64(qs), _f64(ys)
    out = np.empty_like(ys)
    lib().or_phi_sum_plain(_d(xs), _d(qs), len(xs), _d(ys), float(rd2), _d(out), 0, len(ys))
    return out


def phi_sum_kahan(xs, qs, ys, rd2: float) -> np.ndarray:
    """_kernels.py:145-160."""
    xs, qs, ys = _f64(xs), _f64(qs), _f64(ys)
    out = np.empty_like(ys)
    lib().or_phi_sum_kahan(_d(xs), _d(qs), len(xs), _d(ys), float(rd2), _d(out), 0, len(ys))
    return out


# ---------------------------------------------------------------- end to end
def evaluate_tree(xs, qs, r_d: float, p: int, theta: float, leaf_capacity: int,
                  adaptive: bool, tolerance: float, ys, tree: OracleTree | None = None,
                  instrument: bool = False):
    """tree.py:318-373 on sorted sources: e term + tree_phi_sum."""
    xs, qs, ys = _f64(xs), _f64(qs), _f64(ys)
    if tree is None:
        tree = build(xs, qs, p, leaf_capacity, adaptive)
    pre = prefix(qs)
    total = float(pre[-1]) if len(pre) else 0.0
    e = sign_terms(xs, pre, total, ys)
    rd2 = r_d * r_d
    res = tree_phi_sum(tree, xs, qs, rd2, theta, p, adaptive, tol_share(tolerance, tree.depth),
                       ys, instrument)
    if instrument:
        phi, st = res
        return e + phi, tree, st
    return e + res, tree


def evaluate_direct(xs, qs, r_d: float, ys, compensated: bool = False) -> np.ndarray:
    """direct.py:52-88 (plain or Kahan kernel; no symmetric split)."""
    xs, qs, ys = _f64(xs), _f64(qs), _f64(ys)
    pre = prefix(qs)
    total = float(pre[-1]) if len(pre) else 0.0
    e = sign_terms(xs, pre, total, ys)
    fn = phi_sum_kahan if compensated else phi_sum_plain
    return e + fn(xs, qs, ys, r_d * r_d)
