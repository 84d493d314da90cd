"""Binary source tree, node moments and tree field evaluation on the B200.

Mirror of disctree.tree (tree.py:35-373): EvalConfig, Tree, TreeNode, build,
well_separated, evaluate_point, evaluate_all with the reference's names,
argument meaning and errors.  build() runs stages (b) and (c) of the hot
path (csrc/dt_build.cu, csrc/dt_moments.cu); evaluate_all() runs (a) and
(d)+(e) (csrc/dt_scan.cu, csrc/dt_eval.cu).  Node arrays are CUDA tensors
in the reference's breadth-first layout and are bit-identical to it.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np

import torch

from . import _lib
from .charges import (ChargeSystem, _sign_terms, as_targets, check_values, host_targets,
                      permute, sort_stable)
from .direct import FieldResult
from .kernel import DEFAULT_CONTOUR_SAMPLES, DEFAULT_P_MAX, DiscKernel

MAX_DEPTH = 60  # tree.py:32


@dataclass(frozen=True)
class EvalConfig:
    """Truncation order, separation ratio, leaf size, adaptive tolerance
    (tree.py:35-59)."""

    p: int = 10
    theta: float = 1.0 / 3.0
    leaf_capacity: int = 40
    adaptive: bool = False
    tolerance: float = 1e-9

    def __post_init__(self) -> None:
        if self.p < 0:
            raise ValueError(f"p must be >= 0, got {self.p!r}")
        if not 0.0 < self.theta < 1.0:
            raise ValueError(f"theta must lie in (0, 1), got {self.theta!r}")
        if self.leaf_capacity < 1:
            raise ValueError(f"leaf_capacity must be >= 1, got {self.leaf_capacity!r}")
        if self.tolerance <= 0:
            raise ValueError(f"tolerance must be positive, got {self.tolerance!r}")


def moment_order_for(config: EvalConfig) -> int:
    """tree.py:224-226: p, raised to the adaptive cap when adaptive."""
    return max(config.p, DEFAULT_P_MAX) if config.adaptive else config.p


@dataclass
class Tree:
    """Breadth-first node arrays (CUDA tensors; child -1 = absent) and moments
    [nodes, moment_order + 1] (tree.py:62-99)."""

    system: ChargeSystem
    lo: torch.Tensor
    hi: torch.Tensor
    center: torch.Tensor
    half: torch.Tensor
    level: torch.Tensor
    start: torch.Tensor
    end: torch.Tensor
    left: torch.Tensor
    right: torch.Tensor
    moment_order: int
    depth: int
    leaf_count: int
    build_seconds: float  # given as (start, end) CUDA events, read when asked
    # device-side extras for the traversal kernel: meval holds the moments in
    # the traversal layout (dt_moments moments_eval), the only layout the
    # upward pass writes for moment order <= 31
    meval: torch.Tensor = field(repr=False, default=None)
    packed: torch.Tensor = field(repr=False, default=None)
    xq: torch.Tensor = field(repr=False, default=None)
    meta: torch.Tensor = field(repr=False, default=None)
    moments_ref: torch.Tensor | None = field(repr=False, default=None)

    def __getattribute__(self, name):
        if name == "build_seconds":
            v = object.__getattribute__(self, "build_seconds")
            if isinstance(v, tuple):  # events around the build on its stream
                v[1].synchronize()
                v = v[0].elapsed_time(v[1]) * 1e-3
                object.__setattr__(self, "build_seconds", v)
            return v
        return object.__getattribute__(self, name)

    def __len__(self) -> int:
        return int(self.lo.shape[0])

    @property
    def moments(self) -> torch.Tensor:
        """m_k = sum q (x - c)^k / k!, [nodes, moment_order + 1] (tree.py:224-238),
        derived from the traversal rows on first use (dt_moments_from_eval)."""
        if self.moments_ref is None:
            n, o1 = len(self), self.moment_order + 1
            out = torch.empty((n, o1), dtype=torch.float64, device=self.meval.device)
            _lib.check(_lib.load().dt_moments_from_eval(
                _lib.ptr(self.meval), self.meval.shape[1], n, self.moment_order,
                _lib.ptr(out), _lib.stream_handle()), "dt_moments_from_eval")
            self.moments_ref = out
        return self.moments_ref

    def node(self, index: int) -> "TreeNode":
        return TreeNode(self, index)

    @property
    def root(self) -> "TreeNode":
        return TreeNode(self, 0)

    @property
    def mean_leaf_occupancy(self) -> float:
        return len(self.system) / self.leaf_count

    def numpy(self) -> dict:
        """Host copies of the node arrays (reference dtypes)."""
        names = ("lo", "hi", "center", "half", "level", "start", "end", "left", "right",
                 "moments")
        return {k: getattr(self, k).cpu().numpy() for k in names}


@dataclass(frozen=True)
class TreeNode:
    """Read-only view of one node (tree.py:102-147)."""

    tree: Tree
    index: int

    @property
    def interval(self) -> tuple[float, float]:
        return (float(self.tree.lo[self.index]), float(self.tree.hi[self.index]))

    @property
    def center(self) -> float:
        return float(self.tree.center[self.index])

    @property
    def half_width(self) -> float:
        return float(self.tree.half[self.index])

    @property
    def level(self) -> int:
        return int(self.tree.level[self.index])

    @property
    def source_range(self) -> tuple[int, int]:
        return (int(self.tree.start[self.index]), int(self.tree.end[self.index]))

    @property
    def source_count(self) -> int:
        s, e = self.source_range
        return e - s

    @property
    def moments(self) -> np.ndarray:
        return self.tree.moments[self.index].cpu().numpy()

    @property
    def children(self) -> tuple["TreeNode", ...]:
        kids = []
        for c in (int(self.tree.left[self.index]), int(self.tree.right[self.index])):
            if c >= 0:
                kids.append(TreeNode(self.tree, c))
        return tuple(kids)

    @property
    def is_leaf(self) -> bool:
        return int(self.tree.left[self.index]) < 0 and int(self.tree.right[self.index]) < 0


def initial_node_capacity(n: int, leaf_capacity: int) -> int:
    return int(4 * (n // max(1, leaf_capacity) + 1) + 256)


class TreeBuffers:
    """Device buffers for one build at a fixed node capacity (reusable)."""

    F64 = ("lo", "hi", "center", "half")
    I64 = ("level", "start", "end", "left", "right")

    def __init__(self, n: int, capacity: int, device):
        self.n = n
        self.capacity = capacity
        for k in self.F64:
            setattr(self, k, torch.empty(capacity, dtype=torch.float64, device=device))
        for k in self.I64:
            setattr(self, k, torch.empty(capacity, dtype=torch.int64, device=device))
        self.packed = torch.empty(capacity * 32, dtype=torch.uint8, device=device)
        self.meta = _lib.zeros_i64(_lib.DT_META_WORDS, device)
        L = _lib.load()
        self.ws_bytes = int(L.dt_build_workspace(n, capacity))
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=device)
        self.mws_bytes = int(L.dt_moments_workspace(capacity))
        self.mws = torch.empty(self.mws_bytes, dtype=torch.uint8, device=device)

    def launch(self, xs: torch.Tensor, leaf_capacity: int, max_depth: int = MAX_DEPTH,
               p2m=None) -> None:
        """dt_build_tree; with p2m = (qs, order, meval, xq) the build's idle
        blocks also form the leaves of finished levels (dt_build_tree_p2m)."""
        L = _lib.load()
        p = _lib.ptr
        if p2m is not None:
            qs, order, meval, xq = p2m
            _lib.check(
                L.dt_build_tree_p2m(
                    p(xs), p(qs), self.n, int(leaf_capacity), int(max_depth), self.capacity,
                    p(self.lo), p(self.hi), p(self.center), p(self.half), p(self.level),
                    p(self.start), p(self.end), p(self.left), p(self.right), p(self.packed),
                    p(self.meta), int(order), p(meval), meval.shape[1], p(xq), p(self.ws),
                    self.ws_bytes, _lib.stream_handle(),
                ),
                "dt_build_tree_p2m",
            )
            return
        _lib.check(
            L.dt_build_tree(
                p(xs), self.n, int(leaf_capacity), int(max_depth), self.capacity, p(self.lo),
                p(self.hi), p(self.center), p(self.half), p(self.level), p(self.start),
                p(self.end), p(self.left), p(self.right), p(self.packed), p(self.meta),
                p(self.ws), self.ws_bytes, _lib.stream_handle(),
            ),
            "dt_build_tree",
        )


def eval_stride(order: int) -> int:
    """Row stride of the traversal moment layout (even, >= order + 1)."""
    return (order + 2) & ~1


def launch_moments(bufs: TreeBuffers, xs, qs, order: int, moments: torch.Tensor | None,
                   meval: torch.Tensor, xq: torch.Tensor | None = None) -> None:
    """dt_moments: traversal rows into meval; for order > 31 (or when given)
    the reference layout into moments as well; with xq, the interleaved
    (x, q) pairs too (dt_moments_pack: no separate pack pass)."""
    L = _lib.load()
    p = _lib.ptr
    if xq is not None:
        _lib.check(
            L.dt_moments_pack(p(xs), p(qs), xs.numel(), p(bufs.center), p(bufs.start),
                              p(bufs.end), p(bufs.left), p(bufs.right), p(bufs.meta),
                              int(order), p(moments), p(meval), eval_stride(order),
                              bufs.capacity, p(xq), p(bufs.mws), bufs.mws_bytes,
                              _lib.stream_handle()),
            "dt_moments_pack",
        )
        return
    _lib.check(
        L.dt_moments(p(xs), p(qs), p(bufs.center), p(bufs.start), p(bufs.end), p(bufs.left),
                     p(bufs.right), p(bufs.meta), int(order), p(moments), p(meval),
                     eval_stride(order), bufs.capacity, p(bufs.mws), bufs.mws_bytes,
                     _lib.stream_handle()),
        "dt_moments",
    )


def pack_sources(xs: torch.Tensor, qs: torch.Tensor, out: torch.Tensor | None = None):
    n = xs.numel()
    if out is None:
        out = torch.empty(2 * n, dtype=torch.float64, device=xs.device)
    if n:
        _lib.check(
            _lib.load().dt_pack_sources(_lib.ptr(xs), _lib.ptr(qs), n, _lib.ptr(out),
                                        _lib.stream_handle()),
            "dt_pack_sources",
        )
    return out


def build(system: ChargeSystem, kernel: DiscKernel, config: EvalConfig) -> Tree:
    """Build the tree and all node moments on the GPU (tree.py:156-257).

    Bit-identical node arrays, depth and leaf_count; moments agree with the
    reference to round-off.  ``kernel`` is unused, as in the reference.
    """
    if len(system) == 0:
        raise ValueError("cannot build a tree over an empty charge system")
    return _build(system, config, None)


def _build(system: ChargeSystem, config: EvalConfig, upward) -> Tree:
    """Structure + moments; ``upward(bufs, order, moments, meval)`` replaces
    the full upward pass when given (parallel.build_sharded).  For moment
    order <= 31 only the traversal rows are formed (moments is None); the
    reference layout is derived on first access of Tree.moments."""
    dev = _lib.require_device()
    # build time from events on the stream: the host does not wait for the
    # moments (Tree.build_seconds reads the events when asked)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    n = len(system)
    order = moment_order_for(config)
    # orders <= 31 on one device: the build's idle blocks start the leaves'
    # P2M (rows of up to capacity nodes; the tree keeps the first n_nodes)
    fused = upward is None and order + 1 <= 32
    xq = torch.empty(2 * n, dtype=torch.float64, device=dev)
    cap = initial_node_capacity(n, config.leaf_capacity)
    meta_h = torch.empty(8, dtype=torch.int64, pin_memory=True)
    while True:
        bufs = TreeBuffers(n, cap, dev)
        meval = (torch.empty((cap, eval_stride(order)), dtype=torch.float64, device=dev)
                 if fused else None)
        bufs.launch(system.xs, config.leaf_capacity,
                    p2m=(system.qs, order, meval, xq) if fused else None)
        # the host needs the node count; the fused path enqueues the moments
        # first (they read the count on the device and do nothing if the build
        # overflowed), so the GPU does not idle while the host reads it
        meta_h.copy_(bufs.meta[:8], non_blocking=True)
        counted = torch.cuda.Event()
        counted.record()
        if fused:  # moments and the traversal's (x, q) pairs in one pass
            launch_moments(bufs, system.xs, system.qs, order, None, meval, xq=xq)
        counted.synchronize()
        meta = meta_h.tolist()
        if not meta[_lib.DT_META_OVERFLOW]:
            break
        cap *= 4
    n_nodes = int(meta[_lib.DT_META_NODES])
    moments = (torch.empty((n_nodes, order + 1), dtype=torch.float64, device=dev)
               if order + 1 > 32 else None)
    if meval is None:
        meval = torch.empty((n_nodes, eval_stride(order)), dtype=torch.float64, device=dev)
    if upward is None and not fused:  # higher orders: both layouts, then the pairs
        launch_moments(bufs, system.xs, system.qs, order, moments, meval, xq=xq)
    elif upward is not None:
        upward(bufs, order, moments, meval)
        pack_sources(system.xs, system.qs, xq)
    ev1.record()
    return Tree(
        system=system,
        lo=bufs.lo[:n_nodes], hi=bufs.hi[:n_nodes], center=bufs.center[:n_nodes],
        half=bufs.half[:n_nodes], level=bufs.level[:n_nodes], start=bufs.start[:n_nodes],
        end=bufs.end[:n_nodes], left=bufs.left[:n_nodes], right=bufs.right[:n_nodes],
        moment_order=order, depth=int(meta[_lib.DT_META_DEPTH]),
        leaf_count=int(meta[_lib.DT_META_LEAVES]), build_seconds=(ev0, ev1),
        meval=meval[:n_nodes], packed=bufs.packed[: n_nodes * 32], xq=xq, meta=bufs.meta,
        moments_ref=moments,
    )


def well_separated(node: TreeNode, y: float, theta: float) -> bool:
    """half / |y - center| <= theta, false at distance 0 (tree.py:260-265)."""
    dist = abs(y - node.center)
    if dist == 0.0:
        return False
    return node.half_width <= theta * dist


def _tol_share(tree: Tree, config: EvalConfig) -> float:
    return config.tolerance / (3.0 * max(tree.depth, 1))  # tree.py:268-270


_TABLES: dict = {}


def contour_tables(device, samples: int = DEFAULT_CONTOUR_SAMPLES):
    """cos/sin of linspace(0, 2 pi, 64, endpoint=False) from host numpy
    (tree.py:342), cached on the device."""
    key = (str(device), samples)
    if key not in _TABLES:
        ang = np.linspace(0.0, 2.0 * np.pi, samples, endpoint=False)
        _TABLES[key] = (
            torch.from_numpy(np.cos(ang)).to(device),
            torch.from_numpy(np.sin(ang)).to(device),
        )
    return _TABLES[key]


def tree_phi_sum(tree: Tree, kernel: DiscKernel, config: EvalConfig, ys: torch.Tensor,
                 out: torch.Tensor, i0: int = 0, i1: int | None = None,
                 accumulate: bool = True, psel_mode: int = _lib.DT_PSEL_FAST,
                 stats: _lib.EvalStats | None = None,
                 workspace: torch.Tensor | None = None) -> None:
    """Stage (d)+(e) on device targets ys[i0:i1] (the _kernels.tree_phi_sum
    seam); out[i] (+)= phi(y_i)."""
    if i1 is None:
        i1 = ys.numel()
    if i1 <= i0:
        return
    cos_t, sin_t = contour_tables(ys.device)
    if workspace is None:
        workspace = _workspace(ys.device, _lib.DT_EVAL_COUNTER_BYTES)
    p = _lib.ptr
    _lib.check(
        _lib.load().dt_tree_phi_sum_packed(
            p(tree.packed), len(tree), p(tree.meval), tree.meval.shape[1], p(tree.xq),
            len(tree.system), kernel.r_d * kernel.r_d, float(config.theta), int(config.p),
            int(bool(config.adaptive)), _tol_share(tree, config), int(tree.moment_order),
            p(cos_t), p(sin_t), cos_t.numel(), p(ys), p(out), int(i0), int(i1),
            int(bool(accumulate)), int(psel_mode), C.byref(stats) if stats is not None else None,
            p(workspace), workspace.numel(), _lib.stream_handle(),
        ),
        "dt_tree_phi_sum_packed",
    )


def _check_order(tree: Tree, config: EvalConfig) -> None:
    if tree.moment_order < config.p:
        raise ValueError(
            f"tree was built with moment order {tree.moment_order}, "
            f"config.p = {config.p} requires at least that"
        )


def evaluate_point(tree: Tree, kernel: DiscKernel, config: EvalConfig, y: float) -> float:
    """Kernel-sum part of the field at one target (tree.py:273-315); the sign
    term is not included.  Runs the same GPU traversal as evaluate_all."""
    _check_order(tree, config)
    dev = _lib.require_device()
    ys = torch.tensor([float(y)], dtype=torch.float64, device=dev)
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    tree_phi_sum(tree, kernel, config, ys, out, accumulate=False)
    return float(out[0])


_WS = threading.local()


def _workspace(dev, nbytes: int) -> torch.Tensor:
    """A traversal workspace kept per thread and device: reusing it keeps the
    cached adaptive-order tables (their key lives in the slot) and skips an
    allocation per call.  Per thread, since a call owns it until it returns."""
    cache = getattr(_WS, "d", None)
    if cache is None:
        cache = _WS.d = {}
    key = str(dev)
    ws = cache.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = cache[key] = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    return ws


def _timing_events():
    """A start event recorded now on the current stream and its end event:
    evaluation times are taken on the device, so the host does not have to
    drain the stream before it starts enqueueing (no idle gap)."""
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    return ev0, ev1


def _elapsed(ev0, ev1) -> float:
    ev1.record()
    ev1.synchronize()
    return ev0.elapsed_time(ev1) * 1e-3


def evaluate_all(tree: Tree, kernel: DiscKernel, config: EvalConfig, system: ChargeSystem,
                 targets, threads: int | None = 1) -> FieldResult:
    """Field at every target: sign term + tree-accelerated kernel sum
    (tree.py:318-373).

    ``targets`` may be a numpy array / sequence (numpy values returned) or a
    torch tensor (returned on the same device).  Per-target results are
    bit-identical for any ``threads`` value and any target order; ``threads``
    is accepted for API compatibility (the GPU grid replaces the CPU pool).
    """
    _check_order(tree, config)
    host = host_targets(targets)
    if host is not None and host.numel() >= PIPELINE_MIN_TARGETS and _looks_sorted(host):
        numpy_out = not isinstance(targets, torch.Tensor)
        if host.is_pinned():
            return _evaluate_host_mapped(tree, kernel, config, system, host, numpy_out)
        return _evaluate_host_pipelined(tree, kernel, config, system, host, numpy_out)
    t, back = as_targets(targets)
    dev = t.device
    ev0, ev1 = _timing_events()
    values = _sign_terms(system, t)
    T = t.numel()
    if T:
        if T > 1 and check_values(t).tolist()[1]:
            # sorted targets traverse coherently; the field goes back in place
            ys, perm, vs = sort_stable(t, values)
            tree_phi_sum(tree, kernel, config, ys, vs)
            permute(vs, perm, scatter=True, out=values)
        else:
            tree_phi_sum(tree, kernel, config, t, values)
    elapsed = _elapsed(ev0, ev1)
    return FieldResult(values=back(values), build_time=tree.build_seconds, eval_time=elapsed,
                       method="tree")


# Host targets of at least this many points are streamed in chunks: the
# host->device copy of chunk i+1 and the device->host copy of chunk i-1
# overlap the sign term and traversal of chunk i (three CUDA streams).
PIPELINE_MIN_TARGETS = 1 << 20
PIPELINE_CHUNK = 1 << 21


def _looks_sorted(host: torch.Tensor) -> bool:
    """Cheap host-side guess (65 evenly spaced samples: each is a cache miss
    in a large pinned array, and the guess sits before the first launch) that
    the targets are ascending; unsorted targets take the sorting path.
    Results never depend on it: the traversal is exact in any order."""
    n = host.numel()
    s = host.numpy()[np.linspace(0, n - 1, min(n, 65)).astype(np.int64)]
    return bool((s[1:] >= s[:-1]).all())


def _evaluate_host_pipelined(tree: Tree, kernel: DiscKernel, config: EvalConfig,
                             system: ChargeSystem, host: torch.Tensor,
                             numpy_out: bool) -> FieldResult:
    dev = _lib.require_device()
    T = host.numel()
    src = host if host.is_pinned() else None
    out_h = torch.empty(T, dtype=torch.float64, pin_memory=True)
    d_t = torch.empty(T, dtype=torch.float64, device=dev)
    d_o = torch.empty(T, dtype=torch.float64, device=dev)
    flags = _lib.zeros_i64(2, dev)
    chunks = [(i, min(T, i + PIPELINE_CHUNK)) for i in range(0, T, PIPELINE_CHUNK)]
    L = _lib.load()
    p = _lib.ptr
    ws_bytes = int(L.dt_tree_field_workspace(PIPELINE_CHUNK))
    cos_t, sin_t = contour_tables(dev)
    # two compute streams in turn: chunk i+1's traversal fills the SMs that
    # chunk i's tail leaves idle (own workspaces per stream)
    main = torch.cuda.current_stream(dev)
    comps = [main, torch.cuda.Stream(dev)]
    eval_ws = [torch.empty(ws_bytes, dtype=torch.uint8, device=dev) for _ in comps]
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ready = torch.cuda.Event()
    ready.record(main)
    comps[1].wait_event(ready)  # the tree and flags were made on the main stream
    ev0, ev1 = _timing_events()
    keep = []  # pinned staging buffers stay alive until the copies finish
    for c, (i0, i1) in enumerate(chunks):
        comp, k = comps[c % 2], c % 2
        with torch.cuda.stream(s_in):
            if src is None:  # pageable input: stage through pinned memory
                buf = torch.empty(i1 - i0, dtype=torch.float64, pin_memory=True)
                buf.copy_(host[i0:i1])
                keep.append(buf)
                d_t[i0:i1].copy_(buf, non_blocking=True)
            else:
                d_t[i0:i1].copy_(src[i0:i1], non_blocking=True)
            arrived = torch.cuda.Event()
            arrived.record(s_in)
        comp.wait_event(arrived)
        with torch.cuda.stream(comp):
            # sign term + traversal in one kernel; non-finite targets are
            # counted in flags[0] and not traversed (no O(N) walk per NaN)
            _lib.check(
                L.dt_tree_field_packed(
                    p(tree.packed), len(tree), p(tree.meval), tree.meval.shape[1], p(tree.xq),
                    p(system.xs), p(system.prefix), len(system), kernel.r_d * kernel.r_d,
                    float(config.theta), int(config.p), int(bool(config.adaptive)),
                    _tol_share(tree, config), int(tree.moment_order), p(cos_t), p(sin_t),
                    cos_t.numel(), p(d_t), p(d_o), i0, i1, p(flags), p(eval_ws[k]), ws_bytes,
                    _lib.stream_handle(),
                ),
                "dt_tree_field_packed",
            )
            done = torch.cuda.Event()
            done.record(comp)
        s_out.wait_event(done)
        with torch.cuda.stream(s_out):
            out_h[i0:i1].copy_(d_o[i0:i1], non_blocking=True)
    s_out.synchronize()
    fin = torch.cuda.Event()
    fin.record(comps[1])
    main.wait_event(fin)
    elapsed = _elapsed(ev0, ev1)
    bad, _ = flags.tolist()
    if bad:
        raise ValueError("targets must all be finite")
    values = out_h.numpy() if numpy_out else out_h
    return FieldResult(values=values, build_time=tree.build_seconds, eval_time=elapsed,
                       method="tree")


def _evaluate_host_mapped(tree: Tree, kernel: DiscKernel, config: EvalConfig,
                          system: ChargeSystem, host: torch.Tensor,
                          numpy_out: bool) -> FieldResult:
    """Pinned host targets: one fused kernel (dt_tree_field_packed) reads
    each target over the host link and writes E(y) = e(y) + phi(y) straight
    into a pinned result buffer; no device copies of targets or results."""
    dev = _lib.require_device()
    T = host.numel()
    out_h = torch.empty(T, dtype=torch.float64, pin_memory=True)
    flags = _lib.zeros_i64(2, dev)
    ws = _workspace(dev, int(_lib.load().dt_tree_field_workspace(T)))
    cos_t, sin_t = contour_tables(dev)
    p = _lib.ptr
    ev0, ev1 = _timing_events()
    _lib.check(
        _lib.load().dt_tree_field_packed(
            p(tree.packed), len(tree), p(tree.meval), tree.meval.shape[1], p(tree.xq),
            p(system.xs), p(system.prefix), len(system), kernel.r_d * kernel.r_d,
            float(config.theta), int(config.p), int(bool(config.adaptive)),
            _tol_share(tree, config), int(tree.moment_order), p(cos_t), p(sin_t), cos_t.numel(),
            host.data_ptr(), out_h.data_ptr(), 0, T, p(flags), p(ws), ws.numel(),
            _lib.stream_handle(),
        ),
        "dt_tree_field_packed",
    )
    elapsed = _elapsed(ev0, ev1)  # synchronises
    bad, _ = flags.tolist()
    if bad:
        raise ValueError("targets must all be finite")
    values = out_h.numpy() if numpy_out else out_h
    return FieldResult(values=values, build_time=tree.build_seconds, eval_time=elapsed,
                       method="tree")


def evaluate_with_bound(tree: Tree, kernel: DiscKernel, config: EvalConfig,
                        system: ChargeSystem, targets: torch.Tensor):
    """Field and a-posteriori truncation bound per target on the device
    (SURVEY.md §8(f) "next" #4): E(y) as evaluate_all, plus
    B(y) = sum over accepted far nodes of bound_value(M, R, h, p_use) *
    sum_node |q| (kernel.py:130-182) with the exact contour supremum M, so
    |E_tree(y) - E_direct(y)| <= B(y) up to round-off can be checked at any
    size without a CPU replay (test_tree.py:216-250 does it node by node).
    Returns (values, bounds) as device tensors."""
    from .charges import prefix_sum

    t, _ = as_targets(targets)
    _check_order(tree, config)
    values = _sign_terms(system, t)
    bounds = torch.zeros_like(t)
    if t.numel():
        abs_pre = prefix_sum(system.qs.abs())
        st = _lib.EvalStats(None, None, None, None, None, None, bounds.data_ptr(),
                            abs_pre.data_ptr())
        tree_phi_sum(tree, kernel, config, t, values, stats=st)
        torch.cuda.synchronize(t.device)
    return values, bounds
