"""Device-resident evaluation step with no host round trips.

One ``step`` is the whole hot path on inputs already in HBM:
    (a) prefix scan of q and the sign term e(y)      dt_prefix_scan, dt_sign_terms
    (b) tree build                                   dt_build_tree (cooperative)
    (c) P2M / M2M moments, and the (x, q) pairs       dt_moments_pack (prep + fused dataflow)
        for the traversal (sharded: dt_pack_sources)
    (d)+(e) traversal, far + near field, += e(y)     dt_tree_eval_device
All launches are stream-ordered and read sizes (node count, depth, level
ranges, tol_share) from device memory, so the step can be timed back to back
or captured in a CUDA graph.  Buffers are sized once (node capacity from a
planning build); a step whose tree overflows the capacity is detected by
``check()``.  Used by bench.py and by the multi-GPU driver (contiguous target
slices [i0, i1) per rank, sources replicated, world > 1: sharded upward
pass with one all-gather of the cut-level moment rows).
"""

from __future__ import annotations

import os

import torch

from . import _lib
from .kernel import DiscKernel
from .tree import (
    EvalConfig,
    TreeBuffers,
    contour_tables,
    eval_stride,
    initial_node_capacity,
    launch_moments,
    moment_order_for,
    pack_sources,
)

# kernels launched per step (memset of the work counter not counted):
# scan(2) sign(2) build(3: dyadic samples, dyadic searches, the cooperative
# build) moments(2) eval, plus the two order-table kernels
# ahead of an adaptive evaluation with moment order <= 31, theta <= 1/2 (the
# sharded pass adds its own launches and the separate pack)
LAUNCHES_PER_STEP = 2 + 2 + 3 + 2 + 1
ORDER_TABLE_LAUNCHES = 2


class TreePipeline:
    def __init__(self, n: int, n_targets: int, kernel: DiscKernel, config: EvalConfig,
                 node_capacity: int | None = None, device=None, world: int = 1, rank: int = 0,
                 group=None, cut_level: int | None = None, fused_sign: bool | None = None):
        self.dev = device or _lib.require_device()
        self.n, self.T = int(n), int(n_targets)
        self.kernel, self.config = kernel, config
        self.order = moment_order_for(config)
        cap = node_capacity or initial_node_capacity(n, config.leaf_capacity)
        self.bufs = TreeBuffers(self.n, cap, self.dev)
        # the traversal rows are the only layout the step forms (order <= 31);
        # higher orders also need the reference layout as the pass's input
        self.moments = (torch.empty((cap, self.order + 1), dtype=torch.float64, device=self.dev)
                        if self.order + 1 > 32 else None)
        self.estride = eval_stride(self.order)
        self.meval = torch.empty((cap, self.estride), dtype=torch.float64, device=self.dev)
        self.prefix = torch.empty(self.n, dtype=torch.float64, device=self.dev)
        L = _lib.load()
        self.scan_ws_bytes = int(L.dt_prefix_scan_workspace(self.n))
        self.scan_ws = torch.empty(self.scan_ws_bytes, dtype=torch.uint8, device=self.dev)
        self.xq = torch.empty(2 * self.n, dtype=torch.float64, device=self.dev)
        # the sign term as its own kernel on the side stream (dt_sign_terms,
        # default: hidden beside the upward pass) or inside the traversal
        # kernel (dt_tree_field_device: +0.22 ms of traversal at configs[2],
        # step 12.61 against 12.52 ms)
        if fused_sign is None:
            fused_sign = os.environ.get("DT_PIPE_FUSED_SIGN", "0") == "1"
        self.fused_sign = bool(fused_sign)
        ws_bytes = (int(L.dt_tree_field_workspace(self.T)) if self.fused_sign
                    else _lib.DT_EVAL_COUNTER_BYTES)
        self.eval_ws = torch.empty(ws_bytes, dtype=torch.uint8, device=self.dev)
        self.sign_ws_bytes = int(L.dt_sign_terms_workspace(self.T))
        self.sign_ws = torch.empty(self.sign_ws_bytes, dtype=torch.uint8, device=self.dev)
        self.cos_t, self.sin_t = contour_tables(self.dev)
        self.side = torch.cuda.Stream(self.dev)
        # a third stream builds the traversal's order tables beside the upward
        # pass (dt_eval_prepare) instead of in front of the traversal
        self.tabs = torch.cuda.Stream(self.dev)
        self.ev_scan, self.ev_side = torch.cuda.Event(), torch.cuda.Event()
        self.ev_tabs = torch.cuda.Event()
        # world > 1: sharded upward pass (one all-gather of cut-level rows)
        self.shard = None
        if world > 1 and self.order + 1 <= 32:  # higher orders: replicated moments
            from .parallel import ShardedMoments

            self.shard = ShardedMoments(self.bufs, self.order, self.moments, self.meval,
                                        self.estride, config.theta, world, rank, group,
                                        cut_level)
        tables = bool(config.adaptive) and self.order <= 31 and config.theta <= 0.5
        # fused sign: the bracket kernel instead of the two sign-term kernels;
        # sharded: its launches replace the two moments kernels, plus the pack
        self.launches_per_step = LAUNCHES_PER_STEP + (-1 if self.fused_sign else 0) + (
            self.shard.LAUNCHES - 2 + 1 if self.shard else 0) + (
            ORDER_TABLE_LAUNCHES if tables else 0)

    @classmethod
    def planned(cls, xs: torch.Tensor, n_targets: int, kernel: DiscKernel,
                config: EvalConfig, slack: float = 1.25, **kw) -> "TreePipeline":
        """Size the node capacity from one synchronous build of these sources."""
        n = xs.numel()
        cap = initial_node_capacity(n, config.leaf_capacity)
        while True:
            probe = TreeBuffers(n, cap, _lib.require_device())
            probe.launch(xs, config.leaf_capacity)
            meta = probe.meta[:8].cpu().tolist()
            if not meta[_lib.DT_META_OVERFLOW]:
                break
            cap *= 4
        need = int(meta[_lib.DT_META_NODES] * slack) + 64
        del probe
        return cls(n, n_targets, kernel, config, node_capacity=need, **kw)

    def step(self, xs: torch.Tensor, qs: torch.Tensor, ys: torch.Tensor, out: torch.Tensor,
             i0: int = 0, i1: int | None = None, eval_events=None) -> None:
        """out[i0:i1] = E(ys[i0:i1]) for sorted sources (xs, qs); async.

        ``eval_events`` = (start, end) CUDA events recorded on the launching
        stream around the traversal kernel (roofline timing)."""
        if i1 is None:
            i1 = ys.numel()
        L = _lib.load()
        p = _lib.ptr
        main = torch.cuda.current_stream(self.dev)
        s = _lib.stream_handle()
        cfg = self.config
        ys_part = ys[i0:i1]
        out_part = out[i0:i1]
        # side stream: the prefix scan, the (x, q) interleave and the sign
        # term overlap the latency-bound upward pass (none of them feeds the
        # tree).  They start after the build: the build is a cooperative
        # launch, which waits for co-residency with anything already running.
        if self.shard is None and self.order + 1 <= 32:
            # the build's idle blocks start the P2M of the finished levels
            self.bufs.launch(xs, cfg.leaf_capacity, p2m=(qs, self.order, self.meval, self.xq))
        else:
            self.bufs.launch(xs, cfg.leaf_capacity)
        self.ev_scan.record(main)
        eval_args = None
        if not self.fused_sign:
            eval_args = (p(self.bufs.packed), p(self.bufs.meta), self.bufs.capacity,
                         p(self.meval), self.estride, p(self.xq), self.n,
                         self.kernel.r_d * self.kernel.r_d, float(cfg.theta), int(cfg.p),
                         int(bool(cfg.adaptive)), float(cfg.tolerance), self.order,
                         p(self.cos_t), p(self.sin_t), self.cos_t.numel(), p(ys), p(out),
                         int(i0), int(i1), 1, p(self.eval_ws), self.eval_ws.numel())
            # the tables need only the tree's node records and depth
            self.tabs.wait_event(self.ev_scan)
            with torch.cuda.stream(self.tabs):
                _lib.check(L.dt_eval_prepare(*eval_args, _lib.stream_handle()), "dt_eval_prepare")
                # the sign term's tile brackets need no prefix either
                _lib.check(L.dt_sign_bracket(p(xs), self.n, p(ys_part), i1 - i0,
                                             p(self.sign_ws), self.sign_ws_bytes,
                                             _lib.stream_handle()), "dt_sign_bracket")
                self.ev_tabs.record(self.tabs)
        self.side.wait_event(self.ev_scan)
        with torch.cuda.stream(self.side):
            _lib.check(L.dt_prefix_scan(p(qs), p(self.prefix), self.n, p(self.scan_ws),
                                        self.scan_ws_bytes, _lib.stream_handle()),
                       "dt_prefix_scan")
            if self.shard is not None:  # the full upward pass writes xq itself
                pack_sources(xs, qs, self.xq)
            if not self.fused_sign:
                self.side.wait_event(self.ev_tabs)  # the brackets (third stream)
                _lib.check(L.dt_sign_terms_bracketed(p(xs), p(self.prefix), self.n, p(ys_part),
                                                     p(out_part), i1 - i0, p(self.sign_ws),
                                                     self.sign_ws_bytes, _lib.stream_handle()),
                           "dt_sign_terms_bracketed")
            self.ev_side.record(self.side)
        if self.shard is None:  # moments + the traversal's (x, q) pairs (dt_moments_pack)
            launch_moments(self.bufs, xs, qs, self.order, self.moments, self.meval, xq=self.xq)
        else:  # this rank's subtrees + all-gather of the cut-level rows
            self.shard.launch(xs, qs, ys_part, targets_sorted=True)
        main.wait_event(self.ev_side)
        if eval_events is not None:
            eval_events[0].record()
        if self.fused_sign:
            _lib.check(
                L.dt_tree_field_device(
                    p(self.bufs.packed), p(self.bufs.meta), self.bufs.capacity, p(self.meval),
                    self.estride, p(self.xq), p(xs), p(self.prefix), self.n,
                    self.kernel.r_d * self.kernel.r_d, float(cfg.theta), int(cfg.p),
                    int(bool(cfg.adaptive)), float(cfg.tolerance), self.order, p(self.cos_t),
                    p(self.sin_t), self.cos_t.numel(), p(ys), p(out), int(i0), int(i1),
                    p(self.eval_ws), self.eval_ws.numel(), s,
                ),
                "dt_tree_field_device",
            )
        else:
            main.wait_event(self.ev_tabs)
            _lib.check(L.dt_tree_eval_device_prepared(*eval_args, s),
                       "dt_tree_eval_device_prepared")
        if eval_events is not None:
            eval_events[1].record()

    def check(self) -> dict:
        """Synchronise and report the last step's tree (raises on overflow)."""
        meta = self.bufs.meta[:8].cpu().tolist()
        if meta[_lib.DT_META_OVERFLOW]:
            raise RuntimeError("tree exceeded the pipeline's node capacity")
        return {"nodes": int(meta[_lib.DT_META_NODES]), "depth": int(meta[_lib.DT_META_DEPTH]),
                "leaves": int(meta[_lib.DT_META_LEAVES])}
