"""Predict the G-GPU step of bench.py from per-rank components measured on
one GPU (configs[2]).  The traversal of a slice is timed without its
order-table build, which the pipeline runs on a third stream.  Per rank the step is
    scan + build + max(sharded upward pass + all-gather, pack + sign term of
    the slice) + traversal of the slice
(pipeline.TreePipeline.step: the pack and the sign term run on a side stream
beside the upward pass).  Each component is timed with CUDA events
(best of 5); the sharded pass and the traversal take the slowest rank.  The
all-gather of the cut-level rows (2^cut rows x 32 doubles per rank, ~2-8 KB)
cannot run on one GPU: it is charged ALLGATHER_US, an assumed small-message
NCCL latency over NVLink.  Prints one JSON object (profiles/r2_predict_scaling.json)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import _lib
from paper_1710_05781_b200 import workloads as W
from paper_1710_05781_b200.charges import prefix_sum
from paper_1710_05781_b200.parallel import ShardedMoments, shard_bounds
from paper_1710_05781_b200.tree import (TreeBuffers, eval_stride, initial_node_capacity,
                                        launch_moments, moment_order_for, pack_sources,
                                        tree_phi_sum)

ALLGATHER_US = 20.0
w = W.cfg2()
k = dt.DiscKernel(w.r_d)
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
xs, qs, ys = (torch.from_numpy(a).cuda() for a in (w.xs, w.qs, w.targets))
T = ys.numel()
bufs = TreeBuffers(len(xs), initial_node_capacity(len(xs), 64), xs.device)
bufs.launch(xs, 64)
order = moment_order_for(cfg)
es = eval_stride(order)
me = torch.empty((bufs.capacity, es), dtype=torch.float64, device="cuda")
L = _lib.load()
p = _lib.ptr
prefix = prefix_sum(qs)
xq = torch.empty(2 * len(xs), dtype=torch.float64, device="cuda")
system = dt.from_sorted(w.xs, w.qs)
tree = dt.build(system, k, cfg)
out = torch.empty_like(ys)
sign_ws = torch.empty(int(L.dt_sign_terms_workspace(T)), dtype=torch.uint8, device="cuda")


def timeit(fn, reps=5):
    ts = []
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts[1:])


from paper_1710_05781_b200.tree import contour_tables

cos_t, sin_t = contour_tables(ys.device)
eval_ws = torch.empty(_lib.DT_EVAL_COUNTER_BYTES, dtype=torch.uint8, device="cuda")


def traverse(i0, i1):
    """The pipeline's traversal of one slice: the order tables are built on
    a third stream beside the upward pass (dt_eval_prepare), so only the
    traversal kernel (dt_tree_eval_device_prepared) is on the step's path."""
    args = (p(tree.packed), p(tree.meta), tree.packed.numel() // 32, p(tree.meval),
            tree.meval.shape[1], p(tree.xq), len(xs), w.r_d * w.r_d, float(cfg.theta),
            int(cfg.p), 1, float(cfg.tolerance), tree.moment_order, p(cos_t), p(sin_t),
            cos_t.numel(), p(ys), p(out), i0, i1, 0, p(eval_ws), eval_ws.numel(),
            _lib.stream_handle())
    ts = []
    for _ in range(6):  # the prepare call also zeroes the slot's task counters
        _lib.check(L.dt_eval_prepare(*args), "dt_eval_prepare")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.check(L.dt_tree_eval_device_prepared(*args), "dt_tree_eval_device_prepared")
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts[1:])


res = {"workload": "configs[2] (2^24 sources = targets)", "allgather_us_assumed": ALLGATHER_US}
res["scan_ms"] = timeit(lambda: prefix_sum(qs))
res["build_ms"] = timeit(lambda: bufs.launch(xs, 64))
res["moments_full_ms"] = timeit(lambda: launch_moments(bufs, xs, qs, order, None, me))
res["eval_full_ms"] = traverse(0, T)
per_g = {}
for G in (1, 2, 4, 8):
    mom, ev, side = 0.0, 0.0, 0.0
    for r in range(G):
        i0, i1 = shard_bounds(T, G, r)
        yr = ys[i0:i1]
        if G > 1:
            sh = ShardedMoments(bufs, order, None, me, es, cfg.theta, G, r)

            def go():
                sh.local(xs, qs, yr)
                sh.recv[: sh.send.numel()].copy_(sh.send)
                sh.finish()

            mom = max(mom, timeit(go) + ALLGATHER_US * 1e-3)
        else:
            mom = res["moments_full_ms"]
        ev = max(ev, traverse(i0, i1))

        def sidework():
            pack_sources(xs, qs, xq)
            L.dt_sign_terms(p(xs), p(prefix), len(xs), p(ys[i0:i1]), p(out[i0:i1]), i1 - i0,
                            p(sign_ws), sign_ws.numel(), _lib.stream_handle())

        side = max(side, timeit(sidework))
    step = res["scan_ms"] + res["build_ms"] + max(mom, side) + ev
    per_g[G] = {"sharded_upward_ms": mom, "side_stream_ms": side, "eval_slice_ms": ev,
                "predicted_step_ms": step, "predicted_targets_per_s": T / (step * 1e-3)}
base = per_g[1]["predicted_step_ms"]
for G, v in per_g.items():
    v["predicted_efficiency"] = base / (G * v["predicted_step_ms"])
res["per_world"] = per_g
print(json.dumps(res, indent=1))
