"""Own race / stale-read probe (compute-sanitizer is closed on this GPU pool).

For the kernels with inter-block protocols, run them many times on buffers
poisoned with NaN before every run and require every run to be finite and
bit-identical to the first:
  - the upward pass (arrival counters with acquire/release, frontier climb):
    a row read before its writer published it is NaN and poisons the root;
  - the cooperative build (grid barriers, block-0 level runs, flag wait);
  - the two-pass prefix scan (group arrival counters);
  - the traversal (per-SM task segments, work stealing);
  - the sharded upward pass for 2 and 8 ranks (plan, partial, pack, finish).
Usage: python tools/race_probe.py [cells] [reps]   (configs[2] mesh)."""
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
                                        launch_moments, moment_order_for, tree_phi_sum)

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
w = W.cfg2(cells=cells)
k = dt.DiscKernel(w.r_d)
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
xs, qs, ys = (torch.from_numpy(a).cuda() for a in (w.xs, w.qs, w.targets))
order = moment_order_for(cfg)
es = eval_stride(order)
bufs = TreeBuffers(len(xs), initial_node_capacity(len(xs), cfg.leaf_capacity), xs.device)
report = {"cells": cells, "n": len(xs), "reps": reps}
NODE = ("lo", "hi", "center", "half", "level", "start", "end", "left", "right")

# build
ref = None
for i in range(reps):
    for f in NODE:
        getattr(bufs, f).fill_(-7)
    bufs.launch(xs, cfg.leaf_capacity)
    n_nodes = int(bufs.meta[_lib.DT_META_NODES])
    cur = torch.cat([getattr(bufs, f)[:n_nodes].double() for f in NODE])
    if ref is None:
        ref = cur
    assert torch.equal(cur, ref), f"build differs at rep {i}"
report["build"] = {"nodes": n_nodes, "depth": int(bufs.meta[_lib.DT_META_DEPTH]),
                   "identical_runs": reps}

# upward pass
me = torch.empty((bufs.capacity, es), dtype=torch.float64, device="cuda")
ref = None
for i in range(reps):
    me.fill_(float("nan"))
    launch_moments(bufs, xs, qs, order, None, me)
    cur = me[:n_nodes].clone()
    assert bool(torch.isfinite(cur).all()), f"upward pass read an unpublished row (rep {i})"
    if ref is None:
        ref = cur
    assert torch.equal(cur, ref), f"upward pass differs at rep {i}"
report["upward"] = {"identical_finite_runs": reps}

# the build's idle-block P2M followed by the rest of the upward pass
xq = torch.empty(2 * len(xs), dtype=torch.float64, device="cuda")
for i in range(reps):
    me.fill_(float("nan"))
    xq.fill_(float("nan"))
    bufs.launch(xs, cfg.leaf_capacity, p2m=(qs, order, me, xq))
    launch_moments(bufs, xs, qs, order, None, me, xq=xq)
    cur = me[:n_nodes].clone()
    assert bool(torch.isfinite(cur).all()), f"build + upward read an unpublished row (rep {i})"
    assert torch.equal(cur, ref), f"build-time P2M rows differ at rep {i}"
    assert bool(torch.isfinite(xq).all())
report["build_p2m"] = {"identical_finite_runs": reps,
                       "preformed_nodes": int(bufs.meta[_lib.DT_META_P2M_UPTO])}

# prefix scan
ref = None
for i in range(reps):
    p = prefix_sum(qs)
    if ref is None:
        ref = p
    assert torch.equal(p, ref), f"scan differs at rep {i}"
report["scan"] = {"identical_runs": reps}

# traversal
system = dt.from_sorted(w.xs, w.qs)
tree = dt.build(system, k, cfg)
ref = None
for i in range(max(5, reps // 5)):
    out = torch.full_like(ys, float("nan"))
    tree_phi_sum(tree, k, cfg, ys, out, accumulate=False)
    assert bool(torch.isfinite(out).all())
    if ref is None:
        ref = out
    assert torch.equal(out, ref), f"traversal differs at rep {i}"
report["traversal"] = {"identical_runs": max(5, reps // 5)}

# sharded upward pass
full = ref_rows = me[:n_nodes].clone()
for G in (2, 8):
    for i in range(max(3, reps // 10)):
        sends, shards = [], []
        for r in range(G):
            i0, i1 = shard_bounds(ys.numel(), G, r)
            mr = torch.full((bufs.capacity, es), float("nan"), dtype=torch.float64, device="cuda")
            sh = ShardedMoments(bufs, order, None, mr, es, cfg.theta, G, r)
            sends.append(sh.local(xs, qs, ys[i0:i1].contiguous(), True).clone())
            shards.append((sh, mr))
        recv = torch.cat(sends)
        for sh, mr in shards:
            sh.finish(recv)
            rows = mr[:n_nodes]
            held = torch.isfinite(rows).all(dim=1)
            assert torch.equal(rows[held], full[held]), f"G={G}: a held row differs"
    report[f"sharded_G{G}"] = {"runs": max(3, reps // 10)}
torch.cuda.synchronize()
print(json.dumps(report))
