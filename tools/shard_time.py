"""Per-rank cost of the sharded upward pass at configs[2] (one GPU standing
in for rank r of G; the all-gather is replaced by a local copy).  Dev aid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import workloads as W
from paper_1710_05781_b200.parallel import ShardedMoments, shard_bounds
from paper_1710_05781_b200.tree import (TreeBuffers, eval_stride, initial_node_capacity,
                                        launch_moments, moment_order_for)

w = W.cfg2()
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
xs, qs, ys = (torch.from_numpy(a).cuda() for a in (w.xs, w.qs, w.targets))
bufs = TreeBuffers(len(xs), initial_node_capacity(len(xs), 64), xs.device)
bufs.launch(xs, 64)
order = moment_order_for(cfg)
es = eval_stride(order)
me = torch.empty((bufs.capacity, es), dtype=torch.float64, device="cuda")


def timeit(fn, reps=5):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts[1:])


print("full moments ms %.3f" % timeit(lambda: launch_moments(bufs, xs, qs, order, None, me)))
for G in (2, 4, 8):
    for r in (0, G // 2, G - 1):
        i0, i1 = shard_bounds(len(ys), G, r)
        sh = ShardedMoments(bufs, order, None, me, es, cfg.theta, G, r)
        yr = ys[i0:i1]

        def go():
            sh.local(xs, qs, yr)
            sh.recv[: sh.send.numel()].copy_(sh.send)
            sh.finish()

        t = timeit(go)
        p = sh.plan_host()
        print(f"G={G} rank={r}: {t:.3f} ms  src {p['src'][1]-p['src'][0]} of {len(xs)}  cut {p['cut']}")
