"""Time the upward pass (dt_moments) alone at configs[2] (dev aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import workloads as W
from paper_1710_05781_b200.tree import (TreeBuffers, eval_stride, initial_node_capacity,
                                        launch_moments, moment_order_for)

w = W.cfg2() if len(sys.argv) < 2 else W.cfg1(cells=int(sys.argv[1]))
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
xs, qs = (torch.from_numpy(a).cuda() for a in (w.xs, w.qs))
bufs = TreeBuffers(len(xs), initial_node_capacity(len(xs), 64), xs.device)
order = moment_order_for(cfg)
me = torch.zeros((bufs.capacity, eval_stride(order)), dtype=torch.float64, device="cuda")
ts, tb = [], []
for _ in range(6):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    bufs.launch(xs, 64)
    e[1].record()
    launch_moments(bufs, xs, qs, order, None, me)
    e[2].record()
    torch.cuda.synchronize()
    tb.append(e[0].elapsed_time(e[1]))
    ts.append(e[1].elapsed_time(e[2]))
n = int(bufs.meta[0])
print(os.environ.get("DISCTREE_B200_LIB", "default"), "build ms %.3f moments ms %s checksum %.12e"
      % (min(tb[1:]), ["%.3f" % t for t in ts], float(me[:n].abs().sum())))
