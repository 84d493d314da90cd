"""Phase timeline of the cooperative upward pass at configs[2] (dev aid):
build the variant with  make variant-mom NAME=trace DEFS=-DDT_UP_TRACE=1  and
run with DISCTREE_B200_LIB=paper_1710_05781_b200/variants/lib_mom_trace.so."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import workloads as W
from paper_1710_05781_b200.tree import (TreeBuffers, eval_stride, initial_node_capacity,
                                        launch_moments, moment_order_for)

w = W.cfg2()
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
xs, qs = (torch.from_numpy(a).cuda() for a in (w.xs, w.qs))
bufs = TreeBuffers(len(xs), initial_node_capacity(len(xs), 64), xs.device)
order = moment_order_for(cfg)
me = torch.zeros((bufs.capacity, eval_stride(order)), dtype=torch.float64, device="cuda")
bufs.launch(xs, 64)
for _ in range(4):
    launch_moments(bufs, xs, qs, order, None, me)
torch.cuda.synchronize()
meta = bufs.meta.cpu().numpy()
depth = int(meta[1])
raw = bufs.mws.cpu().numpy()
off = 2 * bufs.capacity * 4 + 4 * 8
tr = raw[off: off + 8 * (depth + 3)].view(np.uint64).astype(np.int64)
t0 = tr[0]
print(f"P2M (block 0 done): {(tr[1] - t0) / 1e3:.1f} us")
lv = [int(meta[dt._lib.DT_META_LEVEL0 + l + 1] - meta[dt._lib.DT_META_LEVEL0 + l]) for l in range(depth + 1)]
prev = tr[1]
for lev in range(depth - 1, -1, -1):
    t = tr[2 + lev]
    print(f"level {lev:2d} nodes {lv[lev]:7d}: +{(t - prev) / 1e3:6.1f} us  (at {(t - t0) / 1e3:6.1f})")
    prev = t
