"""Per-level timestamps of m2m_threads_kernel (variant DT_M2M_TRACE; dev aid)."""
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
m = torch.zeros((bufs.capacity, order + 1), dtype=torch.float64, device="cuda")
me = torch.zeros((bufs.capacity, eval_stride(order)), dtype=torch.float64, device="cuda")
bufs.launch(xs, 64)
for _ in range(3):
    launch_moments(bufs, xs, qs, order, m, me)
torch.cuda.synchronize()
# the arrived[] workspace holds one u64 timestamp per level
ts = bufs.mws.view(torch.int64)[bufs.capacity // 2: bufs.capacity // 2 + 40].cpu().numpy()
depth = int(bufs.meta[1])
t = ts[:depth][::-1]
print("level start offsets (us):", np.round((t - t[0]) / 1e3, 1).tolist())
print("per-level us:", np.round(np.diff(t) / 1e3, 1).tolist())
ph = bufs.mws.view(torch.int64)[bufs.capacity // 2 + 64: bufs.capacity // 2 + 64 + 512].cpu().numpy().reshape(64, 8)
lo = bufs.meta[8:8 + depth + 1].cpu().numpy()
for lev in range(depth - 1, -1, -1):
    r = ph[int(lo[lev]) & 63]
    if r[0] and r[3] > r[0]:
        print("level", lev, "load %.2f us, shift %.2f us, store %.2f us" %
              ((r[1] - r[0]) / 1e3, (r[2] - r[1]) / 1e3, (r[3] - r[2]) / 1e3))
