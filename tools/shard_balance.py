"""Eval time of each rank's target slice at G ranks (one GPU, slices run one
after the other; dev aid for multi-GPU load balance)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import workloads as W
from paper_1710_05781_b200.parallel import shard_bounds
from paper_1710_05781_b200.tree import tree_phi_sum

w = W.cfg2()
k = dt.DiscKernel(w.r_d)
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
system = dt.from_sorted(w.xs, w.qs)
tree = dt.build(system, k, cfg)
ys = torch.from_numpy(w.targets).cuda()
out = torch.zeros_like(ys)
for G in (2, 4, 8):
    ts = []
    for r in range(G):
        i0, i1 = shard_bounds(len(ys), G, r)
        best = 1e9
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            tree_phi_sum(tree, k, cfg, ys, out, i0=i0, i1=i1, accumulate=False)
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        ts.append(best)
    print(f"G={G}: per-rank eval ms {['%.3f' % t for t in ts]}  max/mean {max(ts) / (sum(ts) / G):.3f}")
