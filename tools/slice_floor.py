import os, sys
sys.path.insert(0, '/root/repo')
import torch
import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import workloads as W
from paper_1710_05781_b200.tree import tree_phi_sum
w = W.cfg2()
k = dt.DiscKernel(w.r_d)
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
system = dt.from_sorted(w.xs, w.qs)
tree = dt.build(system, k, cfg)
ys = torch.from_numpy(w.targets).cuda()
out = torch.zeros_like(ys)
T = len(ys)
for n in (32, 4096, 65536, 1 << 20, T // 8, T // 4, T):
    for i0 in (0, T // 2):
        i1 = min(T, i0 + n)
        best = 1e9
        for _ in range(4):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            tree_phi_sum(tree, k, cfg, ys, out, i0=i0, i1=i1, accumulate=False)
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        print(f"n={n:9d} i0={i0:9d}: {best:.3f} ms  per 1/8: {best * T / 8 / (i1 - i0):.3f}")
