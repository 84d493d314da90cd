"""Traversal cost breakdown on cfg2: adaptive vs fixed orders (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import workloads as W, _lib
from paper_1710_05781_b200.tree import tree_phi_sum
cells = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 22)
w = W.cfg2(cells=cells)
k = dt.DiscKernel(w.r_d)
cfgA = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
system = dt.from_sorted(w.xs, w.qs)
tree = dt.build(system, k, cfgA)
ys = torch.from_numpy(w.targets).cuda()
out = torch.empty_like(ys)
def t(cfg, mode=0, reps=3):
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); tree_phi_sum(tree, k, cfg, ys, out, accumulate=False, psel_mode=mode); b.record()
        torch.cuda.synchronize(); best = min(best, a.elapsed_time(b))
    return best
print("adaptive fast", t(cfgA))
for p in (0, 1, 2, 4, 8, 12, 18, 24, 30):
    print("fixed p", p, t(dt.EvalConfig(p=p, leaf_capacity=64)))
print("adaptive exact-only", t(cfgA, mode=1, reps=1))
