"""Run the cfg2 pipeline twice (for ncu: profile the 2nd traversal launch)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import workloads as W
from paper_1710_05781_b200.pipeline import TreePipeline

cells = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 22)
w = W.cfg2(cells=cells)
k = dt.DiscKernel(w.r_d)
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
xs, qs, ys = (torch.from_numpy(a).cuda() for a in (w.xs, w.qs, w.targets))
out = torch.empty_like(ys)
pipe = TreePipeline.planned(xs, len(ys), k, cfg)
for _ in range(2):
    pipe.step(xs, qs, ys, out)
torch.cuda.synchronize()
print("ok", pipe.check(), float(out[:4].sum()))
