"""Time the traversal kernel alone on cfg2 (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import workloads as W, _lib
from paper_1710_05781_b200.pipeline import TreePipeline
cells = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 22)
w = W.cfg2(cells=cells)
k = dt.DiscKernel(w.r_d)
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
xs, qs, ys = (torch.from_numpy(a).cuda() for a in (w.xs, w.qs, w.targets))
out = torch.empty_like(ys)
pipe = TreePipeline.planned(xs, len(ys), k, cfg)
ts = []
for i in range(6):
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    pipe.step(xs, qs, ys, out, eval_events=ev)
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
print(os.environ.get("DISCTREE_B200_LIB", "default"), "eval ms", ["%.3f" % t for t in ts], "checksum", float(out.double().abs().sum()))
