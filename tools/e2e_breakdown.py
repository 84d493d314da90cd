"""Time the public-API end-to-end path stage by stage (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import workloads as W
w = W.cfg2()
k = dt.DiscKernel(w.r_d)
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
pairs = torch.from_numpy(np.column_stack([w.xs, w.qs])).pin_memory()
tgt = torch.from_numpy(w.targets.copy()).pin_memory()
for rep in range(3):
    torch.cuda.synchronize(); t = [time.perf_counter()]
    s = dt.from_particles(pairs); torch.cuda.synchronize(); t.append(time.perf_counter())
    tr = dt.build(s, k, cfg); torch.cuda.synchronize(); t.append(time.perf_counter())
    v = dt.evaluate_all(tr, k, cfg, s, tgt).values; torch.cuda.synchronize(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"rep{rep}: from_particles {d[0]:.1f} ms, build {d[1]:.1f} ms, evaluate_all {d[2]:.1f} ms, total {sum(d):.1f}")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    s = dt.from_particles(pairs); tr = dt.build(s, k, cfg); v = dt.evaluate_all(tr, k, cfg, s, tgt).values
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
