"""Timeline of the public-API end-to-end path (dev aid): kernels and copies
with start offsets, from a torch profiler trace."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import workloads as W

w = W.cfg2()
k = dt.DiscKernel(w.r_d)
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
pairs = torch.from_numpy(np.column_stack([w.xs, w.qs])).pin_memory()
tgt = torch.from_numpy(w.targets.copy()).pin_memory()
for _ in range(2):
    s = dt.from_particles(pairs)
    tr = dt.build(s, k, cfg)
    v = dt.evaluate_all(tr, k, cfg, s, tgt).values
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    s = dt.from_particles(pairs)
    tr = dt.build(s, k, cfg)
    v = dt.evaluate_all(tr, k, cfg, s, tgt).values
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/e2e_trace.json")
ev = json.load(open("/tmp/e2e_trace.json"))["traceEvents"]
gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
t0 = min(e["ts"] for e in gpu)
for e in sorted(gpu, key=lambda e: e["ts"]):
    print("%9.3f ms  %8.3f ms  stream %-3s %s" % ((e["ts"] - t0) / 1e3, e["dur"] / 1e3,
          e.get("args", {}).get("stream", "?"), e["name"][:70]))
