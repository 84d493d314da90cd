"""Kernel timeline of one device-resident pipeline step (configs[2]) from a
torch profiler (CUPTI) trace: start offset, duration and stream of every
kernel and memset (dev aid)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import workloads as W
from paper_1710_05781_b200.pipeline import TreePipeline

w = W.cfg2()
k = dt.DiscKernel(w.r_d)
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
xs, qs, ys = (torch.from_numpy(a).cuda() for a in (w.xs, w.qs, w.targets))
out = torch.empty_like(ys)
pipe = TreePipeline.planned(xs, len(ys), k, cfg)
for _ in range(3):
    pipe.step(xs, qs, ys, out)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    pipe.step(xs, qs, ys, out)
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/step_trace.json")
ev = [e for e in json.load(open("/tmp/step_trace.json"))["traceEvents"]
      if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
for e in ev:
    print(f"{e['ts'] - t0:9.1f} us  +{e['dur']:8.1f} us  stream {e['args'].get('stream', '?'):>3}  "
          f"{e['name'][:70]}")
end = max(e["ts"] + e["dur"] for e in ev)
print(f"step span {end - t0:.1f} us")
