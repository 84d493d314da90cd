"""Per-level completion times of the upward pass inside one pipeline step
(variant: make variant-mom NAME=uptrace DEFS=-DDT_UP_TRACE=1; dev aid)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import _lib
from paper_1710_05781_b200 import workloads as W
from paper_1710_05781_b200.pipeline import TreePipeline

w = W.cfg2()
k = dt.DiscKernel(w.r_d)
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
xs, qs, ys = (torch.from_numpy(a).cuda() for a in (w.xs, w.qs, w.targets))
out = torch.empty_like(ys)
pipe = TreePipeline.planned(xs, len(ys), k, cfg)
L = _lib.load()
buf = (C.c_ulonglong * 72)()
for rep in range(3):
    L.dt_debug_uptrace(buf, 1)
    pipe.step(xs, qs, ys, out)
    torch.cuda.synchronize()
L.dt_debug_uptrace(buf, 0)
t0 = buf[0]
meta = pipe.bufs.meta.cpu().tolist()
depth = meta[1]
print("upto (P2M by the build):", meta[_lib.DT_META_P2M_UPTO], "of", meta[0], "nodes")
for lev in range(depth, -1, -1):
    t = buf[1 + lev]
    print(f"level {lev:2d} ({meta[8 + lev + 1] - meta[8 + lev]:6d} nodes): last formed at "
          f"{(t - t0) / 1e3:7.1f} us" if t else f"level {lev}: none")
