"""Lane-utilisation counters of the traversal kernel (variant build
DT_EVAL_UTIL=1; development aid).  Usage:
  DISCTREE_B200_LIB=paper_1710_05781_b200/variants/lib_util.so python tools/eval_util.py [cells]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import _lib
from paper_1710_05781_b200 import workloads as W
from paper_1710_05781_b200.pipeline import TreePipeline

cells = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 22)
w = W.cfg2(cells=cells)
k = dt.DiscKernel(w.r_d)
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
xs, qs, ys = (torch.from_numpy(a).cuda() for a in (w.xs, w.qs, w.targets))
out = torch.empty_like(ys)
pipe = TreePipeline.planned(xs, len(ys), k, cfg)
L = _lib.load()
buf = (C.c_ulonglong * 16)()
pipe.step(xs, qs, ys, out)
L.dt_eval_util(buf, 1)
pipe.step(xs, qs, ys, out)
L.dt_eval_util(buf, 1)
u = list(buf)
names = ["node_visits", "far_visits", "far_lanes", "sum_pmax", "sum_pu", "sum_pmin",
         "near_visits", "near_lanes", "near_warp_pairs", "tasks"]
for n, v in zip(names, u):
    print(f"{n:16s} {v:.6e}")
T = len(ys)
print("per task: node visits %.1f, far visits %.1f, near visits %.1f" %
      (u[0] / u[9], u[1] / u[9], u[6] / u[9]))
print("far lane util (lanes/32 per far visit): %.3f" % (u[2] / (32 * u[1])))
print("far order util (sum pu+1 / 32*(pmax+1)): %.3f" % ((u[4] + u[2]) / (32 * (u[3] + u[1]))))
print("mean pmax %.2f, mean pmin %.2f, mean pu %.2f" % (u[3] / u[1], u[5] / u[1], u[4] / u[2]))
print("near lane util: %.3f" % (u[7] / (32 * u[6])))
print("far events/target %.2f near pairs/target (executed lanes) %.1f" % (u[2] / T, u[8] * 32 / T))
print("table calls (lane 0) %d, table misses (lane 0) %d" % (u[10], u[11]))
print("two-child opens %.1f per task: all lanes accept the first child %.1f, accept both %.1f; "
      "lanes accepting the first child %.1f per open" % (u[12] / u[9], u[13] / u[9], u[14] / u[9],
                                                        u[15] / max(u[12], 1)))
