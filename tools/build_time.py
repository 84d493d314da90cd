"""Build kernel alone (configs[2], leaf 64), CUDA events, median of 30 (dev aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1710_05781_b200 import workloads as W
from paper_1710_05781_b200.tree import TreeBuffers, initial_node_capacity

w = W.cfg2()
xs = torch.from_numpy(w.xs).cuda()
bufs = TreeBuffers(len(xs), initial_node_capacity(len(xs), 64), xs.device)
ts = []
for i in range(33):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    bufs.launch(xs, 64)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print("%s build ms median %.4f min %.4f" % (os.environ.get("DISCTREE_B200_LIB", "default").split("/")[-1],
                                            float(np.median(ts[3:])), min(ts[3:])))
