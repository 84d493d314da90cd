"""Per-level timestamps of build_kernel (variant DT_BUILD_TRACE; dev aid)."""
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
for _ in range(3):
    bufs.launch(xs, 64)
torch.cuda.synchronize()
cap = bufs.capacity
# workspace: scratch_off[cap] i32, scratch_split[cap] i32, block_total[4096] i64
bt = bufs.ws.view(torch.uint8)[cap * 8: cap * 8 + 4096 * 8].view(torch.int64).cpu().numpy()
depth = int(bufs.meta[1])
t = bt[2048: 2048 + depth + 2]
ph = bt[2048 + 70: 2048 + 73]
print("dyadic splits + barrier %.1f us, one-pass top %.1f us" % ((ph[1] - ph[0]) / 1e3, (ph[2] - ph[1]) / 1e3))
dy = bt[2048 + 73: 2048 + 76]
if dy.min() > 0:
    print("  sample copy %.1f us, sample barrier %.1f us, searches %.1f us, final barrier %.1f us" % (
        (dy[0] - ph[0]) / 1e3, (dy[1] - dy[0]) / 1e3, (dy[2] - dy[1]) / 1e3, (ph[1] - dy[2]) / 1e3))
tp = bt[2048 + 76: 2048 + 80]
if tp.min() > 0:
    print("  top: pass 1 %.1f us, barrier %.1f us, bases %.1f us, pass 2 %.1f us, barrier %.1f us" % (
        (tp[0] - ph[1]) / 1e3, (tp[1] - tp[0]) / 1e3, (tp[2] - tp[1]) / 1e3, (tp[3] - tp[2]) / 1e3,
        (ph[2] - tp[3]) / 1e3))
lv = bufs.meta[8: 8 + depth + 2].cpu().numpy()
print("per-level us (level: nodes us):")
for l in range(depth + 1):
    print(l, int(lv[l + 1] - lv[l]), round((t[l + 1] - t[l]) / 1e3, 1) if t[l + 1] > t[l] else None)

fine = bt[2048 + 100: 2048 + 105]
if fine[0] > 0:
    print("level 20 inside (SM cycles): search %d, scan %d, emit %d, tail %d" %
          tuple(int(fine[k + 1] - fine[k]) for k in range(4)))
