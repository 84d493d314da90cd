"""Time the prefix scan (dt_prefix_scan) at 2^24 values, 20 calls back to
back between two events (no host gaps), and check it (determinism, distance
from the sequential cumsum) (dev aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1710_05781_b200 import _lib
from paper_1710_05781_b200 import workloads as W

w = W.cfg2()
q = torch.from_numpy(w.qs).cuda()
n = q.numel()
L = _lib.load()
wsb = int(L.dt_prefix_scan_workspace(n))
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
outs = [torch.empty_like(q) for _ in range(2)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def scan(out):
    _lib.check(L.dt_prefix_scan(_lib.ptr(q), _lib.ptr(out), n, _lib.ptr(ws), wsb,
                                _lib.stream_handle()), "dt_prefix_scan")


for _ in range(3):
    scan(outs[0])
reps = 20
flush.zero_()
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
e[0].record()
for i in range(reps):
    scan(outs[i & 1])
e[1].record()
torch.cuda.synchronize()
ms = e[0].elapsed_time(e[1]) / reps
scan(outs[1])
ref = np.cumsum(w.qs)
err = float(np.max(np.abs(outs[0].cpu().numpy() - ref)) / np.abs(w.qs).sum())
print(os.environ.get("DISCTREE_B200_LIB", "default"),
      "scan ms %.4f (%.0f GB/s of 16N)" % (ms, 16 * n / ms / 1e6),
      "bitwise repeat", bool(torch.equal(outs[0], outs[1])), "max|d|/sum|q| vs cumsum %.2e" % err)
