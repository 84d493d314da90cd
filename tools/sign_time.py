"""Time dt_sign_terms at configs[2] (2^24 sorted targets), 10 calls back to
back between two events (dev aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import _lib
from paper_1710_05781_b200 import workloads as W

w = W.cfg2()
system = dt.from_sorted(w.xs, w.qs)
ys = torch.from_numpy(w.targets).cuda()
out = torch.empty_like(ys)
L = _lib.load()
p = _lib.ptr
wsb = int(L.dt_sign_terms_workspace(ys.numel()))
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")


def go():
    _lib.check(L.dt_sign_terms(p(system.xs), p(system.prefix), len(system), p(ys), p(out),
                               ys.numel(), p(ws), wsb, _lib.stream_handle()), "dt_sign_terms")


for _ in range(3):
    go()
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
e[0].record()
for _ in range(10):
    go()
e[1].record()
torch.cuda.synchronize()
print(os.environ.get("DISCTREE_B200_LIB", "default"), "sign ms %.4f" % (e[0].elapsed_time(e[1]) / 10),
      "checksum %.12e" % float(out.abs().sum()))
