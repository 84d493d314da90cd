"""configs[4] direct sums: plain vs pair-symmetric kernel (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1710_05781_b200 import workloads as W
from paper_1710_05781_b200.direct import phi_sum_direct, phi_sum_symmetric
w = W.cfg4()
x, q = torch.from_numpy(w.xs).cuda(), torch.from_numpy(w.qs).cuda()
rd2 = w.r_d ** 2
for name, fn in (("plain", lambda o: phi_sum_direct(x, q, x, rd2, o, accumulate=False)),
                 ("symmetric", lambda o: phi_sum_symmetric(x, q, rd2, o, accumulate=False))):
    o = torch.zeros_like(x)
    fn(o)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); fn(o); b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"{name}: {ms:.1f} ms, {len(w.xs) ** 2 / ms * 1e3:.3e} interactions/s, checksum {float(o.abs().sum()):.12e}")
