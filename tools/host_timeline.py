"""Host-side timeline of the public API calls (dev aid): when each C-ABI
call is issued, relative to the API call's entry, with the GPU idle before
each call; shows the host work that sits in front of the GPU."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import workloads as W, tree as TR, _lib
w = W.cfg2()
k = dt.DiscKernel(w.r_d)
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
pairs = torch.from_numpy(np.column_stack([w.xs, w.qs])).pin_memory()
tgt = torch.from_numpy(w.targets.copy()).pin_memory()
for _ in range(3):
    s = dt.from_particles(pairs); tr = dt.build(s, k, cfg); v = dt.evaluate_all(tr, k, cfg, s, tgt).values
orig_check = _lib.check
marks = []
def check(rc, name):
    marks.append((time.perf_counter(), name)); return orig_check(rc, name)
_lib.check = check
orig_empty = torch.empty
for rep in range(3):
    s = dt.from_particles(pairs); torch.cuda.synchronize()
    marks.clear(); t0 = time.perf_counter()
    tr = dt.build(s, k, cfg); t1 = time.perf_counter()
    print("build host %.3f ms:" % (1e3*(t1-t0)), " ".join("%s@%.3f" % (n, 1e3*(t-t0)) for t, n in marks))
    torch.cuda.synchronize()
    marks.clear(); t0 = time.perf_counter()
    v = dt.evaluate_all(tr, k, cfg, s, tgt).values; t1 = time.perf_counter()
    print("evaluate host %.3f ms:" % (1e3*(t1-t0)), " ".join("%s@%.3f" % (n, 1e3*(t-t0)) for t, n in marks))
    marks.clear(); torch.cuda.synchronize(); t0 = time.perf_counter()
    s2 = dt.from_particles(pairs); t1 = time.perf_counter()
    print("from_particles host %.3f ms:" % (1e3*(t1-t0)), " ".join("%s@%.3f" % (n, 1e3*(t-t0)) for t, n in marks))
