import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import workloads as W, _lib, pipeline as PL
w = W.cfg2()
k = dt.DiscKernel(w.r_d)
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
xs, qs, ys = (torch.from_numpy(a).cuda() for a in (w.xs, w.qs, w.targets))
out = torch.empty_like(ys)
pipe = PL.TreePipeline.planned(xs, len(ys), k, cfg)
def run(tag):
    ts=[]
    for i in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        a.record(); pipe.step(xs, qs, ys, out, eval_events=ev); b.record(); torch.cuda.synchronize()
        ts.append((a.elapsed_time(b), a.elapsed_time(ev[0]), ev[0].elapsed_time(ev[1])))
    ts=ts[2:]
    print(tag, "step %.3f pre-eval %.3f eval %.3f" % tuple(sum(t[i] for t in ts)/len(ts) for i in range(3)))
run("normal")
L = _lib.load()
orig_sign = L.dt_sign_terms
class Shim:
    def __getattr__(self, n): return getattr(L, n)
    def dt_sign_terms(self, *a): return 0
PL._lib.load = lambda: Shim()
run("no-sign")
orig_pack = PL.pack_sources
PL.pack_sources = lambda *a, **kw: None
run("no-sign-no-pack")
